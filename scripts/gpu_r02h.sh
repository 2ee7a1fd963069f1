#!/bin/bash
# round 2, call H: correction items fused into the main kernel's tail — correctness (stencil tests),
# A/B against the separate items kernel, bench, ncu of the fused kernel
mkdir -p gpurun_out
timeout 900 python -X faulthandler -m pytest tests/test_gpu_stencil.py tests/test_gpu_fullsize.py tests/test_gpu_parity.py -q > gpurun_out/pytest_h.log 2>&1
echo "pytest exit $?: $(tail -1 gpurun_out/pytest_h.log)"; grep -E "^FAILED|^E " gpurun_out/pytest_h.log | head -10
for v in fused split minb4 minb4split; do
  for rep in 1 2; do
    sp=; lib=
    case $v in split) sp=1;; minb4) lib=paper_2604_22087_b200/variants/libafem_minb4.so;; minb4split) sp=1; lib=paper_2604_22087_b200/variants/libafem_minb4.so;; esac
    AFEM_LIBRARY=$lib AFEM_STENCIL_SPLIT=$sp timeout 300 python bench.py --steps 40 --warmup 12 --no-cpu --e2e-steps 1 > gpurun_out/abh_${v}_$rep.json 2>gpurun_out/abh_${v}_$rep.err
    python -c "import json; d=json.loads(open('gpurun_out/abh_${v}_$rep.json').read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step']*1e3,2), 'us', round(d['value']/1e9,2), 'GDOF/s cg', round(d['cg']['solve_s'],3), d['cg']['iterations'])"
  done
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_stencil" -s 20 -c 1 \
  -o gpurun_out/prof_r02h -f python bench.py --steps 5 --warmup 3 --no-cpu --no-cg --e2e-steps 1 > gpurun_out/prof_r02h.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_r02h.csv python bench.py --steps 5 --warmup 3 --no-cpu --no-cg --e2e-steps 1 > gpurun_out/launches_r02h.log 2>&1

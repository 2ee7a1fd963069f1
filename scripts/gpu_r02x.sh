#!/bin/bash
# round 2, call X: axis-factorised interior stencil (plane_sep, default) against the direct 153-DFMA
# sum (variants/libafem_nosep.so): correctness on the default build, then alternated A/B
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stencil.py tests/test_gpu_fullsize.py -q -x > gpurun_out/pytest_x.log 2>&1
echo "stencil tests exit $?: $(tail -1 gpurun_out/pytest_x.log)"; grep -E "^FAILED|Error" gpurun_out/pytest_x.log | head -5
for rep in 1 2; do
for v in default nosep; do
  lib=""; [ $v != default ] && lib=paper_2604_22087_b200/variants/libafem_$v.so
  AFEM_LIBRARY=$lib timeout 300 python bench.py --steps 40 --warmup 12 --no-cpu --e2e-steps 1 > gpurun_out/abx_${v}_$rep.json 2>gpurun_out/abx_${v}_$rep.err
  python -c "import json; d=json.loads(open('gpurun_out/abx_${v}_$rep.json').read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step']*1e3,2), 'us', round(d['value']/1e9,2), 'GDOF/s cg', round(d['cg']['solve_s'],3), d['cg']['iterations'])"
  AFEM_LIBRARY=$lib AFEM_STENCIL_ONLY=main timeout 300 python bench.py --steps 40 --warmup 12 --no-cpu --no-cg --e2e-steps 1 > gpurun_out/abx_${v}_main$rep.json 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/abx_${v}_main$rep.json').read().strip().splitlines()[-1]); print('$v main only', round(d['ms_per_step']*1e3,2), 'us')"
done
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_stencil_tma" -s 20 -c 1 \
  -o gpurun_out/prof_r02x -f python bench.py --steps 5 --warmup 3 --no-cpu --no-cg --e2e-steps 1 > gpurun_out/prof_r02x.log 2>&1
echo "ncu exit $?"

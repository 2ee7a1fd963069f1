#!/bin/bash
# round 2, call F: exact-norm fused GMRES, main kernel with spread TMA issue (88 registers) vs the
# round-start build, the test files touched this round, bench, ncu of the new main kernel
mkdir -p gpurun_out
timeout 600 python scripts/gmres_debug.py > gpurun_out/gmres_debug_f.txt 2>&1; cut -c1-700 gpurun_out/gmres_debug_f.txt
for v in default base; do
  lib=""; [ $v != default ] && lib=paper_2604_22087_b200/variants/libafem_$v.so
  for rep in 1 2; do
    AFEM_LIBRARY=$lib AFEM_NO_APPLY_GRAPH=1 timeout 300 python bench.py --steps 40 --warmup 12 --no-cpu --no-cg --e2e-steps 1 > gpurun_out/abf_${v}_$rep.json 2>gpurun_out/abf_${v}_$rep.err
    python -c "import json; d=json.loads(open('gpurun_out/abf_${v}_$rep.json').read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step']*1e3,2), 'us', round(d['value']/1e9,2), 'GDOF/s')"
  done
done
for f in test_gpu_gmres test_gpu_dist test_gpu_stencil test_gpu_parity test_gpu_ref_suite test_gpu_fullsize; do
  timeout 900 python -X faulthandler -m pytest tests/$f.py -q > gpurun_out/pytest_f_$f.log 2>&1
  echo "$f exit $?: $(tail -1 gpurun_out/pytest_f_$f.log)"
done
timeout 600 python bench.py --steps 30 --warmup 5 > gpurun_out/bench_f.json 2> gpurun_out/bench_f.err
tail -2 gpurun_out/bench_f.err; cut -c1-900 gpurun_out/bench_f.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_stencil" -s 20 -c 2 \
  -o gpurun_out/prof_r02f -f python bench.py --steps 5 --warmup 3 --no-cpu --no-cg --e2e-steps 1 > gpurun_out/prof_r02f.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_r02f.csv python bench.py --steps 5 --warmup 3 --no-cpu --no-cg --e2e-steps 1 > gpurun_out/launches_r02f.log 2>&1

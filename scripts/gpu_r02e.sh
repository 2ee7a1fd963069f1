#!/bin/bash
# round 2, call E: GMRES debug, kernel-variant A/B (items gathers, planes per barrier), the drop-in
# suites with the context-lifetime fix, failing test files, bench
mkdir -p gpurun_out
timeout 600 python scripts/gmres_debug.py > gpurun_out/gmres_debug.txt 2>&1; cat gpurun_out/gmres_debug.txt | cut -c1-1500
for v in default nopipe pipe128 base; do
  lib=""; [ $v != default ] && lib=paper_2604_22087_b200/variants/libafem_$v.so
  for g in 1 0; do
    if [ $g = 1 ]; then ng=1; else ng=; fi
    [ $v = base ] && [ $g = 0 ] && continue
    AFEM_LIBRARY=$lib AFEM_NO_APPLY_GRAPH=$ng timeout 300 python bench.py --steps 40 --warmup 12 --no-cpu --no-cg --e2e-steps 1 > gpurun_out/ab_${v}_g$g.json 2>gpurun_out/ab_${v}_g$g.err
    python -c "import json; d=json.loads(open('gpurun_out/ab_${v}_g$g.json').read().strip().splitlines()[-1]); print('$v nograph=$g', round(d['ms_per_step']*1e3,2), 'us', round(d['value']/1e9,2), 'GDOF/s')"
  done
done
for f in test_gpu_ref_suite test_gpu_nonlinear test_gpu_dist test_gpu_gmres; do
  timeout 900 python -X faulthandler -m pytest tests/$f.py -q > gpurun_out/pytest_e_$f.log 2>&1
  echo "$f exit $?: $(tail -1 gpurun_out/pytest_e_$f.log)"
done
grep -E "FAILED|tests ran|PASSED" gpurun_out/pytest_e_test_gpu_ref_suite.log | head

#!/bin/bash
# round 2, call K: two node rows per warp (AFEM_STENCIL_ROWS=2; ring 3 -> 4 CTAs/SM, ring 4 -> 3)
# against the one-row kernel: correctness (stencil + full-size tests on each build) and A/B
mkdir -p gpurun_out
for v in rw2 rw2r4; do
  AFEM_LIBRARY=paper_2604_22087_b200/variants/libafem_$v.so timeout 900 python -m pytest tests/test_gpu_stencil.py tests/test_gpu_fullsize.py -q -x > gpurun_out/pytest_k_$v.log 2>&1
  echo "$v stencil tests exit $?: $(tail -1 gpurun_out/pytest_k_$v.log)"
done
for v in default rw2 rw2r4; do
  lib=""; [ $v != default ] && lib=paper_2604_22087_b200/variants/libafem_$v.so
  for rep in 1 2; do
    AFEM_LIBRARY=$lib timeout 300 python bench.py --steps 40 --warmup 12 --no-cpu --e2e-steps 1 > gpurun_out/abk_${v}_$rep.json 2>gpurun_out/abk_${v}_$rep.err
    python -c "import json; d=json.loads(open('gpurun_out/abk_${v}_$rep.json').read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step']*1e3,2), 'us', round(d['value']/1e9,2), 'GDOF/s cg', round(d['cg']['solve_s'],3), d['cg']['iterations'])"
  done
  AFEM_LIBRARY=$lib AFEM_STENCIL_ONLY=main timeout 300 python bench.py --steps 40 --warmup 12 --no-cpu --no-cg --e2e-steps 1 > gpurun_out/abk_${v}_main.json 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/abk_${v}_main.json').read().strip().splitlines()[-1]); print('$v main only', round(d['ms_per_step']*1e3,2), 'us')"
done

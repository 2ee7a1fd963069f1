#!/bin/bash
# round 2, call J: items kernel occupancy variants (64-register cap at 4 x 256 threads, 7 x 128 threads)
mkdir -p gpurun_out
for v in default items_minb4 items128; do
  lib=""; [ $v != default ] && lib=paper_2604_22087_b200/variants/libafem_$v.so
  for rep in 1 2; do
    AFEM_LIBRARY=$lib AFEM_STENCIL_ONLY=items timeout 300 python bench.py --steps 40 --warmup 12 --no-cpu --no-cg --e2e-steps 1 > gpurun_out/abj_${v}_$rep.json 2>&1
    python -c "import json; d=json.loads(open('gpurun_out/abj_${v}_$rep.json').read().strip().splitlines()[-1]); print('$v items only', round(d['ms_per_step']*1e3,2), 'us')"
  done
  AFEM_LIBRARY=$lib timeout 300 python bench.py --steps 40 --warmup 12 --no-cpu --no-cg --e2e-steps 1 > gpurun_out/abj_${v}_full.json 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/abj_${v}_full.json').read().strip().splitlines()[-1]); print('$v full', round(d['ms_per_step']*1e3,2), 'us')"
done

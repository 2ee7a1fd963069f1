#!/bin/bash
# round 2, call Y: main-kernel skeleton (staging, masking, barriers, output; no stencil arithmetic)
# against the full main kernel, to split the 50 us between arithmetic and the per-plane pipeline
mkdir -p gpurun_out
for rep in 1 2; do
for v in default nosep nocomp; do
  lib=""; [ $v != default ] && lib=paper_2604_22087_b200/variants/libafem_$v.so
  AFEM_LIBRARY=$lib AFEM_STENCIL_ONLY=main timeout 300 python bench.py --steps 40 --warmup 12 --no-cpu --no-cg --e2e-steps 1 > gpurun_out/aby_${v}_main$rep.json 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/aby_${v}_main$rep.json').read().strip().splitlines()[-1]); print('$v main only', round(d['ms_per_step']*1e3,2), 'us')"
done
done

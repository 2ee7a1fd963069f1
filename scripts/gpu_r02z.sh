#!/bin/bash
# round 2, call Z: what bounds the main kernel's per-plane pipeline (measurement builds):
# skeleton (no arithmetic) with a deeper TMA ring / 3 CTAs per SM / no y stores, and the full kernel
# with the deeper ring and without stores
mkdir -p gpurun_out
for rep in 1 2; do
for v in ${VARIANTS:-nosep nocomp nocomp_r6 nocomp_m3 nocomp_nost r6 nost}; do
  lib=paper_2604_22087_b200/variants/libafem_$v.so
  AFEM_LIBRARY=$lib AFEM_STENCIL_ONLY=main timeout 300 python bench.py --steps 40 --warmup 12 --no-cpu --no-cg --e2e-steps 1 > gpurun_out/abz_${v}_main$rep.json 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/abz_${v}_main$rep.json').read().strip().splitlines()[-1]); print('$v main only', round(d['ms_per_step']*1e3,2), 'us')"
done
done

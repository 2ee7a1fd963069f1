#!/bin/bash
# round 2, call AD: fused corrections with two accumulator chains per row; the fused schedule
# without corrections (variants/libafem_fskip.so, timing only); the separate kernels
mkdir -p gpurun_out
for rep in 1 2; do
for v in ${VARIANTS:-fused fskip nofuse}; do
  env=""; lib=""; [ $v = nofuse ] && env="AFEM_STENCIL_NOFUSE=1"; [ $v = fskip ] && lib=paper_2604_22087_b200/variants/libafem_fskip.so
  env $env AFEM_LIBRARY=$lib AFEM_STENCIL_ONLY=main timeout 300 python bench.py --steps 40 --warmup 12 --no-cpu --no-cg --e2e-steps 1 > gpurun_out/abad_${v}_main$rep.json 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/abad_${v}_main$rep.json').read().strip().splitlines()[-1]); print('$v main only', round(d['ms_per_step']*1e3,2), 'us')"
done
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_stencil_tma" -s 20 -c 1 \
  -o gpurun_out/prof_r02ad -f python bench.py --steps 30 --warmup 3 --no-cpu --no-cg --e2e-steps 0 > gpurun_out/prof_r02ad.log 2>&1
echo "ncu exit $?"

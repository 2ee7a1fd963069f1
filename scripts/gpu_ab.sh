#!/bin/bash
# A/B: default stencil vs AFEM_STENCIL_FUSE_ITEMS=1 (apply time + launch list per variant)
TAG=${1:-ab}
for V in 0 1; do
  AFEM_STENCIL_FUSE_ITEMS=$V timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu --no-cg --e2e-steps 1 > gpurun_out/bench_${TAG}_$V.json 2> gpurun_out/bench_${TAG}_$V.err
  python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print('fuse=$V apply_us', round(d['ms_per_step']*1e3,1))" gpurun_out/bench_${TAG}_$V.json
  AFEM_STENCIL_FUSE_ITEMS=$V timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_stencil -c 20 --csv \
    --log-file gpurun_out/launches_${TAG}_$V.csv python bench.py --steps 3 --warmup 1 --no-cpu --no-cg --e2e-steps 1 > /dev/null 2>&1
done

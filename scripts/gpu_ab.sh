#!/bin/bash
# A/B: stencil apply time + launch list, run twice with env var AFEM_AB=0/1 for experiments
TAG=${1:-ab}
for V in 0 1; do
  AFEM_AB=$V timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu --no-cg --e2e-steps 1 > gpurun_out/bench_${TAG}_$V.json 2> gpurun_out/bench_${TAG}_$V.err
  python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print('ab=$V apply_us', round(d['ms_per_step']*1e3,1))" gpurun_out/bench_${TAG}_$V.json
  AFEM_AB=$V timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_stencil -c 20 --csv \
    --log-file gpurun_out/launches_${TAG}_$V.csv python bench.py --steps 3 --warmup 1 --no-cpu --no-cg --e2e-steps 1 > /dev/null 2>&1
done

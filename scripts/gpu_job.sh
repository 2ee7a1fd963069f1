#!/bin/bash
# GPU-box job: tests, bench, launch list and one ncu --set full capture of the stencil kernels.
# usage: bash scripts/gpu_job.sh TAG [tests|bench|ncu|all]
TAG=${1:-r}
WHAT=${2:-all}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
if [[ $WHAT == all || $WHAT == tests ]]; then
  timeout 1200 python -m pytest tests -q -m gpu 2>&1 | tail -30
fi
if [[ $WHAT == all || $WHAT == bench ]]; then
  timeout 900 python bench.py --steps 30 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
  tail -3 gpurun_out/bench_$TAG.err; cat gpurun_out/bench_$TAG.json
fi
if [[ $WHAT == all || $WHAT == ncu ]]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 5 --warmup 1 --no-cpu --e2e-steps 1 > /dev/null 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stencil -s 3 -c 3 \
    -o gpurun_out/prof_$TAG python bench.py --steps 3 --warmup 1 --no-cpu --no-cg --e2e-steps 1 > gpurun_out/ncu_$TAG.log 2>&1
  tail -3 gpurun_out/ncu_$TAG.log
fi

#!/bin/bash
# ncu --set full of one kernel (regex $2) in a short bench run; report -> gpurun_out/prof_$1
TAG=$1; K=$2
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 1 \
  -o gpurun_out/prof_$TAG python bench.py --steps 3 --warmup 1 --no-cpu --no-cg --e2e-steps 1 > gpurun_out/ncu_$TAG.log 2>&1
tail -1 gpurun_out/ncu_$TAG.log

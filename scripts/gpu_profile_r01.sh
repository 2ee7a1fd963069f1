#!/bin/bash
# Round-1 profile set for the bench kernels: launch list of the bench command, one ncu --set full
# capture of the apply's kernels (main + items) and of the CG vector kernels, in-situ per-kernel
# times. Outputs under gpurun_out/prof_*. usage: bash scripts/gpu_profile_r01.sh
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/prof_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --e2e-steps 1 > gpurun_out/prof_launches.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_stencil" -s 4 -c 2 \
  -o gpurun_out/prof_stencil -f python bench.py --steps 3 --warmup 1 --no-cpu --no-cg --e2e-steps 1 > gpurun_out/prof_stencil.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"k_cg_update|k_cg_p" -s 40 -c 2 \
  -o gpurun_out/prof_cg -f python bench.py --steps 3 --warmup 1 --no-cpu --e2e-steps 1 > gpurun_out/prof_cg.log 2>&1
bash scripts/gpu_insitu.sh r01c > /dev/null 2>&1

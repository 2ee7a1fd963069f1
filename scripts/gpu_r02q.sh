#!/bin/bash
# round 2, call Q: ncu --set full of the matrix-free JVP kernels at 128^3 (config-3 NH element
# pass + gather; config-4 cached J2 element pass)
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:k_grid_elem<3, 1>|k_gather<3>" -c 4 -o gpurun_out/prof_q_nh -f \
  python scripts/jvp_probe.py --n 128 --reps 2 > gpurun_out/prof_q_nh.log 2>&1; echo "nh ncu exit $?"
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k "regex:k_grid_jvp_cached" -c 2 -o gpurun_out/prof_q_j2 -f \
  python scripts/c4_mf.py 128 > gpurun_out/prof_q_j2.log 2>&1; echo "j2 ncu exit $?"
ls -la gpurun_out/*.ncu-rep

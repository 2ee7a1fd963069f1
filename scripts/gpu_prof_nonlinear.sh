#!/bin/bash
# ncu --set full of every nonlinear-path kernel (C4-shaped J2 grid, N = ${1:-128}).
mkdir -p gpurun_out
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_(grid_elem|gather|jacobian|eliminate|csr_apply|history_commit|cg_)" -c 16 \
  -o gpurun_out/prof_nl python scripts/prof_nonlinear.py ${1:-128} > gpurun_out/prof_nl.log 2>&1
tail -2 gpurun_out/prof_nl.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_(grid_elem|gather|jacobian|eliminate|csr_apply|history_commit|cg_)" -c 30 \
  --csv --log-file gpurun_out/launches_nl.csv python scripts/prof_nonlinear.py ${1:-128} > /dev/null 2>&1

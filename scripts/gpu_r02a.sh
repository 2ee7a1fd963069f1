#!/bin/bash
# round 2, call A: full GPU suite (incl. the C2 full-size oracle parity), C5 100 M-dof solve, bench
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc
timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -15
timeout 600 python scripts/solve_c5.py --out gpurun_out/c5_solve.jsonl 2>&1 | tail -3
timeout 600 python bench.py --steps 30 --warmup 5 > gpurun_out/bench_a.json 2> gpurun_out/bench_a.err
tail -3 gpurun_out/bench_a.err; cat gpurun_out/bench_a.json

#!/bin/bash
# round 2, call B (after container re-creation): GPU suite, bench, C3/C4 at stated size
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc
timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -15
timeout 600 python bench.py --steps 30 --warmup 5 > gpurun_out/bench_b.json 2> gpurun_out/bench_b.err
tail -3 gpurun_out/bench_b.err; cat gpurun_out/bench_b.json
timeout 3000 python scripts/solve_configs.py --lin-rtol4 1e-4 --out gpurun_out/configs_b.jsonl > gpurun_out/configs_b.log 2>&1
tail -20 gpurun_out/configs_b.log

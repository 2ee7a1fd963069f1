#!/bin/bash
TAG=${1:-q}
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu --e2e-steps 2 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
python - gpurun_out/bench_$TAG.json <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print("apply_us", round(d["ms_per_step"] * 1e3, 1), "GDOF/s", round(d["value"] / 1e9, 1), "hbm_frac", round(d["roofline"]["frac"], 3),
      "fp64_frac", round(d["roofline"]["fp64"]["frac"], 3), "cg", d["cg"])
PY
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 5 --warmup 1 --no-cpu --e2e-steps 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stencil -s 3 -c 3 \
  -o gpurun_out/prof_$TAG python bench.py --steps 3 --warmup 1 --no-cpu --no-cg --e2e-steps 1 > gpurun_out/ncu_$TAG.log 2>&1
tail -1 gpurun_out/ncu_$TAG.log

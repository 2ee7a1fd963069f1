#!/bin/bash
# Fast stencil iteration on the GPU box: stencil parity tests, a short bench (apply time, HBM
# fraction, CG), and the per-kernel ncu launch times of the apply. usage: bash scripts/gpu_iter.sh TAG
TAG=${1:-it}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_stencil.py -q -x 2>&1 | tail -2
timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu --e2e-steps 2 > gpurun_out/bench_$TAG.json 2>gpurun_out/bench_$TAG.err
python - "$TAG" <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/bench_{sys.argv[1]}.json").read().strip().splitlines()[-1])
print("apply_us", round(d["ms_per_step"] * 1e3, 1), "hbm_frac", round(d["roofline"]["frac"], 3),
      "cg_s", d["cg"]["solve_s"], "cg_it", d["cg"]["iterations"], "e2e", d["e2e"]["value"])
PY
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_stencil|k_fix" -c 9 python bench.py --steps 3 --warmup 1 --no-cpu --no-cg --e2e-steps 1 > gpurun_out/ncu_$TAG.txt 2>&1
python - "$TAG" <<'PY'
import re, sys
name = None
for line in open(f"gpurun_out/ncu_{sys.argv[1]}.txt"):
    m = re.search(r"(k_(?:stencil|fix)_\w+)", line)
    if m and "void" in line:
        name = m.group(1)
    elif "gpu__time_duration.sum" in line and name:
        print(name, line.split()[-1])
        name = None
PY

#!/bin/bash
# C5 single-GPU points: the device-resident matrix-free apply (bench.py --n N, L2 flushed between
# applies; round 2: rotating buffers) of the linear hex8 fibre RVE at N in {128,...,404}: 6.4 M -> 199 M dofs.
mkdir -p gpurun_out
for N in 128 160 202 254 321 404; do
  timeout 900 python bench.py --n $N --steps 10 --warmup 3 --no-cpu --e2e-steps 1 --no-cg > gpurun_out/sweep_$N.json 2> gpurun_out/sweep_$N.err
  python - "$N" <<'PY'
import json, sys
n = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/sweep_{n}.json").read().strip().splitlines()[-1])
    print(n, d["config"]["n_dof"], "apply_us", round(d["ms_per_step"] * 1e3, 1), "GDOF/s", round(d["value"] / 1e9, 1),
          "hbm_frac", round(d["roofline"]["frac"], 3), "fp64_frac", round(d["roofline"]["fp64"]["frac"], 3))
except Exception as e:
    print(n, "failed", e, open(f"gpurun_out/sweep_{n}.err").read()[-400:])
PY
done

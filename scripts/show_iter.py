"""Print the apply time / CG of a gpu_iter bench JSON and the stencil kernel times of its ncu list."""
import json
import re
import sys

t = sys.argv[1]
d = json.loads(open(f"gpurun_out/bench_{t}.json").read().strip().splitlines()[-1])
print(t, "apply_us", round(d["ms_per_step"] * 1e3, 1), "cg_s", round(d["cg"]["solve_s"], 3) if d["cg"] else None)
name = None
ts = {}
for line in open(f"gpurun_out/ncu_{t}.txt"):
    m = re.search(r"(k_(?:stencil|fix)_\w+)", line)
    if m and "Context" in line:
        name = m.group(1)
    elif "gpu__time_duration.sum" in line and name:
        ts.setdefault(name, []).append(float(line.split()[-1]))
        name = None
for k, v in ts.items():
    print("  ", k, [round(x, 1) for x in v])

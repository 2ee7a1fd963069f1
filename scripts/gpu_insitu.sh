#!/bin/bash
# Per-kernel times of the apply with caches as left by the previous kernel (ncu --cache-control none;
# the bench still flushes L2 between applies). usage: bash scripts/gpu_insitu.sh TAG
TAG=${1:-x}
timeout 300 ncu --cache-control none --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  -k regex:"k_stencil" -s 4 -c 6 python bench.py --steps 4 --warmup 2 --no-cpu --no-cg --e2e-steps 1 > gpurun_out/insitu_$TAG.txt 2>&1
python - "$TAG" <<'PY'
import re, sys
name, vals = None, {}
for line in open(f"gpurun_out/insitu_{sys.argv[1]}.txt"):
    m = re.search(r"(k_stencil_\w+)", line)
    if m and "(" in line and "Context" in line:
        name = m.group(1)
    for k in ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum"):
        if k in line and name:
            vals.setdefault(name, []).append((k.split("__")[1].split(".")[0], line.split()[-2], line.split()[-1]))
for k, v in vals.items():
    print(sys.argv[1], k, v[:3])
PY

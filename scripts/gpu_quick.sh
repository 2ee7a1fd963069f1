#!/bin/bash
# Quick GPU iteration: stencil tests, two bench variants, ncu of the main kernel.
# usage: bash scripts/gpu_quick.sh TAG
TAG=${1:-q}
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_stencil.py -q -x 2>&1 | tail -3
for occ in 3 2; do
  AFEM_STENCIL_OCC=$occ timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu --e2e-steps 2 \
    > gpurun_out/bench_${TAG}_occ$occ.json 2> gpurun_out/bench_${TAG}_occ$occ.err
  python - "$occ" gpurun_out/bench_${TAG}_occ$occ.json <<'EOF'
import json, sys
d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
print("occ", sys.argv[1], "apply_us", round(d["ms_per_step"] * 1e3, 1), "GDOF/s", round(d["value"] / 1e9, 1),
      "hbm_frac", round(d["roofline"]["frac"], 3), "fp64_frac", round(d["roofline"]["fp64"]["frac"], 3),
      "cg_s", d["cg"]["solve_s"] if d["cg"] else None, "cg_it", d["cg"]["iterations"] if d["cg"] else None)
EOF
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 5 --warmup 1 --no-cpu --e2e-steps 1 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_stencil -s 3 -c 3 \
  -o gpurun_out/prof_$TAG python bench.py --steps 3 --warmup 1 --no-cpu --no-cg --e2e-steps 1 > gpurun_out/ncu_$TAG.log 2>&1
tail -2 gpurun_out/ncu_$TAG.log

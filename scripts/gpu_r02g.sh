#!/bin/bash
# round 2, call G: the whole GPU suite + smoke (round-end gate), main-kernel A/B (5 CTAs / SM,
# LDS.128 window loads, round-start build), bench, the C5 100 M-dof solve with the current kernels
mkdir -p gpurun_out
timeout 1800 python -X faulthandler -m pytest tests -q -m gpu > gpurun_out/pytest_g_all.log 2>&1
echo "pytest -m gpu exit $?: $(tail -1 gpurun_out/pytest_g_all.log)"
grep -E "^FAILED|^ERROR" gpurun_out/pytest_g_all.log | head -20
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_g.log 2>&1; echo "smoke exit $?: $(tail -1 gpurun_out/smoke_g.log)"
for v in default lds128 base; do
  lib=""; [ $v != default ] && lib=paper_2604_22087_b200/variants/libafem_$v.so
  for rep in 1 2; do
    AFEM_LIBRARY=$lib AFEM_NO_APPLY_GRAPH=1 timeout 300 python bench.py --steps 40 --warmup 12 --no-cpu --no-cg --e2e-steps 1 > gpurun_out/abg_${v}_$rep.json 2>gpurun_out/abg_${v}_$rep.err
    python -c "import json; d=json.loads(open('gpurun_out/abg_${v}_$rep.json').read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step']*1e3,2), 'us', round(d['value']/1e9,2), 'GDOF/s')"
  done
done
timeout 600 python bench.py --steps 30 --warmup 5 > gpurun_out/bench_g.json 2> gpurun_out/bench_g.err
tail -2 gpurun_out/bench_g.err; cut -c1-600 gpurun_out/bench_g.json
timeout 900 python scripts/solve_c5.py --out gpurun_out/c5_solve_g.jsonl > gpurun_out/c5_g.log 2>&1; tail -2 gpurun_out/c5_g.log | cut -c1-600

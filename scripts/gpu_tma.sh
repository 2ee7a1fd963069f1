#!/bin/bash
# TMA main-kernel A/B: parity tests, bench (TMA vs cp.async staging), ncu of the TMA kernel
TAG=${1:-tma}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stencil.py tests/test_gpu_fullsize.py tests/test_gpu_dist.py -x -q 2>&1 | tail -5
for k in 1 2; do
timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu --no-cg --e2e-steps 2 > gpurun_out/bench_${TAG}_$k.json 2>&1
AFEM_STENCIL_LDGSTS=1 timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu --no-cg --e2e-steps 2 > gpurun_out/bench_${TAG}_old$k.json 2>&1
done
for f in gpurun_out/bench_${TAG}_*.json; do echo $f; python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['value']/1e9, d['roofline']['frac'])"; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
    --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 5 --warmup 1 --no-cpu --e2e-steps 1 --no-cg > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_stencil -s 4 -c 2 \
    -o gpurun_out/prof_$TAG python bench.py --steps 3 --warmup 1 --no-cpu --no-cg --e2e-steps 1 > gpurun_out/ncu_$TAG.log 2>&1
tail -2 gpurun_out/ncu_$TAG.log

for v in "" main items; do for k in 1 2; do AFEM_STENCIL_ONLY=$v timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu --no-cg --e2e-steps 1 > gpurun_out/bench_t$v$k.json 2>&1; done; done
for f in gpurun_out/bench_t*.json; do python -c "import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', d['ms_per_step'], d['value']/1e9, d['roofline']['frac'])"; done

#!/bin/bash
# round 2, call W: correction items concurrent with the main kernel vs sequential
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stencil.py tests/test_gpu_fullsize.py tests/test_gpu_parity.py -q -x > gpurun_out/pytest_w.log 2>&1; echo "pytest exit $?: $(tail -1 gpurun_out/pytest_w.log)"; grep -E "^FAILED|^E " gpurun_out/pytest_w.log | head -5
for N in 128 321; do
  for v in conc serial conc serial; do
    if [ $v = serial ]; then se=1; else se=; fi
    AFEM_ITEMS_SERIAL=$se timeout 600 python bench.py --n $N --steps 30 --warmup 8 --no-cpu --no-cg --e2e-steps 1 > gpurun_out/abw_${v}_$N.json 2>&1
    python -c "import json; d=json.loads(open('gpurun_out/abw_${v}_$N.json').read().strip().splitlines()[-1]); print('$N $v', round(d['ms_per_step']*1e3,1), 'us', round(d['value']/1e9,1), 'GDOF/s', round(d['roofline']['frac'],3))"
  done
done

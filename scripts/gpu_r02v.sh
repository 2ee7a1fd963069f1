#!/bin/bash
# round 2, call V: 4 vs 5 main CTAs per SM across sizes (128^3, 254^3, 321^3)
mkdir -p gpurun_out
for N in 128 254 321; do
  for v in default minb5; do
    lib=""; [ $v != default ] && lib=paper_2604_22087_b200/variants/libafem_$v.so
    AFEM_LIBRARY=$lib timeout 600 python bench.py --n $N --steps 20 --warmup 6 --no-cpu --no-cg --e2e-steps 1 > gpurun_out/abv_${v}_$N.json 2>&1
    python -c "import json; d=json.loads(open('gpurun_out/abv_${v}_$N.json').read().strip().splitlines()[-1]); print('$N $v', round(d['ms_per_step']*1e3,1), 'us', round(d['value']/1e9,1), 'GDOF/s', round(d['roofline']['frac'],3))"
  done
done

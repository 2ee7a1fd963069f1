#!/bin/bash
# round 2, call AB: per-plane overhead of the main kernel — plane loop unrolled by three (static
# accumulator roles), one issuing thread, window-only masking test, lean output addressing — alone
# and combined, against the default (role-slot refactor, switches off); stencil tests on default
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stencil.py -q -x > gpurun_out/pytest_ab.log 2>&1
echo "stencil tests exit $?: $(tail -1 gpurun_out/pytest_ab.log)"
for rep in 1 2; do
for v in default u3 is1 mw lo u3mwlo all4; do
  lib=""; [ $v != default ] && lib=paper_2604_22087_b200/variants/libafem_$v.so
  AFEM_LIBRARY=$lib AFEM_STENCIL_ONLY=main timeout 300 python bench.py --steps 40 --warmup 12 --no-cpu --no-cg --e2e-steps 1 > gpurun_out/abab_${v}_main$rep.json 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/abab_${v}_main$rep.json').read().strip().splitlines()[-1]); print('$v main only', round(d['ms_per_step']*1e3,2), 'us')"
done
done

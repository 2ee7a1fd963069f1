#!/bin/bash
# round 2, call AA: z-run correction kernel (k_stencil_items rewritten) — correctness on the
# default build, then items-only and full-apply timings against the previous item kernel
# (variants/libafem_nosep.so) and run-length / occupancy variants
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_stencil.py tests/test_gpu_fullsize.py tests/test_gpu_dist.py -q -x > gpurun_out/pytest_aa.log 2>&1
echo "tests exit $?: $(tail -1 gpurun_out/pytest_aa.log)"; grep -E "^FAILED|Error|assert" gpurun_out/pytest_aa.log | head -8
for rep in 1 2; do
for v in default nosep it_m3 it_r4 it_r16; do
  lib=""; [ $v != default ] && lib=paper_2604_22087_b200/variants/libafem_$v.so
  AFEM_LIBRARY=$lib AFEM_STENCIL_ONLY=items timeout 300 python bench.py --steps 40 --warmup 12 --no-cpu --no-cg --e2e-steps 1 > gpurun_out/abaa_${v}_items$rep.json 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/abaa_${v}_items$rep.json').read().strip().splitlines()[-1]); print('$v items only', round(d['ms_per_step']*1e3,2), 'us')"
done
done
for v in default nosep it_m3; do
  lib=""; [ $v != default ] && lib=paper_2604_22087_b200/variants/libafem_$v.so
  AFEM_LIBRARY=$lib timeout 300 python bench.py --steps 40 --warmup 12 --no-cpu --e2e-steps 1 > gpurun_out/abaa_${v}.json 2>gpurun_out/abaa_${v}.err
  python -c "import json; d=json.loads(open('gpurun_out/abaa_${v}.json').read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step']*1e3,2), 'us', round(d['value']/1e9,2), 'GDOF/s cg', round(d['cg']['solve_s'],3), d['cg']['iterations'])"
done

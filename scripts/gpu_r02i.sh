#!/bin/bash
# round 2, call I: items kernel with scalar loads + sign-bit flips vs the current form; stencil tests
mkdir -p gpurun_out
for v in default iscalar; do
  lib=""; [ $v != default ] && lib=paper_2604_22087_b200/variants/libafem_$v.so
  for rep in 1 2; do
    AFEM_LIBRARY=$lib timeout 300 python bench.py --steps 40 --warmup 12 --no-cpu --no-cg --e2e-steps 1 > gpurun_out/abi_${v}_$rep.json 2>gpurun_out/abi_${v}_$rep.err
    python -c "import json; d=json.loads(open('gpurun_out/abi_${v}_$rep.json').read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step']*1e3,2), 'us', round(d['value']/1e9,2), 'GDOF/s')"
  done
  AFEM_LIBRARY=$lib AFEM_STENCIL_ONLY=items timeout 300 python bench.py --steps 40 --warmup 12 --no-cpu --no-cg --e2e-steps 1 > gpurun_out/abi_${v}_items.json 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/abi_${v}_items.json').read().strip().splitlines()[-1]); print('$v items only', round(d['ms_per_step']*1e3,2), 'us')"
done
AFEM_LIBRARY=paper_2604_22087_b200/variants/libafem_iscalar.so timeout 900 python -m pytest tests/test_gpu_stencil.py tests/test_gpu_fullsize.py -q > gpurun_out/pytest_i.log 2>&1; echo "iscalar stencil tests exit $?: $(tail -1 gpurun_out/pytest_i.log)"

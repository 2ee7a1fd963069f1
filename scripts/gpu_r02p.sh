#!/bin/bash
# round 2, call P: Gauss-point split of the element kernels (AFEM_QSPLIT = 1, 2, 4, 8 lanes per
# element) on the config-3 NH JVP / residual (192^3) and the config-4 cached J2 JVP (256^3); parity
# tests with the split on
mkdir -p gpurun_out
for i in 1 2; do
  for q in 1 8 4 2; do
    echo "{\"qsplit\": $q, \"c3\": $(AFEM_QSPLIT=$q timeout 600 python scripts/jvp_probe.py 2>&1 | tail -1), \"c4\": \"$(AFEM_QSPLIT=$q timeout 600 python scripts/c4_mf.py 256 2>&1 | tail -1)\"}"
  done
done | tee gpurun_out/qsplit_p.jsonl
AFEM_QSPLIT=8 timeout 900 python -m pytest tests/test_gpu_nonlinear.py tests/test_gpu_dist.py -q -x > gpurun_out/t_p.log 2>&1; tail -2 gpurun_out/t_p.log

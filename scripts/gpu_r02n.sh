#!/bin/bash
# round 2, call N: A/B against the previous build (AFEM_LIBRARY=libafem_ab.so): config-3 tangent
# assembly with the Neo-Hookean block coefficients hoisted to the Gauss point, and the slab CG step
# that recomputes u = M r instead of re-reading it (world size 1: no allreduce launch)
mkdir -p gpurun_out
AB=paper_2604_22087_b200/libafem_ab.so
for i in 1 2; do
  timeout 600 python scripts/jvp_probe.py --spmv >> gpurun_out/jac_n.jsonl 2>&1
  AFEM_LIBRARY=$AB timeout 600 python scripts/jvp_probe.py --spmv | sed 's/^{/{"build": "previous", /' >> gpurun_out/jac_n.jsonl 2>&1
done
cat gpurun_out/jac_n.jsonl
timeout 600 python scripts/dist_cg_probe.py > gpurun_out/dist_cg_n.jsonl 2>&1
AFEM_LIBRARY=$AB timeout 600 python scripts/dist_cg_probe.py | sed 's/^{/{"build": "previous", /' >> gpurun_out/dist_cg_n.jsonl 2>&1
cat gpurun_out/dist_cg_n.jsonl
timeout 900 python -m pytest tests/test_gpu_dist.py tests/test_gpu_nonlinear.py tests/test_gpu_parity.py -q -x > gpurun_out/t_n.log 2>&1; tail -2 gpurun_out/t_n.log

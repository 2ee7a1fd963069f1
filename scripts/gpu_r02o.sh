#!/bin/bash
# round 2, call O: C4 cached-tangent JVP with the next Gauss point's tangent prefetched, A/B against
# the previous build (AFEM_LIBRARY=libafem_ab.so), checksums must agree; the J2 parity tests
mkdir -p gpurun_out
AB=paper_2604_22087_b200/libafem_ab.so
for i in 1 2; do
  echo "new: $(timeout 600 python scripts/c4_mf.py 256 2>&1 | tail -1)"
  echo "previous: $(AFEM_LIBRARY=$AB timeout 600 python scripts/c4_mf.py 256 2>&1 | tail -1)"
done | tee gpurun_out/c4_jvp_o.txt
timeout 900 python -m pytest tests/test_gpu_nonlinear.py tests/test_gpu_dist.py -q -x > gpurun_out/t_o.log 2>&1; tail -2 gpurun_out/t_o.log

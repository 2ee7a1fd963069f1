#!/bin/bash
# round 2, call R: config-4 cached J2 JVP with the element's cached tangents staged by cp.async
# (one round trip per element), A/B against the previous build; J2 parity tests
mkdir -p gpurun_out
AB=paper_2604_22087_b200/libafem_ab.so
for i in 1 2; do
  echo "new: $(timeout 600 python scripts/c4_mf.py 256 2>&1 | tail -1)"
  echo "previous: $(AFEM_LIBRARY=$AB timeout 600 python scripts/c4_mf.py 256 2>&1 | tail -1)"
done | tee gpurun_out/c4_jvp_r.txt
timeout 900 python -m pytest tests/test_gpu_nonlinear.py tests/test_gpu_dist.py -q -x > gpurun_out/t_r.log 2>&1; tail -2 gpurun_out/t_r.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_grid_jvp_cached -c 1 -o gpurun_out/prof_r_j2 -f \
  python scripts/c4_mf.py 128 > gpurun_out/prof_r_j2.log 2>&1; echo "ncu exit $?"

#!/bin/bash
# round 2, call C: the reference's own suites on the drop-in, GMRES / dist tests, the B^T D B
# tensor-core probe, the bench (rotating buffers) and the r02 profile set of the bench kernels
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests/test_gpu_ref_suite.py -q -x 2>&1 | tail -5
tests/cpp/build/ref_suite_b200 > gpurun_out/ref_suite_b200.txt 2>&1; echo "ref_suite exit $?"
tests/cpp/build/acceptance_b200 > gpurun_out/acceptance_b200.txt 2>&1; echo "acceptance exit $?"
grep -E "FAILED|PASSED|tests ran" gpurun_out/ref_suite_b200.txt gpurun_out/acceptance_b200.txt | tail -30
timeout 900 python -m pytest tests/test_gpu_gmres.py tests/test_gpu_parity.py tests/test_gpu_nonlinear.py tests/test_gpu_dist.py -q 2>&1 | tail -5
timeout 300 tools/probe/btdb_probe > gpurun_out/btdb_probe.txt 2>&1; cat gpurun_out/btdb_probe.txt
timeout 600 python bench.py --steps 30 --warmup 5 > gpurun_out/bench_c.json 2> gpurun_out/bench_c.err
tail -3 gpurun_out/bench_c.err; cat gpurun_out/bench_c.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_r02c.csv python bench.py --steps 5 --warmup 3 --no-cpu --no-cg --e2e-steps 1 > gpurun_out/launches_r02c.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_stencil" -s 10 -c 2 \
  -o gpurun_out/prof_r02c -f python bench.py --steps 5 --warmup 3 --no-cpu --no-cg --e2e-steps 1 > gpurun_out/prof_r02c.log 2>&1
ls -la gpurun_out/

#!/bin/bash
# round 2, call D: per-file GPU test logs (a pytest process crashed in call C), the drop-in suites,
# the bench with the graph cache + two planes per barrier, and a profile of the new main kernel
mkdir -p gpurun_out
for f in test_gpu_gmres test_gpu_parity test_gpu_nonlinear test_gpu_dist test_gpu_stencil test_gpu_fullsize test_gpu_ref_suite; do
  timeout 900 python -X faulthandler -m pytest tests/$f.py -q -x > gpurun_out/pytest_$f.log 2>&1
  echo "$f exit $?: $(tail -1 gpurun_out/pytest_$f.log)"
done
tests/cpp/build/acceptance_b200 > gpurun_out/acceptance_b200.txt 2>&1; echo "acceptance exit $?"
timeout 600 python bench.py --steps 30 --warmup 5 > gpurun_out/bench_d.json 2> gpurun_out/bench_d.err
tail -3 gpurun_out/bench_d.err; cat gpurun_out/bench_d.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_stencil_tma" -s 10 -c 1 \
  -o gpurun_out/prof_r02d -f python bench.py --steps 5 --warmup 3 --no-cpu --no-cg --e2e-steps 1 > gpurun_out/prof_r02d.log 2>&1

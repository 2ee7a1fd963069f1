#!/bin/bash
# round 2, call L: round-end gate on the current build (whole GPU suite, smoke), the bench line, the
# launch list and one ncu --set full capture of the apply kernels
mkdir -p gpurun_out
timeout 1800 python -X faulthandler -m pytest tests -q -m gpu > gpurun_out/pytest_l_all.log 2>&1
echo "pytest -m gpu exit $?: $(tail -1 gpurun_out/pytest_l_all.log)"; grep -E "^FAILED|^ERROR" gpurun_out/pytest_l_all.log | head
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_l.log 2>&1; echo "smoke exit $?: $(tail -1 gpurun_out/smoke_l.log)"
timeout 900 python bench.py > gpurun_out/bench_l.json 2> gpurun_out/bench_l.err; tail -2 gpurun_out/bench_l.err; cut -c1-400 gpurun_out/bench_l.json
timeout 900 python bench.py --impl reference > gpurun_out/bench_l_ref.json 2> gpurun_out/bench_l_ref.err; cut -c1-300 gpurun_out/bench_l_ref.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_r02l.csv python bench.py --steps 5 --warmup 3 --no-cpu --no-cg --e2e-steps 1 > gpurun_out/launches_r02l.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_stencil" -s 20 -c 2 \
  -o gpurun_out/prof_r02l -f python bench.py --steps 5 --warmup 3 --no-cpu --no-cg --e2e-steps 1 > gpurun_out/prof_r02l.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"k_gm_pass|k_cg_update|k_cg_p" -c 6 \
  -o gpurun_out/prof_r02l_krylov -f python scripts/gmres_debug.py > gpurun_out/prof_r02l_krylov.log 2>&1

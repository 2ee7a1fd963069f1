#!/bin/bash
# round 2, final call: round-end gate on the current build (whole GPU suite, smoke), the bench line, the
# launch list and one ncu --set full capture of the apply kernels
mkdir -p gpurun_out
timeout 1800 python -X faulthandler -m pytest tests -q -m gpu > gpurun_out/pytest_fin_all.log 2>&1
echo "pytest -m gpu exit $?: $(tail -1 gpurun_out/pytest_fin_all.log)"; grep -E "^FAILED|^ERROR" gpurun_out/pytest_fin_all.log | head
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_fin.log 2>&1; echo "smoke exit $?: $(tail -1 gpurun_out/smoke_fin.log)"
timeout 900 python bench.py > gpurun_out/bench_fin.json 2> gpurun_out/bench_fin.err; tail -2 gpurun_out/bench_fin.err; cut -c1-400 gpurun_out/bench_fin.json
timeout 900 python bench.py --impl reference > gpurun_out/bench_fin_ref.json 2> gpurun_out/bench_fin_ref.err; cut -c1-300 gpurun_out/bench_fin_ref.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_r02fin.csv python bench.py --steps 5 --warmup 3 --no-cpu --no-cg --e2e-steps 1 > gpurun_out/launches_r02fin.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_stencil" -s 20 -c 2 \
  -o gpurun_out/prof_r02fin -f python bench.py --steps 5 --warmup 3 --no-cpu --no-cg --e2e-steps 1 > gpurun_out/prof_r02fin.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"k_gm_pass|k_cg_update|k_cg_p" -c 6 \
  -o gpurun_out/prof_r02fin_krylov -f python scripts/gmres_debug.py > gpurun_out/prof_r02fin_krylov.log 2>&1

#!/bin/bash
# round 2, call S (round-end gate of this session): corner-major element scratch A/B against the
# previous build (AFEM_LIBRARY=libafem_ab.so), whole GPU suite, smoke, bench lines (both arms), the
# bench launch list, and ncu of the config-3 element kernels at 128^3
mkdir -p gpurun_out
AB=paper_2604_22087_b200/libafem_ab.so
for i in 1 2; do
  echo "{\"build\": \"new\", \"c3\": $(timeout 600 python scripts/jvp_probe.py 2>&1 | tail -1), \"c4\": \"$(timeout 600 python scripts/c4_mf.py 256 2>&1 | tail -1)\"}"
  echo "{\"build\": \"previous\", \"c3\": $(AFEM_LIBRARY=$AB timeout 600 python scripts/jvp_probe.py 2>&1 | tail -1), \"c4\": \"$(AFEM_LIBRARY=$AB timeout 600 python scripts/c4_mf.py 256 2>&1 | tail -1)\"}"
done | tee gpurun_out/evlayout_s.jsonl
timeout 1800 python -X faulthandler -m pytest tests -q -m gpu > gpurun_out/pytest_s_all.log 2>&1
echo "pytest -m gpu exit $?: $(tail -1 gpurun_out/pytest_s_all.log)"; grep -E "^FAILED|^ERROR" gpurun_out/pytest_s_all.log | head
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_s.log 2>&1; echo "smoke exit $?: $(tail -1 gpurun_out/smoke_s.log)"
timeout 900 python bench.py > gpurun_out/bench_s.json 2> gpurun_out/bench_s.err; tail -2 gpurun_out/bench_s.err; cut -c1-300 gpurun_out/bench_s.json
timeout 900 python bench.py --impl reference > gpurun_out/bench_s_ref.json 2> gpurun_out/bench_s_ref.err; cut -c1-200 gpurun_out/bench_s_ref.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches_r02s.csv python bench.py --steps 5 --warmup 3 --no-cpu --no-cg --e2e-steps 1 > gpurun_out/launches_r02s.log 2>&1; echo "launch list exit $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_grid_elem|k_gather" -c 12 \
  -o gpurun_out/prof_s_nh -f python scripts/jvp_probe.py --n 128 --reps 2 > gpurun_out/prof_s_nh.log 2>&1; echo "nh ncu exit $?"

#!/bin/bash
# round 2, call U (final gate of this session): whole GPU suite + smoke on the build with p.Ap fused
# into the grid gathers (cached J2 and any-law grid operators), bench line
mkdir -p gpurun_out
timeout 1800 python -X faulthandler -m pytest tests -q -m gpu > gpurun_out/pytest_u_all.log 2>&1
echo "pytest -m gpu exit $?: $(tail -1 gpurun_out/pytest_u_all.log)"; grep -E "^FAILED|^ERROR" gpurun_out/pytest_u_all.log | head
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_u.log 2>&1; echo "smoke exit $?: $(tail -1 gpurun_out/smoke_u.log)"
timeout 900 python bench.py > gpurun_out/bench_u.json 2> gpurun_out/bench_u.err; tail -1 gpurun_out/bench_u.err; cut -c1-300 gpurun_out/bench_u.json

#!/bin/bash
# round 2, call M: whole GPU suite + smoke on the single-reduction slab CG build, the slab CG probe,
# and the bench lines (our arm, reference arm)
mkdir -p gpurun_out
timeout 1800 python -X faulthandler -m pytest tests -q -m gpu > gpurun_out/pytest_m_all.log 2>&1
echo "pytest -m gpu exit $?: $(tail -1 gpurun_out/pytest_m_all.log)"; grep -E "^FAILED|^ERROR" gpurun_out/pytest_m_all.log | head
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_m.log 2>&1; echo "smoke exit $?: $(tail -1 gpurun_out/smoke_m.log)"
timeout 900 python scripts/dist_cg_probe.py > gpurun_out/dist_cg_m.jsonl 2>&1; cat gpurun_out/dist_cg_m.jsonl
timeout 900 python bench.py > gpurun_out/bench_m.json 2> gpurun_out/bench_m.err; tail -2 gpurun_out/bench_m.err; cut -c1-400 gpurun_out/bench_m.json
timeout 900 python bench.py --impl reference > gpurun_out/bench_m_ref.json 2> gpurun_out/bench_m_ref.err; cut -c1-300 gpurun_out/bench_m_ref.json

#!/bin/bash
# round 2, call AC: interface corrections fused into the main kernel (computed from its staged
# planes) — parity tests on the default build, then full-apply / CG timings against the separate
# correction kernel (AFEM_STENCIL_NOFUSE=1), alternated
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_stencil.py tests/test_gpu_fullsize.py tests/test_gpu_dist.py -q -x > gpurun_out/pytest_ac.log 2>&1
echo "tests exit $?: $(tail -1 gpurun_out/pytest_ac.log)"; grep -E "^FAILED|^E  " gpurun_out/pytest_ac.log | head -8
for rep in 1 2; do
for v in fused nofuse; do
  env=""; [ $v = nofuse ] && env="AFEM_STENCIL_NOFUSE=1"
  env $env timeout 300 python bench.py --steps 40 --warmup 12 --no-cpu --e2e-steps 1 > gpurun_out/abac_${v}_$rep.json 2>gpurun_out/abac_${v}_$rep.err
  python -c "import json; d=json.loads(open('gpurun_out/abac_${v}_$rep.json').read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step']*1e3,2), 'us', round(d['value']/1e9,2), 'GDOF/s cg', round(d['cg']['solve_s'],3), d['cg']['iterations'], d['cg']['true_rel_residual'])"
  env $env AFEM_STENCIL_ONLY=main timeout 300 python bench.py --steps 40 --warmup 12 --no-cpu --no-cg --e2e-steps 1 > gpurun_out/abac_${v}_main$rep.json 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/abac_${v}_main$rep.json').read().strip().splitlines()[-1]); print('$v main only', round(d['ms_per_step']*1e3,2), 'us')"
done
done

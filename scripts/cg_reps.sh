# CG solve-time spread at 128^3 (cg_probe: 3 reps per process, 3 processes)
for i in 1 2 3; do python scripts/cg_probe.py 128 2>&1 | grep rep; done

#!/usr/bin/env python
"""Config-4 Jacobi-PCG on the matrix-free cached-tangent J2 operator (256^3 by default) at a plastic
state: iterations and ms per CG iteration (the loop C4's load stepping spends its time in).
usage: python scripts/c4_cg_probe.py [n] [max_iter]"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_22087_b200 as afem  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
max_iter = int(sys.argv[2]) if len(sys.argv) > 2 else 3000
ctx = afem.Context(0, stream=torch.cuda.current_stream())
s = afem.System.grid(ctx, 3, n, n, n, inclusions=afem.fibres(12345, 40), radius=0.05,
                     materials=[(afem.J2, 1.0, 0.3, 0.002, 0.1), (afem.LINEAR, 10.0, 0.3)])
s.set_benchmark_dirichlet(0.012)
coords = s.mesh()[0].reshape(-1)
ua = np.zeros(s.n)
ua[0::3] = 0.01 * coords[0::3]
s.commit_history(ua)  # a plastic history
ua[0::3] = 0.012 * coords[0::3]
u = s.impose_dirichlet(ua)
op = afem.matrix_free_operator(s, u)
b = -s.constrain_residual(s.residual(u), u)
out = dict(n=n, n_dof=s.n)
for rep in range(2):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    x, r = afem.run_solver(op, b, method=afem.CG, precond=afem.JACOBI, rtol=1e-30, max_iter=max_iter)
    dt = time.perf_counter() - t0
    out[f"run{rep}"] = dict(iterations=r["iterations"], s=dt, ms_per_iteration=dt / r["iterations"] * 1e3,
                            final_rel_residual=float(r["residual_history"][-1]))
print(json.dumps(out), flush=True)

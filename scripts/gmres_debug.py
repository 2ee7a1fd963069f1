"""Debug: GMRES iteration counts on a small 3D matrix-free system under the fused / MGS Arnoldi
and with / without the apply graph cache (env switches are read once per process: run once per
combination). usage: python scripts/gmres_debug.py"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SNIP = r"""
import sys, json, numpy as np
sys.path.insert(0, %r)
import paper_2604_22087_b200 as afem
ctx = afem.Context(0)
out = {}
for (nx, ny, nz) in ((10, 8, 6), (16, 8, 12)):
    s = afem.System.grid(ctx, 3, nx, ny, nz, inclusions=afem.fibres(12345, 4), radius=0.2,
                         materials=[(0, 1.0, 0.3), (0, 3.0, 0.3)])
    s.set_benchmark_dirichlet(0.01)
    u = s.impose_dirichlet(np.zeros(s.n))
    op = afem.matrix_free_operator(s, u)
    b = -s.constrain_residual(s.residual(u), u)
    for restart in (5, 30):
        x, rep = afem.run_solver(op, b, method=afem.GMRES, precond=afem.JACOBI, rtol=1e-10, restart=restart, max_iter=3000)
        h = rep["residual_history"]
        out[f"{nx}x{ny}x{nz} r{restart}"] = [rep["converged"], rep["iterations"], float(h[-1]), [float(v) for v in h[:8]], op.uses_stencil]
    xc, rc = afem.run_solver(op, b, method=afem.CG, precond=afem.JACOBI, rtol=1e-10)
    out[f"{nx}x{ny}x{nz} cg"] = [rc["converged"], rc["iterations"]]
print(json.dumps(out))
""" % ROOT
for env in ({}, {"AFEM_GMRES_MGS": "1"}, {"AFEM_NO_APPLY_GRAPH": "1"}, {"AFEM_GMRES_MGS": "1", "AFEM_NO_APPLY_GRAPH": "1"}):
    e = dict(os.environ)
    e.update(env)
    p = subprocess.run([sys.executable, "-c", SNIP], capture_output=True, text=True, env=e, timeout=600)
    print(env, p.stdout.strip()[-3000:], p.stderr[-2000:])

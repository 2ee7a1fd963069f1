#!/usr/bin/env python
"""GMRES(30)+Jacobi cost per iteration on config 3's first Newton system (NH 192^3, assembled CSR
tangent, 21.6 M dofs): the fused CGS2 Arnoldi step against the MGS kernels (AFEM_GMRES_MGS=1, run in a
subprocess because the switch is read once per process). Prints one JSON line per variant.
usage: python scripts/gmres_c3.py [--n 192] [--iters 300]"""
import argparse
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run_one(n, iters):
    sys.path.insert(0, ROOT)
    import numpy as np
    import paper_2604_22087_b200 as afem
    ctx = afem.Context(0)
    mats = [(afem.NEOHOOKE, 1.0, 0.3), (afem.LINEAR, 10.0, 0.3)]
    s = afem.System.grid(ctx, 3, n, n, n, inclusions=afem.fibres(12345, 40), radius=0.05, materials=mats)
    s.set_benchmark_dirichlet(0.05)
    c = s.mesh()[0]
    u = np.zeros_like(c)
    u[0::3] = 0.05 * c[0::3]
    u = s.impose_dirichlet(u)
    vals = afem.Values(s)
    vals.assemble(u)
    r = vals.eliminate(s.residual(u), u)
    buf = afem.HandoffBuffer(s)
    buf.handoff(vals)
    op = afem.explicit_operator(buf)
    b = -r
    afem.run_solver(op, b, method=afem.GMRES, precond=afem.JACOBI, rtol=1e-12, max_iter=31, restart=30)  # warm-up
    ctx.synchronize()
    t = time.perf_counter()
    _, rep = afem.run_solver(op, b, method=afem.GMRES, precond=afem.JACOBI, rtol=1e-12, max_iter=iters, restart=30)
    dt = time.perf_counter() - t
    return dict(n=n, n_dof=s.n, iterations=rep["iterations"], time_s=dt, ms_per_iteration=1e3 * dt / rep["iterations"],
                final_rres=float(rep["residual_history"][-1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=192)
    ap.add_argument("--iters", type=int, default=300)
    ap.add_argument("--child", action="store_true")
    a = ap.parse_args()
    if a.child:
        print(json.dumps(run_one(a.n, a.iters)))
        return
    for mgs in (False, True, False, True):  # alternated: the box's power state drifts over a run
        env = dict(os.environ)
        env.pop("AFEM_GMRES_MGS", None)
        if mgs:
            env["AFEM_GMRES_MGS"] = "1"
        p = subprocess.run([sys.executable, __file__, "--child", "--n", str(a.n), "--iters", str(a.iters)],
                           capture_output=True, text=True, env=env)
        rec = json.loads(p.stdout.strip().splitlines()[-1]) if p.returncode == 0 else {"error": p.stderr[-500:]}
        rec["arnoldi"] = "MGS (kernel by kernel)" if mgs else "fused CGS2 (3 passes)"
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()

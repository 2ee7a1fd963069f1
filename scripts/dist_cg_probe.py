#!/usr/bin/env python
"""Slab CG (dist.cu dist_solve: single-reduction Jacobi-PCG, one allreduce per iteration) against
the single-GPU CG on the bench workload (128^3, 40 fibres), at NCCL world size 1 on one B200:
iterations, wall seconds, ms and kernel launches per iteration, agreement of x. A second child
forces the N > 1 apply schedule (AFEM_DIST_FORCE_PIECES=1: shared planes as one-plane launches on
a second stream, interior wave, halo kernel; the dot falls back to the owned-dot kernel) to show a
middle rank's per-iteration cost without peers. usage: python scripts/dist_cg_probe.py [--n 128]"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import sys, json, numpy as np, torch
sys.path.insert(0, %r)
import paper_2604_22087_b200 as afem
n = %d
torch.cuda.set_device(0)
ctx = afem.Context(0)
fib = afem.fibres(12345, 40)
mats = [(0, 1.0, 0.3), (0, 10.0, 0.3)]
s = afem.System.grid(ctx, 3, n, n, n, inclusions=fib, radius=0.05, materials=mats)
s.set_benchmark_dirichlet(0.01)
u0 = s.impose_dirichlet(np.zeros(s.n))
op = afem.matrix_free_operator(s, u0)
b = -s.constrain_residual(s.residual(u0), u0)
d = afem.Dist(ctx, 0, 1, backend="nccl", uid=afem.nccl_unique_id())
ss, _ = afem.slab_system(ctx, n, n, n, 0, 1, inclusions=fib, radius=0.05, materials=mats)
d.set_benchmark_dirichlet(ss, 0.01)
dop = d.matrix_free_operator(ss, ss.impose_dirichlet(np.zeros(ss.n)))
out = dict(n=n, n_dof=s.n, schedule=%r)
xs = {}
for name, solve in (("single_gpu_cg", lambda: afem.run_solver(op, b, method=afem.CG, precond=afem.JACOBI,
                                                              rtol=1e-8, max_iter=20000)),
                    ("slab_cg", lambda: d.run_solver(dop, b, method=afem.CG, precond=afem.JACOBI, rtol=1e-8,
                                                     max_iter=20000))):
    solve()  # warm-up (graph capture, allocations)
    l0 = ctx.launches
    x, rep = solve()
    it = rep["iterations"]
    out[name] = dict(iterations=it, converged=rep["converged"], wall_s=rep["wall_time"],
                     ms_per_iteration=rep["wall_time"] / it * 1e3, launches_per_iteration=(ctx.launches - l0) / it,
                     true_rel_residual=float(np.linalg.norm(b - op.apply(x)) / np.linalg.norm(b)))
    xs[name] = x
out["x_rel_diff"] = float(np.abs(xs["slab_cg"] - xs["single_gpu_cg"]).max() / np.abs(xs["single_gpu_cg"]).max())
print(json.dumps(out))
"""


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=128)
    a = ap.parse_args()
    for sched, extra in (("world1", {}), ("forced_pieces", {"AFEM_DIST_FORCE_PIECES": "1"})):
        env = dict(os.environ, **extra)
        p = subprocess.run([sys.executable, "-c", CHILD % (ROOT, a.n, sched)], capture_output=True, text=True, env=env)
        print(p.stdout.strip() or p.stderr[-2000:], flush=True)


if __name__ == "__main__":
    main()

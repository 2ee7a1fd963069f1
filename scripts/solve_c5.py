#!/usr/bin/env python
"""The north-star target solve on one B200: config 5's linear hex8 fibre RVE at N = 321 (100.2 M
dofs; 40 z-parallel fibres of radius 0.05 from mt19937_64(12345), E 1 / 10, nu 0.3, benchmark BCs at
1 % strain), matrix-free (structured stencil) Jacobi-PCG to rtol 1e-8 with the reference's
true-residual re-verification (krylov.hpp:350-408).

Prints one JSON line: build/setup times, solve time (CUDA events on the context stream), CG
iterations, the solver's reported true relative residual and an independent re-check
||b - A x|| / ||b|| (a fresh apply), clocks sampled during the solve, and the per-iteration cost.
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2604_22087_b200 as afem  # noqa: E402
from bench import ClockSampler  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=321)
    ap.add_argument("--rtol", type=float, default=1e-8)
    ap.add_argument("--max-iter", type=int, default=100000)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    n = a.n
    stream = torch.cuda.current_stream()
    ctx = afem.Context(0, stream=stream)
    t0 = time.perf_counter()
    fib = afem.fibres(12345, 40)
    s = afem.System.grid(ctx, 3, n, n, n, inclusions=fib, radius=0.05,
                         materials=[(afem.LINEAR, 1.0, 0.3), (afem.LINEAR, 10.0, 0.3)])
    s.set_benchmark_dirichlet(0.01)
    u0 = s.impose_dirichlet(np.zeros(s.n))
    ctx.synchronize()
    t_sys = time.perf_counter() - t0
    t0 = time.perf_counter()
    op = afem.matrix_free_operator(s, u0)
    ctx.synchronize()
    t_op = time.perf_counter() - t0
    assert op.uses_stencil
    b = -torch.from_numpy(s.constrain_residual(s.residual(u0), u0)).cuda()
    clk = ClockSampler(0, period_ms=500)
    clk.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    e0.record(stream)
    x, rep = afem.run_solver(op, b, method=afem.CG, precond=afem.JACOBI, rtol=a.rtol, max_iter=a.max_iter)
    e1.record(stream)
    torch.cuda.synchronize()
    wall = time.perf_counter() - w0
    solve_s = e0.elapsed_time(e1) * 1e-3
    clocks = clk.stop()
    xd = torch.as_tensor(x).cuda() if not isinstance(x, torch.Tensor) else x
    y = torch.empty_like(b)
    op.apply_device(xd.data_ptr(), y.data_ptr())
    torch.cuda.synchronize()
    true_rres = float(torch.linalg.norm(b - y) / torch.linalg.norm(b))
    vf = float(s.mesh()[2].mean()) if n <= 200 else None
    rec = {
        "what": "C5 north-star solve, 1 GPU", "n": n, "n_dof": s.n, "n_elem": s.info.n_elem, "nnz_K": s.nnz,
        "fibres": 40, "radius": 0.05, "E": [1.0, 10.0], "nu": 0.3, "strain": 0.01,
        "fibre_volume_fraction": vf, "operator": "matrix-free structured stencil",
        "method": "CG", "precond": "jacobi", "rtol": a.rtol, "converged": rep["converged"],
        "iterations": rep["iterations"], "solve_s": solve_s, "solve_wall_s": wall,
        "ms_per_iteration": 1e3 * solve_s / max(rep["iterations"], 1),
        "reported_true_rel_residual": float(rep["residual_history"][-1]), "recheck_true_rel_residual": true_rres,
        "failure": rep.get("failure", ""), "setup_s": {"system": t_sys, "operator": t_op},
        "device_gb": round(s.info.device_bytes / 1e9, 2), "clocks": clocks, "dtype": "f64", "data": "synthetic",
    }
    line = json.dumps(rec)
    print(line, flush=True)
    if a.out:
        with open(a.out, "a") as f:
            f.write(line + "\n")


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Measurements for BASELINE.json configs 3 and 4 on one B200 (bench.py covers config 2).

  C3  3D Neo-Hookean hex8 RVE N^3 (default 192): matrix Neo-Hookean E=1 nu=0.3, fibres linear
      E=10; Newton-Krylov with the assembled CSR tangent. GMRES(30)+Jacobi stagnates on this 10:1
      contrast RVE (in the CPU restatement as on the GPU: profiles/r01_configs.json), so the solve
      uses Jacobi-PCG on the symmetric Neo-Hookean tangent; GMRES cost per iteration is reported.
  C4  3D J2 hex8 RVE N^3 (default 256): matrix J2 (E=1, nu=0.3, sigma_y=0.002, H=0.1), fibres
      linear E=10; quadrature-point history resident in HBM; strain ramped to 0.02 in 10 steps.

Per config at full size it times every hot-path kernel through the C ABI with device buffers
(torch allocations, CUDA events on the context stream, min over reps): residual, tangent
assembly (CSR values), Dirichlet elimination, CSR SpMV, matrix-free JVP, Jacobi diagonal,
history commit. Then it runs the complete nonlinear solve at a reduced size (--solve-n) on the
GPU and the same solve on the CPU restatement (oracle/, 1 thread) for the speed-up line.
Prints one JSON object per config.
"""
import argparse
import ctypes as C
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2604_22087_b200 as afem  # noqa: E402

SEED, N_FIBRES, RADIUS = 12345, 40, 0.05
CONFIGS = {
    3: dict(mats=[(afem.NEOHOOKE, 1.0, 0.3), (afem.LINEAR, 10.0, 0.3)], strain=0.05, steps=1, n=192,
            workload="C3 hex8 Neo-Hookean RVE, Newton + assembled CSR tangent + GMRES(30)/Jacobi"),
    4: dict(mats=[(afem.J2, 1.0, 0.3, 0.002, 0.1), (afem.LINEAR, 10.0, 0.3)], strain=0.02, steps=10, n=256,
            workload="C4 hex8 J2 RVE, quadrature-point history in HBM, 10 load steps"),
}


def timed(fn, reps, stream):
    best = float("inf")
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fn()
        b.record(stream)
        b.synchronize()
        best = min(best, a.elapsed_time(b) * 1e-3)
    return best


def kernels(cfg, n, reps):
    L = afem.load()
    ctx = afem.Context(0)
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream.cuda_stream)
    fib = afem.fibres(SEED, N_FIBRES)
    s = afem.System.grid(ctx, 3, n, n, n, inclusions=fib, radius=RADIUS, materials=cfg["mats"])
    s.set_benchmark_dirichlet(cfg["strain"] / cfg["steps"])
    nd, nnz, ne = s.n, s.nnz, s.info.n_elem
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(1)
    u = (torch.rand(nd, dtype=torch.float64, device=dev, generator=g) - 0.5) * (0.02 / n)
    x = torch.rand(nd, dtype=torch.float64, device=dev, generator=g) - 0.5
    r = torch.empty_like(u)
    y = torch.empty_like(u)
    d = torch.empty_like(u)
    vals = torch.empty(nnz, dtype=torch.float64, device=dev)
    P = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
    ck = afem._check
    out = dict(n=n, n_dof=nd, n_elem=ne, nnz=nnz, device_gb=round(s.info.device_bytes / 1e9, 2))
    if s.history_size():
        ck(L.afem_history_commit(s.h, P(u * 0.5)))
        out["history_gb"] = round(s.history_size() * 8 / 1e9, 2)
    out["residual_ms"] = timed(lambda: ck(L.afem_residual(s.h, P(u), P(r))), reps, stream) * 1e3
    out["diagonal_ms"] = timed(lambda: ck(L.afem_diagonal(s.h, P(u), P(d))), reps, stream) * 1e3
    out["jacobian_ms"] = timed(lambda: ck(L.afem_jacobian(s.h, P(u), P(vals))), reps, stream) * 1e3
    rr = r.clone()
    out["eliminate_ms"] = timed(lambda: ck(L.afem_eliminate(s.h, P(vals), P(rr), P(u))), 1, stream) * 1e3
    out["csr_spmv_ms"] = timed(lambda: ck(L.afem_csr_apply(s.h, P(vals), P(x), P(y))), reps, stream) * 1e3
    # bytes our CSR layout moves: fp64 values + node-level int32 columns (nnz/9 for dim 3) + the
    # int64 node row pointers + x and y; SURVEY §8(d)'s dof-level formula (12 nnz + 8 n + 16 n) alongside
    out["csr_spmv_gbs"] = (8 * nnz + 4 * nnz / 9 + 8 * nd / 3 + 16 * nd) / (out["csr_spmv_ms"] * 1e-3) / 1e9
    out["csr_spmv_gbs_survey_bytes"] = (12 * nnz + 24 * nd) / (out["csr_spmv_ms"] * 1e-3) / 1e9
    # one bounded GMRES(30)+Jacobi and CG+Jacobi run on the eliminated tangent (cost per iteration)
    buf, hv = C.c_void_p(), C.c_void_p()
    ck(L.afem_buffer_create(s.h, C.byref(buf)))
    ck(L.afem_values_create(s.h, C.byref(hv)))
    ck(L.afem_values_set(hv, P(vals)))
    ck(L.afem_buffer_handoff(buf, C.byref(hv)))
    eop = C.c_void_p()
    ck(L.afem_op_create_explicit(buf, C.byref(eop)))
    del vals
    torch.cuda.empty_cache()
    xs = torch.zeros_like(u)
    for name, meth in (("gmres30", afem.GMRES), ("cg", afem.CG)):
        cfgs = afem.afem_solver_cfg(meth, afem.JACOBI, 1e-30, 200, 30)
        rep = afem.afem_solve_report()
        t0 = time.perf_counter()
        ck(L.afem_solve(eop, C.byref(cfgs), P(rr), None, P(xs), C.byref(rep), None, 0))
        dt = time.perf_counter() - t0
        out[f"{name}_ms_per_iteration"] = dt / max(rep.iterations, 1) * 1e3
    ck(L.afem_op_destroy(eop))
    ck(L.afem_buffer_release(buf))
    ck(L.afem_buffer_destroy(buf))
    op = C.c_void_p()
    ck(L.afem_op_create_mf(s.h, P(u), C.byref(op)))
    out["mf_apply_ms"] = timed(lambda: ck(L.afem_op_apply_async(op, P(x), P(y))), reps, stream) * 1e3
    out["mf_dof_per_s"] = nd / (out["mf_apply_ms"] * 1e-3)
    ck(L.afem_op_destroy(op))
    if s.history_size():
        out["history_commit_ms"] = timed(lambda: ck(L.afem_history_commit(s.h, P(u))), reps, stream) * 1e3
    return out


def affine(coords, strain):
    """Uniaxial predictor u = strain * x e_x (satisfies the benchmark BCs; warm start x0)."""
    u = np.zeros_like(coords)
    u[0::3] = strain * coords[0::3]
    return u


def solve_small(cfg, n, cfgno, cpu):
    """The complete nonlinear solve at N^3: C3 one Newton solve, C4 the incremental load path with a
    history commit after every converged step. Warm start: the uniaxial affine predictor (the
    reference's BC-consistent zero start puts the whole applied displacement into the last element
    layer, strain * N, which inverts elements at these sizes)."""
    from oracle.pyoracle import Oracle
    ctx = afem.Context(0)
    fib = afem.fibres(SEED, N_FIBRES)
    s = afem.System.grid(ctx, 3, n, n, n, inclusions=fib, radius=RADIUS, materials=cfg["mats"])
    coords = s.mesh()[0]
    kw = dict(rtol=1e-10, lin_rtol=1e-12, lin_max_iter=200000, operator_kind=afem.EXPLICIT, method=afem.CG)
    steps, strain = cfg["steps"], cfg["strain"]

    def run(set_bcs, solve, commit):
        u = np.zeros(3 * (n + 1) ** 3)
        its, lin, ok = [], 0, True
        for st in range(1, steps + 1):
            set_bcs(strain * st / steps)
            u, rep = solve(u + affine(coords, strain / steps))
            its.append(int(rep["iterations"]))
            lin += int(rep["total_linear_iterations"])
            if not rep["converged"]:
                ok = False
                break
            commit(u)
        return u, its, lin, ok

    t = time.perf_counter()
    u, its, lin, ok = run(s.set_benchmark_dirichlet, lambda x0: s.solve_bvp(x0=x0, **kw),
                          s.commit_history if s.history_size() else (lambda u: None))
    res = dict(n=n, n_dof=s.n, gpu_s=time.perf_counter() - t, converged=ok, newton_iterations=its,
               linear_iterations=lin)
    if cpu:
        o = Oracle("restate")
        coords_, conn, phase = s.mesh()
        os_ = o.system(3, coords_, conn, phase, cfg["mats"], grid=(n, n, n, 1.0, 1.0, 1.0))
        t = time.perf_counter()
        uo, ito, lino, oko = run(lambda e: os_.set_dirichlet(*o.bcs(3, n, n, n, 1.0, e)),
                                 lambda x0: os_.solve_bvp(x0=x0, **kw),
                                 os_.commit_history if cfgno == 4 else (lambda u: None))
        res.update(cpu_s=time.perf_counter() - t, cpu_newton_iterations=ito, cpu_linear_iterations=lino,
                   cpu_converged=oko, cpu_cores=1, cpu_kind="port (oracle/restate.hpp, single thread)",
                   rel_diff_u=float(np.abs(u - uo).max() / np.abs(uo).max()))
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="3,4")
    ap.add_argument("--n", type=int, default=0, help="override the full size")
    ap.add_argument("--solve-n", type=int, default=16, help="size of the GPU-vs-CPU solve")
    ap.add_argument("--big-n", type=int, default=64, help="size of the GPU-only full solve (0: skip)")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--no-cpu", action="store_true")
    a = ap.parse_args()
    for c in map(int, a.configs.split(",")):
        cfg = CONFIGS[c]
        rec = dict(config=c, workload=cfg["workload"], dtype="f64", data="synthetic")
        rec["kernels"] = kernels(cfg, a.n or cfg["n"], a.reps)
        torch.cuda.empty_cache()
        rec["solve"] = solve_small(cfg, a.solve_n, c, not a.no_cpu)
        if a.big_n:
            rec["solve_gpu_only"] = solve_small(cfg, a.big_n, c, False)
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()

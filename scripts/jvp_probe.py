#!/usr/bin/env python
"""Config-3 element-centric kernels at full size (192^3 Neo-Hookean matrix + linear fibres): the
residual, the matrix-free JVP (k_grid_elem* + k_gather) and the assembled CSR SpMV they are
compared with. One JSON line. Device buffers, CUDA events on the context stream, min over reps.
profiles/r02_jvp_lean_ab.jsonl: the A/B of a shared-memory u_e / x_e element kernel ("lean",
168 registers, 3 CTAs per SM) against the register-resident one (255 registers, 2 CTAs per SM,
AFEM_ELEM_REGS=1 in that build): 3.80 vs 3.61 ms, rejected."""
import argparse
import ctypes as C
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2604_22087_b200 as afem  # noqa: E402
from scripts.bench_configs import CONFIGS, N_FIBRES, RADIUS, SEED, timed  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=192)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--spmv", action="store_true", help="also time the tangent assembly and the CSR SpMV")
    a = ap.parse_args()
    L = afem.load()
    ctx = afem.Context(0)
    stream = torch.cuda.current_stream()
    ctx.set_stream(stream.cuda_stream)
    cfg = CONFIGS[3]
    n = a.n
    s = afem.System.grid(ctx, 3, n, n, n, inclusions=afem.fibres(SEED, N_FIBRES), radius=RADIUS,
                         materials=cfg["mats"])
    s.set_benchmark_dirichlet(cfg["strain"])
    nd = s.n
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(1)
    u = (torch.rand(nd, dtype=torch.float64, device=dev, generator=g) - 0.5) * (0.02 / n)
    x = torch.rand(nd, dtype=torch.float64, device=dev, generator=g) - 0.5
    r, y = torch.empty_like(u), torch.empty_like(u)
    P = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
    ck = afem._check
    out = dict(n=n, n_dof=nd)
    out["residual_ms"] = timed(lambda: ck(L.afem_residual(s.h, P(u), P(r))), a.reps, stream) * 1e3
    op = C.c_void_p()
    ck(L.afem_op_create_mf(s.h, P(u), C.byref(op)))
    out["mf_jvp_ms"] = timed(lambda: ck(L.afem_op_apply_async(op, P(x), P(y))), a.reps, stream) * 1e3
    torch.cuda.synchronize()
    out["jvp_checksum"] = float(y.abs().sum())
    out["residual_checksum"] = float(r.abs().sum())
    ck(L.afem_op_destroy(op))
    if a.spmv:
        vals = torch.empty(s.nnz, dtype=torch.float64, device=dev)
        out["jacobian_ms"] = timed(lambda: ck(L.afem_jacobian(s.h, P(u), P(vals))), 3, stream) * 1e3
        out["jacobian_checksum"] = float(vals.abs().sum())
        out["csr_spmv_ms"] = timed(lambda: ck(L.afem_csr_apply(s.h, P(vals), P(x), P(y))), a.reps, stream) * 1e3
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()

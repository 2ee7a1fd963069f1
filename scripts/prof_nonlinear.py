"""One call of every nonlinear-path kernel on a C4-shaped (J2 + linear fibres) grid, for ncu.

usage: python scripts/prof_nonlinear.py N   (run under ncu --set full; timings here are not measurements)
"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2604_22087_b200 as afem

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
L = afem.load()
ctx = afem.Context(0)
fib = afem.fibres(12345, 40)
s = afem.System.grid(ctx, 3, n, n, n, inclusions=fib, radius=0.05,
                     materials=[(afem.J2, 1.0, 0.3, 0.002, 0.1), (afem.LINEAR, 10.0, 0.3)])
s.set_benchmark_dirichlet(0.002)
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(1)
u = (torch.rand(s.n, dtype=torch.float64, device=dev, generator=g) - 0.5) * (0.02 / n)
x = torch.rand(s.n, dtype=torch.float64, device=dev, generator=g) - 0.5
r, y, d = torch.empty_like(u), torch.empty_like(u), torch.empty_like(u)
P = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
ck = afem._check
ck(L.afem_history_commit(s.h, P(u * 0.5)))
ck(L.afem_residual(s.h, P(u), P(r)))
ck(L.afem_diagonal(s.h, P(u), P(d)))
vals = torch.empty(s.nnz, dtype=torch.float64, device=dev)
ck(L.afem_jacobian(s.h, P(u), P(vals)))
ck(L.afem_eliminate(s.h, P(vals), P(r), P(u)))
ck(L.afem_csr_apply(s.h, P(vals), P(x), P(y)))
buf, hv, eop = C.c_void_p(), C.c_void_p(), C.c_void_p()
ck(L.afem_buffer_create(s.h, C.byref(buf)))
ck(L.afem_values_create(s.h, C.byref(hv)))
ck(L.afem_values_set(hv, P(vals)))
ck(L.afem_buffer_handoff(buf, C.byref(hv)))
ck(L.afem_op_create_explicit(buf, C.byref(eop)))
cfg = afem.afem_solver_cfg(afem.CG, afem.JACOBI, 1e-30, 3, 30)
rep = afem.afem_solve_report()
ck(L.afem_solve(eop, C.byref(cfg), P(r), None, P(y), C.byref(rep), None, 0))
op = C.c_void_p()
ck(L.afem_op_create_mf(s.h, P(u), C.byref(op)))
ck(L.afem_op_apply_async(op, P(x), P(y)))
ctx.synchronize()
print("done", s.n)

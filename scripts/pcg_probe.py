"""Config-1 explicit Jacobi-PCG (rtol 1e-8) solve time on the device: chunked launches vs the
persistent cooperative kernel (AFEM_NO_PERSISTENT_CG / AFEM_PCG_BLOCKS set by the caller)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2604_22087_b200 as afem

ctx = afem.Context(0)
s = afem.System.grid(ctx, 2, 64, 64, materials=[(0, 1.0, 0.3), (0, 10.0, 0.3)])
s.set_benchmark_dirichlet(0.01)
u = s.impose_dirichlet(np.zeros(s.n))
v = afem.Values(s)
v.assemble(u)
r = s.residual(u)
r = v.eliminate(r, u)
buf = afem.HandoffBuffer(s)
buf.handoff(v)
op = afem.explicit_operator(buf)
best = 1e9
for _ in range(5):
    t = time.perf_counter()
    x, rep = afem.run_solver(op, -r, method=afem.CG, precond=afem.JACOBI, rtol=1e-8)
    best = min(best, time.perf_counter() - t)
print(os.environ.get("AFEM_NO_PERSISTENT_CG", "persistent"), os.environ.get("AFEM_PCG_BLOCKS", "-"),
      f"{best*1e3:.2f} ms, {rep['iterations']} it, {best*1e6/rep['iterations']:.1f} us/it, rres {rep['residual_history'][-1]:.2e}")

"""Time the C2 Jacobi-PCG solve several times (device buffers) and report per-iteration cost."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_22087_b200 as afem  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 128
ctx = afem.Context(0, stream=torch.cuda.current_stream())
s = afem.System.grid(ctx, 3, n, n, n, inclusions=afem.fibres(12345, 40), radius=0.05,
                     materials=[(0, 1.0, 0.3), (0, 10.0, 0.3)])
s.set_benchmark_dirichlet(0.01)
u0 = s.impose_dirichlet(np.zeros(s.n))
op = afem.matrix_free_operator(s, u0)
b = -torch.from_numpy(s.constrain_residual(s.residual(u0), u0)).cuda()
for rep in range(3):
    torch.cuda.synchronize()
    l0 = ctx.launches
    t0 = time.perf_counter()
    x, r = afem.run_solver(op, b, method=afem.CG, precond=afem.JACOBI, rtol=1e-8, max_iter=20000)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"rep {rep}: {dt:.3f} s  it={r['iterations']}  {1e3 * dt / r['iterations']:.3f} ms/it  "
          f"launches={ctx.launches - l0} wall_time={r['wall_time']:.3f} rres={r['residual_history'][-1]:.2e}",
          flush=True)

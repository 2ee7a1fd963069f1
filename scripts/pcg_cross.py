"""Per-iteration cost of assembled Jacobi-PCG, persistent cooperative kernel vs the chunked launch
path, across sizes (sets AFEM_NO_PERSISTENT_CG per child process). usage: python scripts/pcg_cross.py"""
import os
import subprocess
import sys
import time

if len(sys.argv) > 1:
    n = int(sys.argv[1])
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import numpy as np
    import torch
    import paper_2604_22087_b200 as afem
    ctx = afem.Context(0)
    s = afem.System.grid(ctx, 3, n, n, n, inclusions=afem.fibres(12345, 40), radius=0.05,
                         materials=[(0, 1.0, 0.3), (0, 10.0, 0.3)])
    s.set_benchmark_dirichlet(0.01)
    u0 = s.impose_dirichlet(np.zeros(s.n))
    vals = afem.Values(s).assemble(u0)
    rhs = vals.eliminate(s.residual(u0), u0)
    buf = afem.HandoffBuffer(s)
    buf.handoff(vals)
    op = afem.explicit_operator(buf)
    b = -torch.as_tensor(np.asarray(rhs)).cuda()
    best = 1e9
    for rep in range(3):
        torch.cuda.synchronize()
        t = time.perf_counter()
        x, r = afem.run_solver(op, b, method=afem.CG, precond=afem.JACOBI, rtol=1e-8, max_iter=100000)
        torch.cuda.synchronize()
        best = min(best, (time.perf_counter() - t) / r["iterations"])
    print(f"n={n} dofs={s.n} its={r['iterations']} us/it={best * 1e6:.1f}", flush=True)
else:
    for n in (16, 24, 32, 48, 64, 96):
        for off in (0, 1):
            env = dict(os.environ)
            if off:
                env["AFEM_NO_PERSISTENT_CG"] = "1"
            out = subprocess.run([sys.executable, __file__, str(n)], env=env, capture_output=True, text=True)
            print("chunked   " if off else "persistent", out.stdout.strip() or out.stderr[-300:], flush=True)

"""C4 at a reduced size: explicit-operator Newton + CG load path (bench_configs' solve_gpu_only),
timed per load step. usage: python scripts/c4_probe.py [N] [ROOT]"""
import os
import subprocess
import sys
import time

import numpy as np

n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
root = sys.argv[2] if len(sys.argv) > 2 else os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, root)
import paper_2604_22087_b200 as afem  # noqa: E402

print("lib", afem.__file__)
ctx = afem.Context(0)
mats = [(afem.J2, 1.0, 0.3, 0.002, 0.1), (afem.LINEAR, 10.0, 0.3)]
s = afem.System.grid(ctx, 3, n, n, n, inclusions=afem.fibres(12345, 40), radius=0.05, materials=mats)
coords = s.mesh()[0]
kw = dict(rtol=1e-10, lin_rtol=1e-12, lin_max_iter=200000, operator_kind=afem.EXPLICIT, method=afem.CG)
u = np.zeros(s.n)
for st in range(1, 4):
    s.set_benchmark_dirichlet(0.02 * st / 10)
    pred = np.zeros(s.n)
    pred[0::3] = 0.002 * coords[0::3]
    t = time.perf_counter()
    u, rep = s.solve_bvp(x0=u + pred, **kw)
    dt = time.perf_counter() - t
    s.commit_history(u)
    li = rep["total_linear_iterations"]
    clk = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks_throttle_reasons.active", "--format=csv,noheader"],
                         capture_output=True, text=True).stdout.strip()
    print(f"step {st}: {dt:.3f} s newton={rep['iterations']} lin={li} {1e6 * dt / max(li, 1):.1f} us/lin-it clk={clk}",
          flush=True)

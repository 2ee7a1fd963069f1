"""Tangent assembly (CSR values) on a C3-type grid: time per assembly. usage: python scripts/jac_probe.py [N] [reps]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_22087_b200 as afem  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
ctx = afem.Context(0)
for name, mats in (("NH", [(afem.NEOHOOKE, 1.0, 0.3), (afem.LINEAR, 10.0, 0.3)]),
                   ("J2", [(afem.J2, 1.0, 0.3, 0.002, 0.1), (afem.LINEAR, 10.0, 0.3)])):
    s = afem.System.grid(ctx, 3, n, n, n, inclusions=afem.fibres(12345, 40), radius=0.05, materials=mats)
    coords = s.mesh()[0]
    u = np.zeros(s.n)
    u[0::3] = 0.01 * coords[0::3]
    u += 1e-3 * np.sin(7.0 * coords)
    vals = afem.Values(s)
    best = 1e9
    for r in range(reps):
        torch.cuda.synchronize()
        t = time.perf_counter()
        vals.assemble(u)
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t)
    import hashlib
    digest = hashlib.sha1(np.ascontiguousarray(vals.numpy()).tobytes()).hexdigest()[:16] if n <= 64 else "-"
    print(f"{name} n={n} assemble {best * 1e3:.2f} ms sha1 {digest}", flush=True)

"""C4 (J2 256^3) matrix-free apply on cached Gauss-point tangents: device-buffer apply time."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_22087_b200 as afem  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
ctx = afem.Context(0, stream=torch.cuda.current_stream())
s = afem.System.grid(ctx, 3, n, n, n, inclusions=afem.fibres(12345, 40), radius=0.05,
                     materials=[(afem.J2, 1.0, 0.3, 0.002, 0.1), (afem.LINEAR, 10.0, 0.3)])
s.set_benchmark_dirichlet(0.002)
u = torch.from_numpy(s.impose_dirichlet(np.zeros(s.n))).cuda()
op = afem.matrix_free_operator(s, u)
torch.manual_seed(0)
x = torch.rand(s.n, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
L = afem.load()
import ctypes as C  # noqa: E402
for _ in range(3):
    L.afem_op_apply_async(op.h, C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()))
ts = []
for _ in range(10):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    L.afem_op_apply_async(op.h, C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()))
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
print(f"n={n} mf apply min {min(ts):.3f} ms median {sorted(ts)[5]:.3f} ms checksum {float(y.abs().sum())!r}")

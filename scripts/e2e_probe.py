import ctypes as C, time, sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2604_22087_b200 as afem
ctx = afem.Context(0)
fib = afem.fibres(12345, 40)
s = afem.System.grid(ctx, 3, 128, 128, 128, inclusions=fib, radius=0.05, materials=[(0,1.0,0.3),(0,10.0,0.3)])
s.set_benchmark_dirichlet(0.01)
u = s.impose_dirichlet(np.zeros(s.n))
op = afem.matrix_free_operator(s, u)
L = afem.load()
xh = torch.rand(s.n, dtype=torch.float64).pin_memory(); yh = torch.empty_like(xh).pin_memory()
xd = xh.cuda(); yd = torch.empty_like(xd)
for name, env in (("pipe", None), ("nopipe", "1")):
    if env: os.environ["AFEM_NO_PIPELINE"] = env
    for _ in range(3): L.afem_op_apply(op.h, C.c_void_p(xh.data_ptr()), C.c_void_p(yh.data_ptr()))
    t = time.perf_counter()
    for _ in range(20): L.afem_op_apply(op.h, C.c_void_p(xh.data_ptr()), C.c_void_p(yh.data_ptr()))
    print(name, (time.perf_counter() - t) / 20 * 1e3, "ms")
# raw copy speeds
for _ in range(2):
    torch.cuda.synchronize(); t = time.perf_counter(); xd.copy_(xh, non_blocking=True); torch.cuda.synchronize(); h2d = time.perf_counter() - t
    t = time.perf_counter(); yh.copy_(xd, non_blocking=True); torch.cuda.synchronize(); d2h = time.perf_counter() - t
print("h2d GB/s", xh.numel()*8/h2d/1e9, "d2h GB/s", xh.numel()*8/d2h/1e9)

"""Config 1 (64x64 quad4, linear E 1/10, benchmark BCs 1 %): solve_bvp (EXPLICIT and MATRIX_FREE,
CG+Jacobi, lin rtol 1e-8) on the GPU vs the reference library (oracle/_ref, 1 core) on the host."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_22087_b200 as afem
from oracle.pyoracle import Oracle

mats = [(0, 1.0, 0.3), (0, 10.0, 0.3)]
ctx = afem.Context(0)
s = afem.System.grid(ctx, 2, 64, 64, materials=mats)
s.set_benchmark_dirichlet(0.01)
R = Oracle("ref")
o = R.system(2, *s.mesh(), mats, grid=(64, 64, 0, 1.0, 1.0, 1.0))
o.set_dirichlet(*R.bcs(2, 64, 64, 0, 1.0, 0.01))
for kind in (0, 1):
    best_g = best_c = 1e9
    for _ in range(3):
        t = time.perf_counter()
        ug, rg = s.solve_bvp(operator_kind=kind, lin_rtol=1e-8)
        best_g = min(best_g, time.perf_counter() - t)
        t = time.perf_counter()
        uc, rc = o.solve_bvp(operator_kind=kind, lin_rtol=1e-8)
        best_c = min(best_c, time.perf_counter() - t)
    print(f"kind {kind}: gpu {best_g*1e3:.1f} ms (newton {rg['iterations']}, lin {rg['total_linear_iterations']}) "
          f"ref-cpu {best_c*1e3:.1f} ms (newton {rc['iterations']}, lin {rc['total_linear_iterations']}) "
          f"speedup {best_c/best_g:.1f}x")

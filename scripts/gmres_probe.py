"""Diagnostic: restarted GMRES(60)+Jacobi on config 1 — reference library (CPU) vs the device
GMRES vs a numpy restatement of the reference algorithm driving the device operator."""
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np

import paper_2604_22087_b200 as afem
from oracle.pyoracle import Oracle

RTOL, MAXIT, RS = float(sys.argv[1]) if len(sys.argv) > 1 else 1e-12, 42250, 60
ctx = afem.Context(0)
mats = [(0, 1.0, 0.3), (0, 10.0, 0.3)]
s = afem.System.grid(ctx, 2, 64, 64, materials=mats)
s.set_benchmark_dirichlet(0.01)
R = Oracle("ref")
o = R.system(2, *s.mesh(), mats, grid=(64, 64, 0, 1.0, 1.0, 1.0))
o.set_dirichlet(*R.bcs(2, 64, 64, 0, 1.0, 0.01))
u = s.impose_dirichlet(np.random.default_rng(2024).uniform(-0.01, 0.01, s.n))
b = -s.constrain_residual(s.residual(u), u)
xr, rr = o.solve(1, u, b, method=1, precond=1, rtol=RTOL, max_iter=MAXIT, restart=RS)
print("ref  ", rr["converged"], rr["iterations"], rr["residual_history"][-1], flush=True)
op = afem.matrix_free_operator(s, u)
xd, rd = afem.run_solver(op, b, method=afem.GMRES, precond=afem.JACOBI, rtol=RTOL, max_iter=MAXIT, restart=RS)
print("dev  ", rd["converged"], rd["iterations"], rd["residual_history"][-1], flush=True)


def gmres_np(A, b, inv, rtol, maxit, m):
    n = len(b)
    x = np.zeros(n)
    bn = np.sqrt(np.dot(b, b))
    r = b - A(x)
    true = np.sqrt(r @ r) / bn
    it = 0
    while true > rtol and it < maxit:
        w = r * inv
        beta = np.sqrt(w @ w)
        tgt = beta * min(1.0, 0.5 * rtol / true)
        V = [w / beta]
        H = np.zeros((m + 1, m))
        cs, sn, g = np.zeros(m), np.zeros(m), np.zeros(m + 1)
        g[0] = beta
        cols = 0
        for j in range(m):
            if it >= maxit:
                break
            w = A(V[j]) * inv
            for i in range(j + 1):
                H[i, j] = V[i] @ w
                w = w - H[i, j] * V[i]
            hn = np.sqrt(w @ w)
            H[j + 1, j] = hn
            happy = hn <= beta * 1e-16
            if not happy:
                V.append(w / hn)
            for i in range(j):
                t = cs[i] * H[i, j] + sn[i] * H[i + 1, j]
                H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
                H[i, j] = t
            rr_ = np.hypot(H[j, j], H[j + 1, j])
            cs[j], sn[j] = (1.0, 0.0) if rr_ == 0 else (H[j, j] / rr_, H[j + 1, j] / rr_)
            H[j, j], H[j + 1, j] = rr_, 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] *= cs[j]
            it += 1
            cols = j + 1
            if abs(g[j + 1]) <= tgt or happy:
                break
        y = np.zeros(cols)
        for i in range(cols - 1, -1, -1):
            y[i] = (g[i] - H[i, i + 1:cols] @ y[i + 1:cols]) / H[i, i]
        for k in range(cols):
            x = x + y[k] * V[k]
        r = b - A(x)
        true = np.sqrt(r @ r) / bn
    return x, it, true


inv = 1.0 / op.diagonal()
xn, itn, tn = gmres_np(op.apply, b, inv, RTOL, MAXIT, RS)
print("numpy", tn <= RTOL, itn, tn, flush=True)

"""Parity at the stated bench size against the CPU oracle (VERDICT r01 "next" 1).

Config 2 exactly as bench.py builds it: 128^3 hex8 elements (6.44 M dofs), 40 z-parallel fibres of
radius 0.05 from mt19937_64(12345), E 1 / 10, nu 0.3, benchmark BCs at 1 % strain, u0 the
BC-consistent zero state. Every GPU output below is compared with oracle/ (the CPU restatement
that follows the reference function by function; the reference itself has no hex8):

  * the residual R(u0) (assemble_residual, assembly.hpp:126-139), single-threaded oracle, 1e-12;
  * the structured-stencil matrix-free apply (backend.hpp:130-147) on a random vector, the oracle's
    per-element Dual<1> JVP on host threads, 1e-12;
  * the matrix-free Jacobi diagonal (backend.hpp:222-236) on the first 8 node planes, computed by
    the oracle on the 8-layer z slab of the same mesh (those planes see exactly the same elements), 1e-12;
  * the Jacobi-PCG solution at rtol 1e-8 (krylov.hpp:350-408): its true residual measured with the
    ORACLE's operator, ||b - A_oracle x|| <= 1e-8 ||b|| (the reference's re-verification contract,
    krylov.hpp:331-342, with an independent apply).
"""
import os

import numpy as np
import pytest

from oracle.pyoracle import Oracle
from tests.helpers import LINEAR, random_vector, rel_err

pytestmark = pytest.mark.gpu
N = 128
THREADS = max(1, min(32, os.cpu_count() or 1))


@pytest.fixture(scope="module")
def c2():
    import paper_2604_22087_b200 as afem
    ctx = afem.Context(0)
    fib = afem.fibres(12345, 40)
    s = afem.System.grid(ctx, 3, N, N, N, inclusions=fib, radius=0.05, materials=LINEAR)
    s.set_benchmark_dirichlet(0.01)
    orc = Oracle("restate")
    coords, conn, phase = s.mesh()
    o = orc.system(3, coords, conn, phase, LINEAR, lite=True)
    o.set_dirichlet(*orc.bcs(3, N, N, N, 1.0, 0.01))
    u0 = s.impose_dirichlet(np.zeros(s.n))
    op = afem.matrix_free_operator(s, u0)
    assert op.uses_stencil
    return afem, ctx, s, o, orc, u0, op, (coords, conn, phase)


def test_c2_residual_vs_oracle(c2):
    afem, ctx, s, o, orc, u0, op, _ = c2
    assert rel_err(s.residual(u0), o.residual(u0)) <= 1e-12


def test_c2_stencil_apply_vs_oracle(c2):
    afem, ctx, s, o, orc, u0, op, _ = c2
    for seed in (1, 2):
        x = random_vector(s.n, 1.0, seed)
        assert rel_err(op.apply(x), o.mf_apply(u0, x, nthreads=THREADS)) <= 1e-12


def test_c2_diagonal_vs_oracle_slab(c2):
    afem, ctx, s, o, orc, u0, op, mesh = c2
    coords, conn, phase = mesh
    L = 8  # element layers of the slab; node planes 0 .. L-1 have all their elements inside it
    nn = (N + 1) ** 2 * (L + 1)
    slab = orc.system(3, coords[: 3 * nn], conn[: 8 * N * N * L], phase[: N * N * L], LINEAR, lite=True)
    slab.set_dirichlet(*orc.bcs(3, N, N, L, 1.0, 0.01))
    d_gpu = op.diagonal()
    d_orc = slab.mf_diagonal(u0[: 3 * nn], nthreads=THREADS)
    m = 3 * (N + 1) ** 2 * L
    assert rel_err(d_gpu[:m], d_orc[:m]) <= 1e-12


def test_c2_cg_true_residual_with_oracle_operator(c2):
    afem, ctx, s, o, orc, u0, op, _ = c2
    b = -s.constrain_residual(s.residual(u0), u0)
    x, rep = afem.run_solver(op, b, method=afem.CG, precond=afem.JACOBI, rtol=1e-8, max_iter=20000)
    assert rep["converged"]
    r = b - o.mf_apply(u0, x, nthreads=THREADS)
    assert np.linalg.norm(r) <= 1.001e-8 * np.linalg.norm(b)

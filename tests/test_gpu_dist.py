"""GPU tests of the slab-decomposed operator and CG (dist.cu) on one B200: the threads backend runs
2-3 subdomains (one host thread + stream each) through the same code path the NCCL backend runs
across GPUs; the NCCL backend itself is exercised at world size 1.
"""
import threading

import numpy as np
import pytest

from tests.helpers import LINEAR, rel_err

pytestmark = pytest.mark.gpu

NX, NY, NZ = 64, 10, 24
STRAIN = 0.01


@pytest.fixture(scope="module")
def afem():
    import paper_2604_22087_b200 as m
    m.load()
    return m


def _global(afem, nz=NZ):
    ctx = afem.Context(0)
    fib = afem.fibres(12345, 6)
    s = afem.System.grid(ctx, 3, NX, NY, nz, inclusions=fib, radius=0.15, materials=LINEAR)
    s.set_benchmark_dirichlet(STRAIN)
    u = s.impose_dirichlet(np.zeros(s.n))
    x = np.random.default_rng(1).uniform(-1, 1, s.n)
    op = afem.matrix_free_operator(s, u)
    b = -s.constrain_residual(s.residual(u), u)
    return ctx, fib, s, u, x, op, b


def _run_threads(afem, size, fib, x, b, results, nz=NZ):
    group = afem.ThreadGroup(size)
    plane = 3 * (NX + 1) * (NY + 1)

    def work(rank):
        try:
            ctx = afem.Context(0)
            sys_, (z0, z1) = afem.slab_system(ctx, NX, NY, nz, rank, size, inclusions=fib, radius=0.15,
                                              materials=LINEAR)
            d = afem.Dist(ctx, rank, size, backend="threads", group=group)
            d.set_benchmark_dirichlet(sys_, STRAIN)
            sl = slice(plane * z0, plane * (z1 + 1))
            u = sys_.impose_dirichlet(np.zeros(sys_.n))
            op = d.matrix_free_operator(sys_, u)
            y = op.apply(x[sl])
            dot = d.dot(op, x[sl], y)
            xs, rep = d.run_solver(op, b[sl], method=afem.CG, precond=afem.JACOBI, rtol=1e-10)
            results[rank] = dict(z=(z0, z1), y=y, dot=dot, x=xs, rep=rep, stencil=op.uses_stencil)
        except Exception as e:  # surfaced by the caller
            results[rank] = e

    th = [threading.Thread(target=work, args=(r,)) for r in range(size)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    return plane


# nz 24: slabs of <= 13 node planes (one-shot apply, then the plane exchange); nz 64: slabs of
# >= 3 z pieces, which run the overlapped apply (shared-plane pieces, exchange, interior pieces)
@pytest.mark.parametrize("size,nz", [(2, 24), (3, 24), (2, 64), (3, 64)])
def test_threads_backend_matches_single_domain(afem, size, nz):
    ctx, fib, s, u, x, op, b = _global(afem, nz)
    y_global = op.apply(x)
    xg, rg = afem.run_solver(op, b, method=afem.CG, precond=afem.JACOBI, rtol=1e-10)
    results = {}
    plane = _run_threads(afem, size, fib, x, b, results, nz)
    for r in range(size):
        assert not isinstance(results[r], Exception), results[r]
    for r in range(size):
        res = results[r]
        z0, z1 = res["z"]
        sl = slice(plane * z0, plane * (z1 + 1))
        assert res["stencil"]
        assert rel_err(res["y"], y_global[sl]) <= 1e-12
        assert abs(res["dot"] - float(x @ y_global)) <= 1e-12 * abs(float(x @ y_global))
        assert res["rep"]["converged"]
        # dot products reduce per slab, then across slabs: a different (fixed) summation order
        assert abs(res["rep"]["iterations"] - rg["iterations"]) <= max(2, rg["iterations"] // 100)
        assert rel_err(res["x"], xg[sl]) <= 1e-8
    # every rank reports the same history (identical global scalars)
    h0 = results[0]["rep"]["residual_history"]
    for r in range(1, size):
        assert np.array_equal(results[r]["rep"]["residual_history"], h0)


def test_nccl_backend_single_rank(afem):
    ctx, fib, s, u, x, op, b = _global(afem)
    xg, rg = afem.run_solver(op, b, method=afem.CG, precond=afem.JACOBI, rtol=1e-10)
    d = afem.Dist(ctx, 0, 1, backend="nccl", uid=afem.nccl_unique_id())
    sys_, _ = afem.slab_system(ctx, NX, NY, NZ, 0, 1, inclusions=fib, radius=0.15, materials=LINEAR)
    d.set_benchmark_dirichlet(sys_, STRAIN)
    dop = d.matrix_free_operator(sys_, sys_.impose_dirichlet(np.zeros(sys_.n)))
    assert rel_err(dop.apply(x), op.apply(x)) <= 1e-12
    xs, rep = d.run_solver(dop, b, method=afem.CG, precond=afem.JACOBI, rtol=1e-10)
    assert rep["converged"] and abs(rep["iterations"] - rg["iterations"]) <= max(2, rg["iterations"] // 100), (rep, rg)
    assert rel_err(xs, xg) <= 1e-8


def test_distributed_cg_one_collective_kernel_count(afem):
    """The slab CG is single-reduction (one allreduce per iteration) with the (u, A u) dot fused into
    the stencil apply: at world size 1 it launches no more kernels per iteration than the
    single-GPU CG (apply with fused p.Ap, update, p update)."""
    ctx, fib, s, u, x, op, b = _global(afem, nz=64)
    l0 = ctx.launches
    xg, rg = afem.run_solver(op, b, method=afem.CG, precond=afem.JACOBI, rtol=1e-10)
    per_single = (ctx.launches - l0) / rg["iterations"]
    d = afem.Dist(ctx, 0, 1, backend="nccl", uid=afem.nccl_unique_id())
    sys_, _ = afem.slab_system(ctx, NX, NY, 64, 0, 1, inclusions=fib, radius=0.15, materials=LINEAR)
    d.set_benchmark_dirichlet(sys_, STRAIN)
    dop = d.matrix_free_operator(sys_, sys_.impose_dirichlet(np.zeros(sys_.n)))
    l1 = ctx.launches
    xs, rep = d.run_solver(dop, b, method=afem.CG, precond=afem.JACOBI, rtol=1e-10)
    per_dist = (ctx.launches - l1) / rep["iterations"]
    assert rep["converged"] and abs(rep["iterations"] - rg["iterations"]) <= max(2, rg["iterations"] // 100), (rep, rg)
    assert rel_err(xs, xg) <= 1e-8
    assert per_dist <= per_single, (per_dist, per_single)


J2_MIX = [(3, 1.0, 0.3, 0.002, 0.1), (0, 10.0, 0.3)]


@pytest.mark.parametrize("size", [2, 3])
def test_distributed_j2_load_stepping_matches_single_domain(afem, size):
    """Config 4 in miniature, slab-sharded: per-rank J2 history, distributed Newton (MF, CG+Jacobi)
    with shared-plane residual assembly and a global free norm; vs the single-domain load path."""
    nx, ny, nz = 8, 8, 12
    ctx = afem.Context(0)
    fib = afem.fibres(12345, 4)
    g = afem.System.grid(ctx, 3, nx, ny, nz, inclusions=fib, radius=0.2, materials=J2_MIX)
    ug, rg = g.load_stepping(0.01, 3, operator_kind=afem.MATRIX_FREE, lin_rtol=1e-12)
    assert rg["converged"]
    hg = g.history().reshape(nz, ny * nx * 8 * 8)
    group = afem.ThreadGroup(size)
    plane = 3 * (nx + 1) * (ny + 1)
    results = {}

    def work(rank):
        try:
            c = afem.Context(0)
            s, (z0, z1) = afem.slab_system(c, nx, ny, nz, rank, size, inclusions=fib, radius=0.2, materials=J2_MIX)
            d = afem.Dist(c, rank, size, backend="threads", group=group)
            u, rep = d.load_stepping(s, 0.01, 3, lx_global=1.0, lin_rtol=1e-12)
            results[rank] = dict(z=(z0, z1), u=u, rep=rep, hist=s.history())
        except Exception as e:  # surfaced below
            results[rank] = e

    th = [threading.Thread(target=work, args=(r,)) for r in range(size)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    for r in range(size):
        assert not isinstance(results[r], Exception), results[r]
        res = results[r]
        z0, z1 = res["z"]
        assert res["rep"]["converged"]
        assert list(res["rep"]["step_iterations"]) == list(rg["step_iterations"])
        assert rel_err(res["u"], ug[plane * z0: plane * (z1 + 1)]) <= 1e-8
        # the rank's committed history is the single-domain history of its element layers
        assert rel_err(res["hist"], hg[z0:z1].ravel()) <= 1e-8


@pytest.mark.parametrize("size", [2, 3])
def test_distributed_explicit_operator_matches_single_domain(afem, size):
    """The assembled (explicit) operator over the slab decomposition: each rank assembles and
    eliminates its own slab's Neo-Hookean tangent at a perturbed state; the local SpMV gives partial
    sums on the shared planes, completed by the plane halo. y = K x and the distributed Jacobi-PCG
    solution equal the single-domain explicit operator's on every slab."""
    nh = [(2, 1.0, 0.3), (0, 10.0, 0.3)]
    ctx = afem.Context(0)
    fib = afem.fibres(12345, 6)
    s = afem.System.grid(ctx, 3, NX, NY, NZ, inclusions=fib, radius=0.15, materials=nh)
    s.set_benchmark_dirichlet(STRAIN)
    u = s.impose_dirichlet(np.random.default_rng(7).uniform(-0.003, 0.003, s.n))
    x = np.random.default_rng(8).uniform(-1, 1, s.n)
    vals = afem.Values(s).assemble(u)
    rhs = vals.eliminate(s.residual(u), u)
    buf = afem.HandoffBuffer(s)
    buf.handoff(vals)
    op = afem.explicit_operator(buf)
    y_global = op.apply(x)
    xg, rg = afem.run_solver(op, -rhs, method=afem.CG, precond=afem.JACOBI, rtol=1e-10)
    buf.release()
    group = afem.ThreadGroup(size)
    plane = 3 * (NX + 1) * (NY + 1)
    results = {}

    def work(rank):
        try:
            c = afem.Context(0)
            sys_, (z0, z1) = afem.slab_system(c, NX, NY, NZ, rank, size, inclusions=fib, radius=0.15, materials=nh)
            d = afem.Dist(c, rank, size, backend="threads", group=group)
            d.set_benchmark_dirichlet(sys_, STRAIN)
            sl = slice(plane * z0, plane * (z1 + 1))
            v = afem.Values(sys_).assemble(u[sl])
            v.eliminate(sys_.residual(u[sl]), u[sl])
            dop = d.explicit_operator(sys_, v.numpy())
            y = dop.apply(x[sl])
            xs, rep = d.run_solver(dop, -rhs[sl], method=afem.CG, precond=afem.JACOBI, rtol=1e-10)
            results[rank] = dict(sl=sl, y=y, x=xs, rep=rep, stencil=dop.uses_stencil)
        except Exception as e:  # surfaced below
            results[rank] = e

    th = [threading.Thread(target=work, args=(r,)) for r in range(size)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    for r in range(size):
        assert not isinstance(results[r], Exception), results[r]
        res = results[r]
        assert not res["stencil"]
        assert rel_err(res["y"], y_global[res["sl"]]) <= 1e-12
        assert res["rep"]["converged"]
        assert abs(res["rep"]["iterations"] - rg["iterations"]) <= max(2, rg["iterations"] // 100)
        assert rel_err(res["x"], xg[res["sl"]]) <= 1e-8


@pytest.mark.parametrize("method", ["gmres", "bicgstab"])
def test_distributed_gmres_bicgstab_match_single_domain(afem, method):
    """GMRES(30) and BiCGStab over the slab decomposition: the same host-driven methods as on one
    GPU, their inner products summed over owned dofs and allreduced (identical scalars on every
    rank). A small mild-contrast RVE (restarted GMRES stagnates near 1e-5 on the large 10:1 one, in
    the single-domain solve as in the reference): solutions equal the single-domain solve,
    iteration counts agree within 15 % (the dots reduce in a different order; BiCGStab's count is
    rounding-sensitive)."""
    size = 2
    meth = afem.GMRES if method == "gmres" else afem.BICGSTAB
    mild = [(0, 1.0, 0.3), (0, 1.5, 0.3)]
    rtol = 1e-10
    nx, ny, nz = 16, 8, 12  # small enough that GMRES(30) does not stagnate
    ctx = afem.Context(0)
    fib = afem.fibres(12345, 6)
    s = afem.System.grid(ctx, 3, nx, ny, nz, inclusions=fib, radius=0.15, materials=mild)
    s.set_benchmark_dirichlet(STRAIN)
    u = s.impose_dirichlet(np.zeros(s.n))
    op = afem.matrix_free_operator(s, u)
    b = -s.constrain_residual(s.residual(u), u)
    xg, rg = afem.run_solver(op, b, method=meth, precond=afem.JACOBI, rtol=rtol, max_iter=5000)
    assert rg["converged"]
    group = afem.ThreadGroup(size)
    plane = 3 * (nx + 1) * (ny + 1)
    results = {}

    def work(rank):
        try:
            c = afem.Context(0)
            sys_, (z0, z1) = afem.slab_system(c, nx, ny, nz, rank, size, inclusions=fib, radius=0.15, materials=mild)
            d = afem.Dist(c, rank, size, backend="threads", group=group)
            d.set_benchmark_dirichlet(sys_, STRAIN)
            sl = slice(plane * z0, plane * (z1 + 1))
            dop = d.matrix_free_operator(sys_, sys_.impose_dirichlet(np.zeros(sys_.n)))
            xs, rep = d.run_solver(dop, b[sl], method=meth, precond=afem.JACOBI, rtol=rtol, max_iter=5000)
            results[rank] = dict(sl=sl, x=xs, rep=rep)
        except Exception as e:  # surfaced below
            results[rank] = e

    th = [threading.Thread(target=work, args=(r,)) for r in range(size)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    for r in range(size):
        assert not isinstance(results[r], Exception), results[r]
        res = results[r]
        assert res["rep"]["converged"]
        # restarted GMRES amplifies the different reduction order over many restart cycles
        slack = 50 if method == "gmres" else 15
        assert abs(res["rep"]["iterations"] - rg["iterations"]) <= max(2, (slack * rg["iterations"]) // 100)
        assert rel_err(res["x"], xg[res["sl"]]) <= 1e-6
    assert results[0]["rep"]["iterations"] == results[1]["rep"]["iterations"]


@pytest.mark.parametrize("method", ["gmres", "bicgstab"])
def test_distributed_newton_with_gmres_bicgstab_linear_steps(afem, method):
    """Distributed solve_bvp whose linear solver is GMRES(30) or BiCGStab (run_solver's method
    dispatch, backend.hpp:241-286, over the slab operator's allreduced inner products): converges
    with the single-domain Newton's iteration count and displacement."""
    nh = [(2, 1.0, 0.3), (0, 10.0, 0.3)]
    nx, ny, nz, size = 6, 6, 8, 2
    meth = afem.GMRES if method == "gmres" else afem.BICGSTAB
    ctx = afem.Context(0)
    fib = afem.fibres(12345, 4)
    g = afem.System.grid(ctx, 3, nx, ny, nz, inclusions=fib, radius=0.2, materials=nh)
    g.set_benchmark_dirichlet(STRAIN)
    ug, rg = g.solve_bvp(operator_kind=afem.MATRIX_FREE, method=meth, lin_rtol=1e-11, lin_max_iter=20000)
    assert rg["converged"]
    group = afem.ThreadGroup(size)
    plane = 3 * (nx + 1) * (ny + 1)
    results = {}

    def work(rank):
        try:
            c = afem.Context(0)
            s, (z0, z1) = afem.slab_system(c, nx, ny, nz, rank, size, inclusions=fib, radius=0.2, materials=nh)
            d = afem.Dist(c, rank, size, backend="threads", group=group)
            d.set_benchmark_dirichlet(s, STRAIN)
            u, rep = d.solve_bvp(s, operator_kind=afem.MATRIX_FREE, method=meth, lin_rtol=1e-11,
                                 lin_max_iter=20000)
            results[rank] = dict(z=(z0, z1), u=u, rep=rep)
        except Exception as e:  # surfaced below
            results[rank] = e

    th = [threading.Thread(target=work, args=(r,)) for r in range(size)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    for r in range(size):
        assert not isinstance(results[r], Exception), results[r]
        res = results[r]
        z0, z1 = res["z"]
        assert res["rep"]["converged"], res["rep"]["failure"]
        assert res["rep"]["iterations"] == rg["iterations"]
        assert rel_err(res["u"], ug[plane * z0: plane * (z1 + 1)]) <= 1e-8


@pytest.mark.parametrize("size", [2, 3])
def test_distributed_newton_assembled_tangent_matches_single_domain(afem, size):
    """Distributed solve_bvp on the assembled tangent (EXPLICIT): every Newton iteration each slab
    assembles and eliminates its own Neo-Hookean tangent (assemble_jacobian + apply_dirichlet,
    newton.hpp:93-104), the distributed CG solves on it; iteration count and u equal the
    single-domain EXPLICIT Newton."""
    nh = [(2, 1.0, 0.3), (0, 10.0, 0.3)]
    nx, ny, nz = 8, 8, 12
    ctx = afem.Context(0)
    fib = afem.fibres(12345, 4)
    g = afem.System.grid(ctx, 3, nx, ny, nz, inclusions=fib, radius=0.2, materials=nh)
    g.set_benchmark_dirichlet(STRAIN)
    ug, rg = g.solve_bvp(operator_kind=afem.EXPLICIT, lin_rtol=1e-12)
    assert rg["converged"]
    group = afem.ThreadGroup(size)
    plane = 3 * (nx + 1) * (ny + 1)
    results = {}

    def work(rank):
        try:
            c = afem.Context(0)
            s, (z0, z1) = afem.slab_system(c, nx, ny, nz, rank, size, inclusions=fib, radius=0.2, materials=nh)
            d = afem.Dist(c, rank, size, backend="threads", group=group)
            d.set_benchmark_dirichlet(s, STRAIN)
            u, rep = d.solve_bvp(s, operator_kind=afem.EXPLICIT, lin_rtol=1e-12)
            results[rank] = dict(z=(z0, z1), u=u, rep=rep)
        except Exception as e:  # surfaced below
            results[rank] = e

    th = [threading.Thread(target=work, args=(r,)) for r in range(size)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=600)
    for r in range(size):
        assert not isinstance(results[r], Exception), results[r]
        res = results[r]
        z0, z1 = res["z"]
        assert res["rep"]["converged"]
        assert res["rep"]["iterations"] == rg["iterations"]
        assert rel_err(res["u"], ug[plane * z0: plane * (z1 + 1)]) <= 1e-8


def test_distributed_capability_errors(afem):
    """The distributed run_solver keeps the reference's error contract: ILU(0) and the direct
    methods need the whole assembled matrix (CapabilityError, backend.hpp:151-156 / 245-269), an
    unknown method is invalid; a non-distributed operator is rejected."""
    ctx, fib, s, u, x, op, b = _global(afem)
    d = afem.Dist(ctx, 0, 1, backend="nccl", uid=afem.nccl_unique_id())
    sys_, _ = afem.slab_system(ctx, NX, NY, NZ, 0, 1, inclusions=fib, radius=0.15, materials=LINEAR)
    d.set_benchmark_dirichlet(sys_, STRAIN)
    dop = d.matrix_free_operator(sys_, sys_.impose_dirichlet(np.zeros(sys_.n)))
    for method, precond in ((afem.CG, afem.ILU0), (afem.GMRES, afem.ILU0), (afem.DIRECT_CHOL, afem.NONE)):
        with pytest.raises(afem.CapabilityError):
            d.run_solver(dop, b, method=method, precond=precond, rtol=1e-8, max_iter=10)
    with pytest.raises(afem.AfemError):
        d.run_solver(op, b, method=afem.CG, precond=afem.JACOBI, rtol=1e-8, max_iter=10)


OVERLAP_SNIPPET = r"""
import sys, threading, numpy as np
sys.path.insert(0, {root!r})
import paper_2604_22087_b200 as afem
NX, NY, NZ, size = 64, 10, 64, 2
LIN = [(0, 1.0, 0.3), (0, 10.0, 0.3)]
ctx = afem.Context(0)
fib = afem.fibres(12345, 6)
s = afem.System.grid(ctx, 3, NX, NY, NZ, inclusions=fib, radius=0.15, materials=LIN)
s.set_benchmark_dirichlet(0.01)
u = s.impose_dirichlet(np.zeros(s.n))
x = np.random.default_rng(1).uniform(-1, 1, s.n)
yg = afem.matrix_free_operator(s, u).apply(x)
group = afem.ThreadGroup(size)
plane = 3 * (NX + 1) * (NY + 1)
res = {{}}
def work(rank):
    c = afem.Context(0)
    ss, (z0, z1) = afem.slab_system(c, NX, NY, NZ, rank, size, inclusions=fib, radius=0.15, materials=LIN)
    d = afem.Dist(c, rank, size, backend="threads", group=group)
    d.set_benchmark_dirichlet(ss, 0.01)
    op = d.matrix_free_operator(ss, ss.impose_dirichlet(np.zeros(ss.n)))
    sl = slice(plane * z0, plane * (z1 + 1))
    res[rank] = float(np.abs(op.apply(x[sl]) - yg[sl]).max() / np.abs(yg).max())
th = [threading.Thread(target=work, args=(r,)) for r in range(size)]
[t.start() for t in th]
[t.join() for t in th]
print(max(res.values()))
"""


def test_sequential_slab_schedule_matches_single_domain():
    """AFEM_DIST_OVERLAP=0 (whole-slab apply, then the exchange and the halo add) gives the
    single-domain apply, like the default overlapped schedule the in-process tests run."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, AFEM_DIST_OVERLAP="0")
    p = subprocess.run([sys.executable, "-c", OVERLAP_SNIPPET.format(root=root)], capture_output=True, text=True,
                       env=env, timeout=600)
    assert p.returncode == 0, p.stderr[-3000:]
    assert float(p.stdout.strip().splitlines()[-1]) <= 1e-12

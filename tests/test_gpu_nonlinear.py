"""GPU parity for the north star's nonlinear laws (configs 3 and 4): compressible Neo-Hookean and
small-strain J2 plasticity with device-resident quadrature-point history, against the CPU
restatement (oracle/restate.hpp; pinned in tests/test_oracle_nonlinear.py by an independent
integrator). Tolerances as DESIGN.md §Parity: residual / tangent / operator <= 1e-12 relative,
history <= 1e-12, converged displacement <= 1e-8, Newton iteration counts equal.
"""
import numpy as np
import pytest

from oracle.pyoracle import Oracle
from tests.helpers import random_vector, rel_err

pytestmark = pytest.mark.gpu

TOL = 1e-12
TOL_U = 1e-8
NH_MIX = [(2, 1.0, 0.3), (0, 10.0, 0.3)]
NH_BOTH = [(2, 1.0, 0.3), (2, 10.0, 0.3)]
J2_MIX = [(3, 1.0, 0.3, 0.002, 0.1), (0, 10.0, 0.3)]


@pytest.fixture(scope="module")
def afem():
    import paper_2604_22087_b200 as m
    m.load()
    return m


@pytest.fixture(scope="module")
def ctx(afem):
    return afem.Context(0)


@pytest.fixture(scope="module")
def orc():
    return Oracle("restate")


def case(afem, ctx, orc, dim, n, mats, strain=0.01):
    if dim == 3:
        fib = afem.fibres(12345, 4)
        s = afem.System.grid(ctx, 3, n, n, n, inclusions=fib, radius=0.2, materials=mats)
    else:
        s = afem.System.grid(ctx, 2, n, n, materials=mats)
    s.set_benchmark_dirichlet(strain)
    coords, conn, phase = s.mesh()
    o = orc.system(dim, coords, conn, phase, mats, grid=(n, n, n if dim == 3 else 0, 1.0, 1.0, 1.0))
    o.set_dirichlet(*orc.bcs(dim, n, n, n if dim == 3 else 0, 1.0, strain))
    return s, o


def assembly_parity(afem, s, o, u, x):
    assert rel_err(s.residual(u), o.residual(u)) <= TOL
    K = s.jacobian(u)
    assert rel_err(K, o.jacobian(u)) <= TOL
    assert rel_err(s.diagonal(u), o.diagonal(u)) <= TOL
    op = afem.matrix_free_operator(s, u)
    assert not op.uses_stencil
    assert rel_err(op.apply(x), o.mf_apply(u, x)) <= TOL
    assert rel_err(op.diagonal(), o.mf_diagonal(u)) <= TOL


@pytest.mark.parametrize("dim,mats", [(3, NH_MIX), (3, NH_BOTH), (2, NH_BOTH)], ids=["3d-mix", "3d-nh", "2d-nh"])
def test_neohooke_assembly_parity(afem, ctx, orc, dim, mats):
    s, o = case(afem, ctx, orc, dim, 5 if dim == 3 else 8, mats)
    u = s.impose_dirichlet(random_vector(s.n, 0.05, 3))
    assembly_parity(afem, s, o, u, random_vector(s.n, 1.0, 4))


@pytest.mark.parametrize("dim", [3, 2])
def test_j2_assembly_parity_with_history(afem, ctx, orc, dim):
    s, o = case(afem, ctx, orc, dim, 5 if dim == 3 else 8, J2_MIX)
    assert s.history_size() == o.history().size > 0
    # a plastic committed state: commit at a large random displacement, then evaluate elsewhere
    u0 = random_vector(s.n, 0.02, 10)
    s.commit_history(u0)
    o.commit_history(u0)
    hg, ho = s.history(), o.history()
    assert np.abs(ho[6::8]).max() > 0  # some Gauss points yielded
    assert rel_err(hg, ho) <= TOL
    u = s.impose_dirichlet(random_vector(s.n, 0.02, 11))
    assembly_parity(afem, s, o, u, random_vector(s.n, 1.0, 12))
    s.reset_history()
    assert not s.history().any()


def test_neohooke_newton_gmres_parity(afem, ctx, orc):
    """Config 3 in miniature: Newton with the assembled tangent and GMRES(30)+Jacobi."""
    s, o = case(afem, ctx, orc, 3, 4, NH_MIX, strain=0.05)
    for kind in (0, 1):
        ug, rg = s.solve_bvp(rtol=1e-10, lin_rtol=1e-12, operator_kind=kind, method=afem.GMRES)
        uo, ro = o.solve_bvp(rtol=1e-10, lin_rtol=1e-12, operator_kind=kind, method=1)
        assert rg["converged"] and ro["converged"] and rg["iterations"] >= 3
        assert rg["iterations"] == ro["iterations"]
        assert rel_err(ug, uo) <= TOL_U


def test_j2_load_stepping_parity(afem, ctx, orc):
    """Config 4 in miniature: incremental loading with committed history between steps."""
    s, o = case(afem, ctx, orc, 3, 4, J2_MIX, strain=0.01)
    ug, rg = s.load_stepping(0.01, 4, lin_rtol=1e-12)
    uo, ro = o.load_stepping(0.01, 4, lin_rtol=1e-12)
    assert rg["converged"] and ro["converged"]
    assert list(rg["step_iterations"]) == list(ro["step_iterations"])
    assert rel_err(ug, uo) <= TOL_U
    assert rel_err(s.history(), o.history()) <= 1e-8
    assert s.history()[6::8].max() > 0


def test_nonlinear_determinism_bitwise(afem, ctx, orc):
    s, _ = case(afem, ctx, orc, 3, 5, J2_MIX)
    s.commit_history(random_vector(s.n, 0.02, 1))
    u = s.impose_dirichlet(random_vector(s.n, 0.02, 2))
    assert s.residual(u).tobytes() == s.residual(u).tobytes()
    assert s.jacobian(u).tobytes() == s.jacobian(u).tobytes()


def test_inverted_element_raises(afem, ctx):
    s = afem.System.grid(ctx, 3, 2, 2, 2, materials=[(2, 1.0, 0.3)])
    u = np.zeros(s.n)
    u[0::3] = -3.0 * s.mesh()[0][0::3]  # x -> -2x: det F < 0
    with pytest.raises(afem.InvertedElementError):
        s.residual(u)


def test_j2_material_validation(afem, ctx):
    with pytest.raises(afem.InvalidArgument):
        afem.System.grid(ctx, 3, 2, 2, 2, materials=[(3, 1.0, 0.3, 0.0, 0.1)])


@pytest.mark.parametrize("mats", [NH_MIX, J2_MIX, [(1, 1.0, 0.3), (0, 10.0, 0.3)], [(0, 1.0, 0.3), (0, 10.0, 0.3)]],
                         ids=["neohooke", "j2", "svk", "linear"])
def test_general_mesh_kernels_all_laws(afem, ctx, orc, mats):
    """Distorted (non-grid) hex8 mesh: the node-centric general kernels vs the restatement, and the
    element-centric grid kernels vs the general kernels on the same undistorted mesh."""
    n = 4
    fib = afem.fibres(12345, 4)
    g = afem.System.grid(ctx, 3, n, n, n, inclusions=fib, radius=0.2, materials=mats)
    coords, conn, phase = g.mesh()
    flat = afem.System(ctx, 3, coords, conn, phase, mats)  # same mesh through the general path
    u = random_vector(g.n, 0.03, 21)
    x = random_vector(g.n, 1.0, 22)
    if g.history_size():
        g.commit_history(u * 0.7)
        flat.commit_history(u * 0.7)
    assert rel_err(g.residual(u), flat.residual(u)) <= 1e-13
    assert rel_err(g.diagonal(u), flat.diagonal(u)) <= 1e-13
    assert rel_err(afem.matrix_free_operator(g, u).apply(x), afem.matrix_free_operator(flat, u).apply(x)) <= 1e-13
    dist = coords + random_vector(len(coords), 0.02, 23)
    s = afem.System(ctx, 3, dist, conn, phase, mats)
    o = orc.system(3, dist, conn, phase, mats)
    if s.history_size():
        s.commit_history(u * 0.7)
        o.commit_history(u * 0.7)
        assert rel_err(s.history(), o.history()) <= TOL
    assembly_parity(afem, s, o, u, x)


@pytest.mark.parametrize("mats", [NH_MIX, J2_MIX], ids=["nh", "j2"])
def test_grid_tangent_slabs_bitwise_and_oracle(afem, ctx, orc, mats, monkeypatch):
    """The 3D grid tangent runs element-centric per z slab of node planes (element blocks in a
    scratch, node rows gathered in incidence order): any slab size gives bitwise the same values,
    and they match the restatement's AD tangent to 1e-12."""
    s, o = case(afem, ctx, orc, 3, 7, mats)
    u = s.impose_dirichlet(random_vector(s.n, 0.02, 5))
    if mats is J2_MIX:  # a plastic history: commit a loaded state first
        s.commit_history(s.impose_dirichlet(random_vector(s.n, 0.05, 6)))
        o.commit_history(s.impose_dirichlet(random_vector(s.n, 0.05, 6)))
    K = s.jacobian(u)
    assert rel_err(K, o.jacobian(u)) <= TOL
    for planes in ("1", "2", "3", "5"):
        monkeypatch.setenv("AFEM_JAC_SLAB", planes)
        assert np.array_equal(s.jacobian(u), K)


# ---- the stated configs' materials and fibre generator at larger sizes
C3_MATS = [(2, 1.0, 0.3), (0, 10.0, 0.3)]
C4_MATS = [(3, 1.0, 0.3, 0.002, 0.1), (0, 10.0, 0.3)]


def stated_case(afem, ctx, orc, n, mats, strain):
    """C2-C5 fibre generator (mt19937_64(12345), 40 fibres, r = 0.05) at n^3."""
    s = afem.System.grid(ctx, 3, n, n, n, inclusions=afem.fibres(12345, 40), radius=0.05, materials=mats)
    s.set_benchmark_dirichlet(strain)
    coords, conn, phase = s.mesh()
    o = orc.system(3, coords, conn, phase, mats, grid=(n, n, n, 1.0, 1.0, 1.0))
    o.set_dirichlet(*orc.bcs(3, n, n, n, 1.0, strain))
    assert 0 < phase.mean() < 1
    return s, o


@pytest.mark.parametrize("cfg", ["c3", "c4"])
def test_stated_config_kernels_n32(afem, ctx, orc, cfg):
    """Residual, tangent, diagonal and matrix-free apply of configs 3 / 4 at 32^3 (107 k dofs, 8.2 M
    tangent values) against the restatement; C4 from a plastic committed history."""
    mats = C3_MATS if cfg == "c3" else C4_MATS
    s, o = stated_case(afem, ctx, orc, 32, mats, 0.05 if cfg == "c3" else 0.02)
    if cfg == "c4":
        u0 = s.impose_dirichlet(random_vector(s.n, 0.5 / 32, 21))  # plastic at the Gauss points
        s.commit_history(u0)
        o.commit_history(u0)
        assert rel_err(s.history(), o.history()) <= TOL and np.abs(o.history()[6::8]).max() > 0
    u = s.impose_dirichlet(random_vector(s.n, 0.1 / 32, 22))  # a tenth of the element size: no inversion
    x = random_vector(s.n, 1.0, 23)
    assert rel_err(s.residual(u), o.residual(u)) <= TOL
    assert rel_err(s.jacobian(u), o.jacobian(u)) <= TOL
    assert rel_err(s.diagonal(u), o.diagonal(u)) <= TOL
    op = afem.matrix_free_operator(s, u)
    assert rel_err(op.apply(x), o.mf_apply(u, x)) <= TOL
    assert rel_err(op.diagonal(), o.mf_diagonal(u)) <= TOL


def _affine(coords, strain):
    u = np.zeros_like(coords)
    u[0::3] = strain * coords[0::3]
    return u


def test_stated_config3_newton_n12(afem, ctx, orc):
    """C3's solve path (Newton, assembled tangent, CG+Jacobi, affine warm start) at 12^3 with the
    stated fibre generator: Newton counts equal, u within 1e-8."""
    s, o = stated_case(afem, ctx, orc, 12, C3_MATS, 0.05)
    x0 = s.impose_dirichlet(_affine(s.mesh()[0], 0.05))
    ug, rg = s.solve_bvp(x0=x0, rtol=1e-10, lin_rtol=1e-12, operator_kind=afem.EXPLICIT, method=afem.CG,
                         precond=afem.JACOBI)
    uo, ro = o.solve_bvp(x0=x0, rtol=1e-10, lin_rtol=1e-12, operator_kind=0, method=0, precond=1)
    assert rg["converged"] and ro["converged"] and rg["iterations"] == ro["iterations"] >= 2
    assert rel_err(ug, uo) <= TOL_U


def test_stated_config4_load_path_n12(afem, ctx, orc):
    """C4's load path (J2, history committed per step, matrix-free cached tangent) at 12^3, 4 steps."""
    s, o = stated_case(afem, ctx, orc, 12, C4_MATS, 0.02)
    ug, rg = s.load_stepping(0.02, 4, lin_rtol=1e-12, operator_kind=afem.MATRIX_FREE)
    uo, ro = o.load_stepping(0.02, 4, lin_rtol=1e-12, operator_kind=1)
    assert rg["converged"] and ro["converged"]
    assert list(rg["step_iterations"]) == list(ro["step_iterations"])
    assert rel_err(ug, uo) <= TOL_U and rel_err(s.history(), o.history()) <= 1e-8

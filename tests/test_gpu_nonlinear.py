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

"""CPU tests: pin the oracle (restatement) against the reference's golden vectors and against the
reference's own frozen facts, then check the hex8 twin by properties the reference tests for 2D.
"""
import numpy as np
import pytest

from oracle.pyoracle import Oracle, OracleError, available
from tests.helpers import LINEAR, SVK_MIX, bc_state, fibre_mesh, golden_cases, load, random_vector, rel_err


@pytest.fixture(scope="module")
def orc():
    return Oracle("restate")


def _system_from_golden(orc, g):
    n = int(g["n"])
    mats = [tuple(m) for m in g["mats"]]
    s = orc.system(2, g["coords"], g["conn"], g["phase"], [(int(m[0]), m[1], m[2]) for m in mats],
                   grid=(n, n, 0, 1.0, 1.0, 1.0))
    s.set_dirichlet(g["bc_node"], g["bc_comp"], g["bc_val"])
    return s


@pytest.mark.parametrize("path", golden_cases())
def test_restatement_matches_reference_golden(orc, path):
    g = load(path)
    n = int(g["n"])
    coords, conn, phase = orc.mesh2d(n, n)
    assert np.array_equal(coords, g["coords"]) and np.array_equal(conn, g["conn"])
    assert np.array_equal(phase, g["phase"])
    node, comp, val = orc.bcs(2, n, n, 0, 1.0, float(g["strain"]))
    assert np.array_equal(node, g["bc_node"]) and np.array_equal(comp, g["bc_comp"])
    assert np.array_equal(val, g["bc_val"])
    s = _system_from_golden(orc, g)
    rp, rows, cols = s.pattern()
    assert np.array_equal(rp, g["row_ptr"]) and np.array_equal(rows, g["rows"]) and np.array_equal(cols, g["cols"])
    u, x = g["u"], g["x"]
    assert rel_err(s.residual(u), g["residual"]) <= 1e-15
    assert rel_err(s.jacobian(u), g["jacobian"]) <= 1e-15
    assert rel_err(s.diagonal(u), g["diagonal"]) <= 1e-15
    v, r = s.eliminate(g["jacobian"], g["residual"], u)
    assert rel_err(v, g["elim_values"]) <= 1e-15 and rel_err(r, g["elim_rhs"]) <= 1e-15
    assert rel_err(s.mf_apply(u, x), g["mf_apply"]) <= 1e-15
    assert rel_err(s.csr_apply(g["elim_values"], x), g["csr_apply"]) <= 1e-15
    xc, rep = s.solve(0, g["elim_values"], -g["elim_rhs"], method=0, precond=1, rtol=1e-10)
    assert rep["iterations"] == int(g["cg_iterations"])
    assert rel_err(xc, g["x_cg"]) <= 1e-14
    ub, rb = s.solve_bvp(rtol=1e-10, lin_rtol=1e-12)
    assert rb["iterations"] == int(g["bvp_iterations"])
    assert rel_err(ub, g["u_bvp"]) <= 1e-14


@pytest.mark.skipif(not available("ref"), reason="oracle/_ref not built")
def test_restatement_bitwise_vs_reference_config1():
    """Config 1 (64x64 quad4, linear E 1/10) through both libraries: identical bits."""
    R, O = Oracle("ref"), Oracle("restate")
    mesh = R.mesh2d(64, 64)
    bc = R.bcs(2, 64, 64, 0, 1.0, 0.01)
    out = []
    for lib in (R, O):
        s = lib.system(2, *mesh, LINEAR, grid=(64, 64, 0, 1.0, 1.0, 1.0))
        s.set_dirichlet(*bc)
        u = bc_state(s.n, 2, *bc, u=random_vector(s.n, 0.01, 7))
        out.append((s.pattern(), s.residual(u), s.jacobian(u), s.mf_apply(u, random_vector(s.n, 1.0, 12345))))
    (pa, ra, ja, ma), (pb, rb, jb, mb) = out
    assert all(np.array_equal(a, b) for a, b in zip(pa, pb))
    assert np.array_equal(ra, rb) and np.array_equal(ja, jb) and np.array_equal(ma, mb)


def test_reference_frozen_facts(orc):
    # phase count 16 on 10x10 r=0.25 (reference test_mesh.cpp:46-60)
    _, _, phase = orc.mesh2d(10, 10)
    assert int(phase.sum()) == 16
    # nnz 64 for one element, 112 for two sharing an edge (test_assembly.cpp:52-67)
    s1 = orc.system(2, *orc.mesh2d(1, 1, radius=0.0), [(0, 1.0, 0.3)])
    assert s1.nnz() == 64
    s2 = orc.system(2, *orc.mesh2d(2, 1, radius=0.0), [(0, 1.0, 0.3)])
    assert s2.nnz() == 112
    # 2(ny+1)+1 benchmark constraints (test_mesh.cpp:117-122)
    assert len(orc.bcs(2, 7, 5, 0, 1.0, 0.01)[0]) == 2 * 6 + 1


def test_error_semantics(orc):
    with pytest.raises(OracleError) as e:
        orc.mesh2d(0, 3)
    assert e.value.code == 1  # invalid_argument
    s = orc.system(2, *orc.mesh2d(2, 2), SVK_MIX)
    with pytest.raises(OracleError) as e:
        s.set_dirichlet([99], [0], [0.0])
    assert e.value.code == 2  # out_of_range
    with pytest.raises(OracleError) as e:
        s.set_dirichlet([0, 0], [0, 0], [0.0, 0.0])
    assert e.value.code == 1  # duplicate pair
    with pytest.raises(OracleError) as e:  # missing material for phase 1
        orc.system(2, *orc.mesh2d(4, 4), [(0, 1.0, 0.3)])
    assert "no material supplied" in e.value.msg


# ------------------------------------------------------------------ hex8 twin (restatement only)

@pytest.fixture(scope="module")
def hex_sys(orc):
    (coords, conn, phase), _ = fibre_mesh(orc, 4, n_fibres=3, radius=0.3)
    s = orc.system(3, coords, conn, phase, SVK_MIX, grid=(4, 4, 4, 1.0, 1.0, 1.0))
    s.set_dirichlet(*orc.bcs(3, 4, 4, 4, 1.0, 0.01))
    return s, coords, phase


def test_hex8_mesh_and_bcs(orc, hex_sys):
    s, coords, phase = hex_sys
    assert s.n == 3 * 125 and len(phase) == 64 and 0 < phase.sum() < 64
    node, comp, _ = orc.bcs(3, 4, 4, 4, 1.0, 0.01)
    assert len(node) == 2 * 25 + 3
    # pattern: nnz = 9 (3N+1)^3 for a structured hex grid
    assert s.nnz() == 9 * 13 ** 3


def test_hex8_rigid_translation_has_zero_residual(orc, hex_sys):
    s, coords, _ = hex_sys
    u = np.tile([0.3, -0.2, 0.1], s.n // 3)
    assert np.abs(s.residual(u)).max() < 1e-13


def test_hex8_linear_residual_equals_jacobian_times_u(orc):
    (coords, conn, phase), _ = fibre_mesh(orc, 3, n_fibres=2, radius=0.3)
    s = orc.system(3, coords, conn, phase, LINEAR)
    u = random_vector(s.n, 0.01, 3)
    rp, rows, cols = s.pattern()
    K = s.jacobian(u)
    Ku = np.zeros(s.n)
    np.add.at(Ku, rows, K * u[cols])
    assert rel_err(s.residual(u), Ku) < 1e-13
    # symmetric
    dense = np.zeros((s.n, s.n))
    dense[rows, cols] = K
    assert np.abs(dense - dense.T).max() < 1e-12 * np.abs(dense).max()


def test_hex8_jacobian_matches_finite_differences(orc, hex_sys):
    s, _, _ = hex_sys
    u = random_vector(s.n, 0.01, 5)
    rp, rows, cols = s.pattern()
    K = s.jacobian(u)
    dense = np.zeros((s.n, s.n))
    dense[rows, cols] = K
    h = 1e-6
    for j in [0, 7, 50, 121, 300]:
        e = np.zeros(s.n)
        e[j] = h
        fd = (s.residual(u + e) - s.residual(u - e)) / (2 * h)
        assert np.abs(fd - dense[:, j]).max() < 1e-6


def test_hex8_mf_equals_eliminated_explicit(orc, hex_sys):
    s, _, _ = hex_sys
    node, comp, val = orc.bcs(3, 4, 4, 4, 1.0, 0.01)
    u = bc_state(s.n, 3, node, comp, val, u=random_vector(s.n, 0.01, 9))
    K = s.jacobian(u)
    vals, _ = s.eliminate(K, s.residual(u), u)
    x = random_vector(s.n, 1.0, 11)
    assert rel_err(s.mf_apply(u, x), s.csr_apply(vals, x)) < 1e-12


def test_hex8_patch_test_linear_field(orc):
    """A homogeneous linear-elastic cube under the benchmark BCs reproduces the uniaxial-strain
    state exactly: u_x = eps*x, u_y = u_z = -nu/(1-nu)*eps*(y|z)... checked via residual = 0 of the
    affine field that satisfies the BCs and the traction-free lateral faces."""
    n = 3
    coords, conn, phase = orc.mesh3d(n, n, n, np.zeros(0), 0.0)
    nu, eps = 0.3, 0.01
    s = orc.system(3, coords, conn, phase, [(0, 1.0, nu)], grid=(n, n, n, 1.0, 1.0, 1.0))
    s.set_dirichlet(*orc.bcs(3, n, n, n, 1.0, eps))
    u, rep = s.solve_bvp(rtol=1e-12, lin_rtol=1e-13)
    assert rep["converged"]
    X = coords.reshape(-1, 3)
    exact = np.stack([eps * X[:, 0], -nu * eps * X[:, 1], -nu * eps * X[:, 2]], 1).ravel()
    assert np.abs(u - exact).max() < 1e-12


def test_hex8_newton_explicit_vs_matrix_free(orc, hex_sys):
    s, _, _ = hex_sys
    ue, re = s.solve_bvp(rtol=1e-10, lin_rtol=1e-12, operator_kind=0)
    um, rm = s.solve_bvp(rtol=1e-10, lin_rtol=1e-12, operator_kind=1)
    assert re["converged"] and rm["converged"]
    assert rel_err(um, ue) < 1e-8


@pytest.mark.skipif(not available("ref"), reason="oracle/_ref not built")
@pytest.mark.parametrize("precond", [0, 1])
def test_restatement_bicgstab_bitwise_vs_reference(precond):
    """BiCGStab (krylov.hpp:535-620), restated for the device path's parity: identical bits."""
    R, O = Oracle("ref"), Oracle("restate")
    mesh = R.mesh2d(16, 16)
    bc = R.bcs(2, 16, 16, 0, 1.0, 0.01)
    out = []
    for lib in (R, O):
        s = lib.system(2, *mesh, LINEAR, grid=(16, 16, 0, 1.0, 1.0, 1.0))
        s.set_dirichlet(*bc)
        u = bc_state(s.n, 2, *bc)
        v, r = s.eliminate(s.jacobian(u), s.residual(u), u)
        x, rep = s.solve(0, v, -r, method=2, precond=precond, rtol=1e-12, max_iter=5000)
        out.append((x, rep))
    (xa, ra), (xb, rb) = out
    assert ra["converged"] and rb["converged"] and ra["iterations"] == rb["iterations"]
    assert np.array_equal(xa, xb) and np.array_equal(ra["residual_history"], rb["residual_history"])


@pytest.mark.skipif(not available("ref"), reason="oracle/_ref not built")
@pytest.mark.parametrize("method", [0, 1, 2], ids=["cg", "gmres", "bicgstab"])
def test_restatement_ilu0_bitwise_vs_reference(method):
    """ILU(0) (krylov.hpp:116-192), restated for the device path's parity: identical bits."""
    R, O = Oracle("ref"), Oracle("restate")
    mesh = R.mesh2d(12, 12)
    bc = R.bcs(2, 12, 12, 0, 1.0, 0.01)
    out = []
    for lib in (R, O):
        s = lib.system(2, *mesh, SVK_MIX, grid=(12, 12, 0, 1.0, 1.0, 1.0))
        s.set_dirichlet(*bc)
        u = bc_state(s.n, 2, *bc, u=random_vector(s.n, 0.01, 5))
        v, r = s.eliminate(s.jacobian(u), s.residual(u), u)
        out.append(s.solve(0, v, -r, method=method, precond=2, rtol=1e-12, max_iter=5000))
    (xa, ra), (xb, rb) = out
    assert ra["converged"] and rb["converged"] and ra["iterations"] == rb["iterations"]
    assert np.array_equal(xa, xb)

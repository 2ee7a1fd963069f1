"""CPU tests: pin the restatement's Neo-Hookean and J2 laws (north-star configs 3 and 4).

The reference has neither law (its material.hpp:13 stops at SVK), so these are pinned the way the
reference pins its own laws: an independent element integrator (numpy, no dual arithmetic, like
test_support.hpp:99-146's oracle_q4_stiffness) for the stress update, closed-form limits (small
strain -> Hooke; below yield -> Hooke), rigid-body invariance (test_element.cpp:104-153), AD tangent
vs finite differences (test_element.cpp:249-262, test_assembly.cpp:429-444), symmetry of the
hyperelastic tangent, and explicit-vs-matrix-free Newton agreement (test_newton.cpp:124-136).
"""
import numpy as np
import pytest

from oracle.pyoracle import Oracle
from tests.helpers import bc_state, fibre_mesh, random_vector, rel_err

NH_MIX = [(2, 1.0, 0.3), (0, 10.0, 0.3)]
J2_MIX = [(3, 1.0, 0.3, 0.002, 0.1), (0, 10.0, 0.3)]

G = 0.57735026918962576451
SX = np.array([-1, 1, 1, -1, -1, 1, 1, -1.0])
SY = np.array([-1, -1, 1, 1, -1, -1, 1, 1.0])
SZ = np.array([-1, -1, -1, -1, 1, 1, 1, 1.0])
QPTS = [(x, y, z) for z in (-G, G) for (x, y) in ((-G, -G), (G, -G), (G, G), (-G, G))]


def lame(E, nu):
    return E * nu / ((1 + nu) * (1 - 2 * nu)), E / (2 * (1 + nu))


def hex_grads(xc, q):
    xi, eta, zeta = q
    dn = np.stack([0.125 * SX * (1 + SY * eta) * (1 + SZ * zeta),
                   0.125 * SY * (1 + SX * xi) * (1 + SZ * zeta),
                   0.125 * SZ * (1 + SX * xi) * (1 + SY * eta)], 1)
    J = dn.T @ xc
    return dn @ np.linalg.inv(J).T, np.linalg.det(J)


def nh_piola(F, E, nu):
    lam, mu = lame(E, nu)
    kappa = lam + 2 * mu / 3
    J = np.linalg.det(F)
    Finv_T = np.linalg.inv(F).T
    return mu * J ** (-2 / 3) * (F - np.trace(F.T @ F) / 3 * Finv_T) + kappa * (J - 1) * J * Finv_T


def j2_stress(eps, h, E, nu, sy, hh):
    lam, mu = lame(E, nu)
    kappa = lam + 2 * mu / 3
    ep = np.array([[h[0], h[5], h[4]], [h[5], h[1], h[3]], [h[4], h[3], h[2]]])
    ee = eps - ep
    tr = np.trace(ee)
    s = 2 * mu * (ee - tr / 3 * np.eye(3))
    q = np.sqrt(1.5 * np.sum(s * s))
    f = q - (sy + hh * h[6])
    if f > 0:
        da = f / (3 * mu + hh)
        s = s * (1 - 3 * mu * da / q)
    return s + kappa * tr * np.eye(3)


def element_force(xc, ue, stress_fn):
    f = np.zeros((8, 3))
    for qi, q in enumerate(QPTS):
        g, detJ = hex_grads(xc, q)
        H = ue.reshape(8, 3).T @ g
        P = stress_fn(H, qi)
        f += detJ * g @ P.T
    return f.ravel()


@pytest.fixture(scope="module")
def orc():
    return Oracle("restate")


def _distorted_cube(orc, mats, seed=4):
    coords, conn, phase = orc.mesh3d(1, 1, 1, np.zeros(0), 0.0)
    coords = coords + random_vector(len(coords), 0.08, seed)
    return orc.system(3, coords, conn, np.zeros(1, np.int32), mats), coords.reshape(8, 3)[conn]


def test_neohooke_element_matches_independent_integrator(orc):
    s, xc = _distorted_cube(orc, [(2, 2.0, 0.3)])
    ue = random_vector(24, 0.1, 8)
    ref = element_force(xc, ue, lambda H, q: nh_piola(np.eye(3) + H, 2.0, 0.3))
    assert rel_err(s.element_residual(0, ue), ref) < 1e-12


def test_j2_element_matches_independent_integrator(orc):
    mat = (3, 1.0, 0.3, 0.002, 0.1)
    s, xc = _distorted_cube(orc, [mat])
    ue = random_vector(24, 0.02, 9)  # well past yield
    h = np.zeros(64)
    h[::8] = 1e-3  # nonzero committed plastic strain and alpha
    h[6::8] = 2e-3
    s.set_history(h)
    ref = element_force(xc, ue, lambda H, q: j2_stress(0.5 * (H + H.T), h[8 * q:8 * q + 8], *mat[1:]))
    assert rel_err(s.element_residual(0, ue), ref) < 1e-12


def test_neohooke_rigid_motions_and_small_strain_limit(orc):
    (coords, conn, phase), _ = fibre_mesh(orc, 3, n_fibres=2, radius=0.3)
    s = orc.system(3, coords, conn, phase, [(2, 1.0, 0.3), (2, 10.0, 0.3)])
    X = coords.reshape(-1, 3)
    th = 0.4
    R = np.array([[np.cos(th), -np.sin(th), 0], [np.sin(th), np.cos(th), 0], [0, 0, 1]])
    u_rot = (X @ R.T - X + np.array([0.1, -0.2, 0.3])).ravel()
    assert np.abs(s.residual(u_rot)).max() < 1e-13
    lin = orc.system(3, coords, conn, phase, [(0, 1.0, 0.3), (0, 10.0, 0.3)])
    u = random_vector(s.n, 1e-7, 3)  # small-strain limit: NH -> Hooke with the same (lam, mu)
    assert rel_err(s.residual(u), lin.residual(u)) < 1e-5


def test_neohooke_tangent_symmetric_and_matches_fd(orc):
    (coords, conn, phase), _ = fibre_mesh(orc, 2, n_fibres=2, radius=0.3)
    s = orc.system(3, coords, conn, phase, NH_MIX)
    u = random_vector(s.n, 0.05, 5)
    _, rows, cols = s.pattern()
    dense = np.zeros((s.n, s.n))
    dense[rows, cols] = s.jacobian(u)
    assert np.abs(dense - dense.T).max() < 1e-12 * np.abs(dense).max()
    h = 1e-6
    for j in [0, 13, 40, 80]:
        e = np.zeros(s.n)
        e[j] = h
        fd = (s.residual(u + e) - s.residual(u - e)) / (2 * h)
        assert np.abs(fd - dense[:, j]).max() < 1e-6


def test_j2_below_yield_is_hooke_and_tangent_matches_fd_past_yield(orc):
    (coords, conn, phase), _ = fibre_mesh(orc, 2, n_fibres=2, radius=0.3)
    s = orc.system(3, coords, conn, phase, J2_MIX)
    lin = orc.system(3, coords, conn, phase, [(0, 1.0, 0.3), (0, 10.0, 0.3)])
    u_small = random_vector(s.n, 1e-5, 2)
    assert rel_err(s.residual(u_small), lin.residual(u_small)) < 1e-14
    u = random_vector(s.n, 0.02, 6)
    _, rows, cols = s.pattern()
    dense = np.zeros((s.n, s.n))
    dense[rows, cols] = s.jacobian(u)
    h = 1e-7
    for j in [1, 17, 44, 70]:
        e = np.zeros(s.n)
        e[j] = h
        fd = (s.residual(u + e) - s.residual(u - e)) / (2 * h)
        assert np.abs(fd - dense[:, j]).max() < 1e-5 * np.abs(dense).max()


def test_j2_load_stepping_commits_history(orc):
    n = 3
    fib = orc.fibres(12345, 2)
    coords, conn, phase = orc.mesh3d(n, n, n, fib, 0.25)
    s = orc.system(3, coords, conn, phase, J2_MIX, grid=(n, n, n, 1.0, 1.0, 1.0))
    u, rep = s.load_stepping(0.01, 4, rtol=1e-10, lin_rtol=1e-12)
    assert rep["converged"]
    h = s.history().reshape(-1, 8, 8)
    alpha = h[:, :, 6]
    assert alpha[phase == 0].max() > 0 and np.all(alpha[phase == 1] == 0)
    # plastic strain is deviatoric
    assert np.abs(h[:, :, 0] + h[:, :, 1] + h[:, :, 2]).max() < 1e-15
    # consistency: the committed state sits on its yield surface, so re-committing at the same u
    # changes nothing beyond rounding
    s.commit_history(u)
    assert rel_err(s.history(), h.ravel()) < 1e-12


@pytest.mark.parametrize("mats", [NH_MIX, J2_MIX], ids=["neohooke", "j2"])
def test_nonlinear_newton_explicit_vs_matrix_free(orc, mats):
    n = 3
    fib = orc.fibres(12345, 2)
    coords, conn, phase = orc.mesh3d(n, n, n, fib, 0.25)
    out = []
    for kind in (0, 1):
        s = orc.system(3, coords, conn, phase, mats, grid=(n, n, n, 1.0, 1.0, 1.0))
        s.set_dirichlet(*orc.bcs(3, n, n, n, 1.0, 0.02))
        u, rep = s.solve_bvp(rtol=1e-10, lin_rtol=1e-12, operator_kind=kind, method=1, restart=30)
        assert rep["converged"] and rep["iterations"] >= 2
        out.append(u)
    assert rel_err(out[1], out[0]) < 1e-8


def test_neohooke_2d_plane_strain(orc):
    coords, conn, phase = orc.mesh2d(4, 4)
    s = orc.system(2, coords, conn, phase, [(2, 1.0, 0.3), (2, 10.0, 0.3)])
    lin = orc.system(2, coords, conn, phase, [(0, 1.0, 0.3), (0, 10.0, 0.3)])
    u = random_vector(s.n, 1e-7, 1)
    assert rel_err(s.residual(u), lin.residual(u)) < 1e-5
    X = coords.reshape(-1, 2)
    th = 0.3
    R = np.array([[np.cos(th), -np.sin(th)], [np.sin(th), np.cos(th)]])
    assert np.abs(s.residual((X @ R.T - X).ravel())).max() < 1e-13

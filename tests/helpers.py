"""Shared fixtures for the parity tests (mirrors reference tests/test_support.hpp:19-39)."""
import glob
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

SVK_MIX = [(1, 1.0, 0.3), (0, 10.0, 0.3)]   # benchmark_materials, test_support.hpp:27-30
LINEAR = [(0, 1.0, 0.3), (0, 10.0, 0.3)]    # linear_materials(10), test_support.hpp:32-35


def golden_cases():
    return sorted(glob.glob(os.path.join(GOLDEN, "*.npz")))


def load(path):
    return dict(np.load(path))


def rel_err(a, b):
    """Normwise relative error max|a-b| / max|b| (the tolerance convention of DESIGN.md §Parity)."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    den = np.abs(b).max() if b.size else 0.0
    return float(np.abs(a - b).max() / (den if den > 0 else 1.0)) if a.size else 0.0


def random_vector(n, scale, seed):
    return np.random.default_rng(seed).uniform(-scale, scale, n)


def bc_state(n_dof, dim, node, comp, val, u=None):
    u = np.zeros(n_dof) if u is None else np.array(u, np.float64)
    u[dim * np.asarray(node) + np.asarray(comp)] = val
    return u


def fibre_mesh(orc, n, n_fibres=6, radius=0.15, seed=12345, nz=None):
    fib = orc.fibres(seed, n_fibres)
    nz = n if nz is None else nz
    return orc.mesh3d(n, n, nz, fib, radius), fib

"""TEST INFRASTRUCTURE ONLY — ctypes view of the parity oracles (oracle/orc_api.h).

Loaded only by tests/, __graft_entry__.smoke() (as the checker) and bench.py's cpu_baseline /
``--impl reference`` leg. The product package never imports this module.

    Oracle("restate")  -> oracle/liboracle.so           CPU restatement (2D + 3D)
    Oracle("ref")      -> oracle/_ref/libadfem_ref.so   the reference headers compiled in place (2D)
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIBS = {
    "restate": os.path.join(HERE, "liboracle.so"),
    "ref": os.path.join(HERE, "_ref", "libadfem_ref.so"),
}


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code
        self.msg = msg


class orc_material(C.Structure):
    _fields_ = [("model", C.c_int32), ("E", C.c_double), ("nu", C.c_double),
                ("sigma_y", C.c_double), ("hardening", C.c_double)]


class orc_solver_cfg(C.Structure):
    _fields_ = [("method", C.c_int32), ("precond", C.c_int32), ("rtol", C.c_double),
                ("max_iter", C.c_int32), ("restart", C.c_int32)]


class orc_solve_report(C.Structure):
    _fields_ = [("converged", C.c_int32), ("iterations", C.c_int32), ("n_history", C.c_int32),
                ("wall_time", C.c_double), ("failure", C.c_char * 256)]


class orc_newton_cfg(C.Structure):
    _fields_ = [("rtol", C.c_double), ("atol", C.c_double), ("max_iter", C.c_int32),
                ("operator_kind", C.c_int32), ("linear", orc_solver_cfg)]


class orc_newton_report(C.Structure):
    _fields_ = [("converged", C.c_int32), ("iterations", C.c_int32),
                ("total_linear_iterations", C.c_int32), ("n_norms", C.c_int32),
                ("total_time", C.c_double), ("failure", C.c_char * 256)]


def build(quiet: bool = True) -> None:
    """Compile the oracles (make -C oracle). Builds _ref only when /root/reference is present."""
    subprocess.run(["make", "-C", HERE], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


def available(kind: str) -> bool:
    return os.path.exists(LIBS[kind])


def _p(a, ct=C.c_double):
    if a is None:
        return None
    return a.ctypes.data_as(C.POINTER(ct))


def materials_array(mats):
    arr = (orc_material * len(mats))()
    for i, m in enumerate(mats):
        model, E, nu = m[0], m[1], m[2]
        sy = float(m[3]) if len(m) > 3 else 0.0
        hh = float(m[4]) if len(m) > 4 else 0.0
        arr[i] = orc_material(int(model), float(E), float(nu), sy, hh)
    return arr


class Oracle:
    def __init__(self, kind: str = "restate"):
        path = LIBS[kind]
        if not os.path.exists(path):
            raise FileNotFoundError(f"oracle library {path} not built (run make -C oracle)")
        self.kind = kind
        L = self.lib = C.CDLL(path)
        L.orc_last_error.restype = C.c_char_p
        L.orc_system_create.restype = C.c_void_p
        L.orc_system_create.argtypes = [C.c_int32, C.c_int64, C.c_int64, C.c_void_p, C.c_void_p,
                                        C.c_void_p, C.c_int32, C.c_void_p]
        L.orc_system_create_lite.restype = C.c_void_p
        L.orc_system_create_lite.argtypes = L.orc_system_create.argtypes
        for name in ["orc_system_destroy"]:
            getattr(L, name).argtypes = [C.c_void_p]
            getattr(L, name).restype = None
        L.orc_n_dof.restype = C.c_int64
        L.orc_n_dof.argtypes = [C.c_void_p]
        L.orc_pattern_nnz.restype = C.c_int64
        L.orc_pattern_nnz.argtypes = [C.c_void_p]
        L.orc_bcs.restype = C.c_int64
        L.orc_bcs.argtypes = [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_double, C.c_double,
                              C.c_void_p, C.c_void_p, C.c_void_p]
        L.orc_fibres.argtypes = [C.c_uint64, C.c_int32, C.c_double, C.c_double, C.c_void_p]
        L.orc_mesh2d.argtypes = [C.c_int32, C.c_int32, C.c_double, C.c_double, C.c_double, C.c_double,
                                 C.c_double, C.c_void_p, C.c_void_p, C.c_void_p]
        L.orc_mesh3d.argtypes = [C.c_int32, C.c_int32, C.c_int32, C.c_double, C.c_double, C.c_double,
                                 C.c_int32, C.c_void_p, C.c_double, C.c_void_p, C.c_void_p, C.c_void_p]
        vp = C.c_void_p
        sig = {
            "orc_system_set_grid": [vp, C.c_int32, C.c_int32, C.c_int32, C.c_double, C.c_double, C.c_double],
            "orc_set_dirichlet": [vp, C.c_int64, vp, vp, vp],
            "orc_pattern": [vp, vp, vp, vp],
            "orc_residual": [vp, vp, vp],
            "orc_element_residual": [vp, C.c_int64, vp, vp],
            "orc_jacobian": [vp, vp, vp],
            "orc_diagonal": [vp, vp, vp],
            "orc_eliminate": [vp, vp, vp, vp],
            "orc_constrain_residual": [vp, vp, vp],
            "orc_mf_apply": [vp, vp, vp, vp],
            "orc_mf_apply_mt": [vp, vp, vp, vp, C.c_int32],
            "orc_mf_diagonal": [vp, vp, vp],
            "orc_mf_diagonal_mt": [vp, vp, vp, C.c_int32],
            "orc_csr_apply": [vp, vp, vp, vp],
            "orc_solve": [vp, C.c_int32, vp, vp, vp, vp, vp, vp, vp, C.c_int32],
            "orc_solve_bvp": [vp, vp, vp, vp, vp, vp, C.c_int32],
            "orc_load_stepping": [vp, C.c_double, C.c_int32, vp, vp, vp, vp, vp],
            "orc_batch_info": [vp, C.c_int32, vp, vp, vp],
            "orc_n_batches": [vp],
        }
        for k, v in sig.items():
            getattr(L, k).argtypes = v
            getattr(L, k).restype = C.c_int32
        if kind == "restate":  # J2 history exists only in the restatement (the reference has no state)
            L.orc_history_size.restype = C.c_int64
            L.orc_history_size.argtypes = [vp]
            for k in ("orc_history_commit", "orc_history_copy", "orc_history_set"):
                getattr(L, k).argtypes = [vp, vp]
                getattr(L, k).restype = C.c_int32

    def check(self, st):
        if st != 0:
            raise OracleError(st, self.lib.orc_last_error().decode())

    # ---- generators
    def mesh2d(self, nx, ny, lx=1.0, ly=1.0, center=(0.5, 0.5), radius=0.25):
        coords = np.zeros((nx + 1) * (ny + 1) * 2)
        conn = np.zeros(nx * ny * 4, np.int32)
        phase = np.zeros(nx * ny, np.int32)
        self.check(self.lib.orc_mesh2d(nx, ny, lx, ly, center[0], center[1], radius,
                                       _p(coords), _p(conn, C.c_int32), _p(phase, C.c_int32)))
        return coords, conn, phase

    def fibres(self, seed, n, lx=1.0, ly=1.0):
        out = np.zeros(2 * n)
        self.check(self.lib.orc_fibres(seed, n, lx, ly, _p(out)))
        return out

    def mesh3d(self, nx, ny, nz, fibres, radius, lx=1.0, ly=1.0, lz=1.0):
        fibres = np.ascontiguousarray(fibres, np.float64)
        coords = np.zeros((nx + 1) * (ny + 1) * (nz + 1) * 3)
        conn = np.zeros(nx * ny * nz * 8, np.int32)
        phase = np.zeros(nx * ny * nz, np.int32)
        self.check(self.lib.orc_mesh3d(nx, ny, nz, lx, ly, lz, len(fibres) // 2, _p(fibres), radius,
                                       _p(coords), _p(conn, C.c_int32), _p(phase, C.c_int32)))
        return coords, conn, phase

    def bcs(self, dim, nx, ny, nz, lx, strain):
        n = self.lib.orc_bcs(dim, nx, ny, nz, lx, strain, None, None, None)
        if n < 0:
            self.check(-n)
        node = np.zeros(n, np.int32)
        comp = np.zeros(n, np.int32)
        val = np.zeros(n)
        self.lib.orc_bcs(dim, nx, ny, nz, lx, strain, _p(node, C.c_int32), _p(comp, C.c_int32), _p(val))
        return node, comp, val

    def system(self, dim, coords, conn, phase, mats, grid=None, lite=False):
        return OracleSystem(self, dim, coords, conn, phase, mats, grid, lite)


class OracleSystem:
    def __init__(self, orc: Oracle, dim, coords, conn, phase, mats, grid=None, lite=False):
        self.o = orc
        L = orc.lib
        self.dim = dim
        self.coords = np.ascontiguousarray(coords, np.float64)
        self.conn = np.ascontiguousarray(conn, np.int32)
        self.phase = np.ascontiguousarray(phase, np.int32)
        n_nodes = len(self.coords) // dim
        n_elem = len(self.phase)
        m = materials_array(mats)
        create = L.orc_system_create_lite if lite else L.orc_system_create
        h = create(dim, n_nodes, n_elem, _p(self.coords), _p(self.conn, C.c_int32),
                   _p(self.phase, C.c_int32), len(mats), m)
        if not h:
            raise OracleError(-1, L.orc_last_error().decode())
        self.h = h
        self.n = L.orc_n_dof(h)
        if grid is not None:
            nx, ny, nz, lx, ly, lz = grid
            orc.check(L.orc_system_set_grid(h, nx, ny, nz, lx, ly, lz))

    def __del__(self):
        if getattr(self, "h", None):
            self.o.lib.orc_system_destroy(self.h)
            self.h = None

    def _c(self, st):
        self.o.check(st)

    def set_dirichlet(self, node, comp, value):
        node = np.ascontiguousarray(node, np.int32)
        comp = np.ascontiguousarray(comp, np.int32)
        value = np.ascontiguousarray(value, np.float64)
        self._c(self.o.lib.orc_set_dirichlet(self.h, len(node), _p(node, C.c_int32), _p(comp, C.c_int32), _p(value)))

    def pattern(self):
        nnz = self.o.lib.orc_pattern_nnz(self.h)
        rp = np.zeros(self.n + 1, np.int64)
        rows = np.zeros(nnz, np.int32)
        cols = np.zeros(nnz, np.int32)
        self._c(self.o.lib.orc_pattern(self.h, _p(rp, C.c_int64), _p(rows, C.c_int32), _p(cols, C.c_int32)))
        return rp, rows, cols

    def nnz(self):
        return self.o.lib.orc_pattern_nnz(self.h)

    def batches(self):
        out = []
        nb = self.o.lib.orc_n_batches(self.h)
        nd = 8 if self.dim == 2 else 24
        for b in range(nb):
            sz = C.c_int64()
            self._c(self.o.lib.orc_batch_info(self.h, b, C.byref(sz), None, None))
            ids = np.zeros(sz.value, np.int32)
            dm = np.zeros(sz.value * nd, np.int32)
            self._c(self.o.lib.orc_batch_info(self.h, b, C.byref(sz), _p(ids, C.c_int32), _p(dm, C.c_int32)))
            out.append((ids, dm.reshape(-1, nd)))
        return out

    def _vec(self, fn, *arrays):
        out = np.zeros(self.n)
        args = [_p(np.ascontiguousarray(a, np.float64)) for a in arrays]
        self._c(fn(self.h, *args, _p(out)))
        return out

    def residual(self, u):
        return self._vec(self.o.lib.orc_residual, u)

    def element_residual(self, e, ue):
        ue = np.ascontiguousarray(ue, np.float64)
        re = np.zeros_like(ue)
        self._c(self.o.lib.orc_element_residual(self.h, e, _p(ue), _p(re)))
        return re

    def jacobian(self, u):
        out = np.zeros(self.nnz())
        u = np.ascontiguousarray(u, np.float64)
        self._c(self.o.lib.orc_jacobian(self.h, _p(u), _p(out)))
        return out

    def diagonal(self, u):
        return self._vec(self.o.lib.orc_diagonal, u)

    def eliminate(self, values, residual, u):
        values = np.array(values, np.float64)
        residual = np.array(residual, np.float64)
        u = np.ascontiguousarray(u, np.float64)
        self._c(self.o.lib.orc_eliminate(self.h, _p(values), _p(residual), _p(u)))
        return values, residual

    def constrain_residual(self, residual, u):
        residual = np.array(residual, np.float64)
        u = np.ascontiguousarray(u, np.float64)
        self._c(self.o.lib.orc_constrain_residual(self.h, _p(residual), _p(u)))
        return residual

    def mf_apply(self, u, x, nthreads=1):
        out = np.zeros(self.n)
        u = np.ascontiguousarray(u, np.float64)
        x = np.ascontiguousarray(x, np.float64)
        self._c(self.o.lib.orc_mf_apply_mt(self.h, _p(u), _p(x), _p(out), nthreads))
        return out

    def mf_diagonal(self, u, nthreads=1):
        if nthreads <= 1:
            return self._vec(self.o.lib.orc_mf_diagonal, u)
        out = np.zeros(self.n)
        u = np.ascontiguousarray(u, np.float64)
        self._c(self.o.lib.orc_mf_diagonal_mt(self.h, _p(u), _p(out), nthreads))
        return out

    def csr_apply(self, values, x):
        out = np.zeros(self.n)
        values = np.ascontiguousarray(values, np.float64)
        x = np.ascontiguousarray(x, np.float64)
        self._c(self.o.lib.orc_csr_apply(self.h, _p(values), _p(x), _p(out)))
        return out

    def solve(self, op_kind, values_or_u, b, method=0, precond=1, rtol=1e-13, max_iter=10000, restart=30,
              x0=None, hist_cap=100000):
        cfg = orc_solver_cfg(method, precond, rtol, max_iter, restart)
        rep = orc_solve_report()
        hist = np.zeros(hist_cap)
        x = np.zeros(self.n)
        vu = np.ascontiguousarray(values_or_u, np.float64)
        b = np.ascontiguousarray(b, np.float64)
        x0a = None if x0 is None else np.ascontiguousarray(x0, np.float64)
        self._c(self.o.lib.orc_solve(self.h, op_kind, _p(vu), C.byref(cfg), _p(b), _p(x0a), _p(x),
                                     C.byref(rep), _p(hist), hist_cap))
        return x, dict(converged=bool(rep.converged), iterations=rep.iterations,
                       residual_history=hist[:min(rep.n_history, hist_cap)].copy(),
                       wall_time=rep.wall_time, failure=rep.failure.decode())

    def solve_bvp(self, rtol=1e-10, atol=1e-14, max_iter=25, operator_kind=0, method=0, precond=1,
                  lin_rtol=1e-13, lin_max_iter=10000, restart=30, x0=None):
        cfg = orc_newton_cfg(rtol, atol, max_iter, operator_kind,
                             orc_solver_cfg(method, precond, lin_rtol, lin_max_iter, restart))
        rep = orc_newton_report()
        norms = np.zeros(max_iter + 2)
        u = np.zeros(self.n)
        x0a = None if x0 is None else np.ascontiguousarray(x0, np.float64)
        self._c(self.o.lib.orc_solve_bvp(self.h, C.byref(cfg), _p(x0a), _p(u), C.byref(rep), _p(norms),
                                         len(norms)))
        return u, dict(converged=bool(rep.converged), iterations=rep.iterations,
                       total_linear_iterations=rep.total_linear_iterations,
                       residual_norms=norms[:rep.n_norms].copy(), total_time=rep.total_time,
                       failure=rep.failure.decode())

    def load_stepping(self, total_strain, n_steps, rtol=1e-10, atol=1e-14, max_iter=25, operator_kind=0,
                      method=0, precond=1, lin_rtol=1e-13, lin_max_iter=10000, restart=30):
        cfg = orc_newton_cfg(rtol, atol, max_iter, operator_kind,
                             orc_solver_cfg(method, precond, lin_rtol, lin_max_iter, restart))
        u = np.zeros(self.n)
        failed = C.c_int32()
        conv = C.c_int32()
        its = np.zeros(n_steps, np.int32)
        self._c(self.o.lib.orc_load_stepping(self.h, total_strain, n_steps, C.byref(cfg), _p(u),
                                             C.byref(failed), C.byref(conv), _p(its, C.c_int32)))
        return u, dict(converged=bool(conv.value), failed_step=failed.value, step_iterations=its)

    def history(self):
        out = np.zeros(self.o.lib.orc_history_size(self.h))
        self._c(self.o.lib.orc_history_copy(self.h, _p(out)))
        return out

    def set_history(self, h):
        h = np.ascontiguousarray(h, np.float64)
        self._c(self.o.lib.orc_history_set(self.h, _p(h)))

    def commit_history(self, u):
        u = np.ascontiguousarray(u, np.float64)
        self._c(self.o.lib.orc_history_commit(self.h, _p(u)))

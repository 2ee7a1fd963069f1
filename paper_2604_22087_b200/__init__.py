"""B200-native matrix-free FEM core (hot path of arXiv 2604.22087 / JetSCI).

The product is ``libafem_b200.so`` (hand-written sm_100a CUDA + the C ABI in include/afem.h).
This module is thin ctypes glue over that ABI for tests, bench.py and Python users; it mirrors the
reference's names (proj/include/adfem: build_batches, precompute_sparsity, assemble_residual,
assemble_jacobian, HandoffBuffer, explicit_operator, matrix_free_operator, run_solver, solve_bvp,
load_stepping) and its exception types. There is no CPU fallback: importing this package on a
machine without the built library raises, and every compute call runs on the GPU.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

__all__ = [
    "AfemError", "InvalidArgument", "OutOfRange", "LogicError", "DomainError", "LeaseError",
    "StaleEpochError", "CapabilityError", "FactorizationError", "InvertedElementError", "CudaError",
    "Context", "System", "Values", "HandoffBuffer", "LinearOperator", "explicit_operator",
    "matrix_free_operator", "run_solver", "fibres", "LINEAR", "SVK", "NEOHOOKE", "J2", "EXPLICIT", "MATRIX_FREE",
    "CG", "GMRES", "BICGSTAB", "DIRECT_CHOL", "DIRECT_LU", "NONE", "JACOBI", "ILU0", "lib_path", "load",
]

HERE = os.path.dirname(os.path.abspath(__file__))
# AFEM_LIBRARY: another build of the same library (A/B measurements of kernel variants)
LIB_PATH = os.environ.get("AFEM_LIBRARY") or os.path.join(HERE, "libafem_b200.so")

LINEAR, SVK = 0, 1                 # MaterialModel (material.hpp:13)
NEOHOOKE, J2 = 2, 3                # north-star laws beyond the reference (configs 3 and 4)
EXPLICIT, MATRIX_FREE = 0, 1       # OperatorKind (backend.hpp:20)
CG, GMRES, BICGSTAB, DIRECT_CHOL, DIRECT_LU = 0, 1, 2, 3, 4  # SolverMethod (krylov.hpp:20)
NONE, JACOBI, ILU0 = 0, 1, 2       # PreconKind (krylov.hpp:21)


class AfemError(RuntimeError):
    code = -1

    def __init__(self, msg, code=None):
        super().__init__(msg)
        if code is not None:
            self.code = code


class InvalidArgument(AfemError, ValueError): code = 1
class OutOfRange(AfemError, IndexError): code = 2
class LogicError(AfemError): code = 3
class DomainError(AfemError): code = 4
class LeaseError(LogicError): code = 5
class StaleEpochError(LogicError): code = 6
class CapabilityError(LogicError): code = 7
class FactorizationError(AfemError): code = 8
class InvertedElementError(AfemError): code = 9
class CudaError(AfemError): code = 10


_ERRORS = {c.code: c for c in [InvalidArgument, OutOfRange, LogicError, DomainError, LeaseError, StaleEpochError,
                               CapabilityError, FactorizationError, InvertedElementError, CudaError]}


class afem_material(C.Structure):
    _fields_ = [("model", C.c_int32), ("E", C.c_double), ("nu", C.c_double),
                ("sigma_y", C.c_double), ("hardening", C.c_double)]


class afem_solver_cfg(C.Structure):
    _fields_ = [("method", C.c_int32), ("precond", C.c_int32), ("rtol", C.c_double),
                ("max_iter", C.c_int32), ("restart", C.c_int32)]


class afem_solve_report(C.Structure):
    _fields_ = [("converged", C.c_int32), ("iterations", C.c_int32), ("n_history", C.c_int32),
                ("wall_time", C.c_double), ("failure", C.c_char * 256)]


class afem_newton_cfg(C.Structure):
    _fields_ = [("rtol", C.c_double), ("atol", C.c_double), ("max_iter", C.c_int32),
                ("operator_kind", C.c_int32), ("linear", afem_solver_cfg)]


class afem_newton_report(C.Structure):
    _fields_ = [("converged", C.c_int32), ("iterations", C.c_int32), ("total_linear_iterations", C.c_int32),
                ("n_norms", C.c_int32), ("total_time", C.c_double), ("failure", C.c_char * 256)]


class afem_system_info(C.Structure):
    _fields_ = [("dim", C.c_int32), ("nodes_per_elem", C.c_int32), ("n_nodes", C.c_int64), ("n_elem", C.c_int64),
                ("n_dof", C.c_int64), ("nnz", C.c_int64), ("n_batches", C.c_int32), ("structured", C.c_int32),
                ("nx", C.c_int32), ("ny", C.c_int32), ("nz", C.c_int32), ("device_bytes", C.c_int64)]


_lib = None


def lib_path() -> str:
    return LIB_PATH


def load():
    """Load libafem_b200.so (fails loudly: there is no fallback implementation)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is not built; run __graft_entry__.build() (make -C paper_2604_22087_b200/csrc)")
    L = C.CDLL(LIB_PATH)
    vp, i32, i64, f64 = C.c_void_p, C.c_int32, C.c_int64, C.c_double
    sigs = {
        "afem_abi_version": ([], i32),
        "afem_ctx_create": ([i32, vp], i32),
        "afem_ctx_destroy": ([vp], i32),
        "afem_ctx_set_stream": ([vp, vp], i32),
        "afem_ctx_synchronize": ([vp], i32),
        "afem_ctx_launch_count": ([vp, vp], i32),
        "afem_probe_fp64": ([vp, vp], i32),
        "afem_fibres": ([C.c_uint64, i32, f64, f64, vp], i32),
        "afem_system_create": ([vp, i32, i64, i64, vp, vp, vp, i32, vp, vp], i32),
        "afem_system_create_grid": ([vp, i32, i32, i32, i32, f64, f64, f64, i32, vp, f64, i32, vp, vp], i32),
        "afem_system_destroy": ([vp], i32),
        "afem_system_get_info": ([vp, vp], i32),
        "afem_system_mesh": ([vp, vp, vp, vp], i32),
        "afem_system_batch": ([vp, i32, vp, vp, vp], i32),
        "afem_set_dirichlet": ([vp, i64, vp, vp, vp], i32),
        "afem_set_benchmark_dirichlet": ([vp, f64], i32),
        "afem_impose_dirichlet": ([vp, vp], i32),
        "afem_pattern_nnz": ([vp, vp], i32),
        "afem_pattern": ([vp, vp, vp, vp], i32),
        "afem_residual": ([vp, vp, vp], i32),
        "afem_jacobian": ([vp, vp, vp], i32),
        "afem_diagonal": ([vp, vp, vp], i32),
        "afem_eliminate": ([vp, vp, vp, vp], i32),
        "afem_op_create_csr": ([vp, i64, i64, vp, vp, vp], i32),
        "afem_op_set_values": ([vp, vp], i32),
        "afem_eliminate_csr": ([vp, i64, i64, vp, vp, vp, vp, vp, vp, vp], i32),
        "afem_constrain_masked": ([vp, i64, vp, vp, vp, vp], i32),
        "afem_solve_bvp_ex": ([vp, vp, vp, vp, vp, vp, i32, vp, i32], i32),
        "afem_constrain_residual": ([vp, vp, vp], i32),
        "afem_csr_apply": ([vp, vp, vp, vp], i32),
        "afem_free_norm": ([vp, vp, vp], i32),
        "afem_values_create": ([vp, vp], i32),
        "afem_values_destroy": ([vp], i32),
        "afem_values_assemble": ([vp, vp], i32),
        "afem_values_eliminate": ([vp, vp, vp], i32),
        "afem_values_set": ([vp, vp], i32),
        "afem_values_device_ptr": ([vp, vp], i32),
        "afem_values_copy": ([vp, vp], i32),
        "afem_buffer_create": ([vp, vp], i32),
        "afem_buffer_destroy": ([vp], i32),
        "afem_buffer_handoff": ([vp, vp], i32),
        "afem_buffer_release": ([vp], i32),
        "afem_buffer_state": ([vp, vp, vp], i32),
        "afem_buffer_assembly_values": ([vp, vp], i32),
        "afem_buffer_solver_values": ([vp, vp], i32),
        "afem_op_create_explicit": ([vp, vp], i32),
        "afem_op_create_mf": ([vp, vp, vp], i32),
        "afem_op_destroy": ([vp], i32),
        "afem_op_kind": ([vp, vp], i32),
        "afem_op_dim": ([vp, vp], i32),
        "afem_op_apply": ([vp, vp, vp], i32),
        "afem_op_apply_async": ([vp, vp, vp], i32),
        "afem_op_diagonal": ([vp, vp], i32),
        "afem_op_csr_values": ([vp, vp], i32),
        "afem_op_uses_stencil": ([vp, vp], i32),
        "afem_solve": ([vp, vp, vp, vp, vp, vp, vp, i32], i32),
        "afem_solve_bvp": ([vp, vp, vp, vp, vp, vp, i32], i32),
        "afem_load_stepping": ([vp, f64, i32, vp, vp, vp, vp, vp], i32),
        "afem_history_size": ([vp, vp], i32),
        "afem_history_commit": ([vp, vp], i32),
        "afem_history_reset": ([vp], i32),
        "afem_history_copy": ([vp, vp], i32),
        "afem_history_set": ([vp, vp], i32),
        "afem_slab_range": ([i32, i32, i32, vp, vp], i32),
        "afem_nccl_unique_id": ([vp], i32),
        "afem_dist_create_nccl": ([vp, vp, i32, i32, vp], i32),
        "afem_thread_group_create": ([i32, vp], i32),
        "afem_thread_group_destroy": ([vp], i32),
        "afem_dist_create_threads": ([vp, vp, i32, vp], i32),
        "afem_dist_destroy": ([vp], i32),
        "afem_dist_set_benchmark_dirichlet": ([vp, vp, f64, f64], i32),
        "afem_dist_op_create_mf": ([vp, vp, vp, vp], i32),
        "afem_dist_op_create_explicit": ([vp, vp, vp, vp], i32),
        "afem_dist_solve": ([vp, vp, vp, vp, vp, vp, vp, vp, i32], i32),
        "afem_dist_dot": ([vp, vp, vp, vp, vp], i32),
        "afem_dist_assemble": ([vp, vp, vp], i32),
        "afem_dist_solve_bvp": ([vp, vp, vp, vp, vp, vp, vp, i32], i32),
        "afem_dist_load_stepping": ([vp, vp, f64, i32, f64, vp, vp, vp, vp, vp], i32),
    }
    for name, (args, res) in sigs.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    L.afem_last_error.restype = C.c_char_p
    L.afem_last_error.argtypes = []
    _lib = L
    return L


def _check(st):
    if st != 0:
        msg = _lib.afem_last_error().decode()
        raise _ERRORS.get(st, AfemError)(msg, st)


def _ptr(a):
    """Host numpy array or device tensor (anything with data_ptr()) -> void*."""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        return C.c_void_p(a.data_ptr())
    return C.c_void_p(a.ctypes.data)


def _f64(a):
    if hasattr(a, "data_ptr"):
        return a
    return np.ascontiguousarray(a, np.float64)


def _i32(a):
    if hasattr(a, "data_ptr"):
        return a
    return np.ascontiguousarray(a, np.int32)


def _mats(mats):
    """Materials as (model, E, nu) or (model, E, nu, sigma_y, hardening) tuples."""
    arr = (afem_material * len(mats))()
    for i, m in enumerate(mats):
        sy = float(m[3]) if len(m) > 3 else 0.0
        hh = float(m[4]) if len(m) > 4 else 0.0
        arr[i] = afem_material(int(m[0]), float(m[1]), float(m[2]), sy, hh)
    return arr


def fibres(seed: int, n: int, lx: float = 1.0, ly: float = 1.0) -> np.ndarray:
    """Fibre centres U(0,lx) x U(0,ly) from mt19937_64(seed), flattened (x0, y0, x1, y1, ...)."""
    L = load()
    out = np.zeros(2 * n)
    _check(L.afem_fibres(seed, n, lx, ly, _ptr(out)))
    return out


def _ctx_alive(obj) -> bool:
    """True unless the Context `obj` depends on (directly, or through its system) is already gone."""
    ctx = getattr(obj, "ctx", None)
    if ctx is None:
        sys_ = getattr(obj, "sys", None)
        ctx = getattr(sys_, "ctx", None) if sys_ is not None else None
    return ctx is None or getattr(ctx, "h", None) is not None


class Context:
    """One device + one stream. ``stream`` may be a torch.cuda.Stream (or raw cudaStream_t int)."""

    def __init__(self, device: int = 0, stream=None):
        L = load()
        h = C.c_void_p()
        _check(L.afem_ctx_create(device, C.byref(h)))
        self.h = h
        self.device = device
        if stream is not None:
            self.set_stream(stream)

    def set_stream(self, stream):
        raw = getattr(stream, "cuda_stream", stream)
        _check(_lib.afem_ctx_set_stream(self.h, C.c_void_p(int(raw))))

    def synchronize(self):
        _check(_lib.afem_ctx_synchronize(self.h))

    def probe_fp64_tflops(self) -> float:
        v = C.c_double()
        _check(_lib.afem_probe_fp64(self.h, C.byref(v)))
        return v.value

    @property
    def launches(self) -> int:
        v = C.c_int64()
        _check(_lib.afem_ctx_launch_count(self.h, C.byref(v)))
        return v.value

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.afem_ctx_destroy(self.h)
            self.h = None


class System:
    """Mesh + batches + sparsity pattern + Dirichlet table, resident in HBM."""

    def __init__(self, ctx: Context, dim: int, coords, conn, phase, materials, _handle=None):
        self.ctx = ctx
        if _handle is None:
            L = load()
            coords, conn, phase = _f64(coords), _i32(conn), _i32(phase)
            npe = 4 if dim == 2 else 8
            n_nodes = len(coords) // dim
            n_elem = len(conn) // npe
            h = C.c_void_p()
            m = _mats(materials)
            _check(L.afem_system_create(ctx.h, dim, n_nodes, n_elem, _ptr(coords), _ptr(conn), _ptr(phase),
                                        len(materials), m, C.byref(h)))
            _handle = h
        self.h = _handle
        info = afem_system_info()
        _check(_lib.afem_system_get_info(self.h, C.byref(info)))
        self.info = info
        self.dim = info.dim
        self.n = info.n_dof

    @classmethod
    def grid(cls, ctx: Context, dim: int, nx: int, ny: int, nz: int = 0, lx=1.0, ly=1.0, lz=1.0,
             inclusions=(0.5, 0.5), radius=0.25, materials=((LINEAR, 1.0, 0.3), (LINEAR, 10.0, 0.3))):
        """generate_two_phase_mesh (mesh.hpp:47-85) / its hex8 fibre twin, generated on the device."""
        L = load()
        incl = np.ascontiguousarray(inclusions, np.float64).ravel()
        h = C.c_void_p()
        m = _mats(materials)
        _check(L.afem_system_create_grid(ctx.h, dim, nx, ny, nz, lx, ly, lz, len(incl) // 2, _ptr(incl), radius,
                                         len(materials), m, C.byref(h)))
        return cls(ctx, dim, None, None, None, materials, _handle=h)

    def __del__(self):
        # a garbage cycle (e.g. a failed test's traceback) may finalise the Context first: then the
        # device objects are left to the process exit rather than destroyed against a dead context
        if getattr(self, "h", None) and _lib is not None and _ctx_alive(self):
            _lib.afem_system_destroy(self.h)
            self.h = None

    @property
    def nnz(self) -> int:
        return self.info.nnz

    def mesh(self):
        i = self.info
        coords = np.zeros(i.n_nodes * i.dim)
        conn = np.zeros(i.n_elem * i.nodes_per_elem, np.int32)
        phase = np.zeros(i.n_elem, np.int32)
        _check(_lib.afem_system_mesh(self.h, _ptr(coords), _ptr(conn), _ptr(phase)))
        return coords, conn, phase

    def batches(self):
        out = []
        nd = self.dim * self.info.nodes_per_elem
        for b in range(self.info.n_batches):
            sz = C.c_int64()
            _check(_lib.afem_system_batch(self.h, b, C.byref(sz), None, None))
            ids = np.zeros(sz.value, np.int32)
            dm = np.zeros(sz.value * nd, np.int32)
            _check(_lib.afem_system_batch(self.h, b, C.byref(sz), _ptr(ids), _ptr(dm)))
            out.append((ids, dm.reshape(-1, nd)))
        return out

    def set_dirichlet(self, node, comp, value):
        node, comp, value = _i32(node), _i32(comp), _f64(value)
        _check(_lib.afem_set_dirichlet(self.h, len(node), _ptr(node), _ptr(comp), _ptr(value)))

    def set_benchmark_dirichlet(self, strain: float):
        _check(_lib.afem_set_benchmark_dirichlet(self.h, strain))

    def impose_dirichlet(self, u):
        u = np.array(u, np.float64)
        _check(_lib.afem_impose_dirichlet(self.h, _ptr(u)))
        return u

    def pattern(self):
        rp = np.zeros(self.n + 1, np.int64)
        rows = np.zeros(self.nnz, np.int32)
        cols = np.zeros(self.nnz, np.int32)
        _check(_lib.afem_pattern(self.h, _ptr(rp), _ptr(rows), _ptr(cols)))
        return rp, rows, cols

    def _vec_op(self, fn, inp, out_len):
        inp = _f64(inp)
        out = np.zeros(out_len)
        _check(fn(self.h, _ptr(inp), _ptr(out)))
        return out

    def residual(self, u):
        return self._vec_op(_lib.afem_residual, u, self.n)

    def jacobian(self, u):
        return self._vec_op(_lib.afem_jacobian, u, self.nnz)

    def diagonal(self, u):
        return self._vec_op(_lib.afem_diagonal, u, self.n)

    def eliminate(self, values, residual, u):
        values = np.array(values, np.float64)
        residual = np.array(residual, np.float64)
        _check(_lib.afem_eliminate(self.h, _ptr(values), _ptr(residual), _ptr(_f64(u))))
        return values, residual

    def constrain_residual(self, residual, u):
        residual = np.array(residual, np.float64)
        _check(_lib.afem_constrain_residual(self.h, _ptr(residual), _ptr(_f64(u))))
        return residual

    def csr_apply(self, values, x):
        out = np.zeros(self.n)
        _check(_lib.afem_csr_apply(self.h, _ptr(_f64(values)), _ptr(_f64(x)), _ptr(out)))
        return out

    def free_norm(self, r):
        out = C.c_double()
        _check(_lib.afem_free_norm(self.h, _ptr(_f64(r)), C.byref(out)))
        return out.value

    def solve_bvp(self, rtol=1e-10, atol=1e-14, max_iter=25, operator_kind=EXPLICIT, method=CG, precond=JACOBI,
                  lin_rtol=1e-13, lin_max_iter=10000, restart=30, x0=None):
        """solve_bvp (newton.hpp:59-152) with the system's Dirichlet table."""
        cfg = afem_newton_cfg(rtol, atol, max_iter, operator_kind,
                              afem_solver_cfg(method, precond, lin_rtol, lin_max_iter, restart))
        rep = afem_newton_report()
        norms = np.zeros(max_iter + 2)
        u = np.zeros(self.n)
        x0 = None if x0 is None else _f64(x0)
        _check(_lib.afem_solve_bvp(self.h, C.byref(cfg), _ptr(x0), _ptr(u), C.byref(rep), _ptr(norms),
                                   len(norms)))
        return u, dict(converged=bool(rep.converged), iterations=rep.iterations,
                       total_linear_iterations=rep.total_linear_iterations,
                       residual_norms=norms[:rep.n_norms].copy(), total_time=rep.total_time,
                       failure=rep.failure.decode())

    def load_stepping(self, total_strain, n_steps, rtol=1e-10, atol=1e-14, max_iter=25, operator_kind=EXPLICIT,
                      method=CG, precond=JACOBI, lin_rtol=1e-13, lin_max_iter=10000, restart=30):
        """load_stepping (newton.hpp:163-186) for grid systems."""
        cfg = afem_newton_cfg(rtol, atol, max_iter, operator_kind,
                              afem_solver_cfg(method, precond, lin_rtol, lin_max_iter, restart))
        u = np.zeros(self.n)
        failed = C.c_int32()
        conv = C.c_int32()
        its = np.zeros(n_steps, np.int32)
        _check(_lib.afem_load_stepping(self.h, total_strain, n_steps, C.byref(cfg), _ptr(u), C.byref(failed),
                                       C.byref(conv), _ptr(its)))
        return u, dict(converged=bool(conv.value), failed_step=failed.value, step_iterations=its)

    # ---- J2 quadrature-point history (device resident; include/afem.h)
    def history_size(self) -> int:
        n = C.c_int64()
        _check(_lib.afem_history_size(self.h, C.byref(n)))
        return n.value

    def history(self):
        out = np.zeros(self.history_size())
        _check(_lib.afem_history_copy(self.h, _ptr(out)))
        return out

    def set_history(self, h):
        h = _f64(h)
        _check(_lib.afem_history_set(self.h, _ptr(h)))

    def commit_history(self, u):
        u = _f64(u)
        _check(_lib.afem_history_commit(self.h, _ptr(u)))

    def reset_history(self):
        _check(_lib.afem_history_reset(self.h))


class Values:
    """Assembled K(u) values in pattern order, device-resident (the CooTriplets.values of the reference)."""

    def __init__(self, sys: System):
        self.sys = sys
        h = C.c_void_p()
        _check(_lib.afem_values_create(sys.h, C.byref(h)))
        self.h = h

    def assemble(self, u):
        _check(_lib.afem_values_assemble(self.h, _ptr(_f64(u))))
        return self

    def set(self, values):
        _check(_lib.afem_values_set(self.h, _ptr(_f64(values))))
        return self

    def eliminate(self, residual, u):
        residual = np.array(residual, np.float64)
        _check(_lib.afem_values_eliminate(self.h, _ptr(residual), _ptr(_f64(u))))
        return residual

    def device_ptr(self) -> int:
        p = C.c_void_p()
        _check(_lib.afem_values_device_ptr(self.h, C.byref(p)))
        return p.value

    def numpy(self):
        out = np.zeros(self.sys.nnz)
        _check(_lib.afem_values_copy(self.h, _ptr(out)))
        return out

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None and _ctx_alive(self):
            _lib.afem_values_destroy(self.h)
            self.h = None


class HandoffBuffer:
    """HandoffBuffer (backend.hpp:33-97): lease state machine + epoch over device storage."""

    OwnedByAssembly, LeasedToSolver = 0, 1

    def __init__(self, sys: System):
        self.sys = sys
        h = C.c_void_p()
        _check(_lib.afem_buffer_create(sys.h, C.byref(h)))
        self.h = h

    def handoff(self, values: Values):
        _check(_lib.afem_buffer_handoff(self.h, C.byref(values.h)))
        values.h = None  # moved into the buffer (no copy)

    def release(self):
        _check(_lib.afem_buffer_release(self.h))

    def _state(self):
        s = C.c_int32()
        e = C.c_uint64()
        _check(_lib.afem_buffer_state(self.h, C.byref(s), C.byref(e)))
        return s.value, e.value

    @property
    def state(self):
        return self._state()[0]

    @property
    def epoch(self):
        return self._state()[1]

    def assembly_values(self) -> int:
        p = C.c_void_p()
        _check(_lib.afem_buffer_assembly_values(self.h, C.byref(p)))
        return p.value

    def solver_values(self) -> int:
        p = C.c_void_p()
        _check(_lib.afem_buffer_solver_values(self.h, C.byref(p)))
        return p.value

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None and _ctx_alive(self):
            _lib.afem_buffer_destroy(self.h)
            self.h = None


class LinearOperator:
    """LinearOperator (backend.hpp:117-195)."""

    def __init__(self, h, sys, keep=None):
        self.h = h
        self.sys = sys
        self._keep = keep
        k = C.c_int32()
        _check(_lib.afem_op_kind(self.h, C.byref(k)))
        self.kind = k.value
        self.n = sys.n

    def dim(self):
        return self.n

    def apply(self, x):
        y = np.zeros(self.n)
        _check(_lib.afem_op_apply(self.h, _ptr(_f64(x)), _ptr(y)))
        return y

    def apply_device(self, x_ptr: int, y_ptr: int):
        """Enqueue y = A x on the context stream (device pointers, no validation, no sync)."""
        _check(_lib.afem_op_apply_async(self.h, C.c_void_p(x_ptr), C.c_void_p(y_ptr)))

    def diagonal(self):
        d = np.zeros(self.n)
        _check(_lib.afem_op_diagonal(self.h, _ptr(d)))
        return d

    def csr_values_ptr(self) -> int:
        p = C.c_void_p()
        _check(_lib.afem_op_csr_values(self.h, C.byref(p)))
        return p.value

    @property
    def uses_stencil(self) -> bool:
        f = C.c_int32()
        _check(_lib.afem_op_uses_stencil(self.h, C.byref(f)))
        return bool(f.value)

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None and _ctx_alive(self):
            _lib.afem_op_destroy(self.h)
            self.h = None


def explicit_operator(buffer: HandoffBuffer) -> LinearOperator:
    """explicit_operator(buffer) (backend.hpp:199-214)."""
    h = C.c_void_p()
    _check(_lib.afem_op_create_explicit(buffer.h, C.byref(h)))
    return LinearOperator(h, buffer.sys, keep=buffer)


def matrix_free_operator(sys: System, u) -> LinearOperator:
    """matrix_free_operator(batches, u, dirichlet) (backend.hpp:222-236)."""
    h = C.c_void_p()
    _check(_lib.afem_op_create_mf(sys.h, _ptr(_f64(u)), C.byref(h)))
    return LinearOperator(h, sys)


def run_solver(op: LinearOperator, b, method=CG, precond=NONE, rtol=1e-13, max_iter=10000, restart=30, x0=None,
               hist_cap=None):
    """run_solver (backend.hpp:241-286) -> (x, report dict)."""
    cfg = afem_solver_cfg(method, precond, rtol, max_iter, restart)
    rep = afem_solve_report()
    cap = hist_cap or (max_iter + 2)
    hist = np.zeros(cap)
    x = b.new_zeros(op.n) if hasattr(b, "data_ptr") else np.zeros(op.n)  # device b -> device x
    x0 = None if x0 is None else _f64(x0)
    _check(_lib.afem_solve(op.h, C.byref(cfg), _ptr(_f64(b)), _ptr(x0), _ptr(x), C.byref(rep), _ptr(hist), cap))
    return x, dict(converged=bool(rep.converged), iterations=rep.iterations,
                   residual_history=hist[:min(rep.n_history, cap)].copy(), wall_time=rep.wall_time,
                   failure=rep.failure.decode())


# ---------------------------------------------------------------------------- multi-GPU (slab)

def slab_range(nz: int, size: int, rank: int):
    """Element layers [z0, z1) of `rank` when nz layers are split over `size` ranks (host only)."""
    L = load()
    z0, z1 = C.c_int32(), C.c_int32()
    _check(L.afem_slab_range(nz, size, rank, C.byref(z0), C.byref(z1)))
    return z0.value, z1.value


def _nccl_first():
    """libafem_b200 binds NCCL with dlopen("libnccl.so.2") and reuses an already-loaded copy. Load
    torch's (the process's NCCL of record) first, so that a later `import torch` does not meet an
    older system libnccl under the same soname."""
    try:
        import torch  # noqa: F401
    except ImportError:
        pass


def nccl_unique_id() -> bytes:
    _nccl_first()
    buf = C.create_string_buffer(128)
    _check(load().afem_nccl_unique_id(buf))
    return buf.raw


class ThreadGroup:
    """Several subdomains of one process on one device (the threads backend of the slab solver)."""

    def __init__(self, size: int):
        h = C.c_void_p()
        _check(load().afem_thread_group_create(size, C.byref(h)))
        self.h = h
        self.size = size

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.afem_thread_group_destroy(self.h)
            self.h = None


class Dist:
    """One rank of the z-slab decomposition: backend 'nccl' (one process per GPU; `uid` from
    nccl_unique_id() on rank 0, broadcast by the host) or 'threads' (a ThreadGroup)."""

    def __init__(self, ctx: Context, rank: int, size: int, backend: str = "nccl", uid: bytes = None,
                 group: ThreadGroup = None):
        L = load()
        h = C.c_void_p()
        if backend == "nccl":
            _nccl_first()
            buf = C.create_string_buffer(uid, 128)
            _check(L.afem_dist_create_nccl(ctx.h, buf, rank, size, C.byref(h)))
        else:
            _check(L.afem_dist_create_threads(ctx.h, group.h, rank, C.byref(h)))
        self.h, self.ctx, self.rank, self.size = h, ctx, rank, size
        self._group = group

    def set_benchmark_dirichlet(self, sys: System, strain: float, lx_global: float = 1.0):
        _check(_lib.afem_dist_set_benchmark_dirichlet(self.h, sys.h, strain, lx_global))

    def matrix_free_operator(self, sys: System, u) -> LinearOperator:
        h = C.c_void_p()
        _check(_lib.afem_dist_op_create_mf(self.h, sys.h, _ptr(_f64(u)), C.byref(h)))
        return LinearOperator(h, sys, keep=self)

    def explicit_operator(self, sys: System, values) -> LinearOperator:
        """The slab's eliminated assembled values (pattern order): local SpMV + the plane halo."""
        h = C.c_void_p()
        _check(_lib.afem_dist_op_create_explicit(self.h, sys.h, _ptr(_f64(values)), C.byref(h)))
        return LinearOperator(h, sys, keep=self)

    def run_solver(self, op: LinearOperator, b, method=CG, precond=JACOBI, rtol=1e-13, max_iter=10000, x0=None):
        cfg = afem_solver_cfg(method, precond, rtol, max_iter, 30)
        rep = afem_solve_report()
        cap = max_iter + 2
        hist = np.zeros(cap)
        x = b.new_zeros(op.n) if hasattr(b, "data_ptr") else np.zeros(op.n)
        x0 = None if x0 is None else _f64(x0)
        _check(_lib.afem_dist_solve(self.h, op.h, C.byref(cfg), _ptr(_f64(b)), _ptr(x0), _ptr(x), C.byref(rep),
                                    _ptr(hist), cap))
        return x, dict(converged=bool(rep.converged), iterations=rep.iterations,
                       residual_history=hist[:min(rep.n_history, cap)].copy(), wall_time=rep.wall_time,
                       failure=rep.failure.decode())

    def solve_bvp(self, sys: System, rtol=1e-10, atol=1e-14, max_iter=25, lin_rtol=1e-13, lin_max_iter=10000,
                  precond=JACOBI, x0=None, operator_kind=MATRIX_FREE, method=CG, restart=30):
        """Distributed solve_bvp (collective): matrix-free or assembled slab tangent; CG, GMRES or
        BiCGStab for the linear steps."""
        cfg = afem_newton_cfg(rtol, atol, max_iter, operator_kind,
                              afem_solver_cfg(method, precond, lin_rtol, lin_max_iter, restart))
        rep = afem_newton_report()
        norms = np.zeros(max_iter + 2)
        u = np.zeros(sys.n)
        x0 = None if x0 is None else _f64(x0)
        _check(_lib.afem_dist_solve_bvp(self.h, sys.h, C.byref(cfg), _ptr(x0), _ptr(u), C.byref(rep), _ptr(norms),
                                        len(norms)))
        return u, dict(converged=bool(rep.converged), iterations=rep.iterations,
                       total_linear_iterations=rep.total_linear_iterations,
                       residual_norms=norms[:rep.n_norms].copy(), failure=rep.failure.decode())

    def load_stepping(self, sys: System, total_strain, n_steps, lx_global=1.0, rtol=1e-10, atol=1e-14, max_iter=25,
                      lin_rtol=1e-13, lin_max_iter=10000, precond=JACOBI):
        """Distributed load_stepping (collective) with per-rank J2 history commits."""
        cfg = afem_newton_cfg(rtol, atol, max_iter, MATRIX_FREE, afem_solver_cfg(CG, precond, lin_rtol, lin_max_iter, 30))
        u = np.zeros(sys.n)
        failed, conv = C.c_int32(), C.c_int32()
        its = np.zeros(n_steps, np.int32)
        _check(_lib.afem_dist_load_stepping(self.h, sys.h, total_strain, n_steps, lx_global, C.byref(cfg), _ptr(u),
                                            C.byref(failed), C.byref(conv), _ptr(its)))
        return u, dict(converged=bool(conv.value), failed_step=failed.value, step_iterations=its)

    def assemble(self, op: LinearOperator, v):
        """Sum the shared planes of a slab-partial vector with the neighbours' partials."""
        v = v if hasattr(v, "data_ptr") else np.array(v, np.float64)
        _check(_lib.afem_dist_assemble(self.h, op.h, _ptr(v)))
        return v

    def dot(self, op: LinearOperator, a, b) -> float:
        out = C.c_double()
        _check(_lib.afem_dist_dot(self.h, op.h, _ptr(_f64(a)), _ptr(_f64(b)), C.byref(out)))
        return out.value

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None and _ctx_alive(self):
            _lib.afem_dist_destroy(self.h)
            self.h = None


def slab_system(ctx: Context, nx: int, ny: int, nz_global: int, rank: int, size: int, lx=1.0, ly=1.0, lz=1.0,
                inclusions=(), radius=0.0, materials=((LINEAR, 1.0, 0.3), (LINEAR, 10.0, 0.3))):
    """The local grid system of one z-slab (fibres are parallel to z, so the slab's phase pattern is
    the global one; the operator is translation invariant, so local z starts at 0)."""
    z0, z1 = slab_range(nz_global, size, rank)
    return System.grid(ctx, 3, nx, ny, z1 - z0, lx, ly, lz * (z1 - z0) / nz_global, inclusions, radius,
                       materials), (z0, z1)

"""The caller-CSR entry points behind the namespace-adfem drop-in (afem_op_create_csr,
afem_op_set_values, afem_eliminate_csr, afem_constrain_masked): bitwise equal to the reference's
host loops (sparse.hpp:105-115 CsrMatrix::apply, assembly.hpp:218-240 eliminate_dirichlet,
assembly.hpp:255-260 constrain_residual), restated here as sequential Python loops (IEEE doubles,
no FMA contraction)."""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def lib():
    import paper_2604_22087_b200 as afem
    return afem, afem.load()


def _p(a):
    return C.c_void_p(a.ctypes.data)


def random_csr(n, per_row, seed):
    rng = np.random.default_rng(seed)
    rp, cols = [0], []
    for i in range(n):
        c = sorted(set(rng.integers(0, n, per_row).tolist()) | {i})
        cols += c
        rp.append(len(cols))
    return np.array(rp, np.int32), np.array(cols, np.int32), rng.uniform(-1, 1, len(cols))


def test_csr_apply_bitwise_equals_host_loop(lib):
    afem, L = lib
    ctx = afem.Context(0)
    n = 300
    rp, ci, v = random_csr(n, 9, 3)
    x = np.random.default_rng(4).uniform(-1, 1, n)
    op = C.c_void_p()
    assert L.afem_op_create_csr(ctx.h, n, len(ci), _p(rp), _p(ci), C.byref(op)) == 0, L.afem_last_error()
    try:
        assert L.afem_op_set_values(op, _p(v)) == 0
        y = np.zeros(n)
        assert L.afem_op_apply(op, _p(x), _p(y)) == 0, L.afem_last_error()
        ref = np.zeros(n)
        for i in range(n):
            s = 0.0
            for k in range(rp[i], rp[i + 1]):
                s += float(v[k]) * float(x[ci[k]])
            ref[i] = s
        assert np.array_equal(y, ref)
        # the diagonal is the stored diagonal entry (csr_diagonal, krylov.hpp:102-111)
        d = np.zeros(n)
        assert L.afem_op_diagonal(op, _p(d)) == 0
        dref = np.array([v[k] for i in range(n) for k in range(rp[i], rp[i + 1]) if ci[k] == i])
        assert np.array_equal(d, dref)
        # a column index outside the matrix is rejected like the reference (out_of_range)
        bad = ci.copy()
        bad[5] = n
        op2 = C.c_void_p()
        assert L.afem_op_create_csr(ctx.h, n, len(bad), _p(rp), _p(bad), C.byref(op2)) == afem.OutOfRange.code
    finally:
        L.afem_op_destroy(op)


def test_eliminate_and_constrain_bitwise_equal_host_loops(lib):
    afem, L = lib
    ctx = afem.Context(0)
    n = 240
    rp, ci, v = random_csr(n, 7, 5)
    rng = np.random.default_rng(6)
    cons = (rng.random(n) < 0.2).astype(np.uint8)
    presc = rng.uniform(-0.1, 0.1, n)
    u = rng.uniform(-0.1, 0.1, n)
    r = rng.uniform(-1, 1, n)
    vg, rg = v.copy(), r.copy()
    assert L.afem_eliminate_csr(ctx.h, n, len(ci), _p(rp), _p(ci), _p(vg), _p(rg), _p(cons), _p(presc), _p(u)) == 0, \
        L.afem_last_error()
    vr, rr = v.copy(), r.copy()
    for i in range(n):
        for k in range(rp[i], rp[i + 1]):
            j = ci[k]
            if not cons[i] and cons[j]:
                rr[i] += float(vr[k]) * (float(presc[j]) - float(u[j]))
                vr[k] = 0.0
            elif cons[i]:
                vr[k] = 1.0 if i == j else 0.0
    for d in range(n):
        if cons[d]:
            rr[d] = u[d] - presc[d]
    assert np.array_equal(vg, vr) and np.array_equal(rg, rr)
    rc = r.copy()
    assert L.afem_constrain_masked(ctx.h, n, _p(rc), _p(cons), _p(presc), _p(u)) == 0
    ref = np.where(cons.astype(bool), u - presc, r)
    assert np.array_equal(rc, ref)

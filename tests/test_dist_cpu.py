"""CPU (gloo, world_size 2-3) test of the slab decomposition the multi-GPU path uses.

Each rank takes its z-slab from the product's own partition (afem_slab_range, host-only), builds the
slab's local operator with the CPU oracle, exchanges the shared node plane's partial sums with its
neighbours over gloo (the NCCL exchange of dist.cu), re-imposes the unit Dirichlet rows, and sums
owned-dof dot products with all_reduce. The assembled result must equal the global operator.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

NX, NY, NZ = 5, 4, 9
STRAIN = 0.01
MATS = [(0, 1.0, 0.3), (0, 10.0, 0.3)]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _global_problem(orc):
    fib = orc.fibres(12345, 3)
    coords, conn, phase = orc.mesh3d(NX, NY, NZ, fib, 0.3)
    g = orc.system(3, coords, conn, phase, MATS, lite=True)
    node, comp, val = orc.bcs(3, NX, NY, NZ, 1.0, STRAIN)
    g.set_dirichlet(node, comp, val)
    u = np.zeros(g.n)
    u[3 * node + comp] = val
    x = np.random.default_rng(0).uniform(-1, 1, g.n)
    return fib, g, u, x


def _slab_bcs(nzl, rank, size):
    """Global benchmark_bcs restricted to the slab (mirror of dist.cu slab_benchmark_bcs)."""
    node = lambda i, j, k: i + (NX + 1) * (j + (NY + 1) * k)  # noqa: E731
    c = [(node(0, j, k), 0, 0.0) for k in range(nzl + 1) for j in range(NY + 1)]
    if rank == 0:
        c += [(node(0, 0, 0), 1, 0.0), (node(0, 0, 0), 2, 0.0)]
    if rank == size - 1:
        c += [(node(0, 0, nzl), 1, 0.0)]
    c += [(node(NX, j, k), 0, STRAIN * 1.0) for k in range(nzl + 1) for j in range(NY + 1)]
    return [np.array([t[i] for t in c]) for i in range(3)]


def _worker(rank, size, port, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=size)
        import paper_2604_22087_b200 as afem
        from oracle.pyoracle import Oracle
        orc = Oracle("restate")
        fib, g, u, x = _global_problem(orc)
        y_global = g.mf_apply(u, x)
        z0, z1 = afem.slab_range(NZ, size, rank)
        nzl = z1 - z0
        plane = 3 * (NX + 1) * (NY + 1)
        sl = slice(plane * z0, plane * (z1 + 1))  # the slab's node planes z0..z1 (both shared planes)
        coords, conn, phase = orc.mesh3d(NX, NY, nzl, fib, 0.3, lz=nzl / NZ)
        loc = orc.system(3, coords, conn, phase, MATS, lite=True)
        node, comp, val = _slab_bcs(nzl, rank, size)
        loc.set_dirichlet(node.astype(np.int32), comp.astype(np.int32), val)
        xl, ul = x[sl].copy(), u[sl].copy()
        y = loc.mf_apply(ul, xl)
        mask = np.zeros(loc.n, bool)
        mask[3 * node + comp] = True
        # halo: add the neighbour's partial sums on each shared plane, then unit Dirichlet rows
        reqs, bufs = [], {}
        if rank > 0:
            bufs["lo"] = torch.zeros(plane, dtype=torch.float64)
            reqs += [dist.isend(torch.from_numpy(y[:plane].copy()), rank - 1), dist.irecv(bufs["lo"], rank - 1)]
        if rank < size - 1:
            bufs["hi"] = torch.zeros(plane, dtype=torch.float64)
            reqs += [dist.isend(torch.from_numpy(y[-plane:].copy()), rank + 1), dist.irecv(bufs["hi"], rank + 1)]
        for r in reqs:
            r.wait()
        if "lo" in bufs:
            y[:plane] += bufs["lo"].numpy()
        if "hi" in bufs:
            y[-plane:] += bufs["hi"].numpy()
        y[mask] = xl[mask]
        err = float(np.abs(y - y_global[sl]).max() / np.abs(y_global).max())
        # owned dot (the bottom plane belongs to rank - 1)
        off = plane if rank > 0 else 0
        d = torch.tensor([float(np.dot(xl[off:], y[off:]))], dtype=torch.float64)
        dist.all_reduce(d)
        dot_err = abs(d.item() - float(np.dot(x, y_global))) / abs(float(np.dot(x, y_global)))
        q.put((rank, err, dot_err, (z0, z1)))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - surfaced by the assertion below
        q.put((rank, repr(e), None, None))


@pytest.mark.parametrize("size", [2, 3])
def test_slab_decomposition_gloo(size):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, size, port, q)) for r in range(size)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(size)]
    for p in procs:
        p.join(timeout=60)
    res.sort()
    ranges = [r[3] for r in res]
    assert all(isinstance(r[1], float) for r in res), res
    assert ranges[0][0] == 0 and ranges[-1][1] == NZ
    assert all(ranges[k][1] == ranges[k + 1][0] for k in range(size - 1))
    for rank, err, dot_err, _ in res:
        assert err < 1e-12, (rank, err)
        assert dot_err < 1e-12, (rank, dot_err)


def _halo(y, rank, size, plane):
    """Neighbour partial sums added into the two shared planes (dist.cu k_halo_fin's assembly)."""
    reqs, bufs = [], {}
    if rank > 0:
        bufs["lo"] = torch.zeros(plane, dtype=torch.float64)
        reqs += [dist.isend(torch.from_numpy(y[:plane].copy()), rank - 1), dist.irecv(bufs["lo"], rank - 1)]
    if rank < size - 1:
        bufs["hi"] = torch.zeros(plane, dtype=torch.float64)
        reqs += [dist.isend(torch.from_numpy(y[-plane:].copy()), rank + 1), dist.irecv(bufs["hi"], rank + 1)]
    for r in reqs:
        r.wait()
    if "lo" in bufs:
        y[:plane] += bufs["lo"].numpy()
    if "hi" in bufs:
        y[-plane:] += bufs["hi"].numpy()
    return y


def _cg_worker(rank, size, port, q):
    """dist.cu dist_solve restated over gloo: single-reduction (Chronopoulos-Gear) Jacobi-PCG on
    the slab operator, ONE all_reduce of (r.u, r.r, u.Au) per iteration, against the oracle's
    single-domain CG (krylov.hpp:350-408) on the global operator."""
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        dist.init_process_group("gloo", rank=rank, world_size=size)
        import paper_2604_22087_b200 as afem
        from oracle.pyoracle import Oracle
        orc = Oracle("restate")
        fib, g, u, _ = _global_problem(orc)
        b = np.random.default_rng(7).uniform(-1, 1, g.n)
        rtol = 1e-10
        xg, rg = g.solve(1, u, b, method=0, precond=1, rtol=rtol)
        z0, z1 = afem.slab_range(NZ, size, rank)
        nzl = z1 - z0
        plane = 3 * (NX + 1) * (NY + 1)
        sl = slice(plane * z0, plane * (z1 + 1))
        coords, conn, phase = orc.mesh3d(NX, NY, nzl, fib, 0.3, lz=nzl / NZ)
        loc = orc.system(3, coords, conn, phase, MATS, lite=True)
        node, comp, val = _slab_bcs(nzl, rank, size)
        loc.set_dirichlet(node.astype(np.int32), comp.astype(np.int32), val)
        ul, bl = u[sl].copy(), b[sl].copy()
        mask = np.zeros(loc.n, bool)
        mask[3 * node + comp] = True
        off = plane if rank > 0 else 0
        ncoll = [0]

        def apply(v):
            y = _halo(loc.mf_apply(ul, v), rank, size, plane)
            y[mask] = v[mask]
            return y

        def allreduce(vals):
            ncoll[0] += 1
            t = torch.tensor(vals, dtype=torch.float64)
            dist.all_reduce(t)
            return t.numpy()

        diag = _halo(loc.mf_diagonal(ul), rank, size, plane)
        diag[mask] = 1.0
        inv = 1.0 / diag
        bn = float(np.sqrt(allreduce([float(bl[off:] @ bl[off:])])[0]))
        x = np.zeros(loc.n)
        r = bl.copy()
        uu = inv * r
        w = apply(uu)
        gam, rr, dlt = allreduce([r[off:] @ uu[off:], r[off:] @ r[off:], uu[off:] @ w[off:]])
        p, s = np.zeros(loc.n), np.zeros(loc.n)
        it, gold, aold, c0 = 0, 0.0, 0.0, ncoll[0]
        while it < 10000:
            if it > 0 and np.sqrt(rr) / bn <= rtol:
                break
            beta = gam / gold if it > 0 else 0.0
            pap = dlt - beta * gam / aold if it > 0 else dlt
            alpha = gam / pap
            p = uu + beta * p
            s = w + beta * s
            x += alpha * p
            r -= alpha * s
            uu = inv * r
            w = apply(uu)
            gold, aold = gam, alpha
            gam, rr, dlt = allreduce([r[off:] @ uu[off:], r[off:] @ r[off:], uu[off:] @ w[off:]])
            it += 1
        per_it = (ncoll[0] - c0) / max(it, 1)
        xerr = float(np.abs(x - xg[sl]).max() / np.abs(xg).max())
        q.put((rank, xerr, it, rg["iterations"], per_it))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - surfaced by the assertion below
        q.put((rank, repr(e), None, None, None))


@pytest.mark.parametrize("size", [2, 3])
def test_single_reduction_slab_cg_gloo(size):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_cg_worker, args=(r, size, port, q)) for r in range(size)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(size)]
    for p in procs:
        p.join(timeout=60)
    assert all(isinstance(r[1], float) for r in res), res
    for rank, xerr, it, it_ref, per_it in res:
        assert xerr <= 1e-8, (rank, xerr)
        assert abs(it - it_ref) <= 2, (rank, it, it_ref)
        assert per_it == 1.0, (rank, per_it)  # one collective per iteration

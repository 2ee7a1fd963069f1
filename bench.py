#!/usr/bin/env python
"""bench.py — BASELINE.json metric: matrix-free operator DOFs/s & CG solve time.

Workload (BASELINE.json configs[1], "config 2"): 3D linear-elastic hex8 RVE, 128^3 elements
(6.44 M dofs), random z-parallel fibres from mt19937_64(12345) (E_m = 1, E_f = 10, nu = 0.3),
benchmark BCs at 1% strain, state u0 = BC-consistent; fp64 matrix-free K(u0) x and Jacobi-PCG.

  step      one matrix-free operator apply y = K x over the whole mesh (inputs resident in HBM);
            back-to-back applies rotate over several (x, y) pairs whose combined footprint is 4x
            the L2 (one event pair around all steps), so every apply reads x from HBM and pays
            the write-back of the y lines earlier applies left dirty in L2
  value     whole-job DOFs/s = global n_dof * steps / max-over-ranks(time of the K applies)
  e2e       the same metric through the C ABI (afem_op_apply) with pinned HOST x/y buffers:
            H2D of x and D2H of y inside every step
  cg        one Jacobi-PCG solve (rtol 1e-8) of K du = -R(u0) on the device: solve time,
            iterations, true relative residual; at N > 1 the gathered solution is compared with a
            1-GPU solve of the same global RVE (cg.check_vs_1gpu)
  roofline  HBM: SURVEY §8(d) algorithmic bytes B_MF = 17 n_dof + 33 n_elem per apply; FP64:
            F_MF = 2 nnz(K) per apply against the live-probed DFMA peak
  cpu_baseline  the CPU restatement (oracle/, the reference has no hex8) timed on this host on a
            z-slab sample of the same mesh: ONE core (the reference's execution model), with the
            threaded port's all-cores figure beside it; its Jacobi-PCG seconds per iteration
            (extrapolated to the full solve) and one complete 16^3 solve on CPU and GPU

--impl reference runs the CPU path only (oracle port, all host threads) on the same metric/config.
Multi-GPU (torchrun, N > 1): --scaling weak (default) — the global RVE is 128 x 128 x (128 N)
elements, each rank owns 128 element layers; --scaling strong — one 128^3 (or --n) RVE split into
N z-slabs. Every apply adds the shared node planes over NCCL and the CG dot products are NCCL
allreduces. Time is the max over ranks.
"""
import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "matrix-free operator DOFs/s & CG solve time at 1/2/4/8 B200 vs host-CPU ref"
UNIT = "DOF/s"
SEED = 12345
N_FIBRES = 40
RADIUS = 0.05
MATS = [(0, 1.0, 0.3), (0, 10.0, 0.3)]
STRAIN = 0.01


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=50)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--n", type=int, default=128, help="elements per axis")
    p.add_argument("--no-cg", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--e2e-steps", type=int, default=10)
    p.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                   help="weak: n^3 elements per GPU (z-stacked); strong: one n^3 RVE split into z-slabs")
    p.add_argument("--no-check", action="store_true", help="N>1: skip the 1-GPU re-solve of the global system")
    return p.parse_args()


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        d = json.load(open(path))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(n):
    """dram bytes per apply of the dominant kernel from the committed ncu --set full summary."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if not os.path.exists(path):
        return None
    d = json.load(open(path))
    rec = d.get(f"n{n}")
    return None if rec is None else rec.get("dram_bytes_per_apply")


class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.sw_power_cap,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,utilization.gpu")

    def __init__(self, device, period_ms=100):
        self.device = device
        self.period_ms = period_ms
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", str(self.period_ms)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        rows = [r.split(",") for r in out.strip().splitlines() if r.count(",") >= 6]
        names = ["sw_power_cap", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"]
        sm, mx, reasons, loaded = [], None, set(), []
        for r in rows:
            try:
                c, m, util = float(r[0]), float(r[1]), float(r[6])
            except ValueError:
                continue
            mx = m
            sm.append(c)
            if util > 0:
                loaded.append(c)
            for k, nm in enumerate(names):
                if "Active" == r[2 + k].strip():
                    reasons.add(nm)
        use = loaded or sm
        return {"sm_mhz": float(np.median(use)) if use else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm), "samples_under_load": len(loaded)}


def host_mesh_slab(sys_, n, nz_s):
    """First nz_s element layers of the GPU-generated mesh (node / element arrays are k-major)."""
    coords, conn, phase = sys_.mesh()
    nn = (n + 1) * (n + 1) * (nz_s + 1)
    ne = n * n * nz_s
    return coords[: 3 * nn], conn[: 8 * ne], phase[:ne]


def cpu_sample(n, nz_s, threads, reps, mesh_arrays=None):
    """Time the CPU restatement's matrix-free apply on a z-slab sample; returns (DOF/s, seconds, n_dof)."""
    from oracle.pyoracle import Oracle, build
    build()
    orc = Oracle("restate")
    if mesh_arrays is None:
        fib = orc.fibres(SEED, N_FIBRES)
        coords, conn, phase = orc.mesh3d(n, n, nz_s, fib, RADIUS, lz=nz_s / n)
    else:
        coords, conn, phase = mesh_arrays
    s = orc.system(3, coords, conn, phase, MATS, lite=True)
    node, comp, val = orc.bcs(3, n, n, nz_s, 1.0, STRAIN)
    s.set_dirichlet(node, comp, val)
    u = np.zeros(s.n)
    u[3 * node + comp] = val
    x = np.random.default_rng(SEED).uniform(-1.0, 1.0, s.n)
    best = float("inf")
    for _ in range(reps):
        t0 = time.perf_counter()
        s.mf_apply(u, x, nthreads=threads)
        best = min(best, time.perf_counter() - t0)
    return s.n / best, best, s.n


def pick_slab(n, threads, target_s):
    """Calibrate the slab thickness so one CPU apply takes about target_s seconds."""
    _, t, _ = cpu_sample(n, 1, threads, 1)
    return max(1, min(n, int(target_s / max(t, 1e-6))))


def check_vs_one_gpu(afem, ctx, D, sys_, du, rep, n, nz_glob, fib, rank, world, z0, z1, dist):
    """N > 1: gather the slab-decomposed CG solution on rank 0 and compare it with a 1-GPU Jacobi-PCG
    solve of the same global RVE (same BCs, rtol 1e-8). Returns the comparison on rank 0."""
    plane = 3 * (n + 1) ** 2
    loc = du.cpu().numpy() if hasattr(du, "cpu") else np.asarray(du)
    parts = [None] * world if rank == 0 else None
    dist.gather_object((z0, z1, loc), parts, dst=0)
    if rank != 0:
        return None
    xg = np.zeros(plane * (nz_glob + 1))
    for a, b_, v in parts:
        xg[plane * a: plane * (b_ + 1)] = v
    g = afem.System.grid(ctx, 3, n, n, nz_glob, lz=nz_glob / n, inclusions=fib, radius=RADIUS, materials=MATS)
    g.set_benchmark_dirichlet(STRAIN)
    ug = g.impose_dirichlet(np.zeros(g.n))
    opg = afem.matrix_free_operator(g, ug)
    bg = -g.constrain_residual(g.residual(ug), ug)
    x1, r1 = afem.run_solver(opg, bg, method=afem.CG, precond=afem.JACOBI, rtol=1e-8, max_iter=200000)
    rel = float(np.abs(xg - x1).max() / max(np.abs(x1).max(), 1e-300))
    return {"rel_diff_u": rel, "tol": 1e-7, "ok": bool(rel <= 1e-7 and r1["converged"]),
            "iterations_1gpu": r1["iterations"], "iterations_ngpu": rep["iterations"],
            "note": "both solves stop at true relative residual <= 1e-8; u agrees to ~cond(K) * 1e-8"}


def cpu_cg_sample(mesh_arrays, n, nz_s, iters):
    """The CPU restatement's Jacobi-PCG (krylov.hpp:350-408, single thread) on a z-slab sample:
    seconds per iteration, from the difference of a 1-iteration and a (1 + iters)-iteration capped
    solve (cancels the setup: Jacobi diagonal, initial and re-verified residuals)."""
    from oracle.pyoracle import Oracle
    orc = Oracle("restate")
    coords, conn, phase = mesh_arrays
    s = orc.system(3, coords, conn, phase, MATS, lite=True)
    node, comp, val = orc.bcs(3, n, n, nz_s, 1.0, STRAIN)
    s.set_dirichlet(node, comp, val)
    u = np.zeros(s.n)
    u[3 * node + comp] = val
    b = -s.constrain_residual(s.residual(u), u)
    t = []
    its = []
    for k in (1, 1 + iters):
        t0 = time.perf_counter()
        _, rep = s.solve(1, u, b, method=0, precond=1, rtol=1e-8, max_iter=k)
        t.append(time.perf_counter() - t0)
        its.append(rep["iterations"])
    return (t[1] - t[0]) / max(its[1] - its[0], 1), its[1] - its[0], s.n


def cpu_small_solve(afem, ctx, n):
    """A complete Jacobi-PCG solve (rtol 1e-8) of the C2 problem at n^3 on the CPU restatement (one
    thread) and on the GPU: end-to-end solve seconds on both and the solution difference."""
    from oracle.pyoracle import Oracle
    fib = afem.fibres(SEED, N_FIBRES)
    g = afem.System.grid(ctx, 3, n, n, n, inclusions=fib, radius=RADIUS, materials=MATS)
    g.set_benchmark_dirichlet(STRAIN)
    ug = g.impose_dirichlet(np.zeros(g.n))
    b = -g.constrain_residual(g.residual(ug), ug)
    t0 = time.perf_counter()
    xg, rg = afem.run_solver(afem.matrix_free_operator(g, ug), b, method=afem.CG, precond=afem.JACOBI, rtol=1e-8,
                             max_iter=200000)
    gpu_s = time.perf_counter() - t0
    orc = Oracle("restate")
    coords, conn, phase = g.mesh()
    o = orc.system(3, coords, conn, phase, MATS, lite=True)
    o.set_dirichlet(*orc.bcs(3, n, n, n, 1.0, STRAIN))
    t0 = time.perf_counter()
    xo, ro = o.solve(1, ug, b, method=0, precond=1, rtol=1e-8, max_iter=200000)
    cpu_s = time.perf_counter() - t0
    return {"n": n, "n_dof": g.n, "cpu_s": cpu_s, "cpu_iterations": ro["iterations"], "gpu_s": gpu_s,
            "gpu_iterations": rg["iterations"], "speedup": cpu_s / gpu_s,
            "rel_diff_u": float(np.abs(xg - xo).max() / max(np.abs(xo).max(), 1e-300)),
            "gpu_path": "afem.run_solver (host b/x, setup + solve)"}


def cpu_baseline(n, sys_, cg):
    """cpu_baseline: the CPU restatement (oracle/, the reference has no hex8) on this host, ONE core —
    the reference's execution model; the all-threads figure of the threaded port is
    reported beside it. CG: seconds per Jacobi-PCG iteration on the same sample, extrapolated to the
    full mesh and the GPU's iteration count, plus a complete small solve on both sides."""
    import paper_2604_22087_b200 as afem
    threads = os.cpu_count() or 1
    nz1 = pick_slab(n, 1, 4.0)
    mesh1 = host_mesh_slab(sys_, n, nz1)
    val1, t1, dofs1 = cpu_sample(n, nz1, 1, 3, mesh_arrays=mesh1)
    nzt = pick_slab(n, threads, 2.0)
    valt, tt, dofst = cpu_sample(n, nzt, threads, 3, mesh_arrays=host_mesh_slab(sys_, n, nzt))
    sec_it, its, _ = cpu_cg_sample(mesh1, n, nz1, 3)
    cpu_cg = {"sec_per_iteration_sample": sec_it, "sample_iterations": its, "sample_dofs": dofs1,
              "cores": 1}
    if cg is not None:
        full = sec_it * sys_.n / dofs1
        cpu_cg.update({"extrapolated_sec_per_iteration_full": full,
                       "extrapolated_solve_s": full * cg["iterations"],
                       "gpu_solve_s": cg["solve_s"], "gpu_iterations": cg["iterations"],
                       "note": "CPU seconds/iteration x (full dofs / sample dofs) x the GPU's iteration count"})
    cpu_cg["small_full_solve"] = cpu_small_solve(afem, sys_.ctx, 16)
    return {"value": val1, "unit": UNIT, "cores": 1, "kind": "port",
            "sample": f"z-slab {n}x{n}x{nz1} elements ({dofs1} dofs) of the same mesh, MF apply, one thread, min of 3",
            "host_cores": threads,
            "all_threads": {"value": valt, "cores": threads,
                            "sample": f"z-slab {n}x{n}x{nzt} ({dofst} dofs), threaded port, min of 3"},
            "cg": cpu_cg}


def reference_arm(args, rank, world):
    """--impl reference: the CPU path (oracle port) on this host's cores, rank 0 only."""
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    nz_s = pick_slab(args.n, threads, 1.0)
    for _ in range(args.warmup):
        cpu_sample(args.n, nz_s, threads, 1)
    times = []
    dofs = 0
    for _ in range(args.steps):
        _, t, dofs = cpu_sample(args.n, nz_s, threads, 1)
        times.append(t)
    T = sum(times)
    value = dofs * len(times) / T
    sample = f"z-slab {args.n}x{args.n}x{nz_s} elements ({dofs} dofs) of the {args.n}^3 workload, one MF apply per step"
    # the CG leg of the metric: the restatement's Jacobi-PCG (single-threaded, like the reference)
    from oracle.pyoracle import Oracle
    nz1 = pick_slab(args.n, 1, 1.0)
    orc = Oracle("restate")
    mesh1 = orc.mesh3d(args.n, args.n, nz1, orc.fibres(SEED, N_FIBRES), RADIUS, lz=nz1 / args.n)
    sec_it, its, d1 = cpu_cg_sample(mesh1, args.n, nz1, 3)
    full_dofs = 3 * (args.n + 1) ** 3
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * T / len(times), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"C2 hex8 {args.n}^3 linear-elastic fibre RVE, matrix-free K(u0)x (CPU port)",
                   "parallelism": "host threads"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample,
                         "note": "threaded restatement (oracle/restate.hpp); the reference itself is single-threaded"},
        "cg": {"sec_per_iteration_sample": sec_it, "sample_dofs": d1, "sample_iterations": its, "cores": 1,
               "extrapolated_sec_per_iteration_full": sec_it * full_dofs / d1},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def ours(args, rank, world, local_rank):
    import torch

    import paper_2604_22087_b200 as afem

    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    stream = torch.cuda.current_stream()
    ctx = afem.Context(local_rank, stream=stream)
    n = args.n
    fib = afem.fibres(SEED, N_FIBRES)
    D = None
    if world > 1:
        # weak scaling over z-slabs: the global RVE is n x n x (n * world) elements of the same size
        # ([0,1]^2 x [0, world]); each rank owns n element layers; NCCL plane halo + allreduces
        uid = [afem.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        D = afem.Dist(ctx, rank, world, backend="nccl", uid=uid[0])
        nz_g = n * world if args.scaling == "weak" else n
        sys_, (z0, z1) = afem.slab_system(ctx, n, n, nz_g, rank, world, lz=nz_g / n, inclusions=fib,
                                          radius=RADIUS, materials=MATS)
        D.set_benchmark_dirichlet(sys_, STRAIN, 1.0)
    else:
        sys_ = afem.System.grid(ctx, 3, n, n, n, inclusions=fib, radius=RADIUS, materials=MATS)
        sys_.set_benchmark_dirichlet(STRAIN)
    n_dof, n_elem = sys_.n, sys_.info.n_elem
    nz_glob = n * world if args.scaling == "weak" else n
    global_dofs = 3 * (n + 1) ** 2 * (nz_glob + 1)
    u0 = sys_.impose_dirichlet(np.zeros(n_dof))
    op = D.matrix_free_operator(sys_, u0) if D else afem.matrix_free_operator(sys_, u0)
    assert op.uses_stencil, "structured stencil path not selected"
    vf = float(sys_.mesh()[2].mean())

    g = torch.Generator(device="cuda").manual_seed(SEED + rank)
    x = torch.rand(n_dof, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    # L2 policy: back-to-back applies rotate over R (x, y) pairs whose combined footprint is >= 4x
    # the 126 MB L2, so every apply streams its x from HBM and pays the write-back of the dirty y
    # lines earlier applies left in L2 (a read flush between timed applies would evict them outside
    # the events); one apply moves B_MF > L2 bytes, so the shared element data is re-read as well
    R = max(2, -(-4 * 126 * 2 ** 20 // (16 * n_dof)))
    xs_ = [x] + [x.clone() for _ in range(R - 1)]
    ys_ = [torch.empty_like(x) for _ in range(R)]
    flush = torch.ones(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
    sink = torch.empty((), dtype=torch.float64, device="cuda")

    # warm-up: >= 2 passes over the rotation (the apply graph of a pointer pair is captured on its
    # second use, outside the timed region)
    for k in range(max(args.warmup, 2 * R)):
        op.apply_device(xs_[k % R].data_ptr(), ys_[k % R].data_ptr())
    torch.cuda.synchronize()
    clocks = ClockSampler(local_rank)
    clocks.start()
    time.sleep(0.3)
    if dist:
        dist.barrier()
    torch.sum(flush, dim=0, out=sink)  # cold start: nothing of the workload in L2
    torch.cuda.synchronize()
    e_start, e_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = ctx.launches
    e_start.record(stream)
    for k in range(args.steps):
        op.apply_device(xs_[k % R].data_ptr(), ys_[k % R].data_ptr())
    e_end.record(stream)
    launches = ctx.launches - l0
    torch.cuda.synchronize()
    T = e_start.elapsed_time(e_end)
    y = ys_[(args.steps - 1) % R]
    del xs_[1:], ys_[:-1]
    if dist:
        t = torch.tensor([T], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        T = float(t.item())
        dist.barrier()
    t_apply = T / args.steps * 1e-3  # s per apply (max over ranks)
    value = global_dofs * args.steps / (T * 1e-3)

    clk = clocks.stop()

    # CG solve time (device-resident, Jacobi-PCG, rtol 1e-8): K du = -R(u0). Timed outside the
    # nvidia-smi polling window (the poller contends for the driver lock the CG loop's per-chunk
    # synchronisations need); clocks are sampled again at a 1 s period around it.
    cg = None
    if not args.no_cg:
        r_loc = sys_.residual(u0)
        if D:  # shared planes hold slab-partial residuals: assemble before constraining
            r_loc = D.assemble(op, r_loc)
        b = -torch.from_numpy(sys_.constrain_residual(r_loc, u0)).cuda()
        solver = D.run_solver if D else afem.run_solver
        cg_clk = ClockSampler(local_rank, period_ms=1000)
        cg_clk.start()
        best = None
        for _ in range(2):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(stream)
            du, rep = solver(op, b, method=afem.CG, precond=afem.JACOBI, rtol=1e-8, max_iter=200000)
            e1.record(stream)
            torch.cuda.synchronize()
            solve_s = e0.elapsed_time(e1) * 1e-3
            if best is None or solve_s < best[0]:
                best = (solve_s, rep)
        solve_s, rep = best
        check = None
        if D and not args.no_check:
            check = check_vs_one_gpu(afem, ctx, D, sys_, du, rep, n, nz_glob, fib, rank, world, z0, z1, dist)
        cg = {"check_vs_1gpu": check,"solve_s": solve_s, "iterations": rep["iterations"], "converged": rep["converged"],
              "true_rel_residual": float(rep["residual_history"][-1]), "rtol": 1e-8, "precond": "jacobi",
              "ms_per_iteration": 1e3 * solve_s / max(rep["iterations"], 1), "best_of": 2,
              "clocks": cg_clk.stop()}

    # end to end through the C ABI with pinned host buffers
    xh = x.cpu().pin_memory()
    yh = torch.empty_like(xh).pin_memory()
    lib = afem.load()
    import ctypes as C
    for _ in range(2):
        lib.afem_op_apply(op.h, C.c_void_p(xh.data_ptr()), C.c_void_p(yh.data_ptr()))
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        st = lib.afem_op_apply(op.h, C.c_void_p(xh.data_ptr()), C.c_void_p(yh.data_ptr()))
        assert st == 0, lib.afem_last_error()
    te = time.perf_counter() - t0
    if dist:
        t = torch.tensor([te], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        te = float(t.item())
    e2e = {"value": global_dofs * args.e2e_steps / te, "unit": UNIT, "h2d_bytes_per_step": 8 * n_dof,
           "d2h_bytes_per_step": 8 * n_dof, "path": "afem_op_apply(op, pinned host x, pinned host y)"}
    if cg is not None:
        bh = b.cpu().numpy()
        t0 = time.perf_counter()
        _, rep2 = solver(op, bh, method=afem.CG, precond=afem.JACOBI, rtol=1e-8, max_iter=200000)
        e2e["cg_solve_s"] = time.perf_counter() - t0
        e2e["cg_iterations"] = rep2["iterations"]

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return

    hbm_peak, peak_src = peaks()
    b_mf = 17 * n_dof + 33 * n_elem
    achieved = b_mf / t_apply / 1e9
    fp64_peak = ctx.probe_fp64_tflops()
    f_mf = 2.0 * sys_.nnz
    roof = {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s", "frac": achieved / hbm_peak,
            "traffic": ncu_traffic(n), "peak_source": peak_src,
            "algorithmic_bytes_per_apply": b_mf, "kernel": "matrix-free apply (k_stencil_main + edge + fix)",
            "fp64": {"achieved_tflops": f_mf / t_apply / 1e12, "peak_tflops": fp64_peak,
                     "frac": f_mf / t_apply / 1e12 / fp64_peak, "flops_per_apply": f_mf,
                     "peak_source": "measured live (afem_probe_fp64 DFMA chains)"}}

    cpu = None
    if world == 1 and not args.no_cpu:
        cpu = cpu_baseline(n, sys_, cg)

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * t_apply, "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"C2 hex8 {n}^3 linear-elastic fibre RVE, matrix-free K(u0)x + Jacobi-PCG",
                   "elements": n_elem, "n_dof": n_dof, "nnz_K": sys_.nnz, "fibres": N_FIBRES, "radius": RADIUS,
                   "fibre_volume_fraction": vf, "E": [1.0, 10.0], "nu": 0.3, "strain": STRAIN,
                   "l2": (f"inputs larger than L2: {R} rotating (x, y) pairs ({R * 16 * n_dof / 2**20:.0f} MiB), "
                          "back-to-back applies, one event pair around all steps; B_MF per apply "
                          f"{(17 * n_dof + 33 * n_elem) / 2**20:.0f} MiB > 126 MB L2"),
                   "scaling": args.scaling,
                   "global_dofs": global_dofs,
                   "parallelism": (f"z-slab decomposition over {world} GPUs (NCCL plane halo + allreduce), "
                                   f"{nz_glob // world}-{-(-nz_glob // world)} element layers per GPU"
                                   if world > 1 else "1 GPU")},
        "cg": cg, "e2e": e2e, "roofline": roof, "cpu_baseline": cpu, "clocks": clk, "gpu_launches": launches,
    }
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def main():
    args = parse()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        reference_arm(args, rank, world)
    else:
        ours(args, rank, world, local_rank)


if __name__ == "__main__":
    main()

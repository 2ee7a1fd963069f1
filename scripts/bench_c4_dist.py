#!/usr/bin/env python
"""Config 4 slab-sharded: J2 hex8 RVE N x N x N, 10 load steps to 2 % strain, one process per GPU
(torchrun), each rank a z-slab with its own Gauss-point history in HBM; distributed Newton with the
matrix-free tangent and the distributed Jacobi-PCG (NCCL plane halo + allreduced dots).

  python -m torch.distributed.run --nproc-per-node G --master-addr 127.0.0.1 scripts/bench_c4_dist.py --size 64
Prints one JSON line on rank 0 (wall time of the whole load path, max over ranks).
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_22087_b200 as afem  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--size", type=int, default=64, help="elements per axis")
ap.add_argument("--steps", type=int, default=10)
ap.add_argument("--strain", type=float, default=0.02)
a = ap.parse_args()
rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
local = int(os.environ.get("LOCAL_RANK", 0))
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
ctx = afem.Context(local)
uid = [afem.nccl_unique_id() if rank == 0 else None]
dist.broadcast_object_list(uid, src=0)
D = afem.Dist(ctx, rank, world, backend="nccl", uid=uid[0])
mats = [(afem.J2, 1.0, 0.3, 0.002, 0.1), (afem.LINEAR, 10.0, 0.3)]
s, (z0, z1) = afem.slab_system(ctx, a.size, a.size, a.size, rank, world, inclusions=afem.fibres(12345, 40), radius=0.05,
                               materials=mats)
# load path: each step warm-starts from the previous state plus the uniaxial affine increment
# (the reference's bare warm start puts the whole increment into the last element layer)
xs = s.mesh()[0][0::3]
dist.barrier()
t = time.perf_counter()
u = np.zeros(s.n)
its, ok = [], True
for st in range(1, a.steps + 1):
    D.set_benchmark_dirichlet(s, a.strain * st / a.steps, 1.0)
    x0 = u.copy()
    x0[0::3] += (a.strain / a.steps) * xs
    u, r = D.solve_bvp(s, rtol=1e-8, lin_rtol=1e-10, lin_max_iter=200000, x0=x0)
    its.append(r["iterations"])
    if not r["converged"]:
        ok = False
        break
    s.commit_history(u)
rep = {"converged": ok, "step_iterations": its}
el = torch.tensor([time.perf_counter() - t], dtype=torch.float64, device="cuda")
dist.all_reduce(el, op=dist.ReduceOp.MAX)
if rank == 0:
    print(json.dumps({"config": 4, "workload": f"C4 J2 hex8 {a.size}^3, {a.steps} load steps to {a.strain}, slab-sharded",
                      "n_gpus": world, "n_dof": 3 * (a.size + 1) ** 3, "wall_s": float(el.item()),
                      "converged": rep["converged"], "newton_iterations": list(map(int, rep["step_iterations"])),
                      "history_gb_per_rank": round(s.history_size() * 8 / 1e9, 3)}), flush=True)
dist.destroy_process_group()

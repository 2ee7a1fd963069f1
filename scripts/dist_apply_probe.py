#!/usr/bin/env python
"""Per-rank cost of the slab-decomposed apply, measured on one GPU: the single-domain apply (the
N = 1 bench path) against the overlapped schedule a rank runs at N > 1 (the shared node planes as
one-plane launches on a second stream, followed there by the plane exchange, concurrent with the
interior planes as one balanced wave; then the halo add), forced at NCCL world size 1 with
AFEM_DIST_FORCE_PIECES=1 (the exchange has no peer). usage: python
scripts/dist_apply_probe.py [--n 128]"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import sys, json, numpy as np, torch
sys.path.insert(0, %r)
import paper_2604_22087_b200 as afem
n = %d
torch.cuda.set_device(0)
stream = torch.cuda.current_stream()
ctx = afem.Context(0, stream=stream)
fib = afem.fibres(12345, 40)
mats = [(0, 1.0, 0.3), (0, 10.0, 0.3)]
out = {}
s = afem.System.grid(ctx, 3, n, n, n, inclusions=fib, radius=0.05, materials=mats)
s.set_benchmark_dirichlet(0.01)
op = afem.matrix_free_operator(s, s.impose_dirichlet(np.zeros(s.n)))
d = afem.Dist(ctx, 0, 1, backend="nccl", uid=afem.nccl_unique_id())
ss, _ = afem.slab_system(ctx, n, n, n, 0, 1, inclusions=fib, radius=0.05, materials=mats)
d.set_benchmark_dirichlet(ss, 0.01)
dop = d.matrix_free_operator(ss, ss.impose_dirichlet(np.zeros(ss.n)))
x = torch.rand(s.n, dtype=torch.float64, device="cuda") * 2 - 1
for name, o in (("single_domain", op), ("slab_overlapped", dop)):
    ys = [torch.empty_like(x) for _ in range(2)]
    for k in range(10):
        o.apply_device(x.data_ptr(), ys[k %% 2].data_ptr())
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for k in range(50):
        o.apply_device(x.data_ptr(), ys[k %% 2].data_ptr())
    e1.record(stream)
    torch.cuda.synchronize()
    out[name + "_us"] = e0.elapsed_time(e1) / 50 * 1e3
yy = [op.apply(x.cpu().numpy()), dop.apply(x.cpu().numpy())]
out["max_rel_diff"] = float(np.abs(yy[0] - yy[1]).max() / np.abs(yy[0]).max())
print(json.dumps(out))
"""


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=128)
    a = ap.parse_args()
    env = dict(os.environ, AFEM_DIST_FORCE_PIECES="1")
    p = subprocess.run([sys.executable, "-c", CHILD % (ROOT, a.n)], capture_output=True, text=True, env=env)
    print(p.stdout.strip() or p.stderr[-2000:])


if __name__ == "__main__":
    main()

"""Small driver for ncu: build the graph of a config and run the (I+L)p kernel a few times."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2101_08143_b200 as fj  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--k", type=int, default=1)
ap.add_argument("--solve", action="store_true")
ap.add_argument("--scale", type=int, default=None)
a = ap.parse_args()
wl = synth.make_config(a.config, k=a.k, kinds=["uniform"] * a.k, scale=a.scale)
u, v = torch.from_numpy(wl.u).cuda(), torch.from_numpy(wl.v).cuda()
w = None if wl.w is None else torch.from_numpy(wl.w).cuda()
G = fj.Graph.from_edges(wl.n, u, v, w)
print(G.info())
x = torch.from_numpy(wl.S.copy()).cuda()
if a.k == 1:
    x = x[:, 0].contiguous()
for _ in range(3):
    y = G.apply(x)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.reps):
    y = G.apply(x)
e1.record()
e1.synchronize()
ms = e0.elapsed_time(e1) / a.reps
nnz = G.info()["nnz"]
print("spmv_ms", ms, "nnz", nnz, "Gnnz/s", nnz / ms / 1e6, "GB/s gathered", nnz * 8 * a.k / ms / 1e6)
if a.solve:
    z, q, rep = G.approxim(x)
    print(rep)
torch.cuda.synchronize()
print("ok")

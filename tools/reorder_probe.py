"""Diagnostic: does relabelling vertices by descending degree speed up the gather-bound product?
Builds the canonical CSR, times fj_time_spmv, then builds P A P^T (P: stable sort by degree,
descending) with torch ops, times it again, and solves both (quantities must agree to rounding).
  python tools/reorder_probe.py --config c5 --k 1 [--sortcols]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2101_08143_b200 as fj  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c5")
ap.add_argument("--k", type=int, default=1)
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--sortcols", action="store_true")
ap.add_argument("--order", default="degree", choices=["degree", "random"])
a = ap.parse_args()
kinds = (["uniform", "exponential", "powerlaw"] * 22)[:a.k]
wl = synth.make_config(a.config, kinds=kinds)
n = wl.n
S = torch.from_numpy(wl.S[:, :a.k].copy()).cuda()
Sq = S if a.k > 1 else S[:, 0].contiguous()
u, v = torch.from_numpy(wl.u).cuda(), torch.from_numpy(wl.v).cuda()
w = None if wl.w is None else torch.from_numpy(wl.w).cuda()
del wl
rp, col, wo, _ = fj.csr_from_edges(n, u, v, w)
del u, v
G = fj.Graph(n, rp, col, wo, validate=False)
z, q, rep = G.approxim(Sq)
z, q, rep = G.approxim(Sq)
t0 = G.time_spmv(k=a.k, reps=a.reps)
res = {"config": a.config, "k": a.k, "orig": {"spmv_ms": t0, "loop_ms": rep["ms_loop"], "iters": rep["iterations"],
                                              "D": q[0]["D"], "P": q[0]["P"]}}
G.close()
del z

torch.cuda.synchronize()
ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ev0.record()
deg = (rp[1:] - rp[:-1])
if a.order == "degree":
    new2old = torch.sort(-deg, stable=True).indices          # hubs first
else:
    new2old = torch.randperm(n, device="cuda")
old2new = torch.empty_like(new2old)
old2new[new2old] = torch.arange(n, device="cuda")
deg2 = deg[new2old]
rp2 = torch.zeros(n + 1, dtype=torch.int64, device="cuda")
rp2[1:] = torch.cumsum(deg2, 0)
shift = rp[:-1][new2old] - rp2[:-1]
idx = torch.repeat_interleave(shift, deg2, output_size=int(rp2[-1]))
idx += torch.arange(idx.numel(), device="cuda")
col2 = old2new[col[idx].long()].int()
w2 = None if wo is None else wo[idx]
del idx
if a.sortcols:
    row2 = torch.repeat_interleave(torch.arange(n, device="cuda"), deg2, output_size=col2.numel())
    key = row2 * n + col2.long()
    del row2
    perm = torch.sort(key).indices
    del key
    col2 = col2[perm]
    if w2 is not None:
        w2 = w2[perm]
    del perm
ev1.record()
torch.cuda.synchronize()
build_ms = ev0.elapsed_time(ev1)
del col
G2 = fj.Graph(n, rp2, col2, w2, validate=False)
S2 = Sq[new2old].contiguous()
z2, q2, rep2 = G2.approxim(S2)
z2, q2, rep2 = G2.approxim(S2)
t1 = G2.time_spmv(k=a.k, reps=a.reps)
res["reordered"] = {"order": a.order, "sortcols": a.sortcols, "torch_build_ms": build_ms, "spmv_ms": t1,
                    "loop_ms": rep2["ms_loop"], "iters": rep2["iterations"], "D": q2[0]["D"], "P": q2[0]["P"]}
res["D_rel_diff"] = abs(q2[0]["D"] - q[0]["D"]) / abs(q[0]["D"])
print(json.dumps(res), flush=True)

"""Column-slab probe: time the PCG product of a config's graph split into S column
slabs, each slab its own square CSR (the entries of every row whose column falls in the slab), so
the sum over slabs bounds a slab-pass product whose gathered block per pass fits in L2.
  python tools/slab_probe.py --config c3 --k 3 --S 1 2 3 4 [--order natural]
One JSON line per S: per-slab product time (fj_time_spmv), their sum, and the slab footprints."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2101_08143_b200 as fj  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--k", type=int, default=3)
ap.add_argument("--S", type=int, nargs="+", default=[1, 2, 3, 4])
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--order", default="natural", choices=["natural", "degree"])
ap.add_argument("--split", default="cols", choices=["cols", "nnz"])
a = ap.parse_args()
wl = synth.make_config(a.config)
u, v = torch.from_numpy(wl.u).cuda(), torch.from_numpy(wl.v).cuda()
w = None if wl.w is None else torch.from_numpy(wl.w).cuda()
G0 = fj.Graph.from_edges(wl.n, u, v, w, order=a.order)
rp, col, wo = G0._keep
n = wl.n
kp = 1 if a.k == 1 else (2 if a.k == 2 else 4)
full = G0.time_spmv(k=a.k, reps=a.reps)
rows = torch.repeat_interleave(torch.arange(n, device="cuda"), torch.diff(rp))
c64 = col.to(torch.int64)
for S in a.S:
    if a.split == "cols":
        bnd = [n * b // S for b in range(S + 1)]
    else:
        cnt = torch.bincount(c64, minlength=n).cumsum(0)
        tot = int(cnt[-1])
        bnd = [0] + [int(torch.searchsorted(cnt, tot * b // S)) for b in range(1, S)] + [n]
    ts, nnzs = [], []
    for b in range(S):
        m = (c64 >= bnd[b]) & (c64 < bnd[b + 1])
        cb = col[m].contiguous()
        wb = None if wo is None else wo[m].contiguous()
        cntb = torch.bincount(rows[m], minlength=n)
        rpb = torch.zeros(n + 1, dtype=torch.int64, device="cuda")
        rpb[1:] = cntb.cumsum(0)
        Gb = fj.Graph(n, rpb, cb, wb, validate=False)
        ts.append(Gb.time_spmv(k=a.k, reps=a.reps))
        nnzs.append(int(cb.numel()))
        Gb.close()
        del cb, wb, rpb, m
        torch.cuda.empty_cache()
    print(json.dumps({"config": a.config, "k": a.k, "order": a.order, "split": a.split, "S": S, "full_ms": full,
                      "sum_ms": sum(ts), "slab_ms": ts, "slab_nnz": nnzs,
                      "slab_MB": [(bnd[b + 1] - bnd[b]) * kp * 8 / 1e6 for b in range(S)]}), flush=True)

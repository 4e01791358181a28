"""Per-process A/B of the row-engine variants (env knobs are read once per process):
prints one JSON line with the PCG product time (fj_time_spmv), the solve loop time and
iterations for a config, so variants can be compared with
  for e in "FJ_L2_HINT=0" "FJ_L2_HINT=1" ...; do env $e python tools/spmv_variants.py --k 3; done"""
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
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--scale", type=int, default=None)
ap.add_argument("--n", type=int, default=None)
ap.add_argument("--order", default="natural", choices=["natural", "degree"])
a = ap.parse_args()
kinds = (["uniform", "exponential", "powerlaw"] * 22)[:a.k]
wl = synth.make_config(a.config, kinds=kinds, scale=a.scale, n=a.n)
S = torch.from_numpy(wl.S[:, :a.k].copy()).cuda()
u, v = torch.from_numpy(wl.u).cuda(), torch.from_numpy(wl.v).cuda()
w = None if wl.w is None else torch.from_numpy(wl.w).cuda()
G = fj.Graph.from_edges(wl.n, u, v, w, order=a.order)
opts = fj.SolveOpts.make(use_cuda_graph=not os.environ.get("FJV_NO_GRAPH"))
z, q, rep = G.approxim(S if a.k > 1 else S[:, 0].contiguous(), opts=opts)
z, q, rep = G.approxim(S if a.k > 1 else S[:, 0].contiguous(), opts=opts)
ms = G.time_spmv(k=a.k, reps=a.reps)
Sq = S if a.k > 1 else S[:, 0].contiguous()
G.quantities(Sq, z)
torch.cuda.synchronize()
import time  # noqa: E402
t0 = time.perf_counter()
for _ in range(3):
    G.quantities(Sq, z)
quant_ms = (time.perf_counter() - t0) / 3 * 1e3
env = {k: v for k, v in os.environ.items() if k.startswith("FJ_")}
print(json.dumps({"env": env, "config": a.config, "n": wl.n, "k": a.k, "spmv_ms": ms, "loop_ms": rep["ms_loop"],
                  "ms": rep["ms"], "quant_ms": quant_ms, "iters": rep["iterations"], "rel_res": rep["rel_res_true"],
                  "D0": q[0]["D"]}), flush=True)

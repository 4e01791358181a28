"""One hot-path step on a config (for ncu launch lists)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2101_08143_b200 as fj  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--k", type=int, default=0)
a = ap.parse_args()
wl = synth.make_config(a.config, k=a.k or None)
u, v = torch.from_numpy(wl.u).cuda(), torch.from_numpy(wl.v).cuda()
w = None if wl.w is None else torch.from_numpy(wl.w).cuda()
S = torch.from_numpy(wl.S).cuda()
for _ in range(2):
    rp, col, wo, st = fj.csr_from_edges(wl.n, u, v, w)
    G = fj.Graph(wl.n, rp, col, wo, validate=False)
    z, q, r = G.approxim(S)
    G.close()
torch.cuda.synchronize()
print("ok", r)

"""Host-side phase timing of one hot-path step (diagnostics only)."""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2101_08143_b200 as fj  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
a = ap.parse_args()
wl = synth.make_config(a.config)
u, v = torch.from_numpy(wl.u).cuda(), torch.from_numpy(wl.v).cuda()
w = None if wl.w is None else torch.from_numpy(wl.w).cuda()
S = torch.from_numpy(wl.S).cuda()


def T(label, f):
    torch.cuda.synchronize()
    t = time.perf_counter()
    r = f()
    torch.cuda.synchronize()
    print(f"{label:28s} {1e3 * (time.perf_counter() - t):9.3f} ms", flush=True)
    return r


for rep in range(3):
    print("--- rep", rep)
    rp, col, wo, st = T("csr_from_edges", lambda: fj.csr_from_edges(wl.n, u, v, w))
    G = T("graph_create", lambda: fj.Graph(wl.n, rp, col, wo, validate=False))
    z, q, r = T("approxim #1", lambda: G.approxim(S))
    print("   report", {k: round(x, 3) if isinstance(x, float) else x for k, x in r.items()})
    z, q, r = T("approxim #2", lambda: G.approxim(S))
    print("   report", {k: round(x, 3) if isinstance(x, float) else x for k, x in r.items()})
    z, rr = T("solve (k cols)", lambda: G.solve(S))
    q = T("quantities", lambda: G.quantities(S, z))
    T("graph destroy", lambda: G.close())

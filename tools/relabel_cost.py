"""Diagnostic: device time of the relabelling steps (fj_degree_order, mapped vs plain CSR build,
fj_permute_rows) on a config, CUDA events around each call (median of 5)."""
import argparse
import os
import statistics
import sys

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


def T(label, f, reps=5):
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        r = f()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"{label:34s} {statistics.median(ts):8.3f} ms", flush=True)
    return r


n2o, o2n = T("degree_order", lambda: fj.degree_order(wl.n, u, v))
T("csr_from_edges", lambda: fj.csr_from_edges(wl.n, u, v, w))
T("csr_from_edges_mapped", lambda: fj.csr_from_edges(wl.n, u, v, w, old2new=o2n))
T("permute_rows S", lambda: fj.permute_rows(S, n2o))
rp, col, wo, _ = fj.csr_from_edges(wl.n, u, v, w)
m2o, m_o2n = T("csr_degree_order", lambda: fj.csr_degree_order(wl.n, rp))
T("csr_permute", lambda: fj.csr_permute(wl.n, rp, col, wo, m2o, m_o2n))
del rp, col, wo
T("Graph.from_edges natural", lambda: fj.Graph.from_edges(wl.n, u, v, w).close())
T("Graph.from_edges degree", lambda: fj.Graph.from_edges(wl.n, u, v, w, order="degree").close())
Gn = fj.Graph.from_edges(wl.n, u, v, w)
Gd = fj.Graph.from_edges(wl.n, u, v, w, order="degree")
T("approxim natural", lambda: Gn.approxim(S), reps=3)
T("approxim degree", lambda: Gd.approxim(S), reps=3)
T("graph create natural", lambda: fj.Graph(wl.n, *Gn._keep, validate=False).close(), reps=3)
T("graph create degree", lambda: fj.Graph(wl.n, *Gd._keep, validate=False).close(), reps=3)

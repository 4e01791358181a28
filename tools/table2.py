"""Table 2's error protocol on the device: sigma = |rho - rho~| / rho for each
quantity, rho from fj_exact_dense (the paper's "Exact": dense Cholesky of I+L) and rho~ from
fj_approxim (Jacobi-PCG to rtol 1e-10 + certificate), for the three opinion distributions of
P:L637-639 on seeded synthetic graphs shaped like the BASELINE configs (n <= 50000: dense limit).
Prints one line per (graph, distribution) with max sigma, the certified bound and the times."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2101_08143_b200 as fj  # noqa: E402
import synth  # noqa: E402

KEYS = ["CI", "D", "P", "C", "Idc", "PDI"]
cases = [("c3", dict(n=40000)), ("c2", dict(n=40000)), ("c4", dict(scale=15, k=3))]
for name, kw in cases:
    wl = synth.make_config(name, kinds=["uniform", "exponential", "powerlaw"], **kw)
    u, v = torch.from_numpy(wl.u).cuda(), torch.from_numpy(wl.v).cuda()
    w = None if wl.w is None else torch.from_numpy(wl.w).cuda()
    G = fj.Graph.from_edges(wl.n, u, v, w)
    S = torch.from_numpy(wl.S).cuda()
    torch.cuda.synchronize(); t = time.perf_counter()
    ze, qe = G.exact_dense(S)
    torch.cuda.synchronize(); te = time.perf_counter() - t
    za, qa, rep = G.approxim(S)
    for c, kind in enumerate(wl.kinds):
        sig = {k: abs(qe[c][k] - qa[c][k]) / qe[c][k] for k in KEYS}
        print(json.dumps({"graph": f"{name} n={wl.n} nnz={G.info()['nnz']}", "opinions": kind,
                          "sigma": sig, "max_sigma": max(sig.values()),
                          "certified_eps": qa[c]["eps"], "exact_s": te, "approxim_ms": rep["ms"],
                          "iterations": rep["iterations"]}), flush=True)
    G.close()

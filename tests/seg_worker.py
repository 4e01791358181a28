"""Subprocess body of test_segmented_product (FJ_SEG_MB is read once per process): a graph whose
gathered vectors exceed a tiny segment size, so every (I+L)p product runs as several L2 column-
segment passes (segments.cu); results checked against the oracle."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import oracle as O  # noqa: E402
import paper_2101_08143_b200 as fj  # noqa: E402

rng = np.random.default_rng(31)
n = 30000
u = np.concatenate([rng.integers(0, n, 150000), np.zeros(9000, np.int64)]).astype(np.int32)   # + a hub row
v = np.concatenate([rng.integers(0, n, 150000), rng.choice(n, 9000, replace=False)]).astype(np.int32)
wk = sys.argv[1]
w = None if wk == "unit" else rng.integers(1, 6, len(u)).astype(np.uint8)
g = O.canonical_csr(n, u, v, w)
dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
G = fj.Graph.from_edges(n, dev(u), dev(v), None if w is None else dev(w))
out = {"nseg_k1": None}
res = {}
for k in (1, 3):
    S = rng.uniform(0, 1, (n, k))
    Sd = dev(S if k > 1 else S[:, 0])
    z1, q1, r1 = G.approxim(Sd)
    z2, q2, r2 = G.approxim(Sd, opts=fj.SolveOpts.make(use_cuda_graph=False))
    Z = z1.cpu().numpy().reshape(n, k)
    err = 0.0
    for c in range(k):
        zo = O.solve_dense(g, S[:, c]) if n <= 4096 else O.solve_pcg(g, S[:, c], tol=1e-13)[0]
        qo = O.quantities(g, S[:, c], zo)
        for key in ["CI", "D", "P", "C", "Idc", "PDI"]:
            err = max(err, abs(q1[c][key] - qo[key]) / abs(qo[key]))
        err = max(err, float(np.max(np.abs(Z[:, c] - zo))))
    Y = G.apply(dev(S if k > 1 else S[:, 0])).cpu().numpy().reshape(n, k)
    aerr = max(float(np.max(np.abs(Y[:, c] - O.ipl_apply(g, S[:, c])) / (1 + np.abs(O.ipl_apply(g, S[:, c])))))
               for c in range(k))
    res[k] = {"err": err, "apply_err": aerr, "bitwise_graph_vs_loop": bool(torch.equal(z1, z2)),
              "rel_res": r1["rel_res_true"], "converged": r1["converged"], "ms_spmv": G.time_spmv(k=k, reps=2)}
print(json.dumps(res))

"""Small cases through every engine of libfj, for compute-sanitizer (memcheck / racecheck /
synccheck, one tool per run; logs under profiles/).  Each case is checked against the oracle
loosely (the sanitizer run is about memory / race / barrier errors, parity is tested elsewhere).

  python tools/sanitize_cases.py [--no-graph]
"""
import argparse
import os
import sys
import threading

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import oracle as O  # noqa: E402
import paper_2101_08143_b200 as fj  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--no-graph", action="store_true")
a = ap.parse_args()
opts = fj.SolveOpts.make(use_cuda_graph=not a.no_graph)


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def check(name, Q, g, S):
    S = S.reshape(g.n, -1)
    for c in range(S.shape[1]):
        qo = O.quantities(g, S[:, c], O.solve_dense(g, S[:, c]))
        for key in ["CI", "D", "P", "C"]:
            assert abs(Q[c][key] - qo[key]) <= 1e-7 * abs(qo[key]) + 1e-12, (name, c, key)
    print("ok", name, flush=True)


# k = 1 scalar engine, C1 (BA 2000), natural and degree-relabelled; validation on
wl = synth.make_config("c1", kinds=["uniform", "exponential", "powerlaw"])
g = O.canonical_csr(wl.n, wl.u, wl.v)
u, v = dev(wl.u), dev(wl.v)
G = fj.Graph.from_edges(wl.n, u, v, validate=True)
_, Q, _ = G.approxim(dev(wl.S[:, 0].copy()), opts=opts)
check("k1", Q, g, wl.S[:, :1])
# k = 3 vector engine (TMA tile prefetch), k = 2
_, Q, _ = G.approxim(dev(wl.S), opts=opts)
check("k3-vec", Q, g, wl.S)
_, Q, _ = G.approxim(dev(wl.S[:, :2].copy()), opts=opts)
check("k2-vec", Q, g, wl.S[:, :2])
G.close()
Gd = fj.Graph.from_edges(wl.n, u, v, order="degree")
_, Q, _ = Gd.approxim(dev(wl.S), opts=opts)
check("k3-degree-order", Q, g, wl.S)
Gd.close()
# k = 64 warp-per-row engine, weighted R-MAT scale 10 (hubs, chunked long rows, isolated rows)
w4 = synth.make_config("c4", scale=10, k=8)
g4 = O.canonical_csr(w4.n, w4.u, w4.v, w4.w)
G4 = fj.Graph.from_edges(w4.n, dev(w4.u), dev(w4.v), dev(w4.w))
S64 = np.ascontiguousarray(np.tile(w4.S, (1, 8)))
_, Q, _ = G4.approxim(dev(S64), opts=opts)
check("k64-spmm", Q[:8], g4, S64[:, :8])
# Algorithm 1 verbatim, forest columns, exact dense, CSR permutation
G4.approxim_alg1(dev(w4.S[:, 0].copy()), opts=opts)
G4.forest_columns([0, 5, 77], opts=opts)
G4.close()
print("ok f2/f4", flush=True)
# row f1: components / LCC / device opinions
lab, nc = fj.connected_components(w4.n, dev(w4.u), dev(w4.v))
fj.lcc(w4.n, dev(w4.u), dev(w4.v), dev(w4.w))
fj.opinions_generate(1000, "powerlaw", 7)
print("ok f1", flush=True)


# LOOPBACK row-partitioned path, P = 2, k = 1 and k = 3
def loop(P, S):
    from paper_2101_08143_b200 import dist as D
    comm = fj.Comm.loopback(P)
    world = D.ThreadWorld(P)
    bounds = fj.partition_rows(wl.n, u, v, P)
    out = [None] * P

    def rank_main(r):
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            Gr, _ = D.build_dist_graph(comm, r, wl.n, u, v, None, D.ThreadGroup(world, r), bounds=bounds, stream=st)
            Sl = dev(S[bounds[r]:bounds[r + 1]])
            _, q, _ = Gr.approxim(Sl, opts=opts, stream=st)
            st.synchronize()
            out[r] = q
            Gr.close()
    ts = [threading.Thread(target=rank_main, args=(r,)) for r in range(P)]
    [t.start() for t in ts]
    [t.join(600) for t in ts]
    comm.close()
    return out[0]


check("dist-P2-k1", loop(2, wl.S[:, :1].copy()), g, wl.S[:, :1])
check("dist-P2-k3", loop(2, wl.S), g, wl.S)
torch.cuda.synchronize()
print("ALL OK", flush=True)

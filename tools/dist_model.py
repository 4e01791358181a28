"""Per-iteration model of the row-partitioned path at P ranks, MEASURED rank by rank on ONE B200
(the round's boxes have one GPU; DESIGN.md §8/§10).  For each rank r of a P-way nnz-balanced
partition (fj_partition_rows) the tool builds that rank's local CSR exactly as the distributed
path does (fj_csr_rows_from_edges, fj_dist_ghosts, own columns -> [0, n_loc), ghosts -> n_loc +
index), wraps it as a square single-GPU graph of n_loc + n_ghost rows (the ghost rows empty, so the
gathered vector is the rank's extended u) and times its PCG product with fj_time_spmv (CUDA events).
The elementwise work of one Chronopoulos-Gear iteration is charged at the measured HBM copy rate;
the halo at the measured NVLink peer rate (B200_PROFILING.md: 770 GB/s per direction), overlapped
with the product's own-column pass; the allreduce at a fixed latency.

  python tools/dist_model.py --config c5 --P 1 2 4 8 [--k 1]
prints one JSON line per P; the speedup column is t_iter(1) / t_iter(P)."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2101_08143_b200 as fj  # noqa: E402
import synth  # noqa: E402

NVLINK_GBS = 770.0           # measured peer copy per direction (B200_PROFILING.md)
HALO_LAT_US = 8.0            # grouped send/recv launch + NVLink latency
ALLREDUCE_US = 12.0          # 3 KP doubles, NCCL (LL protocol) over NVSwitch

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c5")
ap.add_argument("--P", type=int, nargs="+", default=[1, 2, 4, 8])
ap.add_argument("--k", type=int, default=None)
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--order", default="natural", choices=["natural", "degree"],
                help="degree: relabel by descending degree before partitioning (fj_edge_degree_order)")
a = ap.parse_args()
wl = synth.make_config(a.config)
k = a.k or min(wl.k, 4)
kp = 1 if k == 1 else (2 if k == 2 else 4)
u = torch.from_numpy(wl.u).cuda()
v = torch.from_numpy(wl.v).cuda()
w = None if wl.w is None else torch.from_numpy(wl.w).cuda()
wb = 0 if wl.w is None else wl.w.dtype.itemsize
peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
base = None
o2n = fj.binding.edge_degree_order(wl.n, u, v)[1] if a.order == "degree" else None
for P in a.P:
    bounds = fj.partition_rows(wl.n, u, v, P, old2new=o2n)
    ranks = []
    for r in range(P):
        r0, r1 = bounds[r], bounds[r + 1]
        rp, colg, wo, nnz = fj.csr_rows_from_edges(wl.n, u, v, w, r0, r1, old2new=o2n)
        gh = fj.dist_ghosts(colg, r0, r1)
        nl, ng = r1 - r0, int(gh.numel())
        c64 = colg.to(torch.int64)
        own = (c64 >= r0) & (c64 < r1)
        loc = torch.where(own, c64 - r0, nl + torch.searchsorted(gh.to(torch.int64), c64))
        col = loc.to(torch.int32)
        rpx = torch.cat([rp, rp[-1:].expand(ng)]) if ng else rp
        G = fj.Graph(nl + ng, rpx.contiguous(), col.contiguous(), wo, validate=False)
        t_spmv = G.time_spmv(k=k, reps=a.reps)
        G.close()
        n_bnd = int(torch.unique(torch.repeat_interleave(torch.arange(nl, device="cuda"), torch.diff(rp))[~own]).numel()) if ng else 0
        # C-G step: p, s, x, r read+write, u read+write, w read, dinv read (KP-wide rows)
        elem_bytes = nl * (8 * kp * 11 + 8)
        t_elem = elem_bytes / (peak * 1e9) * 1e3
        halo_bytes = 8 * kp * ng
        t_halo = (halo_bytes / (NVLINK_GBS * 1e9) * 1e3 + HALO_LAT_US * 1e-3) if P > 1 else 0.0
        frac_own = float(own.sum()) / max(nnz, 1)
        exposed = max(0.0, t_halo - frac_own * t_spmv)   # the own-column pass covers the halo
        t_iter = t_spmv + t_elem + exposed + (ALLREDUCE_US * 1e-3 if P > 1 else 0.0)
        ranks.append({"rank": r, "n_loc": nl, "nnz_local": nnz, "n_ghost": ng, "n_boundary_rows": n_bnd,
                      "own_nnz_frac": frac_own, "t_spmv_ms": t_spmv, "t_elem_ms": t_elem,
                      "halo_MB": halo_bytes / 1e6, "t_halo_ms": t_halo, "t_iter_ms": t_iter})
        del rp, colg, wo, gh, c64, own, loc, col, rpx
        torch.cuda.empty_cache()
    t = max(x["t_iter_ms"] for x in ranks)
    if P == 1:
        base = t
    print(json.dumps({"config": a.config, "k": k, "P": P, "order": a.order, "t_iter_ms": t,
                      "speedup_vs_P1": (base / t) if base else None,
                      "max_halo_MB": max(x["halo_MB"] for x in ranks),
                      "max_t_spmv_ms": max(x["t_spmv_ms"] for x in ranks), "ranks": ranks}), flush=True)

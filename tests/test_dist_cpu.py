"""CPU tests of the row-partitioned path's host logic (rows a8/e) with world_size-2 gloo and
in-process thread groups.  The halo plan produced by paper_2101_08143_b200.dist.exchange_requests
is exercised end to end: a numpy emulation of the distributed (I+L)p (columns renumbered exactly as
fj_graph_create_dist does, halo values moved with gloo) must equal the oracle's global product, and
the distributed dot products (allreduce) must equal the global ones."""
import os
import socket
import threading

import numpy as np
import pytest

import oracle as O
from paper_2101_08143_b200 import dist as D


def _bounds_by_nnz(row_ptr, P):
    """Same rule as fj_partition_rows (first row whose prefix reaches r/P of the total)."""
    tot = int(row_ptr[-1])
    b = [0]
    for r in range(1, P):
        target = (tot // P) * r + (tot % P) * r // P
        b.append(int(np.searchsorted(row_ptr[:-1], target, side="left")))
    b.append(len(row_ptr) - 1)
    return b


def _local_plan(g, bounds, rank):
    r0, r1 = bounds[rank], bounds[rank + 1]
    a, bnd = g.row_ptr[r0], g.row_ptr[r1]
    rp = g.row_ptr[r0:r1 + 1] - a
    colg = g.col[a:bnd].astype(np.int64)
    ghosts = np.unique(colg[(colg < r0) | (colg >= r1)])
    # renumbering rule of k_renumber: own -> c - r0, ghost -> n_loc + index in the sorted ghost list
    cl = np.where((colg >= r0) & (colg < r1), colg - r0, (r1 - r0) + np.searchsorted(ghosts, colg))
    return rp, cl, ghosts


def _dist_ipl(g, bounds, rank, x_global_local, halo_vals):
    r0, r1 = bounds[rank], bounds[rank + 1]
    rp, cl, ghosts = _local_plan(g, bounds, rank)
    xe = np.concatenate([x_global_local, halo_vals])
    wf = g.wf()[g.row_ptr[r0]:g.row_ptr[r1]]
    rows = np.repeat(np.arange(r1 - r0), np.diff(rp))
    ax = np.bincount(rows, weights=wf * xe[cl], minlength=r1 - r0)
    d = np.bincount(rows, weights=wf, minlength=r1 - r0)
    return x_global_local + d * x_global_local - ax


def test_exchange_requests_threads():
    rng = np.random.default_rng(0)
    P, n = 3, 300
    bounds = [0, 90, 200, 300]
    ghost_sets = []
    for r in range(P):
        cand = np.setdiff1d(np.arange(n), np.arange(bounds[r], bounds[r + 1]))
        ghost_sets.append(np.sort(rng.choice(cand, 40, replace=False)))
    world = D.ThreadWorld(P)
    out = [None] * P

    def run(r):
        out[r] = D.exchange_requests(ghost_sets[r], bounds, D.ThreadGroup(world, r))

    ts = [threading.Thread(target=run, args=(r,)) for r in range(P)]
    [t.start() for t in ts]
    [t.join() for t in ts]
    for o in range(P):
        counts, idx = out[o]
        off = np.concatenate([[0], np.cumsum(counts)])
        for q in range(P):
            want = ghost_sets[q][D.owners(ghost_sets[q], bounds) == o] - bounds[o]
            assert np.array_equal(idx[off[q]:off[q + 1]], want.astype(np.int32))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gloo_worker(rank, P, port, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=P)
    try:
        import synth
        wl = synth.make_config("c4", scale=10, k=1)
        g = O.canonical_csr(wl.n, wl.u, wl.v, wl.w)
        bounds = _bounds_by_nnz(g.row_ptr, P)
        rp, cl, ghosts = _local_plan(g, bounds, rank)
        grp = D.TorchGroup(None, "cpu")
        counts, send_idx = D.exchange_requests(ghosts, bounds, grp)
        x = np.random.default_rng(7).normal(size=wl.n)
        r0, r1 = bounds[rank], bounds[rank + 1]
        xl = x[r0:r1]
        # halo exchange with gloo point-to-point, segment per owner in rank order
        own = D.owners(ghosts, bounds)
        halo = np.zeros(len(ghosts))
        off = np.concatenate([[0], np.cumsum(counts)])
        reqs = []
        for peer in range(P):
            if peer == rank:
                continue
            sbuf = torch.from_numpy(xl[send_idx[off[peer]:off[peer + 1]]].copy())
            reqs.append(dist.isend(sbuf, peer))
        for peer in range(P):
            if peer == rank:
                continue
            rbuf = torch.zeros(int((own == peer).sum()), dtype=torch.float64)
            dist.recv(rbuf, peer)
            halo[own == peer] = rbuf.numpy()
        for r in reqs:
            r.wait()
        y = _dist_ipl(g, bounds, rank, xl, halo)
        ref = O.ipl_apply(g, x)[r0:r1]
        err = float(np.max(np.abs(y - ref) / (1 + np.abs(ref))))
        # distributed dot product x^T (I+L) x = allreduce of the local parts
        t = torch.tensor([float(np.dot(xl, y))], dtype=torch.float64)
        dist.all_reduce(t)
        q.put((rank, err, float(t[0]), float(np.dot(x, O.ipl_apply(g, x)))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("P", [2])
def test_gloo_halo_plan_and_distributed_spmv(P):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, P, port, q)) for r in range(P)]
    [p.start() for p in procs]
    [p.join(120) for p in procs]
    assert all(p.exitcode == 0 for p in procs)
    res = [q.get(timeout=5) for _ in range(P)]
    for rank, err, dot_d, dot_g in res:
        assert err < 1e-13
        assert dot_d == pytest.approx(dot_g, rel=1e-12)


def test_bounds_rule_balances_nnz():
    import synth
    wl = synth.make_config("c4", scale=12, k=1)
    g = O.canonical_csr(wl.n, wl.u, wl.v, wl.w)
    for P in [2, 4, 8]:
        b = _bounds_by_nnz(g.row_ptr, P)
        per = np.diff(g.row_ptr[b])
        assert b[0] == 0 and b[-1] == wl.n and np.all(np.diff(b) >= 0)
        assert per.max() <= g.nnz / P + np.diff(g.row_ptr).max()

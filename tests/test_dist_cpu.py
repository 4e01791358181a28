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


def _bounds_by_nnz(row_ptr, P, row_cost=6):
    """Same rule as fj_partition_rows (first row whose cost prefix, nonzeros + row_cost per row,
    reaches r/P of the total)."""
    pre = row_ptr + row_cost * np.arange(len(row_ptr), dtype=np.int64)
    tot = int(pre[-1])
    b = [0]
    for r in range(1, P):
        target = (tot // P) * r + (tot % P) * r // P
        b.append(int(np.searchsorted(pre[:-1], target, side="left")))
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
        cost = g.row_ptr + 6 * np.arange(wl.n + 1)
        per = np.diff(cost[b])
        assert b[0] == 0 and b[-1] == wl.n and np.all(np.diff(b) >= 0)
        assert per.max() <= cost[-1] / P + np.diff(g.row_ptr).max() + 6


def _gloo_cg_worker(rank, P, port, q):
    """The distributed single-reduction (Chronopoulos-Gear) Jacobi-PCG schedule of dist.cu, emulated
    in numpy over gloo: per iteration one elementwise step, the halo of u, the own-column / ghost-
    column split product, and exactly ONE allreduce of [gamma, delta, rho]."""
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
        counts, send_idx = D.exchange_requests(ghosts, bounds, D.TorchGroup(None, "cpu"))
        own = D.owners(ghosts, bounds)
        off = np.concatenate([[0], np.cumsum(counts)])
        r0, r1 = bounds[rank], bounds[rank + 1]
        nl = r1 - r0
        wf = g.wf()[g.row_ptr[r0]:g.row_ptr[r1]]
        rows = np.repeat(np.arange(nl), np.diff(rp))
        d = np.bincount(rows, weights=wf, minlength=nl)
        dinv = 1.0 / (1.0 + d)
        loc = cl < nl

        def halo(ul):
            hv = np.zeros(len(ghosts))
            reqs = [dist.isend(torch.from_numpy(ul[send_idx[off[p]:off[p + 1]]].copy()), p)
                    for p in range(P) if p != rank]
            for p in range(P):
                if p != rank:
                    rb = torch.zeros(int((own == p).sum()), dtype=torch.float64)
                    dist.recv(rb, p)
                    hv[own == p] = rb.numpy()
            for rq in reqs:
                rq.wait()
            return hv

        def product(ul):   # own-column pass, then the ghost-column pass of the boundary rows
            hv = halo(ul)
            w = (1.0 + d) * ul - np.bincount(rows[loc], weights=wf[loc] * ul[cl[loc]], minlength=nl)
            gh = ~loc
            return w - np.bincount(rows[gh], weights=wf[gh] * hv[cl[gh] - nl], minlength=nl)

        n_allreduce = 0

        def allreduce(vals):
            nonlocal n_allreduce
            n_allreduce += 1
            t = torch.tensor(vals, dtype=torch.float64)
            dist.all_reduce(t)
            return t.numpy()

        s = wl.S[r0:r1, 0]
        x = np.zeros(nl)
        r = s.copy()
        u = dinv * r
        w = product(u)
        gam, dlt, rho, ss = allreduce([r @ u, u @ w, r @ r, s @ s])
        tol2 = 1e-20 * ss
        it, first = 0, True
        p = sv = None
        gp = ap = 0.0
        while rho > tol2 and it < 500:
            if first:
                beta, alpha = 0.0, gam / dlt
                p, sv = u.copy(), w.copy()
            else:
                beta = gam / gp
                alpha = gam / (dlt - beta * gam / ap)
                p = u + beta * p
                sv = w + beta * sv
            x += alpha * p
            r -= alpha * sv
            u = dinv * r
            gp, ap, first = gam, alpha, False
            w = product(u)
            gam, dlt, rho = allreduce([r @ u, u @ w, r @ r])
            it += 1
        mx = max(bounds[k + 1] - bounds[k] for k in range(P))   # gloo all_gather: equal sizes
        xs = [torch.zeros(mx, dtype=torch.float64) for _ in range(P)]
        xp = torch.zeros(mx, dtype=torch.float64)
        xp[:nl] = torch.from_numpy(x)
        dist.all_gather(xs, xp)
        z = np.concatenate([xs[k].numpy()[:bounds[k + 1] - bounds[k]] for k in range(P)])
        q.put((rank, z, it, n_allreduce))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("P", [2])
def test_gloo_single_reduction_pcg_schedule(P):
    import synth
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_cg_worker, args=(r, P, port, q)) for r in range(P)]
    [p.start() for p in procs]
    [p.join(180) for p in procs]
    assert all(p.exitcode == 0 for p in procs)
    res = sorted([q.get(timeout=5) for _ in range(P)], key=lambda t: t[0])
    wl = synth.make_config("c4", scale=10, k=1)
    g = O.canonical_csr(wl.n, wl.u, wl.v, wl.w)
    zo = O.solve_dense(g, wl.S[:, 0])
    its = {t[2] for t in res}
    assert len(its) == 1                                   # identical decisions on every rank
    it = its.pop()
    for rank, z, _, nar in res:
        assert np.max(np.abs(z - zo)) < 1e-8
        assert nar == it + 1                               # one allreduce per iteration (+ the initial one)
    # same iteration count as textbook Jacobi-PCG (the recurrences are equivalent in exact arithmetic)
    _, info = O.solve_pcg(g, wl.S[:, 0], tol=1e-10)
    assert abs(it - info["iterations"]) <= 1

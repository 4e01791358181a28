"""GPU tests of the row-partitioned path (rows a8/e) with the LOOPBACK transport: P virtual ranks
as host threads of one process on one B200, each with its own stream and its own row block, the
halo exchange and allreduces done by the library (barrier-ordered device copies / host sums; no
kernel ever waits on another).  Results must match the single-GPU path and the oracle."""
import threading

import numpy as np
import pytest

import oracle as O
import synth

pytestmark = pytest.mark.gpu
QKEYS = ["CI", "D", "P", "C", "Idc", "PDI"]


@pytest.fixture(scope="module")
def fj():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2101_08143_b200 as m
    from paper_2101_08143_b200 import build as B
    B.build()
    return m


def run_ranks(fj, P, wl, S, opts=None, order="natural"):
    import torch
    from paper_2101_08143_b200 import dist as D
    comm = fj.Comm.loopback(P)
    world = D.ThreadWorld(P)
    u = torch.from_numpy(wl.u).cuda()
    v = torch.from_numpy(wl.v).cuda()
    w = None if wl.w is None else torch.from_numpy(wl.w).cuda()
    o2n = fj.binding.edge_degree_order(wl.n, u, v)[1] if order == "degree" else None
    bounds = fj.partition_rows(wl.n, u, v, P, old2new=o2n)
    Sd = torch.from_numpy(np.ascontiguousarray(S)).cuda()
    out, errs = [None] * P, []

    def rank_main(r):
        try:
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                G, _ = D.build_dist_graph(comm, r, wl.n, u, v, w, D.ThreadGroup(world, r), bounds=bounds, stream=st,
                                          order=order)
                Sl = D.slice_in(G, Sd, bounds, stream=st)
                z, q, rep = G.approxim(Sl, opts=opts, stream=st)
                st.synchronize()
                rows = None if G.rows_global is None else G.rows_global.cpu().numpy()
                out[r] = (z.cpu().numpy(), q, rep, G.plan, rows)
                G.close()
        except Exception as e:  # surface in the main thread
            errs.append(e)
            raise

    ts = [threading.Thread(target=rank_main, args=(r,)) for r in range(P)]
    [t.start() for t in ts]
    [t.join(300) for t in ts]
    comm.close()
    assert not errs, errs
    if order == "natural":
        Z = np.concatenate([o[0] for o in out])
    else:   # z rows back to the input labels
        Z = np.zeros_like(np.asarray(S, dtype=np.float64))
        for o in out:
            Z[o[4]] = o[0]
    return Z, [o[1] for o in out], [o[2] for o in out], bounds, [o[3] for o in out]


@pytest.mark.parametrize("P", [2, 3, 4])
def test_loopback_c1_matches_dense_oracle(fj, P):
    wl = synth.make_config("c1", k=2)
    Z, Q, R, bounds, plans = run_ranks(fj, P, wl, wl.S)
    g = O.canonical_csr(wl.n, wl.u, wl.v)
    for c in range(2):
        zo = O.solve_dense(g, wl.S[:, c])
        qo = O.quantities(g, wl.S[:, c], zo)
        assert np.max(np.abs(Z[:, c] - zo)) < 1e-9
        for r in range(P):                      # identical global quantities on every rank
            for k in QKEYS:
                assert Q[r][c][k] == Q[0][c][k]
                assert abs(Q[r][c][k] - qo[k]) / qo[k] <= 1e-8, (r, c, k)
    assert all(R[r]["iterations"] == R[0]["iterations"] for r in range(P))
    assert sum(p["nnz_local"] for p in plans) == g.nnz


@pytest.mark.parametrize("P", [2, 4])
def test_loopback_weighted_rmat_vs_single(fj, P):
    import torch
    wl = synth.make_config("c4", scale=14, k=1)
    Z, Q, R, bounds, plans = run_ranks(fj, P, wl, wl.S)
    G = fj.Graph.from_edges(wl.n, torch.from_numpy(wl.u).cuda(), torch.from_numpy(wl.v).cuda(),
                            torch.from_numpy(wl.w).cuda())
    z1, q1, r1 = G.approxim(torch.from_numpy(wl.S.copy()).cuda())
    assert np.max(np.abs(Z - z1.cpu().numpy())) < 1e-8
    g = O.canonical_csr(wl.n, wl.u, wl.v, wl.w)
    zo, _ = O.solve_pcg(g, wl.S[:, 0], tol=1e-13)
    qo = O.quantities(g, wl.S[:, 0], zo)
    for k in QKEYS:
        assert abs(Q[0][0][k] - qo[k]) / qo[k] <= 1e-8, k
        assert Q[0][0][k] == pytest.approx(q1[0][k], rel=1e-9)
    assert R[0]["rel_res_true"] <= 1e-10


def test_loopback_rows_build_bit_exact(fj):
    """Row-block CSR (a1 per rank) concatenates to the oracle's canonical CSR."""
    import torch
    wl = synth.make_config("c4", scale=12, k=1)
    u, v, w = (torch.from_numpy(a).cuda() for a in (wl.u, wl.v, wl.w))
    g = O.canonical_csr(wl.n, wl.u, wl.v, wl.w)
    bounds = fj.partition_rows(wl.n, u, v, 3)
    assert bounds[0] == 0 and bounds[-1] == wl.n
    cols, ws, rps = [], [], [np.zeros(1, np.int64)]
    for r in range(3):
        rp, cg, wo, nnz = fj.csr_rows_from_edges(wl.n, u, v, w, bounds[r], bounds[r + 1])
        cols.append(cg.cpu().numpy())
        ws.append(wo.cpu().numpy())
        rps.append(rp.cpu().numpy()[1:] + rps[-1][-1])
    assert np.array_equal(np.concatenate(rps), g.row_ptr)
    assert np.array_equal(np.concatenate(cols), g.col)
    assert np.array_equal(np.concatenate(ws), g.w)


def test_nccl_single_rank_comm(fj, monkeypatch):
    """The NCCL transport on a 1-rank communicator (dlopen, ncclCommInitRank, ncclAllReduce on the
    device scalars) gives the single-GPU result.  Multi-rank NCCL needs several GPUs (bench.py under
    torchrun); its plan / exchange logic is covered by the gloo and loopback tests."""
    import torch
    from paper_2101_08143_b200 import dist as D
    monkeypatch.setenv("FJ_NCCL_FORCE", "1")
    uid = fj.Comm.unique_id()
    assert len(uid) == 128
    comm = fj.Comm.nccl(1, 0, uid)
    wl = synth.make_config("c1", k=1)
    u, v = torch.from_numpy(wl.u).cuda(), torch.from_numpy(wl.v).cuda()
    G, b = D.build_dist_graph(comm, 0, wl.n, u, v, None, D.ThreadGroup(D.ThreadWorld(1), 0))
    assert b == [0, wl.n]
    z, q, rep = G.approxim(torch.from_numpy(wl.S.copy()).cuda())
    G1 = fj.Graph.from_edges(wl.n, u, v)
    z1, q1, rep1 = G1.approxim(torch.from_numpy(wl.S.copy()).cuda())
    assert np.max(np.abs(z.cpu().numpy() - z1.cpu().numpy())) < 1e-12
    for k in QKEYS:
        assert q[0][k] == pytest.approx(q1[0][k], rel=1e-12)
    G.close()
    comm.close()


@pytest.mark.parametrize("P", [2, 3])
def test_loopback_batched_k3_weighted_vs_oracle(fj, P):
    """Rows a8 + a9: three opinion columns of every rank's slice solved together (halo of padded
    KP = 4 rows, allreduce of k-vectors), weighted R-MAT, against the oracle and the 1-GPU path."""
    import torch
    wl = synth.make_config("c4", scale=13, kinds=["uniform", "exponential", "powerlaw"])
    Z, Q, R, bounds, plans = run_ranks(fj, P, wl, wl.S)
    assert all(R[r]["batch_k"] == 3 and R[r]["converged"] == 1 for r in range(P))
    assert all(R[r]["iterations"] == R[0]["iterations"] for r in range(P))
    g = O.canonical_csr(wl.n, wl.u, wl.v, wl.w)
    for c in range(3):
        zo, _ = O.solve_pcg(g, wl.S[:, c], tol=1e-13)
        qo = O.quantities(g, wl.S[:, c], zo)
        assert np.max(np.abs(Z[:, c] - zo)) < 1e-8
        for r in range(P):
            for k in QKEYS:
                assert Q[r][c][k] == Q[0][c][k]
                assert abs(Q[r][c][k] - qo[k]) / qo[k] <= 1e-8, (r, c, k)
    G = fj.Graph.from_edges(wl.n, torch.from_numpy(wl.u).cuda(), torch.from_numpy(wl.v).cuda(),
                            torch.from_numpy(wl.w).cuda())
    z1, q1, r1 = G.approxim(torch.from_numpy(wl.S.copy()).cuda())
    assert np.max(np.abs(Z - z1.cpu().numpy())) < 1e-8


@pytest.mark.parametrize("k", [1, 3])
def test_nccl_single_rank_graph_matches_host_loop(fj, monkeypatch, k):
    """The single-reduction loop captured in a CUDA graph together with its NCCL allreduce (1-rank
    communicator) gives bitwise the iterates of the same kernels launched from the host."""
    import torch
    from paper_2101_08143_b200 import dist as D
    monkeypatch.setenv("FJ_NCCL_FORCE", "1")
    comm = fj.Comm.nccl(1, 0, fj.Comm.unique_id())
    wl = synth.make_config("c4", scale=12, kinds=["uniform", "exponential", "powerlaw"][:k])
    u, v, w = (torch.from_numpy(a).cuda() for a in (wl.u, wl.v, wl.w))
    G, _ = D.build_dist_graph(comm, 0, wl.n, u, v, w, D.ThreadGroup(D.ThreadWorld(1), 0))
    S = torch.from_numpy(np.ascontiguousarray(wl.S)).cuda()
    zg, qg, rg = G.approxim(S, opts=fj.SolveOpts.make(use_cuda_graph=True))
    zh, qh, rh = G.approxim(S, opts=fj.SolveOpts.make(use_cuda_graph=False))
    assert torch.equal(zg, zh) and rg["iterations"] == rh["iterations"]
    g = O.canonical_csr(wl.n, wl.u, wl.v, wl.w)
    for c in range(k):
        zo, _ = O.solve_pcg(g, wl.S[:, c], tol=1e-13)
        qo = O.quantities(g, wl.S[:, c], zo)
        for key in QKEYS:
            assert qg[c][key] == qh[c][key]
            assert abs(qg[c][key] - qo[key]) / qo[key] <= 1e-8, (c, key)
    assert rg["rel_res_true"] <= 1e-10
    G.close()
    comm.close()


def test_loopback_eps_target_warm_restart(fj):
    """eps_target tightens rtol and warm-starts the distributed solve from z (the restart path of
    the single-reduction loop): certified bounds meet the target, results match the oracle."""
    wl = synth.make_config("c1", k=1)
    Z, Q, R, bounds, plans = run_ranks(fj, 3, wl, wl.S, opts=fj.SolveOpts.make(rtol=1e-6, eps_target=1e-9))
    g = O.canonical_csr(wl.n, wl.u, wl.v)
    zo = O.solve_dense(g, wl.S[:, 0])
    qo = O.quantities(g, wl.S[:, 0], zo)
    for key in QKEYS:
        assert Q[0][0]["eps"][key] <= 1e-9
        assert abs(Q[0][0][key] - qo[key]) / qo[key] <= max(Q[0][0]["eps"][key], 1e-12), key
    assert np.max(np.abs(Z[:, 0] - zo)) < 1e-8


@pytest.mark.parametrize("P,k", [(2, 1), (3, 3)])
def test_loopback_degree_relabelled_partition_vs_oracle(fj, P, k):
    """The graph relabelled by descending degree before partitioning (fj_edge_degree_order,
    fj_partition_rows_relabelled, fj_csr_rows_from_edges_relabelled): z mapped back to the input
    labels and the quantities against the oracle on the ORIGINAL graph (P:L88 P L P^T invariance)."""
    import torch
    wl = synth.make_config("c4", scale=13, kinds=["uniform", "exponential", "powerlaw"][:k])
    Z, Q, R, bounds, plans = run_ranks(fj, P, wl, wl.S, order="degree")
    g = O.canonical_csr(wl.n, wl.u, wl.v, wl.w)
    u, v = torch.from_numpy(wl.u).cuda(), torch.from_numpy(wl.v).cuda()
    n2o, o2n = fj.binding.edge_degree_order(wl.n, u, v)
    keep = wl.u != wl.v
    cnt = np.bincount(np.concatenate([wl.u[keep], wl.v[keep]]), minlength=wl.n)
    assert np.array_equal(n2o.cpu().numpy(), np.argsort(-cnt, kind="stable"))
    assert sum(p["nnz_local"] for p in plans) == g.nnz
    for c in range(k):
        zo, _ = O.solve_pcg(g, wl.S[:, c], tol=1e-13)
        qo = O.quantities(g, wl.S[:, c], zo)
        assert np.max(np.abs(Z[:, c] - zo)) < 1e-8
        for r in range(P):
            for key in QKEYS:
                assert Q[r][c][key] == Q[0][c][key]
                assert abs(Q[r][c][key] - qo[key]) / qo[key] <= 1e-8, (r, c, key)


class _WL:   # a minimal workload record for hand-built graphs
    def __init__(self, n, u, v, S, w=None):
        self.n, self.u, self.v, self.S, self.w = n, u.astype(np.int32), v.astype(np.int32), S, w


@pytest.mark.parametrize("P", [2, 3])
def test_loopback_star_hub_and_isolated(fj, P):
    """A star (one hub row holding most of the nonzeros) plus isolated vertices: blocks of very
    unequal row counts, ranks whose halo is the hub only, isolated rows (z_i = s_i)."""
    n = 3000
    leaves = np.arange(1, 2000)
    wl = _WL(n, np.zeros(len(leaves), np.int64), leaves,
             np.random.default_rng(3).uniform(0, 1, (n, 2)))
    Z, Q, R, bounds, plans = run_ranks(fj, P, wl, wl.S)
    g = O.canonical_csr(n, wl.u, wl.v)
    for c in range(2):
        zo = O.solve_dense(g, wl.S[:, c])
        qo = O.quantities(g, wl.S[:, c], zo)
        assert np.max(np.abs(Z[:, c] - zo)) < 1e-9
        assert np.max(np.abs(Z[2000:, c] - wl.S[2000:, c])) < 1e-9   # isolated rows: z_i = s_i
        for key in QKEYS:
            assert abs(Q[0][c][key] - qo[key]) / qo[key] <= 1e-8, (c, key)


def test_loopback_rank_without_halo(fj):
    """Two disjoint graphs split exactly at the component boundary: a rank whose local rows have no
    ghost columns (empty halo, no boundary rows) -- the off-diagonal pass is empty."""
    import torch
    from paper_2101_08143_b200 import dist as D
    a = synth.make_config("c1", n=1500, k=1)
    u = np.concatenate([a.u, a.u + 1500])
    v = np.concatenate([a.v, a.v + 1500])
    S = np.random.default_rng(5).uniform(0, 1, (3000, 1))
    wl = _WL(3000, u, v, S)
    comm = fj.Comm.loopback(2)
    world = D.ThreadWorld(2)
    ud, vd = torch.from_numpy(wl.u).cuda(), torch.from_numpy(wl.v).cuda()
    bounds = [0, 1500, 3000]
    out = [None, None]

    def rank_main(r):
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            G, _ = D.build_dist_graph(comm, r, 3000, ud, vd, None, D.ThreadGroup(world, r), bounds=bounds, stream=st)
            z, q, rep = G.approxim(torch.from_numpy(np.ascontiguousarray(S[bounds[r]:bounds[r + 1]])).cuda(), stream=st)
            st.synchronize()
            out[r] = (z.cpu().numpy(), q, rep, G.plan)
            G.close()
    import threading
    ts = [threading.Thread(target=rank_main, args=(r,)) for r in range(2)]
    [t.start() for t in ts]
    [t.join(300) for t in ts]
    comm.close()
    assert out[0][3]["n_ghost"] == 0 and out[1][3]["n_ghost"] == 0
    g = O.canonical_csr(3000, wl.u, wl.v)
    zo = O.solve_dense(g, S[:, 0])
    qo = O.quantities(g, S[:, 0], zo)
    Z = np.concatenate([out[0][0], out[1][0]]).reshape(-1)
    assert np.max(np.abs(Z - zo)) < 1e-9
    for key in QKEYS:
        assert abs(out[0][1][0][key] - qo[key]) / qo[key] <= 1e-8, key

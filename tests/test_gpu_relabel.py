"""GPU: the locality relabelling of a1 (include/fj.h fj_csr_degree_order,
fj_csr_permute, fj_permute_rows).

The orders and the relabelled CSRs are integer results: bit-exact against numpy's stable argsort
of the row lengths and P A P^T of the oracle's CSR with columns in source order.  Solves on
a relabelled graph are checked against the oracle on the ORIGINAL graph (the quantities are
invariant: P L P^T; sums over vertices and edges) with the usual bars."""
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


def dev(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def host(t):
    return t.cpu().numpy()


def permuted_csr_ref(g, n2o, o2n):
    """P A P^T in numpy: row i' = old row n2o[i'], columns relabelled, source order kept."""
    lens = np.diff(g.row_ptr)[n2o]
    rp = np.zeros(len(n2o) + 1, np.int64)
    rp[1:] = np.cumsum(lens)
    idx = np.concatenate([np.arange(g.row_ptr[r], g.row_ptr[r + 1]) for r in n2o]) if g.nnz else np.zeros(0, int)
    col = o2n[g.col[idx]].astype(np.int32)
    return rp, col, (None if g.w is None else g.w[idx])


@pytest.mark.parametrize("wkind", ["unit", "u8", "f64"])
@pytest.mark.parametrize("order", ["degree", "random"])
def test_csr_permute_exact(fj, wkind, order):
    rng = np.random.default_rng(11)
    n, m = 20000, 30000        # ~half the vertices isolated: random orders put empty rows inside chunks
    u = rng.integers(0, n // 2, m).astype(np.int32)
    v = (rng.zipf(1.5, m) % (n // 2)).astype(np.int32)
    w = None if wkind == "unit" else (rng.integers(1, 6, m).astype(np.uint8) if wkind == "u8"
                                      else rng.uniform(0.1, 4.0, m))
    g = O.canonical_csr(n, u, v, w)
    rp, col, wo, _ = fj.csr_from_edges(n, dev(u), dev(v), None if w is None else dev(w))
    if order == "degree":
        n2o, o2n = fj.csr_degree_order(n, rp)
        ref = np.argsort(-np.diff(g.row_ptr), kind="stable").astype(np.int32)
        assert np.array_equal(host(n2o), ref) and np.array_equal(host(o2n)[ref], np.arange(n))
    else:
        perm = rng.permutation(n).astype(np.int32)
        inv = np.empty_like(perm)
        inv[perm] = np.arange(n, dtype=np.int32)
        n2o, o2n = dev(perm), dev(inv)
    rp2, col2, w2 = fj.csr_permute(n, rp, col, wo, n2o, o2n)
    rr, cr, wr = permuted_csr_ref(g, host(n2o), host(o2n))
    assert np.array_equal(host(rp2), rr) and np.array_equal(host(col2), cr)
    if w is not None:
        assert np.array_equal(host(w2), wr)
    G = fj.Graph(n, rp2, col2, w2, validate=False)   # degrees: same per-row order -> bit-exact
    assert np.array_equal(host(G.degrees()), O.degrees(g)[host(n2o)])


@pytest.mark.parametrize("k", [1, 2, 3, 4, 7, 40])
def test_permute_rows_exact(fj, k):
    import torch
    rng = np.random.default_rng(k)
    n = 1001
    x = rng.standard_normal((n, k)) if k > 1 else rng.standard_normal(n)
    perm = rng.permutation(n).astype(np.int32)
    y = host(fj.permute_rows(dev(x), dev(perm)))
    assert np.array_equal(y, x[perm])
    assert fj.permute_rows(torch.zeros(0, dtype=torch.float64, device="cuda"),
                           torch.zeros(0, dtype=torch.int32, device="cuda")).numel() == 0


def _solve_both(fj, n, u, v, w, S):   # the relabelled handle (csr_degree_order + csr_permute)
    Gd = fj.Graph.from_edges(n, dev(u), dev(v), None if w is None else dev(w), order="degree")
    z, q, rep = Gd.approxim(dev(S))
    return Gd, host(z), q, rep


@pytest.mark.parametrize("name,k", [("c1", 1), ("c1", 3), ("c1", 8), ("c1w", 3)])
def test_relabelled_approxim_vs_oracle(fj, name, k):
    weighted = name == "c1w"
    wl = synth.make_config("c1", kinds=(["uniform", "exponential", "powerlaw"] * 3)[:k])
    if weighted:   # u8 weights 1..5 on the same graph (the C4 weight recipe)
        wl.w = np.random.default_rng(3).integers(1, 6, len(wl.u)).astype(np.uint8)
    S = wl.S[:, :k].copy() if k > 1 else wl.S[:, 0].copy()
    G, z, q, rep = _solve_both(fj, wl.n, wl.u, wl.v, wl.w, S)
    g = O.canonical_csr(wl.n, wl.u, wl.v, wl.w)
    S2 = S.reshape(wl.n, -1)
    Z = z.reshape(wl.n, -1)
    for c in range(k):
        zo = O.solve(g, S2[:, c])
        qo = O.quantities(g, S2[:, c], zo)
        assert np.max(np.abs(Z[:, c] - zo)) <= 1e-8 * np.max(np.abs(zo))
        for key in QKEYS:
            rel = abs(q[c][key] - qo[key]) / abs(qo[key])
            assert rel <= 1e-8 and rel <= q[c]["eps"][key] * (1 + 1e-9) + 1e-15, (c, key, rel)
    # vertex-indexed results come back in the input labels
    assert np.array_equal(host(G.degrees()), O.degrees(g))
    x = np.random.default_rng(1).standard_normal(wl.n)
    assert np.allclose(host(G.apply(dev(x))), O.ipl_apply(g, x), rtol=1e-13, atol=1e-12)
    zs, _ = G.solve(dev(S))
    assert np.max(np.abs(host(zs).reshape(wl.n, -1) - Z)) <= 1e-9 * np.max(np.abs(Z))
    qq = G.quantities(dev(S), dev(z))
    for c in range(k):
        for key in QKEYS:
            assert qq[c][key] == pytest.approx(q[c][key], rel=1e-12), (c, key)


def test_relabelled_forest_columns(fj):
    rng = np.random.default_rng(5)
    n = 400
    u = rng.integers(0, n, 3000).astype(np.int32)
    v = (rng.zipf(1.8, 3000) % n).astype(np.int32)
    G = fj.Graph.from_edges(n, dev(u), dev(v), order="degree")
    cols = [0, 17, 399]
    om, rep = G.forest_columns(cols)
    Om = np.linalg.inv(O.dense_ipl(O.canonical_csr(n, u, v)))
    assert np.max(np.abs(host(om) - Om[:, cols])) <= 1e-9


@pytest.mark.parametrize("name,k", [("c1", 1), ("c1", 3)])
def test_approxim_host_vertex_order(fj, name, k):
    wl = synth.make_config(name, kinds=["uniform", "exponential", "powerlaw"][:k])
    S = wl.S[:, :k].copy() if k > 1 else wl.S[:, 0].copy()
    z0, q0, _ = fj.approxim_host(wl.n, wl.u, wl.v, wl.w, S, want_z=True)
    z1, q1, _ = fj.approxim_host(wl.n, wl.u, wl.v, wl.w, S, opts=fj.SolveOpts.make(vertex_order="degree"),
                                 want_z=True)
    assert np.max(np.abs(z1 - z0)) <= 1e-9 * np.max(np.abs(z0))
    for c in range(k):
        for key in QKEYS:
            assert q1[c][key] == pytest.approx(q0[c][key], rel=1e-9), (c, key)
    z2, q2, _ = fj.approxim_host(wl.n, wl.u, wl.v, wl.w, S, opts=fj.SolveOpts.make(vertex_order="auto"),
                                 want_z=True)   # small graph: auto keeps the input labels
    assert np.array_equal(z2, z0)
    with pytest.raises(fj.FJError):
        o = fj.SolveOpts.make()
        o.vertex_order = 5
        fj.approxim_host(wl.n, wl.u, wl.v, wl.w, S, opts=o)


def test_relabelled_user_buffers(fj):
    """Caller-owned z buffers: approxim and solve write z (input labels) into them."""
    import torch
    wl = synth.make_config("c1", kinds=["uniform", "exponential", "powerlaw"])
    G = fj.Graph.from_edges(wl.n, dev(wl.u), dev(wl.v), order="degree")
    S = dev(wl.S)
    zbuf = torch.full_like(S, 7.0)
    z, q, _ = G.approxim(S, z=zbuf)
    assert z.data_ptr() == zbuf.data_ptr()
    g = O.canonical_csr(wl.n, wl.u, wl.v)
    for c in range(3):
        assert np.max(np.abs(host(zbuf)[:, c] - O.solve(g, wl.S[:, c]))) < 1e-8
    zw = torch.zeros_like(S)
    z2, rep = G.solve(S, z=zw)
    assert z2.data_ptr() == zw.data_ptr()
    assert np.max(np.abs(host(zw) - host(zbuf))) < 1e-9

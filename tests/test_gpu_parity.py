"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the same seeded inputs.

Bars (BASELINE.json north_star): CSR and degrees bit-exact; relative residual <= 1e-10; each
quantity within relative 1e-8 of the oracle.  Operator parity is checked against the oracle's
(I+L)x within a rounding bound derived from the row sums."""
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


def gpu_csr(fj, n, u, v, w=None):
    rp, col, wo, stats = fj.csr_from_edges(n, dev(u.astype(np.int32)), dev(v.astype(np.int32)),
                                           None if w is None else dev(w))
    return rp, col, wo, stats


def assert_csr_equal(fj, n, u, v, w=None):
    g = O.canonical_csr(n, u, v, w)
    rp, col, wo, stats = gpu_csr(fj, n, u, v, w)
    assert np.array_equal(host(rp), g.row_ptr)
    assert np.array_equal(host(col), g.col)
    if w is not None:
        assert np.array_equal(host(wo), g.w)
    assert stats["selfloops"] == g.selfloops and stats["duplicates"] == g.duplicates
    return g, (rp, col, wo)


# ---------------------------------------------------------------- a1 / a2: bit-exact
@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("wkind", ["unit", "u8", "f64"])
def test_csr_bit_exact_random(fj, seed, wkind):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 3000))
    m = int(rng.integers(0, 20000))
    u = rng.integers(0, n, m).astype(np.int32)
    v = rng.integers(0, n, m).astype(np.int32)
    w = None if wkind == "unit" else (rng.integers(1, 6, m).astype(np.uint8) if wkind == "u8"
                                      else rng.uniform(0.1, 4.0, m))
    g, (rp, col, wo) = assert_csr_equal(fj, n, u, v, w)
    G = fj.Graph(n, rp, col, wo, validate=True)
    assert np.array_equal(host(G.degrees()), O.degrees(g))   # bit-exact, ascending-column sums
    info = G.info()
    assert info["nnz"] == g.nnz and info["n_isolated"] == int((np.diff(g.row_ptr) == 0).sum())


def test_csr_edge_cases(fj):
    assert_csr_equal(fj, 1, np.zeros(0, np.int32), np.zeros(0, np.int32))
    assert_csr_equal(fj, 5, np.array([1, 2, 3], np.int32), np.array([1, 2, 3], np.int32))     # all self-loops
    assert_csr_equal(fj, 4, np.array([0, 1, 0, 1], np.int32), np.array([1, 0, 1, 0], np.int32))  # duplicates
    with pytest.raises(fj.FJError):
        gpu_csr(fj, 4, np.array([0], np.int32), np.array([4], np.int32))


@pytest.mark.parametrize("name", ["c1", "c2", "c3"])
def test_csr_bit_exact_configs(fj, name):
    wl = synth.make_config(name, k=1, kinds=["uniform"])
    assert_csr_equal(fj, wl.n, wl.u, wl.v, wl.w)


def test_csr_c4_scale16_bit_exact_and_full_size_sampled(fj):
    wl = synth.make_config("c4", scale=16, k=1)
    assert_csr_equal(fj, wl.n, wl.u, wl.v, wl.w)
    big = synth.make_config("c4", k=1)                           # full scale 22, 67M raw edges
    rp, col, wo, stats = gpu_csr(fj, big.n, big.u, big.v, big.w)
    rp_h = host(rp)
    rng = np.random.default_rng(0)
    deg = np.diff(rp_h)
    rows = list(rng.integers(0, big.n, 40)) + list(np.argsort(deg)[-5:]) + [0, big.n - 1]
    want = O.csr_rows_from_edges(big.n, big.u, big.v, rows, big.w)
    for i, (c_ref, w_ref) in want.items():
        a, b = rp_h[i], rp_h[i + 1]
        assert np.array_equal(host(col[a:b]), c_ref)
        assert np.array_equal(host(wo[a:b]), w_ref)


# ---------------------------------------------------------------- operator
def hub_graph(rng, n, hubs, hub_deg, extra):
    u = [rng.integers(0, n, extra)]
    v = [rng.integers(0, n, extra)]
    for h in range(hubs):
        u.append(np.full(hub_deg, h))
        v.append(rng.choice(n, hub_deg, replace=False))
    return np.concatenate(u).astype(np.int32), np.concatenate(v).astype(np.int32)


@pytest.mark.parametrize("wkind", ["unit", "u8", "f64"])
@pytest.mark.parametrize("op", [0, 1])
def test_apply_matches_oracle(fj, wkind, op):
    rng = np.random.default_rng(7)
    n = 40000
    u, v = hub_graph(rng, n, hubs=3, hub_deg=20000, extra=150000)   # long rows -> multi-chunk path
    m = len(u)
    w = None if wkind == "unit" else (rng.integers(1, 6, m).astype(np.uint8) if wkind == "u8"
                                      else rng.uniform(0.1, 4.0, m))
    g, (rp, col, wo) = assert_csr_equal(fj, n, u, v, w)
    G = fj.Graph(n, rp, col, wo)
    assert G.info()["n_long_rows"] >= 3
    assert np.array_equal(host(G.degrees()), O.degrees(g))   # bit-exact, incl. the warp-summed long u8 rows
    X = rng.normal(size=(n, 3))
    Y = host(G.apply(dev(X), op=op))
    for c in range(3):
        x = X[:, c]
        ref = O.ipl_apply(g, x) - (x if op == 0 else 0.0)
        d = O.degrees(g)
        # rounding bound of a row sum: (len + 2) u ((1+d)|x_i| + sum_j w_ij |x_j|)
        scale = (1 + d) * np.abs(x) + np.bincount(g.rows(), weights=g.wf() * np.abs(x[g.col]), minlength=n)
        err = np.abs(Y[:, c] - ref)
        assert np.all(err <= 2 * (np.diff(g.row_ptr) + 2) * 2.0 ** -53 * scale), c


# ---------------------------------------------------------------- solve + quantities: pins
def solve_quant(fj, n, u, v, w, S, **kw):
    rp, col, wo, _ = gpu_csr(fj, n, np.asarray(u), np.asarray(v), w)
    G = fj.Graph(n, rp, col, wo, validate=True)
    z, q, rep = G.approxim(dev(S), opts=fj.SolveOpts.make(**kw))
    return G, host(z), q, rep


def test_p5_and_path2_golden(fj):
    from conftest import read_golden
    from fractions import Fraction
    gold = {r[0]: Fraction(int(r[1]), int(r[2])) for r in read_golden("p5_e1_quantities.txt")}
    u = np.arange(4); v = u + 1
    _, z, q, rep = solve_quant(fj, 5, u, v, None, np.eye(5)[0], rtol=1e-14)
    assert np.allclose(z * 55, [34, 13, 5, 2, 1], rtol=1e-12)
    for k in QKEYS:
        assert q[0][k] == pytest.approx(float(gold[k]), rel=1e-10), k
    gold2 = {r[0]: Fraction(int(r[1]), int(r[2])) for r in read_golden("path2_quantities.txt")}
    _, z, q, _ = solve_quant(fj, 2, [0], [1], None, np.array([1.0, 0.0]), rtol=1e-14)
    for k in QKEYS:
        assert q[0][k] == pytest.approx(float(gold2[k]), rel=1e-10), k


@pytest.mark.parametrize("n", [300, 3000])
def test_complete_graph_closed_form(fj, n):
    iu, ju = np.triu_indices(n, 1)
    s = np.random.default_rng(n).uniform(0, 1, n)
    _, z, q, rep = solve_quant(fj, n, iu, ju, None, s)
    m = s.mean(); S = ((s - m) ** 2).sum()
    assert np.allclose(z, (s + n * m) / (n + 1), rtol=1e-9)
    for k, ref in [("P", S / (n + 1) ** 2), ("D", n * S / (n + 1) ** 2), ("CI", n * n * S / (n + 1) ** 2),
                   ("C", S / (n + 1) ** 2 + n * m * m), ("PDI", S / (n + 1))]:
        assert q[0][k] == pytest.approx(ref, rel=1e-8), k


def test_star_hub_closed_form(fj):
    n = 200_000   # hub row of 199,999 nonzeros: 98 long-row chunks
    s = np.random.default_rng(3).uniform(0, 1, n)
    G, z, q, rep = solve_quant(fj, n, np.zeros(n - 1, np.int32), np.arange(1, n, dtype=np.int32), None, s)
    assert G.info()["n_long_chunks"] == (n - 1 + 2047) // 2048
    z0 = (2 * s[0] + s[1:].sum()) / (n + 1)
    zc = np.concatenate([[z0], (s[1:] + z0) / 2])
    assert np.allclose(z, zc, rtol=1e-9, atol=0)
    qo = O.quantities(O.canonical_csr(n, np.zeros(n - 1), np.arange(1, n)), s, zc)
    for k in QKEYS:
        assert q[0][k] == pytest.approx(qo[k], rel=1e-8), k


def test_consensus_zero_and_isolated(fj):
    rng = np.random.default_rng(11)
    u = rng.integers(0, 1000, 4000); v = rng.integers(0, 1000, 4000)
    _, z, q, rep = solve_quant(fj, 1200, u, v, None, np.full(1200, 0.3))   # 200 isolated vertices too
    assert np.array_equal(z, np.full(1200, 0.3)) and q[0]["consensus"] == 1
    assert q[0]["C"] == pytest.approx(1200 * 0.09, rel=1e-15) and q[0]["D"] == 0 and q[0]["P"] == 0
    _, z, q, rep = solve_quant(fj, 1200, u, v, None, np.zeros(1200))
    assert not z.any() and q[0]["C"] == 0
    s = rng.uniform(0, 1, 1200)
    _, z, q, rep = solve_quant(fj, 1200, u, v, None, s)
    iso = np.setdiff1d(np.arange(1200), np.concatenate([u, v]))
    assert np.allclose(z[iso], s[iso], rtol=1e-12)


# ---------------------------------------------------------------- solve + quantities: configs
def check_against_oracle(q, qo, S_col, z, zo, cert=True):
    for k in QKEYS:
        rel = abs(q[k] - qo[k]) / abs(qo[k])
        assert rel <= 1e-8, (k, rel)
        if cert:
            assert rel <= q["eps"][k] * (1 + 1e-9) + 1e-15, (k, rel, q["eps"][k])   # certificate holds
    assert q["res_norm"] <= 1e-10 * q["s_norm"] * (1 + 1e-9)


def test_c1_vs_dense_oracle(fj):
    wl = synth.make_config("c1")
    g = O.canonical_csr(wl.n, wl.u, wl.v)
    zo = O.solve_dense(g, wl.S[:, 0])
    qo = O.quantities(g, wl.S[:, 0], zo)
    _, z, q, rep = solve_quant(fj, wl.n, wl.u, wl.v, None, wl.S[:, 0])
    assert rep["converged"] == 1 and rep["rel_res_true"] <= 1e-10
    check_against_oracle(q[0], qo, wl.S[:, 0], z, zo)
    assert np.max(np.abs(z - zo)) < 1e-9


@pytest.mark.parametrize("name", ["c2", "c3"])
def test_full_config_vs_pcg_oracle(fj, name):
    wl = synth.make_config(name)
    g = O.canonical_csr(wl.n, wl.u, wl.v)
    G, Z, Q, rep = solve_quant(fj, wl.n, wl.u, wl.v, None, wl.S)
    assert rep["converged"] == 1 and rep["rel_res_true"] <= 1e-10
    if wl.k == 3:   # c3: the bench's product path (two column slabs)
        assert G.product_path(3) == "rows_slabs"
    for c in range(wl.k):
        zo, info = O.solve_pcg(g, wl.S[:, c], tol=1e-13)
        assert info["converged"]
        qo = O.quantities(g, wl.S[:, c], zo)
        check_against_oracle(Q[c], qo, wl.S[:, c], Z[:, c], zo)


def test_c4_small_weighted_batch(fj):
    wl = synth.make_config("c4", scale=14, k=3)
    g = O.canonical_csr(wl.n, wl.u, wl.v, wl.w)
    _, Z, Q, rep = solve_quant(fj, wl.n, wl.u, wl.v, wl.w, wl.S)
    for c in range(3):
        zo, _ = O.solve_pcg(g, wl.S[:, c], tol=1e-13)
        check_against_oracle(Q[c], O.quantities(g, wl.S[:, c], zo), wl.S[:, c], Z[:, c], zo)


# ---------------------------------------------------------------- behaviour
def test_determinism_and_graph_mode(fj):
    wl = synth.make_config("c2", n=200_000)
    rp, col, wo, _ = gpu_csr(fj, wl.n, wl.u, wl.v)
    G = fj.Graph(wl.n, rp, col, wo)
    s = dev(wl.S[:, 0])
    z1, q1, r1 = G.approxim(s)
    z2, q2, r2 = G.approxim(s)
    z3, q3, r3 = G.approxim(s, opts=fj.SolveOpts.make(use_cuda_graph=False))
    assert np.array_equal(host(z1), host(z2)) and np.array_equal(host(z1), host(z3))
    assert q1[0]["D"] == q2[0]["D"] == q3[0]["D"] and r1["iterations"] == r3["iterations"]


def test_solve_and_quantities_entry_points(fj):
    wl = synth.make_config("c1", k=2)
    rp, col, wo, _ = gpu_csr(fj, wl.n, wl.u, wl.v)
    G = fj.Graph(wl.n, rp, col, wo)
    S = dev(wl.S)
    z, rep = G.solve(S)
    assert rep["converged"] == 1 and rep["rel_res_true"] <= 1e-10
    q = G.quantities(S, z)
    _, qa, _ = G.approxim(S)
    for c in range(2):
        for k in QKEYS:
            assert q[c][k] == pytest.approx(qa[c][k], rel=1e-9)
    st = G.opinion_stats(S)
    assert st[0][0] == pytest.approx(wl.S[:, 0].sum(), rel=1e-13) and st[1][3] == wl.S[:, 1].max()
    with pytest.raises(fj.FJError):
        G.approxim(dev(np.full(wl.n, np.nan)))


def test_eps_target_tightens(fj):
    wl = synth.make_config("c1")
    rp, col, wo, _ = gpu_csr(fj, wl.n, wl.u, wl.v)
    G = fj.Graph(wl.n, rp, col, wo)
    _, q, rep = G.approxim(dev(wl.S[:, 0]), opts=fj.SolveOpts.make(rtol=1e-4, eps_target=1e-9))
    assert max(q[0]["eps"].values()) <= 1e-9


def test_validation_errors(fj):
    import torch
    rp = dev(np.array([0, 1, 1], np.int64)); col = dev(np.array([1], np.int32))
    with pytest.raises(fj.FJError) as e:
        fj.Graph(2, rp, col)                                  # (0,1) without (1,0)
    assert e.value.status == 3
    rp = dev(np.array([0, 1, 2], np.int64)); col = dev(np.array([0, 1], np.int32))
    with pytest.raises(fj.FJError) as e:
        fj.Graph(2, rp, col)                                  # self-loops
    assert e.value.status == 2
    rp = dev(np.array([0, 1, 2], np.int64)); col = dev(np.array([1, 0], np.int32))
    with pytest.raises(fj.FJError) as e:
        fj.Graph(2, rp, col, dev(np.array([-1.0, -1.0])))     # bad weight
    assert e.value.status == 4


def test_e2e_host_matches_device(fj):
    wl = synth.make_config("c4", scale=12, k=2)
    z_h, q_h, rep_h = fj.approxim_host(wl.n, wl.u, wl.v, wl.w, wl.S, want_z=True)
    _, z_d, q_d, rep_d = solve_quant(fj, wl.n, wl.u, wl.v, wl.w, wl.S)
    assert np.array_equal(z_h, z_d)
    assert q_h[1]["D"] == q_d[1]["D"]


# ---------------------------------------------------------------- a9: batched k-column PCG
def test_batched_k_columns_vs_oracle(fj):
    wl = synth.make_config("c4", scale=14, k=8)
    S = wl.S.copy()
    S[:, 3] = 0.25            # consensus column (exact z = s)
    S[:, 5] = 0.0             # zero column
    g = O.canonical_csr(wl.n, wl.u, wl.v, wl.w)
    _, Z, Q, rep = solve_quant(fj, wl.n, wl.u, wl.v, wl.w, S)
    assert rep["converged"] == 1 and rep["rel_res_true"] <= 1e-10
    assert np.array_equal(Z[:, 3], S[:, 3]) and Q[3]["consensus"] == 1
    assert not Z[:, 5].any()
    for c in [0, 1, 2, 4, 6, 7]:
        zo, _ = O.solve_pcg(g, S[:, c], tol=1e-13)
        check_against_oracle(Q[c], O.quantities(g, S[:, c], zo), S[:, c], Z[:, c], zo)


def test_batched_k64_deterministic_and_matches_single(fj):
    wl = synth.make_config("c4", scale=13, k=64)
    rp, col, wo, _ = gpu_csr(fj, wl.n, wl.u, wl.v, wl.w)
    G = fj.Graph(wl.n, rp, col, wo)
    S = dev(wl.S)
    z1, q1, r1 = G.approxim(S)
    z2, q2, r2 = G.approxim(S)
    z3, q3, r3 = G.approxim(S, opts=fj.SolveOpts.make(use_cuda_graph=False))
    assert np.array_equal(host(z1), host(z2)) and np.array_equal(host(z1), host(z3))
    for c in [0, 17, 63]:                      # batched columns agree with the k = 1 path
        zc, qc, rc = G.approxim(dev(wl.S[:, c].copy()))
        for k in QKEYS:
            assert q1[c][k] == pytest.approx(qc[0][k], rel=1e-8), (c, k)
        assert np.max(np.abs(host(z1)[:, c] - host(zc))) < 1e-8


def test_batched_apply_and_solve_entry(fj):
    wl = synth.make_config("c1", k=5)
    g = O.canonical_csr(wl.n, wl.u, wl.v)
    rp, col, wo, _ = gpu_csr(fj, wl.n, wl.u, wl.v)
    G = fj.Graph(wl.n, rp, col, wo)
    Z, rep = G.solve(dev(wl.S))
    Z = host(Z)
    for c in range(5):
        assert np.max(np.abs(Z[:, c] - O.solve_dense(g, wl.S[:, c]))) < 1e-9
    Y = host(G.apply(dev(wl.S), op=0))
    for c in range(5):
        assert np.allclose(Y[:, c], O.ipl_apply(g, wl.S[:, c]) - wl.S[:, c], rtol=1e-12, atol=1e-12)


# ---------------------------------------------------------------- a9, small k: vector warp-item engine
@pytest.mark.parametrize("k,wkind", [(2, "unit"), (3, "u8"), (4, "f64"), (3, "unit")])
def test_small_k_vector_engine_vs_oracle(fj, k, wkind):
    """2 <= k <= 4 columns solved together on padded [n][KP] blocks (spmv_vec.cu): every column
    against the oracle, a consensus column exact, bitwise graph / host-loop agreement."""
    rng = np.random.default_rng(20 + k)
    n = 30000
    u, v = hub_graph(rng, n, hubs=2, hub_deg=9000, extra=120000)   # T tiles + W rows + long chunks
    m = len(u)
    w = None if wkind == "unit" else (rng.integers(1, 6, m).astype(np.uint8) if wkind == "u8"
                                      else rng.uniform(0.1, 4.0, m))
    S = rng.uniform(0, 1, (n, k))
    S[:, k - 1] = 0.375                    # consensus column: z = s exactly
    g = O.canonical_csr(n, u, v, w)
    G, Z, Q, rep = solve_quant(fj, n, u, v, w, S)
    assert rep["batch_k"] == k and rep["converged"] == 1 and rep["rel_res_true"] <= 1e-10
    assert np.array_equal(Z[:, k - 1], S[:, k - 1]) and Q[k - 1]["consensus"] == 1
    for c in range(k - 1):
        zo, _ = O.solve_pcg(g, S[:, c], tol=1e-13)
        check_against_oracle(Q[c], O.quantities(g, S[:, c], zo), S[:, c], Z[:, c], zo)
    Sd = dev(S)
    z1, q1, r1 = G.approxim(Sd)
    z2, q2, r2 = G.approxim(Sd, opts=fj.SolveOpts.make(use_cuda_graph=False))
    assert np.array_equal(host(z1), host(z2)) and r1["iterations"] == r2["iterations"]
    qs = G.quantities(Sd, z1)                  # stand-alone entry packs z itself
    for c in range(k):
        for key in QKEYS:
            assert qs[c][key] == q1[c][key], (c, key)
    assert G.time_spmv(k=k, reps=2) > 0


def test_small_k_solve_entry_and_ragged(fj):
    """fj_solve with k = 3 on a graph with isolated vertices and a single edge component."""
    n = 5000
    rng = np.random.default_rng(5)
    u = rng.integers(0, 4000, 12000); v = rng.integers(0, 4000, 12000)     # 1000 isolated rows
    g = O.canonical_csr(n, u, v)
    rp, col, wo, _ = gpu_csr(fj, n, u.astype(np.int32), v.astype(np.int32))
    G = fj.Graph(n, rp, col, wo)
    S = rng.uniform(0, 1, (n, 3))
    Z, rep = G.solve(dev(S))
    Z = host(Z)
    assert rep["batch_k"] == 3 and rep["converged"] == 1
    for c in range(3):
        assert np.max(np.abs(Z[:, c] - O.solve_dense(g, S[:, c]) if n <= 4096 else
                             Z[:, c] - O.solve_pcg(g, S[:, c], tol=1e-13)[0])) < 1e-9
    assert np.allclose(Z[4000:], S[4000:], rtol=1e-12)


# ---------------------------------------------------------------- f2: Algorithm 1 verbatim
@pytest.mark.parametrize("name", ["c1", "c4s"])
def test_alg1_verbatim_vs_oracle(fj, name):
    """fj_approxim_alg1 (both solves as one k = 2 batch, lines 5-9 norms) against the oracle's
    line-by-line Algorithm 1 with exact solves; delta / clamp / rtol equal the oracle's transcription."""
    if name == "c1":
        wl = synth.make_config("c1")
        w = None
    else:
        wl = synth.make_config("c4", scale=9, k=1)
        w = wl.w
    s = wl.S[:, 0].copy()
    g = O.canonical_csr(wl.n, wl.u, wl.v, w)
    rp, col, wo, _ = gpu_csr(fj, wl.n, wl.u, wl.v, w)
    G = fj.Graph(wl.n, rp, col, wo)
    r, rep = G.approxim_alg1(dev(s), eps=1e-6)
    o = O.alg1(g, s, 1e-6)
    assert rep["converged"] == 1 and rep["batch_k"] == 2 and rep["rel_res_true"] <= r["rtol"] * (1 + 1e-9)
    for k in ["CI", "D", "P", "C", "Idc", "PDI"]:
        assert r[k] == pytest.approx(o[k], rel=1e-8), k
    assert r["D_from_z"] == pytest.approx(r["D"], rel=1e-9)        # D from s or s_bar
    assert r["CI_def"] == pytest.approx(r["CI"], rel=1e-8)         # ||Lz||^2 = sum (z - s)^2 (Lemma 4.1)
    for a, b in [("delta", "delta"), ("delta_eff", "delta_eff"), ("rtol", "rtol")]:
        assert r[a] == pytest.approx(o[b], rel=1e-12), a
    assert bool(r["clamped"]) == o["clamped"] and bool(r["rtol_floored"]) == o["floored"]


def test_alg1_path2_and_consensus(fj):
    gold = {"CI": 2 / 9, "D": 1 / 9, "P": 1 / 18, "C": 5 / 9, "Idc": 2 / 3}      # S:L311 example (golden path2)
    rp, col, wo, _ = gpu_csr(fj, 2, np.array([0], np.int32), np.array([1], np.int32))
    G = fj.Graph(2, rp, col, wo)
    r, rep = G.approxim_alg1(dev(np.array([1.0, 0.0])), eps=1e-6)
    for k, v in gold.items():
        assert r[k] == pytest.approx(v, rel=1e-12), k
    wl = synth.make_config("c1")
    rp, col, wo, _ = gpu_csr(fj, wl.n, wl.u, wl.v)
    G = fj.Graph(wl.n, rp, col, wo)
    r, rep = G.approxim_alg1(dev(np.full(wl.n, 0.4)), eps=1e-6)        # consensus
    assert r["D"] == 0 and r["P"] == 0 and r["CI"] < 1e-20 and r["C"] == pytest.approx(wl.n * 0.16, rel=1e-12)


# ---------------------------------------------------------------- f4: forest-matrix entries
@pytest.mark.parametrize("m", [1, 3, 5, 70])
def test_forest_columns_vs_dense_inverse(fj, m):
    """Columns of Omega = (I+L)^{-1} against the oracle's dense inverse on C1 (k = 1, vector
    engine, warp-per-row engine, and two batches 64 + 6)."""
    wl = synth.make_config("c1")
    g = O.canonical_csr(wl.n, wl.u, wl.v)
    rp, col, wo, _ = gpu_csr(fj, wl.n, wl.u, wl.v)
    G = fj.Graph(wl.n, rp, col, wo)
    cols = np.random.default_rng(m).choice(wl.n, m, replace=False)
    Om, rep = G.forest_columns(cols, opts=fj.SolveOpts.make(rtol=1e-12))
    Om = host(Om)
    inv = np.linalg.inv(O.dense_ipl(g))
    assert rep["converged"] == 1
    assert np.max(np.abs(Om - inv[:, cols])) < 1e-11
    assert np.allclose(Om.sum(axis=0), 1.0, atol=1e-10)              # Omega 1 = 1, symmetric


def test_forest_columns_p5_golden(fj):
    """P5: 55 * Omega is the paper's integer matrix (golden p5_forest_matrix)."""
    from conftest import read_golden
    M = np.array([[int(x) for x in r] for r in read_golden("p5_forest_matrix.txt")], dtype=float)
    u = np.arange(4, dtype=np.int32)
    rp, col, wo, _ = gpu_csr(fj, 5, u, u + 1)
    G = fj.Graph(5, rp, col, wo)
    Om, _ = G.forest_columns(np.arange(5), opts=fj.SolveOpts.make(rtol=1e-14))
    assert np.allclose(host(Om) * 55, M, rtol=0, atol=1e-10)


# ---------------------------------------------------------------- f1: ingest on the device
@pytest.mark.parametrize("kind", ["uniform", "exponential", "powerlaw"])
def test_device_opinions_match_generator(fj, kind):
    """fj_opinions_generate re-implements the workloads' counter-based generator (DESIGN.md §5,
    R10): uniform bit-exact; exponential / power law within 4 ulp (device log1p / pow vs libm),
    max s = 1 exactly after the rescale."""
    n = 1_000_003
    g = host(fj.opinions_generate(n, kind, 7))
    ref = synth.opinions(kind, n, 7)
    if kind == "uniform":
        assert np.array_equal(g, ref)
    else:
        assert np.max(np.abs(g - ref) / ref) <= 4 * 2.0 ** -52
        assert g.max() == 1.0


def test_components_and_lcc_vs_oracle(fj):
    rng = np.random.default_rng(12)
    n, m = 20000, 16000                         # below the giant-component threshold: many pieces
    u = rng.integers(0, n, m).astype(np.int32)
    v = rng.integers(0, n, m).astype(np.int32)
    u[:50] = v[:50]                             # self-loops
    u[50:60] = u[60:70]; v[50:60] = v[60:70]    # duplicates
    w = rng.integers(1, 6, m).astype(np.uint8)
    lab, nc = fj.connected_components(n, dev(u), dev(v))
    ref = O.components(n, u, v)
    assert np.array_equal(host(lab), ref) and nc == len(np.unique(ref))
    vmap, u2, v2, w2, nl = fj.lcc(n, dev(u), dev(v), dev(w))
    rv, ru2, rv2, rw2, rnl = O.lcc(n, u, v, w)
    assert nl == rnl and np.array_equal(host(vmap), rv)
    assert np.array_equal(host(u2), ru2) and np.array_equal(host(v2), rv2) and np.array_equal(host(w2), rw2)
    # the LCC through the rest of the path: CSR bit-exact, quantities vs the oracle
    g = O.canonical_csr(nl, ru2, rv2, rw2)
    rp, col, wo, _ = fj.csr_from_edges(nl, u2.contiguous(), v2.contiguous(), w2.contiguous())
    assert np.array_equal(host(rp), g.row_ptr) and np.array_equal(host(col), g.col)
    G = fj.Graph(nl, rp, col, wo)
    s = host(fj.opinions_generate(nl, "exponential", 3))
    z, q, rep = G.approxim(dev(s))
    qo = O.quantities(g, s, O.solve(g, s))
    for k in QKEYS:
        assert q[0][k] == pytest.approx(qo[k], rel=1e-8), k


def test_components_long_path_and_errors(fj):
    n = 300000                                   # one path in shuffled id order: many hook rounds
    perm = np.random.default_rng(2).permutation(n).astype(np.int32)
    lab, nc = fj.connected_components(n, dev(perm[:-1]), dev(perm[1:]))
    assert nc == 1 and not host(lab).any()
    with pytest.raises(fj.FJError):
        fj.connected_components(10, dev(np.array([0], np.int32)), dev(np.array([10], np.int32)))


# ---------------------------------------------------------------- f3: Exact on the device + Table 2 protocol
def test_exact_dense_vs_oracle_and_table2_protocol(fj):
    """fj_exact_dense (dense Cholesky) on C1 against the oracle's LAPACK solve, then Table 2's
    error protocol (sigma = |rho - rho~| / rho) for fj_approxim against it on a 12000-node BA
    graph with the three opinion distributions: every sigma <= 1e-8 and within its certificate."""
    wl = synth.make_config("c1")
    g = O.canonical_csr(wl.n, wl.u, wl.v)
    rp, col, wo, _ = gpu_csr(fj, wl.n, wl.u, wl.v)
    G = fj.Graph(wl.n, rp, col, wo)
    s = wl.S[:, 0].copy()
    z, q = G.exact_dense(dev(s))
    zo = O.solve_dense(g, s)
    assert np.max(np.abs(host(z) - zo)) < 1e-13
    qo = O.quantities(g, s, zo)
    for k in QKEYS:
        assert q[0][k] == pytest.approx(qo[k], rel=1e-12), k
    wl = synth.make_config("c3", n=12000)
    rp, col, wo, _ = gpu_csr(fj, wl.n, wl.u, wl.v)
    G = fj.Graph(wl.n, rp, col, wo)
    S = dev(wl.S)
    ze, qe = G.exact_dense(S)
    za, qa, rep = G.approxim(S)
    for c in range(3):
        for k in QKEYS:
            sigma = abs(qe[c][k] - qa[c][k]) / qe[c][k]
            assert sigma <= 1e-8 and sigma <= qa[c]["eps"][k] * (1 + 1e-9) + 1e-15, (c, k, sigma)


# ---------------------------------------------------------------- degenerate graphs on every engine
@pytest.mark.parametrize("k", [1, 3, 64])
@pytest.mark.parametrize("case", ["single", "edgeless", "one_edge"])
def test_degenerate_graphs_all_engines(fj, k, case):
    """L = 0 (single node, no edges: z = s exactly, D = C_I = 0) and the 2-node path (S:L218 closed
    form) through the k = 1 engine, the vector engine (k = 3) and the warp-per-row engine (k = 64)."""
    n = {"single": 1, "edgeless": 7, "one_edge": 2}[case]
    u = np.array([0] if case == "one_edge" else [], np.int32)
    v = np.array([1] if case == "one_edge" else [], np.int32)
    rp, col, wo, _ = gpu_csr(fj, n, u, v)
    G = fj.Graph(n, rp, col, wo)
    S = np.random.default_rng(k).uniform(0.1, 1.0, (n, k))
    z, q, rep = G.approxim(dev(S if k > 1 else S[:, 0].copy()))
    Z = host(z).reshape(n, k)
    assert rep["converged"] == 1
    if case == "one_edge":
        inv = np.array([[2.0, 1.0], [1.0, 2.0]]) / 3.0          # (I+L)^{-1} of the unit 2-node path
        for c in range(k):
            assert np.allclose(Z[:, c], inv @ S[:, c], rtol=1e-10, atol=0)
            assert q[c]["D"] == pytest.approx((Z[0, c] - Z[1, c]) ** 2, rel=1e-9)
    else:
        assert np.allclose(Z, S, rtol=1e-13, atol=0)
        for c in range(k):
            assert q[c]["D"] == 0 and q[c]["CI"] <= 1e-26
            assert q[c]["C"] == pytest.approx(float((S[:, c] ** 2).sum()), rel=1e-12)


# ---------------------------------------------------------------- allocator hook
@pytest.mark.parametrize("k", [1, 3, 8])
def test_torch_allocator_hook(fj, k):
    """fj_set_allocator bound to torch's caching allocator: the library's workspace shows up in
    torch.cuda.memory_allocated() while the handle lives, every block goes back on close, and the
    results are bitwise those of the library pool."""
    import torch
    wl = synth.make_config("c2", n=200_000, k=k)
    S = dev(wl.S if k > 1 else wl.S[:, 0].copy())
    u, v = dev(wl.u), dev(wl.v)
    G0 = fj.Graph.from_edges(wl.n, u, v)
    z0, q0, _ = G0.approxim(S)
    G0.close()
    torch.cuda.synchronize()
    fj.use_torch_allocator(True)
    try:
        base = torch.cuda.memory_allocated()
        G = fj.Graph.from_edges(wl.n, u, v)
        z1, q1, rep = G.approxim(S)
        torch.cuda.synchronize()
        assert fj.allocator_live_blocks() > 0
        held = torch.cuda.memory_allocated() - base
        # at least the degree / Jacobi arrays and the solver vectors (>= 4 n k doubles) are torch's
        assert held >= 8 * wl.n * (2 + 4 * k) - 8 * wl.n * k * 2, held
        G.close()
        del G
        torch.cuda.synchronize()
        assert fj.allocator_live_blocks() == 0
    finally:
        fj.use_torch_allocator(False)
    assert torch.equal(z0, z1)
    for c in range(k):
        for key in QKEYS:
            assert q0[c][key] == q1[c][key], (c, key)
    assert rep["converged"] == 1


# ---------------------------------------------------------------- on-chip small-graph path (onchip.cu)
@pytest.mark.parametrize("name,wkind", [("c1", "unit"), ("rmat", "u8"), ("rmat", "f64"), ("iso", "unit")])
def test_onchip_small_graph_vs_oracle_and_kernel_path(fj, name, wkind):
    """fj_approxim on a graph that fits one block's shared memory runs onchip.cu (the whole solve and
    the quantities pass in one 1024-thread block); against the dense oracle, and against the multi-
    kernel path (fj_solve + fj_quantities) on the same graph."""
    rng = np.random.default_rng(11)
    if name == "c1":
        wl = synth.make_config("c1")
        n, u, v, w = wl.n, wl.u, wl.v, None
        s = wl.S[:, 0].copy()
    elif name == "rmat":
        wl = synth.make_config("c4", scale=9, k=1)
        n, u, v = wl.n, wl.u, wl.v
        w = wl.w if wkind == "u8" else rng.uniform(0.1, 4.0, len(u))
        s = wl.S[:, 0].copy()
    else:   # isolated vertices and a hub
        n = 3000
        u = np.zeros(1200, np.int64)
        v = np.arange(1, 1201)
        w = None
        s = rng.uniform(0, 1, n)
    rp, col, wo, _ = gpu_csr(fj, n, np.asarray(u), np.asarray(v), w)
    G = fj.Graph(n, rp, col, wo)
    G.approxim(dev(s))                       # warm (workspace, schedules)
    l0, _ = fj.binding.kernel_launches()
    z, q, rep = G.approxim(dev(s))
    l1, _ = fj.binding.kernel_launches()
    assert l1 - l0 <= 4, l1 - l0             # statistics + the one on-chip kernel (no PCG loop graph)
    assert rep["converged"] == 1 and rep["rel_res_true"] <= 1e-10
    g = O.canonical_csr(n, np.asarray(u), np.asarray(v), w)
    zo = O.solve_dense(g, s)
    qo = O.quantities(g, s, zo)
    assert np.max(np.abs(host(z) - zo)) < 1e-9
    for key in QKEYS:
        assert abs(q[0][key] - qo[key]) <= 1e-8 * abs(qo[key]) + 1e-300, key
        assert abs(q[0][key] - qo[key]) / qo[key] <= q[0]["eps"][key] * (1 + 1e-9) + 1e-15, key
    z2, rep2 = G.solve(dev(s))           # the multi-kernel PCG (pcg.cu) + the engine's quantities pass
    q2 = G.quantities(dev(s), z2)
    assert rep2["iterations"] == rep["iterations"]
    assert np.max(np.abs(host(z2) - host(z))) < 1e-12
    for key in QKEYS:
        assert q2[0][key] == pytest.approx(q[0][key], rel=1e-11), key

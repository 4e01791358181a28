"""Pins of the CPU oracle against values fixed by the paper and by mathematics, never against
itself (DESIGN.md §Oracle / task ③).  All run on CPU (-m "not gpu")."""
from fractions import Fraction

import numpy as np
import pytest

import oracle as O
from conftest import read_golden


def path_graph(n, w=None):
    u = np.arange(n - 1)
    v = u + 1
    return O.canonical_csr(n, u, v, w)


def complete_graph(n):
    iu, ju = np.triu_indices(n, 1)
    return O.canonical_csr(n, iu, ju)


def star_graph(n):  # hub 0, leaves 1..n-1
    return O.canonical_csr(n, np.zeros(n - 1, dtype=np.int64), np.arange(1, n))


def random_graph(n, m, rng, weighted=False, connected=False):
    u = rng.integers(0, n, m)
    v = rng.integers(0, n, m)
    if connected:  # add a random spanning path so the graph is connected
        perm = rng.permutation(n)
        u = np.concatenate([u, perm[:-1]])
        v = np.concatenate([v, perm[1:]])
    w = rng.uniform(0.2, 3.0, len(u)) if weighted else None
    return O.canonical_csr(n, u, v, w)


# ---------------------------------------------------------------- P5 worked example (paper)
def test_p5_forest_matrix_matches_paper():
    M = np.array([[int(x) for x in r] for r in read_golden("p5_forest_matrix.txt")])
    g = path_graph(5)
    Om = np.linalg.inv(O.dense_ipl(g))
    assert np.allclose(Om * 55, M, atol=1e-12, rtol=0)
    # dense solve of each unit vector reproduces the columns (P:L152 z_i = sum_j w_ij s_j)
    Z = O.solve_dense(g, np.eye(5))
    assert np.allclose(Z * 55, M, atol=1e-12, rtol=0)


def test_p5_forest_census_counts_55_and_13():
    total, E = O.forest_census(5, [(0, 1), (1, 2), (2, 3), (3, 4)])
    assert total == 55                       # P:L105 "exactly 55 spanning rooted forests"
    assert E[0][1] == 13                     # P:L105 "13 forests where v2 ... rooted at v1"
    M = np.array([[int(x) for x in r] for r in read_golden("p5_forest_matrix.txt")])
    assert (np.array(E) == M).all()          # whole matrix of P:L107-114


def _golden_fracs(name):
    return {r[0]: Fraction(int(r[1]), int(r[2])) for r in read_golden(name)}


def test_p5_e1_quantities_exact_rationals():
    gold = _golden_fracs("p5_e1_quantities.txt")
    g = path_graph(5)
    s = np.eye(5)[0]
    z = O.solve_dense(g, s)
    q = O.quantities(g, s, z)
    for k in ["CI", "D", "P", "C", "Idc", "PDI"]:
        assert q[k] == pytest.approx(float(gold[k]), rel=1e-14, abs=0), k
    # D counted once per undirected edge: C_I + 2D + C = s^T s (DESIGN reading R2)
    assert gold["CI"] + 2 * gold["D"] + gold["C"] == 1
    assert gold["CI"] + gold["D"] + gold["C"] != 1


def test_path2_quantities():
    gold = _golden_fracs("path2_quantities.txt")
    g = path_graph(2)
    s = np.array([1.0, 0.0])
    z = O.solve_dense(g, s)
    assert z == pytest.approx([float(gold["z1"]), float(gold["z2"])], rel=1e-15)
    q = O.quantities(g, s, z)
    for k in ["CI", "D", "P", "C", "Idc", "PDI"]:
        assert q[k] == pytest.approx(float(gold[k]), rel=1e-14), k


# ---------------------------------------------------------------- closed forms
@pytest.mark.parametrize("n", [2, 7, 9, 40])
def test_complete_graph_closed_form(n):
    """K_n: (I+L)^{-1} = (I+J)/(n+1) (BASELINE.json north_star)."""
    rng = np.random.default_rng(n)
    g = complete_graph(n)
    s = rng.uniform(0, 1, n)
    m = s.mean()
    S = ((s - m) ** 2).sum()
    z = O.solve_dense(g, s)
    assert np.allclose(z, (s + n * m) / (n + 1), rtol=1e-13, atol=1e-14)
    q = O.quantities(g, s, z)
    assert q["P"] == pytest.approx(S / (n + 1) ** 2, rel=1e-12)
    assert q["D"] == pytest.approx(n * S / (n + 1) ** 2, rel=1e-12)
    assert q["CI"] == pytest.approx(n * n * S / (n + 1) ** 2, rel=1e-12)
    assert q["C"] == pytest.approx(S / (n + 1) ** 2 + n * m * m, rel=1e-12)
    assert q["PDI"] == pytest.approx(S / (n + 1), rel=1e-12)
    # closed form z plugged straight into the definitions (no solve)
    q2 = O.quantities(g, s, (s + n * m) / (n + 1))
    assert q2["D"] == pytest.approx(n * S / (n + 1) ** 2, rel=1e-12)


@pytest.mark.parametrize("n", [4, 50, 1000])
def test_star_closed_form(n):
    rng = np.random.default_rng(n)
    g = star_graph(n)
    s = rng.uniform(0, 1, n)
    z0 = (2 * s[0] + s[1:].sum()) / (n + 1)
    zc = np.concatenate([[z0], (s[1:] + z0) / 2])
    z = O.solve_dense(g, s)
    assert np.allclose(z, zc, rtol=1e-13, atol=1e-15)
    zp, info = O.solve_pcg(g, s, tol=1e-14)
    assert np.allclose(zp, zc, rtol=1e-12, atol=1e-14)


def _fib(k):
    a, b = 0, 1
    for _ in range(k):
        a, b = b, a + b
    return a


@pytest.mark.parametrize("n", [5, 8, 13, 20])
def test_path_fibonacci_forest_matrix(n):
    """omega_ij = F_{2 min(i,j)-1} F_{2(n-max(i,j))+1} / F_{2n} (1-indexed); reproduces P5's 55/13."""
    g = path_graph(n)
    Om = np.linalg.inv(O.dense_ipl(g))
    F2n = _fib(2 * n)
    for i in range(1, n + 1):
        for j in range(1, n + 1):
            a, b = min(i, j), max(i, j)
            assert Om[i - 1, j - 1] == pytest.approx(_fib(2 * a - 1) * _fib(2 * (n - b) + 1) / F2n, rel=1e-12)


# ---------------------------------------------------------------- brute force
@pytest.mark.parametrize("seed", range(6))
def test_forest_census_matches_dense_inverse_weighted(seed):
    rng = np.random.default_rng(100 + seed)
    n = 6
    g = random_graph(n, 9, rng, connected=True)
    rows = g.rows()
    up = g.col > rows
    edges = list(zip(rows[up].tolist(), g.col[up].tolist()))
    wint = rng.integers(1, 4, len(edges))
    gw = O.canonical_csr(n, rows[up], g.col[up], wint.astype(np.float64))
    total, E = O.forest_census(n, edges, [int(x) for x in wint])
    Om = np.linalg.inv(O.dense_ipl(gw))
    assert np.allclose(np.array(E, dtype=float) / total, Om, rtol=1e-12, atol=1e-15)
    assert np.allclose(Om.sum(0), 1) and np.allclose(Om.sum(1), 1)   # doubly stochastic


@pytest.mark.parametrize("seed", range(8))
def test_fj_iteration_matches_dense(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(3, 30))
    g = random_graph(n, 3 * n, rng, weighted=bool(seed % 2))
    s = rng.uniform(0, 1, n)
    zi, steps = O.fj_iterate(g, s)
    assert np.allclose(zi, O.solve_dense(g, s), rtol=1e-11, atol=1e-12)


# ---------------------------------------------------------------- invariants
@pytest.mark.parametrize("seed", range(10))
def test_invariants_random(seed):
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.integers(5, 120))
    g = random_graph(n, int(rng.integers(n, 5 * n)), rng, weighted=bool(seed % 2))
    s = rng.uniform(0, 1, n)
    z = O.solve_dense(g, s)
    q = O.quantities(g, s, z)
    assert z.sum() == pytest.approx(s.sum(), rel=1e-12)                    # P:L152 conservation
    assert z.min() >= -1e-15 and z.max() <= 1 + 1e-15                       # P:L152 z in [0,1]
    assert q["CI"] + 2 * q["D"] + q["C"] == pytest.approx(q["ss"], rel=1e-11)
    assert q["Idc"] == pytest.approx(q["sz"], rel=1e-11)
    assert q["PDI"] == pytest.approx(q["sbzb"], rel=1e-10, abs=1e-13)
    assert q["CI"] == pytest.approx(q["Lz2"], rel=1e-9, abs=1e-13)          # Lz = s - z
    # Idc - PDI = n mean(s)^2 (DESIGN reading R1)
    assert q["Idc"] - q["PDI"] == pytest.approx(n * s.mean() ** 2, rel=1e-10)
    # ||W^{1/2} B x||^2 = x^T L x
    x = rng.normal(size=n)
    assert (O.incidence_apply(g, x) ** 2).sum() == pytest.approx(x @ O.laplacian_apply(g, x), rel=1e-12)
    # shift invariance of C_I, D, P
    z2 = O.solve_dense(g, s + 0.37)
    q2 = O.quantities(g, s + 0.37, z2)
    for k in ["CI", "D", "P"]:
        assert q2[k] == pytest.approx(q[k], rel=1e-9, abs=1e-13)
    # permutation invariance
    perm = rng.permutation(n)
    inv = np.argsort(perm)
    rows = g.rows()
    gp = O.canonical_csr(n, inv[rows], inv[g.col], None if g.w is None else g.w)
    sp = np.empty(n); sp[inv] = s
    qp = O.quantities(gp, sp, O.solve_dense(gp, sp))
    for k in ["CI", "D", "P", "C", "Idc", "PDI"]:
        assert qp[k] == pytest.approx(q[k], rel=1e-11, abs=1e-14)


def test_isolated_vertices_and_disjoint_union():
    rng = np.random.default_rng(5)
    g1 = random_graph(20, 40, rng)
    g2 = random_graph(15, 30, rng)
    s1, s2 = rng.uniform(0, 1, 20), rng.uniform(0, 1, 15)
    r1, r2 = g1.rows(), g2.rows()
    u = np.concatenate([r1, r2 + 20])
    v = np.concatenate([g1.col, g2.col + 20])
    g = O.canonical_csr(20 + 15 + 3, u, v)   # + 3 isolated vertices
    s = np.concatenate([s1, s2, [0.1, 0.5, 0.9]])
    z = O.solve_dense(g, s)
    assert np.array_equal(z[-3:], s[-3:]) or np.allclose(z[-3:], s[-3:], rtol=1e-15)
    q = O.quantities(g, s, z)
    qa = O.quantities(g1, s1, O.solve_dense(g1, s1))
    qb = O.quantities(g2, s2, O.solve_dense(g2, s2))
    for k in ["CI", "D", "C", "Idc"]:
        assert q[k] == pytest.approx(qa[k] + qb[k] + (k in ("C", "Idc")) * (0.01 + 0.25 + 0.81), rel=1e-12)


def test_consensus_input():
    rng = np.random.default_rng(9)
    g = random_graph(30, 90, rng)
    s = np.full(30, 0.4)
    z = O.solve_dense(g, s)
    assert np.allclose(z, s, rtol=1e-14)
    q = O.quantities(g, s, z)
    assert q["CI"] < 1e-28 and q["D"] < 1e-28 and q["P"] < 1e-28
    assert q["C"] == pytest.approx(30 * 0.16, rel=1e-14)


# ---------------------------------------------------------------- the C PCG oracle
@pytest.mark.parametrize("weighted", [False, True])
def test_pcg_oracle_matches_dense(weighted):
    import synth
    wl = synth.make_config("c1")
    w = synth.weights_u8(wl.u, wl.v, 1) if weighted else None
    g = O.canonical_csr(wl.n, wl.u, wl.v, w)
    s = wl.S[:, 0]
    zd = O.solve_dense(g, s)
    zp, info = O.solve_pcg(g, s, tol=1e-13)
    assert info["converged"] and info["rel_res"] <= 1e-13
    assert np.max(np.abs(zp - zd)) < 1e-12
    zc, info_cg = O.solve_pcg(g, s, tol=1e-13, precond=False)   # plain-CG cross-check mode
    assert info_cg["converged"] and np.max(np.abs(zc - zd)) < 1e-12
    qd, qp = O.quantities(g, s, zd), O.quantities(g, s, zp)
    for k in ["CI", "D", "P", "C", "Idc", "PDI"]:
        assert qp[k] == pytest.approx(qd[k], rel=1e-11)
    # residual of the oracle's own apply matches the numpy laplacian
    y = O.ipl_apply(g, zp)
    assert np.allclose(y, zp + O.laplacian_apply(g, zp), rtol=1e-14, atol=1e-14)


def test_pcg_oracle_zero_rhs():
    g = path_graph(10)
    z, info = O.solve_pcg(g, np.zeros(10))
    assert info["iterations"] == 0 and not z.any()


# ---------------------------------------------------------------- canonical CSR
def _brute_csr(n, u, v, w):
    first = {}
    for e, (a, b) in enumerate(zip(u.tolist(), v.tolist())):
        if a == b:
            continue
        key = (min(a, b), max(a, b))
        if key not in first:
            first[key] = e
    adj = [[] for _ in range(n)]
    for (a, b), e in first.items():
        ww = None if w is None else w[e]
        adj[a].append((b, ww))
        adj[b].append((a, ww))
    rp, cl, wl = [0], [], []
    for i in range(n):
        for j, ww in sorted(adj[i], key=lambda t: t[0]):
            cl.append(j)
            wl.append(ww)
        rp.append(len(cl))
    return np.array(rp), np.array(cl, dtype=np.int32), (None if w is None else np.array(wl))


@pytest.mark.parametrize("seed", range(8))
def test_canonical_csr_bruteforce(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 40))
    m = int(rng.integers(0, 200))
    u = rng.integers(0, n, m)
    v = rng.integers(0, n, m)
    w = rng.integers(1, 6, m).astype(np.uint8) if seed % 2 else None
    g = O.canonical_csr(n, u, v, w)
    rp, cl, wl = _brute_csr(n, u, v, w)
    assert np.array_equal(g.row_ptr, rp) and np.array_equal(g.col, cl)
    if w is not None:
        assert np.array_equal(g.w, wl)
    assert g.selfloops == int((u == v).sum())
    d = O.degrees(g)
    dd = [sum(1 if w is None else int(x) for x in (wl[rp[i]:rp[i + 1]] if w is not None else range(rp[i + 1] - rp[i])))
          for i in range(n)]
    assert np.array_equal(d, np.array(dd, dtype=float))


def test_csr_sampled_rows_match_full():
    import synth
    u, v = synth.rmat(12, 16, 0.57, 0.19, 0.19, 1)
    w = synth.weights_u8(u, v, 1)
    g = O.canonical_csr(1 << 12, u, v, w)
    rows = [0, 1, 5, 100, 4095, 2048]
    got = O.csr_rows_from_edges(1 << 12, u, v, rows, w)
    for i in rows:
        a, b = g.row_ptr[i], g.row_ptr[i + 1]
        assert np.array_equal(got[i][0], g.col[a:b])
        assert np.array_equal(got[i][1], g.w[a:b])


# ---------------------------------------------------------------- Algorithm 1 (row f2)
def test_alg1_delta_spec_examples_and_hand_value():
    """SPEC S:L139 examples of the residual map (single node: tau = delta; n = 2, w_max = 1:
    tau = delta / sqrt(3) -- the Gershgorin form 1 + 2 d_max equals SPEC's 1 + n w_max there),
    and line 1's delta for the 2-node path by hand:
    eps w_min ||s_bar|| / (3 w_max n^3 (n w_max + 1) sqrt n) = 1e-6 * sqrt(1/2) / (3 * 8 * 3 * sqrt 2)
    = 1e-6 / 144."""
    d, de, tau, cl, fl = O.alg1_delta(1, 0.0, 0.0, 0.0, 1.0, 0.1)          # L = 0
    assert tau == pytest.approx(de) and not fl
    d, de, tau, cl, fl = O.alg1_delta(2, 1.0, 1.0, 1.0, np.sqrt(0.5), 1e-6)
    assert d == pytest.approx(1e-6 / 144, rel=1e-15) and not cl and de == d
    assert tau == pytest.approx(d / np.sqrt(3), rel=1e-15)
    d, de, tau, cl, fl = O.alg1_delta(4_000_000, 1.0, 1.0, 9507.0, 577.0, 1e-6)   # C3-sized: clamped
    assert d < 1e-14 and cl and de == 1e-12 and fl and tau == 1e-14


def test_alg1_path2_matches_spec_example():
    """SPEC S:L311 example: 2-node path, s = (1, 0), eps = 1e-6 -> (C_I, D, P, C, I_dc) =
    (2/9, 1/9, 1/18, 5/9, 2/3) (golden path2); q = z - mean(s)."""
    gold = _golden_fracs("path2_quantities.txt")
    r = O.alg1(path_graph(2), np.array([1.0, 0.0]), 1e-6)
    for k in ["CI", "D", "P", "C", "Idc", "PDI"]:
        assert r[k] == pytest.approx(float(gold[k]), rel=1e-14), k
    assert r["q"] == pytest.approx(r["z"] - 0.5, abs=1e-15)


def test_alg1_equals_definitions_random_weighted():
    """For exact solves Algorithm 1's norms equal Definitions 3.1-3.4 (Lemma 4.1):
    ||L z||^2 = sum (z - s)^2, ||W^{1/2} B q||^2 = D (shift invariance), ||q||^2 = P."""
    rng = np.random.default_rng(9)
    g = random_graph(300, 1500, rng, weighted=True, connected=True)
    s = rng.uniform(0, 1, 300)
    r = O.alg1(g, s, 1e-3)
    qd = O.quantities(g, s, O.solve_dense(g, s))
    for k in ["CI", "D", "P", "C", "Idc", "PDI"]:
        assert r[k] == pytest.approx(qd[k], rel=1e-10), k


def test_alg1_consensus():
    """s = c 1 -> C_I = D = P = 0, C = n c^2 (s_bar = 0 makes the second solve trivial)."""
    g = random_graph(50, 200, np.random.default_rng(1), connected=True)
    r = O.alg1(g, np.full(50, 0.4), 1e-6)
    assert r["D"] == 0 and r["P"] == 0 and r["CI"] < 1e-28
    assert r["C"] == pytest.approx(50 * 0.16, rel=1e-13)


# ---------------------------------------------------------------- ingest (row f1)
def test_components_vs_scipy_and_lcc_by_hand():
    from scipy.sparse import coo_matrix
    from scipy.sparse.csgraph import connected_components
    rng = np.random.default_rng(4)
    n, m = 3000, 2500            # sparse: many components
    u = rng.integers(0, n, m)
    v = rng.integers(0, n, m)
    lab = O.components(n, u, v)
    nc, sl = connected_components(coo_matrix((np.ones(m), (u, v)), shape=(n, n)), directed=False)
    assert len(np.unique(lab)) == nc
    for c in range(nc):                       # same partition, label = smallest member
        members = np.flatnonzero(sl == c)
        assert np.all(lab[members] == members.min())
    # hand-built: triangle {5,6,7}, path 0-1-2-3, isolated 4, triangle {8,9,10} (ties with {5,6,7})
    u = np.array([5, 6, 7, 0, 1, 2, 8, 9, 10, 3])
    v = np.array([6, 7, 5, 1, 2, 3, 9, 10, 8, 3])
    vmap, u2, v2, w2, nl = O.lcc(11, u, v)
    assert nl == 4 and list(vmap[:5]) == [0, 1, 2, 3, -1] and np.all(vmap[5:] == -1)
    assert list(u2) == [0, 1, 2, 3] and list(v2) == [1, 2, 3, 3]            # input order, self-loop kept
    vmap, u2, v2, w2, nl = O.lcc(11, u[[0, 1, 2, 6, 7, 8]], v[[0, 1, 2, 6, 7, 8]], np.arange(6))
    assert nl == 3 and list(np.flatnonzero(vmap >= 0)) == [5, 6, 7] and list(w2) == [0, 1, 2]   # tie -> smaller ids


# ---------------------------------------------------------------- C-loop oracle for C4 / C5 scale
@pytest.mark.parametrize("seed", range(8))
def test_canonical_csr_big_bruteforce(seed):
    """oracle_csr_blocked (row block by row block) against the brute-force dict construction of the
    O-1 rules; block sizes down to one row per block force every block boundary."""
    rng = np.random.default_rng(50 + seed)
    n = int(rng.integers(1, 60))
    m = int(rng.integers(0, 400))
    u = rng.integers(0, n, m)
    v = (rng.zipf(1.5, m) % n) if seed % 3 == 0 else rng.integers(0, n, m)
    w = [None, rng.integers(1, 6, m).astype(np.uint8), rng.uniform(0.1, 3.0, m)][seed % 3]
    rp, cl, wl = _brute_csr(n, u, v, w)
    for blk in [1, 7, 1 << 20]:
        g = O.canonical_csr_big(n, u, v, w, block_entries=blk)
        assert np.array_equal(g.row_ptr, rp) and np.array_equal(g.col, cl), blk
        if w is not None:
            assert np.array_equal(g.w, wl)
        assert g.selfloops == int((u == v).sum())
        assert g.duplicates == (m - g.selfloops) - g.nnz // 2


def test_canonical_csr_big_edge_cases():
    e = np.zeros(0, dtype=np.int32)
    g = O.canonical_csr_big(5, e, e)
    assert np.array_equal(g.row_ptr, np.zeros(6, np.int64)) and g.nnz == 0
    g = O.canonical_csr_big(3, np.array([0, 1, 2]), np.array([0, 1, 2]))   # only self-loops
    assert g.nnz == 0 and g.selfloops == 3
    with pytest.raises(ValueError):
        O.canonical_csr_big(3, np.array([0]), np.array([3]))
    import synth   # R-MAT multigraph with hubs, duplicates and self-loops, u8 weights
    u, v = synth.rmat(12, 16, 0.57, 0.19, 0.19, 1)
    w = synth.weights_u8(u, v, 1)
    a, b = O.canonical_csr(1 << 12, u, v, w), O.canonical_csr_big(1 << 12, u, v, w, block_entries=5000)
    assert np.array_equal(a.row_ptr, b.row_ptr) and np.array_equal(a.col, b.col) and np.array_equal(a.w, b.w)
    assert (a.selfloops, a.duplicates) == (b.selfloops, b.duplicates)


def test_quantities_c_p5_exact_rationals_and_path2():
    """The C definitions against the paper's P5 example (s = e1, exact rationals, golden) and the
    2-node path (golden)."""
    gold = _golden_fracs("p5_e1_quantities.txt")
    g = O.canonical_csr_big(5, np.arange(4), np.arange(1, 5))
    s = np.eye(5)[0]
    q = O.quantities_c(g, s, O.solve_dense(g, s))
    for k in ["CI", "D", "P", "C", "Idc", "PDI"]:
        assert q[k] == pytest.approx(float(gold[k]), rel=1e-14, abs=0), k
    gold = _golden_fracs("path2_quantities.txt")
    g = O.canonical_csr_big(2, np.array([0]), np.array([1]))
    q = O.quantities_c(g, np.array([1.0, 0.0]), np.array([2 / 3, 1 / 3]))
    for k in ["CI", "D", "P", "C", "Idc"]:
        assert q[k] == pytest.approx(float(gold[k]), rel=1e-15), k


@pytest.mark.parametrize("seed", range(4))
def test_quantities_c_matches_definitions(seed):
    """Against the fsum definitions on random weighted graphs (both read Defs. 3.1-3.5) and the
    identities C_I + 2D + C = s^T s (R2), I_dc = s^T z, PDI = s_bar^T z_bar."""
    rng = np.random.default_rng(seed)
    n = 300
    g = random_graph(n, 1500, rng, weighted=seed % 2 == 1)
    s = rng.uniform(0, 1, n)
    z = O.solve_dense(g, s)
    a, b = O.quantities(g, s, z), O.quantities_c(g, s, z)
    for k in ["CI", "D", "P", "C", "Idc", "PDI", "sz", "sbzb", "ss"]:
        assert b[k] == pytest.approx(a[k], rel=1e-13), k
    assert b["CI"] + 2 * b["D"] + b["C"] == pytest.approx(b["ss"], rel=1e-11)
    assert b["Idc"] == pytest.approx(b["sz"], rel=1e-11)
    assert b["PDI"] == pytest.approx(b["sbzb"], rel=1e-11)


def _permute_ref(g, n2o, o2n):
    lens = np.diff(g.row_ptr)[n2o]
    rp = np.zeros(g.n + 1, np.int64)
    rp[1:] = np.cumsum(lens)
    idx = np.concatenate([np.arange(g.row_ptr[r], g.row_ptr[r + 1]) for r in n2o]) if g.nnz else np.zeros(0, int)
    return rp, o2n[g.col[idx]].astype(np.int32), (None if g.w is None else g.w[idx])


@pytest.mark.parametrize("weighted", [False, True])
def test_csr_permute_matches_transcription_and_invariance(weighted):
    """P A P^T against a numpy transcription; the quantities of the permuted graph with P s equal
    those of the original (P:L88 L -> P L P^T; sums over vertices and edges)."""
    rng = np.random.default_rng(3)
    n = 200
    g = random_graph(n, 900, rng, weighted=weighted)
    n2o = rng.permutation(n).astype(np.int32)
    o2n = np.empty(n, np.int32)
    o2n[n2o] = np.arange(n, dtype=np.int32)
    h = O.csr_permute(g, n2o, o2n)
    rp, cl, wl = _permute_ref(g, n2o, o2n)
    assert np.array_equal(h.row_ptr, rp) and np.array_equal(h.col, cl)
    if weighted:
        assert np.array_equal(h.w, wl)
    s = rng.uniform(0, 1, n)
    qa = O.quantities_c(g, s, O.solve_dense(g, s))
    hs = O.canonical_csr(n, h.rows(), h.col, h.w)   # re-sorted columns for the dense oracle
    qb = O.quantities_c(hs, s[n2o], O.solve_dense(hs, s[n2o]))
    for k in ["CI", "D", "P", "C", "Idc", "PDI"]:
        assert qb[k] == pytest.approx(qa[k], rel=1e-12), k

"""ORACLE — test infrastructure only.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs may import this package.  The product path (paper_2101_08143_b200) never
imports it, and this package never imports the product path: they share no code,
headers, tables or constants.  Only the seeded input generators (synth/) serve both.

A plain, slow, obviously-correct CPU fp64 implementation of what the hot path
computes, written from PAPER.md (/root/reference/PAPER.md, cited as P:L<n>) and
SURVEY.md §8(c).  Every function cites the passage it follows.  Pins (tests/
test_oracle_pins.py) tie each function to something other than itself: the
paper's P5 forest matrix, closed forms (K_n, star, path via Fibonacci, 2-node
path), brute-force forest enumeration and the FJ iteration (Eq. 1), and exact
identities.  No function here is "parity unpinned".

Functions
---------
canonical_csr     O-1: simple undirected graph from raw edges -> CSR ("simple graph",
                  P:L88 adjacency A=(w_ij) symmetric; SURVEY §8(c) O-1 readings for self-loops
                  and duplicates).
canonical_csr_big O-1 as plain C loops, row block by row block (C4, C5 scale).  Pinned against
                  canonical_csr on random multigraphs, many blocks forced.
csr_permute       P A P^T of a CSR (relabelling check).  Pinned against a numpy transcription and
                  against the solve invariance under relabelling.
quantities_c      Defs. 3.1-3.5 as C loops with Neumaier sums (C5 scale).  Pinned against the
                  paper's P5 example (golden) and against `quantities` on random graphs.
degrees           O-2: d_i = sum_j w_ij.
ipl_apply         (I + L) x with L = D - A.
incidence_apply   W^{1/2} B x, one entry per edge, head = lower id.
dense_ipl         dense I + L (P:L103 forest matrix Omega = (I+L)^{-1}).
solve_dense       z = (I+L)^{-1} s by dense Cholesky (Eq. (2); "Exact" P:L631).
solve_pcg         z by plain fp64 Jacobi-PCG in C, for n too large for dense.
quantities        C_I, D, P, C, I_dc by Definitions 3.1-3.5,
                  PDI = P + D (BASELINE.json north_star), cross-checks s^T z.
fj_iterate        synchronous iteration of the FJ update rule, Eq. (1).
forest_census     spanning rooted forest weights eps(Gamma), eps(Gamma_ij).
alg1_delta        Algorithm 1 line 1 delta, SPEC's clamp and the residual map.
components / lcc  connected components by union-find and the largest component's relabelled edge
                  list ("largest connected components"; row f1).  Pinned against
                  scipy.sparse.csgraph.connected_components and hand-built graphs.
alg1              Algorithm 1 Approxim step by step, both solves.
                  Pinned: SPEC's residual-map examples and a hand-computed delta (alg1_delta);
                  the 2-node path example (golden path2), consensus, and equality with
                  Definitions 3.1-3.4 on exact solves (Lemma 4.1).
"""
from __future__ import annotations

import ctypes
import itertools
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_lib = None

WT_UNIT, WT_U8, WT_F64 = 0, 1, 3


def build(force: bool = False) -> str:
    srcs = [os.path.join(_HERE, "oracle_cg.c"), os.path.join(_HERE, "oracle_big.c")]
    if force or not os.path.exists(_SO) or any(os.path.getmtime(_SO) < os.path.getmtime(f) for f in srcs):
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", _SO, *srcs, "-lm"])
    return _SO


def _L():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_SO)
        i64, ptr, dbl, cint = ctypes.c_int64, ctypes.c_void_p, ctypes.c_double, ctypes.c_int
        lib.oracle_degrees.argtypes = [i64, ptr, cint, ptr, ptr]
        lib.oracle_ipl_apply.argtypes = [i64, ptr, ptr, cint, ptr, ptr, ptr, ptr]
        lib.oracle_pcg.argtypes = [i64, ptr, ptr, cint, ptr, ptr, dbl, i64, cint, ptr, ptr]
        lib.oracle_pcg.restype = cint
        lib.oracle_pcg_fixed_iters.argtypes = [i64, ptr, ptr, cint, ptr, ptr, i64, ptr]
        lib.oracle_pcg_fixed_iters.restype = cint
        lib.oracle_num_threads.restype = cint
        lib.oracle_set_num_threads.argtypes = [cint]
        lib.oracle_set_num_threads.restype = None
        lib.oracle_csr_blocked.argtypes = [i64, i64, ptr, ptr, cint, ptr, i64, ptr, ptr, ptr, ptr]
        lib.oracle_csr_blocked.restype = i64
        lib.oracle_quantities.argtypes = [i64, ptr, ptr, cint, ptr, ptr, ptr, ptr]
        lib.oracle_quantities.restype = cint
        lib.oracle_csr_permute.argtypes = [i64, ptr, ptr, cint, ptr, ptr, ptr, ptr, ptr, ptr]
        lib.oracle_csr_permute.restype = cint
        _lib = lib
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def num_threads() -> int:
    return int(_L().oracle_num_threads())


def set_num_threads(t: int) -> None:
    _L().oracle_set_num_threads(int(t))


# --------------------------------------------------------------------------- graph
class CSR:
    """Canonical CSR of a simple undirected graph: int64 row_ptr, int32 col, weights or None."""

    def __init__(self, n, row_ptr, col, w, selfloops=0, duplicates=0):
        self.n, self.row_ptr, self.col, self.w = int(n), row_ptr, col, w
        self.selfloops, self.duplicates = int(selfloops), int(duplicates)

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1])

    @property
    def wtype(self) -> int:
        if self.w is None:
            return WT_UNIT
        return WT_U8 if self.w.dtype == np.uint8 else WT_F64

    def rows(self) -> np.ndarray:
        return np.repeat(np.arange(self.n, dtype=np.int64), np.diff(self.row_ptr))

    def wf(self) -> np.ndarray:
        return np.ones(self.nnz) if self.w is None else self.w.astype(np.float64)


def canonical_csr(n: int, u, v, w=None) -> CSR:
    """SURVEY §8(c) O-1, from the simple-graph assumption of P:L86 and the symmetric
    adjacency of P:L88 ("w_ij = w_ji = w_e"):
      1. drop self-loops (u == v);
      2. canonical key (min(u,v), max(u,v));
      3. duplicates: keep the FIRST occurrence in input order (stable sort);
      4. mirror each kept edge (lo,hi,w), (hi,lo,w);
      5. row i holds its neighbours in ascending column order; row_ptr int64."""
    u = np.asarray(u, dtype=np.int64)
    v = np.asarray(v, dtype=np.int64)
    if len(u) and (u.min() < 0 or v.min() < 0 or u.max() >= n or v.max() >= n):
        raise ValueError("vertex id out of range")
    keep = u != v
    selfloops = int(len(u) - keep.sum())
    idx = np.nonzero(keep)[0]
    lo = np.minimum(u[idx], v[idx])
    hi = np.maximum(u[idx], v[idx])
    key = lo * np.int64(n) + hi
    order = np.argsort(key, kind="stable")
    ks = key[order]
    first = np.ones(len(ks), dtype=bool)
    first[1:] = ks[1:] != ks[:-1]
    kept = idx[order[first]]                 # original edge indices, first occurrence per key
    duplicates = int(len(idx) - len(kept))
    lo = np.minimum(u[kept], v[kept])
    hi = np.maximum(u[kept], v[kept])
    rows = np.concatenate([lo, hi])
    cols = np.concatenate([hi, lo])
    o = np.lexsort((cols, rows))
    rows, cols = rows[o], cols[o]
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=n), out=row_ptr[1:])
    wo = None
    if w is not None:
        w = np.asarray(w)
        wk = w[kept]
        wo = np.concatenate([wk, wk])[o]
        if np.any(~np.isfinite(wo.astype(np.float64))) or np.any(wo.astype(np.float64) <= 0):
            raise ValueError("weights must be finite and > 0 (P:L86, w: E -> R_+)")
    return CSR(n, row_ptr, cols.astype(np.int32), wo, selfloops, duplicates)


def canonical_csr_big(n: int, u, v, w=None, block_entries: int = 1 << 28) -> CSR:
    """O-1 (same rules and citations as canonical_csr) as plain C loops, row block by row block
    (oracle_big.c), for the configs where numpy's sort keys would not fit: C4 and C5."""
    u = np.ascontiguousarray(u, dtype=np.int32)
    v = np.ascontiguousarray(v, dtype=np.int32)
    m = len(u)
    wsize, wo = 0, None
    if w is not None:
        w = np.ascontiguousarray(w)
        wsize = w.dtype.itemsize
        if w.dtype not in (np.uint8, np.float64):
            raise ValueError("weights must be uint8 or float64")
        wo = np.empty(max(2 * m, 1), dtype=w.dtype)
    row_ptr = np.empty(n + 1, dtype=np.int64)
    col = np.empty(max(2 * m, 1), dtype=np.int32)
    stats = np.zeros(2, dtype=np.int64)
    nnz = _L().oracle_csr_blocked(n, m, _p(u), _p(v), wsize, _p(w), int(block_entries), _p(row_ptr), _p(col),
                                  _p(wo), _p(stats))
    if nnz == -1:
        raise ValueError("vertex id out of range")
    if nnz < 0:
        raise MemoryError(f"oracle_csr_blocked failed ({nnz})")
    col = col[:nnz]
    if wo is not None:
        wo = wo[:nnz]
        if np.any(~np.isfinite(wo.astype(np.float64))) or np.any(wo.astype(np.float64) <= 0):
            raise ValueError("weights must be finite and > 0 (P:L86, w: E -> R_+)")
    return CSR(n, row_ptr, col, wo, int(stats[0]), int(stats[1]))


def csr_permute(g: CSR, new2old, old2new) -> CSR:
    """P A P^T: row i' = old row new2old[i'], columns mapped by old2new,
    entries in the old row's order (oracle_big.c)."""
    n2o = np.ascontiguousarray(new2old, dtype=np.int32)
    o2n = np.ascontiguousarray(old2new, dtype=np.int32)
    rp = np.empty(g.n + 1, dtype=np.int64)
    col = np.empty(max(g.nnz, 1), dtype=np.int32)
    wo = None if g.w is None else np.empty(max(g.nnz, 1), dtype=g.w.dtype)
    _L().oracle_csr_permute(g.n, _p(g.row_ptr), _p(g.col), 0 if g.w is None else g.w.dtype.itemsize, _p(g.w),
                            _p(n2o), _p(o2n), _p(rp), _p(col), _p(wo))
    return CSR(g.n, rp, col[:g.nnz], None if wo is None else wo[:g.nnz])


def degrees(g: CSR) -> np.ndarray:
    """O-2: d_i = sum_{j in Theta_i} w_ij, summed in ascending column order (C loop)."""
    d = np.empty(g.n, dtype=np.float64)
    _L().oracle_degrees(g.n, _p(g.row_ptr), g.wtype, _p(g.w), _p(d))
    return d


def ipl_apply(g: CSR, x: np.ndarray) -> np.ndarray:
    """y = (I + L) x, L = D - A."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    d = degrees(g)
    y = np.empty(g.n, dtype=np.float64)
    _L().oracle_ipl_apply(g.n, _p(g.row_ptr), _p(g.col), g.wtype, _p(g.w), _p(d), _p(x), _p(y))
    return y


def laplacian_apply(g: CSR, x: np.ndarray) -> np.ndarray:
    """(Lx)_i = d_i x_i - sum_j w_ij x_j, plain numpy."""
    rows = g.rows()
    ax = np.bincount(rows, weights=g.wf() * x[g.col], minlength=g.n)
    return np.bincount(rows, weights=g.wf(), minlength=g.n) * x - ax


def incidence_apply(g: CSR, x: np.ndarray) -> np.ndarray:
    """W^{1/2} B x: one entry per undirected edge e = (i, j), i < j (head = lower id),
    value sqrt(w_e) (x_i - x_j)  (b_e = e_i - e_j, W = diag(w_e))."""
    rows = g.rows()
    up = g.col > rows
    return np.sqrt(g.wf()[up]) * (x[rows[up]] - x[g.col[up]])


def dense_ipl(g: CSR) -> np.ndarray:
    """Dense I + L = I + D - A."""
    M = np.zeros((g.n, g.n))
    rows = g.rows()
    np.add.at(M, (rows, g.col), -g.wf())
    M[np.arange(g.n), np.arange(g.n)] += 1.0 + degrees(g)
    return M


# --------------------------------------------------------------------------- solves
def solve_dense(g: CSR, s: np.ndarray) -> np.ndarray:
    """z = (I + L)^{-1} s (Eq. (2)) via LAPACK Cholesky of the SPD matrix I + L
    (the paper's Exact).  s may be [n] or [n][k]."""
    import scipy.linalg as sla
    c = sla.cho_factor(dense_ipl(g), lower=False)
    return sla.cho_solve(c, s)


def solve_pcg(g: CSR, s: np.ndarray, tol: float = 1e-13, max_iter: int = 100000,
              precond: bool = True):
    """z = (I + L)^{-1} s by plain fp64 Jacobi-PCG (C). Returns (z, info)."""
    s2 = np.asarray(s, dtype=np.float64)
    cols = s2.reshape(g.n, -1)
    Z = np.empty_like(cols)
    infos = []
    for j in range(cols.shape[1]):
        sj = np.ascontiguousarray(cols[:, j])
        x = np.empty(g.n)
        out = np.zeros(3)
        st = _L().oracle_pcg(g.n, _p(g.row_ptr), _p(g.col), g.wtype, _p(g.w), _p(sj), tol,
                             max_iter, 1 if precond else 0, _p(x), _p(out))
        if st < 0:
            raise MemoryError("oracle_pcg allocation failed")
        Z[:, j] = x
        infos.append({"converged": st == 0, "iterations": int(out[0]), "rel_res": float(out[1]),
                      "restarts": int(out[2])})
    return Z.reshape(s2.shape), (infos[0] if s2.ndim == 1 else infos)


def pcg_fixed_iters(g: CSR, s: np.ndarray, iters: int) -> np.ndarray:
    x = np.empty(g.n)
    s = np.ascontiguousarray(s, dtype=np.float64)
    _L().oracle_pcg_fixed_iters(g.n, _p(g.row_ptr), _p(g.col), g.wtype, _p(g.w), _p(s), iters, _p(x))
    return x


def solve(g: CSR, s: np.ndarray, dense_max: int = 4096, tol: float = 1e-13):
    """Dense Cholesky for n <= 4096 (BASELINE.json north_star), PCG at rtol 1e-13 above."""
    if g.n <= dense_max:
        return solve_dense(g, s)
    return solve_pcg(g, s, tol=tol)[0]


# --------------------------------------------------------------------------- quantities
def _fsum(a: np.ndarray) -> float:
    return math.fsum(np.asarray(a, dtype=np.float64).ravel().tolist())


def quantities(g: CSR, s: np.ndarray, z: np.ndarray) -> dict:
    """The five quantities by their definitions, on a given z, summed with math.fsum
    (correctly-rounded summation):
      C_I  = sum_i (z_i - s_i)^2                          Def. 3.1
      D    = sum_{(i,j) in E} w_ij (z_i - z_j)^2          Def. 3.2, P:L183 (each edge once)
      P    = sum_i (z_i - mean(z))^2                       Def. 3.3
      C    = sum_i z_i^2                                   Def. 3.4
      I_dc = D + C                                         Def. 3.5
      PDI  = P + D                                         BASELINE.json north_star (DESIGN reading R1)
    cross-checks: sz = s^T z (= I_dc), sbzb = s_bar^T z_bar (= PDI), ss = s^T s
    (= C_I + 2D + C, DESIGN reading R2), Lz2 = ||L z||^2 (Alg. 1 line 5 form of C_I)."""
    s = np.asarray(s, dtype=np.float64)
    z = np.asarray(z, dtype=np.float64)
    n = g.n
    rows = g.rows()
    up = g.col > rows
    wu = g.wf()[up]
    CI = _fsum((z - s) ** 2)
    D = _fsum(wu * (z[rows[up]] - z[g.col[up]]) ** 2)
    mz = _fsum(z) / n
    P = _fsum((z - mz) ** 2)
    C = _fsum(z * z)
    ms = _fsum(s) / n
    return {
        "CI": CI, "D": D, "P": P, "C": C, "Idc": D + C, "PDI": P + D,
        "sz": _fsum(s * z), "sbzb": _fsum((s - ms) * (z - mz)), "ss": _fsum(s * s),
        "mean_s": ms, "mean_z": mz, "Lz2": _fsum(laplacian_apply(g, z) ** 2),
    }


def quantities_c(g: CSR, s: np.ndarray, z: np.ndarray) -> dict:
    """The same definitions as `quantities` (Defs. 3.1-3.5; PDI = P + D, reading R1)
    as C loops with Neumaier-compensated per-thread sums (oracle_big.c), for graphs whose per-edge
    terms would not fit a Python list (C5: 1.05e9 edges).  No ||Lz||^2 diagnostic."""
    s = np.ascontiguousarray(s, dtype=np.float64)
    z = np.ascontiguousarray(z, dtype=np.float64)
    out = np.zeros(9)
    wsize = 0 if g.w is None else g.w.dtype.itemsize
    _L().oracle_quantities(g.n, _p(g.row_ptr), _p(g.col), wsize, _p(g.w), _p(s), _p(z), _p(out))
    CI, D, P, C, sz, sbzb, ss, mz, ms = [float(x) for x in out]
    return {"CI": CI, "D": D, "P": P, "C": C, "Idc": D + C, "PDI": P + D, "sz": sz, "sbzb": sbzb, "ss": ss,
            "mean_s": ms, "mean_z": mz}


# --------------------------------------------------------------------------- tiny-graph pins
def fj_iterate(g: CSR, s: np.ndarray, tol: float = 1e-14, max_steps: int = 10_000_000):
    """Synchronous iteration of the FJ update rule, Eq. (1):
        z_i <- (s_i + sum_{j in Theta_i} w_ij z_j) / (1 + sum_{j in Theta_i} w_ij),
    from z^0 = s, until max_i |z^{t+1}_i - z^t_i| < tol (S:L263-279 reading).  Converges since
    the iteration matrix (I+D)^{-1}A has spectral radius <= max d_i/(1+d_i) < 1."""
    s = np.asarray(s, dtype=np.float64)
    rows = g.rows()
    wf = g.wf()
    d = np.bincount(rows, weights=wf, minlength=g.n)
    z = s.copy()
    for step in range(max_steps):
        az = np.bincount(rows, weights=wf * z[g.col], minlength=g.n)
        zn = (s + az) / (1.0 + d)
        if np.max(np.abs(zn - z), initial=0.0) < tol:
            return zn, step + 1
        z = zn
    raise RuntimeError("FJ iteration did not converge")


def forest_census(n: int, edges, weights=None):
    """Spanning rooted forests by brute-force enumeration, n <= ~8:
    a spanning forest F (acyclic edge subset) with trees T_1..T_r yields prod |T| rooted
    forests (one root per tree), each of weight eps(F) = prod_{e in F} w_e.
      eps(Gamma)    = sum_F eps(F) prod_T |T|
      eps(Gamma_ij) = sum_{F: i,j in same tree} eps(F) prod_{T not containing i} |T|
                      (the tree holding i and j is rooted at i).
    Returns (eps_Gamma, E) with E[i][j] = eps(Gamma_ij); Omega = E / eps_Gamma."""
    edges = [tuple(e) for e in edges]
    m = len(edges)
    wts = [1] * m if weights is None else list(weights)
    total = 0
    E = [[0] * n for _ in range(n)]
    for r in range(m + 1):
        for sub in itertools.combinations(range(m), r):
            parent = list(range(n))

            def find(a):
                while parent[a] != a:
                    parent[a] = parent[parent[a]]
                    a = parent[a]
                return a
            acyclic = True
            for e in sub:
                a, b = find(edges[e][0]), find(edges[e][1])
                if a == b:
                    acyclic = False
                    break
                parent[a] = b
            if not acyclic:
                continue
            wF = 1
            for e in sub:
                wF *= wts[e]
            comp = [find(a) for a in range(n)]
            size = {}
            for c in comp:
                size[c] = size.get(c, 0) + 1
            prod_all = 1
            for c in size.values():
                prod_all *= c
            total += wF * prod_all
            for i in range(n):
                rest = prod_all // size[comp[i]]   # product over trees not containing i
                for j in range(n):
                    if comp[j] == comp[i]:
                        E[i][j] += wF * rest
    return total, E


# --------------------------------------------------------------------------- sampled checks
def csr_rows_from_edges(n: int, u, v, rows_wanted, w=None):
    """Rows of the canonical CSR for a SAMPLE of vertices, computed one by one from the raw
    edge list (same O-1 rules: drop self-loops, keep-first duplicates, ascending columns).
    For full-size parity where the whole oracle CSR would be too slow.  Returns
    {i: (cols int32 array, weights or None)}."""
    u = np.asarray(u, dtype=np.int64)
    v = np.asarray(v, dtype=np.int64)
    out = {}
    want = np.asarray(sorted(set(int(i) for i in rows_wanted)), dtype=np.int64)
    hit = np.isin(u, want) | np.isin(v, want)
    eidx = np.nonzero(hit & (u != v))[0]           # input order preserved
    for i in want:
        sel = eidx[(u[eidx] == i) | (v[eidx] == i)]
        nb = np.where(u[sel] == i, v[sel], u[sel])
        _, first = np.unique(nb, return_index=True)   # first occurrence in input order
        keep = sel[np.sort(first)]
        nbk = np.where(u[keep] == i, v[keep], u[keep])
        o = np.argsort(nbk, kind="stable")
        out[int(i)] = (nbk[o].astype(np.int32), None if w is None else np.asarray(w)[keep][o])
    return out


# --------------------------------------------------------------------------- Algorithm 1 (row f2)
def alg1_delta(n: int, w_min: float, w_max: float, d_max: float, sbar_norm: float, eps: float):
    """Algorithm 1 line 1:
        delta = eps * w_min * ||s_bar|| / (3 * w_max * n^3 * (n * w_max + 1) * sqrt(n)),
    then SPEC's solver decision: used verbatim when delta >= 1e-14, else delta_eff = 1e-12
    (clamped).  Residual stop implying Lemma 4.2's T-norm bound with T = I + L: every eigenvalue of T
    lies in [1, 1 + 2 d_max] (Gershgorin; SPEC's S:L139 map uses the looser 1 + n w_max), so
    ||y - y*||_T / ||y*||_T <= sqrt(1 + 2 d_max) * ||x - T y|| / ||x||  =>  rtol = delta_eff / sqrt(1 + 2 d_max),
    floored at 1e-14 (fp64-attainable; reading R14).  Edgeless graphs (w_max = 0) use
    w_min = w_max = 1 in the formula (their solve is exact at any tolerance).
    Returns (delta, delta_eff, rtol, clamped, floored)."""
    if w_max > 0:
        delta = eps * w_min * sbar_norm / (3.0 * w_max * n ** 3 * (n * w_max + 1.0) * math.sqrt(n))
    else:
        delta = eps * sbar_norm / (3.0 * n ** 3 * math.sqrt(n))
    clamped = delta < 1e-14
    delta_eff = 1e-12 if clamped else delta
    rtol = delta_eff / math.sqrt(1.0 + 2.0 * d_max)
    floored = rtol < 1e-14
    return delta, delta_eff, (1e-14 if floored else rtol), clamped, floored


def alg1(g: CSR, s: np.ndarray, eps: float, tol: float = 1e-13) -> dict:
    """Approxim(G, s, eps), Algorithm 1, line by line; the two Solve calls are the
    oracle's own exact solves (dense Cholesky for n <= 4096, else Jacobi-PCG at rtol 1e-13, which
    meets any delta the clamp admits):
      1  delta                 (alg1_delta)
      2  s_bar = s - (1^T s / n) 1
      3  z = Solve(I + L, s, delta)
      4  q = Solve(I + L, s_bar, delta)
      5  C_I = ||L z||^2
      6  D   = ||W^{1/2} B q||^2
      7  P   = ||q||^2
      8  C   = ||z||^2
      9  I_dc = D + C"""
    s = np.asarray(s, dtype=np.float64)
    n = g.n
    wf = g.wf()
    w_min = float(wf.min()) if g.nnz else 0.0
    w_max = float(wf.max()) if g.nnz else 0.0
    d = degrees(g)
    sbar = s - _fsum(s) / n                                          # line 2
    delta = alg1_delta(n, w_min, w_max, float(d.max(initial=0.0)), math.sqrt(_fsum(sbar * sbar)), eps)
    z = solve(g, s, tol=tol)                                         # line 3
    q = solve(g, sbar, tol=tol)                                      # line 4
    CI = _fsum(laplacian_apply(g, z) ** 2)                           # line 5
    D = _fsum(incidence_apply(g, q) ** 2)                            # line 6
    P = _fsum(q * q)                                                 # line 7
    C = _fsum(z * z)                                                 # line 8
    return {"CI": CI, "D": D, "P": P, "C": C, "Idc": D + C, "PDI": P + D,   # line 9
            "delta": delta[0], "delta_eff": delta[1], "rtol": delta[2], "clamped": delta[3],
            "floored": delta[4], "z": z, "q": q}


# --------------------------------------------------------------------------- ingest (row f1)
def components(n: int, u, v) -> np.ndarray:
    """Connected components of the raw edge list by union-find (path halving, union by smaller
    id): label[i] = smallest vertex id in i's component."""
    parent = list(range(n))

    def find(x):
        while parent[x] != x:
            parent[x] = parent[parent[x]]
            x = parent[x]
        return x
    for a, b in zip(np.asarray(u).tolist(), np.asarray(v).tolist()):
        ra, rb = find(a), find(b)
        if ra != rb:
            if ra < rb:
                parent[rb] = ra
            else:
                parent[ra] = rb
    return np.array([find(i) for i in range(n)], dtype=np.int64)


def lcc(n: int, u, v, w=None):
    """Largest connected component, ties -> the component holding the smallest vertex id.
    Returns (vmap, u2, v2, w2, n_lcc): vmap[i] = new id (increasing old id) or -1; the LCC's raw
    edges relabelled in input order (self-loops / duplicates kept for the CSR rules of a1)."""
    lab = components(n, u, v)
    sizes = np.bincount(lab, minlength=n)
    roots = np.flatnonzero(lab == np.arange(n))
    best = roots[np.lexsort((roots, -sizes[roots]))[0]]
    inside = lab == best
    vmap = np.full(n, -1, dtype=np.int64)
    vmap[inside] = np.arange(int(inside.sum()))
    u = np.asarray(u)
    v = np.asarray(v)
    keep = inside[u]
    w2 = None if w is None else np.asarray(w)[keep]
    return vmap, vmap[u[keep]], vmap[v[keep]], w2, int(inside.sum())

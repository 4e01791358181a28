"""Graphs of tests/test_gpu_rows.py (shared by the test and its subprocess worker; inputs only)."""
import numpy as np

CASES = ["hub_k3_unit", "hub_k2_u8", "hub_k4_f64", "ragged_k3", "tiny_k3", "hub_k1_unit", "hub_k1_u8", "ragged_k1"]


def _hubs(rng, n, degs, extra, lo=0):
    """Random edges among [lo, n) plus hub h (< len(degs)) joined to degs[h] distinct vertices of
    [lo, n); with lo >= len(degs) every hub row has exactly degs[h] entries."""
    u = [rng.integers(lo, n, extra)]
    v = [rng.integers(lo, n, extra)]
    for h, d in enumerate(degs):
        u.append(np.full(d, h))
        v.append(lo + rng.choice(n - lo, d, replace=False))
    return np.concatenate(u).astype(np.int32), np.concatenate(v).astype(np.int32)


def case_inputs(name):
    """(n, u, v, w or None, S [n][k]) for one case, seeded."""
    rng = np.random.default_rng(sum(map(ord, name)))
    if name.startswith("hub_"):
        n = 30001                                      # odd: the slab split n // 2 is not a row boundary
        u, v = _hubs(rng, n, [9000, 4000, 1025, 300], 120000)   # chunked rows (9, 4, 2, 1 chunks)
        k = int(name[5])
        w = None
        if name.endswith("u8"):
            w = rng.integers(1, 6, len(u)).astype(np.uint8)
        elif name.endswith("f64"):
            w = rng.uniform(0.1, 4.0, len(u))
        S = rng.uniform(0, 1, (n, k))
        if k == 4:
            S[:, 3] = 0.375                            # consensus column: z = s exactly
        return n, u, v, w, S
    if name.startswith("ragged_k"):
        n = 5003
        # rows of exactly 256 / 257 / 1024 / 1025 neighbours (long-row and chunk boundaries), 1000
        # isolated vertices (rows 4003..5002), a single-edge component
        u, v = _hubs(rng, 4000, [256, 257, 1024, 1025], 9000, lo=10)
        u = np.concatenate([u, [4001]]).astype(np.int32)
        v = np.concatenate([v, [4002]]).astype(np.int32)
        return n, u, v, None, rng.uniform(0, 1, (n, int(name[-1])))
    if name == "tiny_k3":
        n = 7                                          # fewer rows than a warp's row groups
        u = np.array([0, 1, 2, 3, 0, 5], dtype=np.int32)
        v = np.array([1, 2, 3, 4, 6, 6], dtype=np.int32)
        return n, u, v, None, rng.uniform(0, 1, (n, 3))
    raise KeyError(name)

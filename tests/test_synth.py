"""Generator reproducibility and recipe checks (synth/ holds no method arithmetic)."""
import numpy as np
import pytest

import synth


def test_rand64_c_matches_numpy_mirror():
    ctr = np.arange(0, 5000, 7, dtype=np.uint64)
    a = synth.rand64_np(12345, synth.STREAM_OPINION, ctr)
    b = np.array([synth.rand64(12345, synth.STREAM_OPINION, int(c)) for c in ctr], dtype=np.uint64)
    assert np.array_equal(a, b)


def test_opinions_recipe():
    s = synth.opinions("uniform", 100_000, 2)
    assert s.min() >= 0 and s.max() < 1 and abs(s.mean() - 0.5) < 0.01
    u = (synth.rand64_np(2, synth.STREAM_OPINION, np.arange(10, dtype=np.uint64)) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    assert np.array_equal(s[:10], u)
    for kind in ["exponential", "powerlaw"]:
        x = synth.opinions(kind, 10_000, 3)
        assert x.max() == 1.0 and x.min() > 0           # divided by the max
    assert synth.opinions("exponential", 1, 3)[0] == 1.0


def test_ba_edge_count_and_structure():
    u, v = synth.barabasi_albert(2000, 3, 1)
    assert len(u) == 3 + (2000 - 3 - 1) * 3 == 5991
    assert not np.any(u == v)
    key = np.minimum(u, v).astype(np.int64) * 2000 + np.maximum(u, v)
    assert len(np.unique(key)) == len(key)              # targets distinct per new node
    u2, v2 = synth.barabasi_albert(2000, 3, 1)
    assert np.array_equal(u, u2) and np.array_equal(v, v2)


def test_er_degree():
    n = 200_000
    u, v = synth.erdos_renyi(n, 10.0 / (n - 1), 1)
    assert abs(2 * len(u) / n - 10) < 0.1
    assert np.all(u < v)


def test_rmat_and_weights():
    u, v = synth.rmat(10, 16, 0.57, 0.19, 0.19, 1)
    assert len(u) == 16 << 10 and u.max() < 1024 and v.max() < 1024
    w = synth.weights_u8(u, v, 1)
    assert w.min() >= 1 and w.max() <= 5
    w_sw = synth.weights_u8(v, u, 1)
    assert np.array_equal(w, w_sw)                     # keyed on the canonical pair

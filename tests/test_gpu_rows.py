"""The lean row product of the small-k PCG (csrc/rows.cuh) in its selections --
FJ_ROWS=0 (merge-path engine), 1 (one row pass), 2 (two column slabs; unit weights read the
slab-major column copies), "2s" (two slabs with FJ_ROWS_SPLIT=0: both passes on the CSR) -- each run
in its own process (the knob is read once per process): every column against the CPU oracle
(quantities <= 1e-8 and inside their certificates, z to 1e-9), the product (I+L)S against the
oracle's, bitwise repeatability and graph / host-loop agreement, and the path each run took."""
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle as O
from rows_cases import CASES, case_inputs

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["CI", "D", "P", "C", "Idc", "PDI"]
MODES = (0, 1, 2, "2s")
PATHS = {0: "engine", 1: "rows", 2: "rows_slabs", "2s": "rows_slabs"}


@pytest.fixture(scope="module")
def runs(tmp_path_factory):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2101_08143_b200 import build as B
    B.build()
    out = {}
    for mode in MODES:
        f = str(tmp_path_factory.mktemp("rows") / f"m{mode}.npz")
        env = dict(os.environ, FJ_ROWS=str(mode)[0], FJ_ROWS_SPLIT="0" if mode == "2s" else "1")
        r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "rows_worker.py"), f], env=env,
                           capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-3000:]
        out[mode] = dict(np.load(f))
    return out


@pytest.fixture(scope="module")
def oracle_results():
    res = {}
    for name in CASES:
        n, u, v, w, S = case_inputs(name)
        g = O.canonical_csr(n, u, v, w)
        cols = []
        for c in range(S.shape[1]):
            zo = O.solve_dense(g, S[:, c]) if n <= 4096 else O.solve_pcg(g, S[:, c], tol=1e-13)[0]
            cols.append((zo, O.quantities(g, S[:, c], zo)))
        Y = np.stack([O.ipl_apply(g, S[:, c]) for c in range(S.shape[1])], axis=1)
        # rounding scale of each row sum: (1+d_i)|x_i| + sum_j w_ij |x_j| = 2(1+d_i)|x_i| - ((I+L)|x|)_i
        d = O.degrees(g)[:, None]
        A = np.abs(S)
        T = 2 * (1 + d) * A - np.stack([O.ipl_apply(g, A[:, c]) for c in range(S.shape[1])], axis=1)
        res[name] = (g, S, cols, Y, T)
    return res


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("name", CASES)
def test_rows_product_modes_vs_oracle(runs, oracle_results, mode, name):
    r = runs[mode]
    g, S, cols, Y, T = oracle_results[name]
    path = str(r[name + "/path"])
    assert path == PATHS[mode], path
    it, conv, rel, bk = r[name + "/rep"]
    assert conv == 1 and rel <= 1e-10 and bk == (S.shape[1] if S.shape[1] > 1 else 0)
    assert r[name + "/same"].all(), r[name + "/same"]     # repeat bitwise, graph == host loop
    assert np.all(np.abs(r[name + "/y"] - Y) <= 1e-13 * T + 1e-300)   # any summation order
    rs, cs = r[name + "/solve"]
    assert cs == 1 and rs <= 1e-10                         # fj_solve's true-residual pass
    Zs = r[name + "/zs"].reshape(S.shape)
    Z, Q, E, RS = r[name + "/z"], r[name + "/q"], r[name + "/eps"], r[name + "/res"]
    for c, (zo, qo) in enumerate(cols):
        assert np.max(np.abs(Z[:, c] - zo)) < 1e-9
        assert np.max(np.abs(Zs[:, c] - zo)) < 1e-9
        if np.ptp(S[:, c]) == 0:                           # consensus column: z = s exactly
            assert np.array_equal(Z[:, c], S[:, c])
            continue
        for j, key in enumerate(KEYS):
            relq = abs(Q[c, j] - qo[key]) / abs(qo[key])
            assert relq <= 1e-8, (key, relq)
            assert relq <= E[c, j] * (1 + 1e-9) + 1e-15, (key, relq, E[c, j])
        assert RS[c, 0] <= 1e-10 * RS[c, 1] * (1 + 1e-9)


@pytest.mark.parametrize("name", CASES)
def test_rows_modes_agree(runs, name):
    """The three product paths reach the same iterates up to rounding (same iteration count +-1)."""
    its = [int(runs[m][name + "/rep"][0]) for m in MODES]
    assert max(its) - min(its) <= 1, its
    for m in MODES[1:]:
        assert np.max(np.abs(runs[m][name + "/z"] - runs[0][name + "/z"])) < 1e-9

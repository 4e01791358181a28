"""Full-size parity at BASELINE.json's largest configs, in the launch configuration bench.py times:
sampled outputs the oracle computes one by one, plus properties that hold at any size.

C4 (R-MAT 22, weights 1..5, k = 64 batched): sampled columns against the oracle's own CSR and
Jacobi-PCG at rtol 1e-13 and its definitions of the quantities.
C5 (R-MAT 26, 1.07e9 raw edges): CSR rows sampled and rebuilt by the oracle from the raw edge
list; the residual (I+L)z - s on those rows recomputed by the oracle from its own rows; global
identities C_I + 2D + C = s^T s, I_dc = s^T z, mean conservation; quantities C, C_I, P recomputed
by the oracle's definitions from z."""
import math

import numpy as np
import pytest

import oracle as O
import synth

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
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


def test_c4_full_k64_sampled_columns(fj):
    import torch
    wl = synth.make_config("c4")                       # k = 64
    G = fj.Graph.from_edges(wl.n, torch.from_numpy(wl.u).cuda(), torch.from_numpy(wl.v).cuda(),
                            torch.from_numpy(wl.w).cuda())
    Z, Q, rep = G.approxim(torch.from_numpy(wl.S).cuda())
    assert rep["batch_k"] == 64 and rep["converged"] == 1 and rep["rel_res_true"] <= 1e-10
    Z = Z.cpu().numpy()
    g = O.canonical_csr(wl.n, wl.u, wl.v, wl.w)
    for c in [0, 37]:
        # hub rows (d ~ 8e5 with weights) put the fp64 residual floor near 1e-13: ask for 1e-12
        zo, info = O.solve_pcg(g, wl.S[:, c], tol=1e-12)
        assert info["converged"] and info["rel_res"] <= 1e-12, info
        qo = O.quantities(g, wl.S[:, c], zo)
        for k in QKEYS:
            rel = abs(Q[c][k] - qo[k]) / qo[k]
            assert rel <= 1e-8, (c, k, rel)
            assert rel <= Q[c]["eps"][k] * (1 + 1e-9) + 1e-15
        assert np.max(np.abs(Z[:, c] - zo)) < 1e-8


def test_c5_full_sampled_rows_and_identities(fj):
    import torch
    wl = synth.make_config("c5")
    u, v = torch.from_numpy(wl.u).cuda(), torch.from_numpy(wl.v).cuda()
    rp, col, _, stats = fj.csr_from_edges(wl.n, u, v)
    G = fj.Graph(wl.n, rp, col, None, validate=False)
    s = wl.S[:, 0]
    z, q, rep = G.approxim(torch.from_numpy(s.copy()).cuda())
    assert rep["converged"] == 1 and rep["rel_res_true"] <= 1e-10
    z = z.cpu().numpy()
    q = q[0]
    rp_h = rp.cpu().numpy()
    deg = np.diff(rp_h)
    rng = np.random.default_rng(1)
    rows = sorted(set(rng.integers(0, wl.n, 60).tolist() + np.argsort(deg)[-3:].tolist()))
    want = O.csr_rows_from_edges(wl.n, wl.u, wl.v, rows)
    snorm = math.sqrt(math.fsum((s * s).tolist()))
    for i, (cref, _) in want.items():
        a, b = rp_h[i], rp_h[i + 1]
        assert np.array_equal(col[a:b].cpu().numpy(), cref), i
        # oracle residual row from its own neighbour list: |(s - (I+L)z)_i| <= ||r|| <= 1e-10 ||s||
        t = z[i] * (1 + len(cref)) - math.fsum(z[cref].tolist())
        assert abs(s[i] - t) <= 1e-10 * snorm * 1.01 + 1e-13 * (1 + len(cref)), i
    # identities at any size (DESIGN reading R2)
    ss = math.fsum((s * s).tolist())
    assert (q["CI"] + 2 * q["D"] + q["C"]) == pytest.approx(ss, rel=1e-9)
    assert q["Idc"] == pytest.approx(math.fsum((s * z).tolist()), rel=1e-10)
    assert math.fsum(z.tolist()) == pytest.approx(math.fsum(s.tolist()), rel=1e-10)
    # definitions recomputed by the oracle from the GPU's z (no CSR needed for these three)
    m = math.fsum(z.tolist()) / wl.n
    assert q["C"] == pytest.approx(math.fsum((z * z).tolist()), rel=1e-12)
    assert q["CI"] == pytest.approx(math.fsum(((z - s) ** 2).tolist()), rel=1e-12)
    assert q["P"] == pytest.approx(math.fsum(((z - m) ** 2).tolist()), rel=1e-8)
    iso = deg == 0
    assert np.array_equal(z[iso], s[iso]) or np.allclose(z[iso], s[iso], rtol=1e-12)

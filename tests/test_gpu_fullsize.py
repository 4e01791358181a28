"""Full-size parity at BASELINE.json's largest configs, in the launch configuration bench.py times:
sampled outputs the oracle computes one by one, plus properties that hold at any size.

C4 (R-MAT 22, weights 1..5, k = 64 batched): sampled columns against the oracle's own CSR and
Jacobi-PCG at rtol 1e-13 and its definitions of the quantities.
C5 (R-MAT 26, 1.07e9 raw edges), in the input labels and through the degree relabelling the bench
uses: the whole CSR bit-exact against the oracle's C-loop builder, z element by element against
the oracle's Jacobi-PCG at rtol 1e-12, and the six quantities within 1e-8 of the oracle's
definitions (and within their certificates)."""
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


@pytest.fixture(scope="module")
def c5():
    """C5 (BASELINE configs[4]: R-MAT 26, 1.07e9 raw edges) and its oracle: the canonical CSR by
    the C-loop builder (row block by row block), z by the oracle's Jacobi-PCG at rtol 1e-12, the
    quantities by the definitions with compensated sums.  Nothing here comes from the GPU."""
    import time
    t0 = time.time()
    wl = synth.make_config("c5")
    g = O.canonical_csr_big(wl.n, wl.u, wl.v, block_entries=1 << 29)
    s = np.ascontiguousarray(wl.S[:, 0])
    zo, info = O.solve_pcg(g, s, tol=1e-12)
    assert info["converged"] and info["rel_res"] <= 1e-12, info
    qo = O.quantities_c(g, s, zo)
    rnorm_o = info["rel_res"] * math.sqrt(qo["ss"])
    print(f"c5 oracle: nnz={g.nnz} pcg={info} {time.time() - t0:.0f} s")
    return wl, g, s, zo, qo, rnorm_o


def _check_c5(q, z, zo, qo, rnorm_gpu, rnorm_o):
    # z element by element: |z - z*| <= ||z - z*||_2 <= ||r|| (lambda_min(I+L) = 1),
    # so two solves differ by at most the sum of their residual norms (rigorous, any size)
    err = float(np.max(np.abs(z - zo)))
    assert err <= rnorm_gpu + rnorm_o, (err, rnorm_gpu, rnorm_o)
    for k in QKEYS:
        rel = abs(q[k] - qo[k]) / abs(qo[k])
        assert rel <= 1e-8, (k, rel)
        assert rel <= q["eps"][k] * (1 + 1e-9) + 1e-15, (k, rel, q["eps"][k])
    return err


def test_c5_full_vs_oracle_natural(fj, c5):
    """C5 in the input labels: the GPU CSR bit-exact against the oracle's, z element by element,
    the six quantities within 1e-8 of the oracle's definitions and within their certificates."""
    import torch
    wl, g, s, zo, qo, rnorm_o = c5
    u, v = torch.from_numpy(wl.u).cuda(), torch.from_numpy(wl.v).cuda()
    rp, col, _, stats = fj.csr_from_edges(wl.n, u, v)
    del u, v
    assert stats["nnz"] == g.nnz and stats["selfloops"] == g.selfloops and stats["duplicates"] == g.duplicates
    assert np.array_equal(rp.cpu().numpy(), g.row_ptr)
    step = 1 << 28
    for a in range(0, g.nnz, step):      # block by block (bounded host copies)
        b = min(a + step, g.nnz)
        assert np.array_equal(col[a:b].cpu().numpy(), g.col[a:b]), a
    G = fj.Graph(wl.n, rp, col, None, validate=False)
    z, q, rep = G.approxim(torch.from_numpy(s.copy()).cuda())
    assert rep["converged"] == 1 and rep["rel_res_true"] <= 1e-10
    q = q[0]
    err = _check_c5(q, z.cpu().numpy(), zo, qo, q["res_norm"], rnorm_o)
    print(f"c5 natural: max|z - z_oracle| = {err:.3e}, iterations {rep['iterations']}")
    G.close()


def test_c5_full_vs_oracle_degree_order(fj, c5):
    """C5 through the relabelled handle the bench uses (FJ_ORDER_AUTO picks it for C5): the degree
    order and P A P^T bit-exact against the oracle's stable argsort and permutation of its own CSR;
    z (mapped back to the input labels) and the quantities against the oracle on the ORIGINAL graph."""
    import torch
    wl, g, s, zo, qo, rnorm_o = c5
    u, v = torch.from_numpy(wl.u).cuda(), torch.from_numpy(wl.v).cuda()
    G = fj.Graph.from_edges(wl.n, u, v, order="degree")
    del u, v
    deg = np.diff(g.row_ptr)
    n2o_ref = np.argsort(-deg, kind="stable").astype(np.int32)
    n2o = G.new2old.cpu().numpy()
    assert np.array_equal(n2o, n2o_ref)
    o2n = G.old2new.cpu().numpy()
    assert np.array_equal(o2n[n2o_ref], np.arange(wl.n, dtype=np.int32))
    h = O.csr_permute(g, n2o_ref, o2n)
    rp, col = G._keep[0], G._keep[1]
    assert np.array_equal(rp.cpu().numpy(), h.row_ptr)
    step = 1 << 28
    for a in range(0, h.nnz, step):
        b = min(a + step, h.nnz)
        assert np.array_equal(col[a:b].cpu().numpy(), h.col[a:b]), a
    del h
    z, q, rep = G.approxim(torch.from_numpy(s.copy()).cuda())
    assert rep["converged"] == 1 and rep["rel_res_true"] <= 1e-10
    q = q[0]
    err = _check_c5(q, z.cpu().numpy(), zo, qo, q["res_norm"], rnorm_o)
    print(f"c5 degree order: max|z - z_oracle| = {err:.3e}, iterations {rep['iterations']}")
    G.close()

"""Subprocess worker of tests/test_gpu_rows.py (not a test module): runs the small-k solve, the
quantities and the product on the graphs of that test with the product path selected by the
environment (FJ_ROWS is read once per process), and saves the GPU results to an .npz.
  FJ_ROWS=<0|1|2> python tests/rows_worker.py <out.npz>"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2101_08143_b200 as fj  # noqa: E402
from rows_cases import CASES, case_inputs  # noqa: E402

out = {}
for name in CASES:
    n, u, v, w, S = case_inputs(name)
    k = S.shape[1]
    G = fj.Graph.from_edges(n, torch.from_numpy(u).cuda(), torch.from_numpy(v).cuda(),
                            None if w is None else torch.from_numpy(w).cuda())
    Sd = torch.from_numpy(S).cuda()
    z, q, rep = G.approxim(Sd)
    z2, _, rep2 = G.approxim(Sd)                                                   # repeat: bitwise
    z3, _, rep3 = G.approxim(Sd, opts=fj.SolveOpts.make(use_cuda_graph=False))   # host-driven loop
    y = G.apply(Sd)                                                              # (I+L) S
    zs, reps = G.solve(Sd)                                   # fj_solve: the true-residual pass runs
    out[name + "/zs"] = zs.cpu().numpy()
    out[name + "/solve"] = np.array([reps["rel_res_true"], reps["converged"]])
    out[name + "/z"] = z.cpu().numpy()
    out[name + "/y"] = y.cpu().numpy()
    out[name + "/q"] = np.array([[qc[key] for key in ["CI", "D", "P", "C", "Idc", "PDI"]] for qc in q])
    out[name + "/eps"] = np.array([[qc["eps"][key] for key in ["CI", "D", "P", "C", "Idc", "PDI"]] for qc in q])
    out[name + "/res"] = np.array([[qc["res_norm"], qc["s_norm"]] for qc in q])
    out[name + "/rep"] = np.array([rep["iterations"], rep["converged"], rep["rel_res_true"], rep["batch_k"]])
    out[name + "/same"] = np.array([bool(torch.equal(z, z2)), bool(torch.equal(z, z3)),
                                    rep["iterations"] == rep2["iterations"] == rep3["iterations"]])
    out[name + "/path"] = np.array(G.product_path(k))
    G.close()
np.savez(sys.argv[1], **out)
print("ok", len(CASES))

"""Lean column-slab product probe: the C3 k = 3 product q = (I+L)p computed by the
lean row kernel of tools/slab2_probe.cu, as one pass over the whole CSR or as S passes over column
slabs, against the engine's product (fj_time_spmv) and its result (fj_apply).
  python tools/slab2_probe.py --config c3
One JSON line per variant: ms per product (CUDA events, back to back), max |q - q_engine|."""
import argparse
import ctypes
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2101_08143_b200 as fj  # noqa: E402
import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--order", default="natural", choices=["natural", "degree"])
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--S", type=int, nargs="+", default=[1, 2, 3, 4])
ap.add_argument("--GU", default="1x4,2x4,4x4,8x2,8x4,16x1,16x2,32x1")
ap.add_argument("--minb", type=int, nargs="+", default=[4])
ap.add_argument("--fracs", type=float, nargs="*", default=[])
ap.add_argument("--splits", default="cols,nnz")
a = ap.parse_args()

libs = {}
for mb in a.minb:
    so = f"/tmp/slab2_probe_{mb}.so"
    subprocess.check_call(["nvcc", "-O3", "-shared", "-Xcompiler", "-fPIC", "-gencode", "arch=compute_100a,code=sm_100a",
                           f"-DFJ_MINB={mb}", "-o", so, os.path.join(ROOT, "tools", "slab2_probe.cu")])
    L = ctypes.CDLL(so)
    L.slab_pass.restype = ctypes.c_int
    L.slab_pass.argtypes = [ctypes.c_int] * 4 + [ctypes.c_int64] + [ctypes.c_void_p] * 5 + [ctypes.c_int, ctypes.c_void_p]
    L.slab_chunks.restype = ctypes.c_int
    L.slab_chunks.argtypes = [ctypes.c_int64] + [ctypes.c_void_p] * 5
    libs[mb] = L

wl = synth.make_config(a.config)
u, v = torch.from_numpy(wl.u).cuda(), torch.from_numpy(wl.v).cuda()
G0 = fj.Graph.from_edges(wl.n, u, v, order=a.order)
rp, col, _ = G0._keep
n = wl.n
deg = G0.degrees() if a.order == "natural" else None
if deg is None:   # relabelled handle: degrees in the handle's labels
    deg = torch.diff(rp).to(torch.float64)
g = torch.Generator(device="cuda").manual_seed(7)
p4 = torch.zeros(n, 4, dtype=torch.float64, device="cuda")
p4[:, :3] = torch.rand(n, 3, generator=g, device="cuda", dtype=torch.float64)
q_eng = G0.apply(p4[:, :3].contiguous()) if a.order == "natural" else None
t_eng = G0.time_spmv(k=3, reps=a.reps)
print(json.dumps({"variant": "engine", "ms": t_eng}), flush=True)

rows = torch.repeat_interleave(torch.arange(n, device="cuda"), torch.diff(rp))
c64 = col.to(torch.int64)
st = torch.cuda.current_stream().cuda_stream


LONG_ROW, CH = 256, 512


def chunks(rpb):
    ln = torch.diff(rpb)
    lr = torch.nonzero(ln > LONG_ROW).flatten()
    out = []
    for i in lr.tolist():
        b, e = int(rpb[i]), int(rpb[i + 1])
        out += [(i, k, min(k + CH, e)) for k in range(b, e, CH)]
    return torch.tensor(out, dtype=torch.int64, device="cuda").reshape(-1, 3)


def slabs(S, split):
    if S == 1:
        return [(rp, col, chunks(rp))]
    if split == "cols":
        bnd = [n * b // S for b in range(S + 1)]
    elif split.startswith("f"):
        bnd = [0, int(n * float(split[1:])), n]
    else:
        cnt = torch.bincount(c64, minlength=n).cumsum(0)
        tot = int(cnt[-1])
        bnd = [0] + [int(torch.searchsorted(cnt, tot * b // S)) for b in range(1, S)] + [n]
    out = []
    for b in range(S):
        m = (c64 >= bnd[b]) & (c64 < bnd[b + 1])
        cb = col[m].contiguous()
        rpb = torch.zeros(n + 1, dtype=torch.int64, device="cuda")
        rpb[1:] = torch.bincount(rows[m], minlength=n).cumsum(0)
        out.append((rpb, cb, chunks(rpb)))
    return out


def run(L, parts, G, U, blocks, q):
    S = len(parts)
    for b, (rpb, cb, ch) in enumerate(parts):
        rc = L.slab_pass(G, U, int(b == 0), int(b == S - 1), n, rpb.data_ptr(), cb.data_ptr(), p4.data_ptr(),
                         deg.data_ptr(), q.data_ptr(), blocks, st)
        assert rc == 0, rc
        rc = L.slab_chunks(ch.shape[0], ch.data_ptr(), cb.data_ptr(), p4.data_ptr(), q.data_ptr(), st)
        assert rc == 0, rc


cases = [(S, sp) for S in a.S for sp in (a.splits.split(",") if S > 1 else ["cols"])]
cases += [(2, f"f{f}") for f in a.fracs]
for S, split in cases:
    if True:
        parts = slabs(S, split)
        for mb, L in libs.items():
            for gu in a.GU.split(","):
                G, U = map(int, gu.split("x"))
                for bpsm in sorted({mb, 2 * mb}):
                    blocks = 148 * bpsm
                    q = torch.empty(n, 3, dtype=torch.float64, device="cuda")
                    run(L, parts, G, U, blocks, q)
                    torch.cuda.synchronize()
                    err = float((q - q_eng).abs().max()) if q_eng is not None else None
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record()
                    for _ in range(a.reps):
                        run(L, parts, G, U, blocks, q)
                    e1.record()
                    torch.cuda.synchronize()
                    tot = e0.elapsed_time(e1) / a.reps
                    per = []
                    for b in range(len(parts)):
                        one = [parts[b]]
                        e0.record()
                        for _ in range(a.reps):
                            L.slab_pass(G, U, 1, 1, n, one[0][0].data_ptr(), one[0][1].data_ptr(), p4.data_ptr(),
                                        deg.data_ptr(), q.data_ptr(), blocks, st)
                            L.slab_chunks(one[0][2].shape[0], one[0][2].data_ptr(), one[0][1].data_ptr(), p4.data_ptr(),
                                          q.data_ptr(), st)
                        e1.record()
                        torch.cuda.synchronize()
                        per.append(round(e0.elapsed_time(e1) / a.reps, 4))
                    print(json.dumps({"variant": "lean", "per_slab_ms": per, "S": S, "split": split, "G": G, "U": U, "minb": mb,
                                      "blocks_per_sm": bpsm, "ms": tot, "max_err": err,
                                      "slab_nnz": [int(c.numel()) for _, c, _ in parts], "chunks": [int(h.shape[0]) for _, _, h in parts]}), flush=True)
        del parts
        torch.cuda.empty_cache()

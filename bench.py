#!/usr/bin/env python
"""Benchmark of the hot path on B200: one JSON line on rank 0.

A "step" = one pass of the whole hot path over one batch of synthetic input resident in HBM:
  a1 fj_csr_from_edges (raw edges -> canonical CSR)  a2 fj_graph_create (degrees, schedule)
  a3-a7 fj_approxim (statistics, Jacobi-PCG solve per opinion column, fused quantities pass,
  certificate).  Default workload: BASELINE.json configs[2] (C3: BA n=4e6, m=8, three opinion
  distributions), the config the metric is quoted on at 1/2/4/8 B200.

value = CG-iteration GB/s = canonical bytes per PCG iteration B(k) x PCG iterations
        / device time of the PCG iterations (CUDA events inside the library, on the caller's stream),
        summed over the K timed steps (max over ranks for the time).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "CG-iteration GB/s & fraction of HBM roofline; time-to-{P,D,I,C} at 1/2/4/8 B200"
L2_FLUSH_BYTES = 512 << 20


def canonical_bytes(n, nnz, wb, k):
    """B(k) = (4 + w_b) nnz + 8 (n+1) + 16 n + 88 n k  (one PCG iteration)."""
    return (4 + wb) * nnz + 8 * (n + 1) + 16 * n + 88 * n * k


def spmv_bytes(n, nnz, wb, k):
    """B_spmv = (4 + w_b) nnz + 8 (n+1) + 16 n k  (one (I+L)p product)."""
    return (4 + wb) * nnz + 8 * (n + 1) + 16 * n * k


def spmv_kernel_name(k, path="engine"):
    if k == 1 and path == "rows":
        return "k_rows_chunks + k_rows<PASS 2> ((I+L)p SpMV, lean row kernel, one pass, k = 1; DESIGN.md 6.10)"
    if k == 1 and path == "rows_slabs":
        return "k_rows<PASS 0> + k_rows<PASS 1> ((I+L)p SpMV, lean row kernel over two column slabs, k = 1)"
    if k == 1:
        return "warp_kernel<ApplyOp> ((I+L)p SpMV, warp-item engine, k = 1)"
    kp = 2 if k <= 2 else 4
    if k <= 4 and path == "rows_slabs":
        return (f"k_rows_chunks + k_rows<PASS 0> + k_rows<PASS 1> ((I+L)P, lean row kernel over two column "
                f"slabs, k = {k} padded to {kp}; one product = these launches, DESIGN.md 6.10)")
    if k <= 4 and path == "rows":
        return f"k_rows_chunks + k_rows<PASS 2> ((I+L)P, lean row kernel, one pass, k = {k} padded to {kp})"
    if k <= 4:
        return f"warp_kernel<ApplyOpV<KP={kp}>> ((I+L)P SpMM, warp-item engine, k = {k} padded)"
    return f"spmm_kernel<BM_APPLY> ((I+L)P SpMM, warp per row, k = {k})"


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons DURING the timed region (B200_PROFILING.md)."""

    def __init__(self, index=0):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(index), f"--query-gpu={q}",
                                       "--format=csv,noheader,nounits", "-lms", "50"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except FileNotFoundError:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.p.kill()
        self.f.flush()
        rows = []
        with open(self.f.name) as fh:
            for line in fh:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 8:
                    rows.append(parts)
        os.unlink(self.f.name)
        if not rows:
            return None
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = max(float(r[1]) for r in rows if r[1].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[4 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(rows)}


def dist_init():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def cpu_model():
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def oracle_ttq(g, s, rtol):
    """The oracle as it stands: Jacobi-PCG to `rtol` on the true residual (restarts included), then
    the quantities by their definitions.  Returns (seconds, solve seconds, iterations)."""
    import oracle as O
    t = time.perf_counter()
    z, info = O.solve_pcg(g, s, tol=rtol)
    t_solve = time.perf_counter() - t
    O.quantities_c(g, s, z)
    return time.perf_counter() - t, t_solve, info["iterations"]


def cpu_baseline(wl, g, rtol, one_core_budget_s=40.0):
    """SURVEY §8(d) protocol: the oracle's time-to-quantities at the GPU's rtol on all host cores
    (every opinion column of the workload, up to 3) and on one core (column 0, when its estimate
    fits the budget), with the CPU model; value = CG-iteration GB/s of the all-core solves."""
    import oracle as O
    wb = 0 if wl.w is None else wl.w.dtype.itemsize
    B1 = canonical_bytes(g.n, g.nnz, wb, 1)
    allc = O.num_threads()
    cols = []
    tot_solve, tot_it = 0.0, 0
    for c in range(min(wl.k, 3)):
        s = np.ascontiguousarray(wl.S[:, c])
        ttq, t_solve, it = oracle_ttq(g, s, rtol)
        cols.append({"opinions": wl.kinds[c], "time_to_quantities_ms": 1e3 * ttq, "iterations": it})
        tot_solve += t_solve
        tot_it += it
    one = None
    est = tot_solve / max(len(cols), 1) * allc
    if est <= one_core_budget_s:
        O.set_num_threads(1)
        try:
            ttq1, ts1, it1 = oracle_ttq(g, np.ascontiguousarray(wl.S[:, 0]), rtol)
        finally:
            O.set_num_threads(allc)
        one = {"cores": 1, "time_to_quantities_ms": 1e3 * ttq1, "iterations": it1, "value": B1 * it1 / ts1 / 1e9}
    return {"value": B1 * tot_it / tot_solve / 1e9, "unit": "GB/s", "cores": allc, "kind": "oracle",
            "cpu_model": cpu_model(), "rtol": rtol, "per_column": cols, "one_core": one,
            "sample": f"oracle Jacobi-PCG to rtol {rtol:g} (true residual, restarts included) + the quantities "
                      f"by definition, per opinion column ({len(cols)} of {wl.k}) of the full {wl.name} graph "
                      f"(n={g.n}, nnz={g.nnz}), CSR built untimed; value = B(1) x iterations / solve time"}


def run_reference(args, ws, rank):
    """--impl reference: the CPU oracle as it stands, on this arm's config / metric / unit.  Each
    step = the oracle's time-to-quantities of opinion column 0 at the GPU's rtol (all host cores)."""
    if rank != 0:
        return 0
    import oracle as O
    import synth
    wl = synth.make_config(args.config)
    big = wl.name in ("c4", "c5")
    g = O.canonical_csr_big(wl.n, wl.u, wl.v, wl.w) if big else O.canonical_csr(wl.n, wl.u, wl.v, wl.w)
    wb = 0 if wl.w is None else wl.w.dtype.itemsize
    B = canonical_bytes(g.n, g.nnz, wb, 1)
    s = np.ascontiguousarray(wl.S[:, 0])
    for _ in range(args.warmup):
        oracle_ttq(g, s, args.rtol)
    times, solve_s, iters = [], 0.0, 0
    for _ in range(args.steps):
        ttq, t_solve, it = oracle_ttq(g, s, args.rtol)
        times.append(ttq)
        solve_s += t_solve
        iters += it
    tot = sum(times)
    value = B * iters / solve_s / 1e9
    sample = (f"each step: the oracle's time-to-quantities of opinion column 0 ({wl.kinds[0]}) at rtol {args.rtol:g} "
              f"(Jacobi-PCG, true-residual restarts, definitions) on the full {wl.name} graph (n={g.n}, "
              f"nnz={g.nnz}), CSR built once untimed")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{wl.name}: {wl.desc}", "n": g.n, "nnz": g.nnz, "rtol": args.rtol},
            "time_to_quantities_ms": 1e3 * statistics.median(times),
            "cpu_baseline": {"value": value, "unit": "GB/s", "cores": O.num_threads(), "kind": "oracle",
                             "cpu_model": cpu_model(), "sample": sample},
            "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="fj", choices=["fj", "reference"])
    ap.add_argument("--config", default="c3")
    ap.add_argument("--rtol", type=float, default=1e-10)
    ap.add_argument("--vertex-order", default="auto", choices=["auto", "degree", "natural"],
                    help="a1 locality relabelling by descending degree, inside the timed step (DESIGN.md "
                         "§6.7); auto = FJ_ORDER_AUTO's rule (k <= 2 and the gathered vector exceeds L2); "
                         "on the row-partitioned N>1 path the relabelling precedes the partition")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--dist-selftest", action="store_true",
                    help="run the row-partitioned (multi-GPU) code path on ONE GPU through a 1-rank NCCL "
                         "communicator (no halo); checks that bench.py --gpus N is ready")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the per-distribution k = 1 lines and the gather probe (profiling runs)")
    ap.add_argument("--spmv-reps", type=int, default=20)
    ap.add_argument("--no-cuda-graph", action="store_true",
                    help="host-driven PCG loop (same kernels); ncu cannot see kernels inside conditional graphs")
    args = ap.parse_args()
    os.environ.setdefault("NCCL_DEBUG", "WARN")
    # NCCL prints its version banner (and any warning) on stdout at WARN: send it to stderr so that
    # rank 0's stdout is the one JSON line
    os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    ws, rank, local = dist_init()
    if args.impl == "reference":
        return run_reference(args, ws, rank)

    import torch
    import torch.distributed as dist
    import paper_2101_08143_b200 as fj
    import synth
    from paper_2101_08143_b200 import binding

    torch.cuda.set_device(local)
    dist_mode = ws > 1 or args.dist_selftest
    if args.dist_selftest and ws == 1:   # the row-partitioned path on a 1-rank NCCL communicator
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29577")
        os.environ["FJ_NCCL_FORCE"] = "1"
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", local))
    elif ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    fj.load_library()
    wl = synth.make_config(args.config)
    n, k = wl.n, wl.k
    wb = 0 if wl.w is None else wl.w.dtype.itemsize
    u = torch.from_numpy(wl.u).cuda()
    v = torch.from_numpy(wl.v).cuda()
    w = None if wl.w is None else torch.from_numpy(wl.w).cuda()
    S = torch.from_numpy(wl.S).cuda()
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.int32, device="cuda")
    order = args.vertex_order
    if order == "auto":   # same rule on 1 GPU and on the row-partitioned path
        order = "degree" if binding.relabel_pays(n, k) else "natural"
    opts = fj.SolveOpts.make(rtol=args.rtol, use_cuda_graph=not args.no_cuda_graph, vertex_order=order)
    stream = torch.cuda.current_stream()

    if dist_mode:   # rows a8/e: the graph row-partitioned over the ranks, NCCL halo + allreduce
        from paper_2101_08143_b200 import dist as FD
        uid = [fj.Comm.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        comm = fj.Comm.nccl(ws, rank, uid[0])
        grp = FD.TorchGroup(None, device=f"cuda:{local}")

    def step():
        if dist_mode:
            G, b = FD.build_dist_graph(comm, rank, n, u, v, w, grp, order=order)   # partition + a1 + ghosts + a2
            Sl = FD.slice_in(G, S, b)
            z, q, rep = G.approxim(Sl, opts=opts)
            info = {"nnz": G.plan["nnz_local"], "bounds": b}
            G.close()
            return q, rep, info, G.plan
        G = fj.Graph.from_edges(n, u, v, w, order=order)   # a1 (+ relabelling) + a2
        z, q, rep = G.approxim(S, opts=opts)                 # s mapped in, z mapped back out
        info = G.info()
        G.close()
        return q, rep, info, G.build_stats

    for _ in range(args.warmup):
        q, rep, info, bst = step()
    torch.cuda.synchronize()
    nnz = info["nnz"]
    if dist_mode:   # global nonzeros = sum of the ranks' blocks
        t = torch.tensor([float(nnz)], dtype=torch.float64, device="cuda")
        dist.all_reduce(t)
        nnz = int(t[0])
    kb = k if rep["batch_k"] else 1
    B = canonical_bytes(n, nnz, wb, kb)      # one PCG iteration (batched over kb columns)

    sampler = ClockSampler(local)
    launches0, cub0 = binding.kernel_launches()
    if dist_mode:
        dist.barrier()
    torch.cuda.synchronize()
    t_wall = time.perf_counter()
    step_ms, loop_ms, iters, ttq_ms, results = [], 0.0, 0, [], []
    for _ in range(args.steps):
        flush.fill_(1)                                   # L2 flush (512 MiB write), outside the events
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        q, rep, info, bst = step()
        e1.record(stream)
        e1.synchronize()
        step_ms.append(e0.elapsed_time(e1))
        loop_ms += rep["ms_loop"]
        # batched (row a9): B(k) per batch iteration; per-column solves: B(1) per column iteration
        iters += rep["iterations"] if rep["batch_k"] else rep["iterations_total"]
        batched = bool(rep["batch_k"])
        ttq_ms.append(rep["ms"])
        results.append((q, rep))
    torch.cuda.synchronize()
    if dist_mode:
        dist.barrier()
    wall = time.perf_counter() - t_wall
    launches1, cub1 = binding.kernel_launches()
    clocks = sampler.stop()

    # dominant kernel: the PCG's (I+L)p product exactly as the solve loop launches it (k columns,
    # solver buffers), timed live inside the library with CUDA events on the launching stream
    spmv_ms, prod_path = None, "engine"
    if not dist_mode:
        G = fj.Graph.from_edges(n, u, v, w, order=order)
        G.approxim(S, opts=opts)          # fills the solver buffers with a real search direction
        flush.fill_(1)
        spmv_ms = G.time_spmv(k=kb, reps=args.spmv_reps)
        prod_path = G.product_path(kb)
        G.close()

    # aggregate over ranks: time = max over ranks, bytes = sum over ranks
    tot_loop_ms = loop_ms
    tot_bytes = B * iters
    max_step_ms = sum(step_ms)
    if dist_mode:   # B is already the GLOBAL per-iteration traffic (all ranks iterate together)
        t = torch.tensor([loop_ms, sum(step_ms)], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        tot_loop_ms, max_step_ms = float(t[0]), float(t[1])
    value = tot_bytes / (tot_loop_ms / 1e3) / 1e9

    peak, peak_src = load_peaks()
    Bs = spmv_bytes(n, nnz, wb, kb)
    if dist_mode:   # fj_apply is not available on a distributed handle: per-rank whole iteration
        t_iter_ms = tot_loop_ms / max(iters, 1)
        Bs = B / ws
        achieved = Bs / (t_iter_ms / 1e3) / 1e9
        spmv_ms = t_iter_ms
    else:
        achieved = Bs / (spmv_ms / 1e3) / 1e9
    # the SpMV's real bound: random gathers (one L2 sector request per nonzero), measured live by
    # fj_probe_gather on the same vector size, index count and gather width
    gather_roof = None
    if not dist_mode and not args.no_extras:
        width = 1 if kb == 1 else (2 if kb == 2 else 4)
        probe = binding.probe_gather(n, nnz, width=width, reps=5)
        ach = nnz / (spmv_ms / 1e3)
        gather_roof = {"achieved_gathers_per_s": ach, "peak_gathers_per_s": probe, "frac": ach / probe,
                       "width_doubles": width,
                       "note": "peak = fj_probe_gather: nnz uniform random int32 indices streamed once, one "
                               f"{8 * width}-byte gather each from an n-row vector, no row logic; achieved = "
                               "nnz / SpMV launch time"}
    # ncu DRAM bytes of one launch of this product, only if captured for this exact config, k,
    # vertex order and CUDA build (profiles/ncu_traffic.json, tools/record_traffic.py)
    from paper_2101_08143_b200 import build as FB
    traffic, traffic_key = None, f"{args.config}/k{kb}/{order}/{FB.source_hash()}"
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp) and not dist_mode:
        traffic = json.load(open(tp)).get(traffic_key, {}).get("spmv_dram_bytes_per_launch")

    # C3 also as separate k = 1 solves, one per opinion distribution (outside the
    # timed region; same graph build, each column's own solve + quantities pass)
    per_dist = None
    if not dist_mode and k > 1 and k <= 4 and not args.no_extras:
        G = fj.Graph.from_edges(n, u, v, w, order=order)
        per_dist = []
        for c in range(k):
            sc = S[:, c].contiguous()
            G.approxim(sc, opts=opts)
            reps1 = []
            for _ in range(3):
                flush.fill_(1)
                _, q1, r1 = G.approxim(sc, opts=opts)
                reps1.append(r1)
            r1 = min(reps1, key=lambda r: r["ms"])
            B1 = canonical_bytes(n, nnz, wb, 1)
            per_dist.append({"opinions": wl.kinds[c], "iterations": r1["iterations"],
                             "cg_gbs": B1 * r1["iterations_total"] / (r1["ms_loop"] / 1e3) / 1e9,
                             "time_to_quantities_ms": r1["ms"], "rel_res_true": r1["rel_res_true"],
                             "D": q1[0]["D"]})
        G.close()

    line = {
        "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": max_step_ms / args.steps, "higher_is_better": True,
        "scaling": "strong" if dist_mode else "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{wl.name}: {wl.desc}", "n": n, "nnz": nnz, "k": k, "rtol": args.rtol,
                   "opinions": wl.kinds, "vertex_order": order,
                   "parallelism": f"row-partition x{ws} (NCCL halo + allreduce)" if dist_mode else "1 GPU",
                   "l2": "flushed between steps (512 MiB write, outside the timed events)",
                   "pcg_iterations_per_step": iters / args.steps,
                   "bytes_per_iteration": B, "fraction_of_measured_hbm": value / peak},
        "time_to_quantities_ms": statistics.median(ttq_ms),
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": None if dist_mode else traffic, "traffic_key": traffic_key,
                     "kernel": ("whole distributed PCG iteration per rank (B(k)/N per iteration time)" if dist_mode
                                else spmv_kernel_name(kb, prod_path)),
                     "algorithmic_bytes_per_launch": Bs, "launch_ms": spmv_ms, "peak_source": peak_src},
        "gather_roofline": gather_roof,
        "per_distribution_k1": per_dist, "build": FB.source_hash(),
        "clocks": clocks, "gpu_launches": launches1 - launches0,
        "cub_calls": cub1 - cub0, "wall_s_timed_region": wall,
        "quantities_step0": {kk: results[0][0][0][kk] for kk in ["CI", "D", "P", "C", "Idc", "PDI"]},
        "max_rel_res_true": max(r[1]["rel_res_true"] for r in results),
    }

    # e2e: the public host-buffer call; H2D of the inputs and D2H of z + quantities inside the timing
    if not args.no_e2e and dist_mode:
        # distributed e2e: every step copies the raw edge list and this rank's opinion slice from
        # pinned host memory, runs the row-partitioned path and reads z + quantities back
        uh, vh = torch.from_numpy(wl.u).pin_memory(), torch.from_numpy(wl.v).pin_memory()
        wh = None if wl.w is None else torch.from_numpy(wl.w).pin_memory()
        b = info["bounds"]
        Sh = torch.from_numpy(np.ascontiguousarray(wl.S)).pin_memory()   # every rank slices on the device
        h2d = uh.nbytes + vh.nbytes + (0 if wh is None else wh.nbytes) + Sh.nbytes
        d2h = 8 * k * (b[rank + 1] - b[rank]) + k * 200
        e_ms, e_iters, reps = 0.0, 0, max(1, min(args.steps, 3))
        for _ in range(reps):
            torch.cuda.synchronize()
            dist.barrier()
            t = time.perf_counter()
            ud, vd = uh.cuda(non_blocking=True), vh.cuda(non_blocking=True)
            wd = None if wh is None else wh.cuda(non_blocking=True)
            Sd = Sh.cuda(non_blocking=True)
            G, _ = FD.build_dist_graph(comm, rank, n, ud, vd, wd, grp, order=order)
            zd, qh, reph = G.approxim(FD.slice_in(G, Sd, b), opts=opts)
            zh = zd.cpu()
            G.close()
            e_ms += (time.perf_counter() - t) * 1e3
            e_iters += reph["iterations_total"]
        t = torch.tensor([e_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e_ms = float(t[0])
        line["e2e"] = {"value": B * e_iters / (e_ms / 1e3) / 1e9, "unit": "GB/s", "h2d_bytes_per_step": h2d,
                       "d2h_bytes_per_step": d2h, "ms_per_step": e_ms / reps,
                       "note": "per rank: pinned H2D of the raw edges + opinions, (relabelling,) partition, "
                               "row-block CSR, halo plan, distributed Algorithm 1, D2H of the rank's z; host wall "
                               "clock, max over ranks"}
    if not args.no_e2e and not dist_mode:
        uh = torch.from_numpy(wl.u).pin_memory().numpy()
        vh = torch.from_numpy(wl.v).pin_memory().numpy()
        wh = None if wl.w is None else torch.from_numpy(wl.w).pin_memory().numpy()
        Sh = torch.from_numpy(wl.S).pin_memory().numpy()
        h2d = uh.nbytes + vh.nbytes + (0 if wh is None else wh.nbytes) + Sh.nbytes
        d2h = Sh.nbytes + k * 200
        zbuf = torch.empty(Sh.shape, dtype=torch.float64, pin_memory=True).numpy()   # caller's output
        for _ in range(2):                                                             # warm
            fj.approxim_host(n, uh, vh, wh, Sh, opts=opts, z_out=zbuf)
        e_loop, e_iters, e_ms = 0.0, 0, 0.0
        reps = max(1, min(args.steps, 3))
        for _ in range(reps):
            flush.fill_(1)
            torch.cuda.synchronize()
            t = time.perf_counter()
            zh, qh, reph = fj.approxim_host(n, uh, vh, wh, Sh, opts=opts, z_out=zbuf)
            e_ms += (time.perf_counter() - t) * 1e3
            e_iters += reph["iterations"] if reph["batch_k"] else reph["iterations_total"]
        e_bytes = B * e_iters
        if ws > 1:
            t = torch.tensor([e_ms], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            tb = torch.tensor([float(e_bytes)], dtype=torch.float64, device="cuda")
            dist.all_reduce(tb, op=dist.ReduceOp.SUM)
            e_ms, e_bytes = float(t[0]), float(tb[0])
        line["e2e"] = {"value": e_bytes / (e_ms / 1e3) / 1e9, "unit": "GB/s", "h2d_bytes_per_step": h2d,
                       "d2h_bytes_per_step": d2h, "ms_per_step": e_ms / reps,
                       "note": "fj_approxim_host from pinned host buffers: H2D edges (opinions on a side stream, "
                               "overlapping the CSR build), CSR build, graph, Algorithm 1, D2H z into the "
                               "caller's pinned buffer; host wall clock"}

    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        import oracle as O
        big = wl.name in ("c4", "c5")
        g = O.canonical_csr_big(wl.n, wl.u, wl.v, wl.w) if big else O.canonical_csr(wl.n, wl.u, wl.v, wl.w)
        line["cpu_baseline"] = cpu_baseline(wl, g, args.rtol)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist_mode:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())

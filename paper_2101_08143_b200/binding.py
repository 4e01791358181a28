"""ctypes binding of include/fj.h.  Marshalling only (pointers, sizes, streams, result structs)."""
from __future__ import annotations

import ctypes
import math
import os

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.environ.get("FJ_LIBRARY") or os.path.join(HERE, "libfj.so")   # FJ_LIBRARY: A/B builds (tools/)

FJ_W_UNIT, FJ_W_U8, FJ_W_F32, FJ_W_F64 = 0, 1, 2, 3
FJ_OP_L, FJ_OP_IPL = 0, 1
FJ_E_NO_CONVERGENCE = 6

_i64, _i32, _dbl, _vp = ctypes.c_int64, ctypes.c_int32, ctypes.c_double, ctypes.c_void_p


class GraphInfo(ctypes.Structure):
    _fields_ = [("n", _i64), ("nnz", _i64), ("m", _i64), ("n_isolated", _i64), ("deg_max", _i64),
                ("w_min", _dbl), ("w_max", _dbl), ("d_max", _dbl), ("n_tiles", _i64), ("n_wrows", _i64),
                ("n_long_rows", _i64), ("n_long_chunks", _i64), ("wtype", _i32), ("reserved", _i32)]


class SolveOpts(ctypes.Structure):
    _fields_ = [("rtol", _dbl), ("eps_target", _dbl), ("max_iter", _i32), ("max_restarts", _i32),
                ("use_cuda_graph", _i32), ("vertex_order", _i32)]

    @classmethod
    def make(cls, rtol=1e-10, eps_target=0.0, max_iter=10000, max_restarts=3, use_cuda_graph=True,
             vertex_order="natural"):
        """vertex_order ("natural" | "degree" | "auto"): fj_approxim_host's a1 relabelling (fj.h FJ_ORDER_*)."""
        vo = {"natural": 0, "degree": 1, "auto": 2}[vertex_order] if isinstance(vertex_order, str) else int(vertex_order)
        return cls(rtol, eps_target, max_iter, max_restarts, 1 if use_cuda_graph else 0, vo)


class SolveReport(ctypes.Structure):
    _fields_ = [("iterations", _i32), ("converged", _i32), ("restarts", _i32), ("batch_k", _i32),
                ("rel_res_recursive", _dbl), ("rel_res_true", _dbl), ("ms", _dbl), ("ms_loop", _dbl),
                ("iterations_total", _i64)]

    def to_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_ if f != "reserved"}


class Quantities(ctypes.Structure):
    _fields_ = [("CI", _dbl), ("D", _dbl), ("P", _dbl), ("C", _dbl), ("Idc", _dbl), ("PDI", _dbl),
                ("mean_s", _dbl), ("ss", _dbl), ("sz", _dbl), ("sbzb", _dbl), ("Lz2", _dbl),
                ("res_norm", _dbl), ("s_norm", _dbl), ("fp_bound", _dbl), ("eps", _dbl * 6),
                ("consensus", _i32), ("certified", _i32)]

    def to_dict(self):
        d = {f: getattr(self, f) for f, _ in self._fields_ if f != "eps"}
        d["eps"] = dict(zip(["CI", "D", "P", "C", "Idc", "PDI"], list(self.eps)))
        return d


class Alg1Result(ctypes.Structure):
    _fields_ = [("CI", _dbl), ("D", _dbl), ("P", _dbl), ("C", _dbl), ("Idc", _dbl), ("PDI", _dbl),
                ("delta", _dbl), ("delta_eff", _dbl), ("rtol", _dbl), ("D_from_z", _dbl), ("CI_def", _dbl),
                ("mean_s", _dbl), ("sbar_norm", _dbl), ("clamped", _i32), ("rtol_floored", _i32)]

    def to_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class FJError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_lib.fj_status_str(status).decode()}: {msg}")
        self.status = status


_lib = None


def load_library(path: str = SO):
    """Load libfj.so.  Raises (never falls back) if the CUDA extension has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} is missing: build it with `python __graft_entry__.py build` "
                          "(the CUDA extension is required; there is no CPU fallback)")
    L = ctypes.CDLL(path)
    P = ctypes.POINTER
    L.fj_abi_version.restype = ctypes.c_int
    L.fj_kernel_launches.restype = _i64
    L.fj_kernel_launches.argtypes = [P(_i64)]
    L.fj_status_str.restype = ctypes.c_char_p
    L.fj_status_str.argtypes = [ctypes.c_int]
    L.fj_last_error.restype = ctypes.c_char_p
    L.fj_default_solve_opts.argtypes = [P(SolveOpts)]
    L.fj_default_solve_opts.restype = None
    L.fj_csr_from_edges.argtypes = [_i64, _i64, _vp, _vp, _vp, ctypes.c_int, _vp, _vp, _vp, P(_i64), P(_i64),
                                    P(_i64), _vp]
    relabel_sigs = {   # DESIGN.md §6.7 (looked up leniently so older A/B builds still load)
        "fj_permute_rows": [_i64, ctypes.c_int, _vp, _vp, _vp, _vp],
        "fj_csr_degree_order": [_i64, _vp, _vp, _vp, _vp],
        "fj_csr_permute": [_i64, _i64, _vp, _vp, _vp, ctypes.c_int, _vp, _vp, _vp, _vp, _vp, _vp],
    }
    for name, sig in relabel_sigs.items():
        if hasattr(L, name):
            getattr(L, name).argtypes = sig
    L.fj_set_allocator.argtypes = [_ALLOC_FN, _FREE_FN, _vp]
    L.fj_allocator_live_blocks.restype = _i64
    L.fj_graph_create.argtypes = [_i64, _i64, _vp, _vp, _vp, ctypes.c_int, ctypes.c_int, _vp, P(_vp)]
    L.fj_graph_info.argtypes = [_vp, P(GraphInfo)]
    L.fj_graph_degrees.argtypes = [_vp, _vp, _vp]
    L.fj_graph_destroy.argtypes = [_vp]
    L.fj_apply.argtypes = [_vp, ctypes.c_int, ctypes.c_int, _vp, _vp, _vp]
    L.fj_time_spmv.argtypes = [_vp, ctypes.c_int, ctypes.c_int, P(ctypes.c_float), _vp]
    L.fj_product_path.argtypes = [_vp, ctypes.c_int, P(ctypes.c_int), _vp]
    L.fj_probe_gather.argtypes = [_i64, _i64, ctypes.c_int, ctypes.c_int, P(ctypes.c_double), _vp]
    L.fj_alg1_delta.argtypes = [_i64, _dbl, _dbl, _dbl, _dbl, _dbl, P(_dbl), P(_dbl), P(_dbl),
                                P(ctypes.c_int), P(ctypes.c_int)]
    L.fj_approxim_alg1.argtypes = [_vp, _vp, _dbl, P(SolveOpts), P(Alg1Result), P(SolveReport), _vp]
    L.fj_forest_columns.argtypes = [_vp, _i64, _vp, _vp, P(SolveOpts), P(SolveReport), _vp]
    L.fj_opinions_generate.argtypes = [_i64, ctypes.c_int, ctypes.c_uint64, _vp, _vp]
    L.fj_exact_dense.argtypes = [_vp, ctypes.c_int, _vp, _vp, _vp, _vp]
    L.fj_connected_components.argtypes = [_i64, _i64, _vp, _vp, _vp, P(_i64), _vp]
    L.fj_lcc.argtypes = [_i64, _i64, _vp, _vp, _vp, ctypes.c_int, _vp, _vp, _vp, _vp, P(_i64), P(_i64), _vp]
    L.fj_opinion_stats.argtypes = [_vp, ctypes.c_int, _vp, _vp, _vp]
    L.fj_solve.argtypes = [_vp, ctypes.c_int, _vp, _vp, P(SolveOpts), P(SolveReport), _vp]
    L.fj_quantities.argtypes = [_vp, ctypes.c_int, _vp, _vp, P(Quantities), _vp]
    L.fj_approxim.argtypes = [_vp, ctypes.c_int, _vp, _vp, P(SolveOpts), P(Quantities), P(SolveReport), _vp]
    L.fj_approxim_host.argtypes = [_i64, _i64, _vp, _vp, _vp, ctypes.c_int, ctypes.c_int, _vp, _vp,
                                   P(SolveOpts), P(Quantities), P(SolveReport), _vp]
    L.fj_comm_unique_id.argtypes = [_vp]
    L.fj_comm_init.argtypes = [ctypes.c_int, ctypes.c_int, _vp, P(_vp)]
    L.fj_comm_init_loopback.argtypes = [ctypes.c_int, P(_vp)]
    L.fj_comm_destroy.argtypes = [_vp]
    L.fj_partition_rows.argtypes = [_i64, _i64, _vp, _vp, ctypes.c_int, _vp, _vp]
    L.fj_csr_rows_from_edges.argtypes = [_i64, _i64, _vp, _vp, _vp, ctypes.c_int, _i64, _i64, _vp, _vp, _vp,
                                         P(_i64), _vp]
    L.fj_dist_ghosts.argtypes = [_i64, _vp, _i64, _i64, _vp, P(_i64), _vp]
    L.fj_edge_degree_order.argtypes = [_i64, _i64, _vp, _vp, _vp, _vp, _vp]
    L.fj_partition_rows_relabelled.argtypes = [_i64, _i64, _vp, _vp, _vp, ctypes.c_int, _vp, _vp]
    L.fj_csr_rows_from_edges_relabelled.argtypes = [_i64, _i64, _vp, _vp, _vp, _vp, ctypes.c_int, _i64, _i64, _vp,
                                                    _vp, _vp, P(_i64), _vp]
    L.fj_graph_create_dist.argtypes = [_vp, ctypes.c_int, _i64, _vp, _i64, _vp, _vp, _vp, ctypes.c_int, _i64, _vp,
                                       _vp, _vp, _vp, P(_vp)]
    for name in ["fj_csr_from_edges", "fj_graph_create", "fj_graph_info", "fj_graph_degrees", "fj_graph_destroy",
                 "fj_apply", "fj_time_spmv", "fj_product_path", "fj_probe_gather",
                 "fj_alg1_delta", "fj_approxim_alg1", "fj_forest_columns", "fj_opinions_generate",
                 "fj_connected_components", "fj_lcc", "fj_exact_dense", "fj_opinion_stats", "fj_solve", "fj_quantities", "fj_approxim", "fj_approxim_host",
                 "fj_comm_unique_id", "fj_comm_init", "fj_comm_init_loopback", "fj_comm_destroy",
                 "fj_partition_rows", "fj_csr_rows_from_edges", "fj_dist_ghosts", "fj_graph_create_dist",
                 "fj_edge_degree_order", "fj_partition_rows_relabelled", "fj_csr_rows_from_edges_relabelled"]:
        getattr(L, name).restype = ctypes.c_int
    _lib = L
    return L


def lib():
    return load_library()


def kernel_launches():
    """(own kernels launched, CUB library calls) so far in this process."""
    c = _i64()
    n = lib().fj_kernel_launches(ctypes.byref(c))
    return int(n), int(c.value)


def probe_gather(n_vec: int, m: int, width: int = 1, reps: int = 10, stream=None) -> float:
    """Random-gather rate (indices / s) of fj_probe_gather: the SpMV's measured gather bound."""
    r = ctypes.c_double()
    _check(lib().fj_probe_gather(int(n_vec), int(m), int(width), int(reps), ctypes.byref(r), _stream(stream)))
    return float(r.value)


OPINION_KINDS = {"uniform": 0, "exponential": 1, "powerlaw": 2}


def opinions_generate(n: int, kind: str, seed: int, device=None, stream=None):
    """Row f1: an opinion vector drawn on the device (fj_opinions_generate) -> fp64 CUDA tensor [n]."""
    import torch
    s = torch.empty(n, dtype=torch.float64, device=device or "cuda")
    _check(lib().fj_opinions_generate(int(n), OPINION_KINDS[kind], int(seed), _ptr(s), _stream(stream)))
    return s


def connected_components(n: int, u, v, stream=None):
    """Row f1: (labels int32 CUDA tensor [n] = smallest vertex id of the component, count)."""
    import torch
    _need_cuda(u, v)
    lab = torch.empty(n, dtype=torch.int32, device=u.device)
    nc = _i64()
    _check(lib().fj_connected_components(int(n), u.numel(), _ptr(u), _ptr(v), _ptr(lab), ctypes.byref(nc),
                                         _stream(stream)))
    return lab, int(nc.value)


def lcc(n: int, u, v, w=None, stream=None):
    """Row f1: largest connected component -> (vmap [n], u', v', w' or None, n_lcc); edges in input order."""
    import torch
    _need_cuda(u, v)
    m = u.numel()
    vmap = torch.empty(n, dtype=torch.int32, device=u.device)
    u2 = torch.empty(max(m, 1), dtype=torch.int32, device=u.device)
    v2 = torch.empty(max(m, 1), dtype=torch.int32, device=u.device)
    w2 = None if w is None else torch.empty(max(m, 1), dtype=w.dtype, device=u.device)
    nl, ml = _i64(), _i64()
    _check(lib().fj_lcc(int(n), m, _ptr(u), _ptr(v), None if w is None else _ptr(w), _wtype(w), _ptr(vmap),
                        _ptr(u2), _ptr(v2), None if w2 is None else _ptr(w2), ctypes.byref(nl), ctypes.byref(ml),
                        _stream(stream)))
    k = int(ml.value)
    return vmap, u2[:k], v2[:k], (None if w2 is None else w2[:k]), int(nl.value)


def alg1_delta(n, w_min, w_max, d_max, sbar_norm, eps):
    """Host arithmetic of Algorithm 1 line 1 + clamp + residual map (fj_alg1_delta; no device work)."""
    d, de, rt = _dbl(), _dbl(), _dbl()
    cl, fl = ctypes.c_int(), ctypes.c_int()
    _check(lib().fj_alg1_delta(int(n), float(w_min), float(w_max), float(d_max), float(sbar_norm), float(eps),
                               ctypes.byref(d), ctypes.byref(de), ctypes.byref(rt), ctypes.byref(cl),
                               ctypes.byref(fl)))
    return d.value, de.value, rt.value, bool(cl.value), bool(fl.value)


def _check(st: int, allow=()):
    if st != 0 and st not in allow:
        raise FJError(st, _lib.fj_last_error().decode(errors="replace"))
    return st


def _stream(stream=None):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _on(stream=None):
    """Allocate temporaries on the stream the library works on: torch's caching allocator then
    reuses their memory only after that stream's pending work (a temporary allocated on
    the current stream and freed on return could be handed out while `stream` still reads it)."""
    import contextlib
    import torch
    return contextlib.nullcontext() if stream is None else torch.cuda.stream(stream)


def _check_out(z, like, what="z"):
    """A caller-supplied output must be a contiguous CUDA tensor shaped and typed like `like`."""
    _need_cuda(z)
    if z.shape != like.shape or z.dtype != like.dtype or z.device != like.device:
        raise ValueError(f"{what} must match s in shape, dtype and device")


def _wtype(w):
    if w is None:
        return FJ_W_UNIT
    import torch
    return {torch.uint8: FJ_W_U8, torch.float32: FJ_W_F32, torch.float64: FJ_W_F64}[w.dtype]


_ALLOC_FN = ctypes.CFUNCTYPE(_vp, ctypes.c_size_t, _vp, _vp)
_FREE_FN = ctypes.CFUNCTYPE(None, _vp, ctypes.c_size_t, _vp, _vp)
_torch_alloc_cbs = None   # keep the ctypes callbacks alive while installed


def use_torch_allocator(enable: bool = True):
    """fj_set_allocator: route the library's device workspace through torch's caching allocator
    (torch.cuda.caching_allocator_alloc / _delete, on the stream the library names), or back to the
    library's own pool (enable=False)."""
    import torch
    global _torch_alloc_cbs
    L = lib()
    if not enable:
        _check(L.fj_set_allocator(ctypes.cast(None, _ALLOC_FN), ctypes.cast(None, _FREE_FN), None))
        _torch_alloc_cbs = None
        return

    def _alloc(nbytes, stream, ctx):
        try:
            return torch.cuda.caching_allocator_alloc(int(nbytes), torch.cuda.current_device(), stream=int(stream or 0))
        except Exception as e:   # OOM -> NULL -> the library reports an allocation failure
            import sys
            print(f"fj torch allocator: {e!r}", file=sys.stderr)
            return None

    def _free(ptr, nbytes, stream, ctx):
        torch.cuda.caching_allocator_delete(int(ptr))

    cbs = (_ALLOC_FN(_alloc), _FREE_FN(_free))
    _check(L.fj_set_allocator(cbs[0], cbs[1], None))
    _torch_alloc_cbs = cbs


def allocator_live_blocks() -> int:
    return int(lib().fj_allocator_live_blocks())


def _need_cuda(*ts):
    for t in ts:
        if t is not None and not t.is_cuda:
            raise ValueError("device tensors required (torch CUDA tensors)")
        if t is not None and not t.is_contiguous():
            raise ValueError("contiguous tensors required")


def relabel_pays(n: int, k: int) -> bool:
    """FJ_ORDER_AUTO's rule: relabel only for rows narrower than a 32-byte L2 sector
    (k <= 2) whose gathered [n][k] vector exceeds the L2."""
    import torch
    l2 = getattr(torch.cuda.get_device_properties(torch.cuda.current_device()), "L2_cache_size", 126 << 20)
    return k <= 2 and n * 8 * k > l2


def csr_degree_order(n: int, row_ptr, stream=None):
    """fj_csr_degree_order: (new2old, old2new) by descending row length of a built CSR."""
    import torch
    _need_cuda(row_ptr)
    new2old = torch.empty(n, dtype=torch.int32, device=row_ptr.device)
    old2new = torch.empty(n, dtype=torch.int32, device=row_ptr.device)
    _check(lib().fj_csr_degree_order(n, _ptr(row_ptr), _ptr(new2old), _ptr(old2new), _stream(stream)))
    return new2old, old2new


def csr_permute(n: int, row_ptr, col, w, new2old, old2new, stream=None):
    """fj_csr_permute: (row_ptr, col, w) of P A P^T (columns in their source order)."""
    import torch
    _need_cuda(row_ptr, col, w, new2old, old2new)
    rp2 = torch.empty_like(row_ptr)
    col2 = torch.empty_like(col)
    w2 = None if w is None else torch.empty_like(w)
    _check(lib().fj_csr_permute(n, int(col.numel()), _ptr(row_ptr), _ptr(col), _ptr(w), _wtype(w), _ptr(new2old),
                                _ptr(old2new), _ptr(rp2), _ptr(col2), _ptr(w2), _stream(stream)))
    return rp2, col2, w2


def permute_rows(x, idx, stream=None):
    """fj_permute_rows: out[i] = x[idx[i]] for a [n] or [n][k] fp64 device tensor."""
    import torch
    _need_cuda(x, idx)
    n = int(idx.numel())
    k = _cols(x, n)
    out = torch.empty_like(x)
    _check(lib().fj_permute_rows(n, k, _ptr(idx), _ptr(x), _ptr(out), _stream(stream)))
    return out


def csr_from_edges(n: int, u, v, w=None, stream=None):
    """Row a1: canonical CSR (device) from a raw device edge list.  Returns
    (row_ptr int64 [n+1], col int32 [nnz], w_out or None, stats dict)."""
    import torch
    L = lib()
    _need_cuda(u, v, w)
    m = int(u.numel())
    dev = u.device
    row_ptr = torch.empty(n + 1, dtype=torch.int64, device=dev)
    col = torch.empty(max(2 * m, 1), dtype=torch.int32, device=dev)
    w_out = None if w is None else torch.empty(max(2 * m, 1), dtype=w.dtype, device=dev)
    nnz, loops, dups = _i64(), _i64(), _i64()
    _check(L.fj_csr_from_edges(n, m, _ptr(u), _ptr(v), _ptr(w), _wtype(w), _ptr(row_ptr), _ptr(col),
                               _ptr(w_out), ctypes.byref(nnz), ctypes.byref(loops), ctypes.byref(dups),
                               _stream(stream)))
    k = nnz.value
    col = col[:k]
    if w_out is not None:
        w_out = w_out[:k]
    return row_ptr, col, w_out, {"nnz": k, "selfloops": loops.value, "duplicates": dups.value}


def _cols(t, n):
    if t.dim() == 1:
        if t.numel() != n:
            raise ValueError("length mismatch")
        return 1
    if t.dim() != 2 or t.shape[0] != n:
        raise ValueError("expected [n] or [n][k]")
    return int(t.shape[1])


class Graph:
    """Handle over a borrowed device CSR (rows a2..a7).  Keeps references to the CSR tensors.
    A graph built with from_edges(..., order="degree") holds the relabelled CSR
    and maps every vertex-indexed argument in (fj_permute_rows with new2old) and every
    vertex-indexed result back (old2new): callers always see the input labels."""

    new2old = None   # class defaults: subclasses (DistGraph) build their handles without __init__
    old2new = None

    def __init__(self, n: int, row_ptr, col, w=None, validate: bool = True, stream=None):
        L = lib()
        _need_cuda(row_ptr, col, w)
        self.n = int(n)
        self.new2old = self.old2new = None
        self._keep = (row_ptr, col, w)
        h = _vp()
        _check(L.fj_graph_create(self.n, int(col.numel()), _ptr(row_ptr), _ptr(col), _ptr(w), _wtype(w),
                                 1 if validate else 0, _stream(stream), ctypes.byref(h)))
        self._h = h

    @classmethod
    def from_edges(cls, n, u, v, w=None, validate=False, stream=None, order: str = "natural"):
        """a1 + a2 from a raw device edge list; order="degree" relabels the built CSR by descending
        degree (fj_csr_degree_order + fj_csr_permute)."""
        if order not in ("natural", "degree"):
            raise ValueError("order must be 'natural' or 'degree'")
        n2o = o2n = None
        rp, col, wo, stats = csr_from_edges(n, u, v, w, stream)
        if order == "degree":
            n2o, o2n = csr_degree_order(n, rp, stream)
            rp, col, wo = csr_permute(n, rp, col, wo, n2o, o2n, stream)
            validate = False   # columns are in source order, not ascending in the new labels
        g = cls(n, rp, col, wo, validate=validate, stream=stream)
        g.new2old, g.old2new = n2o, o2n
        g.build_stats = stats
        return g

    def _in(self, x, stream=None):      # input labels -> the handle's labels
        return x if self.new2old is None else permute_rows(x, self.new2old, stream)

    def _out(self, x, stream=None, out=None):   # the handle's labels -> input labels (into `out` if given)
        if self.old2new is None:
            return x
        if out is None:
            return permute_rows(x, self.old2new, stream)
        _need_cuda(out)
        if out.shape != x.shape or out.dtype != x.dtype:
            raise ValueError("z must match s in shape and dtype")
        _check(lib().fj_permute_rows(self.n, _cols(x, self.n), _ptr(self.old2new), _ptr(x), _ptr(out),
                                     _stream(stream)))
        return out

    @property
    def handle(self):
        if self._h is None:
            raise RuntimeError("graph destroyed")
        return self._h

    def info(self) -> dict:
        gi = GraphInfo()
        _check(lib().fj_graph_info(self.handle, ctypes.byref(gi)))
        return {f: getattr(gi, f) for f, _ in gi._fields_ if f != "reserved"}

    def degrees(self, stream=None):
        import torch
        with _on(stream):
            d = torch.empty(self.n, dtype=torch.float64, device=self._keep[0].device)
            _check(lib().fj_graph_degrees(self.handle, _ptr(d), _stream(stream)))
            return self._out(d, stream)

    def apply(self, x, op: int = FJ_OP_IPL, stream=None):
        import torch
        _need_cuda(x)
        k = _cols(x, self.n)
        with _on(stream):
            xi = self._in(x, stream)
            y = torch.empty_like(x)
            _check(lib().fj_apply(self.handle, op, k, _ptr(xi), _ptr(y), _stream(stream)))
            return self._out(y, stream)

    def time_spmv(self, k: int = 1, reps: int = 20, stream=None) -> float:
        """ms per launch of the k-column PCG product q = (I+L)p (fj_time_spmv; CUDA events)."""
        ms = ctypes.c_float()
        _check(lib().fj_time_spmv(self.handle, int(k), int(reps), ctypes.byref(ms), _stream(stream)))
        return float(ms.value)

    def product_path(self, k: int = 1, stream=None) -> str:
        """Kernel path of the k-column PCG product (fj_product_path): engine / rows / rows_slabs / batch."""
        v = ctypes.c_int()
        _check(lib().fj_product_path(self.handle, int(k), ctypes.byref(v), _stream(stream)))
        return ["engine", "rows", "rows_slabs", "batch"][v.value]

    def opinion_stats(self, s, stream=None):
        import numpy as np
        _need_cuda(s)
        k = _cols(s, self.n)
        out = np.zeros(4 * k)
        _check(lib().fj_opinion_stats(self.handle, k, _ptr(s), ctypes.c_void_p(out.ctypes.data), _stream(stream)))
        return out.reshape(k, 4)

    def solve(self, s, opts: SolveOpts | None = None, z=None, stream=None, allow_no_convergence=False):
        with _on(stream):
            return self._solve(s, opts, z, stream, allow_no_convergence)

    def _solve(self, s, opts, z, stream, allow_no_convergence):
        import torch
        _need_cuda(s)
        k = _cols(s, self.n)
        if z is not None:
            _check_out(z, s)
        z_user = z
        si = self._in(s, stream)
        if self.new2old is not None:   # solve in the handle's labels; z_user receives the input labels
            z = torch.empty_like(s)
        else:
            z = torch.empty_like(s) if z is None else z
        rep = SolveReport()
        o = opts or SolveOpts.make()
        _check(lib().fj_solve(self.handle, k, _ptr(si), _ptr(z), ctypes.byref(o), ctypes.byref(rep), _stream(stream)),
               allow=(FJ_E_NO_CONVERGENCE,) if allow_no_convergence else ())
        return self._out(z, stream, out=z_user), rep.to_dict()

    def quantities(self, s, z, stream=None):
        _need_cuda(s, z)
        _check_out(z, s)
        k = _cols(s, self.n)
        q = (Quantities * k)()
        with _on(stream):
            si, zi = self._in(s, stream), self._in(z, stream)
            _check(lib().fj_quantities(self.handle, k, _ptr(si), _ptr(zi), q, _stream(stream)))
        return [x.to_dict() for x in q]

    def approxim(self, s, opts: SolveOpts | None = None, z=None, stream=None):
        """Algorithm 1 (single-solve form): returns (z, [quantities per column], report)."""
        with _on(stream):
            return self._approxim(s, opts, z, stream)

    def _approxim(self, s, opts, z, stream):
        import torch
        _need_cuda(s)
        k = _cols(s, self.n)
        if z is not None:
            _check_out(z, s)
        z_user = z
        z = torch.empty_like(s) if (z is None or self.new2old is not None) else z
        q = (Quantities * k)()
        rep = SolveReport()
        o = opts or SolveOpts.make()
        si = self._in(s, stream)
        _check(lib().fj_approxim(self.handle, k, _ptr(si), _ptr(z), ctypes.byref(o), q, ctypes.byref(rep),
                                 _stream(stream)))
        return self._out(z, stream, out=z_user), [x.to_dict() for x in q], rep.to_dict()

    def approxim_alg1(self, s, eps: float = 1e-6, opts: SolveOpts | None = None, stream=None):
        """Algorithm 1 verbatim (row f2): both solves, lines 5-9 norms.  Returns (dict, report)."""
        _need_cuda(s)
        if _cols(s, self.n) != 1:
            raise ValueError("approxim_alg1 takes one opinion vector")
        r = Alg1Result()
        rep = SolveReport()
        o = opts or SolveOpts.make()
        with _on(stream):
            s = self._in(s, stream)
            _check(lib().fj_approxim_alg1(self.handle, _ptr(s), float(eps), ctypes.byref(o), ctypes.byref(r),
                                          ctypes.byref(rep), _stream(stream)))
        return r.to_dict(), rep.to_dict()

    def exact_dense(self, s, stream=None):
        """Row f3: the paper's Exact (dense Cholesky of I+L on the device) -> (z, [quantities])."""
        import torch
        _need_cuda(s)
        k = _cols(s, self.n)
        q = (Quantities * k)()
        with _on(stream):
            z = torch.empty_like(s)
            si = self._in(s, stream)
            _check(lib().fj_exact_dense(self.handle, k, _ptr(si), _ptr(z), q, _stream(stream)))
            return self._out(z, stream), [x.to_dict() for x in q]

    def forest_columns(self, cols, opts: SolveOpts | None = None, stream=None):
        """Columns `cols` of Omega = (I+L)^{-1} (row f4): a [n][len(cols)] fp64 CUDA tensor + report."""
        import numpy as np
        import torch
        c = np.ascontiguousarray(cols, dtype=np.int32)
        if self.old2new is not None:   # Omega' = P Omega P^T: column c of Omega is column old2new[c] of Omega'
            if len(c) and (c.min() < 0 or c.max() >= self.n):
                raise ValueError("column index out of range")
            c = np.ascontiguousarray(self.old2new.cpu().numpy()[c], dtype=np.int32)
        rep = SolveReport()
        o = opts or SolveOpts.make()
        with _on(stream):
            out = torch.empty((self.n, len(c)), dtype=torch.float64, device=self._keep[0].device)
            _check(lib().fj_forest_columns(self.handle, len(c), ctypes.c_void_p(c.ctypes.data), _ptr(out),
                                           ctypes.byref(o), ctypes.byref(rep), _stream(stream)))
            return self._out(out, stream), rep.to_dict()

    def close(self):
        if getattr(self, "_h", None) is not None and _lib is not None:
            _lib.fj_graph_destroy(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Comm:
    """Communicator of the row-partitioned path (rows a8/e): NCCL, or LOOPBACK for virtual ranks in one process."""

    def __init__(self, handle, nranks, kind):
        self._h, self.nranks, self.kind = handle, nranks, kind

    @staticmethod
    def unique_id() -> bytes:
        buf = ctypes.create_string_buffer(128)
        _check(lib().fj_comm_unique_id(buf))
        return buf.raw

    @classmethod
    def nccl(cls, nranks: int, rank: int, uid: bytes):
        h = _vp()
        buf = ctypes.create_string_buffer(bytes(uid), 128)
        _check(lib().fj_comm_init(nranks, rank, buf, ctypes.byref(h)))
        return cls(h, nranks, "nccl")

    @classmethod
    def loopback(cls, nranks: int):
        h = _vp()
        _check(lib().fj_comm_init_loopback(nranks, ctypes.byref(h)))
        return cls(h, nranks, "loopback")

    def close(self):
        if getattr(self, "_h", None) is not None and _lib is not None:
            _lib.fj_comm_destroy(self._h)
        self._h = None


def edge_degree_order(n: int, u, v, stream=None):
    """fj_edge_degree_order: (new2old, old2new) int32 device permutations from the raw edge list."""
    import torch
    _need_cuda(u, v)
    new2old = torch.empty(n, dtype=torch.int32, device=u.device)
    old2new = torch.empty(n, dtype=torch.int32, device=u.device)
    _check(lib().fj_edge_degree_order(n, int(u.numel()), _ptr(u), _ptr(v), _ptr(new2old), _ptr(old2new),
                                      _stream(stream)))
    return new2old, old2new


def partition_rows(n: int, u, v, nranks: int, stream=None, old2new=None):
    """Contiguous nnz-balanced row blocks (in the relabelled ids when old2new is given)."""
    import numpy as np
    _need_cuda(u, v, old2new)
    b = np.zeros(nranks + 1, dtype=np.int64)
    if old2new is None:
        _check(lib().fj_partition_rows(n, int(u.numel()), _ptr(u), _ptr(v), nranks, ctypes.c_void_p(b.ctypes.data),
                                       _stream(stream)))
    else:
        _check(lib().fj_partition_rows_relabelled(n, int(u.numel()), _ptr(u), _ptr(v), _ptr(old2new), nranks,
                                                  ctypes.c_void_p(b.ctypes.data), _stream(stream)))
    return [int(x) for x in b]


def csr_rows_from_edges(n: int, u, v, w, r0: int, r1: int, stream=None, old2new=None):
    """Row a1 for rows [r0, r1) (of the relabelled graph when old2new is given):
    (row_ptr_local, col_global, w_out, nnz)."""
    import torch
    _need_cuda(u, v, w, old2new)
    m = int(u.numel())
    dev = u.device
    rp = torch.empty(r1 - r0 + 1, dtype=torch.int64, device=dev)
    col = torch.empty(max(2 * m, 1), dtype=torch.int32, device=dev)
    wo = None if w is None else torch.empty(max(2 * m, 1), dtype=w.dtype, device=dev)
    nnz = _i64()
    if old2new is None:
        _check(lib().fj_csr_rows_from_edges(n, m, _ptr(u), _ptr(v), _ptr(w), _wtype(w), r0, r1, _ptr(rp), _ptr(col),
                                            _ptr(wo), ctypes.byref(nnz), _stream(stream)))
    else:
        _check(lib().fj_csr_rows_from_edges_relabelled(n, m, _ptr(u), _ptr(v), _ptr(old2new), _ptr(w), _wtype(w), r0,
                                                       r1, _ptr(rp), _ptr(col), _ptr(wo), ctypes.byref(nnz),
                                                       _stream(stream)))
    k = nnz.value
    return rp, col[:k], (None if wo is None else wo[:k]), k


def dist_ghosts(col_global, r0: int, r1: int, stream=None):
    import torch
    _need_cuda(col_global)
    nnz = int(col_global.numel())
    out = torch.empty(max(nnz, 1), dtype=torch.int32, device=col_global.device)
    ng = _i64()
    _check(lib().fj_dist_ghosts(nnz, _ptr(col_global), r0, r1, _ptr(out), ctypes.byref(ng), _stream(stream)))
    return out[:ng.value]


class DistGraph(Graph):
    """One rank's handle of a row-partitioned graph."""

    def __init__(self, comm: Comm, rank: int, n_global: int, bounds, row_ptr, col_global, w, ghosts,
                 send_counts, send_idx, stream=None):
        import numpy as np
        L = lib()
        _need_cuda(row_ptr, col_global, w, ghosts, send_idx)
        self.n = int(bounds[rank + 1] - bounds[rank])
        self.rank, self.bounds, self.n_global = rank, list(bounds), n_global
        self._keep = (row_ptr, col_global, w, ghosts, send_idx, comm)
        b = np.asarray(bounds, dtype=np.int64)
        sc = np.asarray(send_counts, dtype=np.int64)
        h = _vp()
        _check(L.fj_graph_create_dist(comm._h, rank, n_global, ctypes.c_void_p(b.ctypes.data), int(col_global.numel()),
                                      _ptr(row_ptr), _ptr(col_global), _ptr(w), _wtype(w), int(ghosts.numel()),
                                      _ptr(ghosts), ctypes.c_void_p(sc.ctypes.data), _ptr(send_idx), _stream(stream),
                                      ctypes.byref(h)))
        self._h = h


def approxim_host(n, u, v, w, S, opts: SolveOpts | None = None, want_z=False, stream=None, z_out=None):
    """End-to-end from HOST numpy buffers (pinned memory recommended): H2D copies, CSR build, handle,
    Algorithm 1, D2H.  Returns (z or None, [quantities], report).  z_out: optional caller-owned host
    float64 array shaped like S (pinned for full link speed) that receives z."""
    import numpy as np
    L = lib()
    S = np.ascontiguousarray(S, dtype=np.float64)
    k = 1 if S.ndim == 1 else S.shape[1]
    u = np.ascontiguousarray(u, dtype=np.int32)
    v = np.ascontiguousarray(v, dtype=np.int32)
    wt = FJ_W_UNIT if w is None else {np.dtype(np.uint8): FJ_W_U8, np.dtype(np.float32): FJ_W_F32,
                                      np.dtype(np.float64): FJ_W_F64}[np.asarray(w).dtype]
    z = None
    if z_out is not None:
        if z_out.shape != S.shape or z_out.dtype != np.float64 or not z_out.flags.c_contiguous:
            raise ValueError("z_out must be a C-contiguous float64 array shaped like S")
        z = z_out
    elif want_z:   # pinned, so the D2H of z runs at full link speed
        import torch
        z = torch.empty(S.shape, dtype=torch.float64, pin_memory=True).numpy()
    q = (Quantities * k)()
    rep = SolveReport()
    o = opts or SolveOpts.make()
    wc = None if w is None else np.ascontiguousarray(w)   # keep alive across the call

    def ptr(a):
        return None if a is None else ctypes.c_void_p(a.ctypes.data)
    _check(L.fj_approxim_host(n, len(u), ptr(u), ptr(v), ptr(wc), wt, k, ptr(S), ptr(z), ctypes.byref(o), q,
                              ctypes.byref(rep), _stream(stream)))
    return z, [x.to_dict() for x in q], rep.to_dict()


def _isnan(x):
    return isinstance(x, float) and math.isnan(x)

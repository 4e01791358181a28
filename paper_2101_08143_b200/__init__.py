"""B200-native Friedkin-Johnsen opinion quantities (arXiv 2101.08143).

Thin Python binding over the C ABI in include/fj.h (libfj.so, built in-tree for sm_100a).
Argument marshalling only: every step of the path runs in the library's CUDA kernels.  There
is no CPU fallback: if libfj.so or a CUDA device is missing, calls raise.
"""
from .binding import (  # noqa: F401
    FJError, Graph, SolveOpts, approxim_host, csr_from_edges, lib, load_library, FJ_W_UNIT, FJ_W_U8,
    FJ_W_F32, FJ_W_F64, FJ_OP_L, FJ_OP_IPL, Comm, DistGraph, partition_rows, csr_rows_from_edges, dist_ghosts,
    probe_gather, alg1_delta, opinions_generate, connected_components, lcc, permute_rows,
    csr_degree_order, csr_permute, use_torch_allocator, allocator_live_blocks,
)

__all__ = ["FJError", "Graph", "SolveOpts", "approxim_host", "csr_from_edges", "lib", "load_library"]

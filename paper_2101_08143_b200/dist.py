"""Set-up plumbing of the row-partitioned path.

The per-iteration exchange (halo of p, allreduce of dot products) runs inside libfj over NCCL.
This module only wires the ONE set-up exchange the library cannot do alone: each rank tells the
owners of its ghost columns which rows it needs (an all-to-all of index lists), through an
`AllToAll` object: `TorchGroup` (torch.distributed, gloo on CPU or NCCL on GPU) or `ThreadGroup`
(virtual ranks as threads of one process, used with the library's LOOPBACK transport).
"""
from __future__ import annotations

import threading

import numpy as np


class TorchGroup:
    """all_to_all over a torch.distributed process group (gloo: CPU tensors, nccl: CUDA tensors)."""

    def __init__(self, group=None, device="cpu"):
        import torch.distributed as dist
        self.dist, self.group, self.device = dist, group, device
        self.rank = dist.get_rank(group)
        self.nranks = dist.get_world_size(group)

    def all_to_all(self, send_chunks):
        """send_chunks[q]: 1-D int64 numpy array for rank q -> list of arrays received from each rank."""
        import torch
        counts = torch.tensor([len(c) for c in send_chunks], dtype=torch.int64, device=self.device)
        rcounts = torch.empty_like(counts)
        self.dist.all_to_all_single(rcounts, counts, group=self.group)
        rc = rcounts.cpu().tolist()
        flat = np.concatenate([np.asarray(c, dtype=np.int64) for c in send_chunks]) if send_chunks else np.zeros(0)
        inp = torch.from_numpy(flat.astype(np.int64)).to(self.device)
        out = torch.empty(sum(rc), dtype=torch.int64, device=self.device)
        self.dist.all_to_all_single(out, inp, output_split_sizes=rc,
                                    input_split_sizes=[len(c) for c in send_chunks], group=self.group)
        o = out.cpu().numpy()
        res, p = [], 0
        for c in rc:
            res.append(o[p:p + c])
            p += c
        return res


class ThreadWorld:
    """Shared state of in-process virtual ranks (one thread each)."""

    def __init__(self, nranks):
        self.nranks = nranks
        self.barrier = threading.Barrier(nranks)
        self.box = [None] * nranks


class ThreadGroup:
    def __init__(self, world: ThreadWorld, rank: int):
        self.world, self.rank, self.nranks = world, rank, world.nranks

    def all_to_all(self, send_chunks):
        w = self.world
        w.box[self.rank] = [np.asarray(c, dtype=np.int64) for c in send_chunks]
        w.barrier.wait()
        res = [w.box[q][self.rank].copy() for q in range(self.nranks)]
        w.barrier.wait()
        return res


def owners(ids: np.ndarray, bounds) -> np.ndarray:
    """Owner rank of each global row id under contiguous row blocks `bounds` (len nranks + 1)."""
    return np.searchsorted(np.asarray(bounds[1:], dtype=np.int64), ids, side="right")


def exchange_requests(ghosts: np.ndarray, bounds, group):
    """Given this rank's sorted ghost ids, return (send_counts[q], send_idx) where send_idx holds the
    LOCAL indices of this rank's rows that rank q needs, concatenated in q order (the halo plan)."""
    rank, P = group.rank, group.nranks
    ghosts = np.asarray(ghosts, dtype=np.int64)
    own = owners(ghosts, bounds)
    chunks = [ghosts[own == q] for q in range(P)]
    if len(chunks[rank]):
        raise ValueError("ghost list contains own rows")
    got = group.all_to_all(chunks)
    r0 = int(bounds[rank])
    counts = [len(x) for x in got]
    idx = np.concatenate(got).astype(np.int64) - r0 if sum(counts) else np.zeros(0, dtype=np.int64)
    if len(idx) and (idx.min() < 0 or idx.max() >= int(bounds[rank + 1]) - r0):
        raise ValueError("requested rows outside this rank's block")
    return counts, idx.astype(np.int32)


def build_dist_graph(comm, rank, n, u, v, w, group, bounds=None, stream=None, order="natural"):
    """One rank's DistGraph from the full raw edge list on this rank's device (rows a1 + a2, a8 set-up).
    order="degree": the graph is relabelled by descending degree BEFORE partitioning
    (fj_edge_degree_order), so every rank's gathered vector packs its hot rows; the
    rank's opinion slice is then rows new2old[r0:r1] of s (slice_in below) and row i of the rank's z
    is row G.rows_global[i] of the global z."""
    import torch
    from . import binding as B
    n2o = o2n = None
    if order == "degree":
        n2o, o2n = B.edge_degree_order(n, u, v, stream)
    elif order != "natural":
        raise ValueError("order must be 'natural' or 'degree'")
    if bounds is None:
        bounds = B.partition_rows(n, u, v, comm.nranks, stream, old2new=o2n)
    r0, r1 = bounds[rank], bounds[rank + 1]
    rp, colg, wo, nnz = B.csr_rows_from_edges(n, u, v, w, r0, r1, stream, old2new=o2n)
    gh = B.dist_ghosts(colg, r0, r1, stream)
    counts, idx = exchange_requests(gh.cpu().numpy(), bounds, group)
    send_idx = torch.from_numpy(idx).to(u.device)
    G = B.DistGraph(comm, rank, n, bounds, rp, colg, wo, gh, counts, send_idx, stream)
    G.plan = {"n_ghost": int(gh.numel()), "send": counts, "nnz_local": nnz, "order": order}
    G.rows_global = None if n2o is None else n2o[r0:r1].contiguous()   # input id of each local row
    return G, bounds


def slice_in(G, S, bounds, stream=None):
    """This rank's opinion rows: S[r0:r1] (natural order) or S[new2old[r0:r1]] (degree order),
    gathered by the library's fj_permute_rows."""
    r0, r1 = bounds[G.rank], bounds[G.rank + 1]
    if G.rows_global is None:
        return S[r0:r1].contiguous()
    return _gather_rows(S, G.rows_global, stream)


def _gather_rows(S, idx, stream=None):
    """out[i] = S[idx[i]] for a global S (more rows than idx): fj_permute_rows over len(idx) rows."""
    import torch
    from . import binding as B
    k = 1 if S.dim() == 1 else S.shape[1]
    out = torch.empty((idx.numel(),) + tuple(S.shape[1:]), dtype=S.dtype, device=S.device)
    B._check(B.lib().fj_permute_rows(int(idx.numel()), k, B._ptr(idx), B._ptr(S), B._ptr(out), B._stream(stream)))
    return out

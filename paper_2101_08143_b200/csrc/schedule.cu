// schedule.cu — builds a warp-item list of the row engine on the device, once per graph and
// parameter set.  Row classes: T (len <= trow_max), W (trow_max < len <= chunk), C (len > chunk).
//   items = [ C chunks (per long row, in row order) | W rows | T tiles ]
// T tiles are maximal runs of consecutive T rows cut where the merge coordinate
// e_i = sum_{j<i, T rows} max(1 + len_j, t_min_cost) crosses a multiple of t_units, so a tile holds
// <= t_units - 1 + (1 + trow_max) merge items (row ends + nonzeros) and <= (that)/t_min_cost rows.
//   k = 1 engine (tiles.cuh):  trow_max 64, t_units 319 (=> <= 384 merge items = 32 lanes x 12),
//                              t_min_cost 12 (=> <= 32 rows), chunk 2048
//   batched engine (spmm.cu):  trow_max 64, t_units 160, t_min_cost 8, chunk 1024
#include "tiles.cuh"
#include "workspace.cuh"

namespace fj {

__device__ __forceinline__ int row_class(const int64_t* rp, int64_t i, const SchedParams& P) {
  const int64_t len = rp[i + 1] - rp[i];
  return len <= P.trow_max ? IT_T : (len <= P.chunk ? IT_W : IT_C);
}

__global__ void k_units(int64_t n, const int64_t* __restrict__ rp, SchedParams P, int64_t* __restrict__ c) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i > n) return;
  if (i == n) { c[i] = 0; return; }
  const int64_t len = rp[i + 1] - rp[i];
  c[i] = len <= P.trow_max ? (1 + len > P.t_min_cost ? 1 + len : P.t_min_cost) : 0;
}

// boundary flags over i in [0, n]
__global__ void k_bflags(int64_t n, const int64_t* __restrict__ rp, const int64_t* __restrict__ e, SchedParams P,
                         uint8_t* __restrict__ f) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i > n) return;
  bool b = (i == 0) || (i == n);
  if (!b)
    b = row_class(rp, i, P) != IT_T || row_class(rp, i - 1, P) != IT_T || (e[i] / P.t_units != e[i - 1] / P.t_units);
  f[i] = b ? 1 : 0;
}

// per segment j = [B[j], B[j+1]): counts of C chunks, W rows, T tiles, long rows
__global__ void k_segcount(int64_t nseg, const int32_t* __restrict__ B, const int64_t* __restrict__ rp,
                           SchedParams P, int64_t* __restrict__ nc, int64_t* __restrict__ nw,
                           int64_t* __restrict__ nt, int64_t* __restrict__ nl) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j > nseg) return;
  if (j == nseg) { nc[j] = nw[j] = nt[j] = nl[j] = 0; return; }
  const int64_t r = B[j];
  const int cls = row_class(rp, r, P);
  const int64_t len = rp[r + 1] - rp[r];
  nc[j] = cls == IT_C ? (len + P.chunk - 1) / P.chunk : 0;
  nw[j] = cls == IT_W ? 1 : 0;
  nt[j] = cls == IT_T ? 1 : 0;
  nl[j] = cls == IT_C ? 1 : 0;
}

__global__ void k_items(int64_t nseg, const int32_t* __restrict__ B, const int64_t* __restrict__ rp, SchedParams P,
                        const int64_t* __restrict__ pc, const int64_t* __restrict__ pw,
                        const int64_t* __restrict__ pt, const int64_t* __restrict__ pl, int64_t n_chunks,
                        int64_t n_w, ItemMeta* __restrict__ items, int32_t* __restrict__ lnch,
                        int32_t* __restrict__ litem0) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= nseg) return;
  const int64_t r = B[j], r1 = B[j + 1];
  const int cls = row_class(rp, r, P);
  const int64_t k0 = rp[r];
  if (cls == IT_T) {
    const int64_t nk = rp[r1] - k0;
    ItemMeta m;
    m.r0 = (int32_t)r;
    m.info = ((uint32_t)IT_T << 30) | (uint32_t)(r1 - r) | ((uint32_t)nk << 7);   // tiles.cuh tile_rows / tile_nnz
    m.k0 = k0;
    items[n_chunks + n_w + pt[j]] = m;
  } else if (cls == IT_W) {
    ItemMeta m;
    m.r0 = (int32_t)r;
    m.info = ((uint32_t)IT_W << 30) | (uint32_t)(rp[r + 1] - k0);
    m.k0 = k0;
    items[n_chunks + pw[j]] = m;
  } else {
    const int64_t len = rp[r + 1] - k0;
    const int64_t nch = (len + P.chunk - 1) / P.chunk;
    const int64_t l = pl[j];
    lnch[l] = (int32_t)nch;
    litem0[l] = (int32_t)pc[j];
    for (int64_t c = 0; c < nch; ++c) {
      ItemMeta m;
      m.r0 = (int32_t)r;
      m.info = ((uint32_t)IT_C << 30) | (uint32_t)l;
      m.k0 = k0 + c * P.chunk;
      items[pc[j] + c] = m;
    }
  }
}

static inline unsigned nb256(int64_t n) { return (unsigned)((n + 255) / 256); }

void free_sched(Sched& s) {
  dfree(s.items); dfree(s.long_nchunks); dfree(s.long_item0);
  s = Sched();
}

fj_status build_schedule(fj_graph* g, const SchedParams& P, Sched& out, cudaStream_t st) {
  const int64_t n = g->n;
  DevBuf<int64_t> c, e;
  DevBuf<uint8_t> f;
  DevBuf<int32_t> B, nsel;
  FJ_TRY(c.alloc(n + 1, st));
  FJ_TRY(e.alloc(n + 1, st));
  FJ_TRY(f.alloc(n + 1, st));
  FJ_TRY(B.alloc(n + 1, st));
  FJ_TRY(nsel.alloc(1, st));
  k_units<<<nb256(n + 1), 256, 0, st>>>(n, g->row_ptr, P, c.p);
  FJ_CK_LAUNCH();
  FJ_TRY(cub_exclusive_sum(c.p, e.p, n + 1, st));
  k_bflags<<<nb256(n + 1), 256, 0, st>>>(n, g->row_ptr, e.p, P, f.p);
  FJ_CK_LAUNCH();
  FJ_TRY(cub_select_index(f.p, B.p, nsel.p, n + 1, st));
  c.release(); e.release(); f.release();
  int32_t nb = 0;
  FJ_CK(cudaMemcpyAsync(&nb, nsel.p, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  FJ_CK(cudaStreamSynchronize(st));
  const int64_t nseg = nb - 1;
  DevBuf<int64_t> nc, nw, nt, nl, pc, pw, pt, pl;
  for (auto* d : {&nc, &nw, &nt, &nl, &pc, &pw, &pt, &pl}) FJ_TRY(d->alloc(nseg + 1, st));
  k_segcount<<<nb256(nseg + 1), 256, 0, st>>>(nseg, B.p, g->row_ptr, P, nc.p, nw.p, nt.p, nl.p);
  FJ_CK_LAUNCH();
  FJ_TRY(cub_exclusive_sum(nc.p, pc.p, nseg + 1, st));
  FJ_TRY(cub_exclusive_sum(nw.p, pw.p, nseg + 1, st));
  FJ_TRY(cub_exclusive_sum(nt.p, pt.p, nseg + 1, st));
  FJ_TRY(cub_exclusive_sum(nl.p, pl.p, nseg + 1, st));
  int64_t tot[4];
  FJ_CK(cudaMemcpyAsync(&tot[0], pc.p + nseg, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  FJ_CK(cudaMemcpyAsync(&tot[1], pw.p + nseg, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  FJ_CK(cudaMemcpyAsync(&tot[2], pt.p + nseg, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  FJ_CK(cudaMemcpyAsync(&tot[3], pl.p + nseg, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  FJ_CK(cudaStreamSynchronize(st));
  free_sched(out);
  out.n_long_chunks = tot[0];
  out.n_wrows = tot[1];
  out.n_tiles = tot[2];
  out.n_long = tot[3];
  out.n_items = tot[0] + tot[1] + tot[2];
  out.chunk = P.chunk;
  FJ_CK(dmalloc(&out.items, sizeof(ItemMeta) * (size_t)std::max<int64_t>(out.n_items, 1), st));
  FJ_CK(dmalloc(&out.long_nchunks, sizeof(int32_t) * (size_t)std::max<int64_t>(out.n_long, 1), st));
  FJ_CK(dmalloc(&out.long_item0, sizeof(int32_t) * (size_t)std::max<int64_t>(out.n_long, 1), st));
  if (nseg > 0) {
    k_items<<<nb256(nseg), 256, 0, st>>>(nseg, B.p, g->row_ptr, P, pc.p, pw.p, pt.p, pl.p, tot[0], tot[1],
                                         reinterpret_cast<ItemMeta*>(out.items), out.long_nchunks, out.long_item0);
    FJ_CK_LAUNCH();
  }
  FJ_CK(cudaStreamSynchronize(st));
  out.built = true;
  return FJ_OK;
}

}  // namespace fj

// schedule.cu — builds the warp-item list of the row engine (tiles.cuh) on the device, once per
// graph.  Row classes: T (len <= T_ROW_MAX), W (T_ROW_MAX < len <= CHUNK), C (len > CHUNK).
//   items = [ C chunks (per long row, in row order) | W rows | T tiles ]
// T tiles are maximal runs of consecutive T rows cut where the merge coordinate
// e_i = sum_{j<i, T rows} max(1 + len_j, T_ROW_MIN_COST) crosses a multiple of T_UNITS, so a tile
// holds <= T_UNITS - 1 + (1 + T_ROW_MAX) = T_CAP merge items (row ends + nonzeros) and <= 32 rows.
#include "tiles.cuh"
#include "workspace.cuh"

namespace fj {

__device__ __forceinline__ int row_class(const int64_t* rp, int64_t i) {
  const int64_t len = rp[i + 1] - rp[i];
  return len <= T_ROW_MAX ? IT_T : (len <= CHUNK ? IT_W : IT_C);
}

__global__ void k_units(int64_t n, const int64_t* __restrict__ rp, int64_t* __restrict__ c) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i > n) return;
  if (i == n) { c[i] = 0; return; }
  const int64_t len = rp[i + 1] - rp[i];
  // a T row is 1 + len merge items; charging at least T_ROW_MIN_COST caps a tile at 32 rows
  c[i] = len <= T_ROW_MAX ? (1 + len > T_ROW_MIN_COST ? 1 + len : T_ROW_MIN_COST) : 0;
}

// boundary flags over i in [0, n]
__global__ void k_bflags(int64_t n, const int64_t* __restrict__ rp, const int64_t* __restrict__ e,
                         uint8_t* __restrict__ f) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i > n) return;
  bool b = (i == 0) || (i == n);
  if (!b)
    b = row_class(rp, i) != IT_T || row_class(rp, i - 1) != IT_T || (e[i] / T_UNITS != e[i - 1] / T_UNITS);
  f[i] = b ? 1 : 0;
}

// per segment j = [B[j], B[j+1]): counts of heavy items (C chunks / W rows), tiles, long rows
__global__ void k_segcount(int64_t nseg, const int32_t* __restrict__ B, const int64_t* __restrict__ rp,
                           int64_t* __restrict__ nc, int64_t* __restrict__ nw, int64_t* __restrict__ nt,
                           int64_t* __restrict__ nl) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j > nseg) return;
  if (j == nseg) { nc[j] = nw[j] = nt[j] = nl[j] = 0; return; }
  const int64_t r = B[j];
  const int cls = row_class(rp, r);
  const int64_t len = rp[r + 1] - rp[r];
  nc[j] = cls == IT_C ? (len + CHUNK - 1) / CHUNK : 0;
  nw[j] = cls == IT_W ? 1 : 0;
  nt[j] = cls == IT_T ? 1 : 0;
  nl[j] = cls == IT_C ? 1 : 0;
}

__global__ void k_items(int64_t nseg, const int32_t* __restrict__ B, const int64_t* __restrict__ rp,
                        const int64_t* __restrict__ pc, const int64_t* __restrict__ pw,
                        const int64_t* __restrict__ pt, const int64_t* __restrict__ pl, int64_t n_chunks,
                        int64_t n_w, ItemMeta* __restrict__ items, int32_t* __restrict__ lnch,
                        int32_t* __restrict__ litem0) {
  const int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (j >= nseg) return;
  const int64_t r = B[j], r1 = B[j + 1];
  const int cls = row_class(rp, r);
  const int64_t k0 = rp[r];
  if (cls == IT_T) {
    const int64_t nk = rp[r1] - k0;
    ItemMeta m;
    m.r0 = (int32_t)r;
    m.info = ((uint32_t)IT_T << 30) | (uint32_t)(r1 - r) | ((uint32_t)nk << 6);
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
    const int64_t nch = (len + CHUNK - 1) / CHUNK;
    const int64_t l = pl[j];
    lnch[l] = (int32_t)nch;
    litem0[l] = (int32_t)pc[j];
    for (int64_t c = 0; c < nch; ++c) {
      ItemMeta m;
      m.r0 = (int32_t)r;
      m.info = ((uint32_t)IT_C << 30) | (uint32_t)l;
      m.k0 = k0 + c * CHUNK;
      items[pc[j] + c] = m;
    }
  }
}

static inline unsigned nb256(int64_t n) { return (unsigned)((n + 255) / 256); }

fj_status build_schedule(fj_graph* g, cudaStream_t st) {
  const int64_t n = g->n;
  DevBuf<int64_t> c, e;
  DevBuf<uint8_t> f;
  DevBuf<int32_t> B, nsel;
  FJ_TRY(c.alloc(n + 1, st));
  FJ_TRY(e.alloc(n + 1, st));
  FJ_TRY(f.alloc(n + 1, st));
  FJ_TRY(B.alloc(n + 1, st));
  FJ_TRY(nsel.alloc(1, st));
  k_units<<<nb256(n + 1), 256, 0, st>>>(n, g->row_ptr, c.p);
  FJ_CK_LAUNCH();
  FJ_TRY(cub_exclusive_sum(c.p, e.p, n + 1, st));
  k_bflags<<<nb256(n + 1), 256, 0, st>>>(n, g->row_ptr, e.p, f.p);
  FJ_CK_LAUNCH();
  FJ_TRY(cub_select_index(f.p, B.p, nsel.p, n + 1, st));
  c.release(); e.release(); f.release();
  int32_t nb = 0;
  FJ_CK(cudaMemcpyAsync(&nb, nsel.p, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  FJ_CK(cudaStreamSynchronize(st));
  const int64_t nseg = nb - 1;
  DevBuf<int64_t> nc, nw, nt, nl, pc, pw, pt, pl;
  for (auto* d : {&nc, &nw, &nt, &nl, &pc, &pw, &pt, &pl}) FJ_TRY(d->alloc(nseg + 1, st));
  k_segcount<<<nb256(nseg + 1), 256, 0, st>>>(nseg, B.p, g->row_ptr, nc.p, nw.p, nt.p, nl.p);
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
  g->n_long_chunks = tot[0];
  g->n_wrows = tot[1];
  g->n_tiles = tot[2];
  g->n_long = tot[3];
  g->n_items = tot[0] + tot[1] + tot[2];
  FJ_CK(dmalloc(&g->items, sizeof(ItemMeta) * (size_t)std::max<int64_t>(g->n_items, 1), st));
  FJ_CK(dmalloc(&g->long_nchunks, sizeof(int32_t) * (size_t)std::max<int64_t>(g->n_long, 1), st));
  FJ_CK(dmalloc(&g->long_item0, sizeof(int32_t) * (size_t)std::max<int64_t>(g->n_long, 1), st));
  if (nseg > 0) {
    k_items<<<nb256(nseg), 256, 0, st>>>(nseg, B.p, g->row_ptr, pc.p, pw.p, pt.p, pl.p, tot[0], tot[1],
                                         reinterpret_cast<ItemMeta*>(g->items), g->long_nchunks, g->long_item0);
    FJ_CK_LAUNCH();
  }
  FJ_CK(cudaStreamSynchronize(st));
  return FJ_OK;
}

}  // namespace fj

// segments.cu — L2-sized column segments of the CSR for the PCG product.
//
// The (I+L)p product gathers p at random rows.  While the gathered block (n rows x KP doubles)
// fits in L2 the gathers are L2 hits at ~250-270 G gathers/s on B200; once it exceeds the part
// of the 126 MB L2 that survives the CSR streams, the rate collapses (fj_probe_gather: 113 G/s at
// 128 MB, 47 G/s at 512 MB).  So when n * KP * 8 bytes exceeds kSegBytes, the columns are cut
// into nseg equal ranges and the CSR is re-laid out as nseg column-segment CSRs (same rows, the
// nonzeros of each row whose column falls in the range, still ascending).  One product is then
// nseg passes of the warp-item engine; pass s gathers only from p's s-th slice, which stays
// L2-resident.  Pass 0 writes y_i = (1 + d_i) x_i - acc, later passes subtract their partial
// sums from y_i, the last pass forms the p^T q partials and finalises alpha on device.
//
// Cost: one extra copy of col (+ weights) and nseg row_ptr arrays, built once per (graph, KP);
// per product the row_ptr of every segment and a read-modify-write of y per extra pass.
//
// MEASURED NEGATIVE (B200, round 1): OFF by default (FJ_SEG_MB=<MB> enables it; tests force it on a
// small graph).  C3 k = 3 (128 MB padded p): 1 segment 1.05 ms, 2 x 64 MB 1.83 ms, 3 x 48 MB 2.67 ms;
// C5 k = 1 (537 MB): 25 ms unsegmented vs 91 ms with 11 x 48 MB.  ncu of a 64 MB pass: L2 hit rate
// only 47-54 % (the x_i / y / col streams of the pass still evict the p slice), and the extra
// y read-modify-write lifts the vector operator to 2 blocks / SM.  R-MAT's hub skew already gives the
// unsegmented product L2 hits (C5: 84 G nonzeros/s vs the 47 G/s uniform-random probe).
#include <algorithm>
#include <cstdlib>

#include "tiles.cuh"
#include "workspace.cuh"

namespace fj {

int64_t seg_bytes() {
  static const int64_t v = [] {
    const char* e = getenv("FJ_SEG_MB");
    return (int64_t)((e ? atof(e) : 0.0) * (1 << 20));   // default 0: off (see below)
  }();
  return v;
}

int seg_count(const fj_graph* g, int kp) {
  const int64_t bytes = g->n * (int64_t)kp * 8;
  const int64_t sb = seg_bytes();
  if (sb <= 0 || bytes <= sb) return 1;
  return (int)std::min<int64_t>((bytes + sb - 1) / sb, MAXSEG);
}

__device__ __forceinline__ int64_t lower_bound_col(const int32_t* __restrict__ col, int64_t b, int64_t e, int64_t v) {
  while (b < e) {
    const int64_t m = (b + e) >> 1;
    if (col[m] < v) b = m + 1; else e = m;
  }
  return b;
}

// cnt[i] = #{ p in row i : lo <= col[p] < hi }, cnt[n] = 0
__global__ void k_seg_count(int64_t n, const int64_t* __restrict__ rp, const int32_t* __restrict__ col, int64_t lo,
                            int64_t hi, int64_t* __restrict__ cnt) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i > n) return;
  if (i == n) { cnt[n] = 0; return; }
  const int64_t b = rp[i], e = rp[i + 1];
  const int64_t a = lower_bound_col(col, b, e, lo);
  cnt[i] = lower_bound_col(col, a, e, hi) - a;
}

// warp per row: copy the row's [lo, hi) columns (and weights) to the segment CSR
__global__ void k_seg_copy(int64_t n, const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                           const unsigned char* __restrict__ w, int wbytes, int64_t lo, int64_t hi,
                           const int64_t* __restrict__ rps, int32_t* __restrict__ cols, unsigned char* __restrict__ ws) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t i = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); i < n; i += nw) {
    const int64_t b = rp[i], e = rp[i + 1];
    const int64_t a = lower_bound_col(col, b, e, lo);
    const int64_t o = rps[i], len = rps[i + 1] - o;
    for (int64_t t = lane; t < len; t += 32) {
      cols[o + t] = col[a + t];
      for (int q = 0; q < wbytes; ++q) ws[(o + t) * wbytes + q] = w[(a + t) * wbytes + q];
    }
  }
}

static void free_layout(SegLayout* L) {
  for (int s = 0; s < L->nseg; ++s) {
    dfree(L->rp[s]); dfree(L->col[s]); dfree(L->w[s]);
    free_sched(L->sched[s]);
  }
  dfree(L->ts.block_part); dfree(L->ts.long_part); dfree(L->ts.chunk_acc);
  dfree(L->ts.long_ticket); dfree(L->ts.grid_ticket);
  delete L;
}

void free_segments(fj_graph* g) {
  for (int kp = 0; kp < 5; ++kp) {
    if (g->seg[kp]) free_layout(reinterpret_cast<SegLayout*>(g->seg[kp]));
    g->seg[kp] = nullptr;
  }
}

static fj_status build_layout(fj_graph* g, int kp, int nseg, SegLayout* L, cudaStream_t st);

// The segment layout for gathered width kp (1..4), built on first use and kept until the graph is
// destroyed (captured solve loops reference it); nullptr when one segment suffices.
fj_status get_segments(fj_graph* g, int kp, cudaStream_t st, const SegLayout** out) {
  *out = nullptr;
  if (g->dist || kp < 1 || kp > 4) return FJ_OK;
  const int nseg = seg_count(g, kp);
  if (nseg <= 1) return FJ_OK;
  if (g->seg[kp]) { *out = reinterpret_cast<const SegLayout*>(g->seg[kp]); return FJ_OK; }
  SegLayout* L = new SegLayout();
  const fj_status s = build_layout(g, kp, nseg, L, st);
  if (s != FJ_OK) {
    cudaStreamSynchronize(st);
    free_layout(L);
    return s;
  }
  g->seg[kp] = L;   // published only when complete
  *out = L;
  return FJ_OK;
}

static fj_status build_layout(fj_graph* g, int kp, int nseg, SegLayout* L, cudaStream_t st) {
  const int64_t n = g->n;
  const int wbytes = g->wtype == FJ_W_UNIT ? 0 : g->wtype == FJ_W_U8 ? 1 : g->wtype == FJ_W_F32 ? 4 : 8;
  DevBuf<int64_t> cnt;
  FJ_TRY(cnt.alloc(n + 1, st));
  int64_t max_long = 0, max_chunks = 0;
  for (int s = 0; s < nseg; ++s) {
    const int64_t lo = n * s / nseg, hi = n * (s + 1) / nseg;
    L->bounds[s] = lo;
    L->bounds[s + 1] = hi;
    k_seg_count<<<(unsigned)((n + 256) / 256), 256, 0, st>>>(n, g->row_ptr, g->col, lo, hi, cnt.p);
    FJ_CK_LAUNCH();
    FJ_CK(dmalloc(&L->rp[s], sizeof(int64_t) * (size_t)(n + 1), st));
    L->nseg = s + 1;   // free_layout releases what exists so far on error
    FJ_TRY(cub_exclusive_sum(cnt.p, L->rp[s], n + 1, st));
    int64_t nnz_s = 0;
    FJ_CK(cudaMemcpyAsync(&nnz_s, L->rp[s] + n, sizeof nnz_s, cudaMemcpyDeviceToHost, st));
    FJ_CK(cudaStreamSynchronize(st));
    L->nnz[s] = nnz_s;
    FJ_CK(dmalloc(&L->col[s], sizeof(int32_t) * (size_t)std::max<int64_t>(nnz_s, 4), st));
    if (wbytes) FJ_CK(dmalloc(reinterpret_cast<unsigned char**>(&L->w[s]), (size_t)std::max<int64_t>(nnz_s, 4) * wbytes, st));
    k_seg_copy<<<g->num_sms * 16, 256, 0, st>>>(n, g->row_ptr, g->col,
                                                 reinterpret_cast<const unsigned char*>(g->w), wbytes, lo, hi,
                                                 L->rp[s], L->col[s], reinterpret_cast<unsigned char*>(L->w[s]));
    FJ_CK_LAUNCH();
    fj_graph tmp = *g;   // shallow view for the schedule builder (reads n and row_ptr only)
    tmp.row_ptr = L->rp[s];
    tmp.col = L->col[s];
    tmp.nnz = nnz_s;
    FJ_TRY(build_schedule(&tmp, kp == 1 ? kSchedK1 : kSchedVec, L->sched[s], st));
    max_long = std::max(max_long, L->sched[s].n_long);
    max_chunks = std::max(max_chunks, L->sched[s].n_long_chunks);
  }
  L->kp = kp;
  L->grid_max = g->num_sms * (2048 / WTPB);
  constexpr int NPMAX = 4, NAMAX = 4;   // the segmented passes run ApplyOp / ApplyOpV (KP <= 4)
  FJ_CK(dmalloc(&L->ts.block_part, sizeof(double) * (size_t)L->grid_max * NPMAX, st));
  FJ_CK(dmalloc(&L->ts.long_part, sizeof(double) * (size_t)std::max<int64_t>(max_long, 1) * NPMAX, st));
  FJ_CK(dmalloc(&L->ts.chunk_acc, sizeof(double) * (size_t)std::max<int64_t>(max_chunks, 1) * NAMAX, st));
  FJ_CK(dmalloc(&L->ts.long_ticket, sizeof(unsigned) * (size_t)std::max<int64_t>(max_long, 1), st));
  FJ_CK(cudaMemsetAsync(L->ts.long_ticket, 0, sizeof(unsigned) * (size_t)std::max<int64_t>(max_long, 1), st));
  FJ_CK(dmalloc(&L->ts.grid_ticket, sizeof(unsigned), st));
  FJ_CK(cudaMemsetAsync(L->ts.grid_ticket, 0, sizeof(unsigned), st));
  FJ_CK(cudaStreamSynchronize(st));
  return FJ_OK;
}

}  // namespace fj

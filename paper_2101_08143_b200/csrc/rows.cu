// rows.cu — the plan of the lean row product (rows.cuh), built once per graph
// and gathered row width with the solver workspace.
#include <algorithm>
#include <climits>
#include <cstdlib>
#include <type_traits>

#include "rows.cuh"
#include "workspace.cuh"

namespace fj {

// ---------------------------------------------------------------- plan (built once per graph)
// nch[i] = chunks of a long row; off[i] = entries with column < split; *bad |= 1 if some row's
// slab-A entries are not a prefix of the row (columns not ascending: the 2-slab split is off).
__global__ void k_rows_plan1(int64_t n, const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                             int64_t split, int64_t long_row, int32_t* __restrict__ nch, uint16_t* __restrict__ off,
                             int32_t* __restrict__ rp32, int* bad) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = rp[i], e = rp[i + 1];
    rp32[i + 1] = (int32_t)e;
    if (i == 0) rp32[0] = (int32_t)b;
    nch[i] = e - b > long_row ? (int32_t)((e - b + ROWS_CH - 1) / ROWS_CH) : 0;
    if (!off) continue;
    if (e - b > long_row) { off[i] = 0; continue; }   // long rows are summed whole by chunk warps
    int32_t lo = 0;
    bool hi_seen = false, viol = false;
    for (int64_t k = b; k < e; ++k) {
      if (col[k] < split) { ++lo; viol |= hi_seen; } else { hi_seen = true; }
    }
    off[i] = (uint16_t)lo;   // <= long_row < 2^16
    if (viol) atomicOr(bad, 1);
  }
}
__global__ void k_rows_plan2(int64_t n, const int64_t* __restrict__ rp, const int32_t* __restrict__ nch,
                             const int32_t* __restrict__ c0, int64_t* __restrict__ tab) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t m = nch[i];
    for (int32_t c = 0; c < m; ++c) {
      tab[2 * ((int64_t)c0[i] + c)] = i;
      tab[2 * ((int64_t)c0[i] + c) + 1] = rp[i] + (int64_t)c * ROWS_CH;
    }
  }
}
// Slab-major copies (mode 2, unit weights): cA[i] / cB[i] = slab-A / slab-B entries of short row i
// (0 for long rows, whose entries the chunk warps sum from col), cA[n] = cB[n] = 0 so their
// exclusive scans are rpA / rpB with the totals at [n].
__global__ void k_rows_plan3(int64_t n, const int32_t* __restrict__ rp32, const uint16_t* __restrict__ off,
                             int64_t long_row, int32_t* __restrict__ cA, int32_t* __restrict__ cB) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= n; i += (int64_t)gridDim.x * blockDim.x) {
    if (i == n) { cA[n] = cB[n] = 0; continue; }
    const int32_t len = rp32[i + 1] - rp32[i];
    const bool lng = len > long_row;
    const int32_t na = lng ? 0 : off[i], nb = lng ? 0 : len - off[i];
    cA[i] = FJ_ROWS_PAD_A ? (na + FJ_ROWS_PAD_A - 1) / FJ_ROWS_PAD_A * FJ_ROWS_PAD_A : na;   // padded row lengths
    cB[i] = FJ_ROWS_PAD_B ? (nb + FJ_ROWS_PAD_B - 1) / FJ_ROWS_PAD_B * FJ_ROWS_PAD_B : nb;
  }
}
// one warp per row: colA[rpA[i] + t] = col[rp[i] + t], colB[rpB[i] + t] = col[rp[i] + off[i] + t]
// (and the weights alike, T the weight type; T = void: unit weights, no array)
template <class T>
__global__ void k_rows_plan4(int64_t n, const int32_t* __restrict__ rp32, const uint16_t* __restrict__ off,
                             const int32_t* __restrict__ col, const void* __restrict__ w,
                             const int32_t* __restrict__ rpA, const int32_t* __restrict__ rpB,
                             int32_t* __restrict__ colA, int32_t* __restrict__ colB, void* __restrict__ wA,
                             void* __restrict__ wB) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x / 32);
  for (int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; i < n; i += nw) {
    // pa / pb: the copy's (possibly padded) row lengths; na / nb the entries (0 for long rows, whose
    // ranges are empty); pads are column -1 with weight 0
    const int32_t b = rp32[i], a0 = rpA[i], pa = rpA[i + 1] - a0, b0 = rpB[i], pb = rpB[i + 1] - b0;
    const int32_t o = off[i];
    const int32_t na = pa ? o : 0, nb = pb ? rp32[i + 1] - b - o : 0;
    for (int32_t t = lane; t < pa; t += 32) colA[a0 + t] = t < na ? col[b + t] : -1;
    for (int32_t t = lane; t < pb; t += 32) colB[b0 + t] = t < nb ? col[b + o + t] : -1;
    if constexpr (!std::is_void<T>::value) {
      const T* ws = reinterpret_cast<const T*>(w);
      for (int32_t t = lane; t < pa; t += 32) reinterpret_cast<T*>(wA)[a0 + t] = t < na ? ws[b + t] : T(0);
      for (int32_t t = lane; t < pb; t += 32) reinterpret_cast<T*>(wB)[b0 + t] = t < nb ? ws[b + o + t] : T(0);
    }
  }
}
template <class T> struct WTag { using type = T; };

// FJ_ROWS_SPLIT (A/B): 1 (default) builds the slab-major copies for mode 2, 0 not
static int rows_split_knob() {
  static const int v = [] { const char* e = getenv("FJ_ROWS_SPLIT"); return e ? atoi(e) : 1; }();
  return v;
}

// FJ_ROWS (A/B, tests): -1 auto (default), 0 merge-path engine, 1 one row pass, 2 two column
// slabs.  Auto: two slabs when the gathered block (n x kp doubles) is in (64 MB, 160 MB] -- each half
// then fits the ~80 MB the L2 holds for random gathers -- and every row's columns
// ascend; else one row pass.
static int rows_knob() {
  static const int v = [] { const char* e = getenv("FJ_ROWS"); return e ? atoi(e) : -1; }();
  return v;
}
constexpr int64_t kRowsSlabMin = 64ll << 20, kRowsSlabMax = 160ll << 20;

void rows_plan_free(RowsPlan& R) {
  dfree(R.off); dfree(R.rp32); dfree(R.c0); dfree(R.tab); dfree(R.chunk_acc); dfree(R.part); dfree(R.ticket);
  dfree(R.op_acc); dfree(R.op_part); dfree(R.op_ticket);
  dfree(R.rpA); dfree(R.rpB); dfree(R.colA); dfree(R.colB); dfree(R.wA); dfree(R.wB);
  R = RowsPlan{};
}

template <class T>
static fj_status ralloc(T** p, int64_t count, cudaStream_t st) {
  if (count < 1) count = 1;
  FJ_CK(dmalloc(p, sizeof(T) * (size_t)count, st));
  return FJ_OK;
}

// mode 2 allowed only for a graph's own CSR (two_ok); the knob and the size rule as described above
static fj_status plan_core(int64_t n, int64_t nnz, const int64_t* row_ptr, const int32_t* col, int kp, int num_sms,
                           bool two_ok, const void* w, int wtype, RowsPlan& R, cudaStream_t st) {
  rows_plan_free(R);
  const int knob = rows_knob();
  // mode 0, the engine: forced, or a CSR beyond the plan's int32 row_ptr
  if (knob == 0 || nnz >= (int64_t)INT32_MAX) return FJ_OK;
  R.num_sms = num_sms;
  const int64_t bytes_p = n * (int64_t)kp * 8;
  bool two = two_ok && (knob == 2 || (knob < 0 && bytes_p > kRowsSlabMin && bytes_p <= kRowsSlabMax));
  R.long_row = kp == 1 ? FJ_ROWS_LONG1 : FJ_ROWS_LONG;
  const unsigned cb = (unsigned)std::min<int64_t>((n + 255) / 256, 8192);
  DevBuf<int32_t> nch;
  DevBuf<int> bad;
  FJ_TRY(nch.alloc(n, st));
  FJ_TRY(bad.alloc(1, st));
  FJ_CK(cudaMemsetAsync(bad.p, 0, sizeof(int), st));
  FJ_TRY(ralloc(&R.c0, n, st));
  FJ_TRY(ralloc(&R.rp32, n + 1, st));
  if (n == 0) FJ_CK(cudaMemsetAsync(R.rp32, 0, sizeof(int32_t), st));
  if (two) FJ_TRY(ralloc(&R.off, n, st));
  if (n > 0) {
    k_rows_plan1<<<cb, 256, 0, st>>>(n, row_ptr, col, n / 2, R.long_row, nch.p, two ? R.off : nullptr, R.rp32,
                                     bad.p);
    FJ_CK_LAUNCH();
    size_t tb = 0;
    FJ_CK(cub::DeviceScan::ExclusiveSum(nullptr, tb, nch.p, R.c0, n, st));
    DevBuf<uint8_t> tmp;
    FJ_TRY(tmp.alloc((int64_t)tb, st));
    FJ_CK(cub::DeviceScan::ExclusiveSum(tmp.p, tb, nch.p, R.c0, n, st));
    count_cub();
  }
  int32_t last[2] = {0, 0};
  int hbad = 0;
  if (n > 0) {
    FJ_CK(cudaMemcpyAsync(&last[0], R.c0 + n - 1, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    FJ_CK(cudaMemcpyAsync(&last[1], nch.p + n - 1, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  }
  FJ_CK(cudaMemcpyAsync(&hbad, bad.p, sizeof(int), cudaMemcpyDeviceToHost, st));
  FJ_CK(cudaStreamSynchronize(st));
  R.n_chunks = (int64_t)last[0] + last[1];
  if (two && hbad) {   // columns not ascending in some row: slab A is not a prefix -> one pass
    if (knob == 2) return fail(FJ_E_INVALID_ARG, "FJ_ROWS=2 needs ascending columns in every row");
    two = false;
    dfree(R.off);
    R.off = nullptr;
  }
  if (two && rows_split_knob() && n > 0) {
    DevBuf<int32_t> cA, cB;
    FJ_TRY(cA.alloc(n + 1, st));
    FJ_TRY(cB.alloc(n + 1, st));
    const unsigned cb1 = (unsigned)std::min<int64_t>((n + 256) / 256, 8192);
    k_rows_plan3<<<cb1, 256, 0, st>>>(n, R.rp32, R.off, R.long_row, cA.p, cB.p);
    FJ_CK_LAUNCH();
    FJ_TRY(ralloc(&R.rpA, n + 1, st));
    FJ_TRY(ralloc(&R.rpB, n + 1, st));
    size_t tb = 0;
    FJ_CK(cub::DeviceScan::ExclusiveSum(nullptr, tb, cA.p, R.rpA, n + 1, st));
    DevBuf<uint8_t> tmp;
    FJ_TRY(tmp.alloc((int64_t)tb, st));
    FJ_CK(cub::DeviceScan::ExclusiveSum(tmp.p, tb, cA.p, R.rpA, n + 1, st));
    FJ_CK(cub::DeviceScan::ExclusiveSum(tmp.p, tb, cB.p, R.rpB, n + 1, st));
    count_cub();
    count_cub();
    int32_t tot[2] = {0, 0};
    FJ_CK(cudaMemcpyAsync(&tot[0], R.rpA + n, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    FJ_CK(cudaMemcpyAsync(&tot[1], R.rpB + n, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    FJ_CK(cudaStreamSynchronize(st));
    FJ_TRY(ralloc(&R.colA, tot[0], st));
    FJ_TRY(ralloc(&R.colB, tot[1], st));
    const int wsz = wtype == FJ_W_U8 ? 1 : wtype == FJ_W_F32 ? 4 : wtype == FJ_W_F64 ? 8 : 0;
    if (wsz) {
      FJ_TRY(ralloc(reinterpret_cast<uint8_t**>(&R.wA), (int64_t)tot[0] * wsz, st));
      FJ_TRY(ralloc(reinterpret_cast<uint8_t**>(&R.wB), (int64_t)tot[1] * wsz, st));
    }
    const unsigned cb4 = (unsigned)std::min<int64_t>((n * 32 + 255) / 256, (int64_t)num_sms * 64);
    auto copy = [&](auto tag) {
      using T = typename decltype(tag)::type;
      k_rows_plan4<T><<<cb4, 256, 0, st>>>(n, R.rp32, R.off, col, w, R.rpA, R.rpB, R.colA, R.colB, R.wA, R.wB);
    };
    switch (wsz) {
      case 1: copy(WTag<uint8_t>()); break;
      case 4: copy(WTag<float>()); break;
      case 8: copy(WTag<double>()); break;
      default: copy(WTag<void>()); break;
    }
    FJ_CK_LAUNCH();
  }
  FJ_TRY(ralloc(&R.tab, 2 * R.n_chunks, st));
  FJ_TRY(ralloc(&R.chunk_acc, 4 * R.n_chunks, st));
  FJ_TRY(ralloc(&R.op_acc, ROWS_NA_MAX * R.n_chunks, st));
  if (R.n_chunks > 0) {
    k_rows_plan2<<<cb, 256, 0, st>>>(n, row_ptr, nch.p, R.c0, R.tab);
    FJ_CK_LAUNCH();
  }
  int occ = 0;
  FJ_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_rows<FJ_W_UNIT, 4, 3, 2>, RTB, 0));
  if (occ < 1) occ = 1;
  // Grid: `waves` x the resident blocks, waves = rows / (8 x resident row groups) clamped to [1, 4]
  // (measured, profiles/r02_ab_rows_variants.log: C3 (4e6 rows) 4 waves 0.496 ms vs 1 wave 0.514;
  // C2 (1e6 rows) 1 wave 61.5 us vs 4 waves 71 us).  FJ_ROWS_WAVES > 0 fixes it (A/B).
#ifndef FJ_ROWS_WAVES
#define FJ_ROWS_WAVES 0
#endif
  const int64_t resident_groups = (int64_t)num_sms * occ * (RTB / FJ_ROWS_G);
  const int64_t waves = FJ_ROWS_WAVES > 0 ? FJ_ROWS_WAVES
                                          : std::max<int64_t>(1, std::min<int64_t>(4, n / (8 * resident_groups)));
  int64_t grid = (int64_t)num_sms * occ * waves;
  const int64_t need = (n * FJ_ROWS_G + RTB - 1) / RTB;
  if (grid > need) grid = need > 0 ? need : 1;
  R.grid = (int)grid;
  R.grid_chunks = (int)std::max<int64_t>(1, std::min<int64_t>((R.n_chunks * 32 + RTB - 1) / RTB, (int64_t)num_sms * 8));
  FJ_TRY(ralloc(&R.part, 4 * grid, st));
  FJ_TRY(ralloc(&R.ticket, 1, st));
  FJ_CK(cudaMemsetAsync(R.ticket, 0, sizeof(unsigned int), st));
  R.grid_op_max = num_sms * (2048 / RTB);
  FJ_TRY(ralloc(&R.op_part, (int64_t)ROWS_NP_MAX * R.grid_op_max, st));
  FJ_TRY(ralloc(&R.op_ticket, 1, st));
  FJ_CK(cudaMemsetAsync(R.op_ticket, 0, sizeof(unsigned int), st));
  R.mode = two ? 2 : 1;
  return FJ_OK;
}

fj_status rows_plan_build(fj_graph* g, int kp, RowsPlan& R, cudaStream_t st) {
  if (g->dist) { rows_plan_free(R); return FJ_OK; }   // the distributed path plans its own views
  return plan_core(g->n, g->nnz, g->row_ptr, g->col, kp, g->num_sms, true, g->w, g->wtype, R, st);
}

fj_status rows_plan_build_csr(int64_t n, int64_t nnz, const int64_t* row_ptr, const int32_t* col, int kp,
                              int num_sms, RowsPlan& R, cudaStream_t st) {
  return plan_core(n, nnz, row_ptr, col, kp, num_sms, false, nullptr, FJ_W_UNIT, R, st);
}

}  // namespace fj

// tiles.cuh — the load-balanced CSR row engine shared by the SpMV (q = (I+L)p), the true residual
// and the fused quantities pass.  DESIGN.md §Kernels "warp-item engine".
//
// Work items (built once per graph in graph.cu), each processed by ONE WARP, independently of the
// other warps (no block barriers on the hot loop, so warps hide each other's latency):
//   T  tile  : a run of <= 32 consecutive short rows (<= T_ROW_MAX nonzeros each) with <= ~576
//              nonzeros.  The warp loads the tile's col indices coalesced, gathers x[col] (up to
//              18 independent loads per lane), stages them in its shared-memory slice, then each
//              lane reduces one row.
//   W  row   : one row with T_ROW_MAX < len <= CHUNK nonzeros, lanes stride, shuffle reduction.
//   C  chunk : CHUNK nonzeros of a row longer than CHUNK.  The warp that finishes a row's last
//              chunk (atomic ticket) merges the chunk partials IN CHUNK ORDER and finishes the row.
// Items are assigned to warps round-robin over a FIXED grid, so every partial sum is formed in a
// fixed order and reduced in a fixed order: results are bitwise reproducible run to run.
#pragma once
#include <climits>
#include <type_traits>

#include "common.cuh"

namespace fj {

constexpr int WTPB = 128;                 // 4 warps per block
constexpr int WPB = WTPB / 32;
constexpr int ITEMS = 12;                 // merge items (row ends + nonzeros) per lane in a T tile
constexpr int T_CAP = 32 * ITEMS;         // 384 merge items per tile
constexpr int T_ROW_MAX = 64;             // rows longer than this are W rows or chunked
constexpr int T_ROW_MIN_COST = 12;        // schedule units per row are max(1 + len, 12): <= 32 rows
constexpr int T_UNITS = T_CAP - (T_ROW_MAX + 1);   // 319: a tile holds <= T_CAP merge items
constexpr int CHUNK = 2048;               // nonzeros per W row (max) / per long-row chunk
constexpr int IT_T = 0, IT_W = 1, IT_C = 2;

struct ItemMeta {   // 16 bytes
  int32_t r0;
  uint32_t info;    // type << 30 | (T: nrows | nk << 6) | (W: nk) | (C: long-row index)
  int64_t k0;
};

struct TileSched {
  int64_t n;
  const int64_t* __restrict__ row_ptr;
  const int32_t* __restrict__ col;
  const void* __restrict__ w;
  const ItemMeta* __restrict__ items;
  int64_t n_items;
  const int32_t* __restrict__ long_nchunks;   // [n_long]
  const int32_t* __restrict__ long_item0;     // [n_long] item index of chunk 0
  int64_t n_long, n_chunks;
  int chunk;                                  // nonzeros per long-row chunk
};

inline TileSched make_sched(const fj_graph* g, const Sched& S) {
  TileSched s;
  s.n = g->n; s.row_ptr = g->row_ptr; s.col = g->col; s.w = g->w;
  s.items = reinterpret_cast<const ItemMeta*>(S.items);
  s.n_items = S.n_items;
  s.long_nchunks = S.long_nchunks; s.long_item0 = S.long_item0;
  s.n_long = S.n_long; s.n_chunks = S.n_long_chunks;
  s.chunk = S.chunk;
  return s;
}

// the k = 1 engine's schedule (ITEMS x 32 lanes = T_CAP merge items per tile)
constexpr SchedParams kSchedK1{T_ROW_MAX, T_UNITS, T_ROW_MIN_COST, CHUNK};
fj_status build_schedule(fj_graph* g, const SchedParams& P, Sched& out, cudaStream_t st);
void free_sched(Sched& s);

// Scratch for the cross-warp parts of a launch (device memory, owned by the workspace).
struct TileScratch {
  double* block_part;          // [max grid][NP]
  double* long_part;           // [n_long][NP]
  double* chunk_acc;           // [n_chunks][NA]
  unsigned int* long_ticket;   // [n_long], zero-initialised, self-resetting
  unsigned int* grid_ticket;   // [1], zero-initialised, self-resetting
};

// Op interface:
//   static constexpr int NA, NP; static constexpr bool NEEDS_XI;
//   __device__ bool skip() const;                  // uniform early exit (solver finished)
//   __device__ double gather(int32_t j) const;     // x_j for a nonzero (i, j)
//   __device__ double row_value(int64_t i) const;  // x_i
//   __device__ void add(double (&a)[NA], double w, double xj, double xi) const;
//   __device__ void finish_row(int64_t i, int64_t len, double xi, const double (&a)[NA], double (&part)[NP]) const;
//   __device__ void finalize(const double (&tot)[NP]) const;   // single thread of the last block

// Merge-path split (Merrill & Garland): on the merge of the row-end offsets A[0..R) with the nonzero
// indices 0..N-1, the number of row ends consumed before diagonal d.
__device__ __forceinline__ int merge_rows_before(int d, const int32_t* A, int R, int N) {
  int lo = max(d - N, 0), hi = min(d, R);
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (A[mid] <= d - mid - 1) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// One T tile, one warp.  Every lane owns ITEMS consecutive merge items (row ends + nonzeros) of
// the tile: it gathers its <= ITEMS values with independent loads, walks them finishing every row
// that ends inside its range, and hands the partial of the row it ends inside to the next lanes
// (warp segmented scan).  No shared-memory reduction, no idle lanes on ragged rows.
template <int WT, class Op>
__device__ __forceinline__ void t_tile(const TileSched& sc, const Op& op, const ItemMeta& cur, int lane,
                                       int32_t* s_e, int32_t* s_col, double* s_xi,
                                       double (&part)[Op::NP]) {
  constexpr int NA = Op::NA;
  constexpr bool WEIGHTED = (WT != FJ_W_UNIT);
  const int R = cur.info & 63;
  const int N = (cur.info >> 6) & 0xFFFFF;
  const int64_t r0 = cur.r0, k0 = cur.k0;
  if (lane < R) {
    s_e[lane] = (int32_t)(__ldg(sc.row_ptr + r0 + lane + 1) - k0);
    s_xi[lane] = op.row_value(r0 + lane);
  }
#pragma unroll
  for (int u = 0; u < ITEMS; ++u) {
    const int k = lane + 32 * u;
    if (k < N) s_col[k] = __ldg(sc.col + k0 + k);
  }
  __syncwarp();
  const int M = R + N;
  const int d0 = min(lane * ITEMS, M), d1 = min(d0 + ITEMS, M);
  const int row_s = merge_rows_before(d0, s_e, R, N);
  const int row_n = __shfl_down_sync(0xffffffffu, row_s, 1);    // next lane's split = this lane's end
  const int row_e = lane == 31 ? R : row_n;
  const int nz_s = d0 - row_s, nz_e = d1 - row_e;
  using WS = typename std::conditional<WT == FJ_W_F64, double, float>::type;   // exact for u8 / f32
  double xv[ITEMS];
  WS wv[ITEMS];
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) {
    const int k = nz_s + j;
    xv[j] = 0.0;
    wv[j] = 1.0;
    if (k < nz_e) {
      xv[j] = op.gather(s_col[k]);
      if (WEIGHTED) wv[j] = (WS)WeightT<WT>::get(sc.w, k0 + k);
    }
  }
  double a[NA], a_first[NA];
#pragma unroll
  for (int f = 0; f < NA; ++f) { a[f] = 0.0; a_first[f] = 0.0; }
  bool has_first = false;
  int row = row_s;
  int re = row < R ? s_e[row] : INT_MAX;
  double xi = row < R ? s_xi[row] : 0.0;
  auto close_row = [&](int r) {
    if (r == row_s) {           // may have started in earlier lanes: finish after the carry scan
      has_first = true;
#pragma unroll
      for (int f = 0; f < NA; ++f) a_first[f] = a[f];
    } else {
      const int rb = r == 0 ? 0 : s_e[r - 1];
      op.finish_row(r0 + r, s_e[r] - rb, s_xi[r], a, part);
    }
#pragma unroll
    for (int f = 0; f < NA; ++f) a[f] = 0.0;
  };
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) {
    const int k = nz_s + j;
    if (k < nz_e) {
      while (row < row_e && re <= k) {
        close_row(row);
        ++row;
        re = row < R ? s_e[row] : INT_MAX;
        xi = row < R ? s_xi[row] : 0.0;
      }
      op.add(a, (double)wv[j], xv[j], xi);
    }
  }
  while (row < row_e) {
    close_row(row);
    ++row;
  }
  // a = partial of row `row_e` (continues in later lanes); segmented inclusive scan by row key
  int key = row_e;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int kup = __shfl_up_sync(0xffffffffu, key, off);
#pragma unroll
    for (int f = 0; f < NA; ++f) {
      const double v = __shfl_up_sync(0xffffffffu, a[f], off);
      if (lane >= off && kup == key) a[f] += v;
    }
  }
  // carry into this lane's first finished row = scanned partial of the previous lane
#pragma unroll
  for (int f = 0; f < NA; ++f) {
    const double cin = __shfl_up_sync(0xffffffffu, a[f], 1);
    if (lane > 0) a_first[f] += cin;
  }
  if (has_first) {
    const int rb = row_s == 0 ? 0 : s_e[row_s - 1];
    op.finish_row(r0 + row_s, s_e[row_s] - rb, s_xi[row_s], a_first, part);
  }
  __syncwarp();
}

template <int WT, class Op>
__global__ void __launch_bounds__(WTPB) warp_kernel(const TileSched sc, const Op op, const TileScratch ws) {
  constexpr int NA = Op::NA, NP = Op::NP;
  constexpr bool WEIGHTED = (WT != FJ_W_UNIT);
  __shared__ int32_t s_col[WPB][T_CAP];
  __shared__ int32_t s_e[WPB][32];
  __shared__ double s_xi[WPB][32];
  __shared__ double s_red[(NP > NA ? NP : NA) * WPB];
  __shared__ bool s_last;

  if (op.skip()) return;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  double part[NP];
#pragma unroll
  for (int j = 0; j < NP; ++j) part[j] = 0.0;

  const int64_t nwarps = (int64_t)gridDim.x * WPB;
  int64_t it = (int64_t)blockIdx.x * WPB + wib;
  ItemMeta m{};
  if (it < sc.n_items) m = sc.items[it];
  for (; it < sc.n_items; it += nwarps) {
    const ItemMeta cur = m;
    if (it + nwarps < sc.n_items) m = sc.items[it + nwarps];   // prefetch the next item's meta
    const uint32_t type = cur.info >> 30;
    if (type == IT_T) {
      t_tile<WT, Op>(sc, op, cur, lane, s_e[wib], s_col[wib], s_xi[wib], part);
    } else {
      // ------------------------------------------------ W row or C chunk: lanes stride
      const int64_t r = cur.r0;
      const int64_t rb = __ldg(sc.row_ptr + r), re = __ldg(sc.row_ptr + r + 1);
      const int64_t kb = cur.k0;
      const int64_t ke = (type == IT_W) ? re : min(kb + (int64_t)sc.chunk, re);
      const double xi = op.row_value(r);
      double a[NA];
#pragma unroll
      for (int f = 0; f < NA; ++f) a[f] = 0.0;
      for (int64_t k = kb + lane; k < ke; k += 32 * 8) {
        int32_t c8[8];
        double w8[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int64_t kk = k + 32 * u;
          c8[u] = kk < ke ? __ldg(sc.col + kk) : -1;
          w8[u] = (WEIGHTED && kk < ke) ? WeightT<WT>::get(sc.w, kk) : 1.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (c8[u] >= 0) op.add(a, w8[u], op.gather(c8[u]), xi);
      }
#pragma unroll
      for (int f = 0; f < NA; ++f) a[f] = warp_sum(a[f]);
      if (type == IT_W) {
        if (lane == 0) op.finish_row(r, re - rb, xi, a, part);
      } else {
        const uint32_t l = cur.info & 0x3FFFFFFFu;
        const int64_t first = sc.long_item0[l];
        const int32_t nch = sc.long_nchunks[l];
        bool last = false;
        if (lane == 0) {
#pragma unroll
          for (int f = 0; f < NA; ++f) ws.chunk_acc[it * NA + f] = a[f];
          __threadfence();
          last = atomicAdd(ws.long_ticket + l, 1u) == (unsigned)nch - 1u;
          if (last) {
            __threadfence();
            double acc[NA];
#pragma unroll
            for (int f = 0; f < NA; ++f) acc[f] = 0.0;
            for (int32_t c = 0; c < nch; ++c) {
#pragma unroll
              for (int f = 0; f < NA; ++f) acc[f] += ld_cg(ws.chunk_acc + (first + c) * NA + f);
            }
            double lp[NP];
#pragma unroll
            for (int j = 0; j < NP; ++j) lp[j] = 0.0;
            op.finish_row(r, re - rb, xi, acc, lp);
#pragma unroll
            for (int j = 0; j < NP; ++j) ws.long_part[(int64_t)l * NP + j] = lp[j];
            ws.long_ticket[l] = 0u;
          }
        }
      }
    }
  }

  // ---------------------------------------------------- grid-level deterministic reduction
  block_sum<NP, WTPB>(part, s_red);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int j = 0; j < NP; ++j) ws.block_part[(int64_t)blockIdx.x * NP + j] = part[j];
    __threadfence();
    s_last = atomicAdd(ws.grid_ticket, 1u) == gridDim.x - 1u;
  }
  __syncthreads();
  if (s_last) {
    __threadfence();
    double tot[NP];
#pragma unroll
    for (int j = 0; j < NP; ++j) tot[j] = 0.0;
    for (int64_t q = threadIdx.x; q < (int64_t)gridDim.x; q += WTPB) {
#pragma unroll
      for (int j = 0; j < NP; ++j) tot[j] += ld_cg(ws.block_part + q * NP + j);
    }
    for (int64_t q = threadIdx.x; q < sc.n_long; q += WTPB) {
#pragma unroll
      for (int j = 0; j < NP; ++j) tot[j] += ld_cg(ws.long_part + q * NP + j);
    }
    block_sum<NP, WTPB>(tot, s_red);
    if (threadIdx.x == 0) {
      op.finalize(tot);
      *ws.grid_ticket = 0u;
    }
  }
}

}  // namespace fj

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
#include <cstring>
#include <type_traits>

#include "common.cuh"

namespace fj {

constexpr int WTPB = 128;                 // 4 warps per block
constexpr int WPB = WTPB / 32;
#ifndef FJ_ITEMS
#define FJ_ITEMS 12
#endif
#ifndef FJ_K1_MIN_BLOCKS
#define FJ_K1_MIN_BLOCKS 0
#endif
// Register caps of the engine (__launch_bounds__ min blocks / SM) per gathered value width; 0 = no
// hint.  (A hint of 1 is NOT neutral: ptxas then spends registers on ILP -- 106 instead of 72 for
// k = 1, 25 % slower.)  Measured on B200 (C2, C3, C4): k = 1 best with no hint (72 regs, 7 blocks);
// KP = 4 at 4 blocks (128 regs, no spill) 1.2-1.5x faster than 160 regs / 3 blocks; KP = 2 at 5.
#ifndef FJ_K1_TMA
#define FJ_K1_TMA 0
#endif
#ifndef FJ_VEC_MIN_BLOCKS
#define FJ_VEC_MIN_BLOCKS 4
#endif
#ifndef FJ_QUANTV_MIN_BLOCKS   // -1: 4 blocks/SM for unit weights and k <= 3, else 3 (no spills with
#define FJ_QUANTV_MIN_BLOCKS -1  // the partials in shared memory); 0: no hint
#endif
#ifndef FJ_VEC2_MIN_BLOCKS
#define FJ_VEC2_MIN_BLOCKS 5
#endif
template <class V>
constexpr int engine_min_blocks() {
  return sizeof(V) == 8 ? FJ_K1_MIN_BLOCKS : (sizeof(V) == 16 ? FJ_VEC2_MIN_BLOCKS : FJ_VEC_MIN_BLOCKS);
}
#ifndef FJ_VEC_ITEMS
#define FJ_VEC_ITEMS 10   // r02: 10 once the product carries only the KQ real columns (C3 k = 3
#endif                    // 0.643 -> 0.607 ms, C2 k = 2 80.6 -> 74.3 us; R-MAT k = 4 +3 %)
// Merge items (row ends + nonzeros) per lane in a T tile, per engine: the k = 1 operators use
// ITEMS (32 x 12 = 384 per tile); the vector operators (spmv_vec.cu) hold KP doubles per item and
// use VEC_ITEMS (32 x 10 = 320): 4 blocks / SM at 128 registers (12 overflows the quantities
// pass's 48 KB of static shared memory).
constexpr int ITEMS = FJ_ITEMS;
constexpr int VEC_ITEMS = FJ_VEC_ITEMS;
constexpr int T_ROW_MAX = 64;             // rows longer than this are W rows or chunked
template <int IT> constexpr int t_cap() { return 32 * IT; }
// a tile holds <= t_cap merge items: cut the merge coordinate every t_units = t_cap - (T_ROW_MAX + 1)
template <int IT> constexpr int t_units() { return t_cap<IT>() - (T_ROW_MAX + 1); }
// schedule units per row are max(1 + len, t_min_cost): <= TILE_ROWS rows per tile
// rows per T tile: up to ROWS (each lane stages ROWS / 32 row ends).  The scalar engine takes 64,
// which packs the short rows of power-law graphs (measured: C5 product 16.8 -> 15.8 ms, C2 61.6 ->
// 59.0 us); the vector engine keeps 32 (64 cost it 28 % on C3: larger shared staging per block).
#ifndef FJ_TILE_ROWS
#define FJ_TILE_ROWS 64
#endif
constexpr int TILE_ROWS = FJ_TILE_ROWS;   // scalar engine
constexpr int VEC_TILE_ROWS = 32;
template <int ROWS> constexpr int t_min_cost_floor() { return ROWS == 32 ? 12 : 6; }
template <int IT, int ROWS> constexpr int t_min_cost() {
  return (t_units<IT>() + ROWS - 2) / (ROWS - 1) > t_min_cost_floor<ROWS>()
             ? (t_units<IT>() + ROWS - 2) / (ROWS - 1) : t_min_cost_floor<ROWS>();
}
constexpr int T_CAP = t_cap<ITEMS>();
constexpr int CHUNK = 2048;               // nonzeros per W row (max) / per long-row chunk
constexpr int IT_T = 0, IT_W = 1, IT_C = 2;

struct ItemMeta {   // 16 bytes
  int32_t r0;
  uint32_t info;    // type << 30 | (T: nrows | nk << 7) | (W: nk) | (C: long-row index)
  int64_t k0;
};
__host__ __device__ __forceinline__ int tile_rows(uint32_t info) { return (int)(info & 127u); }
__host__ __device__ __forceinline__ int tile_nnz(uint32_t info) { return (int)((info >> 7) & 0x7FFFFu); }

struct TileSched {
  int64_t n, nnz;
  int64_t ncol;                               // gathered rows: n, or n_loc + ghosts on a rank
  const int64_t* __restrict__ row_ptr;
  const int32_t* __restrict__ col;
  const void* __restrict__ w;
  const ItemMeta* __restrict__ items;
  int64_t n_items;
  const int32_t* __restrict__ long_nchunks;   // [n_long]
  const int32_t* __restrict__ long_item0;     // [n_long] item index of chunk 0
  int64_t n_long, n_chunks;
  int chunk;                                  // nonzeros per long-row chunk
  int hint;                                   // bit 1: disable the TMA tile prefetch (FJ_L2_HINT=2)
};

// Loads of the CSR streams outside the TMA prefetch.  (An evict-first .cs variant was measured
// 25 % slower on C2 and is not used.)
__device__ __forceinline__ int32_t ld_col(const TileSched& sc, int64_t p) { return __ldg(sc.col + p); }
__device__ __forceinline__ int64_t ld_rp(const TileSched& sc, int64_t i) { return __ldg(sc.row_ptr + i); }

int64_t dist_n_ghost(const fj_graph* g);   // dist.cu
inline TileSched make_sched(const fj_graph* g, const Sched& S) {
  TileSched s;
  s.n = g->n; s.nnz = g->nnz;
  s.ncol = g->n + dist_n_ghost(g); s.row_ptr = g->row_ptr; s.col = g->col; s.w = g->w;
  s.items = reinterpret_cast<const ItemMeta*>(S.items);
  s.n_items = S.n_items;
  s.long_nchunks = S.long_nchunks; s.long_item0 = S.long_item0;
  s.n_long = S.n_long; s.n_chunks = S.n_long_chunks;
  s.chunk = S.chunk;
  s.hint = l2_hint();
  return s;
}

// the k = 1 engine's schedule (ITEMS x 32 lanes = T_CAP merge items per tile)
template <int IT, int ROWS> constexpr SchedParams sched_params() {
  return SchedParams{T_ROW_MAX, t_units<IT>(), t_min_cost<IT, ROWS>(), CHUNK};
}
constexpr SchedParams kSchedK1 = sched_params<ITEMS, TILE_ROWS>();
constexpr SchedParams kSchedVec = sched_params<VEC_ITEMS, VEC_TILE_ROWS>();
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
//   using V;                                       // gathered value: double (k = 1) or DVec<KP> (k <= 4)
//   static constexpr int ITEMS;                    // merge items per lane (the schedule's t_cap / 32)
//   static constexpr int TILE_ROWS;                // rows per T tile (32 or 64; the schedule's)
//   static constexpr int MIN_BLOCKS;               // __launch_bounds__ min blocks / SM (register cap)
//   static constexpr bool TMA;                     // stage tiles by the TMA bulk-copy prefetch
//   static constexpr int NA, NP; static constexpr bool NEEDS_XI;   // NEEDS_XI: add() reads x_i
//   static __device__ V vzero();
//   __device__ bool skip() const;                  // uniform early exit (solver finished)
//   __device__ V gather(int32_t j) const;          // x_j for a nonzero (i, j)
//   __device__ V row_value(int64_t i) const;       // x_i
//   __device__ const V* xi_base() const;           // x_i = xi_base()[i] (contiguous), or nullptr
//   __device__ bool wants_xi() const;              // false: x_i unused by finish_row (not loaded)
//   __device__ void add(double (&a)[NA], double w, V xj, V xi) const;
//   template <class P>                             // P: double[NP] or PartStore (part[j] += ...)
//   __device__ void finish_row(int64_t i, int64_t len, V xi, const double (&a)[NA], P& part) const;
//   static constexpr bool PART_SMEM;               // optional: per-thread partials in shared memory
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
// Tile inputs staged by the TMA bulk-copy prefetch (warp_kernel): the tile's col indices, row_ptr
// entries and row values already sit in shared memory (null members: load them here).
// Per-thread partial sums of finish_row: registers, or (Op::PART_SMEM, for operators with many
// partials) a [NP][WTPB] shared-memory column per thread, freeing 2 NP registers in the main loop.
template <class Op, class = void>
struct PartSmemT : std::false_type {};
template <class Op>
struct PartSmemT<Op, std::void_t<decltype(Op::PART_SMEM)>> : std::integral_constant<bool, Op::PART_SMEM> {};
template <int NP, bool SMEM>
struct PartStore {
  double v[NP];
  __device__ __forceinline__ double& operator[](int j) { return v[j]; }
};
template <int NP>
struct PartStore<NP, true> {
  double* b;   // s_part + threadIdx.x, stride WTPB
  __device__ __forceinline__ double& operator[](int j) { return b[j * WTPB]; }
};

// Deferred row finish (r02): rows that close inside a lane's merge range park their sums in a
// per-warp shared-memory slot instead of running finish_row at the close (divergent: 1-2 lanes
// active, ~10 times per tile); after the carry scan lane r finishes row r of the tile, all lanes
// together, and the row results are stored coalesced.  Used when the slots fit FJ_DEFER_BYTES per
// block.  FJ_DEFER: 0 off, 1 every operator, 2 (default) operators without the TMA tile staging
// (the scalar k = 1 engine).  Measured (profiles/r02_ab_defer_prefetch.log): k = 1 C2 product
// 58.1 -> 53.6 us; but the k = 3 C3 product 0.611 -> 0.690 ms, whose gathers miss L2: the finish
// work done at the row closes overlaps the gathers still in flight, deferred it does not.
#ifndef FJ_DEFER
#define FJ_DEFER 2
#endif
#ifndef FJ_DEFER_BYTES
#define FJ_DEFER_BYTES 4096
#endif
template <class Op>
constexpr bool defer_finish() {
  return (FJ_DEFER == 1 || (FJ_DEFER == 2 && !Op::TMA)) && Op::TILE_ROWS * Op::NA * 8 * WPB <= FJ_DEFER_BYTES;
}

template <class V>
struct TilePre {
  const int32_t* col;     // col[k0 .. k0+N)
  const int64_t* rp;      // row_ptr[r0+1 .. r0+R]
  const V* xi;            // x[r0 .. r0+R)
};

template <int WT, class Op, bool PRE, class P>
__device__ __forceinline__ void t_tile(const TileSched& sc, const Op& op, const ItemMeta& cur, int lane,
                                       int32_t* s_e, int32_t* s_col_own, typename Op::V* s_xi_own,
                                       double* s_acc, P& part, const TilePre<typename Op::V>& pre) {
  using V = typename Op::V;
  constexpr int NA = Op::NA;
  constexpr int ITEMS = Op::ITEMS;
  constexpr bool WEIGHTED = (WT != FJ_W_UNIT);
  const int R = tile_rows(cur.info);
  const int N = tile_nnz(cur.info);
  const int64_t r0 = cur.r0, k0 = cur.k0;
  FJ_DCHECK(R >= 1 && R <= Op::TILE_ROWS && N >= 0 && R + N <= 32 * Op::ITEMS);
  FJ_DCHECK(r0 >= 0 && r0 + R <= sc.n && k0 >= 0 && k0 + N <= sc.nnz);
  const int32_t* s_col = (PRE && pre.col) ? pre.col : s_col_own;
  const V* s_xi = (PRE && pre.xi) ? pre.xi : s_xi_own;
#pragma unroll
  for (int rr = lane; rr < Op::TILE_ROWS; rr += 32) {
    if (rr < R) {
      s_e[rr] = (int32_t)(((PRE && pre.rp) ? pre.rp[rr] : ld_rp(sc, r0 + rr + 1)) - k0);
      if (!(PRE && pre.xi) && op.wants_xi()) s_xi_own[rr] = op.row_value(r0 + rr);
    }
  }
  if (!(PRE && pre.col)) {
#pragma unroll
    for (int u = 0; u < ITEMS; ++u) {
      const int k = lane + 32 * u;
      if (k < N) s_col_own[k] = ld_col(sc, k0 + k);
    }
  }
  __syncwarp();
  const int M = R + N;
  const int d0 = min(lane * ITEMS, M), d1 = min(d0 + ITEMS, M);
  const int row_s = merge_rows_before(d0, s_e, R, N);
  const int row_n = __shfl_down_sync(0xffffffffu, row_s, 1);    // next lane's split = this lane's end
  const int row_e = lane == 31 ? R : row_n;
  const int nz_s = d0 - row_s, nz_e = d1 - row_e;
  using WS = typename std::conditional<WT == FJ_W_F64, double, float>::type;   // exact for u8 / f32
  V xv[ITEMS];
  WS wv[ITEMS];
#pragma unroll
  for (int j = 0; j < ITEMS; ++j) {
    const int k = nz_s + j;
    xv[j] = Op::vzero();
    wv[j] = 1.0;
    if (k < nz_e) {
      FJ_DCHECK(s_col[k] >= 0 && s_col[k] < sc.ncol);
      xv[j] = op.gather(s_col[k]);
      if (WEIGHTED) wv[j] = (WS)WeightT<WT>::get(sc.w, k0 + k);
    }
  }
  double a[NA], a_first[NA];
#pragma unroll
  for (int f = 0; f < NA; ++f) { a[f] = 0.0; a_first[f] = 0.0; }
  bool has_first = false;
  int row = row_s;
  // the next row end inside this lane's range (rows [row_s, row_e) end here; the row it ends inside
  // continues in later lanes: INT_MAX), so the per-nonzero test is one compare
  int re = row < row_e ? s_e[row] : INT_MAX;
  V xi = Op::vzero();   // x_i for operators whose add() uses it (NEEDS_XI)
  if constexpr (Op::NEEDS_XI) xi = row < R ? s_xi[row] : Op::vzero();
  constexpr bool DEFER = defer_finish<Op>();
  auto close_row = [&](int r) {
    if (r == row_s) {           // may have started in earlier lanes: finish after the carry scan
      has_first = true;
#pragma unroll
      for (int f = 0; f < NA; ++f) a_first[f] = a[f];
    } else if constexpr (DEFER) {
#pragma unroll
      for (int f = 0; f < NA; ++f) s_acc[r * NA + f] = a[f];
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
      while (re <= k) {
        close_row(row);
        ++row;
        re = row < row_e ? s_e[row] : INT_MAX;
        if constexpr (Op::NEEDS_XI) xi = row < R ? s_xi[row] : Op::vzero();
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
    if constexpr (DEFER) {
#pragma unroll
      for (int f = 0; f < NA; ++f) s_acc[row_s * NA + f] = a_first[f];
    } else {
      const int rb = row_s == 0 ? 0 : s_e[row_s - 1];
      op.finish_row(r0 + row_s, s_e[row_s] - rb, s_xi[row_s], a_first, part);
    }
  }
  if constexpr (DEFER) {   // every row of the tile was parked by exactly one lane
    __syncwarp();
#pragma unroll
    for (int rr = lane; rr < Op::TILE_ROWS; rr += 32) {
      if (rr < R) {
        double acc[NA];
#pragma unroll
        for (int f = 0; f < NA; ++f) acc[f] = s_acc[rr * NA + f];
        const int rb = rr == 0 ? 0 : s_e[rr - 1];
        op.finish_row(r0 + rr, s_e[rr] - rb, s_xi[rr], acc, part);
      }
    }
  }
  __syncwarp();
}

#ifndef FJ_TMA_PREFETCH
#define FJ_TMA_PREFETCH 1
#endif
#ifndef FJ_SLOT_STAGE
#define FJ_SLOT_STAGE 1
#endif
// ---------------------------------------------------------------- TMA bulk-copy tile prefetch
// While a warp works on one T tile, the TMA engine copies the NEXT tile's three contiguous input
// ranges (col indices, row_ptr entries, row values) global -> shared (cp.async.bulk, completion on
// a per-warp mbarrier, two slots).  The CSR stream latency then overlaps the current tile's gathers
// instead of stalling the warp at the start of every tile.  Copies are 16-byte granular: each range
// is widened to 16-byte boundaries (never past the array's last full 16-byte unit; such a tile,
// and any tile whose base pointers are not 16-byte aligned, takes the plain-load path).
template <class Op>
struct PfSlot {   // [cols | row_ptr | row values] of one tile
  static constexpr int COL_BYTES = t_cap<Op::ITEMS>() * 4 + 32;
  static constexpr int RP_BYTES = Op::TILE_ROWS * 8 + 32;
  static constexpr int XI_BYTES = Op::TILE_ROWS * (int)sizeof(typename Op::V) + 32;
  static constexpr int BYTES = ((COL_BYTES + RP_BYTES + XI_BYTES) + 15) & ~15;
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile("{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
               " @!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}

struct PfRange {   // one widened 16-byte-granular copy [b0, b1) of an array, in bytes from its base
  int64_t b0, b1;
};
__device__ __forceinline__ PfRange pf_range(int64_t byte_begin, int64_t byte_end) {
  return PfRange{byte_begin & ~(int64_t)15, (byte_end + 15) & ~(int64_t)15};
}

// Per-kernel limits (uniform): last full 16-byte unit of each array, or -1 if its base is unaligned.
struct PfLimits {
  int64_t col, rp, xi;
};

template <class Op>
__device__ __forceinline__ bool pf_ok(const TileSched& sc, const Op& op, const ItemMeta& m, const PfLimits& L) {
  using V = typename Op::V;
  if ((m.info >> 30) != IT_T || L.col < 0 || L.rp < 0) return false;
  const int R = tile_rows(m.info), N = tile_nnz(m.info);
  const PfRange c = pf_range(4 * m.k0, 4 * (m.k0 + N));
  const PfRange r = pf_range(8 * ((int64_t)m.r0 + 1), 8 * ((int64_t)m.r0 + R + 1));
  if (c.b1 > L.col || r.b1 > L.rp) return false;
  if (L.xi >= 0) {
    const PfRange x = pf_range((int64_t)sizeof(V) * m.r0, (int64_t)sizeof(V) * (m.r0 + R));
    if (x.b1 > L.xi) return false;
  }
  return true;
}

// lane 0 only: arm the slot's barrier and issue the (up to) three bulk copies of tile m.
template <class Op>
__device__ __forceinline__ void pf_issue(const TileSched& sc, const Op& op, const ItemMeta& m, const PfLimits& L,
                                         unsigned char* slot, uint64_t* bar) {
  using V = typename Op::V;
  const int R = tile_rows(m.info), N = tile_nnz(m.info);
  const PfRange c = pf_range(4 * m.k0, 4 * (m.k0 + N));
  const PfRange r = pf_range(8 * ((int64_t)m.r0 + 1), 8 * ((int64_t)m.r0 + R + 1));
  PfRange x{0, 0};
  if (L.xi >= 0) x = pf_range((int64_t)sizeof(V) * m.r0, (int64_t)sizeof(V) * (m.r0 + R));
  FJ_DCHECK(c.b1 - c.b0 <= PfSlot<Op>::COL_BYTES && r.b1 - r.b0 <= PfSlot<Op>::RP_BYTES &&
            x.b1 - x.b0 <= PfSlot<Op>::XI_BYTES);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic reads of the slot are done
  mbar_expect_tx(bar, (uint32_t)((c.b1 - c.b0) + (r.b1 - r.b0) + (x.b1 - x.b0)));
  if (c.b1 > c.b0)
    bulk_g2s(slot, reinterpret_cast<const unsigned char*>(sc.col) + c.b0, (uint32_t)(c.b1 - c.b0), bar);
  constexpr int PF_COL_BYTES = PfSlot<Op>::COL_BYTES;
  bulk_g2s(slot + PF_COL_BYTES, reinterpret_cast<const unsigned char*>(sc.row_ptr) + r.b0, (uint32_t)(r.b1 - r.b0),
           bar);
  if (x.b1 > x.b0)
    bulk_g2s(slot + PF_COL_BYTES + PfSlot<Op>::RP_BYTES, reinterpret_cast<const unsigned char*>(op.xi_base()) + x.b0,
             (uint32_t)(x.b1 - x.b0), bar);
}

// Pointers into a filled slot for tile m (byte shifts undo the 16-byte widening).
template <class Op>
__device__ __forceinline__ TilePre<typename Op::V> pf_view(const ItemMeta& m, const PfLimits& L,
                                                          unsigned char* slot) {
  using V = typename Op::V;
  constexpr int PF_COL_BYTES = PfSlot<Op>::COL_BYTES;
  TilePre<V> p;
  p.col = reinterpret_cast<const int32_t*>(slot + ((4 * m.k0) & 15));
  p.rp = reinterpret_cast<const int64_t*>(slot + PF_COL_BYTES + ((8 * ((int64_t)m.r0 + 1)) & 15));
  p.xi = L.xi >= 0 ? reinterpret_cast<const V*>(slot + PF_COL_BYTES + PfSlot<Op>::RP_BYTES +
                                                 (((int64_t)sizeof(V) * m.r0) & 15))
                   : nullptr;
  return p;
}

// W row or C chunk item (lanes stride over the row's nonzeros; chunk partials merged in chunk
// order by the warp that completes the row).
template <int WT, class Op, class P>
__device__ __forceinline__ void wc_item(const TileSched& sc, const Op& op, const TileScratch& ws, const ItemMeta& cur,
                                        int64_t it, int lane, P& part) {
  using V = typename Op::V;
  constexpr int NA = Op::NA, NP = Op::NP;
  constexpr bool WEIGHTED = (WT != FJ_W_UNIT);
  const uint32_t type = cur.info >> 30;
  // ------------------------------------------------ W row or C chunk: lanes stride
  const int64_t r = cur.r0;
  const int64_t rb = ld_rp(sc, r), re = ld_rp(sc, r + 1);
  const int64_t kb = cur.k0;
  const int64_t ke = (type == IT_W) ? re : min(kb + (int64_t)sc.chunk, re);
  const V xi = op.wants_xi() ? op.row_value(r) : Op::vzero();
  double a[NA];
#pragma unroll
  for (int f = 0; f < NA; ++f) a[f] = 0.0;
  for (int64_t k = kb + lane; k < ke; k += 32 * 8) {
    int32_t c8[8];
    double w8[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int64_t kk = k + 32 * u;
      c8[u] = kk < ke ? ld_col(sc, kk) : -1;
      w8[u] = (WEIGHTED && kk < ke) ? WeightT<WT>::get(sc.w, kk) : 1.0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      FJ_DCHECK(c8[u] < sc.ncol);
      if (c8[u] >= 0) op.add(a, w8[u], op.gather(c8[u]), xi);
    }
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

template <int WT, class Op>
__global__ void __launch_bounds__(WTPB, Op::MIN_BLOCKS) warp_kernel(const TileSched sc, const Op op, const TileScratch ws) {
  using V = typename Op::V;
  constexpr int NA = Op::NA, NP = Op::NP;
  constexpr bool TMA = Op::TMA && FJ_TMA_PREFETCH != 0;
  // with the TMA ring, a tile that was not prefetched stages its cols / row values in its own idle
  // slot, so the block needs no separate staging arrays (r02: C3 k = 3 engine 32.2 -> 23.0 KB of
  // shared memory per block).  Shared memory per block is a measured lever here: 6.6 KB MORE (any
  // use: a pad, a shared-memory carry, the deferred finish) made the C3 product 13 % slower at the
  // same occupancy and instruction count (more short-scoreboard stalls; profiles/r02_ab_smem.log)
  constexpr bool SLOT = TMA && FJ_SLOT_STAGE != 0;
  __shared__ int32_t s_col[WPB][SLOT ? 1 : t_cap<Op::ITEMS>()];
  __shared__ int32_t s_e[WPB][Op::TILE_ROWS];
  __shared__ V s_xi[WPB][SLOT ? 1 : Op::TILE_ROWS];
  __shared__ double s_acc[WPB][defer_finish<Op>() ? Op::TILE_ROWS * NA : 1];
  __shared__ double s_red[(NP > NA ? NP : NA) * WPB];
  __shared__ bool s_last;
  __shared__ __align__(128) unsigned char s_pf[WPB][TMA ? 2 : 1][TMA ? PfSlot<Op>::BYTES : 16];
  __shared__ uint64_t s_bar[WPB][2];

  pdl_prologue();   // solver iterations chain this kernel with PDL (no-op otherwise)
  if (op.skip()) return;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  constexpr bool PS = PartSmemT<Op>::value;
  __shared__ double s_part[PS ? NP * WTPB : 1];
  PartStore<NP, PS> part;
  if constexpr (PS) part.b = s_part + threadIdx.x;
#pragma unroll
  for (int j = 0; j < NP; ++j) part[j] = 0.0;

  if constexpr (!TMA) {   // scalar operators: plain loads, next item's meta one ahead
    const int64_t nwarps = (int64_t)gridDim.x * WPB;
    int64_t it = (int64_t)blockIdx.x * WPB + wib;
    ItemMeta m{};
    if (it < sc.n_items) m = sc.items[it];
    for (; it < sc.n_items; it += nwarps) {
      const ItemMeta cur = m;
      if (it + nwarps < sc.n_items) m = sc.items[it + nwarps];
      if ((cur.info >> 30) == IT_T) {
        const TilePre<V> pre{nullptr, nullptr, nullptr};
        t_tile<WT, Op, false>(sc, op, cur, lane, s_e[wib], s_col[wib], s_xi[wib], s_acc[wib], part, pre);
      } else {
        wc_item<WT, Op>(sc, op, ws, cur, it, lane, part);
      }
    }
  } else {
    PfLimits L;
    L.col = !TMA || (sc.hint & 2) || (reinterpret_cast<uintptr_t>(sc.col) & 15) ? -1 : ((4 * sc.nnz) & ~(int64_t)15);
    L.rp = (reinterpret_cast<uintptr_t>(sc.row_ptr) & 15) ? -1 : ((8 * (sc.n + 1)) & ~(int64_t)15);
    const V* xb = op.xi_base();
    L.xi = (!xb || !op.wants_xi() || (reinterpret_cast<uintptr_t>(xb) & 15)) ? -1
                                                                           : (((int64_t)sizeof(V) * sc.n) & ~(int64_t)15);
    if (TMA && lane == 0) {
      mbar_init(&s_bar[wib][0]);
      mbar_init(&s_bar[wib][1]);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();

    const int64_t nwarps = (int64_t)gridDim.x * WPB;
    int64_t it = (int64_t)blockIdx.x * WPB + wib;
    ItemMeta m{}, m1{};   // current and next item
    if (it < sc.n_items) m = sc.items[it];
    if (it + nwarps < sc.n_items) m1 = sc.items[it + nwarps];
    uint32_t pend = 0, par = 0;   // per slot: copy in flight / barrier phase parity
    int slot = 0;
    if (TMA && it < sc.n_items && pf_ok(sc, op, m, L)) {
      if (lane == 0) pf_issue(sc, op, m, L, s_pf[wib][0], &s_bar[wib][0]);
      pend = 1;
    }
    for (; it < sc.n_items; it += nwarps) {
      const ItemMeta cur = m;
      ItemMeta m2{};
      if (it + 2 * nwarps < sc.n_items) m2 = sc.items[it + 2 * nwarps];   // meta two items ahead
      if (TMA && it + nwarps < sc.n_items && pf_ok(sc, op, m1, L)) {       // stage the next tile
        __syncwarp();
        if (lane == 0) pf_issue(sc, op, m1, L, s_pf[wib][slot ^ 1], &s_bar[wib][slot ^ 1]);
        pend |= 1u << (slot ^ 1);
      }
      const uint32_t type = cur.info >> 30;
      if (type == IT_T) {
        TilePre<V> pre{nullptr, nullptr, nullptr};
        if (TMA && (pend & (1u << slot))) {
          mbar_wait(&s_bar[wib][slot], (par >> slot) & 1u);
          par ^= 1u << slot;
          pend &= ~(1u << slot);
          pre = pf_view<Op>(cur, L, s_pf[wib][slot]);
        }
        int32_t* own_col = s_col[wib];
        V* own_xi = s_xi[wib];
        if constexpr (SLOT) {   // this tile's slot: in use by its own TMA copy, or idle
          own_col = reinterpret_cast<int32_t*>(s_pf[wib][slot]);
          own_xi = reinterpret_cast<V*>(s_pf[wib][slot] + PfSlot<Op>::COL_BYTES + PfSlot<Op>::RP_BYTES);
        }
        if (pre.col) t_tile<WT, Op, true>(sc, op, cur, lane, s_e[wib], own_col, own_xi, s_acc[wib], part, pre);
        else t_tile<WT, Op, false>(sc, op, cur, lane, s_e[wib], own_col, own_xi, s_acc[wib], part, pre);
      } else {
        wc_item<WT, Op>(sc, op, ws, cur, it, lane, part);
      }
      m = m1;
      m1 = m2;
      slot ^= 1;
    }
  }

  // ---------------------------------------------------- grid-level deterministic reduction
  double pr[NP];
#pragma unroll
  for (int j = 0; j < NP; ++j) pr[j] = part[j];
  block_sum<NP, WTPB>(pr, s_red);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int j = 0; j < NP; ++j) ws.block_part[(int64_t)blockIdx.x * NP + j] = pr[j];
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

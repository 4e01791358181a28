// tiles.cuh — the load-balanced CSR row engine shared by the SpMV (q = (I+L)p) and the fused
// quantities pass.  DESIGN.md §Kernels "tile engine".
//
// Work items (built once per graph in graph.cu):
//   * long-row chunks: rows with > LONG_ROW nonzeros are cut into LONG_CHUNK-nonzero chunks; each
//     chunk is reduced by one block, the block that finishes a row last (atomic ticket) merges the
//     chunk partials IN CHUNK ORDER and finishes the row;
//   * tiles: maximal runs of short rows with <= TILE_UNITS merge units (4 per row + 1 per
//     nonzero), i.e. <= 256 rows and <= 2048 nonzeros.  A block stages the tile's gathered
//     x[col] values in shared memory with coalesced col loads (8 independent gathers per thread),
//     then reduces rows: one thread per row of <= 32 nonzeros, one warp per longer row.
// Items are assigned to a fixed grid round-robin (static), so every partial sum is formed in a
// fixed order: results are bitwise reproducible run to run.
#pragma once
#include "common.cuh"

namespace fj {

struct TileSched {
  int64_t n;
  const int64_t* __restrict__ row_ptr;
  const int32_t* __restrict__ col;
  const void* __restrict__ w;
  const int32_t* __restrict__ tile_begin;
  const int32_t* __restrict__ tile_end;
  const int32_t* __restrict__ long_row;
  const int32_t* __restrict__ chunk_row;
  const int32_t* __restrict__ chunk_idx;
  const int32_t* __restrict__ long_nchunks;
  int64_t n_tiles, n_long, n_long_chunks;
};

inline TileSched make_sched(const fj_graph* g) {
  TileSched s;
  s.n = g->n; s.row_ptr = g->row_ptr; s.col = g->col; s.w = g->w;
  s.tile_begin = g->tile_begin; s.tile_end = g->tile_end; s.long_row = g->long_row;
  s.chunk_row = g->chunk_row; s.chunk_idx = g->chunk_idx; s.long_nchunks = g->long_nchunks;
  s.n_tiles = g->n_tiles; s.n_long = g->n_long; s.n_long_chunks = g->n_long_chunks;
  return s;
}

// Scratch for the cross-block parts of a tile launch (device memory, owned by the caller).
struct TileScratch {
  double* block_part;      // [grid][NP]
  double* long_part;       // [n_long][NP]
  double* chunk_acc;       // [n_long_chunks][NA]
  unsigned int* long_ticket;   // [n_long], zero-initialised, self-resetting
  unsigned int* grid_ticket;   // [1], zero-initialised, self-resetting
};

// Op interface:
//   static constexpr int NA, NP; static constexpr bool NEEDS_XI;
//   __device__ bool skip() const;                  // uniform early exit (solver finished)
//   __device__ double gather(int32_t j) const;     // value staged per nonzero
//   __device__ double row_value(int64_t i) const;  // x_i (only if NEEDS_XI)
//   __device__ void add(double (&a)[NA], double w, double xj, double xi) const;
//   __device__ void finish_row(int64_t i, int64_t len, const double (&a)[NA], double (&part)[NP]) const;
//   __device__ void finalize(const double (&tot)[NP]) const;   // single thread of the last block
template <int WT, class Op>
__global__ void __launch_bounds__(TPB) tile_kernel(const TileSched sc, const Op op, const TileScratch ws) {
  constexpr int NA = Op::NA, NP = Op::NP;
  constexpr bool WEIGHTED = (WT != FJ_W_UNIT);
  constexpr int NW = TPB / 32;
  __shared__ double s_x[TILE_MAX_NNZ];
  __shared__ double s_w[WEIGHTED ? TILE_MAX_NNZ : 1];
  __shared__ int32_t s_off[TILE_MAX_ROWS + 1];
  __shared__ int32_t s_big[TILE_MAX_ROWS];
  __shared__ int32_t s_wcount[NW + 1];
  __shared__ double s_red[(NP > NA ? NP : NA) * NW];
  __shared__ bool s_last;

  if (op.skip()) return;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  double part[NP];
#pragma unroll
  for (int j = 0; j < NP; ++j) part[j] = 0.0;

  const int64_t n_items = sc.n_long_chunks + sc.n_tiles;
  for (int64_t it = blockIdx.x; it < n_items; it += gridDim.x) {
    if (it < sc.n_long_chunks) {
      // ------------------------------------------------ long-row chunk
      const int32_t l = sc.chunk_row[it];
      const int32_t ci = sc.chunk_idx[it];
      const int64_t i = sc.long_row[l];
      const int64_t rb = sc.row_ptr[i], re = sc.row_ptr[i + 1];
      const int64_t kb = rb + (int64_t)ci * LONG_CHUNK;
      const int64_t ke = min(kb + (int64_t)LONG_CHUNK, re);
      const double xi = Op::NEEDS_XI ? op.row_value(i) : 0.0;
      double a[NA];
#pragma unroll
      for (int f = 0; f < NA; ++f) a[f] = 0.0;
#pragma unroll 4
      for (int64_t k = kb + tid; k < ke; k += TPB) {
        const double wk = WeightT<WT>::get(sc.w, k);
        op.add(a, wk, op.gather(__ldg(sc.col + k)), xi);
      }
      block_sum<NA, TPB>(a, s_red);
      if (tid == 0) {
#pragma unroll
        for (int f = 0; f < NA; ++f) ws.chunk_acc[it * NA + f] = a[f];
        __threadfence();
        unsigned int t = atomicAdd(ws.long_ticket + l, 1u);
        s_last = (t == (unsigned)sc.long_nchunks[l] - 1u);
      }
      __syncthreads();
      if (s_last && tid == 0) {
        __threadfence();
        const int64_t c0 = it - ci;
        double acc[NA];
#pragma unroll
        for (int f = 0; f < NA; ++f) acc[f] = 0.0;
        for (int32_t c = 0; c < sc.long_nchunks[l]; ++c) {
#pragma unroll
          for (int f = 0; f < NA; ++f) acc[f] += ld_cg(ws.chunk_acc + (c0 + c) * NA + f);
        }
        double lp[NP];
#pragma unroll
        for (int j = 0; j < NP; ++j) lp[j] = 0.0;
        op.finish_row(i, re - rb, acc, lp);
#pragma unroll
        for (int j = 0; j < NP; ++j) ws.long_part[(int64_t)l * NP + j] = lp[j];
        ws.long_ticket[l] = 0u;
      }
      __syncthreads();
    } else {
      // ------------------------------------------------ tile of short rows
      const int64_t t = it - sc.n_long_chunks;
      const int32_t r0 = sc.tile_begin[t], r1 = sc.tile_end[t];
      const int nrows = r1 - r0;
      const int64_t k0 = sc.row_ptr[r0];
      if (tid <= nrows) s_off[tid] = (int32_t)(sc.row_ptr[r0 + tid] - k0);
      __syncthreads();
      const int nk = s_off[nrows];
      // stage: coalesced col loads, independent gathers (<= 8 per thread)
#pragma unroll
      for (int u = 0; u < TILE_MAX_NNZ / TPB; ++u) {
        const int k = tid + u * TPB;
        if (k < nk) {
          s_x[k] = op.gather(__ldg(sc.col + k0 + k));
          if (WEIGHTED) s_w[k] = WeightT<WT>::get(sc.w, k0 + k);
        }
      }
      // rows longer than 32 go to warps: deterministic compaction by thread id
      const bool mine = tid < nrows;
      const int b = mine ? s_off[tid] : 0;
      const int e = mine ? s_off[tid + 1] : 0;
      const bool big = mine && (e - b) > 32;
      const unsigned bal = __ballot_sync(0xffffffffu, big);
      if (lane == 0) s_wcount[wid] = __popc(bal);
      __syncthreads();   // also publishes s_x / s_w
      if (tid == 0) {
        int acc = 0;
        for (int q = 0; q < NW; ++q) { int c = s_wcount[q]; s_wcount[q] = acc; acc += c; }
        s_wcount[NW] = acc;
      }
      __syncthreads();
      if (big) s_big[s_wcount[wid] + __popc(bal & ((1u << lane) - 1u))] = tid;
      if (mine && !big) {
        const int64_t i = r0 + tid;
        const double xi = Op::NEEDS_XI ? op.row_value(i) : 0.0;
        double a[NA];
#pragma unroll
        for (int f = 0; f < NA; ++f) a[f] = 0.0;
        for (int k = b; k < e; ++k) op.add(a, WEIGHTED ? s_w[k] : 1.0, s_x[k], xi);
        op.finish_row(i, e - b, a, part);
      }
      __syncthreads();
      const int nbig = s_wcount[NW];
      for (int q = wid; q < nbig; q += NW) {
        const int rt = s_big[q];
        const int bb = s_off[rt], ee = s_off[rt + 1];
        const int64_t i = r0 + rt;
        const double xi = Op::NEEDS_XI ? op.row_value(i) : 0.0;
        double a[NA];
#pragma unroll
        for (int f = 0; f < NA; ++f) a[f] = 0.0;
        for (int k = bb + lane; k < ee; k += 32) op.add(a, WEIGHTED ? s_w[k] : 1.0, s_x[k], xi);
#pragma unroll
        for (int f = 0; f < NA; ++f) a[f] = warp_sum(a[f]);
        if (lane == 0) op.finish_row(i, ee - bb, a, part);
      }
      __syncthreads();
    }
  }

  // ---------------------------------------------------- grid-level deterministic reduction
  block_sum<NP, TPB>(part, s_red);
  if (tid == 0) {
#pragma unroll
    for (int j = 0; j < NP; ++j) ws.block_part[(int64_t)blockIdx.x * NP + j] = part[j];
  }
  if (last_block_ticket(ws.grid_ticket, gridDim.x)) {
    double tot[NP];
#pragma unroll
    for (int j = 0; j < NP; ++j) tot[j] = 0.0;
    for (int64_t q = tid; q < (int64_t)gridDim.x; q += TPB) {
#pragma unroll
      for (int j = 0; j < NP; ++j) tot[j] += ld_cg(ws.block_part + q * NP + j);
    }
    for (int64_t q = tid; q < sc.n_long; q += TPB) {
#pragma unroll
      for (int j = 0; j < NP; ++j) tot[j] += ld_cg(ws.long_part + q * NP + j);
    }
    block_sum<NP, TPB>(tot, s_red);
    if (tid == 0) {
      op.finalize(tot);
      *ws.grid_ticket = 0u;
    }
  }
}

}  // namespace fj

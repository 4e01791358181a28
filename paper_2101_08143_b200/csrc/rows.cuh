// rows.cuh — the small-k PCG product q = (I+L)p (rows a4/a9, KP = 2 or 4 padded gathered rows) as a
// lean row kernel over COLUMN SLABS.  DESIGN.md §6.10.
//
// Why (measured, profiles/r02_slab2_probe_*.jsonl): on C3 (BA 4e6, k = 3) the gathered block p is
// [n][4] fp64 = 128 MB, above the ~80 MB the L2 holds for random 32-byte gathers, so the merge-path
// engine (tiles.cuh) runs at the DRAM-miss bound of that footprint (0.61 ms, 3.06 GB DRAM per
// launch for 0.48 GB algorithmic).  Splitting each row's entries at the column n/2 into two slabs
// and running one pass per slab keeps every pass's gathered half of p (64 MB) L2-resident; with a
// lean row kernel (G lanes per row, U gathers in flight per lane, no shared-memory staging, no
// merge-path search or carry scan) the two passes cost less than the one engine pass.
//
// Layout: the canonical CSR has ascending columns in every row, so a row's slab-A entries are a
// PREFIX of the row: per row one int32 offset (off[i] = #cols < n/2) is the whole slab split, no
// second copy of col.  Rows longer than ROWS_LONG nonzeros (hubs) are cut into ROWS_CH-nonzero
// chunks, each summed by one warp into chunk_acc (in the first pass); the finishing
// pass adds a long row's chunk sums in chunk order.  Every partial is formed and combined in a fixed
// order (lane-strided sums, xor-shuffle tree, chunks in order, pass A + pass B, blocks in order):
// results are bitwise reproducible run to run.
//
// Per launch sequence (single GPU, inside the PCG graph):
//   k_rows<PASS 0>  long-row chunk warps: chunk_acc[c] = sum over the chunk of w p_j; then slab A of
//                   every short row: q_i = sum_{j < n/2} w_ij p_j                  (partial)
//   k_rows<PASS 1>  slab B + finish                 q_i = (1+d_i) p_i - (q_i + sum_{j >= n/2})
//   (or k_rows_chunks + k_rows<PASS 2>: one pass over whole rows when the block fits the L2 or
//   some row's columns do not ascend)
// The finishing pass also forms p_c^T q_c (deterministic two-stage reduction) and alpha_c on device,
// exactly as ApplyOpV::finalize (spmv_vec.cu).
#pragma once
#include "ops.cuh"
#include "vec.cuh"

namespace fj {

#ifndef FJ_ROWS_LONG1
#define FJ_ROWS_LONG1 128       // k = 1 (one 8-byte gather per nonzero)
#endif
#ifndef FJ_ROWS_LONG
#define FJ_ROWS_LONG 128        // KP = 2, 4; measured C3 k = 3: 128 0.478 ms, 64 0.496, 256 0.487, 512 0.504
#endif
#ifndef FJ_ROWS_CH
#define FJ_ROWS_CH 256          // measured C3: 256 0.481 ms vs 1024 0.487
#endif
// rows with more nonzeros than the plan's long_row (FJ_ROWS_LONG, or FJ_ROWS_LONG1 for k = 1) are
// summed by chunk warps
constexpr int ROWS_CH = FJ_ROWS_CH;       // nonzeros per long-row chunk
constexpr int RTB = 256;         // threads per block of the row kernels
static_assert(FJ_ROWS_LONG < 65536 && FJ_ROWS_LONG1 < 65536, "slab offsets are uint16");
#ifndef FJ_ROWS_G
#define FJ_ROWS_G 2              // lanes per row (measured on C3: 2 > 1, 4 > 8 > 16, 32)
#endif
#ifndef FJ_ROWS_U
#define FJ_ROWS_U 4              // independent gathers in flight per lane
#endif
#ifndef FJ_ROWS_G_B
#define FJ_ROWS_G_B 1            // lanes per row in the slab-B pass (C3: 1 0.465 ms, 2 0.475, 4 0.527)
#endif
#ifndef FJ_ROWS_U_B
#define FJ_ROWS_U_B FJ_ROWS_U
#endif
#ifndef FJ_ROWS_MINB
#define FJ_ROWS_MINB 8           // slab-A pass: 8 x 256 threads per SM (32 registers, no spill)
#endif
#ifndef FJ_ROWS_MINB_FIN
#define FJ_ROWS_MINB_FIN 6       // finishing passes (p^T q partials, the epilogue): 40 registers
#endif

// Gathered row of p through the non-coherent path (p is read-only during a product).  Plain (not
// volatile) asm so the U loads of a batch are issued back to back.
template <int KP> __device__ __forceinline__ DVec<KP> ldg_vec(const double* p);
template <> __device__ __forceinline__ DVec<1> ldg_vec<1>(const double* p) {
  DVec<1> r;
  asm("ld.global.nc.f64 %0, [%1];" : "=d"(r.v[0]) : "l"(p));
  return r;
}
template <> __device__ __forceinline__ DVec<2> ldg_vec<2>(const double* p) {
  DVec<2> r;
  asm("ld.global.nc.v2.f64 {%0, %1}, [%2];" : "=d"(r.v[0]), "=d"(r.v[1]) : "l"(p));
  return r;
}
template <> __device__ __forceinline__ DVec<4> ldg_vec<4>(const double* p) {
  DVec<4> r;
  asm("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(r.v[0]), "=d"(r.v[1]), "=d"(r.v[2]), "=d"(r.v[3])
      : "l"(p));
  return r;
}

// L2 eviction hints (FJ_ROWS_HINT bits, A/B): 1 = the streams (col, row_ptr, off) evict-first,
// 2 = the gathers of p evict-last, 4 = the own-row read of p in the finishing pass evict-first.
#ifndef FJ_ROWS_HINT
#define FJ_ROWS_HINT 0
#endif
__device__ __forceinline__ uint64_t pol_first() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t pol_last() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ int32_t ldh_i32(const int32_t* a, uint64_t pol) {
  int32_t r;
  asm("ld.global.nc.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(r) : "l"(a), "l"(pol));
  return r;
}
template <int KP> __device__ __forceinline__ DVec<KP> ldgh_vec(const double* p, uint64_t pol);
template <> __device__ __forceinline__ DVec<1> ldgh_vec<1>(const double* p, uint64_t pol) {
  DVec<1> r;
  asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(r.v[0]) : "l"(p), "l"(pol));
  return r;
}
template <> __device__ __forceinline__ DVec<2> ldgh_vec<2>(const double* p, uint64_t pol) {
  DVec<2> r;
  asm("ld.global.nc.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(r.v[0]), "=d"(r.v[1]) : "l"(p), "l"(pol));
  return r;
}
template <> __device__ __forceinline__ DVec<4> ldgh_vec<4>(const double* p, uint64_t pol) {
  DVec<4> r;
  asm("ld.global.nc.L2::cache_hint.v4.f64 {%0, %1, %2, %3}, [%4], %5;"
      : "=d"(r.v[0]), "=d"(r.v[1]), "=d"(r.v[2]), "=d"(r.v[3]) : "l"(p), "l"(pol));
  return r;
}
template <int KP> __device__ __forceinline__ DVec<KP> ld_gather(const double* p, uint64_t pol) {
  if constexpr ((FJ_ROWS_HINT & 2) != 0) return ldgh_vec<KP>(p, pol); else return ldg_vec<KP>(p);
}
__device__ __forceinline__ int32_t ld_colh(const int32_t* a, uint64_t pol) {
  if constexpr ((FJ_ROWS_HINT & 1) != 0) return ldh_i32(a, pol); else return __ldg(a);
}

struct RowsArgs {
  int64_t n;
  const int64_t* __restrict__ rp;
  const int32_t* __restrict__ col;
  const void* __restrict__ w;
  const int32_t* __restrict__ rp32;     // [n+1] row_ptr as int32 (the plan's copy: nnz < 2^31)
  const uint16_t* __restrict__ off;     // [n] slab-A entries per short row (2-slab mode)
  const int32_t* __restrict__ c0;       // [n] first chunk of a long row
  const int64_t* __restrict__ tab;      // [n_chunks][2] (row, first nonzero)
  int64_t n_chunks;
  int64_t long_row;                     // rows longer than this are summed by chunk warps
  double* chunk_acc;                    // [n_chunks][4]
  const double* __restrict__ x;         // gathered block, padded [n][KP]
  double* y;                            // [n][KQ]
  const double* __restrict__ deg;
  int opL, k;
  VecScalars* sc;                       // small-k PCG mode: alpha_c on device (null: plain apply)
  PcgScalars* sc1;                      // k = 1 PCG mode (pcg.cu): alpha on device
  double* part;                         // [grid][4] block partials of p^T q
  unsigned int* ticket;                 // [1], self-resetting
  // slab-major copies of the short rows' entries (FJ_ROWS_SPLIT; null: not built): colA[rpA[i],
  // rpA[i+1]) = row i's slab-A columns, colB[rpB[i], rpB[i+1]) its slab-B columns; wA / wB their
  // weights (null for unit weights)
  const int32_t* __restrict__ rpA;
  const int32_t* __restrict__ rpB;
  const int32_t* __restrict__ colA;
  const int32_t* __restrict__ colB;
  const void* __restrict__ wA;
  const void* __restrict__ wB;
};

template <int WT, int KP, int KQ, int U>
__device__ __forceinline__ void rows_accumulate(const RowsArgs& a, const int32_t* __restrict__ col,
                                                const void* __restrict__ w, int64_t k, int64_t ke, int stride,
                                                double (&acc)[KQ], uint64_t ps = 0, uint64_t pg = 0) {
  using WS = typename std::conditional<WT == FJ_W_F64, double, float>::type;   // exact for u8 / f32
  for (; k + (int64_t)(U - 1) * stride < ke; k += (int64_t)U * stride) {   // full batches
    int32_t j[U];
    WS wv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      j[u] = ld_colh(col + k + u * stride, ps);
      wv[u] = (WT == FJ_W_UNIT) ? (WS)1 : (WS)WeightT<WT>::get(w, k + u * stride);
    }
    DVec<KP> v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = ld_gather<KP>(a.x + (int64_t)j[u] * KP, pg);
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
      for (int c = 0; c < KQ; ++c) acc[c] = (WT == FJ_W_UNIT) ? acc[c] + v[u].v[c] : fma((double)wv[u], v[u].v[c], acc[c]);
  }
  for (; k < ke; k += stride) {
    const DVec<KP> v = ld_gather<KP>(a.x + (int64_t)ld_colh(col + k, ps) * KP, pg);
    const double wk = (WT == FJ_W_UNIT) ? 1.0 : (double)WeightT<WT>::get(w, k);
#pragma unroll
    for (int c = 0; c < KQ; ++c) acc[c] = (WT == FJ_W_UNIT) ? acc[c] + v.v[c] : fma(wk, v.v[c], acc[c]);
  }
}

// Padded slab-major copies (FJ_ROWS_PAD_A / FJ_ROWS_PAD_B = 4; 0: unpadded): each row's entries of the
// copy start at a multiple of 4 and are padded to a multiple of 4 with column -1 (weight 0), so a
// lane reads FOUR column indices with one aligned 16-byte load (one L1 wavefront per lane group
// instead of four, no tail loop) and issues their gathers together; pads gather nothing and add 0.
// Measured on C3 k = 3 (profiles/r02_ab_rows_pad.log): slab A padded 0.4476 -> 0.4313 ms (kept: the
// pass is L1TEX-wavefront bound); slab B padded (its rows hold ~5 entries: +30 % of
// its column stream) 0.470 ms, both 0.453 ms (not kept).
#ifndef FJ_ROWS_PAD_A
#define FJ_ROWS_PAD_A 4
#endif
#ifndef FJ_ROWS_PAD_B
#define FJ_ROWS_PAD_B 0
#endif
template <int WT, int KP, int KQ>
__device__ __forceinline__ void rows_accumulate_pad4(const RowsArgs& a, const int32_t* __restrict__ col,
                                                     const void* __restrict__ w, int64_t k4, int64_t k4e, int stride,
                                                     double (&acc)[KQ]) {
  using WS = typename std::conditional<WT == FJ_W_F64, double, float>::type;
  for (; k4 < k4e; k4 += stride) {
    const int4 c = __ldg(reinterpret_cast<const int4*>(col) + k4);
    const int32_t j[4] = {c.x, c.y, c.z, c.w};
    WS wv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) wv[u] = (WT == FJ_W_UNIT) ? (WS)1 : (WS)WeightT<WT>::get(w, 4 * k4 + u);
    DVec<KP> v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (j[u] >= 0) {
        v[u] = ldg_vec<KP>(a.x + (int64_t)j[u] * KP);
      } else {
#pragma unroll
        for (int c2 = 0; c2 < KP; ++c2) v[u].v[c2] = 0.0;
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
      for (int c2 = 0; c2 < KQ; ++c2)
        acc[c2] = (WT == FJ_W_UNIT) ? acc[c2] + v[u].v[c2] : fma((double)wv[u], v[u].v[c2], acc[c2]);
  }
}

// Long-row chunks: one warp per chunk (grid-stride over the launch's warps), chunk_acc[c] = sum
// w p_j over the chunk.
template <int WT, int KP, int KQ>
__device__ __forceinline__ void rows_chunk_items(const RowsArgs& a, uint64_t ps, uint64_t pg) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (RTB / 32);
  for (int64_t c = (blockIdx.x * (int64_t)RTB + threadIdx.x) >> 5; c < a.n_chunks; c += nw) {
    const int64_t r = a.tab[2 * c], k0 = a.tab[2 * c + 1];
    const int64_t k1 = min(k0 + (int64_t)ROWS_CH, (int64_t)a.rp32[r + 1]);
    FJ_DCHECK(r >= 0 && r < a.n && k0 >= a.rp32[r] && k0 < k1);
    double acc[KQ];
#pragma unroll
    for (int f = 0; f < KQ; ++f) acc[f] = 0.0;
    rows_accumulate<WT, KP, KQ, 4>(a, a.col, a.w, k0 + lane, k1, 32, acc, ps, pg);
#pragma unroll
    for (int f = 0; f < KQ; ++f) acc[f] = warp_sum(acc[f]);
    if (lane == 0) {
#pragma unroll
      for (int f = 0; f < KQ; ++f) a.chunk_acc[c * 4 + f] = acc[f];
    }
  }
}
// One-pass mode: the chunks in their own launch before k_rows<PASS 2> (which reads them).
__device__ __forceinline__ bool rows_skip(const RowsArgs& a) {   // the solver has finished
  return (a.sc && *(volatile int32_t*)&a.sc->done) || (a.sc1 && *(volatile int32_t*)&a.sc1->done);
}
template <int WT, int KP, int KQ>
__global__ void __launch_bounds__(RTB) k_rows_chunks(const RowsArgs a) {
  if (rows_skip(a)) return;
  const uint64_t ps = (FJ_ROWS_HINT & 1) ? pol_first() : 0, pg = (FJ_ROWS_HINT & 2) ? pol_last() : 0;
  rows_chunk_items<WT, KP, KQ>(a, ps, pg);
}

// PASS 0: the long-row chunks (fused: the chunk warps run beside the row groups of other warps;
// FJ_ROWS_FUSE_CHUNKS=0 launches them apart) then slab A partial sums; PASS 1: slab B + finish;
// PASS 2: whole rows + finish.
#ifndef FJ_ROWS_FUSE_CHUNKS
#define FJ_ROWS_FUSE_CHUNKS 1
#endif
template <int WT, int KP, int KQ, int PASS>
__global__ void __launch_bounds__(RTB, PASS == 0 ? FJ_ROWS_MINB : FJ_ROWS_MINB_FIN) k_rows(const RowsArgs a) {
  constexpr int G = PASS == 1 ? FJ_ROWS_G_B : FJ_ROWS_G, U = PASS == 1 ? FJ_ROWS_U_B : FJ_ROWS_U;
  constexpr bool FIN = PASS != 0;
  __shared__ double s_red[4 * RTB / 32];
  if (rows_skip(a)) return;
  const int64_t ng = (int64_t)gridDim.x * (RTB / G);
  const int sub = threadIdx.x % G;
  const uint64_t ps = (FJ_ROWS_HINT & 5) ? pol_first() : 0, pg = (FJ_ROWS_HINT & 2) ? pol_last() : 0;
  if constexpr (PASS == 0 && FJ_ROWS_FUSE_CHUNKS) rows_chunk_items<WT, KP, KQ>(a, ps, pg);
  double part[KQ];
#pragma unroll
  for (int f = 0; f < KQ; ++f) part[f] = 0.0;
  // the loop runs on the warp's first row (warp-uniform trip count: the group shuffles below use
  // the full mask); groups past the last row take an empty range
  for (int64_t i0 = (blockIdx.x * (int64_t)RTB + (threadIdx.x & ~31)) / G; i0 < a.n; i0 += ng) {
    const int64_t i = i0 + (threadIdx.x & 31) / G;
    const bool valid = i < a.n;
    const bool split = PASS != 2 && a.colA != nullptr;   // uniform over the launch
    int64_t b = 0, e = 0, kb = 0, ke = 0;
    bool lng = false;
    if (PASS == 0 && split) {   // slab-major: the row's slab-A entries only (long rows: empty)
      if (valid) { kb = ld_colh(a.rpA + i, ps); ke = ld_colh(a.rpA + i + 1, ps); }
    } else {
      if (valid) { b = ld_colh(a.rp32 + i, ps); e = ld_colh(a.rp32 + i + 1, ps); }
      lng = e - b > a.long_row;
      kb = b; ke = e;
      if (PASS == 1 && split) {
        if (valid) { kb = ld_colh(a.rpB + i, ps); ke = ld_colh(a.rpB + i + 1, ps); }
      } else {
        if (PASS == 0 && valid) ke = b + __ldg(a.off + i);
        if (PASS == 1 && valid) kb = b + __ldg(a.off + i);
        FJ_DCHECK(kb >= b && ke <= e && kb <= ke);
      }
    }
    FJ_DCHECK(kb <= ke);
    const int32_t* __restrict__ colp = !split ? a.col : PASS == 0 ? a.colA : a.colB;
    const void* __restrict__ wp = !split ? a.w : PASS == 0 ? a.wA : a.wB;
    double acc[KQ];
#pragma unroll
    for (int f = 0; f < KQ; ++f) acc[f] = 0.0;
    constexpr int PAD = PASS == 0 ? FJ_ROWS_PAD_A : PASS == 1 ? FJ_ROWS_PAD_B : 0;
    if (PAD == 4 && split) {   // padded copies: kb, ke are multiples of 4 (long rows: empty)
      rows_accumulate_pad4<WT, KP, KQ>(a, colp, wp, (kb >> 2) + sub, ke >> 2, G, acc);
    } else if (!lng) {
      rows_accumulate<WT, KP, KQ, U>(a, colp, wp, kb + sub, ke, G, acc, ps, pg);
    }
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1)
#pragma unroll
      for (int f = 0; f < KQ; ++f) acc[f] += __shfl_xor_sync(0xffffffffu, acc[f], o, G);
    if (sub != 0 || !valid) continue;
    DVec<KP> yv;
#pragma unroll
    for (int c = 0; c < KP; ++c) yv.v[c] = c < KQ ? acc[c < KQ ? c : 0] : 0.0;
    if (PASS == 0) { st_q<KP, KQ>(a.y, i, yv); continue; }
    double tot[KQ];
    if (lng) {   // chunk sums in chunk order
#pragma unroll
      for (int f = 0; f < KQ; ++f) tot[f] = 0.0;
      const int64_t c0 = a.c0[i], nch = (e - b + ROWS_CH - 1) / ROWS_CH;
      for (int64_t c = c0; c < c0 + nch; ++c)
#pragma unroll
        for (int f = 0; f < KQ; ++f) tot[f] += __ldcg(a.chunk_acc + c * 4 + f);
    } else if (PASS == 1) {
      const DVec<KP> ya = ld_q<KP, KQ>(a.y, i);
#pragma unroll
      for (int f = 0; f < KQ; ++f) tot[f] = ya.v[f] + acc[f];
    } else {
#pragma unroll
      for (int f = 0; f < KQ; ++f) tot[f] = acc[f];
    }
    const double d = (WT == FJ_W_UNIT) ? (double)(e - b) : a.deg[i];
    const double dd = a.opL ? d : 1.0 + d;
    // own row of p: in the finishing pass of two slabs, rows of slab A are not being gathered
    const DVec<KP> xi = ((FJ_ROWS_HINT & 4) && PASS == 1 && i < a.n / 2) ? ldgh_vec<KP>(a.x + i * KP, ps)
                                                                       : ldg_vec<KP>(a.x + i * KP);
#pragma unroll
    for (int c = 0; c < KQ; ++c) {
      yv.v[c] = fma(dd, xi.v[c], -tot[c]);
      part[c] = fma(xi.v[c], yv.v[c], part[c]);
    }
    st_q<KP, KQ>(a.y, i, yv);
  }
  if constexpr (FIN) {
    block_sum<KQ, RTB>(part, s_red);
    if (threadIdx.x == 0) {
#pragma unroll
      for (int f = 0; f < KQ; ++f) a.part[(int64_t)blockIdx.x * 4 + f] = part[f];
    }
    if (!last_block_ticket(a.ticket, gridDim.x)) return;
    double t[KQ];
#pragma unroll
    for (int f = 0; f < KQ; ++f) t[f] = 0.0;
    for (int bb = threadIdx.x; bb < (int)gridDim.x; bb += RTB)
#pragma unroll
      for (int f = 0; f < KQ; ++f) t[f] += __ldcg(a.part + (int64_t)bb * 4 + f);
    block_sum<KQ, RTB>(t, s_red);
    if (threadIdx.x != 0) return;
    *a.ticket = 0u;
    if (PcgScalars* s1 = a.sc1) {   // k = 1 (as ApplyOp::finalize)
      s1->pq = t[0];
      if (!(t[0] > 0.0) || !isfinite(t[0])) {   // (I+L) is SPD: p^T q > 0 unless p = 0
        s1->alpha = 0.0;
        s1->breakdown = 1;
        s1->done = 1;
      } else {
        s1->alpha = s1->rho / t[0];
      }
      return;
    }
    VecScalars* sc = a.sc;
    if (!sc) return;
#pragma unroll
    for (int c = 0; c < KQ; ++c) {   // alpha_c = rho_c / p_c^T q_c (as ApplyOpV::finalize)
      if (c >= a.k) break;
      sc->pq[c] = t[c];
      if (sc->active[c]) {
        if (!(t[c] > 0.0) || !isfinite(t[c])) {
          sc->alpha[c] = 0.0;
          sc->active[c] = 0;
          sc->breakdown[c] = 1;
        } else {
          sc->alpha[c] = sc->rho[c] / t[c];
        }
      } else {
        sc->alpha[c] = 0.0;
      }
    }
  }
}

// ---------------------------------------------------------------- plan + launcher (host)
// The rows product of one graph for one gathered row width KP: built once with the solver
// workspace (rows.cu).  mode 0: the merge-path engine (tiles.cuh) computes the product instead.
struct RowsPlan {
  int mode = 0;                      // 0: engine; 1: one row pass; 2: two column slabs
  int grid = 0, grid_chunks = 0;
  int32_t* rp32 = nullptr;           // [n+1] int32 copy of row_ptr
  uint16_t* off = nullptr;           // [n] slab-A entries per short row (mode 2)
  int32_t* c0 = nullptr;             // [n] first long-row chunk
  int64_t* tab = nullptr;            // [n_chunks][2]
  int64_t n_chunks = 0;
  int64_t long_row = 0;
  // mode 2 (FJ_ROWS_SPLIT, default on): the short rows' entries (and weights) in slab-major copies,
  // so each pass streams only its own entries (no sector of col read by both passes)
  int32_t* rpA = nullptr;            // [n+1]
  int32_t* rpB = nullptr;            // [n+1]
  int32_t* colA = nullptr;           // [rpA[n]]
  int32_t* colB = nullptr;           // [rpB[n]]
  void* wA = nullptr;                // weights of colA / colB (null: unit weights)
  void* wB = nullptr;
  double* chunk_acc = nullptr;       // [n_chunks][4]
  double* part = nullptr;            // [grid][4]
  unsigned int* ticket = nullptr;
  // generic row operators (k_op_rows): chunk partials [n_chunks][ROWS_NA_MAX], block partials
  // [grid][ROWS_NP_MAX]
  double* op_acc = nullptr;
  double* op_part = nullptr;
  unsigned int* op_ticket = nullptr;
  int num_sms = 148;
  int grid_op_max = 0;               // rows of op_part (>= #SMs x occupancy of any k_op_rows)
};
// Selection (FJ_ROWS: -1 auto (default), 0 engine, 1 one pass, 2 two slabs): see rows.cu.
fj_status rows_plan_build(fj_graph* g, int kp, RowsPlan& R, cudaStream_t st);
// The plan of any CSR view (rows [0, n), int64 row_ptr, columns < ncol): one row pass, no slabs
// (the distributed path's diagonal / ghost CSRs).  Mode 0 if forced (FJ_ROWS=0) or nnz >= 2^31.
fj_status rows_plan_build_csr(int64_t n, int64_t nnz, const int64_t* row_ptr, const int32_t* col, int kp,
                              int num_sms, RowsPlan& R, cudaStream_t st);
void rows_plan_free(RowsPlan& R);
inline int rows_launches(const RowsPlan& R) {   // kernel launches of one product
  if (R.mode == 0) return 1;
  return (R.mode == 2 ? 2 : 1) + (R.n_chunks > 0 && (R.mode == 1 || !FJ_ROWS_FUSE_CHUNKS) ? 1 : 0);
}

// y = (I+L) x (or L x) on the rows plan; PCG mode with vsc (small k) or psc (k = 1).
template <int WT, int KP, int KQ>
fj_status rows_product(const fj_graph* g, const RowsPlan& R, const double* x, double* y, int opL, int k,
                       VecScalars* vsc, PcgScalars* psc, cudaStream_t st) {
  RowsArgs a{g->n, g->row_ptr, g->col, g->w, R.rp32, R.off, R.c0, R.tab, R.n_chunks, R.long_row, R.chunk_acc,
             x, y, g->deg, opL, k, vsc, psc, R.part, R.ticket, R.rpA, R.rpB, R.colA, R.colB, R.wA, R.wB};
  if (R.n_chunks > 0 && (R.mode == 1 || !FJ_ROWS_FUSE_CHUNKS)) {
    k_rows_chunks<WT, KP, KQ><<<R.grid_chunks, RTB, 0, st>>>(a);
    FJ_CK_LAUNCH();
  }
  if (R.mode == 2) {
    k_rows<WT, KP, KQ, 0><<<R.grid, RTB, 0, st>>>(a);
    FJ_CK_LAUNCH();
    k_rows<WT, KP, KQ, 1><<<R.grid, RTB, 0, st>>>(a);
  } else {
    k_rows<WT, KP, KQ, 2><<<R.grid, RTB, 0, st>>>(a);
  }
  FJ_CK_LAUNCH();
  return FJ_OK;
}


// ---------------------------------------------------------------- any row operator (tiles.cuh Op)
// The same lean scheme for the engine's other row operators (the fused quantities pass, the true
// residual; the distributed product's diagonal and ghost passes): G lanes per row gather through
// op.gather(), accumulate with op.add() (x_i = op.row_value(i) for operators that read it), the
// group's sums are reduced by an xor-shuffle tree, long rows are summed by chunk warps in a launch
// before (k_op_chunks, their NA partials in chunk order), then op.finish_row() on the group's first
// lane and op.finalize() on the fixed-order grid reduction.  One pass over whole rows (no slabs).
constexpr int ROWS_NA_MAX = 12, ROWS_NP_MAX = 16;
struct RowsView {   // a CSR (rows [0, nrows)) and its rows plan
  int64_t nrows;
  const int32_t* __restrict__ rp32;
  const int32_t* __restrict__ col;
  const void* __restrict__ w;
  int64_t long_row;
  const int32_t* __restrict__ c0;
  const int64_t* __restrict__ tab;
  int64_t n_chunks;
  double* acc;              // [n_chunks][ROWS_NA_MAX]
  double* part;             // [grid][ROWS_NP_MAX]
  unsigned int* ticket;
};

template <int WT, class Op, int U>
__device__ __forceinline__ void op_accumulate(const RowsView& v, const Op& op, int64_t k, int64_t ke, int stride,
                                              const typename Op::V& xi, double (&acc)[Op::NA]) {
  using V = typename Op::V;
  for (; k + (int64_t)(U - 1) * stride < ke; k += (int64_t)U * stride) {
    int32_t j[U];
    double wv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      j[u] = __ldg(v.col + k + u * stride);
      wv[u] = (WT == FJ_W_UNIT) ? 1.0 : WeightT<WT>::get(v.w, k + u * stride);
    }
    V xv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) xv[u] = op.gather(j[u]);
#pragma unroll
    for (int u = 0; u < U; ++u) op.add(acc, wv[u], xv[u], xi);
  }
  for (; k < ke; k += stride) {
    const double wk = (WT == FJ_W_UNIT) ? 1.0 : WeightT<WT>::get(v.w, k);
    op.add(acc, wk, op.gather(__ldg(v.col + k)), xi);
  }
}

template <int WT, class Op>
__global__ void __launch_bounds__(RTB) k_op_chunks(const RowsView v, const Op op) {
  constexpr int NA = Op::NA;
  static_assert(NA <= ROWS_NA_MAX, "row operator accumulators");
  if (op.skip()) return;
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (RTB / 32);
  for (int64_t c = (blockIdx.x * (int64_t)RTB + threadIdx.x) >> 5; c < v.n_chunks; c += nw) {
    const int64_t r = v.tab[2 * c], k0 = v.tab[2 * c + 1];
    const int64_t k1 = min(k0 + (int64_t)ROWS_CH, (int64_t)v.rp32[r + 1]);
    FJ_DCHECK(r >= 0 && r < v.nrows && k0 >= v.rp32[r] && k0 < k1);
    const typename Op::V xi = Op::NEEDS_XI ? op.row_value(r) : Op::vzero();
    double acc[NA];
#pragma unroll
    for (int f = 0; f < NA; ++f) acc[f] = 0.0;
    op_accumulate<WT, Op, 4>(v, op, k0 + lane, k1, 32, xi, acc);
#pragma unroll
    for (int f = 0; f < NA; ++f) acc[f] = warp_sum(acc[f]);
    if (lane == 0) {
#pragma unroll
      for (int f = 0; f < NA; ++f) v.acc[c * ROWS_NA_MAX + f] = acc[f];
    }
  }
}

#ifndef FJ_ROWS_OP_MINB
#define FJ_ROWS_OP_MINB 3
#endif
template <int WT, class Op>
__global__ void __launch_bounds__(RTB, FJ_ROWS_OP_MINB) k_op_rows(const RowsView v, const Op op) {
  constexpr int G = FJ_ROWS_G, U = FJ_ROWS_U, NA = Op::NA, NP = Op::NP;
  static_assert(NP <= ROWS_NP_MAX, "row operator partials");
  using V = typename Op::V;
  __shared__ double s_red[ROWS_NP_MAX * RTB / 32];
  if (op.skip()) return;
  const int64_t ng = (int64_t)gridDim.x * (RTB / G);
  const int sub = threadIdx.x % G;
  double part[NP];
#pragma unroll
  for (int f = 0; f < NP; ++f) part[f] = 0.0;
  for (int64_t i0 = (blockIdx.x * (int64_t)RTB + (threadIdx.x & ~31)) / G; i0 < v.nrows; i0 += ng) {
    const int64_t i = i0 + (threadIdx.x & 31) / G;
    const bool valid = i < v.nrows;
    const int64_t b = valid ? __ldg(v.rp32 + i) : 0, e = valid ? __ldg(v.rp32 + i + 1) : 0;
    const bool lng = e - b > v.long_row;
    const V xi = valid ? op.row_value(i) : Op::vzero();
    double acc[NA];
#pragma unroll
    for (int f = 0; f < NA; ++f) acc[f] = 0.0;
    if (!lng) op_accumulate<WT, Op, U>(v, op, b + sub, e, G, xi, acc);
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1)
#pragma unroll
      for (int f = 0; f < NA; ++f) acc[f] += __shfl_xor_sync(0xffffffffu, acc[f], o, G);
    if (sub != 0 || !valid) continue;
    if (lng) {   // chunk partials in chunk order
#pragma unroll
      for (int f = 0; f < NA; ++f) acc[f] = 0.0;
      const int64_t c0 = v.c0[i], nch = (e - b + ROWS_CH - 1) / ROWS_CH;
      for (int64_t c = c0; c < c0 + nch; ++c)
#pragma unroll
        for (int f = 0; f < NA; ++f) acc[f] += __ldcg(v.acc + c * ROWS_NA_MAX + f);
    }
    op.finish_row(i, e - b, xi, acc, part);
  }
  block_sum<NP, RTB>(part, s_red);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int f = 0; f < NP; ++f) v.part[(int64_t)blockIdx.x * ROWS_NP_MAX + f] = part[f];
  }
  if (!last_block_ticket(v.ticket, gridDim.x)) return;
  double t[NP];
#pragma unroll
  for (int f = 0; f < NP; ++f) t[f] = 0.0;
  for (int bb = threadIdx.x; bb < (int)gridDim.x; bb += RTB)
#pragma unroll
    for (int f = 0; f < NP; ++f) t[f] += __ldcg(v.part + (int64_t)bb * ROWS_NP_MAX + f);
  block_sum<NP, RTB>(t, s_red);
  if (threadIdx.x == 0) {
    op.finalize(t);
    *v.ticket = 0u;
  }
}

inline int rows_op_launches(const RowsPlan& R) { return R.mode == 0 ? 1 : (R.n_chunks > 0 ? 2 : 1); }

// Launch a row operator on a plan built for (rp, col) with nrows rows.  The grid is fixed per
// (plan, operator instantiation): #SMs x occupancy, so partials are reduced in a fixed order.
template <int WT, class Op>
fj_status rows_op(const RowsPlan& R, int64_t nrows, const int32_t* col, const void* w, const Op& op,
                  cudaStream_t st) {
  static int occ = 0;   // per instantiation
  if (occ == 0) {
    FJ_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_op_rows<WT, Op>, RTB, 0));
    if (occ < 1) occ = 1;
  }
  RowsView v{nrows, R.rp32, col, w, R.long_row, R.c0, R.tab, R.n_chunks, R.op_acc, R.op_part, R.op_ticket};
  if (R.n_chunks > 0) {
    k_op_chunks<WT, Op><<<R.grid_chunks, RTB, 0, st>>>(v, op);
    FJ_CK_LAUNCH();
  }
  int64_t grid = (int64_t)R.num_sms * occ;
  const int64_t need = (nrows * FJ_ROWS_G + RTB - 1) / RTB;
  if (grid > need) grid = need > 0 ? need : 1;
  if (grid > R.grid_op_max) grid = R.grid_op_max;
  k_op_rows<WT, Op><<<(unsigned)grid, RTB, 0, st>>>(v, op);
  FJ_CK_LAUNCH();
  return FJ_OK;
}

}  // namespace fj

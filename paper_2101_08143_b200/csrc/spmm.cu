// spmm.cu — row a9: k <= 64 opinion vectors solved TOGETHER (batched Jacobi-PCG on I+L with
// per-column alpha_j, beta_j and a per-column convergence mask).  Row-major [n][k] fp64 blocks:
// one neighbour row is k*8 bytes (512 B at k = 64), gathered by a warp as two fully coalesced
// 256-byte loads (lane l owns columns l and l+32).  Same work items as the k = 1 row engine
// (tiles.cuh): T tiles are walked row by row, W rows and C chunks stride over their nonzeros;
// per-column dot products are per-lane (columns never mix), reduced over warps and blocks in a
// fixed order, so results are bitwise reproducible.
#include <cstring>
#include <vector>

#include "ops.cuh"
#include "workspace.cuh"

namespace fj {

#ifndef FJ_SPMM_NB
#define FJ_SPMM_NB 8                   // neighbour rows in flight per warp (measured: 8 at 8 blocks/SM
                                       // 7.6 ms per C4 product, 16 unconstrained 8.5 ms)
#endif
#ifndef FJ_QB_MIN_BLOCKS
#define FJ_QB_MIN_BLOCKS 0             // batched quantities pass
#endif
#ifndef FJ_SPMM_MIN_BLOCKS
#define FJ_SPMM_MIN_BLOCKS 8
#endif
constexpr int BTPB = 128;              // 4 warps
constexpr int BWPB = BTPB / 32;

// Deterministic grid tail of the k > 4 kernels (last block, all BTPB threads): the total of column
// c = t % 64 over nb block partials and nl long-row partials (entries `stride` doubles apart).  Thread
// group t / 64 folds entries g*8.., 8 independent accumulators (8 loads in flight), groups summed in
// order: a fixed order, and ~16x less tail latency than one thread per column walking every entry
// (C4: 1184 blocks + 12 140 long rows per launch).
__device__ __forceinline__ double tail_sum(const double* bp, int64_t nb, const double* lp, int64_t nl,
                                           int64_t stride, double* s_tail /*[BTPB]*/) {
  constexpr int NG = BTPB / MAXK;
  const int c = threadIdx.x % MAXK, grp = threadIdx.x / MAXK;
  double acc[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) acc[u] = 0.0;
  for (int64_t b0 = (int64_t)grp * 8; b0 < nb; b0 += NG * 8) {
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (b0 + u < nb) acc[u] += __ldcg(bp + (b0 + u) * stride);
  }
  for (int64_t l0 = (int64_t)grp * 8; l0 < nl; l0 += NG * 8) {
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (l0 + u < nl) acc[u] += __ldcg(lp + (l0 + u) * stride);
  }
  s_tail[threadIdx.x] = ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));
  __syncthreads();
  double tot = 0.0;
  for (int g2 = 0; g2 < NG; ++g2) tot += s_tail[g2 * MAXK + c];
  __syncthreads();
  return tot;
}
// batched schedule: short rows in tiles of <= ~224 nonzeros, W rows up to 1024, chunks of 1024
constexpr SchedParams kSchedBatch{64, 160, 8, 1024};

struct BatchScalars {
  double rho[MAXK], alpha[MAXK], beta[MAXK], pq[MAXK], rr[MAXK], ss[MAXK], tol2[MAXK], res2[MAXK];
  int32_t active[MAXK], conv[MAXK], breakdown[MAXK];
  int32_t iter, max_iter, done, k;
};

enum { BM_PCG = 0, BM_RESID = 1, BM_APPLY = 2 };

struct BatchArgs {
  int k;
  int ldmode;                      // gather load flavour (ld_gather2)
  const double* __restrict__ x;    // [n][k] input (p, or the iterate for the residual)
  double* __restrict__ y;          // [n][k] output (q)           (BM_PCG, BM_APPLY)
  const double* __restrict__ s;    // [n][k] right-hand side      (BM_RESID)
  const double* __restrict__ deg;
  int opL;
  BatchScalars* bs;
  double* chunk_acc;               // [n_chunks][64]
  double* long_part;               // [n_long][64]
  unsigned int* long_ticket;
  double* block_part;              // [grid][64]
  unsigned int* grid_ticket;
};

// 16-byte gather of two adjacent columns; mode 0: read-only path (ld.global.nc), 1: plain
// ld.global, 2: ld.global.nc.L1::no_allocate (experiment knob FJ_GATHER_MODE)
__device__ __forceinline__ double2 ld_gather2(const double* p, int mode) {
  double2 r;
  if (mode == 1) {
    asm volatile("ld.global.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
  } else if (mode == 2) {
    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
  } else {
    r = __ldg(reinterpret_cast<const double2*>(p));
  }
  return r;
}

// Column ownership of a lane: PAIR (k even) -> columns 2l, 2l+1 loaded as one 16-byte double2;
// otherwise columns l and l+32 as two coalesced 8-byte loads.
template <bool PAIR>
__device__ __forceinline__ int col0(int lane) { return PAIR ? 2 * lane : lane; }
template <bool PAIR>
__device__ __forceinline__ int col1(int lane) { return PAIR ? 2 * lane + 1 : lane + 32; }

// finish row i: y = (1+d) x_i - acc (or d x_i - acc), per-lane column partials
template <int WT, int MODE, bool PAIR>
__device__ __forceinline__ void b_finish(const BatchArgs& a, int64_t i, int64_t len, int lane, double acc0,
                                         double acc1, double& p0, double& p1) {
  const int k = a.k;
  const double d = (WT == FJ_W_UNIT) ? (double)len : a.deg[i];
  const double dd = (MODE == BM_APPLY && a.opL) ? d : 1.0 + d;
  const int c0 = col0<PAIR>(lane), c1 = col1<PAIR>(lane);
  if (c0 < k) {
    const double xi = a.x[i * k + c0];
    const double yi = fma(dd, xi, -acc0);
    if (MODE == BM_RESID) {
      const double r = a.s[i * k + c0] - yi;
      p0 = fma(r, r, p0);
    } else {
      a.y[i * k + c0] = yi;
      p0 = fma(xi, yi, p0);
    }
  }
  if (c1 < k) {
    const double xi = a.x[i * k + c1];
    const double yi = fma(dd, xi, -acc1);
    if (MODE == BM_RESID) {
      const double r = a.s[i * k + c1] - yi;
      p1 = fma(r, r, p1);
    } else {
      a.y[i * k + c1] = yi;
      p1 = fma(xi, yi, p1);
    }
  }
}

// acc += sum_{p in [kb, ke)} w_p x[col_p][:]   (NB neighbour rows in flight per warp)
template <int WT, bool PAIR>
__device__ __forceinline__ void b_accumulate(const TileSched& sc, const BatchArgs& a, int64_t kb, int64_t ke,
                                             int lane, double& acc0, double& acc1) {
  constexpr int NB = FJ_SPMM_NB;
  const int k = a.k;
  const int c0 = col0<PAIR>(lane), c1 = col1<PAIR>(lane);
  const bool h0 = c0 < k, h1 = c1 < k;
  for (int64_t kk = kb; kk < ke; kk += NB) {
    const int nb = (int)min((int64_t)NB, ke - kk);
    int32_t cl = 0;
    double wl = 1.0;
    if (lane < nb) {
      cl = __ldg(sc.col + kk + lane);
      FJ_DCHECK(cl >= 0 && cl < sc.ncol);
      if (WT != FJ_W_UNIT) wl = WeightT<WT>::get(sc.w, kk + lane);
    }
    double v0[NB], v1[NB];
#pragma unroll
    for (int u = 0; u < NB; ++u) {
      const int64_t j = __shfl_sync(0xffffffffu, cl, u);
      v0[u] = 0.0;
      v1[u] = 0.0;
      if (u < nb) {
        if (PAIR) {
          if (h0) {
            const double2 t = ld_gather2(a.x + j * k + c0, a.ldmode);
            v0[u] = t.x;
            v1[u] = t.y;
          }
        } else {
          if (h0) v0[u] = __ldg(a.x + j * k + c0);
          if (h1) v1[u] = __ldg(a.x + j * k + c1);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < NB; ++u) {
      if (WT == FJ_W_UNIT) {
        acc0 += v0[u];
        acc1 += v1[u];
      } else {
        const double wu = __shfl_sync(0xffffffffu, wl, u);
        acc0 = fma(wu, v0[u], acc0);
        acc1 = fma(wu, v1[u], acc1);
      }
    }
  }
}

template <int WT, int MODE, bool PAIR>
__global__ void __launch_bounds__(BTPB, FJ_SPMM_MIN_BLOCKS) spmm_kernel(const TileSched sc, const BatchArgs a) {
  __shared__ double s_red[BWPB][MAXK];
  __shared__ bool s_last;
  if (MODE == BM_PCG && *(volatile int32_t*)&a.bs->done) return;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int k = a.k;
  const int c0 = col0<PAIR>(lane), c1 = col1<PAIR>(lane);
  double p0 = 0.0, p1 = 0.0;
  const int64_t nwarps = (int64_t)gridDim.x * BWPB;
  for (int64_t it = (int64_t)blockIdx.x * BWPB + wib; it < sc.n_items; it += nwarps) {
    const ItemMeta cur = sc.items[it];
    const uint32_t type = cur.info >> 30;
    if (type == IT_T) {
      const int R = tile_rows(cur.info);
      const int64_t r0 = cur.r0;
      int64_t rb = cur.k0;
      for (int t = 0; t < R; ++t) {
        const int64_t re = __ldg(sc.row_ptr + r0 + t + 1);
        double acc0 = 0.0, acc1 = 0.0;
        b_accumulate<WT, PAIR>(sc, a, rb, re, lane, acc0, acc1);
        b_finish<WT, MODE, PAIR>(a, r0 + t, re - rb, lane, acc0, acc1, p0, p1);
        rb = re;
      }
    } else {
      const int64_t r = cur.r0;
      const int64_t rb = __ldg(sc.row_ptr + r), re = __ldg(sc.row_ptr + r + 1);
      const int64_t kb = cur.k0;
      const int64_t ke = (type == IT_W) ? re : min(kb + (int64_t)sc.chunk, re);
      double acc0 = 0.0, acc1 = 0.0;
      b_accumulate<WT, PAIR>(sc, a, kb, ke, lane, acc0, acc1);
      if (type == IT_W) {
        b_finish<WT, MODE, PAIR>(a, r, re - rb, lane, acc0, acc1, p0, p1);
      } else {
        const uint32_t l = cur.info & 0x3FFFFFFFu;
        const int64_t first = sc.long_item0[l];
        const int32_t nch = sc.long_nchunks[l];
        if (c0 < MAXK) a.chunk_acc[it * MAXK + c0] = acc0;
        if (c1 < MAXK) a.chunk_acc[it * MAXK + c1] = acc1;
        __threadfence();
        __syncwarp();
        unsigned last = 0;
        if (lane == 0) last = atomicAdd(a.long_ticket + l, 1u) == (unsigned)nch - 1u;
        last = __shfl_sync(0xffffffffu, last, 0);
        if (last) {
          __threadfence();
          double m0 = 0.0, m1 = 0.0;
          for (int32_t c = 0; c < nch; ++c) {   // chunk order
            if (c0 < MAXK) m0 += __ldcg(a.chunk_acc + (first + c) * MAXK + c0);
            if (c1 < MAXK) m1 += __ldcg(a.chunk_acc + (first + c) * MAXK + c1);
          }
          double lp0 = 0.0, lp1 = 0.0;
          b_finish<WT, MODE, PAIR>(a, r, re - rb, lane, m0, m1, lp0, lp1);
          if (c0 < MAXK) a.long_part[(int64_t)l * MAXK + c0] = lp0;
          if (c1 < MAXK) a.long_part[(int64_t)l * MAXK + c1] = lp1;
          if (lane == 0) a.long_ticket[l] = 0u;
        }
      }
    }
  }
  // ---------------- per-column partials: warps in order, then blocks in order (last block)
  if (c0 < MAXK) s_red[wib][c0] = p0;
  if (c1 < MAXK) s_red[wib][c1] = p1;
  __syncthreads();
  if (threadIdx.x < MAXK) {
    double t = 0.0;
    for (int w = 0; w < BWPB; ++w) t += s_red[w][threadIdx.x];
    a.block_part[(int64_t)blockIdx.x * MAXK + threadIdx.x] = t;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(a.grid_ticket, 1u) == gridDim.x - 1u;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  __shared__ double s_tail[BTPB];
  const double t = tail_sum(a.block_part + threadIdx.x % MAXK, gridDim.x, a.long_part + threadIdx.x % MAXK,
                            sc.n_long, MAXK, s_tail);
  if (threadIdx.x < MAXK) {
    const int c = threadIdx.x;
    if (c < k) {
      BatchScalars* bs = a.bs;
      if (MODE == BM_PCG) {
        bs->pq[c] = t;
        if (bs->active[c]) {
          if (!(t > 0.0) || !isfinite(t)) { bs->alpha[c] = 0.0; bs->active[c] = 0; bs->breakdown[c] = 1; }
          else bs->alpha[c] = bs->rho[c] / t;
        } else {
          bs->alpha[c] = 0.0;
        }
      } else if (MODE == BM_RESID) {
        bs->res2[c] = t;
      }
    }
  }
  if (threadIdx.x == 0) *a.grid_ticket = 0u;
}

// ---------------------------------------------------------------- elementwise batched kernels
// warp per row, lane l owns columns l and l+32; per-column partials reduced warps -> blocks.
constexpr int ETB = 256;
constexpr int EWB = ETB / 32;

template <int NP>
__device__ __forceinline__ bool b_elem_reduce(double (&v0)[NP], double (&v1)[NP], double* part /*[grid][NP][64]*/,
                                              unsigned int* ticket, double (*s_red)[NP][MAXK], double (&tot)[NP]) {
  __shared__ bool s_last;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
#pragma unroll
  for (int j = 0; j < NP; ++j) { s_red[wib][j][lane] = v0[j]; s_red[wib][j][lane + 32] = v1[j]; }
  __syncthreads();
  if (threadIdx.x < MAXK) {
#pragma unroll
    for (int j = 0; j < NP; ++j) {
      double t = 0.0;
      for (int w = 0; w < EWB; ++w) t += s_red[w][j][threadIdx.x];
      part[((int64_t)blockIdx.x * NP + j) * MAXK + threadIdx.x] = t;
    }
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(ticket, 1u) == gridDim.x - 1u;
  __syncthreads();
  if (!s_last) return false;
  __threadfence();
  {   // thread group g = t / 64 folds blocks b = g, g + 4, ... for column t % 64; groups summed in order
    constexpr int NG = ETB / MAXK;
    const int c = threadIdx.x & (MAXK - 1), grp = threadIdx.x / MAXK;
    double t[NP];
#pragma unroll
    for (int j = 0; j < NP; ++j) t[j] = 0.0;
    for (unsigned b = grp; b < gridDim.x; b += NG) {
#pragma unroll
      for (int j = 0; j < NP; ++j) t[j] += __ldcg(part + ((int64_t)b * NP + j) * MAXK + c);
    }
    __syncthreads();   // s_red reused: [group][j][column]
#pragma unroll
    for (int j = 0; j < NP; ++j) s_red[grp][j][c] = t[j];
    __syncthreads();
    if (threadIdx.x < MAXK) {
#pragma unroll
      for (int j = 0; j < NP; ++j) {
        double u = 0.0;
        for (int g2 = 0; g2 < NG; ++g2) u += s_red[g2][j][c];
        tot[j] = u;
      }
    }
  }
  return true;
}

__global__ void __launch_bounds__(ETB) k_b_init(int64_t n, int k, const double* __restrict__ s,
                                                const double* __restrict__ dinv, const double* __restrict__ q,
                                                int restart, double* __restrict__ x, double* __restrict__ r,
                                                double* __restrict__ p, BatchScalars* bs, double rtol, int max_iter,
                                                double* part, unsigned int* ticket) {
  __shared__ double s_red[EWB][3][MAXK];
  const int lane = threadIdx.x & 31;
  double v0[3] = {0, 0, 0}, v1[3] = {0, 0, 0};
  const int64_t w0 = (int64_t)blockIdx.x * EWB + (threadIdx.x >> 5), nw = (int64_t)gridDim.x * EWB;
  for (int64_t i = w0; i < n; i += nw) {
    const double di = dinv[i];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int c = lane + 32 * h;
      if (c < k) {
        const int64_t o = i * k + c;
        const double si = s[o];
        const double ri = restart ? si - q[o] : si;
        if (!restart) x[o] = 0.0;
        const double yi = di * ri;
        r[o] = ri;
        p[o] = yi;
        double* v = h ? v1 : v0;
        v[0] = fma(ri, yi, v[0]);
        v[1] = fma(ri, ri, v[1]);
        v[2] = fma(si, si, v[2]);
      }
    }
  }
  double tot[3];
  if (b_elem_reduce<3>(v0, v1, part, ticket, s_red, tot)) {
    const int c = threadIdx.x;
    if (c < k) {
      bs->rho[c] = tot[0];
      bs->rr[c] = tot[1];
      bs->ss[c] = tot[2];
      bs->tol2[c] = rtol * rtol * tot[2];
      const int conv = tot[1] <= rtol * rtol * tot[2];
      bs->conv[c] = conv;
      bs->active[c] = conv ? 0 : 1;
      bs->breakdown[c] = 0;
      bs->alpha[c] = bs->beta[c] = 0.0;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int any = 0;
      for (int j = 0; j < k; ++j) any |= bs->active[j];
      bs->iter = 0;
      bs->max_iter = max_iter;
      bs->k = k;
      bs->done = (!any || max_iter <= 0) ? 1 : 0;
      *ticket = 0u;
    }
  }
}

__global__ void __launch_bounds__(ETB, 8) k_b_update(int64_t n, int k, const double* __restrict__ dinv,
                                                  const double* __restrict__ p, const double* __restrict__ q,
                                                  double* __restrict__ x, double* __restrict__ r, BatchScalars* bs,
                                                  double* part, unsigned int* ticket, cudaGraphConditionalHandle h,
                                                  int use_h) {
  __shared__ double s_red[EWB][2][MAXK];
  if (*(volatile int32_t*)&bs->done) {
    if (use_h && blockIdx.x == 0 && threadIdx.x == 0) cudaGraphSetConditional(h, 0);
    return;
  }
  const int lane = threadIdx.x & 31;
  const bool a0 = lane < k && bs->active[lane], a1 = lane + 32 < k && bs->active[lane + 32];
  const double al0 = a0 ? bs->alpha[lane] : 0.0, al1 = a1 ? bs->alpha[lane + 32] : 0.0;
  double v0[2] = {0, 0}, v1[2] = {0, 0};
  const int64_t w0 = (int64_t)blockIdx.x * EWB + (threadIdx.x >> 5), nw = (int64_t)gridDim.x * EWB;
  for (int64_t i = w0; i < n; i += nw) {
    const double di = dinv[i];
    if (a0) {
      const int64_t o = i * k + lane;
      x[o] = fma(al0, p[o], x[o]);
      const double ri = fma(-al0, q[o], r[o]);
      r[o] = ri;
      v0[0] = fma(ri, di * ri, v0[0]);
      v0[1] = fma(ri, ri, v0[1]);
    }
    if (a1) {
      const int64_t o = i * k + lane + 32;
      x[o] = fma(al1, p[o], x[o]);
      const double ri = fma(-al1, q[o], r[o]);
      r[o] = ri;
      v1[0] = fma(ri, di * ri, v1[0]);
      v1[1] = fma(ri, ri, v1[1]);
    }
  }
  double tot[2];
  if (b_elem_reduce<2>(v0, v1, part, ticket, s_red, tot)) {
    const int c = threadIdx.x;
    if (c < k && bs->active[c]) {
      bs->beta[c] = tot[0] / bs->rho[c];
      bs->rho[c] = tot[0];
      bs->rr[c] = tot[1];
      if (tot[1] <= bs->tol2[c] || !isfinite(tot[1])) { bs->active[c] = 0; bs->conv[c] = tot[1] <= bs->tol2[c]; }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      const int it = bs->iter + 1;
      bs->iter = it;
      int any = 0;
      for (int j = 0; j < k; ++j) any |= bs->active[j];
      if (!any || it >= bs->max_iter) {
        bs->done = 1;
        if (use_h) cudaGraphSetConditional(h, 0);
      }
      *ticket = 0u;
    }
  }
}

__global__ void __launch_bounds__(ETB) k_b_dir(int64_t n, int k, const double* __restrict__ dinv,
                                               const double* __restrict__ r, double* __restrict__ p,
                                               const BatchScalars* bs) {
  if (*(volatile const int32_t*)&bs->done) return;
  const int lane = threadIdx.x & 31;
  const bool a0 = lane < k && bs->active[lane], a1 = lane + 32 < k && bs->active[lane + 32];
  const double b0 = a0 ? bs->beta[lane] : 0.0, b1 = a1 ? bs->beta[lane + 32] : 0.0;
  const int64_t w0 = (int64_t)blockIdx.x * EWB + (threadIdx.x >> 5), nw = (int64_t)gridDim.x * EWB;
  for (int64_t i = w0; i < n; i += nw) {
    const double di = dinv[i];
    if (a0) { const int64_t o = i * k + lane; p[o] = fma(b0, p[o], di * r[o]); }
    if (a1) { const int64_t o = i * k + lane + 32; p[o] = fma(b1, p[o], di * r[o]); }
  }
}

__global__ void k_b_copy(int64_t nk, const double* __restrict__ src, double* __restrict__ dst) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nk; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

// ---------------------------------------------------------------- workspace + launch
struct BatchWs {
  int k = 0;
  int grid_spmm[4] = {0, 0, 0, 0};
  int grid_elem = 0;
  double *r = nullptr, *p = nullptr, *q = nullptr, *x = nullptr;
  BatchScalars* bs = nullptr;
  double *chunk_acc = nullptr, *long_part = nullptr, *block_part = nullptr, *elem_part = nullptr;
  unsigned int *long_ticket = nullptr, *grid_ticket = nullptr, *elem_ticket = nullptr;
  double *q_chunk = nullptr, *q_long = nullptr, *q_block = nullptr, *q_out = nullptr;   // quant_batch
  cudaGraphExec_t exec = nullptr;
  cudaGraph_t graph = nullptr;
  cudaStream_t cap_stream = nullptr;
  cudaEvent_t ev2 = nullptr, ev3 = nullptr;
};

static BatchWs* g_batch_cache(fj_graph* g) { return reinterpret_cast<BatchWs*>(g->batch_ws); }

void free_batch_ws(fj_graph* g) {
  BatchWs* w = g_batch_cache(g);
  if (!w) return;
  if (w->exec) cudaGraphExecDestroy(w->exec);
  if (w->graph) cudaGraphDestroy(w->graph);
  if (w->cap_stream) cudaStreamDestroy(w->cap_stream);
  if (w->ev2) cudaEventDestroy(w->ev2);
  if (w->ev3) cudaEventDestroy(w->ev3);
  dfree(w->r); dfree(w->p); dfree(w->q); dfree(w->x); dfree(w->bs);
  dfree(w->chunk_acc); dfree(w->long_part); dfree(w->block_part); dfree(w->elem_part);
  dfree(w->long_ticket); dfree(w->grid_ticket); dfree(w->elem_ticket);
  dfree(w->q_chunk); dfree(w->q_long); dfree(w->q_block); dfree(w->q_out);
  delete w;
  g->batch_ws = nullptr;
}

template <class T>
static fj_status balloc(T** p, int64_t count, cudaStream_t st, bool zero = false) {
  if (count < 1) count = 1;
  FJ_CK(dmalloc(p, sizeof(T) * (size_t)count, st));
  if (zero) FJ_CK(cudaMemsetAsync(*p, 0, sizeof(T) * (size_t)count, st));
  return FJ_OK;
}

static fj_status get_batch_ws(fj_graph* g, int k, cudaStream_t st, BatchWs** out) {
  BatchWs* w = g_batch_cache(g);
  if (w && w->k == k) { *out = w; return FJ_OK; }
  if (w) {
    FJ_CK(cudaStreamSynchronize(st));   // the old buffers may still be in use on st
    free_batch_ws(g);
  }
  w = new BatchWs();
  g->batch_ws = w;
  w->k = k;
  const int64_t nk = g->n * (int64_t)k;
  FJ_TRY(balloc(&w->r, nk, st)); FJ_TRY(balloc(&w->p, nk, st));
  FJ_TRY(balloc(&w->q, nk, st)); FJ_TRY(balloc(&w->x, nk, st));
  FJ_TRY(balloc(&w->bs, 1, st, true));
  const int64_t gmax = (int64_t)g->num_sms * (2048 / BTPB);
  if (!g->sb.built) FJ_TRY(build_schedule(g, kSchedBatch, g->sb, st));
  FJ_TRY(balloc(&w->chunk_acc, g->sb.n_long_chunks * MAXK, st));
  FJ_TRY(balloc(&w->long_part, g->sb.n_long * MAXK, st));
  FJ_TRY(balloc(&w->block_part, gmax * MAXK, st));
  FJ_TRY(balloc(&w->long_ticket, g->sb.n_long, st, true));
  FJ_TRY(balloc(&w->grid_ticket, 1, st, true));
  int64_t ge = (int64_t)g->num_sms * (2048 / ETB);
  const int64_t need = (g->n + EWB - 1) / EWB;
  if (ge > need) ge = need > 0 ? need : 1;
  w->grid_elem = (int)ge;
  FJ_TRY(balloc(&w->elem_part, ge * 3 * MAXK, st));
  FJ_TRY(balloc(&w->elem_ticket, 1, st, true));
  FJ_CK(cudaEventCreate(&w->ev2));
  FJ_CK(cudaEventCreate(&w->ev3));
  *out = w;
  return FJ_OK;
}

template <int WT, int MODE, bool PAIR>
static fj_status launch_spmm_p(const fj_graph* g, BatchWs* w, const BatchArgs& a, cudaStream_t st) {
  static int occ = 0;
  if (occ == 0) {
    FJ_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, spmm_kernel<WT, MODE, PAIR>, BTPB, 0));
    if (occ < 1) occ = 1;
  }
  int64_t grid = (int64_t)g->num_sms * occ;
  const int64_t need = (g->sb.n_items + BWPB - 1) / BWPB;
  if (grid > need) grid = need > 0 ? need : 1;
  const int64_t gmax = (int64_t)g->num_sms * (2048 / BTPB);
  if (grid > gmax) grid = gmax;
  spmm_kernel<WT, MODE, PAIR><<<(unsigned)grid, BTPB, 0, st>>>(make_sched(g, g->sb), a);
  FJ_CK_LAUNCH();
  return FJ_OK;
}

template <int WT, int MODE>
static fj_status launch_spmm_wt(const fj_graph* g, BatchWs* w, const BatchArgs& a, cudaStream_t st) {
  const bool pair = (a.k % 2 == 0) && ((reinterpret_cast<uintptr_t>(a.x) & 15) == 0);
  return pair ? launch_spmm_p<WT, MODE, true>(g, w, a, st) : launch_spmm_p<WT, MODE, false>(g, w, a, st);
}

template <int MODE>
static fj_status launch_spmm(const fj_graph* g, BatchWs* w, const BatchArgs& a, cudaStream_t st) {
  switch (g->wtype) {
    case FJ_W_UNIT: return launch_spmm_wt<FJ_W_UNIT, MODE>(g, w, a, st);
    case FJ_W_U8: return launch_spmm_wt<FJ_W_U8, MODE>(g, w, a, st);
    case FJ_W_F32: return launch_spmm_wt<FJ_W_F32, MODE>(g, w, a, st);
    default: return launch_spmm_wt<FJ_W_F64, MODE>(g, w, a, st);
  }
}

static BatchArgs make_args(const fj_graph* g, BatchWs* w, int k, const double* x, double* y, const double* s, int opL) {
  BatchArgs a;
  // measured on B200 (C4 scale 22, k = 64): plain ld.global 8.4 ms, ld.global.nc 8.9 ms,
  // ld.global.nc.L1::no_allocate 9.6 ms per product -> default 1
  static const int ldmode = [] { const char* e = getenv("FJ_GATHER_MODE"); return e ? atoi(e) : 1; }();
  a.k = k; a.ldmode = ldmode; a.x = x; a.y = y; a.s = s; a.deg = g->deg; a.opL = opL; a.bs = w->bs;
  a.chunk_acc = w->chunk_acc; a.long_part = w->long_part; a.long_ticket = w->long_ticket;
  a.block_part = w->block_part; a.grid_ticket = w->grid_ticket;
  return a;
}

static fj_status batch_iteration(const fj_graph* g, BatchWs* w, cudaStream_t st, cudaGraphConditionalHandle h,
                                 int use_h) {
  const int k = w->k;
  FJ_TRY(launch_spmm<BM_PCG>(g, w, make_args(g, w, k, w->p, w->q, nullptr, 0), st));
  k_b_update<<<w->grid_elem, ETB, 0, st>>>(g->n, k, g->dinv, w->p, w->q, w->x, w->r, w->bs, w->elem_part,
                                           w->elem_ticket, h, use_h);
  FJ_CK_LAUNCH();
  k_b_dir<<<w->grid_elem, ETB, 0, st>>>(g->n, k, g->dinv, w->r, w->p, w->bs);
  FJ_CK_LAUNCH();
  return FJ_OK;
}

static fj_status build_batch_graph(fj_graph* g, BatchWs* w) {
  if (w->exec) return FJ_OK;
  FJ_CK(cudaStreamCreateWithFlags(&w->cap_stream, cudaStreamNonBlocking));
  FJ_CK(cudaGraphCreate(&w->graph, 0));
  cudaGraphConditionalHandle h;
  FJ_CK(cudaGraphConditionalHandleCreate(&h, w->graph, 1, cudaGraphCondAssignDefault));
  alignas(cudaGraphNodeParams) unsigned char raw[sizeof(cudaGraphNodeParams)];
  memset(raw, 0, sizeof raw);
  cudaGraphNodeParams& cp = *reinterpret_cast<cudaGraphNodeParams*>(raw);
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = h;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t node;
  FJ_CK(cudaGraphAddNode(&node, w->graph, nullptr, 0, &cp));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  FJ_CK(cudaStreamBeginCaptureToGraph(w->cap_stream, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  g_capturing = true;
  fj_status s = batch_iteration(g, w, w->cap_stream, h, 1);
  g_capturing = false;
  cudaGraph_t captured = nullptr;
  cudaError_t e = cudaStreamEndCapture(w->cap_stream, &captured);
  FJ_TRY(s);
  FJ_CK(e);
  FJ_CK(cudaGraphInstantiate(&w->exec, w->graph, 0));
  return FJ_OK;
}

// Batched solve of all k columns of s [n][k] into z [n][k].  warm: z holds the starting iterate.
// Per-column true residuals are recomputed after the loop; columns missing rtol restart (all
// columns together, warm) up to max_restarts times.
fj_status solve_batch(fj_graph* g, int k, const double* s, double* z, const fj_solve_opts& o, int warm,
                      fj_solve_report* rep, cudaStream_t st, bool defer_true_residual) {
  if (vec_supported(k)) return solve_vec(g, k, s, z, o, warm, rep, st, defer_true_residual);
  BatchWs* w = nullptr;
  FJ_TRY(get_batch_ws(g, k, st, &w));
  const int64_t nk = g->n * (int64_t)k;
  const unsigned cb = (unsigned)std::min<int64_t>((nk + 255) / 256, 8192);
  if (o.use_cuda_graph) FJ_TRY(build_batch_graph(g, w));
  BatchScalars h;
  int restarts = 0, total_iter = 0;
  bool first = true;
  for (;;) {
    const bool restart = !first || warm;
    if (restart) {
      if (first) { k_b_copy<<<cb, 256, 0, st>>>(nk, z, w->x); FJ_CK_LAUNCH(); }
      FJ_TRY(launch_spmm<BM_APPLY>(g, w, make_args(g, w, k, w->x, w->q, nullptr, 0), st));
    }
    const int budget = std::max(0, o.max_iter - total_iter);
    FJ_CK(cudaEventRecord(w->ev2, st));
    k_b_init<<<w->grid_elem, ETB, 0, st>>>(g->n, k, s, g->dinv, w->q, restart ? 1 : 0, w->x, w->r, w->p, w->bs,
                                           o.rtol, budget, w->elem_part, w->elem_ticket);
    FJ_CK_LAUNCH();
    first = false;
    if (o.use_cuda_graph) {
      FJ_CK(cudaGraphLaunch(w->exec, st));
    } else {
      for (;;) {
        for (int u = 0; u < 8; ++u) FJ_TRY(batch_iteration(g, w, st, 0, 0));
        int32_t done = 0;
        FJ_CK(cudaMemcpyAsync(&done, &w->bs->done, sizeof done, cudaMemcpyDeviceToHost, st));
        FJ_CK(cudaStreamSynchronize(st));
        if (done) break;
      }
    }
    FJ_CK(cudaEventRecord(w->ev3, st));
    FJ_TRY(launch_spmm<BM_RESID>(g, w, make_args(g, w, k, w->x, nullptr, s, 0), st));
    FJ_CK(cudaMemcpyAsync(&h, w->bs, sizeof h, cudaMemcpyDeviceToHost, st));
    FJ_CK(cudaStreamSynchronize(st));
    total_iter += h.iter;
    if (o.use_cuda_graph) count_launch(3 * std::max(h.iter, 1));
    float lms = 0.f;
    cudaEventElapsedTime(&lms, w->ev2, w->ev3);
    if (rep) { rep->ms_loop += lms; rep->iterations_total += (int64_t)h.iter * k; }
    bool ok = true, brk = false;
    for (int c = 0; c < k; ++c) {
      if (h.res2[c] > h.tol2[c]) ok = false;
      if (h.breakdown[c]) brk = true;
    }
    if (ok || restarts >= o.max_restarts || total_iter >= o.max_iter || brk) break;
    ++restarts;
  }
  k_b_copy<<<cb, 256, 0, st>>>(nk, w->x, z);
  FJ_CK_LAUNCH();
  bool converged = true;
  double worst_true = 0.0, worst_rec = 0.0;
  for (int c = 0; c < k; ++c) {
    if (h.res2[c] > h.tol2[c]) converged = false;
    if (h.ss[c] > 0) {
      worst_true = std::max(worst_true, std::sqrt(h.res2[c] / h.ss[c]));
      worst_rec = std::max(worst_rec, std::sqrt(h.rr[c] / h.ss[c]));
    }
  }
  if (rep) {
    rep->iterations = std::max(rep->iterations, total_iter);
    rep->restarts = std::max(rep->restarts, restarts);
    rep->batch_k = k;
    rep->rel_res_recursive = std::max(rep->rel_res_recursive, worst_rec);
    rep->rel_res_true = std::isnan(rep->rel_res_true) ? worst_true : std::max(rep->rel_res_true, worst_true);
    if (!converged) rep->converged = 0;
  }
  return converged ? FJ_OK : fail(FJ_E_NO_CONVERGENCE, "batched PCG did not reach rtol on the true residual");
}

fj_status apply_batch(fj_graph* g, int k, const double* x, double* y, int opL, cudaStream_t st) {
  if (vec_supported(k)) return apply_vec(g, k, x, y, opL, st);
  BatchWs* w = nullptr;
  FJ_TRY(get_batch_ws(g, k, st, &w));
  return launch_spmm<BM_APPLY>(g, w, make_args(g, w, k, x, y, nullptr, opL), st);
}

// Device time of one batched product q = (I+L) p on the solver's own buffers (bench roofline).
fj_status time_batch_spmv(fj_graph* g, int k, int reps, float* ms_out, cudaStream_t st) {
  if (vec_supported(k)) return time_vec_spmv(g, k, reps, ms_out, st);
  BatchWs* w = nullptr;
  FJ_TRY(get_batch_ws(g, k, st, &w));
  const BatchArgs a = make_args(g, w, k, w->p, w->q, nullptr, 0);
  FJ_TRY(launch_spmm<BM_APPLY>(g, w, a, st));
  FJ_CK(cudaEventRecord(w->ev2, st));
  for (int i = 0; i < reps; ++i) FJ_TRY(launch_spmm<BM_APPLY>(g, w, a, st));
  FJ_CK(cudaEventRecord(w->ev3, st));
  FJ_CK(cudaEventSynchronize(w->ev3));
  float ms = 0.f;
  FJ_CK(cudaEventElapsedTime(&ms, w->ev2, w->ev3));
  *ms_out = ms / (float)std::max(reps, 1);
  return FJ_OK;
}

// ---------------------------------------------------------------- batched fused quantities (a6, k cols)
// Same traversal as spmm_kernel; per row and column: A = sum w z_j, Dd = sum w (z_i - z_j)^2,
// Aa = sum w |z_j|, then the 10 per-row contributions of QuantOp (ops.cuh) for each column.
constexpr int QNP = 10;

struct QuantArgs {
  int k;
  const double* __restrict__ z;    // [n][k]
  const double* __restrict__ s;    // [n][k]
  const double* __restrict__ deg;
  const double* __restrict__ mean; // [k] mean of s per column
  double* chunk_acc;               // [n_chunks][3][64]
  double* long_part;               // [n_long][10][64]
  unsigned int* long_ticket;
  double* block_part;              // [grid][10][64]
  unsigned int* grid_ticket;
  double* out;                     // [10][64]
};

template <int WT, bool PAIR>
__device__ __forceinline__ void q_accumulate(const TileSched& sc, const QuantArgs& a, int64_t kb, int64_t ke, int lane,
                                             double zi0, double zi1, double (&acc)[6]) {
  constexpr int NB = 8;
  const int k = a.k;
  const int c0 = col0<PAIR>(lane), c1 = col1<PAIR>(lane);
  const bool h0 = c0 < k, h1 = c1 < k;
  for (int64_t kk = kb; kk < ke; kk += NB) {
    const int nb = (int)min((int64_t)NB, ke - kk);
    int32_t cl = 0;
    double wl = 1.0;
    if (lane < nb) {
      cl = __ldg(sc.col + kk + lane);
      FJ_DCHECK(cl >= 0 && cl < sc.ncol);
      if (WT != FJ_W_UNIT) wl = WeightT<WT>::get(sc.w, kk + lane);
    }
    double v0[NB], v1[NB];
#pragma unroll
    for (int u = 0; u < NB; ++u) {
      const int64_t j = __shfl_sync(0xffffffffu, cl, u);
      v0[u] = 0.0;
      v1[u] = 0.0;
      if (u < nb) {
        if (PAIR) {
          if (h0) { const double2 t = ld_gather2(a.z + j * k + c0, 1); v0[u] = t.x; v1[u] = t.y; }
        } else {
          if (h0) v0[u] = ld_plain(a.z + j * k + c0);
          if (h1) v1[u] = ld_plain(a.z + j * k + c1);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < NB; ++u) {
      const double wu = (WT == FJ_W_UNIT) ? 1.0 : __shfl_sync(0xffffffffu, wl, u);
      if (u < nb) {
        const double d0 = zi0 - v0[u], d1 = zi1 - v1[u];
        acc[0] = fma(wu, v0[u], acc[0]);
        acc[1] = fma(wu * d0, d0, acc[1]);
        acc[2] = fma(wu, fabs(v0[u]), acc[2]);
        acc[3] = fma(wu, v1[u], acc[3]);
        acc[4] = fma(wu * d1, d1, acc[4]);
        acc[5] = fma(wu, fabs(v1[u]), acc[5]);
      }
    }
  }
}

template <int WT>
__device__ __forceinline__ void q_finish_col(const QuantArgs& a, int64_t i, int c, double d, double zi, double A,
                                             double Dd, double Aa, double (&p)[QNP]) {
  const double si = a.s[i * a.k + c], m = a.mean[c];
  const double t = fma(1.0 + d, zi, -A);
  const double lz = fma(d, zi, -A);
  const double r = si - t;
  const double e1 = zi - si, e2 = zi - m, e3 = si - m;
  const double ab = fabs(si) + fma(1.0 + d, fabs(zi), Aa);
  p[0] = fma(e1, e1, p[0]);
  p[1] += Dd;
  p[2] = fma(e2, e2, p[2]);
  p[3] = fma(zi, zi, p[3]);
  p[4] = fma(si, zi, p[4]);
  p[5] = fma(e3, e2, p[5]);
  p[6] = fma(r, r, p[6]);
  p[7] = fma(lz, lz, p[7]);
  p[8] = fma(ab, ab, p[8]);
  p[9] = fma(si, si, p[9]);
}

template <int WT, bool PAIR>
__device__ __forceinline__ void q_row(const QuantArgs& a, int64_t i, int64_t len, int lane, double zi0, double zi1,
                                      const double (&acc)[6], double (&p0)[QNP], double (&p1)[QNP]) {
  const double d = (WT == FJ_W_UNIT) ? (double)len : a.deg[i];
  const int c0 = col0<PAIR>(lane), c1 = col1<PAIR>(lane);
  if (c0 < a.k) q_finish_col<WT>(a, i, c0, d, zi0, acc[0], acc[1], acc[2], p0);
  if (c1 < a.k) q_finish_col<WT>(a, i, c1, d, zi1, acc[3], acc[4], acc[5], p1);
}

template <int WT, bool PAIR>
__global__ void __launch_bounds__(BTPB, FJ_QB_MIN_BLOCKS) quant_batch_kernel(const TileSched sc, const QuantArgs a) {
  __shared__ double s_red[BWPB][MAXK];
  __shared__ bool s_last;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int k = a.k;
  const int c0 = col0<PAIR>(lane), c1 = col1<PAIR>(lane);
  double p0[QNP], p1[QNP];
#pragma unroll
  for (int j = 0; j < QNP; ++j) { p0[j] = 0.0; p1[j] = 0.0; }
  auto zrow = [&](int64_t i, double& z0, double& z1) {
    z0 = c0 < k ? a.z[i * k + c0] : 0.0;
    z1 = c1 < k ? a.z[i * k + c1] : 0.0;
  };
  const int64_t nwarps = (int64_t)gridDim.x * BWPB;
  for (int64_t it = (int64_t)blockIdx.x * BWPB + wib; it < sc.n_items; it += nwarps) {
    const ItemMeta cur = sc.items[it];
    const uint32_t type = cur.info >> 30;
    if (type == IT_T) {
      const int R = tile_rows(cur.info);
      const int64_t r0 = cur.r0;
      int64_t rb = cur.k0;
      for (int t = 0; t < R; ++t) {
        const int64_t re = __ldg(sc.row_ptr + r0 + t + 1);
        double z0, z1, acc[6] = {0, 0, 0, 0, 0, 0};
        zrow(r0 + t, z0, z1);
        q_accumulate<WT, PAIR>(sc, a, rb, re, lane, z0, z1, acc);
        q_row<WT, PAIR>(a, r0 + t, re - rb, lane, z0, z1, acc, p0, p1);
        rb = re;
      }
    } else {
      const int64_t r = cur.r0;
      const int64_t rb = __ldg(sc.row_ptr + r), re = __ldg(sc.row_ptr + r + 1);
      const int64_t kb = cur.k0;
      const int64_t ke = (type == IT_W) ? re : min(kb + (int64_t)sc.chunk, re);
      double z0, z1, acc[6] = {0, 0, 0, 0, 0, 0};
      zrow(r, z0, z1);
      q_accumulate<WT, PAIR>(sc, a, kb, ke, lane, z0, z1, acc);
      if (type == IT_W) {
        q_row<WT, PAIR>(a, r, re - rb, lane, z0, z1, acc, p0, p1);
      } else {
        const uint32_t l = cur.info & 0x3FFFFFFFu;
        const int64_t first = sc.long_item0[l];
        const int32_t nch = sc.long_nchunks[l];
#pragma unroll
        for (int f = 0; f < 3; ++f) {
          if (c0 < MAXK) a.chunk_acc[(it * 3 + f) * MAXK + c0] = acc[f];
          if (c1 < MAXK) a.chunk_acc[(it * 3 + f) * MAXK + c1] = acc[3 + f];
        }
        __threadfence();
        __syncwarp();
        unsigned last = 0;
        if (lane == 0) last = atomicAdd(a.long_ticket + l, 1u) == (unsigned)nch - 1u;
        last = __shfl_sync(0xffffffffu, last, 0);
        if (last) {
          __threadfence();
          double m[6] = {0, 0, 0, 0, 0, 0};
          for (int32_t c = 0; c < nch; ++c) {   // chunk order
#pragma unroll
            for (int f = 0; f < 3; ++f) {
              if (c0 < MAXK) m[f] += __ldcg(a.chunk_acc + ((first + c) * 3 + f) * MAXK + c0);
              if (c1 < MAXK) m[3 + f] += __ldcg(a.chunk_acc + ((first + c) * 3 + f) * MAXK + c1);
            }
          }
          double l0[QNP], l1[QNP];
#pragma unroll
          for (int j = 0; j < QNP; ++j) { l0[j] = 0.0; l1[j] = 0.0; }
          q_row<WT, PAIR>(a, r, re - rb, lane, z0, z1, m, l0, l1);
#pragma unroll
          for (int j = 0; j < QNP; ++j) {
            if (c0 < MAXK) a.long_part[((int64_t)l * QNP + j) * MAXK + c0] = l0[j];
            if (c1 < MAXK) a.long_part[((int64_t)l * QNP + j) * MAXK + c1] = l1[j];
          }
          if (lane == 0) a.long_ticket[l] = 0u;
        }
      }
    }
  }
  // per-column partials, one quantity at a time: warps in order, then blocks in order
#pragma unroll
  for (int j = 0; j < QNP; ++j) {
    if (c0 < MAXK) s_red[wib][c0] = p0[j];
    if (c1 < MAXK) s_red[wib][c1] = p1[j];
    __syncthreads();
    if (threadIdx.x < MAXK) {
      double t = 0.0;
      for (int w = 0; w < BWPB; ++w) t += s_red[w][threadIdx.x];
      a.block_part[((int64_t)blockIdx.x * QNP + j) * MAXK + threadIdx.x] = t;
    }
    __syncthreads();
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(a.grid_ticket, 1u) == gridDim.x - 1u;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  __shared__ double s_tail[BTPB];
  for (int j = 0; j < QNP; ++j) {
    const int c = threadIdx.x % MAXK;
    const double t = tail_sum(a.block_part + (int64_t)j * MAXK + c, gridDim.x, a.long_part + (int64_t)j * MAXK + c,
                              sc.n_long, (int64_t)QNP * MAXK, s_tail);
    if (threadIdx.x < MAXK) a.out[j * MAXK + c] = t;
  }
  if (threadIdx.x == 0) *a.grid_ticket = 0u;
}

template <int WT, bool PAIR>
static fj_status launch_quant_batch_p(const fj_graph* g, const QuantArgs& a, cudaStream_t st) {
  static int occ = 0;
  if (occ == 0) {
    FJ_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, quant_batch_kernel<WT, PAIR>, BTPB, 0));
    if (occ < 1) occ = 1;
  }
  int64_t grid = (int64_t)g->num_sms * occ;
  const int64_t need = (g->sb.n_items + BWPB - 1) / BWPB;
  if (grid > need) grid = need > 0 ? need : 1;
  quant_batch_kernel<WT, PAIR><<<(unsigned)grid, BTPB, 0, st>>>(make_sched(g, g->sb), a);
  FJ_CK_LAUNCH();
  return FJ_OK;
}

template <int WT>
static fj_status launch_quant_batch_wt(const fj_graph* g, const QuantArgs& a, cudaStream_t st) {
  const bool pair = (a.k % 2 == 0) && ((reinterpret_cast<uintptr_t>(a.z) & 15) == 0);
  return pair ? launch_quant_batch_p<WT, true>(g, a, st) : launch_quant_batch_p<WT, false>(g, a, st);
}

// All k columns' 10 sums in one pass: host_out[c * 10 + j] (same order as QuantOp's partials).
fj_status quant_batch(fj_graph* g, int k, const double* s, const double* z, const double* mean_host,
                      double* host_out, cudaStream_t st, bool z_from_solve) {
  if (vec_supported(k)) return quant_vec(g, k, s, z, mean_host, host_out, z_from_solve, st);
  BatchWs* w = nullptr;
  FJ_TRY(get_batch_ws(g, k, st, &w));
  if (!w->q_chunk) {
    FJ_TRY(balloc(&w->q_chunk, g->sb.n_long_chunks * 3 * MAXK, st));
    FJ_TRY(balloc(&w->q_long, g->sb.n_long * QNP * MAXK, st));
    FJ_TRY(balloc(&w->q_block, (int64_t)g->num_sms * (2048 / BTPB) * QNP * MAXK, st));
    FJ_TRY(balloc(&w->q_out, QNP * MAXK + MAXK, st));
  }
  FJ_CK(cudaMemcpyAsync(w->q_out + QNP * MAXK, mean_host, sizeof(double) * k, cudaMemcpyHostToDevice, st));
  QuantArgs a;
  a.k = k; a.z = z; a.s = s; a.deg = g->deg; a.mean = w->q_out + QNP * MAXK;
  a.chunk_acc = w->q_chunk; a.long_part = w->q_long; a.long_ticket = w->long_ticket;
  a.block_part = w->q_block; a.grid_ticket = w->grid_ticket; a.out = w->q_out;
  switch (g->wtype) {
    case FJ_W_UNIT: FJ_TRY(launch_quant_batch_wt<FJ_W_UNIT>(g, a, st)); break;
    case FJ_W_U8: FJ_TRY(launch_quant_batch_wt<FJ_W_U8>(g, a, st)); break;
    case FJ_W_F32: FJ_TRY(launch_quant_batch_wt<FJ_W_F32>(g, a, st)); break;
    default: FJ_TRY(launch_quant_batch_wt<FJ_W_F64>(g, a, st)); break;
  }
  std::vector<double> h(QNP * MAXK);
  FJ_CK(cudaMemcpyAsync(h.data(), w->q_out, sizeof(double) * QNP * MAXK, cudaMemcpyDeviceToHost, st));
  FJ_CK(cudaStreamSynchronize(st));
  for (int c = 0; c < k; ++c)
    for (int j = 0; j < QNP; ++j) host_out[c * QNP + j] = h[j * MAXK + c];
  return FJ_OK;
}

}  // namespace fj

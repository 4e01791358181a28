// spmv_vec.cu — row a9 for SMALL k (2 <= k <= 4): the k opinion columns are solved together on
// the k = 1 warp-item engine (tiles.cuh) with a VECTOR value per nonzero.
//
// Why: the SpMV on these graphs is bound by the random 8-byte gathers (one L2 sector request per
// nonzero), not by HBM.  Solving the columns one by one pays that request cost k
// times.  Here the solver's vectors are row-major [n][KP] with KP = 2 (k = 2) or KP = 4 (k = 3, 4),
// zero-padded, 32-byte aligned, so one neighbour row is ONE aligned 16/32-byte load (LDG.128 /
// LDG.E.ENL2.256) = one L2 sector for all k columns.  The warp-per-row batched engine (spmm.cu)
// would leave 32 - k lanes idle at this k.
//
// Per PCG iteration (same algebra as pcg.cu, per column):
//   K_A warp_kernel<ApplyOpV>  q = (I+L) p (all columns), pq_c = p_c^T q_c -> alpha_c   (last block)
//   K_B k_v_update             r -= alpha q, rho'_c, ||r_c||^2 -> beta_c,
//                              per-column convergence mask, loop condition             (last block)
//   K_C k_v_dir                x += alpha p (old p), then p = dinv o r + beta p; after the final
//                              iteration only the x update (the multi-GPU path keeps x in K_B)
// in one CUDA graph with a device-driven conditional WHILE node.  Columns that converged keep
// alpha_c = 0 (x_c, r_c frozen).  All partial sums are formed and combined in a fixed order:
// results are bitwise reproducible.
#include <cstring>
#include <vector>

#include "ops.cuh"
#include "rows.cuh"
#include "vec.cuh"
#include "workspace.cuh"

namespace fj {

// ---------------------------------------------------------------- row operators (tiles.cuh Op)
// q = (I+L) p or L p for the KQ real columns of a padded [n][KP] block (P:L88 L = D - A): the
// gathered row is the whole KP-wide vector (one aligned load), but only the KQ real columns are
// accumulated, carried through the warp's segmented scan and stored (k = 3: 3 of 4 lanes of work).
template <int WT, int KP, int KQ = KP>   // y stored KQ wide
struct ApplyOpV {
  using V = DVec<KP>;
  static constexpr int ITEMS = VEC_ITEMS;
  static constexpr int TILE_ROWS = VEC_TILE_ROWS;
  static constexpr int MIN_BLOCKS = engine_min_blocks<V>();
  static constexpr bool TMA = true;
  static constexpr int NA = KQ, NP = KQ;
  static constexpr bool NEEDS_XI = false;
  static __device__ __forceinline__ V vzero() { return vzero_kp<KP>(); }
  const double* __restrict__ x;
  double* __restrict__ y;
  const double* __restrict__ deg;
  int opL;
  VecScalars* sc;   // PCG mode when non-null: alpha_c = rho_c / p_c^T q_c on device
  int k;
  double* dot_out = nullptr;   // optional: p_c^T q_c per column (distributed: local part)
  int alpha_on_device = 1;     // 0 (distributed): alpha after the allreduce of dot_out
  __device__ __forceinline__ bool skip() const { return sc && *(volatile int32_t*)&sc->done; }
  __device__ __forceinline__ bool wants_xi() const { return true; }
  __device__ __forceinline__ V gather(int32_t j) const { return ld_vec<KP>(x + (int64_t)j * KP); }
  __device__ __forceinline__ V row_value(int64_t i) const { return ld_vec<KP>(x + i * KP); }
  __device__ __forceinline__ const V* xi_base() const { return reinterpret_cast<const V*>(x); }
  __device__ __forceinline__ void add(double (&a)[NA], double w, const V& xj, const V&) const {
#pragma unroll
    for (int c = 0; c < KQ; ++c) a[c] = (WT == FJ_W_UNIT) ? a[c] + xj.v[c] : fma(w, xj.v[c], a[c]);
  }
  template <class P>
  __device__ __forceinline__ void finish_row(int64_t i, int64_t len, const V& xi, const double (&a)[NA],
                                             P& part) const {
    V yv;
    const double d = (WT == FJ_W_UNIT) ? (double)len : deg[i];
    const double dd = opL ? d : 1.0 + d;
#pragma unroll
    for (int c = 0; c < KP; ++c) yv.v[c] = c < KQ ? fma(dd, xi.v[c], -a[c < KQ ? c : 0]) : 0.0;
#pragma unroll
    for (int c = 0; c < KQ; ++c) part[c] = fma(xi.v[c], yv.v[c], part[c]);
    st_q<KP, KQ>(y, i, yv);
  }
  __device__ __forceinline__ void finalize(const double (&tot)[NP]) const {
    if (dot_out) {
#pragma unroll
      for (int c = 0; c < KQ; ++c) dot_out[c] = tot[c];
    }
    if (!sc || !alpha_on_device) return;
#pragma unroll
    for (int c = 0; c < KQ; ++c) {
      if (c >= k) break;
      sc->pq[c] = tot[c];
      if (sc->active[c]) {
        if (!(tot[c] > 0.0) || !isfinite(tot[c])) {   // I+L is SPD: p^T q > 0 unless p = 0
          sc->alpha[c] = 0.0;
          sc->active[c] = 0;
          sc->breakdown[c] = 1;
        } else {
          sc->alpha[c] = sc->rho[c] / tot[c];
        }
      } else {
        sc->alpha[c] = 0.0;
      }
    }
  }
};

// ||s_c - (I+L) z_c||^2 per column: z padded [n][KP], s the caller's [n][k].
template <int WT, int KP>
struct ResidOpV {
  using V = DVec<KP>;
  static constexpr int ITEMS = VEC_ITEMS;
  static constexpr int TILE_ROWS = VEC_TILE_ROWS;
  static constexpr int MIN_BLOCKS = engine_min_blocks<V>();
  static constexpr bool TMA = true;
  static constexpr int NA = KP, NP = KP;
  static constexpr bool NEEDS_XI = false;
  static __device__ __forceinline__ V vzero() { return vzero_kp<KP>(); }
  const double* __restrict__ z;
  const double* __restrict__ s;
  const double* __restrict__ deg;
  int k;
  VecScalars* sc;
  __device__ __forceinline__ bool skip() const { return false; }
  __device__ __forceinline__ bool wants_xi() const { return true; }
  __device__ __forceinline__ V gather(int32_t j) const { return ld_vec<KP>(z + (int64_t)j * KP); }
  __device__ __forceinline__ V row_value(int64_t i) const { return ld_vec<KP>(z + i * KP); }
  __device__ __forceinline__ const V* xi_base() const { return reinterpret_cast<const V*>(z); }
  __device__ __forceinline__ void add(double (&a)[NA], double w, const V& xj, const V&) const {
#pragma unroll
    for (int c = 0; c < KP; ++c) a[c] = (WT == FJ_W_UNIT) ? a[c] + xj.v[c] : fma(w, xj.v[c], a[c]);
  }
  template <class P>
  __device__ __forceinline__ void finish_row(int64_t i, int64_t len, const V& zi, const double (&a)[NA],
                                             P& part) const {
    const double d = (WT == FJ_W_UNIT) ? (double)len : deg[i];
#pragma unroll
    for (int c = 0; c < KP; ++c) {
      if (c < k) {
        const double r = s[i * k + c] - fma(1.0 + d, zi.v[c], -a[c]);
        part[c] = fma(r, r, part[c]);
      }
    }
  }
  __device__ __forceinline__ void finalize(const double (&tot)[NP]) const {
#pragma unroll
    for (int c = 0; c < KP; ++c)
      if (c < k) sc->res2[c] = tot[c];
  }
};

// Quantities pass (rows a5-a7) for all columns at once, split in two: the four sums that need the
// neighbours (this row operator: part[j * KP + c], j = 0 Dd = sum_j w (z_i - z_j)^2, 1 (s - (I+L)z)^2,
// 2 (Lz)^2, 3 rounding allowance^2) and the six row-local sums of QuantOp (k_quant_local).  40
// per-thread partials in one kernel cost 255 registers and 2 blocks / SM (2.2 ms on C3); split,
// the row operator runs at the product's occupancy.
#ifndef FJ_QUANTV_PART_SMEM
#define FJ_QUANTV_PART_SMEM 1
#endif
template <int WT, int KP, int KQ>
struct QuantOpV {   // gathers the padded [n][KP] z; accumulates only the KQ = k real columns
  using V = DVec<KP>;
  static constexpr int ITEMS = VEC_ITEMS;
  static constexpr int TILE_ROWS = VEC_TILE_ROWS;
  static constexpr int MIN_BLOCKS = FJ_QUANTV_MIN_BLOCKS >= 0 ? FJ_QUANTV_MIN_BLOCKS : (KQ <= 3 && WT == FJ_W_UNIT ? 4 : 3);
  static constexpr bool TMA = true;
  static constexpr int NA = 3 * KQ, NP = 4 * KQ;
  static constexpr bool NEEDS_XI = true;
  static constexpr bool PART_SMEM = FJ_QUANTV_PART_SMEM != 0;   // 4 KQ partials off the registers
  static __device__ __forceinline__ V vzero() { return vzero_kp<KP>(); }
  const double* __restrict__ z;   // padded [n][KP]
  const double* __restrict__ s;   // [n][k]
  const double* __restrict__ deg;
  double* out;                    // [4][KP]
  __device__ __forceinline__ bool skip() const { return false; }
  __device__ __forceinline__ bool wants_xi() const { return true; }
  __device__ __forceinline__ V gather(int32_t j) const { return ld_vec<KP>(z + (int64_t)j * KP); }
  __device__ __forceinline__ V row_value(int64_t i) const { return ld_vec<KP>(z + i * KP); }
  __device__ __forceinline__ const V* xi_base() const { return reinterpret_cast<const V*>(z); }
  __device__ __forceinline__ void add(double (&a)[NA], double w, const V& zj, const V& zi) const {
#pragma unroll
    for (int c = 0; c < KQ; ++c) {
      const double df = zi.v[c] - zj.v[c];
      a[c] = fma(w, zj.v[c], a[c]);
      a[KQ + c] = fma(w * df, df, a[KQ + c]);
      a[2 * KQ + c] = fma(w, fabs(zj.v[c]), a[2 * KQ + c]);
    }
  }
  template <class P>
  __device__ __forceinline__ void finish_row(int64_t i, int64_t len, const V& zv, const double (&a)[NA],
                                             P& part) const {
    const double d = (WT == FJ_W_UNIT) ? (double)len : deg[i];
#pragma unroll
    for (int c = 0; c < KQ; ++c) {
      const double zi = zv.v[c];
      const double si = s[i * KQ + c];
      const double t = fma(1.0 + d, zi, -a[c]);
      const double lz = fma(d, zi, -a[c]);
      const double r = si - t;
      const double ab = fabs(si) + fma(1.0 + d, fabs(zi), a[2 * KQ + c]);
      part[0 * KQ + c] += a[KQ + c];
      part[1 * KQ + c] = fma(r, r, part[1 * KQ + c]);
      part[2 * KQ + c] = fma(lz, lz, part[2 * KQ + c]);
      part[3 * KQ + c] = fma(ab, ab, part[3 * KQ + c]);
    }
  }
  __device__ __forceinline__ void finalize(const double (&tot)[NP]) const {
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int c = 0; c < KQ; ++c) out[j * KP + c] = tot[j * KQ + c];
  }
};

// ---------------------------------------------------------------- elementwise kernels
// One thread per row (KP values, one aligned vector load per array); fixed grid, per-column
// partials reduced block -> last block in block order (deterministic).
template <int NPART>
__device__ __forceinline__ bool vec_reduce(double (&v)[NPART], double* part, unsigned int* ticket, double* s_red);
template <int NPART>
__device__ __forceinline__ bool vec_reduce(double (&v)[NPART], double* part, unsigned int* ticket, double* s_red) {
  block_sum<NPART, VETB>(v, s_red);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int j = 0; j < NPART; ++j) part[(int64_t)blockIdx.x * NPART + j] = v[j];
  }
  if (!last_block_ticket(ticket, gridDim.x)) return false;
  double t[NPART];
#pragma unroll
  for (int j = 0; j < NPART; ++j) t[j] = 0.0;
  for (int b = threadIdx.x; b < (int)gridDim.x; b += VETB) {
#pragma unroll
    for (int j = 0; j < NPART; ++j) t[j] += __ldcg(part + (int64_t)b * NPART + j);
  }
  block_sum<NPART, VETB>(t, s_red);
#pragma unroll
  for (int j = 0; j < NPART; ++j) v[j] = t[j];
  return true;
}

// Row-local quantity sums (QuantOp order 0 (z-s)^2, 2 (z-m)^2, 3 z^2, 4 s z, 5 (s-m)(z-m), 9 s^2):
// out[j * KP + c], j = 0..5 in that order.
template <int KP>
__global__ void __launch_bounds__(VETB) k_quant_local(int64_t n, int k, const double* __restrict__ s,
                                                      const double* __restrict__ z, const double* __restrict__ mean,
                                                      double* part, unsigned int* ticket, double* out) {
  __shared__ double s_red[6 * KP * VETB / 32];
  double v[6 * KP];
#pragma unroll
  for (int j = 0; j < 6 * KP; ++j) v[j] = 0.0;
  double m[KP];
#pragma unroll
  for (int c = 0; c < KP; ++c) m[c] = c < k ? mean[c] : 0.0;
  for (int64_t i = blockIdx.x * (int64_t)VETB + threadIdx.x; i < n; i += (int64_t)gridDim.x * VETB) {
    const DVec<KP> zv = ld_vec<KP>(z + i * KP);
#pragma unroll
    for (int c = 0; c < KP; ++c) {
      if (c < k) {
        const double zi = zv.v[c], si = s[i * k + c];
        const double e1 = zi - si, e2 = zi - m[c], e3 = si - m[c];
        v[0 * KP + c] = fma(e1, e1, v[0 * KP + c]);
        v[1 * KP + c] = fma(e2, e2, v[1 * KP + c]);
        v[2 * KP + c] = fma(zi, zi, v[2 * KP + c]);
        v[3 * KP + c] = fma(si, zi, v[3 * KP + c]);
        v[4 * KP + c] = fma(e3, e2, v[4 * KP + c]);
        v[5 * KP + c] = fma(si, si, v[5 * KP + c]);
      }
    }
  }
  if (vec_reduce<6 * KP>(v, part, ticket, s_red) && threadIdx.x == 0) {
#pragma unroll
    for (int j = 0; j < 6 * KP; ++j) out[j] = v[j];
    *ticket = 0u;
  }
}

// fresh start (x = 0, r = s) or restart (r = s - q, q = (I+L) x precomputed); p = dinv o r.
template <int KP, int KQ>
__global__ void __launch_bounds__(VETB) k_v_init(int64_t n, int k, const double* __restrict__ s,
                                                 const double* __restrict__ dinv, const double* __restrict__ q,
                                                 int restart, double* __restrict__ x, double* __restrict__ r,
                                                 double* __restrict__ p, VecScalars* sc, double rtol, int max_iter,
                                                 double* part, unsigned int* ticket) {
  __shared__ double s_red[3 * KP * VETB / 32];
  double v[3 * KP];
#pragma unroll
  for (int j = 0; j < 3 * KP; ++j) v[j] = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)VETB + threadIdx.x; i < n; i += (int64_t)gridDim.x * VETB) {
    DVec<KP> sv, rv, pv;
#pragma unroll
    for (int c = 0; c < KP; ++c) sv.v[c] = c < k ? s[i * k + c] : 0.0;
    if (restart) {
      const DVec<KP> qv = ld_q<KP, KQ>(q, i);
#pragma unroll
      for (int c = 0; c < KP; ++c) rv.v[c] = c < k ? sv.v[c] - qv.v[c] : 0.0;
    } else {
      rv = sv;
      st_q<KP, KQ>(x, i, vzero_kp<KP>());
    }
    const double di = dinv[i];
#pragma unroll
    for (int c = 0; c < KP; ++c) {
      pv.v[c] = di * rv.v[c];
      v[c] = fma(rv.v[c], pv.v[c], v[c]);
      v[KP + c] = fma(rv.v[c], rv.v[c], v[KP + c]);
      v[2 * KP + c] = fma(sv.v[c], sv.v[c], v[2 * KP + c]);
    }
    st_q<KP, KQ>(r, i, rv);
    st_vec<KP>(p + i * KP, pv);
  }
  if (vec_reduce<3 * KP>(v, part, ticket, s_red) && threadIdx.x == 0) {
    int any = 0;
    for (int c = 0; c < k; ++c) {
      sc->rho[c] = v[c];
      sc->rr[c] = v[KP + c];
      sc->ss[c] = v[2 * KP + c];
      sc->tol2[c] = rtol * rtol * v[2 * KP + c];
      const int conv = v[KP + c] <= sc->tol2[c];
      sc->conv[c] = conv;
      sc->active[c] = conv ? 0 : 1;
      sc->breakdown[c] = 0;
      sc->alpha[c] = sc->beta[c] = 0.0;
      any |= sc->active[c];
    }
    sc->iter = 0;
    sc->xpend = 0;
    sc->max_iter = max_iter;
    sc->k = k;
    sc->done = (!any || max_iter <= 0) ? 1 : 0;
    *ticket = 0u;
  }
}

// XD: the x update x += alpha p moves to k_v_dir (which reads p anyway), so this pass streams
// only q and r (one vector stream fewer per iteration); the last block hands the alphas it applied
// to k_v_dir through sc->alx / sc->xpend.
template <int KP, int KQ, bool XD>
__global__ void __launch_bounds__(VETB) k_v_update(int64_t n, int k, const double* __restrict__ dinv,
                                                   const double* __restrict__ p, const double* __restrict__ q,
                                                   double* __restrict__ x, double* __restrict__ r, VecScalars* sc,
                                                   double* part, unsigned int* ticket, cudaGraphConditionalHandle h,
                                                   int use_h) {
  __shared__ double s_red[2 * KP * VETB / 32];
  pdl_prologue();
  if (*(volatile int32_t*)&sc->done) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      if (XD) sc->xpend = 0;    // the loop ended earlier: nothing owed to x any more
      if (use_h) cudaGraphSetConditional(h, 0);
    }
    return;
  }
  double al[KP];
#pragma unroll
  for (int c = 0; c < KP; ++c) al[c] = (c < k && sc->active[c]) ? sc->alpha[c] : 0.0;
  double v[2 * KP];
#pragma unroll
  for (int j = 0; j < 2 * KP; ++j) v[j] = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)VETB + threadIdx.x; i < n; i += (int64_t)gridDim.x * VETB) {
    const DVec<KP> qv = ld_q<KP, KQ>(q, i);
    DVec<KP> rv = ld_q<KP, KQ>(r, i);
    const double di = dinv[i];
    if (!XD) {
      const DVec<KP> pv = ld_vec<KP>(p + i * KP);
      DVec<KP> xv = ld_q<KP, KQ>(x, i);
#pragma unroll
      for (int c = 0; c < KP; ++c) xv.v[c] = fma(al[c], pv.v[c], xv.v[c]);
      st_q<KP, KQ>(x, i, xv);
    }
#pragma unroll
    for (int c = 0; c < KP; ++c) {
      rv.v[c] = fma(-al[c], qv.v[c], rv.v[c]);
      v[c] = fma(rv.v[c], di * rv.v[c], v[c]);
      v[KP + c] = fma(rv.v[c], rv.v[c], v[KP + c]);
    }
    st_q<KP, KQ>(r, i, rv);
  }
  if (vec_reduce<2 * KP>(v, part, ticket, s_red) && threadIdx.x == 0) {
    if (XD) {
#pragma unroll
      for (int c = 0; c < KP; ++c) sc->alx[c] = al[c];
      sc->xpend = 1;
    }
    int any = 0;
    for (int c = 0; c < k; ++c) {
      if (sc->active[c]) {
        sc->beta[c] = v[c] / sc->rho[c];
        sc->rho[c] = v[c];
        sc->rr[c] = v[KP + c];
        const bool conv = v[KP + c] <= sc->tol2[c];
        if (conv || !isfinite(v[KP + c])) { sc->active[c] = 0; sc->conv[c] = conv ? 1 : 0; }
      }
      any |= sc->active[c];
    }
    const int it = sc->iter + 1;
    sc->iter = it;
    if (!any || it >= sc->max_iter) {
      sc->done = 1;
      if (use_h) cudaGraphSetConditional(h, 0);
    }
    *ticket = 0u;
  }
}
// p = dinv o r + beta p (and, XD, first x += alx p with the old p; after the final iteration only that)
template <int KP, int KQ, bool XD>
__global__ void __launch_bounds__(VETB) k_v_dir(int64_t n, int k, const double* __restrict__ dinv,
                                                const double* __restrict__ r, double* __restrict__ p,
                                                double* __restrict__ x, const VecScalars* sc) {
  pdl_prologue();
  const bool done = *(volatile const int32_t*)&sc->done;
  if (XD ? !*(volatile const int32_t*)&sc->xpend : done) return;
  double be[KP], al[KP];
#pragma unroll
  for (int c = 0; c < KP; ++c) {
    be[c] = (c < k && sc->active[c]) ? sc->beta[c] : 0.0;
    al[c] = XD ? sc->alx[c] : 0.0;
  }
  for (int64_t i = blockIdx.x * (int64_t)VETB + threadIdx.x; i < n; i += (int64_t)gridDim.x * VETB) {
    DVec<KP> pv = ld_vec<KP>(p + i * KP);
    if (XD) {
      DVec<KP> xv = ld_q<KP, KQ>(x, i);
#pragma unroll
      for (int c = 0; c < KP; ++c) xv.v[c] = fma(al[c], pv.v[c], xv.v[c]);
      st_q<KP, KQ>(x, i, xv);
      if (done) continue;
    }
    const DVec<KP> rv = ld_q<KP, KQ>(r, i);
    const double di = dinv[i];
#pragma unroll
    for (int c = 0; c < KP; ++c) pv.v[c] = fma(be[c], pv.v[c], di * rv.v[c]);
    st_vec<KP>(p + i * KP, pv);
  }
}

// [n][k] <-> padded [n][KP]
template <int KP>
__global__ void k_v_pack(int64_t n, int k, const double* __restrict__ src, double* __restrict__ dst) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    DVec<KP> v;
#pragma unroll
    for (int c = 0; c < KP; ++c) v.v[c] = c < k ? src[i * k + c] : 0.0;
    st_vec<KP>(dst + i * KP, v);
  }
}
template <int KP, int KQ>
__global__ void k_v_pack_from(int64_t n, const double* __restrict__ src, double* __restrict__ dst) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    st_vec<KP>(dst + i * KP, ld_q<KP, KQ>(src, i));
}
template <int KP>
__global__ void k_v_unpack(int64_t n, int k, const double* __restrict__ src, double* __restrict__ dst) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const DVec<KP> v = ld_vec<KP>(src + i * KP);
#pragma unroll
    for (int c = 0; c < KP; ++c)
      if (c < k) dst[i * k + c] = v.v[c];
  }
}

// ---------------------------------------------------------------- workspace
constexpr int VNP_MAX = 10 * KVMAX, VNA_MAX = 3 * KVMAX;

struct VecWs {
  int k = 0, kp = 0, kq = 0;
  RowsPlan rows;         // k columns; p rows KP wide (gathered), x / r / q rows KQ wide
  int grid_elem = 0, grid_max = 0;
  double *r = nullptr, *p = nullptr, *q = nullptr, *x = nullptr;
  bool x_is_solution = false;        // x holds z ([n][KQ]) of the last solve_vec (for quant_vec)
  VecScalars* sc = nullptr;
  double* elem_part = nullptr;       // [grid_elem][6 * KVMAX]
  unsigned int* elem_ticket = nullptr;
  TileScratch ts{};
  double* qout = nullptr;            // [VNP_MAX]
  double* dred = nullptr;            // [8 * KVMAX] distributed allreduce payloads
  cudaGraphExec_t exec = nullptr;
  cudaGraph_t graph = nullptr;
  cudaStream_t cap_stream = nullptr;
  cudaEvent_t ev2 = nullptr, ev3 = nullptr, ev4 = nullptr;
};

static VecWs* vec_cache(fj_graph* g) { return reinterpret_cast<VecWs*>(g->vec_ws); }

// kernel launches of one PCG iteration (product + k_v_update + k_v_dir), for fj_kernel_launches
static int vec_iter_launches(const VecWs* w) { return rows_launches(w->rows) + 2; }

void free_vec_ws(fj_graph* g) {
  VecWs* w = vec_cache(g);
  if (!w) return;
  if (w->exec) cudaGraphExecDestroy(w->exec);
  if (w->graph) cudaGraphDestroy(w->graph);
  if (w->cap_stream) cudaStreamDestroy(w->cap_stream);
  if (w->ev2) cudaEventDestroy(w->ev2);
  if (w->ev3) cudaEventDestroy(w->ev3);
  if (w->ev4) cudaEventDestroy(w->ev4);
  dfree(w->r); dfree(w->p); dfree(w->q); dfree(w->x); dfree(w->sc);
  dfree(w->elem_part); dfree(w->elem_ticket);
  dfree(w->ts.block_part); dfree(w->ts.long_part); dfree(w->ts.chunk_acc);
  dfree(w->ts.long_ticket); dfree(w->ts.grid_ticket); dfree(w->qout); dfree(w->dred);
  rows_plan_free(w->rows);
  delete w;
  g->vec_ws = nullptr;
}

template <class T>
static fj_status valloc(T** p, int64_t count, cudaStream_t st, bool zero = false) {
  if (count < 1) count = 1;
  FJ_CK(dmalloc(p, sizeof(T) * (size_t)count, st));
  if (zero) FJ_CK(cudaMemsetAsync(*p, 0, sizeof(T) * (size_t)count, st));
  return FJ_OK;
}

static int kp_of(int k) { return k <= 2 ? 2 : k == 3 ? vec_pad3() : 4; }
static int kq_of(int k) { return k <= 2 ? 2 : k == 3 ? 3 : 4; }   // x, r, q: unpadded


static fj_status get_vec_ws(fj_graph* g, int k, cudaStream_t st, VecWs** out) {
  VecWs* w = vec_cache(g);
  const int kp = kp_of(k), kq = kq_of(k);
  if (w && w->kp == kp && w->kq == kq) { w->k = k; *out = w; return FJ_OK; }
  if (w) {
    FJ_CK(cudaStreamSynchronize(st));   // old buffers may still be in use on st
    free_vec_ws(g);
  }
  w = new VecWs();
  g->vec_ws = w;
  w->k = k;
  w->kp = kp;
  w->kq = kq;
  // p has the ghost rows of a distributed slice appended (the halo exchange fills them)
  const int64_t nkp = (g->n + dist_n_ghost(g)) * (int64_t)kp, nkq = g->n * (int64_t)kq;
  FJ_TRY(valloc(&w->r, nkq, st)); FJ_TRY(valloc(&w->p, nkp, st));
  FJ_TRY(valloc(&w->q, nkq, st)); FJ_TRY(valloc(&w->x, nkq, st));
  FJ_TRY(valloc(&w->sc, 1, st, true));
  int64_t ge = (int64_t)g->num_sms * (2048 / VETB);
  const int64_t need = (g->n + VETB - 1) / VETB;
  if (ge > need) ge = need > 0 ? need : 1;
  w->grid_elem = (int)ge;
  FJ_TRY(valloc(&w->elem_part, ge * 6 * KVMAX, st));
  FJ_TRY(valloc(&w->elem_ticket, 1, st, true));
  w->grid_max = g->num_sms * (2048 / WTPB);
  FJ_TRY(valloc(&w->ts.block_part, (int64_t)w->grid_max * VNP_MAX, st));
  if (!g->sv.built) FJ_TRY(build_schedule(g, kSchedVec, g->sv, st));
  FJ_TRY(valloc(&w->ts.long_part, g->sv.n_long * VNP_MAX, st));
  FJ_TRY(valloc(&w->ts.chunk_acc, g->sv.n_long_chunks * VNA_MAX, st));
  FJ_TRY(valloc(&w->ts.long_ticket, g->sv.n_long, st, true));
  FJ_TRY(valloc(&w->ts.grid_ticket, 1, st, true));
  FJ_TRY(valloc(&w->qout, VNP_MAX + 6 * KVMAX + KVMAX, st));
  FJ_TRY(valloc(&w->dred, 8 * KVMAX, st));   // [4][KP] engine sums, [6][KP] local, means
  FJ_CK(cudaEventCreate(&w->ev2));
  FJ_CK(cudaEventCreate(&w->ev3));
  FJ_CK(cudaEventCreate(&w->ev4));
  FJ_TRY(rows_plan_build(g, kp, w->rows, st));
  *out = w;
  return FJ_OK;
}

// The warp-item engine on the vector schedule (sv: VEC_ITEMS merge items per lane), vector values.
template <int WT, class Op>
static fj_status launch_vec_items(const fj_graph* g, const VecWs* w, const Op& op, cudaStream_t st) {
  if (w->rows.mode != 0) return rows_op<WT>(w->rows, g->n, g->col, g->w, op, st);   // rows.cuh
  static int occ = 0;   // per instantiation
  if (occ == 0) {
    FJ_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, warp_kernel<WT, Op>, WTPB, 0));
    if (occ < 1) occ = 1;
  }
  int64_t grid = (int64_t)g->num_sms * occ;
  const int64_t need = (g->sv.n_items + WPB - 1) / WPB;
  if (grid > need) grid = need > 0 ? need : 1;
  if (grid > w->grid_max) grid = w->grid_max;
  warp_kernel<WT, Op><<<(unsigned)grid, WTPB, 0, st>>>(make_sched(g, g->sv), op, w->ts);
  FJ_CK_LAUNCH();
  return FJ_OK;
}

template <int KP, class F>
static fj_status by_wtype(const fj_graph* g, F&& f) {
  switch (g->wtype) {
    case FJ_W_UNIT: return f(std::integral_constant<int, FJ_W_UNIT>());
    case FJ_W_U8: return f(std::integral_constant<int, FJ_W_U8>());
    case FJ_W_F32: return f(std::integral_constant<int, FJ_W_F32>());
    default: return f(std::integral_constant<int, FJ_W_F64>());
  }
}

// y [n][KQ] = (I+L) x (or L x) for x the padded [n][KP] block
template <int KP, int KQ>
static fj_status vec_apply_padded(const fj_graph* g, const VecWs* w, const double* x, double* y, int opL,
                                  VecScalars* sc, cudaStream_t st, bool pdl = false) {
  return by_wtype<KP>(g, [&](auto wt) {
    constexpr int WT = decltype(wt)::value;
    if constexpr (KP == 2 || KP == 4) {
      if (w->rows.mode != 0) return rows_product<WT, KP, KQ>(g, w->rows, x, y, opL, w->k, sc, nullptr, st);
    }
    ApplyOpV<WT, KP, KQ> op{x, y, g->deg, opL, sc, w->k};
    int nl = 0;
    FJ_CK(launch_product<WT>(g, w->ts, w->grid_max, op, st, &nl, pdl));
    if (!g_capturing) count_launch(nl);
    return FJ_OK;
  });
}

template <int KP, int KQ>
static fj_status vec_iteration(const fj_graph* g, VecWs* w, cudaStream_t st, cudaGraphConditionalHandle h, int use_h) {
  // the three kernels of an iteration are chained by programmatic dependent launch (PDL)
  FJ_TRY((vec_apply_padded<KP, KQ>(g, w, w->p, w->q, 0, w->sc, st, true)));
  FJ_CK(pdl_launch(k_v_update<KP, KQ, true>, dim3(w->grid_elem), dim3(VETB), st, g->n, w->k, g->dinv,
                   (const double*)w->p, (const double*)w->q, w->x, w->r, w->sc, w->elem_part, w->elem_ticket, h, use_h));
  FJ_CK_LAUNCH();
  FJ_CK(pdl_launch(k_v_dir<KP, KQ, true>, dim3(w->grid_elem), dim3(VETB), st, g->n, w->k, g->dinv,
                   (const double*)w->r, w->p, w->x, (const VecScalars*)w->sc));
  FJ_CK_LAUNCH();
  return FJ_OK;
}

template <int KP, int KQ>
static fj_status build_vec_graph(fj_graph* g, VecWs* w) {
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
  fj_status s = vec_iteration<KP, KQ>(g, w, w->cap_stream, h, 1);
  g_capturing = false;
  cudaGraph_t captured = nullptr;
  cudaError_t e = cudaStreamEndCapture(w->cap_stream, &captured);
  FJ_TRY(s);
  FJ_CK(e);
  FJ_CK(cudaGraphInstantiate(&w->exec, w->graph, 0));
  return FJ_OK;
}

template <int KP, int KQ>
static fj_status solve_vec_t(fj_graph* g, VecWs* w, int k, const double* s, double* z, const fj_solve_opts& o,
                             int warm, fj_solve_report* rep, cudaStream_t st, bool defer) {
  const int64_t n = g->n;
  const unsigned cb = (unsigned)std::min<int64_t>((n + 255) / 256, 8192);
  w->x_is_solution = false;
  if (o.use_cuda_graph) FJ_TRY((build_vec_graph<KP, KQ>(g, w)));
  phase_tick("vec: loop graph capture", st);
  VecScalars h{};
  int restarts = 0, total_iter = 0;
  bool first = true;
  for (;;) {
    const bool restart = !first || warm;
    if (restart) {
      // restart: q = (I+L) x with x the current iterate (warm: from z), gathered from a padded copy
      if (first) { k_v_pack<KQ><<<cb, 256, 0, st>>>(n, k, z, w->x); FJ_CK_LAUNCH(); }
      k_v_pack_from<KP, KQ><<<cb, 256, 0, st>>>(n, w->x, w->p);
      FJ_CK_LAUNCH();
      FJ_TRY((vec_apply_padded<KP, KQ>(g, w, w->p, w->q, 0, nullptr, st)));
    }
    const int budget = std::max(0, o.max_iter - total_iter);
    FJ_CK(cudaEventRecord(w->ev2, st));
    k_v_init<KP, KQ><<<w->grid_elem, VETB, 0, st>>>(n, k, s, g->dinv, w->q, restart ? 1 : 0, w->x, w->r, w->p, w->sc,
                                                o.rtol, budget, w->elem_part, w->elem_ticket);
    FJ_CK_LAUNCH();
    first = false;
    if (o.use_cuda_graph) {
      FJ_CK(cudaGraphLaunch(w->exec, st));
    } else {
      for (;;) {
        for (int u = 0; u < 8; ++u) FJ_TRY((vec_iteration<KP, KQ>(g, w, st, 0, 0)));
        int32_t done = 0;
        FJ_CK(cudaMemcpyAsync(&done, &w->sc->done, sizeof done, cudaMemcpyDeviceToHost, st));
        FJ_CK(cudaStreamSynchronize(st));
        if (done) break;
      }
    }
    FJ_CK(cudaEventRecord(w->ev3, st));
    phase_tick("vec: init + PCG loop", st);
    if (defer) {   // the caller checks the true residual (fused quantities pass)
      FJ_CK(cudaMemcpyAsync(&h, w->sc, sizeof h, cudaMemcpyDeviceToHost, st));
      FJ_CK(cudaStreamSynchronize(st));
      total_iter += h.iter;
      if (o.use_cuda_graph) count_launch((int64_t)vec_iter_launches(w) * std::max(h.iter, 1));
      float lms = 0.f;
      cudaEventElapsedTime(&lms, w->ev2, w->ev3);
      if (rep) { rep->ms_loop += lms; rep->iterations_total += (int64_t)h.iter * k; }
      for (int c = 0; c < k; ++c) h.res2[c] = h.rr[c];   // recursive residual stands in
      break;
    }
    FJ_TRY(by_wtype<KP>(g, [&](auto wt) {   // true residual per column (x gathered KQ wide)
      constexpr int WT = decltype(wt)::value;
      ResidOpV<WT, KQ> op{w->x, s, g->deg, k, w->sc};
      return launch_vec_items<WT>(g, w, op, st);
    }));
    FJ_CK(cudaMemcpyAsync(&h, w->sc, sizeof h, cudaMemcpyDeviceToHost, st));
    FJ_CK(cudaStreamSynchronize(st));
    phase_tick("vec: true residual", st);
    total_iter += h.iter;
    if (o.use_cuda_graph) count_launch((int64_t)vec_iter_launches(w) * std::max(h.iter, 1));
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
  k_v_unpack<KQ><<<cb, 256, 0, st>>>(n, k, w->x, z);
  FJ_CK_LAUNCH();
  w->x_is_solution = true;
  bool converged = true;
  double worst_true = 0.0, worst_rec = 0.0;
  for (int c = 0; c < k; ++c) {
    if (h.res2[c] > h.tol2[c] && !(defer && h.conv[c])) converged = false;
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
    if (!defer)
      rep->rel_res_true = std::isnan(rep->rel_res_true) ? worst_true : std::max(rep->rel_res_true, worst_true);
    if (!converged) rep->converged = 0;
  }
  return converged ? FJ_OK : fail(FJ_E_NO_CONVERGENCE, "batched PCG did not reach rtol on the true residual");
}

// ---------------------------------------------------------------- entry points (workspace.cuh)
bool vec_supported(int k) { return k >= 2 && k <= KVMAX; }

fj_status solve_vec(fj_graph* g, int k, const double* s, double* z, const fj_solve_opts& o, int warm,
                    fj_solve_report* rep, cudaStream_t st, bool defer) {
  VecWs* w = nullptr;
  phase_tick("vec: enter", st);
  FJ_TRY(get_vec_ws(g, k, st, &w));
  phase_tick("vec: workspace + schedule", st);
  switch (w->kp) {
    case 2: return solve_vec_t<2, 2>(g, w, k, s, z, o, warm, rep, st, defer);
    case 3: return solve_vec_t<3, 3>(g, w, k, s, z, o, warm, rep, st, defer);
    default: return w->kq == 3 ? solve_vec_t<4, 3>(g, w, k, s, z, o, warm, rep, st, defer)
                               : solve_vec_t<4, 4>(g, w, k, s, z, o, warm, rep, st, defer);
  }
}

fj_status apply_vec(fj_graph* g, int k, const double* x, double* y, int opL, cudaStream_t st) {
  VecWs* w = nullptr;
  FJ_TRY(get_vec_ws(g, k, st, &w));
  w->x_is_solution = false;
  const unsigned cb = (unsigned)std::min<int64_t>((g->n + 255) / 256, 8192);
  auto run = [&](auto kpc, auto kqc) -> fj_status {
    constexpr int KP = decltype(kpc)::value, KQ = decltype(kqc)::value;
    k_v_pack<KP><<<cb, 256, 0, st>>>(g->n, k, x, w->p);
    FJ_CK_LAUNCH();
    FJ_TRY((vec_apply_padded<KP, KQ>(g, w, w->p, w->q, opL, nullptr, st)));
    k_v_unpack<KQ><<<cb, 256, 0, st>>>(g->n, k, w->q, y);
    FJ_CK_LAUNCH();
    return FJ_OK;
  };
  using I2 = std::integral_constant<int, 2>;
  using I3 = std::integral_constant<int, 3>;
  using I4 = std::integral_constant<int, 4>;
  switch (w->kp) {
    case 2: return run(I2(), I2());
    case 3: return run(I3(), I3());
    default: return w->kq == 3 ? run(I4(), I3()) : run(I4(), I4());
  }
}

fj_status vec_product_mode(fj_graph* g, int k, cudaStream_t st, int* mode) {
  VecWs* w = nullptr;
  FJ_TRY(get_vec_ws(g, k, st, &w));
  *mode = w->kp == 3 ? 0 : w->rows.mode;
  return FJ_OK;
}

// Time `reps` launches of the PCG-mode product q = (I+L) p on the solver's own padded buffers
// (the kernel the solve loop runs), CUDA events on st.  Diagnostic for the bench roofline.
fj_status time_vec_spmv(fj_graph* g, int k, int reps, float* ms_out, cudaStream_t st) {
  VecWs* w = nullptr;
  FJ_TRY(get_vec_ws(g, k, st, &w));
  w->x_is_solution = false;
  auto run = [&]() -> fj_status {
    switch (w->kp) {
      case 2: return vec_apply_padded<2, 2>(g, w, w->p, w->q, 0, nullptr, st);
      case 3: return vec_apply_padded<3, 3>(g, w, w->p, w->q, 0, nullptr, st);
      default: return w->kq == 3 ? vec_apply_padded<4, 3>(g, w, w->p, w->q, 0, nullptr, st)
                                 : vec_apply_padded<4, 4>(g, w, w->p, w->q, 0, nullptr, st);
    }
  };
  FJ_TRY(run());
  FJ_CK(cudaEventRecord(w->ev2, st));
  for (int i = 0; i < reps; ++i) FJ_TRY(run());
  FJ_CK(cudaEventRecord(w->ev3, st));
  FJ_CK(cudaEventSynchronize(w->ev3));
  float ms = 0.f;
  FJ_CK(cudaEventElapsedTime(&ms, w->ev2, w->ev3));
  *ms_out = ms / (float)std::max(reps, 1);
  return FJ_OK;
}

// All k columns' 10 sums in one pass: host_out[c * 10 + j] (same order as QuantOp's partials).
// If the last solve_vec on this graph produced z, its padded copy is gathered directly.
fj_status quant_vec(fj_graph* g, int k, const double* s, const double* z, const double* mean_host,
                    double* host_out, bool z_from_solve, cudaStream_t st) {
  VecWs* w = nullptr;
  FJ_TRY(get_vec_ws(g, k, st, &w));
  const int kp = w->kp;
  const unsigned cb = (unsigned)std::min<int64_t>((g->n + 255) / 256, 8192);
  // z gathered from a padded [n][KP] copy in the (free) search-direction buffer p; the source is the
  // solver's own x when it holds this z, else the caller's [n][k] z
  const double* zsrc = (z_from_solve && w->x_is_solution && w->k == k) ? w->x : z;
  if (kp == 2) k_v_pack<2><<<cb, 256, 0, st>>>(g->n, k, zsrc, w->p);
  else if (kp == 3) k_v_pack<3><<<cb, 256, 0, st>>>(g->n, k, zsrc, w->p);
  else k_v_pack<4><<<cb, 256, 0, st>>>(g->n, k, zsrc, w->p);
  FJ_CK_LAUNCH();
  w->x_is_solution = false;   // p is overwritten by the next solve / apply anyway
  const double* zp = w->p;
  double* loc = w->qout + 4 * KVMAX;         // [6][KP]
  double* dmean = loc + 6 * KVMAX;            // [KP]
  FJ_CK(cudaMemcpyAsync(dmean, mean_host, sizeof(double) * k, cudaMemcpyHostToDevice, st));
  auto launch = [&](auto kpc) -> fj_status {
    constexpr int KP = decltype(kpc)::value;
    phase_tick("quant: enter", st);
    k_quant_local<KP><<<w->grid_elem, VETB, 0, st>>>(g->n, k, s, zp, dmean, w->elem_part, w->elem_ticket, loc);
    FJ_CK_LAUNCH();
    phase_tick("quant: local sums", st);
    return by_wtype<KP>(g, [&](auto wt) {
      constexpr int WT = decltype(wt)::value;
      auto go = [&](auto kqc) -> fj_status {
        constexpr int KQ = decltype(kqc)::value;
        QuantOpV<WT, KP, KQ> op;
        op.z = zp; op.s = s; op.deg = g->deg; op.out = w->qout;
        return launch_vec_items<WT>(g, w, op, st);
      };
      if (KP == 4 && k == 3) return go(std::integral_constant<int, 3>());
      return go(std::integral_constant<int, KP>());
    });
  };
  if (kp == 2) FJ_TRY(launch(std::integral_constant<int, 2>()));
  else if (kp == 3) FJ_TRY(launch(std::integral_constant<int, 3>()));
  else FJ_TRY(launch(std::integral_constant<int, 4>()));
  phase_tick("quant: neighbour sums", st);
  std::vector<double> h(4 * kp + 6 * kp);
  FJ_CK(cudaMemcpyAsync(h.data(), w->qout, sizeof(double) * 4 * kp, cudaMemcpyDeviceToHost, st));
  FJ_CK(cudaMemcpyAsync(h.data() + 4 * kp, loc, sizeof(double) * 6 * kp, cudaMemcpyDeviceToHost, st));
  FJ_CK(cudaStreamSynchronize(st));
  // QuantOp order: 0 (z-s)^2, 1 Dd, 2 (z-m)^2, 3 z^2, 4 sz, 5 (s-m)(z-m), 6 res^2, 7 (Lz)^2, 8 allow^2, 9 s^2
  static const int src[10] = {4 + 0, 0, 4 + 1, 4 + 2, 4 + 3, 4 + 4, 1, 2, 3, 4 + 5};
  for (int c = 0; c < k; ++c)
    for (int j = 0; j < 10; ++j) host_out[c * 10 + j] = h[src[j] * kp + c];
  return FJ_OK;
}

}  // namespace fj

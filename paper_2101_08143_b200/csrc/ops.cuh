// ops.cuh — row operators plugged into the tile engine (tiles.cuh) and the per-solve workspace.
#pragma once
#include "tiles.cuh"

namespace fj {

// Device scalars of one PCG solve (one column).  Written only by "last block" finalisers.
struct PcgScalars {
  double rho;        // r^T y, y = dinv o r
  double alpha, beta;
  double pq;         // p^T (I+L) p
  double rr;         // ||r||^2 (recursive)
  double ss;         // ||s||^2
  double tol2;       // rtol^2 ||s||^2
  double res2;       // ||s - (I+L) x||^2 (true residual, when computed)
  int32_t iter, max_iter, done, converged, breakdown, pad;
};

// y = (I+L) x  (mode IPL) or y = L x (mode L) for column c of row-major [n][ld] arrays.
// (I+L)x_i = (1 + d_i) x_i - sum_j w_ij x_j   (P:L88 L = D - A).
// If sc != nullptr this is the PCG search-direction product: skip when the solve is done and
// finalise alpha = rho / p^T q on device.
template <int WT>
struct ApplyOp {
  static constexpr int NA = 1, NP = 1;
  static constexpr bool NEEDS_XI = false;
  using V = double;
  static constexpr int ITEMS = fj::ITEMS;
  static constexpr int TILE_ROWS = fj::TILE_ROWS;
  static constexpr int MIN_BLOCKS = engine_min_blocks<double>();
  static constexpr bool TMA = FJ_K1_TMA != 0;   // measured: the plain loop is faster for 8-byte values
  static __device__ __forceinline__ V vzero() { return 0.0; }
  const double* __restrict__ x;
  double* __restrict__ y;
  const double* __restrict__ deg;   // weighted degree (unused for unit weights)
  int64_t ld, c;
  int opL;                          // 1: L x, 0: (I + L) x
  PcgScalars* sc;                   // PCG mode when non-null
  double* dot_out;                  // optional: x^T y
  int alpha_on_device = 1;          // 0 (distributed): leave alpha to the caller after the allreduce
  __device__ __forceinline__ bool skip() const { return sc && *(volatile int32_t*)&sc->done; }
  __device__ __forceinline__ bool wants_xi() const { return true; }
  __device__ __forceinline__ double gather(int32_t j) const {
#ifdef FJ_GATHER_NC
    return __ldg(x + (int64_t)j * ld + c);
#else
    return ld_plain(x + (int64_t)j * ld + c);
#endif
  }
  __device__ __forceinline__ double row_value(int64_t i) const { return __ldg(x + i * ld + c); }
  __device__ __forceinline__ const double* xi_base() const { return ld == 1 ? x : nullptr; }
  __device__ __forceinline__ void add(double (&a)[NA], double w, double xj, double) const {
    if (WT == FJ_W_UNIT) a[0] += xj; else a[0] = fma(w, xj, a[0]);
  }
  template <class P>
  __device__ __forceinline__ void finish_row(int64_t i, int64_t len, double xi, const double (&a)[NA],
                                             P& part) const {
    const double d = (WT == FJ_W_UNIT) ? (double)len : deg[i];
    const double yi = opL ? fma(d, xi, -a[0]) : fma(1.0 + d, xi, -a[0]);
    y[i * ld + c] = yi;
    part[0] = fma(xi, yi, part[0]);
  }
  __device__ __forceinline__ void finalize(const double (&tot)[NP]) const {
    if (dot_out) *dot_out = tot[0];
    if (sc && alpha_on_device) {
      sc->pq = tot[0];
      if (!(tot[0] > 0.0) || !isfinite(tot[0])) {   // (I+L) is SPD: p^T q > 0 unless p = 0
        sc->alpha = 0.0;
        sc->breakdown = 1;
        sc->done = 1;
      } else {
        sc->alpha = sc->rho / tot[0];
      }
    }
  }
};

// ||s - (I+L) z||^2 for column c (true residual).
template <int WT>
struct ResidOp {
  static constexpr int NA = 1, NP = 1;
  static constexpr bool NEEDS_XI = false;
  using V = double;
  static constexpr int ITEMS = fj::ITEMS;
  static constexpr int TILE_ROWS = fj::TILE_ROWS;
  static constexpr int MIN_BLOCKS = engine_min_blocks<double>();
  static constexpr bool TMA = FJ_K1_TMA != 0;   // measured: the plain loop is faster for 8-byte values
  static __device__ __forceinline__ V vzero() { return 0.0; }
  const double* __restrict__ z;     // contiguous [n]
  const double* __restrict__ s;     // column c of row-major [n][ld]
  const double* __restrict__ deg;
  int64_t ld, c;
  double* res2_out;
  __device__ __forceinline__ bool skip() const { return false; }
  __device__ __forceinline__ bool wants_xi() const { return true; }
  __device__ __forceinline__ double gather(int32_t j) const { return __ldg(z + j); }
  __device__ __forceinline__ double row_value(int64_t i) const { return __ldg(z + i); }
  __device__ __forceinline__ const double* xi_base() const { return z; }
  __device__ __forceinline__ void add(double (&a)[NA], double w, double xj, double) const {
    if (WT == FJ_W_UNIT) a[0] += xj; else a[0] = fma(w, xj, a[0]);
  }
  template <class P>
  __device__ __forceinline__ void finish_row(int64_t i, int64_t len, double zi, const double (&a)[NA],
                                             P& part) const {
    const double d = (WT == FJ_W_UNIT) ? (double)len : deg[i];
    const double r = s[i * ld + c] - fma(1.0 + d, zi, -a[0]);
    part[0] = fma(r, r, part[0]);
  }
  __device__ __forceinline__ void finalize(const double (&tot)[NP]) const { *res2_out = tot[0]; }
};

// Fused quantities pass (rows a5-a7) for column c.  Per row i, with A = sum_j w_ij z_j,
// Dd = sum_j w_ij (z_i - z_j)^2, Aa = sum_j w_ij |z_j|, t = (I+L)z_i, m = mean(s):
//  0 (z-s)^2 [CI, Def 3.1]   1 Dd [2D, Def 3.2 counts each edge from both ends]
//  2 (z-m)^2 [P, Def 3.3]    3 z^2 [C, Def 3.4]   4 s z [= Idc, P:L228]
//  5 (s-m)(z-m) [= PDI]      6 (s - t)^2 [true residual]   7 (d z - A)^2 [||Lz||^2, Alg.1 l.5]
//  8 (|s| + (1+d)|z| + Aa)^2 [rounding allowance]          9 s^2
template <int WT>
struct QuantOp {
  static constexpr int NA = 3, NP = 10;
  static constexpr bool NEEDS_XI = true;
  using V = double;
  static constexpr int ITEMS = fj::ITEMS;
  static constexpr int TILE_ROWS = fj::TILE_ROWS;
  static constexpr int MIN_BLOCKS = engine_min_blocks<double>();
  static constexpr bool TMA = FJ_K1_TMA != 0;   // measured: the plain loop is faster for 8-byte values
  static __device__ __forceinline__ V vzero() { return 0.0; }
  const double* __restrict__ z;
  const double* __restrict__ s;
  const double* __restrict__ deg;
  int64_t ld, c;
  double m;
  double* out;   // [NP]
  int64_t zld = -1, zc = 0;   // z layout if it differs from s (distributed: contiguous extended z)
  __device__ __forceinline__ bool skip() const { return false; }
  __device__ __forceinline__ bool wants_xi() const { return true; }
  __device__ __forceinline__ int64_t zi(int64_t i) const { return zld < 0 ? i * ld + c : i * zld + zc; }
  __device__ __forceinline__ double gather(int32_t j) const { return __ldg(z + zi(j)); }
  __device__ __forceinline__ double row_value(int64_t i) const { return __ldg(z + zi(i)); }
  __device__ __forceinline__ const double* xi_base() const {
    return (zld < 0 ? (ld == 1 && c == 0) : (zld == 1 && zc == 0)) ? z : nullptr;
  }
  __device__ __forceinline__ void add(double (&a)[NA], double w, double zj, double zi) const {
    const double df = zi - zj;
    a[0] = fma(w, zj, a[0]);
    a[1] = fma(w * df, df, a[1]);
    a[2] = fma(w, fabs(zj), a[2]);
  }
  template <class P>
  __device__ __forceinline__ void finish_row(int64_t i, int64_t len, double zi, const double (&a)[NA],
                                             P& part) const {
    const double d = (WT == FJ_W_UNIT) ? (double)len : deg[i];
    const double si = s[i * ld + c];
    const double t = fma(1.0 + d, zi, -a[0]);
    const double lz = fma(d, zi, -a[0]);
    const double r = si - t;
    const double e1 = zi - si, e2 = zi - m, e3 = si - m;
    const double ab = fabs(si) + fma(1.0 + d, fabs(zi), a[2]);
    part[0] = fma(e1, e1, part[0]);
    part[1] += a[1];
    part[2] = fma(e2, e2, part[2]);
    part[3] = fma(zi, zi, part[3]);
    part[4] = fma(si, zi, part[4]);
    part[5] = fma(e3, e2, part[5]);
    part[6] = fma(r, r, part[6]);
    part[7] = fma(lz, lz, part[7]);
    part[8] = fma(ab, ab, part[8]);
    part[9] = fma(si, si, part[9]);
  }
  __device__ __forceinline__ void finalize(const double (&tot)[NP]) const {
#pragma unroll
    for (int j = 0; j < NP; ++j) out[j] = tot[j];
  }
};

struct RowsPlan;   // rows.cuh: the lean row product of the k = 1 PCG (built with this workspace)

// Per-graph workspace shared by the solver and the quantities pass (stream-ordered use only).
struct SolveWs {
  int64_t n = 0;
  RowsPlan* rows = nullptr;
  int grid_max = 0, grid_elem = 0;
  double *r = nullptr, *p = nullptr, *q = nullptr, *x = nullptr, *col_s = nullptr;
  PcgScalars* sc = nullptr;
  double* elem_part = nullptr;       // [grid_elem][16]
  unsigned int* elem_ticket = nullptr;
  TileScratch ts{};
  double* qout = nullptr;            // [16] quantities totals
  double* stat = nullptr;            // [4 * MAXK] opinion statistics
  // captured loop
  cudaGraphExec_t exec = nullptr;
  cudaGraph_t graph = nullptr;
  cudaStream_t cap_stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr, ev2 = nullptr, ev3 = nullptr;
};

fj_status get_ws(fj_graph* g, cudaStream_t st, SolveWs** out);

// Launch the warp-item engine for one operator.  The grid is fixed per (graph, operator):
// #SMs x occupancy of this instantiation, capped by the item count -> deterministic partials.
template <int WT, class Op>
inline cudaError_t launch_warp_items(const fj_graph* g, const SolveWs* ws, const Op& op, cudaStream_t st) {
  static int occ = 0;   // per template instantiation
  if (occ == 0) {
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, warp_kernel<WT, Op>, WTPB, 0);
    if (e != cudaSuccess) return e;
    if (occ < 1) occ = 1;
  }
  int64_t grid = (int64_t)g->num_sms * occ;
  const int64_t need = (g->s1.n_items + WPB - 1) / WPB;
  if (grid > need) grid = need > 0 ? need : 1;
  if (grid > ws->grid_max) grid = ws->grid_max;
  warp_kernel<WT, Op><<<(unsigned)grid, WTPB, 0, st>>>(make_sched(g, g->s1), op, ws->ts);
  return cudaGetLastError();
}

// The engine on an explicit schedule / scratch.
template <int WT, class Op>
inline cudaError_t launch_items_on(const fj_graph* g, const Sched& S, const TileSched& ts, const Op& op,
                                   const TileScratch& scr, int grid_max, cudaStream_t st, bool pdl = false) {
  static int occ = 0;   // per template instantiation
  if (occ == 0) {
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, warp_kernel<WT, Op>, WTPB, 0);
    if (e != cudaSuccess) return e;
    if (occ < 1) occ = 1;
  }
  int64_t grid = (int64_t)g->num_sms * occ;
  const int64_t need = (S.n_items + WPB - 1) / WPB;
  if (grid > need) grid = need > 0 ? need : 1;
  if (grid > grid_max) grid = grid_max;
  if (pdl) return pdl_launch(warp_kernel<WT, Op>, dim3((unsigned)grid), dim3(WTPB), st, ts, op, scr);
  warp_kernel<WT, Op><<<(unsigned)grid, WTPB, 0, st>>>(ts, op, scr);
  return cudaGetLastError();
}

// The work-item list matching an operator's tile size (Op::ITEMS).
template <class Op>
inline const Sched& sched_of(const fj_graph* g) {
  return Op::ITEMS == ITEMS ? g->s1 : g->sv;
}

// A product of the ApplyOp family (ApplyOp / ApplyOpV): one whole-row launch with the workspace
// scratch.  Returns the number of kernel launches (for accounting) through *launches.
template <int WT, class Op>
inline cudaError_t launch_product(const fj_graph* g, const TileScratch& scr, int grid_max, const Op& op,
                                  cudaStream_t st, int* launches, bool pdl = false) {
  *launches = 1;
  const Sched& S = sched_of<Op>(g);
  return launch_items_on<WT>(g, S, make_sched(g, S), op, scr, grid_max, st, pdl);
}

}  // namespace fj

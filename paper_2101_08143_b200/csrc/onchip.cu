// onchip.cu — rows a4-a6 for SMALL graphs in ONE thread block, everything in shared memory.
//
// The paper's workloads include many small graphs (Table 1: n' = 5 K .. 100 K) and
// BASELINE configs[0] is BA n = 2000.  There the multi-kernel path is launch- and latency-bound
// (C1: 24 iterations x 3 kernels + graph launch + separate residual and quantities passes,
// ~30 us per iteration for ~0.1 MB of data).  When the CSR and the solver's vectors fit in one SM's
// shared memory (up to 227 KB), one 1024-thread block runs the whole solve of a column -- Jacobi-PCG
// from x0 = 0 with the true-residual check and restarts (same algebra and stopping rule as pcg.cu),
// then the fused quantities pass (the 10 sums of QuantOp, ops.cuh) -- with block barriers instead of
// kernel boundaries and no global memory traffic beyond loading the graph once and writing z.
// Reductions are fixed block trees (bitwise reproducible).
#include <cstring>

#include "ops.cuh"
#include "workspace.cuh"

namespace fj {

constexpr int OC_TPB = 1024;
constexpr size_t OC_SMEM_MAX = 220 * 1024;

struct OnchipOut {
  double t[10];       // QuantOp sums (ops.cuh order)
  double rr, ss;      // recursive ||r||^2 and ||s||^2 at exit
  int32_t iters, restarts, converged, breakdown;
};

// bytes of dynamic shared memory for a graph: row ends (int32 n+1), cols (int32), weights,
// 6 fp64 vectors (s, x, r, p, q, dinv) and the degrees (weighted graphs)
inline size_t onchip_bytes(int64_t n, int64_t nnz, int wbytes) {
  size_t b = 0;
  auto add = [&](size_t x) { b = (b + x + 15) & ~(size_t)15; };
  add(4 * (size_t)(n + 1));
  add(4 * (size_t)nnz);
  add((size_t)wbytes * nnz);
  for (int v = 0; v < (wbytes ? 7 : 6); ++v) add(8 * (size_t)n);   // carved one by one, as k_onchip does
  return b;
}

template <int NP>
__device__ __forceinline__ void oc_sum(double (&v)[NP], double* s_red, double* s_out) {
  block_sum<NP, OC_TPB>(v, s_red);   // result in thread 0
  if (threadIdx.x == 0) {
#pragma unroll
    for (int j = 0; j < NP; ++j) s_out[j] = v[j];
  }
  __syncthreads();
#pragma unroll
  for (int j = 0; j < NP; ++j) v[j] = s_out[j];
  __syncthreads();
}

template <int WT>
__global__ void __launch_bounds__(OC_TPB, 1) k_onchip(int n, int nnz, const int64_t* __restrict__ rp_g,
                                                      const int32_t* __restrict__ col_g, const void* __restrict__ w_g,
                                                      const double* __restrict__ s_g, int64_t ld, int64_t cc,
                                                      double mean, double rtol, int max_iter, int max_restarts,
                                                      double* __restrict__ z_g, OnchipOut* out) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ double s_red[16 * OC_TPB / 32];
  __shared__ double s_bc[16];
  constexpr bool WEIGHTED = WT != FJ_W_UNIT;
  constexpr int WB = WT == FJ_W_UNIT ? 0 : WT == FJ_W_U8 ? 1 : WT == FJ_W_F32 ? 4 : 8;
  size_t off = 0;
  auto carve = [&](size_t bytes) { unsigned char* p = smem + off; off = (off + bytes + 15) & ~(size_t)15; return p; };
  int32_t* rp = reinterpret_cast<int32_t*>(carve(4 * (size_t)(n + 1)));
  int32_t* col = reinterpret_cast<int32_t*>(carve(4 * (size_t)nnz));
  unsigned char* wv = carve((size_t)WB * nnz);
  double* s = reinterpret_cast<double*>(carve(8 * (size_t)n));
  double* x = reinterpret_cast<double*>(carve(8 * (size_t)n));
  double* r = reinterpret_cast<double*>(carve(8 * (size_t)n));
  double* p = reinterpret_cast<double*>(carve(8 * (size_t)n));
  double* q = reinterpret_cast<double*>(carve(8 * (size_t)n));
  double* dinv = reinterpret_cast<double*>(carve(8 * (size_t)n));
  double* deg = WEIGHTED ? reinterpret_cast<double*>(carve(8 * (size_t)n)) : nullptr;
  const int tid = threadIdx.x;
  // ---- load the graph and the column
  for (int i = tid; i <= n; i += OC_TPB) rp[i] = (int32_t)rp_g[i];
  for (int e = tid; e < nnz; e += OC_TPB) col[e] = col_g[e];
  if (WEIGHTED)
    for (int e = tid; e < nnz * WB; e += OC_TPB) wv[e] = reinterpret_cast<const unsigned char*>(w_g)[e];
  for (int i = tid; i < n; i += OC_TPB) s[i] = s_g[(int64_t)i * ld + cc];
  __syncthreads();
  auto wgt = [&](int e) -> double {
    if (WT == FJ_W_U8) return (double)wv[e];
    if (WT == FJ_W_F32) return (double)reinterpret_cast<const float*>(wv)[e];
    if (WT == FJ_W_F64) return reinterpret_cast<const double*>(wv)[e];
    return 1.0;
  };
  // degrees in ascending column order (bit-exact with graph.cu and the oracle), Jacobi diagonal
  for (int i = tid; i < n; i += OC_TPB) {
    double d = 0.0;
    if (WEIGHTED) {
      for (int e = rp[i]; e < rp[i + 1]; ++e) d += wgt(e);
      deg[i] = d;
    } else {
      d = (double)(rp[i + 1] - rp[i]);
    }
    dinv[i] = 1.0 / (1.0 + d);
  }
  __syncthreads();
  auto degree = [&](int i) -> double { return WEIGHTED ? deg[i] : (double)(rp[i + 1] - rp[i]); };
  // y = (I+L) v at row i
  auto ipl = [&](const double* v, int i) -> double {
    double a = 0.0;
    for (int e = rp[i]; e < rp[i + 1]; ++e) a = WEIGHTED ? fma(wgt(e), v[col[e]], a) : a + v[col[e]];
    return fma(1.0 + degree(i), v[i], -a);
  };
  double acc1[1];
  acc1[0] = 0.0;
  for (int i = tid; i < n; i += OC_TPB) acc1[0] = fma(s[i], s[i], acc1[0]);
  oc_sum<1>(acc1, s_red, s_bc);
  const double ss = acc1[0], tol2 = rtol * rtol * ss;
  int iters = 0, restarts = 0, breakdown = 0, converged = 0;
  double rr = ss;
  bool first = true;
  for (;;) {
    // (re)start: r = s - (I+L) x (x = 0 on the first pass), p = dinv o r, rho = r^T p
    double v2[2] = {0.0, 0.0};
    for (int i = tid; i < n; i += OC_TPB) {
      double ri = s[i];
      if (first) x[i] = 0.0;
      else ri = s[i] - ipl(x, i);
      r[i] = ri;
      const double pi = dinv[i] * ri;
      p[i] = pi;
      v2[0] = fma(ri, pi, v2[0]);
      v2[1] = fma(ri, ri, v2[1]);
    }
    oc_sum<2>(v2, s_red, s_bc);
    double rho = v2[0];
    rr = v2[1];
    first = false;
    while (rr > tol2 && iters < max_iter) {
      double v1[1] = {0.0};
      for (int i = tid; i < n; i += OC_TPB) {
        const double qi = ipl(p, i);
        q[i] = qi;
        v1[0] = fma(p[i], qi, v1[0]);
      }
      oc_sum<1>(v1, s_red, s_bc);   // the barrier also orders q before the update
      const double pq = v1[0];
      if (!(pq > 0.0) || !isfinite(pq)) { breakdown = 1; break; }
      const double alpha = rho / pq;
      double v3[2] = {0.0, 0.0};
      for (int i = tid; i < n; i += OC_TPB) {
        x[i] = fma(alpha, p[i], x[i]);
        const double ri = fma(-alpha, q[i], r[i]);
        r[i] = ri;
        v3[0] = fma(ri, dinv[i] * ri, v3[0]);
        v3[1] = fma(ri, ri, v3[1]);
      }
      oc_sum<2>(v3, s_red, s_bc);
      ++iters;
      rr = v3[1];
      if (rr <= tol2) break;
      const double beta = v3[0] / rho;
      rho = v3[0];
      for (int i = tid; i < n; i += OC_TPB) p[i] = fma(beta, p[i], dinv[i] * r[i]);
      __syncthreads();
    }
    // true residual ||s - (I+L) x||^2
    double vt[1] = {0.0};
    for (int i = tid; i < n; i += OC_TPB) {
      const double e = s[i] - ipl(x, i);
      vt[0] = fma(e, e, vt[0]);
    }
    oc_sum<1>(vt, s_red, s_bc);
    converged = vt[0] <= tol2;
    if (converged || breakdown || restarts >= max_restarts || iters >= max_iter) break;
    ++restarts;
  }
  // ---- fused quantities pass (QuantOp order): 0 (z-s)^2, 1 sum_j w (z_i - z_j)^2, 2 (z-m)^2, 3 z^2,
  // 4 s z, 5 (s-m)(z-m), 6 (s - (I+L)z)^2, 7 (Lz)^2, 8 rounding allowance^2, 9 s^2
  double t[10];
#pragma unroll
  for (int j = 0; j < 10; ++j) t[j] = 0.0;
  for (int i = tid; i < n; i += OC_TPB) {
    const double zi = x[i], si = s[i];
    double A = 0.0, Dd = 0.0, Aa = 0.0;
    for (int e = rp[i]; e < rp[i + 1]; ++e) {
      const double wgt_e = wgt(e), zj = x[col[e]], df = zi - zj;
      A = fma(wgt_e, zj, A);
      Dd = fma(wgt_e * df, df, Dd);
      Aa = fma(wgt_e, fabs(zj), Aa);
    }
    const double d = degree(i);
    const double tt = fma(1.0 + d, zi, -A), lz = fma(d, zi, -A), rres = si - tt;
    const double e1 = zi - si, e2 = zi - mean, e3 = si - mean;
    const double ab = fabs(si) + fma(1.0 + d, fabs(zi), Aa);
    t[0] = fma(e1, e1, t[0]);
    t[1] += Dd;
    t[2] = fma(e2, e2, t[2]);
    t[3] = fma(zi, zi, t[3]);
    t[4] = fma(si, zi, t[4]);
    t[5] = fma(e3, e2, t[5]);
    t[6] = fma(rres, rres, t[6]);
    t[7] = fma(lz, lz, t[7]);
    t[8] = fma(ab, ab, t[8]);
    t[9] = fma(si, si, t[9]);
    z_g[(int64_t)i * ld + cc] = zi;
  }
  block_sum<10, OC_TPB>(t, s_red);
  if (tid == 0) {
#pragma unroll
    for (int j = 0; j < 10; ++j) out->t[j] = t[j];
    out->rr = rr;
    out->ss = ss;
    out->iters = iters;
    out->restarts = restarts;
    out->converged = converged;
    out->breakdown = breakdown;
  }
}

// Whole-solve fast path for column c of [n][ld] s -> z: *used = false when the graph does not fit.
fj_status onchip_col(fj_graph* g, const double* s, double* z, int64_t ld, int64_t c, double mean,
                     const fj_solve_opts& o, double* t10, int* iters, int* restarts, double* rel_true,
                     double* rel_rec, bool* converged, bool* used, cudaStream_t st) {
  *used = false;
  const int wb = g->wtype == FJ_W_UNIT ? 0 : g->wtype == FJ_W_U8 ? 1 : g->wtype == FJ_W_F32 ? 4 : 8;
  const size_t bytes = onchip_bytes(g->n, g->nnz, wb);
  static const bool off = getenv("FJ_ONCHIP") && atoi(getenv("FJ_ONCHIP")) == 0;   // A/B knob
  if (off || g->dist || g->n < 1 || g->nnz >= INT32_MAX || bytes > OC_SMEM_MAX) return FJ_OK;
  OnchipOut* dout = nullptr;
  FJ_CK(dmalloc(&dout, sizeof(OnchipOut), st));
  cudaError_t e = cudaSuccess;
  auto go = [&](auto kern) {
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e == cudaSuccess) {
      kern<<<1, OC_TPB, bytes, st>>>((int)g->n, (int)g->nnz, g->row_ptr, g->col, g->w, s, ld, c, mean, o.rtol,
                                    o.max_iter, o.max_restarts, z, dout);
      e = cudaGetLastError();
    }
  };
  switch (g->wtype) {
    case FJ_W_UNIT: go(k_onchip<FJ_W_UNIT>); break;
    case FJ_W_U8: go(k_onchip<FJ_W_U8>); break;
    case FJ_W_F32: go(k_onchip<FJ_W_F32>); break;
    default: go(k_onchip<FJ_W_F64>); break;
  }
  OnchipOut h{};
  if (e == cudaSuccess) {
    count_launch();
    e = cudaMemcpyAsync(&h, dout, sizeof h, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  }
  dfree_on(dout, st);
  if (e != cudaSuccess) return cuda_fail(e, "k_onchip", __FILE__, __LINE__);
  memcpy(t10, h.t, sizeof h.t);
  *iters = h.iters;
  *restarts = h.restarts;
  *rel_true = h.ss > 0 ? std::sqrt(h.t[6] / h.ss) : 0.0;
  *rel_rec = h.ss > 0 ? std::sqrt(h.rr / h.ss) : 0.0;
  *converged = h.converged != 0;
  *used = true;
  return FJ_OK;
}

}  // namespace fj

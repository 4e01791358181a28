// quantities.cu — rows a3 (opinion statistics), a5-a7 (fused quantities pass + certificate) and
// Algorithm 1 in single-solve form (fj_approxim), plus the host-buffer e2e entry point.
#include <cmath>
#include <cstring>
#include <limits>
#include <vector>

#include "ops.cuh"
#include "rows.cuh"
#include "workspace.cuh"

namespace fj {

fj_status solve_col(fj_graph* g, const double* s, double* z, int64_t ld, int64_t c, const fj_solve_opts& o,
                    int warm, fj_solve_report* rep, cudaStream_t st, int* iters_out,
                    bool defer = false);

void free_quant_ws(fj_graph*) {}

// ---------------------------------------------------------------- a3: statistics of column c
constexpr int STPB = 256;

// Last block of a stats kernel: K columns of (sum, sum of squares, min, max) quads at
// part[q * 4K + 4c + j] for the grid's blocks q.  Every thread folds the blocks q = t, t + STPB, ...
// (fixed order), then fixed-order block sums / min-max trees: deterministic, and STPB loads in
// flight instead of one thread walking all blocks (that serial walk cost ~0.25 ms per call).
template <int K>
__device__ __forceinline__ void stats_last_block(const double* part, int kk, unsigned nblocks, double* out,
                                                 const int* nonfinite, double* s_red, double (*s_mm)[STPB / 32]) {
  double v[2 * K], mn[K], mx[K];
#pragma unroll
  for (int c = 0; c < K; ++c) { v[2 * c] = 0.0; v[2 * c + 1] = 0.0; mn[c] = INFINITY; mx[c] = -INFINITY; }
  for (unsigned q = threadIdx.x; q < nblocks; q += STPB) {
#pragma unroll
    for (int c = 0; c < K; ++c) {
      const double* pq = part + (int64_t)q * 4 * K + 4 * c;
      v[2 * c] += __ldcg(pq + 0);
      v[2 * c + 1] += __ldcg(pq + 1);
      mn[c] = fmin(mn[c], __ldcg(pq + 2));
      mx[c] = fmax(mx[c], __ldcg(pq + 3));
    }
  }
  block_sum<2 * K, STPB>(v, s_red);
#pragma unroll
  for (int c = 0; c < K; ++c) {
    for (int o = 16; o > 0; o >>= 1) {
      mn[c] = fmin(mn[c], __shfl_xor_sync(0xffffffffu, mn[c], o));
      mx[c] = fmax(mx[c], __shfl_xor_sync(0xffffffffu, mx[c], o));
    }
  }
  __syncthreads();   // s_mm is reused
  if ((threadIdx.x & 31) == 0) {
#pragma unroll
    for (int c = 0; c < K; ++c) { s_mm[2 * c][threadIdx.x >> 5] = mn[c]; s_mm[2 * c + 1][threadIdx.x >> 5] = mx[c]; }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const bool bad = *(volatile const int*)nonfinite != 0;
    for (int c = 0; c < kk && c < K; ++c) {
      for (int w = 1; w < STPB / 32; ++w) { mn[c] = fmin(mn[c], s_mm[2 * c][w]); mx[c] = fmax(mx[c], s_mm[2 * c + 1][w]); }
      out[4 * c + 0] = bad ? NAN : v[2 * c];   // NaN marks a non-finite input (propagates over ranks)
      out[4 * c + 1] = v[2 * c + 1];
      out[4 * c + 2] = mn[c];
      out[4 * c + 3] = mx[c];
    }
  }
}

__global__ void __launch_bounds__(STPB) k_stats(int64_t n, const double* __restrict__ s, int64_t ld, int64_t c,
                                                double* part /*[grid][4]*/, unsigned int* ticket, double* out,
                                                int* nonfinite) {
  __shared__ double s_red[4 * STPB / 32];
  __shared__ bool s_last;
  double sm = 0.0, sq = 0.0, mn = INFINITY, mx = -INFINITY;
  int bad = 0;
  for (int64_t i = blockIdx.x * (int64_t)STPB + threadIdx.x; i < n; i += (int64_t)gridDim.x * STPB) {
    const double x = s[i * ld + c];
    if (!isfinite(x)) { bad = 1; continue; }
    sm += x;
    sq = fma(x, x, sq);
    mn = fmin(mn, x);
    mx = fmax(mx, x);
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(nonfinite, 1);
  double v[2] = {sm, sq};
  block_sum<2, STPB>(v, s_red);
  // min / max: warp + smem
  for (int o = 16; o > 0; o >>= 1) {
    mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  __shared__ double s_mm[2 * STPB / 32];
  if ((threadIdx.x & 31) == 0) { s_mm[threadIdx.x >> 5] = mn; s_mm[STPB / 32 + (threadIdx.x >> 5)] = mx; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < STPB / 32; ++w) { mn = fmin(mn, s_mm[w]); mx = fmax(mx, s_mm[STPB / 32 + w]); }
    part[blockIdx.x * 4 + 0] = v[0];
    part[blockIdx.x * 4 + 1] = v[1];
    part[blockIdx.x * 4 + 2] = mn;
    part[blockIdx.x * 4 + 3] = mx;
    __threadfence();
    s_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (s_last) {
    __threadfence();
    __shared__ double s_mm2[2][STPB / 32];
    stats_last_block<1>(part, 1, gridDim.x, out, nonfinite, s_red, s_mm2);
    if (threadIdx.x == 0) *ticket = 0u;
  }
}

// All k <= 4 columns of row-major [n][k] in one pass (one thread per row); same outputs as k_stats
// per column: out[4c + {0,1,2,3}] = (sum, sum of squares, min, max), NaN sum on non-finite input.
template <int K>
__global__ void __launch_bounds__(STPB) k_stats_k(int64_t n, int k, const double* __restrict__ s,
                                                  double* part /*[grid][4K]*/, unsigned int* ticket, double* out,
                                                  int* nonfinite) {
  __shared__ double s_red[2 * K * STPB / 32];
  __shared__ double s_mm[2 * K][STPB / 32];
  __shared__ bool s_last;
  double v[2 * K], mn[K], mx[K];
#pragma unroll
  for (int c = 0; c < K; ++c) { v[2 * c] = 0.0; v[2 * c + 1] = 0.0; mn[c] = INFINITY; mx[c] = -INFINITY; }
  int bad = 0;
  for (int64_t i = blockIdx.x * (int64_t)STPB + threadIdx.x; i < n; i += (int64_t)gridDim.x * STPB) {
#pragma unroll
    for (int c = 0; c < K; ++c) {
      if (c < k) {
        const double x = s[i * k + c];
        if (!isfinite(x)) { bad = 1; continue; }
        v[2 * c] += x;
        v[2 * c + 1] = fma(x, x, v[2 * c + 1]);
        mn[c] = fmin(mn[c], x);
        mx[c] = fmax(mx[c], x);
      }
    }
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(nonfinite, 1);
  block_sum<2 * K, STPB>(v, s_red);
#pragma unroll
  for (int c = 0; c < K; ++c) {
    for (int o = 16; o > 0; o >>= 1) {
      mn[c] = fmin(mn[c], __shfl_xor_sync(0xffffffffu, mn[c], o));
      mx[c] = fmax(mx[c], __shfl_xor_sync(0xffffffffu, mx[c], o));
    }
    if ((threadIdx.x & 31) == 0) { s_mm[2 * c][threadIdx.x >> 5] = mn[c]; s_mm[2 * c + 1][threadIdx.x >> 5] = mx[c]; }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int c = 0; c < K; ++c) {
      for (int w = 1; w < STPB / 32; ++w) { mn[c] = fmin(mn[c], s_mm[2 * c][w]); mx[c] = fmax(mx[c], s_mm[2 * c + 1][w]); }
      part[blockIdx.x * 4 * K + 4 * c + 0] = v[2 * c];
      part[blockIdx.x * 4 * K + 4 * c + 1] = v[2 * c + 1];
      part[blockIdx.x * 4 * K + 4 * c + 2] = mn[c];
      part[blockIdx.x * 4 * K + 4 * c + 3] = mx[c];
    }
    __threadfence();
    s_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (s_last) {
    __threadfence();
    stats_last_block<K>(part, k, gridDim.x, out, nonfinite, s_red, s_mm);
    if (threadIdx.x == 0) *ticket = 0u;
  }
}

// All k <= 64 columns of row-major [n][k] in one pass: warp per row, lane l owns columns l and l + 32
// (coalesced row reads), per-column partials reduced warps -> blocks in a fixed order; same outputs
// as k_stats per column.
__global__ void __launch_bounds__(STPB) k_stats_wide(int64_t n, int k, const double* __restrict__ s,
                                                     double* part /*[grid][4][64]*/, unsigned int* ticket,
                                                     double* out, int* nonfinite) {
  constexpr int NW = STPB / 32;
  __shared__ double s_v[NW][4][64];
  __shared__ bool s_last;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  double sm[2] = {0.0, 0.0}, sq[2] = {0.0, 0.0}, mn[2] = {INFINITY, INFINITY}, mx[2] = {-INFINITY, -INFINITY};
  int bad = 0;
  for (int64_t i = blockIdx.x * (int64_t)NW + wib; i < n; i += (int64_t)gridDim.x * NW) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int c = lane + 32 * h;
      if (c < k) {
        const double x = s[i * k + c];
        if (!isfinite(x)) { bad = 1; continue; }
        sm[h] += x;
        sq[h] = fma(x, x, sq[h]);
        mn[h] = fmin(mn[h], x);
        mx[h] = fmax(mx[h], x);
      }
    }
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(nonfinite, 1);
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int c = lane + 32 * h;
    s_v[wib][0][c] = sm[h]; s_v[wib][1][c] = sq[h]; s_v[wib][2][c] = mn[h]; s_v[wib][3][c] = mx[h];
  }
  __syncthreads();
  if (threadIdx.x < 64) {
    const int c = threadIdx.x;
    double a = 0.0, b = 0.0, lo = INFINITY, hi = -INFINITY;
    for (int w = 0; w < NW; ++w) {   // warps in order
      a += s_v[w][0][c]; b += s_v[w][1][c]; lo = fmin(lo, s_v[w][2][c]); hi = fmax(hi, s_v[w][3][c]);
    }
    double* pb = part + (int64_t)blockIdx.x * 256;
    pb[c] = a; pb[64 + c] = b; pb[128 + c] = lo; pb[192 + c] = hi;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  {   // thread group g = t / 64 folds blocks q = g, g + 4, ... for column c = t % 64; groups in order
    constexpr int NG = STPB / 64;
    const int c = threadIdx.x & 63, grp = threadIdx.x >> 6;
    double a = 0.0, b = 0.0, lo = INFINITY, hi = -INFINITY;
    if (c < k) {
      for (unsigned q = grp; q < gridDim.x; q += NG) {
        const double* pb = part + (int64_t)q * 256;
        a += __ldcg(pb + c); b += __ldcg(pb + 64 + c);
        lo = fmin(lo, __ldcg(pb + 128 + c)); hi = fmax(hi, __ldcg(pb + 192 + c));
      }
    }
    __syncthreads();   // s_v reused: [group][quantity][column]
    s_v[grp][0][c] = a; s_v[grp][1][c] = b; s_v[grp][2][c] = lo; s_v[grp][3][c] = hi;
    __syncthreads();
    if (threadIdx.x < 64 && threadIdx.x < k) {
      a = 0.0; b = 0.0; lo = INFINITY; hi = -INFINITY;
      for (int g2 = 0; g2 < NG; ++g2) {
        a += s_v[g2][0][c]; b += s_v[g2][1][c]; lo = fmin(lo, s_v[g2][2][c]); hi = fmax(hi, s_v[g2][3][c]);
      }
      out[4 * c + 0] = *(volatile int*)nonfinite ? NAN : a;
      out[4 * c + 1] = b; out[4 * c + 2] = lo; out[4 * c + 3] = hi;
    }
  }
  if (threadIdx.x == 0) *ticket = 0u;
}

static fj_status stats_cols(fj_graph* g, SolveWs* w, int k, const double* s, std::vector<double>& st4,
                            cudaStream_t st) {
  int* d_bad = nullptr;
  FJ_CK(dmalloc(&d_bad, sizeof(int), st));
  FJ_CK(cudaMemsetAsync(d_bad, 0, sizeof(int), st));
  if (k > 1 && k <= 4) {   // one pass over all columns (SolveWs::elem_part holds grid x 16 doubles)
    k_stats_k<4><<<w->grid_elem, STPB, 0, st>>>(g->n, k, s, w->elem_part, w->elem_ticket, w->stat, d_bad);
    FJ_CK_LAUNCH();
  } else if (k > 4) {   // one pass, warp per row (part: grid x 256 doubles in a transient buffer)
    double* part = nullptr;
    FJ_CK(dmalloc(&part, sizeof(double) * 256 * (size_t)w->grid_elem, st));
    k_stats_wide<<<w->grid_elem, STPB, 0, st>>>(g->n, k, s, part, w->elem_ticket, w->stat, d_bad);
    FJ_CK_LAUNCH();
    dfree_on(part, st);
  } else {
    for (int c = 0; c < k; ++c) {
      k_stats<<<w->grid_elem, STPB, 0, st>>>(g->n, s, k, c, w->elem_part, w->elem_ticket, w->stat + 4 * c, d_bad);
      FJ_CK_LAUNCH();
    }
  }
  if (is_dist(g)) FJ_TRY(dist_stats_combine(g, k, w->stat, st));   // global over the ranks' slices
  st4.assign(4 * k, 0.0);
  FJ_CK(cudaMemcpyAsync(st4.data(), w->stat, sizeof(double) * 4 * k, cudaMemcpyDeviceToHost, st));
  dfree_on(d_bad, st);
  FJ_CK(cudaStreamSynchronize(st));
  for (int c = 0; c < k; ++c)   // k_stats poisons the sum with NaN when a slice held NaN / Inf
    if (std::isnan(st4[4 * c])) return fail(FJ_E_NONFINITE_INPUT, "opinion vector contains NaN or Inf");
  return FJ_OK;
}

// ---------------------------------------------------------------- a6: fused pass for column c
template <int WT>
static fj_status launch_quant_wt(const fj_graph* g, const SolveWs* w, const double* s, const double* z, int64_t ld,
                                 int64_t c, double m, cudaStream_t st) {
  QuantOp<WT> op{z, s, g->deg, ld, c, m, w->qout};
  if (w->rows && w->rows->mode != 0) return rows_op<WT>(*w->rows, g->n, g->col, g->w, op, st);   // rows.cuh
  FJ_CK(launch_warp_items<WT>(g, w, op, st));
  FJ_CK_LAUNCH();
  return FJ_OK;
}

static fj_status quant_pass(const fj_graph* g, const SolveWs* w, const double* s, const double* z, int64_t ld,
                            int64_t c, double m, double* host10, cudaStream_t st) {
  if (is_dist(g)) return dist_quant_pass(g, s, z, ld, c, m, host10, st);
  fj_status r;
  switch (g->wtype) {
    case FJ_W_UNIT: r = launch_quant_wt<FJ_W_UNIT>(g, w, s, z, ld, c, m, st); break;
    case FJ_W_U8: r = launch_quant_wt<FJ_W_U8>(g, w, s, z, ld, c, m, st); break;
    case FJ_W_F32: r = launch_quant_wt<FJ_W_F32>(g, w, s, z, ld, c, m, st); break;
    default: r = launch_quant_wt<FJ_W_F64>(g, w, s, z, ld, c, m, st); break;
  }
  FJ_TRY(r);
  FJ_CK(cudaMemcpyAsync(host10, w->qout, sizeof(double) * 10, cudaMemcpyDeviceToHost, st));
  FJ_CK(cudaStreamSynchronize(st));
  return FJ_OK;
}

// ---------------------------------------------------------------- a7: certificate (host)
// For Q = ||v||^2 computed as Qt = ||vt||^2 with ||vt - v|| <= R:
//   Q in [(a - R)^2, (a + R)^2], a = sqrt(Qt)  =>  |Qt - Q| / Q <= (2 a R + R^2) / (a - R)^2.
// R bounds ||z - z*||: lambda_min(I+L) = 1 gives ||e|| <= ||e||_{I+L} <= ||r|| and
// ||W^{1/2} B e|| = ||e||_L <= ||e||_{I+L} <= ||r||; this is the proof pattern of Lemma 4.3
// applied a posteriori.  R = computed ||r|| + rounding allowance gamma ||a||.
static double cert_eps(double Qt, double R, double rel_sum) {
  if (Qt <= 0.0) return R == 0.0 ? 0.0 : std::numeric_limits<double>::infinity();
  const double a = std::sqrt(Qt);
  if (!(a > R)) return std::numeric_limits<double>::infinity();
  return (2.0 * a * R + R * R) / ((a - R) * (a - R)) + rel_sum;
}

static void fill_quantities(const fj_graph* g, const double* t, double mean_s, fj_quantities_t& q) {
  const double n = (double)global_n(g);
  q.CI = t[0];
  q.D = 0.5 * t[1];   // each undirected edge was visited from both ends
  q.P = t[2];
  q.C = t[3];
  q.Idc = q.D + q.C;
  q.PDI = q.P + q.D;
  q.mean_s = mean_s;
  q.sz = t[4];
  q.sbzb = t[5];
  q.Lz2 = t[7];
  q.ss = t[9];
  q.res_norm = std::sqrt(t[6]);
  q.s_norm = std::sqrt(t[9]);
  const double u = std::ldexp(1.0, -53);
  const double lg = std::ceil(std::log2(global_dmax(g) + 2.0));
  const double gamma = (32.0 + lg + 4.0) * u;     // row sums: <= 32 sequential + tree levels
  q.fp_bound = gamma * std::sqrt(t[8]);
  const double R = q.res_norm * (1.0 + 1e-12) + q.fp_bound;
  const double rel_sum = (std::ceil(std::log2(n + 1.0)) + 40.0) * u;   // summation of the squares
  const double eC = cert_eps(q.C, R, rel_sum), eD = cert_eps(q.D, R, rel_sum);
  const double eP = cert_eps(q.P, R, rel_sum), eI = cert_eps(q.CI, R, rel_sum);
  q.eps[0] = eI;
  q.eps[1] = eD;
  q.eps[2] = eP;
  q.eps[3] = eC;
  q.eps[4] = std::max(eD, eC);   // eps-approximation closed under sums
  q.eps[5] = std::max(eP, eD);
  q.certified = 1;
  for (int j = 0; j < 6; ++j)
    if (!std::isfinite(q.eps[j])) q.certified = 0;
  q.consensus = 0;
}

static void consensus_quantities(const fj_graph* g, double c, fj_quantities_t& q) {
  memset(&q, 0, sizeof q);
  const double n = (double)global_n(g);
  q.C = n * c * c;          // z = s = c 1 exactly (Omega 1 = 1)
  q.Idc = q.C;
  q.mean_s = c;
  q.ss = q.C;
  q.sz = q.C;
  q.s_norm = std::sqrt(q.C);
  q.consensus = 1;
  q.certified = 1;
}

__global__ void k_copy_cols(int64_t n, int64_t k, int64_t c, const double* __restrict__ s, double* __restrict__ z) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    z[i * k + c] = s[i * k + c];
}

}  // namespace fj

using namespace fj;

extern "C" {

fj_status fj_opinion_stats(const fj_graph* gc, int k, const double* s, double* stats_host, void* stream) {
  FJ_RANGE("fj_opinion_stats");
  if (!gc || !s || !stats_host) return fail(FJ_E_INVALID_ARG, "null argument");
  if (k < 1 || k > MAXK) return fail(FJ_E_INVALID_ARG, "k must be in [1, 64]");
  fj_graph* g = const_cast<fj_graph*>(gc);
  cudaStream_t st = S(stream);
  SolveWs* w = nullptr;
  FJ_TRY(get_ws(g, st, &w));
  std::vector<double> v;
  FJ_TRY(stats_cols(g, w, k, s, v, st));
  memcpy(stats_host, v.data(), sizeof(double) * 4 * k);
  return FJ_OK;
}

fj_status fj_quantities(const fj_graph* gc, int k, const double* s, const double* z, fj_quantities_t* out,
                        void* stream) {
  FJ_RANGE("fj_quantities");
  if (!gc || !s || !z || !out) return fail(FJ_E_INVALID_ARG, "null argument");
  if (k < 1 || k > MAXK) return fail(FJ_E_INVALID_ARG, "k must be in [1, 64]");
  fj_graph* g = const_cast<fj_graph*>(gc);
  cudaStream_t st = S(stream);
  SolveWs* w = nullptr;
  FJ_TRY(get_ws(g, st, &w));
  std::vector<double> v;
  FJ_TRY(stats_cols(g, w, k, s, v, st));
  if (k >= batch_min_k() && !is_dist(g)) {   // all columns in one pass
    std::vector<double> means(k), sums(10 * (size_t)k);
    for (int c = 0; c < k; ++c) means[c] = v[4 * c] / (double)global_n(g);
    FJ_TRY(quant_batch(g, k, s, z, means.data(), sums.data(), st));
    for (int c = 0; c < k; ++c) {
      memset(&out[c], 0, sizeof(fj_quantities_t));
      fill_quantities(g, &sums[10 * (size_t)c], means[c], out[c]);
    }
    return FJ_OK;
  }
  for (int c = 0; c < k; ++c) {
    double t[10];
    const double m = v[4 * c] / (double)global_n(g);
    FJ_TRY(quant_pass(g, w, s, z, k, c, m, t, st));
    memset(&out[c], 0, sizeof(fj_quantities_t));
    fill_quantities(g, t, m, out[c]);
  }
  return FJ_OK;
}

}  // extern "C"

// Algorithm 1 (fj_approxim).  z_host (host-buffer entry point only): after the batched solve the
// D2H of z runs on a side stream while the fused quantities pass runs on `stream`.
// z_host_perm (relabelled graph): z_host receives z[z_host_perm[i]] (staged in z_perm_buf).
static fj_status approxim_impl(const fj_graph* gc, int k, const double* s, double* z_user, const fj_solve_opts* opts,
                               fj_quantities_t* qout, fj_solve_report* rep, void* stream, double* z_host,
                               bool* z_host_done, const int32_t* z_host_perm = nullptr,
                               double* z_perm_buf = nullptr) {
  if (z_host_done) *z_host_done = false;
  if (!gc || !s || !qout) return fail(FJ_E_INVALID_ARG, "null argument");
  if (k < 1 || k > MAXK) return fail(FJ_E_INVALID_ARG, "k must be in [1, 64]");
  if (z_user == s) return fail(FJ_E_INVALID_ARG, "s and z must not alias");
  fj_solve_opts o;
  fj_default_solve_opts(&o);
  if (opts) o = *opts;
  if (!(o.rtol > 0.0) || o.max_iter < 0 || o.max_restarts < 0 || o.eps_target < 0)
    return fail(FJ_E_INVALID_ARG, "bad solve options");
  fj_graph* g = const_cast<fj_graph*>(gc);
  cudaStream_t st = S(stream);
  SolveWs* w = nullptr;
  FJ_TRY(get_ws(g, st, &w));
  double* z = z_user;
  DevBuf<double> zbuf;
  if (!z) {
    FJ_TRY(zbuf.alloc(g->n * (int64_t)k, st));
    z = zbuf.p;
  }
  FJ_CK(cudaEventRecord(w->ev0, st));
  // Algorithm 1 line 2: mean of s, plus the consensus short-circuit
  std::vector<double> v;
  FJ_TRY(stats_cols(g, w, k, s, v, st));
  fj_solve_report r{};
  r.converged = 1;
  r.rel_res_true = NAN;
  const unsigned cb = (unsigned)std::min<int64_t>((g->n + 255) / 256, 4096);
  fj_status worst = FJ_OK;
  SideStream side;            // z_host: D2H of z overlapping the quantities pass
  bool d2h_issued = false;
  if (k >= batch_min_k() && !is_dist(g)) {
    // row a9: all k columns in ONE batched PCG (per-column alpha/beta, convergence mask)
    // The solve defers its true-residual pass: the fused quantities pass computes ||s - (I+L)z||^2
    // per column anyway (QuantOp sum 6), so the restart decision is taken on it (one CSR pass less).
    fj_solve_opts oc = o;
    int warm = 0, spent = 0, restarts = 0;
    for (;;) {
      fj_solve_opts ob = oc;
      ob.max_iter = std::max(0, o.max_iter - spent);
      fj_solve_report rb{};
      rb.converged = 1;
      rb.rel_res_true = NAN;
      phase_tick("approxim: before solve", st);
      fj_status sc = solve_batch(g, k, s, z, ob, warm, &rb, st, /*defer_true_residual=*/true);   // Alg. 1 l.3
      if (sc != FJ_OK && sc != FJ_E_NO_CONVERGENCE) return sc;
      phase_tick("approxim: batched solve", st);
      spent += rb.iterations;
      r.ms_loop += rb.ms_loop;
      r.iterations_total += rb.iterations_total;
      r.restarts += rb.restarts;
      r.rel_res_recursive = rb.rel_res_recursive;
      r.batch_k = k;
      double emax = 0.0;
      std::vector<double> means(k), sums(10 * (size_t)k);
      bool z_is_solve = true;   // z untouched since the solve: its padded solver copy may be gathered
      for (int c = 0; c < k; ++c) {
        means[c] = v[4 * c] / (double)global_n(g);
        if (v[4 * c + 2] == v[4 * c + 3]) {   // s = c 1: z = s exactly (P:L129 Omega 1 = 1)
          k_copy_cols<<<cb, 256, 0, st>>>(g->n, k, c, s, z);
          FJ_CK_LAUNCH();
          z_is_solve = false;
        }
      }
      if (z_host) {   // z is final unless the residual check below restarts: copy it out meanwhile
        if (!side.s) FJ_TRY(side.init());
        FJ_CK(cudaEventRecord(side.ev_in, st));
        FJ_CK(cudaStreamWaitEvent(side.s, side.ev_in, 0));
        const double* zsrc = z;
        if (z_host_perm) {   // back to the input labels first (fj_permute_rows, on the side stream)
          FJ_TRY(fj_permute_rows(g->n, k, z_host_perm, z, z_perm_buf, side.s));
          zsrc = z_perm_buf;
        }
        FJ_CK(cudaMemcpyAsync(z_host, zsrc, sizeof(double) * g->n * k, cudaMemcpyDeviceToHost, side.s));
        FJ_CK(cudaEventRecord(side.ev_out, side.s));
        d2h_issued = true;
      }
      FJ_TRY(quant_batch(g, k, s, z, means.data(), sums.data(), st, z_is_solve));   // Alg. 1 lines 5-9
      bool res_ok = true;
      double worst_true = 0.0;
      for (int c = 0; c < k; ++c) {
        if (v[4 * c + 2] == v[4 * c + 3]) {
          consensus_quantities(g, v[4 * c + 2], qout[c]);
          continue;
        }
        memset(&qout[c], 0, sizeof(fj_quantities_t));
        fill_quantities(g, &sums[10 * (size_t)c], means[c], qout[c]);
        for (int j = 0; j < 6; ++j) emax = std::max(emax, qout[c].eps[j]);
        const double res2 = sums[10 * (size_t)c + 6], ss = sums[10 * (size_t)c + 9];
        if (res2 > oc.rtol * oc.rtol * ss) res_ok = false;
        if (ss > 0) worst_true = std::max(worst_true, std::sqrt(res2 / ss));
      }
      r.rel_res_true = worst_true;
      phase_tick("approxim: quantities", st);
      if (sc == FJ_OK && !res_ok) {   // true residual missed rtol: restart from z (warm)
        if (restarts < o.max_restarts && spent < o.max_iter) {
          ++restarts;
          ++r.restarts;
          warm = 1;
          if (d2h_issued) FJ_CK(cudaStreamWaitEvent(st, side.ev_out, 0));   // z is read by the copy
          d2h_issued = false;
          continue;
        }
        sc = FJ_E_NO_CONVERGENCE;
      }
      if (sc != FJ_OK) { worst = sc; break; }
      if (o.eps_target <= 0.0 || emax <= o.eps_target || oc.rtol <= 1e-15 || spent >= o.max_iter) break;
      oc.rtol = std::max(oc.rtol * 1e-2, 1e-15);   // tighten and continue from z (warm start)
      warm = 1;
      if (d2h_issued) FJ_CK(cudaStreamWaitEvent(st, side.ev_out, 0));
      d2h_issued = false;
    }
    r.iterations = spent;
  } else if (is_dist(g) && k <= 4) {
    // rows a8 + a9: the k <= 4 columns of this rank's slice solved together by the single-reduction
    // distributed PCG (dist.cu), then the per-column distributed quantities passes
    fj_solve_opts oc = o;
    int warm = 0, spent = 0;
    for (;;) {
      fj_solve_opts ob = oc;
      ob.max_iter = std::max(0, o.max_iter - spent);
      fj_solve_report rb{};
      rb.converged = 1;
      rb.rel_res_true = NAN;
      fj_status sc = dist_solve_cg(g, k, s, z, k, 0, ob, warm, &rb, st);   // Alg. 1 line 3
      if (sc != FJ_OK && sc != FJ_E_NO_CONVERGENCE) return sc;
      spent += rb.iterations;
      r.ms_loop += rb.ms_loop;
      r.iterations_total += rb.iterations_total;
      r.restarts += rb.restarts;
      r.rel_res_true = rb.rel_res_true;
      r.rel_res_recursive = rb.rel_res_recursive;
      r.batch_k = k;
      double emax = 0.0;
      for (int c = 0; c < k; ++c) {
        const double m = v[4 * c] / (double)global_n(g);
        if (v[4 * c + 2] == v[4 * c + 3]) {   // s = c 1: z = s exactly (P:L129 Omega 1 = 1)
          k_copy_cols<<<cb, 256, 0, st>>>(g->n, k, c, s, z);
          FJ_CK_LAUNCH();
          consensus_quantities(g, v[4 * c + 2], qout[c]);
          continue;
        }
        double t[10];
        FJ_TRY(quant_pass(g, w, s, z, k, c, m, t, st));   // Alg. 1 lines 5-9
        memset(&qout[c], 0, sizeof(fj_quantities_t));
        fill_quantities(g, t, m, qout[c]);
        for (int j = 0; j < 6; ++j) emax = std::max(emax, qout[c].eps[j]);
      }
      if (sc != FJ_OK) { worst = sc; break; }
      if (o.eps_target <= 0.0 || emax <= o.eps_target || oc.rtol <= 1e-15 || spent >= o.max_iter) break;
      oc.rtol = std::max(oc.rtol * 1e-2, 1e-15);   // tighten and continue from z (warm start)
      warm = 1;
    }
    r.iterations = spent;
  } else {
  for (int c = 0; c < k; ++c) {
    const double m = v[4 * c] / (double)global_n(g);
    if (v[4 * c + 2] == v[4 * c + 3]) {   // s = c 1: z = s exactly (P:L129 Omega 1 = 1)
      k_copy_cols<<<cb, 256, 0, st>>>(g->n, k, c, s, z);
      FJ_CK_LAUNCH();
      consensus_quantities(g, v[4 * c + 2], qout[c]);
      r.rel_res_true = std::isnan(r.rel_res_true) ? 0.0 : r.rel_res_true;
      continue;
    }
    fj_solve_opts oc = o;
    int iters = 0, warm = 0, spent = 0;
    double t[10];
    if (!is_dist(g) && o.eps_target <= 0.0) {   // small graph: the whole column in one block (onchip.cu)
      bool used = false, conv = false;
      int it = 0, rs = 0;
      double rt = 0.0, rrec = 0.0;
      FJ_CK(cudaEventRecord(w->ev2, st));
      FJ_TRY(onchip_col(g, s, z, k, c, m, o, t, &it, &rs, &rt, &rrec, &conv, &used, st));
      if (used) {
        FJ_CK(cudaEventRecord(w->ev3, st));
        FJ_CK(cudaEventSynchronize(w->ev3));
        float lms = 0.f;
        cudaEventElapsedTime(&lms, w->ev2, w->ev3);
        r.ms_loop += lms;
        r.iterations = std::max(r.iterations, it);
        r.iterations_total += it;
        r.restarts = std::max(r.restarts, rs);
        r.rel_res_recursive = std::max(r.rel_res_recursive, rrec);
        r.rel_res_true = std::isnan(r.rel_res_true) ? rt : std::max(r.rel_res_true, rt);
        memset(&qout[c], 0, sizeof(fj_quantities_t));
        fill_quantities(g, t, m, qout[c]);
        if (!conv) worst = FJ_E_NO_CONVERGENCE;
        continue;
      }
    }
    int true_restarts = 0;
    for (int round = 0;; ++round) {
      fj_solve_opts ob = oc;
      ob.max_iter = std::max(0, o.max_iter - spent);
      phase_tick("approxim: before solve", st);
      fj_status sc;
      const bool deferred = !is_dist(g);
      if (is_dist(g)) {   // row a8: this rank's slice, halo exchange + allreduce inside
        const int before = r.iterations;
        r.iterations = 0;
        sc = dist_solve_cg(g, 1, s, z, k, c, ob, warm, &r, st);
        iters = r.iterations;
        r.iterations = std::max(before, iters);
      } else {   // Alg. 1 line 3; the true residual comes from the quantities pass below
        sc = solve_col(g, s, z, k, c, ob, warm, &r, st, &iters, true);
      }
      spent += iters;
      if (sc != FJ_OK && sc != FJ_E_NO_CONVERGENCE) return sc;
      phase_tick("approxim: solve", st);
      FJ_TRY(quant_pass(g, w, s, z, k, c, m, t, st));                   // Alg. 1 lines 5-9
      phase_tick("approxim: quantities", st);
      memset(&qout[c], 0, sizeof(fj_quantities_t));
      fill_quantities(g, t, m, qout[c]);
      if (deferred) {   // t[6] = ||s - (I+L) z||^2 of the fused pass decides convergence / restart
        const double rel = t[9] > 0 ? std::sqrt(t[6] / t[9]) : 0.0;
        const bool ok = t[6] <= ob.rtol * ob.rtol * t[9];
        if (!ok && true_restarts < o.max_restarts && spent < o.max_iter) {
          ++true_restarts;
          r.restarts = std::max(r.restarts, true_restarts);
          warm = 1;   // restart from z
          continue;
        }
        r.rel_res_true = std::isnan(r.rel_res_true) ? rel : std::max(r.rel_res_true, rel);
        if (!ok) sc = FJ_E_NO_CONVERGENCE;
      }
      if (sc != FJ_OK) { worst = sc; break; }
      double emax = 0.0;
      for (int j = 0; j < 6; ++j) emax = std::max(emax, qout[c].eps[j]);
      if (o.eps_target <= 0.0 || emax <= o.eps_target || oc.rtol <= 1e-15 || spent >= o.max_iter) break;
      oc.rtol = std::max(oc.rtol * 1e-2, 1e-15);   // tighten and continue from z (warm start)
      warm = 1;
    }
    r.iterations = std::max(r.iterations, spent);
  }
  }
  FJ_CK(cudaEventRecord(w->ev1, st));
  FJ_CK(cudaEventSynchronize(w->ev1));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, w->ev0, w->ev1);
  r.ms = ms;
  if (worst != FJ_OK) r.converged = 0;
  if (rep) *rep = r;
  if (d2h_issued) {
    FJ_CK(cudaStreamSynchronize(side.s));
    if (z_host_done) *z_host_done = true;
  }
  if (worst != FJ_OK) return fail(worst, "PCG did not reach rtol on the true residual");
  return FJ_OK;
}

extern "C" {

fj_status fj_approxim(const fj_graph* gc, int k, const double* s, double* z_user, const fj_solve_opts* opts,
                      fj_quantities_t* qout, fj_solve_report* rep, void* stream) {
  FJ_RANGE("fj_approxim");
  return approxim_impl(gc, k, s, z_user, opts, qout, rep, stream, nullptr, nullptr);
}

// FJ_ORDER_AUTO: relabelling packs several hot x_j into one 32-byte L2 sector, so
// it pays only for rows narrower than a sector (k = 1: 8 bytes, k = 2: 16) whose gathered vector
// does not fit the L2 anyway.
static bool relabel_pays(int64_t n, int k) {
  if (k > 2) return false;
  int dev = 0, l2 = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
  return (double)n * 8.0 * k > (double)(l2 > 0 ? l2 : (126 << 20));
}

fj_status fj_approxim_host(int64_t n, int64_t m_in, const int32_t* u_h, const int32_t* v_h, const void* w_h,
                           int wtype, int k, const double* s_h, double* z_h, const fj_solve_opts* opts,
                           fj_quantities_t* q_h, fj_solve_report* rep, void* stream) {
  FJ_RANGE("fj_approxim_host");
  if (n < 1 || m_in < 0 || !s_h || !q_h || (m_in > 0 && (!u_h || !v_h))) return fail(FJ_E_INVALID_ARG, "null argument");
  if (k < 1 || k > MAXK) return fail(FJ_E_INVALID_ARG, "k must be in [1, 64]");
  if (wtype < FJ_W_UNIT || wtype > FJ_W_F64) return fail(FJ_E_INVALID_ARG, "bad wtype");
  const int wbytes = wtype == FJ_W_UNIT ? 0 : wtype == FJ_W_U8 ? 1 : wtype == FJ_W_F32 ? 4 : 8;
  if (wbytes && m_in > 0 && !w_h) return fail(FJ_E_INVALID_ARG, "weights are NULL");
  cudaStream_t st = S(stream);
  DevBuf<int32_t> du, dv, dcol;
  DevBuf<uint8_t> dw, dwo;
  DevBuf<int64_t> drp;
  DevBuf<double> ds, dz, ds2;
  DevBuf<int32_t> n2o, o2n;
  if (opts && (opts->vertex_order < FJ_ORDER_NATURAL || opts->vertex_order > FJ_ORDER_AUTO))
    return fail(FJ_E_INVALID_ARG, "bad vertex_order");
  bool relabel = opts && opts->vertex_order == FJ_ORDER_DEGREE;
  if (opts && opts->vertex_order == FJ_ORDER_AUTO) relabel = relabel_pays(n, k);
  FJ_TRY(du.alloc(m_in, st)); FJ_TRY(dv.alloc(m_in, st));
  if (relabel) { FJ_TRY(n2o.alloc(n, st)); FJ_TRY(o2n.alloc(n, st)); FJ_TRY(ds2.alloc(n * (int64_t)k, st)); }
  FJ_TRY(ds.alloc(n * (int64_t)k, st)); FJ_TRY(dz.alloc(n * (int64_t)k, st));
  FJ_TRY(drp.alloc(n + 1, st)); FJ_TRY(dcol.alloc(2 * m_in, st));
  if (wbytes) { FJ_TRY(dw.alloc(m_in * wbytes, st)); FJ_TRY(dwo.alloc(2 * m_in * wbytes, st)); }
  if (m_in > 0) {
    FJ_CK(cudaMemcpyAsync(du.p, u_h, sizeof(int32_t) * m_in, cudaMemcpyHostToDevice, st));
    FJ_CK(cudaMemcpyAsync(dv.p, v_h, sizeof(int32_t) * m_in, cudaMemcpyHostToDevice, st));
    if (wbytes) FJ_CK(cudaMemcpyAsync(dw.p, w_h, (size_t)wbytes * m_in, cudaMemcpyHostToDevice, st));
  }
  // the opinions are not needed before the solve: their H2D runs on a side stream after the edge
  // copies, overlapping the CSR build and the graph setup (a1, a2) on `st`
  SideStream side;
  FJ_TRY(side.init());
  FJ_CK(cudaEventRecord(side.ev_in, st));
  FJ_CK(cudaStreamWaitEvent(side.s, side.ev_in, 0));
  FJ_CK(cudaMemcpyAsync(ds.p, s_h, sizeof(double) * n * k, cudaMemcpyHostToDevice, side.s));
  FJ_CK(cudaEventRecord(side.ev_out, side.s));
  int64_t nnz = 0;
  FJ_TRY(fj_csr_from_edges(n, m_in, du.p, dv.p, wbytes ? dw.p : nullptr, wtype, drp.p, dcol.p,
                           wbytes ? dwo.p : nullptr, &nnz, nullptr, nullptr, stream));
  du.release(); dv.release(); dw.release();
  DevBuf<int64_t> drp2;
  DevBuf<int32_t> dcol2;
  DevBuf<uint8_t> dwo2;
  const int64_t* rp_g = drp.p;
  const int32_t* col_g = dcol.p;
  const void* w_g = wbytes ? dwo.p : nullptr;
  if (relabel) {   // relabel the built CSR by descending degree (P A P^T)
    FJ_TRY(drp2.alloc(n + 1, st)); FJ_TRY(dcol2.alloc(nnz, st));
    if (wbytes) FJ_TRY(dwo2.alloc(nnz * wbytes, st));
    FJ_TRY(fj_csr_degree_order(n, drp.p, n2o.p, o2n.p, stream));
    FJ_TRY(fj_csr_permute(n, nnz, drp.p, dcol.p, w_g, wtype, n2o.p, o2n.p, drp2.p, dcol2.p,
                          wbytes ? dwo2.p : nullptr, stream));
    drp.release(); dcol.release(); dwo.release();
    rp_g = drp2.p; col_g = dcol2.p; w_g = wbytes ? dwo2.p : nullptr;
  }
  fj_graph* g = nullptr;
  FJ_TRY(fj_graph_create(n, nnz, rp_g, col_g, w_g, wtype, 0, stream, &g));
  struct GraphGuard {   // the handle (workspace, schedules) is released on every return path
    fj_graph* g;
    ~GraphGuard() { if (g) fj_graph_destroy(g); }
  } guard{g};
  FJ_CK(cudaStreamWaitEvent(st, side.ev_out, 0));
  const double* s_in = ds.p;
  if (relabel) {   // s into the new labels; ds then serves as the old-label staging buffer of z
    FJ_TRY(fj_permute_rows(n, k, n2o.p, ds.p, ds2.p, stream));
    s_in = ds2.p;
  }
  bool z_done = false;
  fj_status s = approxim_impl(g, k, s_in, dz.p, opts, q_h, rep, stream, z_h, &z_done, relabel ? o2n.p : nullptr,
                              relabel ? ds.p : nullptr);
  if ((s == FJ_OK || s == FJ_E_NO_CONVERGENCE) && z_h && !z_done) {
    const double* zsrc = dz.p;
    if (relabel) {
      FJ_TRY(fj_permute_rows(n, k, o2n.p, dz.p, ds.p, stream));
      zsrc = ds.p;
    }
    cudaError_t e = cudaMemcpyAsync(z_h, zsrc, sizeof(double) * n * k, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) s = cuda_fail(e, "z readback", __FILE__, __LINE__);
  }
  return s;
}

}  // extern "C"

// ---------------------------------------------------------------- Algorithm 1 verbatim
// Approxim(G, s, eps) with BOTH solves: z~ = Solve(I+L, s, delta) (line 3) and
// q = Solve(I+L, s_bar, delta) (line 4), run together as one k = 2 batch [s, s_bar]; then
// C_I = ||L z~||^2 (line 5), D = ||W^{1/2} B q||^2 (line 6), P = ||q||^2 (line 7), C = ||z~||^2 (line 8),
// I_dc = D + C (line 9).  delta per line 1, clamped as SPEC's solver decision, mapped to a
// relative-residual stop by the Gershgorin form of SPEC's map (R14).
namespace fj {

constexpr int ATPB = 256;

// S2[i] = (s_i, s_i - m); part[b] = this block's sum of (s_i - m)^2 (host sums the blocks in order)
__global__ void __launch_bounds__(ATPB) k_alg1_rhs(int64_t n, const double* __restrict__ s, double m,
                                                   double* __restrict__ S2, double* __restrict__ part) {
  __shared__ double s_red[ATPB / 32];
  double acc = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)ATPB + threadIdx.x; i < n; i += (int64_t)gridDim.x * ATPB) {
    const double si = s[i], b = si - m;
    S2[2 * i] = si;
    S2[2 * i + 1] = b;
    acc = fma(b, b, acc);
  }
  double v[1] = {acc};
  block_sum<1, ATPB>(v, s_red);
  if (threadIdx.x == 0) part[blockIdx.x] = v[0];
}

}  // namespace fj

extern "C" {

fj_status fj_alg1_delta(int64_t n, double w_min, double w_max, double d_max, double sbar_norm, double eps,
                        double* delta, double* delta_eff, double* rtol, int* clamped, int* floored) {
  if (n < 1 || !(w_min >= 0.0) || !(w_max >= w_min) || !(d_max >= 0.0) || !(sbar_norm >= 0.0) || !(eps > 0.0) ||
      !(eps < 0.5) || !delta || !delta_eff || !rtol || !clamped || !floored)
    return fail(FJ_E_INVALID_ARG, "fj_alg1_delta: n >= 1, 0 <= w_min <= w_max, d_max >= 0, eps in (0, 1/2)");
  const double nn = (double)n;
  // line 1: delta = eps w_min ||s_bar|| / (3 w_max n^3 (n w_max + 1) sqrt(n))   (w_max = 0: no edges)
  const double den = 3.0 * (w_max > 0.0 ? w_max : 1.0) * nn * nn * nn * (nn * w_max + 1.0) * std::sqrt(nn);
  *delta = eps * (w_max > 0.0 ? w_min : 1.0) * sbar_norm / den;
  // the theoretical delta is used verbatim when >= 1e-14, else clamped to 1e-12 (recorded)
  *clamped = *delta >= 1e-14 ? 0 : 1;
  *delta_eff = *clamped ? 1e-12 : *delta;
  // Residual stop that implies the Lemma 4.2 T-norm contract: lambda(I+L) in [1, 1 + 2 d_max]
  // (Gershgorin), so ||y - y*||_T / ||y*||_T <= sqrt(1 + 2 d_max) ||r|| / ||x||.
  *rtol = *delta_eff / std::sqrt(1.0 + 2.0 * d_max);
  // fp64 floor of an attainable relative residual; recorded when it binds
  *floored = *rtol < 1e-14 ? 1 : 0;
  if (*floored) *rtol = 1e-14;
  return FJ_OK;
}

fj_status fj_approxim_alg1(const fj_graph* gc, const double* s, double eps, const fj_solve_opts* opts,
                           fj_alg1_t* out, fj_solve_report* rep, void* stream) {
  FJ_RANGE("fj_approxim_alg1");
  if (!gc || !s || !out) return fail(FJ_E_INVALID_ARG, "null argument");
  fj_graph* g = const_cast<fj_graph*>(gc);
  if (is_dist(g)) return fail(FJ_E_UNSUPPORTED, "fj_approxim_alg1 on a distributed graph");
  if (!(eps > 0.0) || !(eps < 0.5)) return fail(FJ_E_INVALID_ARG, "eps must lie in (0, 1/2) (Algorithm 1 input)");
  cudaStream_t st = S(stream);
  SolveWs* w = nullptr;
  FJ_TRY(get_ws(g, st, &w));
  std::vector<double> v;
  FJ_TRY(stats_cols(g, w, 1, s, v, st));   // line 2: 1^T s / n
  const int64_t n = g->n;
  const double m = v[0] / (double)n;
  DevBuf<double> S2, Z2, part;
  FJ_TRY(S2.alloc(2 * n, st));
  FJ_TRY(Z2.alloc(2 * n, st));
  const int grid = (int)std::min<int64_t>((n + ATPB - 1) / ATPB, (int64_t)g->num_sms * 8);
  FJ_TRY(part.alloc(grid, st));
  k_alg1_rhs<<<grid, ATPB, 0, st>>>(n, s, m, S2.p, part.p);   // line 2: s_bar = s - (1^T s / n) 1
  FJ_CK_LAUNCH();
  std::vector<double> hp(grid);
  FJ_CK(cudaMemcpyAsync(hp.data(), part.p, sizeof(double) * grid, cudaMemcpyDeviceToHost, st));
  FJ_CK(cudaStreamSynchronize(st));
  double sb2 = 0.0;
  for (int b = 0; b < grid; ++b) sb2 += hp[b];   // block order: deterministic
  fj_alg1_t r;
  memset(&r, 0, sizeof r);
  const fj_graph_info_t& I = g->info;
  FJ_TRY(fj_alg1_delta(n, I.w_min, I.w_max, I.d_max, std::sqrt(sb2), eps, &r.delta, &r.delta_eff, &r.rtol,
                       &r.clamped, &r.rtol_floored));   // line 1
  fj_solve_opts o;
  fj_default_solve_opts(&o);
  if (opts) o = *opts;
  o.rtol = r.rtol;
  fj_solve_report sr{};
  sr.converged = 1;
  sr.rel_res_true = NAN;
  const fj_status ss = solve_batch(g, 2, S2.p, Z2.p, o, 0, &sr, st);   // lines 3-4, one k = 2 batch
  if (ss != FJ_OK && ss != FJ_E_NO_CONVERGENCE) return ss;
  const double means[2] = {m, 0.0};
  double sums[20];
  FJ_TRY(quant_batch(g, 2, S2.p, Z2.p, means, sums, st, true));
  // QuantOp sums per column: [0] (z-s)^2 [1] sum_i sum_j w (z_i - z_j)^2 [3] z^2 [7] ||L z||^2 ...
  r.CI = sums[7];               // line 5: ||L z~||^2
  r.D = 0.5 * sums[10 + 1];     // line 6: ||W^{1/2} B q||^2 (each edge once)
  r.P = sums[10 + 3];           // line 7: ||q||^2
  r.C = sums[3];                // line 8: ||z~||^2
  r.Idc = r.D + r.C;            // line 9
  r.PDI = r.P + r.D;
  r.D_from_z = 0.5 * sums[1];   // SPEC note: D from the s-solve agrees at solver tolerance
  r.CI_def = sums[0];           // Def. 3.1 form sum (z~ - s)^2
  r.mean_s = m;
  r.sbar_norm = std::sqrt(sb2);
  *out = r;
  if (rep) *rep = sr;
  if (ss != FJ_OK) return fail(ss, "PCG did not reach the Algorithm 1 tolerance on the true residual");
  return FJ_OK;
}

}  // extern "C"

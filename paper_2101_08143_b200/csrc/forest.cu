// forest.cu — SURVEY §8 row f4: entries of the forest matrix Omega = (I + L)^{-1} (P:L101-103,
// omega_ij = eps(Gamma_ij) / eps(Gamma), the fraction of spanning rooted forests in which
// i and j share a root; "proximity" between i and j).  Column j of Omega solves (I+L) x = e_j, and
// Omega is symmetric, so m requested columns are m right-hand sides e_{c_t} solved together by the
// batched PCG (row a9: 2-4 columns per vector-engine batch, 5-64 per warp-per-row batch).
#include <algorithm>
#include <vector>

#include "common.cuh"
#include "workspace.cuh"

namespace fj {

// E[i][t] = (i == cols[t]) for the kk columns of this batch; E row-major [n][kk]
__global__ void k_unit_columns(int64_t n, int kk, const int32_t* __restrict__ cols, double* __restrict__ E) {
  const int64_t total = n * (int64_t)kk;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = q / kk;
    const int t = (int)(q - i * kk);
    E[q] = (i == cols[t]) ? 1.0 : 0.0;
  }
}

// out[:, t0 : t0+kk] (row-major [n][m]) = X[n][kk]
__global__ void k_scatter_columns(int64_t n, int kk, int64_t m, int64_t t0, const double* __restrict__ X,
                                  double* __restrict__ out) {
  const int64_t total = n * (int64_t)kk;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = q / kk;
    const int64_t t = q - i * kk;
    out[i * m + t0 + t] = X[q];
  }
}

}  // namespace fj

using namespace fj;

extern "C" fj_status fj_forest_columns(const fj_graph* gc, int64_t m, const int32_t* cols_host, double* omega_dev,
                                       const fj_solve_opts* opts, fj_solve_report* rep, void* stream) {
  FJ_RANGE("fj_forest_columns");
  if (!gc || !cols_host || !omega_dev || m < 1) return fail(FJ_E_INVALID_ARG, "null argument or m < 1");
  fj_graph* g = const_cast<fj_graph*>(gc);
  if (g->dist) return fail(FJ_E_UNSUPPORTED, "fj_forest_columns on a distributed graph");
  for (int64_t t = 0; t < m; ++t)
    if (cols_host[t] < 0 || cols_host[t] >= g->n) return fail(FJ_E_INVALID_ARG, "column index out of range");
  cudaStream_t st = S(stream);
  const int64_t n = g->n;
  const int kb = (int)std::min<int64_t>(m, MAXK);   // columns per batch
  DevBuf<double> E, X;
  DevBuf<int32_t> dcols;
  FJ_TRY(E.alloc(n * kb, st));
  FJ_TRY(X.alloc(n * kb, st));
  FJ_TRY(dcols.alloc(kb, st));
  const unsigned cb = (unsigned)std::min<int64_t>((n * kb + 255) / 256, (int64_t)g->num_sms * 16);
  fj_solve_report total{};
  total.converged = 1;
  total.rel_res_true = 0.0;
  fj_status worst = FJ_OK;
  for (int64_t t0 = 0; t0 < m; t0 += kb) {
    const int kk = (int)std::min<int64_t>(kb, m - t0);
    FJ_CK(cudaMemcpyAsync(dcols.p, cols_host + t0, sizeof(int32_t) * kk, cudaMemcpyHostToDevice, st));
    k_unit_columns<<<cb, 256, 0, st>>>(n, kk, dcols.p, E.p);
    FJ_CK_LAUNCH();
    fj_solve_report r{};
    const fj_status s = fj_solve(gc, kk, E.p, X.p, opts, &r, stream);   // Omega[:, c] = (I+L)^{-1} e_c
    if (s != FJ_OK && s != FJ_E_NO_CONVERGENCE) return s;
    if (s != FJ_OK) worst = s;
    k_scatter_columns<<<cb, 256, 0, st>>>(n, kk, m, t0, X.p, omega_dev);
    FJ_CK_LAUNCH();
    total.iterations = std::max(total.iterations, r.iterations);
    total.iterations_total += r.iterations_total;
    total.restarts = std::max(total.restarts, r.restarts);
    total.batch_k = std::max(total.batch_k, r.batch_k);
    total.rel_res_true = std::max(total.rel_res_true, r.rel_res_true);
    total.rel_res_recursive = std::max(total.rel_res_recursive, r.rel_res_recursive);
    total.ms += r.ms;
    total.ms_loop += r.ms_loop;
    if (!r.converged) total.converged = 0;
  }
  FJ_CK(cudaStreamSynchronize(st));
  if (rep) *rep = total;
  return worst == FJ_OK ? FJ_OK : fail(worst, "PCG did not reach rtol on the true residual");
}

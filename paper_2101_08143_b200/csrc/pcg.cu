// pcg.cu — operators (fj_apply) and the Jacobi-preconditioned CG solve of (I+L) z = s
// (row a4; Eq. (2); SOLVE contract Lemma 4.2).
//
// One PCG iteration is three stream-ordered kernels:
//   K_A tile_kernel<ApplyOp>  q = (I+L) p, pq = p^T q   -> alpha = rho / pq      (last block)
//   K_B k_pcg_update          x += alpha p, r -= alpha q, y = dinv o r,
//                             rho' = r^T y, rr = r^T r  -> beta, convergence     (last block)
//   K_C k_pcg_dir             p = y + beta p
// The loop runs inside a CUDA graph with a device-driven conditional WHILE node: K_B's last
// block clears the condition when ||r||^2 <= rtol^2 ||s||^2 or the iteration cap is hit, so a
// whole solve is one graph launch with no host round trip.  All scalars live on the device.
#include <cstring>

#include "ops.cuh"
#include "rows.cuh"
#include "workspace.cuh"

namespace fj {

constexpr int ETPB = 256;

template <int WT, class Op>
inline fj_status launch_tiles_wt(const fj_graph* g, const SolveWs* ws, const Op& op, cudaStream_t st) {
  if (ws->rows && ws->rows->mode != 0) return rows_op<WT>(*ws->rows, g->n, g->col, g->w, op, st);   // rows.cuh
  FJ_CK(launch_warp_items<WT>(g, ws, op, st));
  FJ_CK_LAUNCH();
  return FJ_OK;
}

void free_solve_ws(fj_graph* g) {
  SolveWs* w = g->solve_ws;
  if (!w) return;
  if (w->exec) cudaGraphExecDestroy(w->exec);
  if (w->graph) cudaGraphDestroy(w->graph);
  if (w->cap_stream) cudaStreamDestroy(w->cap_stream);
  if (w->ev0) cudaEventDestroy(w->ev0);
  if (w->ev1) cudaEventDestroy(w->ev1);
  if (w->ev2) cudaEventDestroy(w->ev2);
  if (w->ev3) cudaEventDestroy(w->ev3);
  dfree(w->r); dfree(w->p); dfree(w->q); dfree(w->x); dfree(w->col_s);
  dfree(w->sc); dfree(w->elem_part); dfree(w->elem_ticket);
  dfree(w->ts.block_part); dfree(w->ts.long_part); dfree(w->ts.chunk_acc);
  dfree(w->ts.long_ticket); dfree(w->ts.grid_ticket);
  dfree(w->qout); dfree(w->stat);
  if (w->rows) { rows_plan_free(*w->rows); delete w->rows; }
  delete w;
  g->solve_ws = nullptr;
}

template <class T>
static fj_status dalloc(T** p, int64_t count, cudaStream_t st, bool zero = false) {
  if (count < 1) count = 1;
  FJ_CK(dmalloc(p, sizeof(T) * (size_t)count, st));
  if (zero) FJ_CK(cudaMemsetAsync(*p, 0, sizeof(T) * (size_t)count, st));
  return FJ_OK;
}

fj_status get_ws(fj_graph* g, cudaStream_t st, SolveWs** out) {
  if (g->solve_ws) { *out = g->solve_ws; return FJ_OK; }
  SolveWs* w = new SolveWs();
  g->solve_ws = w;
  w->n = g->n;
  w->grid_max = g->num_sms * (2048 / WTPB);   // upper bound of any warp-engine grid
  int64_t ge = (int64_t)g->num_sms * (2048 / ETPB);
  const int64_t need = (g->n + ETPB - 1) / ETPB;
  if (ge > need) ge = need > 0 ? need : 1;
  w->grid_elem = (int)ge;
  const int64_t n = g->n;
  FJ_TRY(dalloc(&w->r, n, st));
  FJ_TRY(dalloc(&w->p, n, st));
  FJ_TRY(dalloc(&w->q, n, st));
  FJ_TRY(dalloc(&w->x, n, st));
  FJ_TRY(dalloc(&w->sc, 1, st, true));
  FJ_TRY(dalloc(&w->elem_part, (int64_t)w->grid_elem * 16, st));   // k_stats_k: 4 x 4 per block
  FJ_TRY(dalloc(&w->elem_ticket, 1, st, true));
  constexpr int NPMAX = 16, NAMAX = 4;
  FJ_TRY(dalloc(&w->ts.block_part, (int64_t)w->grid_max * NPMAX, st));
  FJ_TRY(dalloc(&w->ts.long_part, g->s1.n_long * NPMAX, st));
  FJ_TRY(dalloc(&w->ts.chunk_acc, g->s1.n_long_chunks * NAMAX, st));
  FJ_TRY(dalloc(&w->ts.long_ticket, g->s1.n_long, st, true));
  FJ_TRY(dalloc(&w->ts.grid_ticket, 1, st, true));
  FJ_TRY(dalloc(&w->qout, 16, st));
  FJ_TRY(dalloc(&w->stat, 4 * MAXK, st));
  FJ_CK(cudaEventCreate(&w->ev0));
  FJ_CK(cudaEventCreate(&w->ev1));
  FJ_CK(cudaEventCreate(&w->ev2));
  FJ_CK(cudaEventCreate(&w->ev3));
  w->rows = new RowsPlan();
  FJ_TRY(rows_plan_build(g, 1, *w->rows, st));
  *out = w;
  return FJ_OK;
}

// ---------------------------------------------------------------- elementwise PCG kernels
// Grid-stride with a FIXED grid: each block's elements are fixed, so partial sums are formed in a
// fixed order and combined in block order by the last block (deterministic).
template <int NPART>
__device__ __forceinline__ bool elem_reduce(double (&v)[NPART], double* part, unsigned int* ticket,
                                            double* s_red) {
  block_sum<NPART, ETPB>(v, s_red);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int j = 0; j < NPART; ++j) part[blockIdx.x * 4 + j] = v[j];
  }
  if (!last_block_ticket(ticket, gridDim.x)) return false;
  double t[NPART];
#pragma unroll
  for (int j = 0; j < NPART; ++j) t[j] = 0.0;
  for (int b = threadIdx.x; b < (int)gridDim.x; b += ETPB) {
#pragma unroll
    for (int j = 0; j < NPART; ++j) t[j] += __ldcg(part + b * 4 + j);
  }
  block_sum<NPART, ETPB>(t, s_red);
#pragma unroll
  for (int j = 0; j < NPART; ++j) v[j] = t[j];
  return true;
}

// fresh start (x = 0, r = s) or restart (r = s - q with q = (I+L) x precomputed).
__global__ void __launch_bounds__(ETPB) k_pcg_init(int64_t n, const double* __restrict__ s, int64_t ld, int64_t c,
                                                   const double* __restrict__ dinv, const double* __restrict__ q,
                                                   int restart, double* __restrict__ x, double* __restrict__ r,
                                                   double* __restrict__ p, PcgScalars* sc, double rtol,
                                                   int max_iter, double* part, unsigned int* ticket) {
  __shared__ double s_red[3 * ETPB / 32];
  double v[3] = {0.0, 0.0, 0.0};
  for (int64_t i = blockIdx.x * (int64_t)ETPB + threadIdx.x; i < n; i += (int64_t)gridDim.x * ETPB) {
    const double si = s[i * ld + c];
    double ri = si;
    if (restart) ri = si - q[i];
    else x[i] = 0.0;
    const double yi = dinv[i] * ri;
    r[i] = ri;
    p[i] = yi;
    v[0] = fma(ri, yi, v[0]);
    v[1] = fma(ri, ri, v[1]);
    v[2] = fma(si, si, v[2]);
  }
  if (elem_reduce<3>(v, part, ticket, s_red) && threadIdx.x == 0) {
    sc->rho = v[0];
    sc->rr = v[1];
    sc->ss = v[2];
    sc->tol2 = rtol * rtol * v[2];
    sc->iter = 0;   // per (re)start; the host accumulates the total
    sc->max_iter = max_iter;
    sc->converged = (v[1] <= sc->tol2) ? 1 : 0;
    sc->done = (sc->converged || sc->iter >= max_iter) ? 1 : 0;
    sc->breakdown = 0;
    sc->alpha = sc->beta = 0.0;
    *ticket = 0u;
  }
}

__global__ void __launch_bounds__(ETPB) k_pcg_update(int64_t n, const double* __restrict__ dinv,
                                                     const double* __restrict__ p, const double* __restrict__ q,
                                                     double* __restrict__ x, double* __restrict__ r,
                                                     PcgScalars* sc, double* part, unsigned int* ticket,
                                                     cudaGraphConditionalHandle h, int use_h) {
  __shared__ double s_red[2 * ETPB / 32];
  if (*(volatile int32_t*)&sc->done) {
    if (use_h && blockIdx.x == 0 && threadIdx.x == 0) cudaGraphSetConditional(h, 0);
    return;
  }
  const double alpha = sc->alpha;
  double v[2] = {0.0, 0.0};
  for (int64_t i = blockIdx.x * (int64_t)ETPB + threadIdx.x; i < n; i += (int64_t)gridDim.x * ETPB) {
    x[i] = fma(alpha, p[i], x[i]);
    const double ri = fma(-alpha, q[i], r[i]);
    r[i] = ri;
    v[0] = fma(ri, dinv[i] * ri, v[0]);
    v[1] = fma(ri, ri, v[1]);
  }
  if (elem_reduce<2>(v, part, ticket, s_red) && threadIdx.x == 0) {
    const int it = sc->iter + 1;
    sc->iter = it;
    sc->beta = v[0] / sc->rho;
    sc->rho = v[0];
    sc->rr = v[1];
    const bool conv = v[1] <= sc->tol2;
    sc->converged = conv ? 1 : 0;
    if (conv || it >= sc->max_iter || !isfinite(v[1])) {
      sc->done = 1;
      if (use_h) cudaGraphSetConditional(h, 0);
    }
    *ticket = 0u;
  }
}

__global__ void __launch_bounds__(ETPB) k_pcg_dir(int64_t n, const double* __restrict__ dinv,
                                                  const double* __restrict__ r, double* __restrict__ p,
                                                  const PcgScalars* sc) {
  if (*(volatile const int32_t*)&sc->done) return;
  const double beta = sc->beta;
  for (int64_t i = blockIdx.x * (int64_t)ETPB + threadIdx.x; i < n; i += (int64_t)gridDim.x * ETPB)
    p[i] = fma(beta, p[i], dinv[i] * r[i]);
}

__global__ void k_copy_col(int64_t n, const double* __restrict__ src, int64_t sld, int64_t sc_,
                           double* __restrict__ dst, int64_t dld, int64_t dc) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i * dld + dc] = src[i * sld + sc_];
}

// q = (I+L) x for contiguous x, y
template <int WT>
static fj_status launch_product1(const fj_graph* g, const SolveWs* w, const double* x, double* y, int opL,
                                 PcgScalars* sc, cudaStream_t st) {
  if (w->rows && w->rows->mode != 0)   // lean row kernel (rows.cuh)
    return rows_product<WT, 1, 1>(g, *w->rows, x, y, opL, 1, nullptr, sc, st);
  ApplyOp<WT> op{x, y, g->deg, 1, 0, opL, sc, nullptr};
  int nl = 0;
  FJ_CK(launch_product<WT>(g, w->ts, w->grid_max, op, st, &nl));
  if (!g_capturing) count_launch(nl);
  return FJ_OK;
}

template <int WT>
static fj_status launch_iteration(const fj_graph* g, SolveWs* w, cudaStream_t st, cudaGraphConditionalHandle h, int use_h) {
  FJ_TRY(launch_product1<WT>(g, w, w->p, w->q, 0, w->sc, st));
  k_pcg_update<<<w->grid_elem, ETPB, 0, st>>>(g->n, g->dinv, w->p, w->q, w->x, w->r, w->sc, w->elem_part,
                                               w->elem_ticket, h, use_h);
  FJ_CK_LAUNCH();
  k_pcg_dir<<<w->grid_elem, ETPB, 0, st>>>(g->n, g->dinv, w->r, w->p, w->sc);
  FJ_CK_LAUNCH();
  return FJ_OK;
}

static fj_status launch_iteration_any(const fj_graph* g, SolveWs* w, cudaStream_t st, cudaGraphConditionalHandle h, int use_h) {
  switch (g->wtype) {
    case FJ_W_UNIT: return launch_iteration<FJ_W_UNIT>(g, w, st, h, use_h);
    case FJ_W_U8: return launch_iteration<FJ_W_U8>(g, w, st, h, use_h);
    case FJ_W_F32: return launch_iteration<FJ_W_F32>(g, w, st, h, use_h);
    default: return launch_iteration<FJ_W_F64>(g, w, st, h, use_h);
  }
}

static fj_status build_loop_graph(fj_graph* g, SolveWs* w) {
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
  fj_status s = launch_iteration_any(g, w, w->cap_stream, h, 1);
  g_capturing = false;
  cudaGraph_t captured = nullptr;
  cudaError_t e = cudaStreamEndCapture(w->cap_stream, &captured);
  FJ_TRY(s);
  FJ_CK(e);
  FJ_CK(cudaGraphInstantiate(&w->exec, w->graph, 0));
  return FJ_OK;
}

template <int WT>
static fj_status launch_apply(const fj_graph* g, const SolveWs* w, const double* x, double* y, int64_t ld,
                              int64_t c, int opL, cudaStream_t st) {
  if (ld == 1) return launch_product1<WT>(g, w, x, y, opL, nullptr, st);
  ApplyOp<WT> op{x, y, g->deg, ld, c, opL, nullptr, nullptr};
  return launch_tiles_wt<WT>(g, w, op, st);
}

fj_status apply_col(const fj_graph* g, const SolveWs* w, const double* x, double* y, int64_t ld, int64_t c,
                    int opL, cudaStream_t st) {
  switch (g->wtype) {
    case FJ_W_UNIT: return launch_apply<FJ_W_UNIT>(g, w, x, y, ld, c, opL, st);
    case FJ_W_U8: return launch_apply<FJ_W_U8>(g, w, x, y, ld, c, opL, st);
    case FJ_W_F32: return launch_apply<FJ_W_F32>(g, w, x, y, ld, c, opL, st);
    default: return launch_apply<FJ_W_F64>(g, w, x, y, ld, c, opL, st);
  }
}

template <int WT>
static fj_status launch_resid(const fj_graph* g, const SolveWs* w, const double* z, const double* s, int64_t ld,
                              int64_t c, double* out, cudaStream_t st) {
  ResidOp<WT> op{z, s, g->deg, ld, c, out};
  return launch_tiles_wt<WT>(g, w, op, st);
}

fj_status resid_col(const fj_graph* g, const SolveWs* w, const double* z, const double* s, int64_t ld, int64_t c,
                    double* out, cudaStream_t st) {
  switch (g->wtype) {
    case FJ_W_UNIT: return launch_resid<FJ_W_UNIT>(g, w, z, s, ld, c, out, st);
    case FJ_W_U8: return launch_resid<FJ_W_U8>(g, w, z, s, ld, c, out, st);
    case FJ_W_F32: return launch_resid<FJ_W_F32>(g, w, z, s, ld, c, out, st);
    default: return launch_resid<FJ_W_F64>(g, w, z, s, ld, c, out, st);
  }
}

// Solve one column c of row-major s [n][ld] into column c of z.  If warm != 0, z already holds
// the starting iterate.  Always ends with a recomputed true residual (restarting while it misses
// rtol); *iters_out receives the iterations spent on this column.
fj_status solve_col(fj_graph* g, const double* s, double* z, int64_t ld, int64_t c, const fj_solve_opts& o,
                    int warm, fj_solve_report* rep, cudaStream_t st, int* iters_out, bool defer) {
  SolveWs* w = nullptr;
  FJ_TRY(get_ws(g, st, &w));
  const int64_t n = g->n;
  const unsigned cb = (unsigned)std::min<int64_t>((n + 255) / 256, 4096);
  if (o.use_cuda_graph) FJ_TRY(build_loop_graph(g, w));
  int restarts = 0, total_iter = 0;
  PcgScalars h{};
  bool first = true;
  double rel_true = NAN;
  for (;;) {
    const bool restart = !first || warm;
    if (restart) {
      if (first) {   // warm start: x = z
        k_copy_col<<<cb, 256, 0, st>>>(n, z, ld, c, w->x, 1, 0);
        FJ_CK_LAUNCH();
      }
      FJ_TRY(apply_col(g, w, w->x, w->q, 1, 0, 0, st));
    }
    // iteration budget left for this (re)start
    const int budget = std::max(0, o.max_iter - total_iter);
    FJ_CK(cudaEventRecord(w->ev2, st));
    k_pcg_init<<<w->grid_elem, ETPB, 0, st>>>(n, s, ld, c, g->dinv, w->q, restart ? 1 : 0, w->x, w->r, w->p, w->sc,
                                              o.rtol, budget, w->elem_part, w->elem_ticket);
    FJ_CK_LAUNCH();
    first = false;
    if (o.use_cuda_graph) {
      FJ_CK(cudaGraphLaunch(w->exec, st));
    } else {
      for (;;) {
        for (int u = 0; u < 8; ++u) FJ_TRY(launch_iteration_any(g, w, st, 0, 0));
        FJ_CK(cudaMemcpyAsync(&h, w->sc, sizeof h, cudaMemcpyDeviceToHost, st));
        FJ_CK(cudaStreamSynchronize(st));
        if (h.done) break;
      }
    }
    FJ_CK(cudaEventRecord(w->ev3, st));
    // true residual ||s - (I+L) x||^2 (defer: the caller's fused quantities pass computes it and
    // decides the restart, one CSR pass less per solve)
    if (!defer) FJ_TRY(resid_col(g, w, w->x, s, ld, c, &w->sc->res2, st));
    FJ_CK(cudaMemcpyAsync(&h, w->sc, sizeof h, cudaMemcpyDeviceToHost, st));
    FJ_CK(cudaStreamSynchronize(st));
    if (defer) h.res2 = h.rr;   // recursive residual stands in
    total_iter += h.iter;
    if (o.use_cuda_graph) count_launch((int64_t)(rows_launches(*w->rows) + 2) * std::max(h.iter, 1));
    float lms = 0.f;
    cudaEventElapsedTime(&lms, w->ev2, w->ev3);
    if (rep) { rep->ms_loop += lms; rep->iterations_total += h.iter; }
    rel_true = h.ss > 0 ? sqrt(h.res2 / h.ss) : 0.0;
    const bool ok = h.res2 <= h.tol2;
    if (defer || ok || restarts >= o.max_restarts || total_iter >= o.max_iter || h.breakdown) break;
    ++restarts;
  }
  k_copy_col<<<cb, 256, 0, st>>>(n, w->x, 1, 0, z, ld, c);
  FJ_CK_LAUNCH();
  if (rep) {
    rep->iterations = std::max(rep->iterations, total_iter);
    rep->restarts = std::max(rep->restarts, restarts);
    const double rr = h.ss > 0 ? sqrt(h.rr / h.ss) : 0.0;
    rep->rel_res_recursive = std::max(rep->rel_res_recursive, rr);
    if (!defer) rep->rel_res_true = std::isnan(rep->rel_res_true) ? rel_true : std::max(rep->rel_res_true, rel_true);
  }
  const bool converged = h.res2 <= h.tol2;
  if (rep && !converged && !defer) rep->converged = 0;
  if (iters_out) *iters_out = total_iter;
  return converged ? FJ_OK : fail(FJ_E_NO_CONVERGENCE, "PCG did not reach rtol on the true residual");
}

}  // namespace fj

using namespace fj;

extern "C" {

fj_status fj_apply(const fj_graph* gc, int op, int k, const double* x, double* y, void* stream) {
  FJ_RANGE("fj_apply");
  if (!gc || !x || !y) return fail(FJ_E_INVALID_ARG, "null argument");
  if (k < 1 || k > MAXK) return fail(FJ_E_INVALID_ARG, "k must be in [1, 64]");
  if (op != FJ_OP_L && op != FJ_OP_IPL) return fail(FJ_E_INVALID_ARG, "bad op");
  if (x == y) return fail(FJ_E_INVALID_ARG, "x and y must not alias");
  fj_graph* g = const_cast<fj_graph*>(gc);
  cudaStream_t st = S(stream);
  if (is_dist(g)) return fail(FJ_E_UNSUPPORTED, "fj_apply on a distributed graph (use fj_solve / fj_quantities)");
  if (k > 1) return apply_batch(g, k, x, y, op == FJ_OP_L ? 1 : 0, st);
  SolveWs* w = nullptr;
  FJ_TRY(get_ws(g, st, &w));
  return apply_col(g, w, x, y, 1, 0, op == FJ_OP_L ? 1 : 0, st);
}

fj_status fj_time_spmv(const fj_graph* gc, int k, int reps, float* ms_host, void* stream) {
  if (!gc || !ms_host) return fail(FJ_E_INVALID_ARG, "null argument");
  if (k < 1 || k > MAXK || reps < 1) return fail(FJ_E_INVALID_ARG, "k must be in [1, 64], reps >= 1");
  fj_graph* g = const_cast<fj_graph*>(gc);
  cudaStream_t st = S(stream);
  if (is_dist(g)) return fail(FJ_E_UNSUPPORTED, "fj_time_spmv on a distributed graph");
  if (k >= batch_min_k()) return time_batch_spmv(g, k, reps, ms_host, st);
  SolveWs* w = nullptr;
  FJ_TRY(get_ws(g, st, &w));
  FJ_TRY(apply_col(g, w, w->p, w->q, 1, 0, 0, st));
  FJ_CK(cudaEventRecord(w->ev2, st));
  for (int i = 0; i < reps; ++i) FJ_TRY(apply_col(g, w, w->p, w->q, 1, 0, 0, st));
  FJ_CK(cudaEventRecord(w->ev3, st));
  FJ_CK(cudaEventSynchronize(w->ev3));
  float ms = 0.f;
  FJ_CK(cudaEventElapsedTime(&ms, w->ev2, w->ev3));
  *ms_host = ms / (float)reps;
  return FJ_OK;
}

fj_status fj_product_path(const fj_graph* gc, int k, int* path, void* stream) {
  if (!gc || !path) return fail(FJ_E_INVALID_ARG, "null argument");
  if (k < 1 || k > MAXK) return fail(FJ_E_INVALID_ARG, "k must be in [1, 64]");
  fj_graph* g = const_cast<fj_graph*>(gc);
  if (is_dist(g)) return fail(FJ_E_UNSUPPORTED, "fj_product_path on a distributed graph");
  if (k < batch_min_k()) {
    SolveWs* w = nullptr;
    FJ_TRY(get_ws(g, S(stream), &w));
    const int m = w->rows ? w->rows->mode : 0;
    *path = m == 0 ? FJ_PATH_ENGINE : (m == 2 ? FJ_PATH_ROWS_SLABS : FJ_PATH_ROWS);
    return FJ_OK;
  }
  if (!vec_supported(k)) { *path = FJ_PATH_BATCH; return FJ_OK; }
  int mode = 0;
  FJ_TRY(vec_product_mode(g, k, S(stream), &mode));
  *path = mode == 0 ? FJ_PATH_ENGINE : (mode == 2 ? FJ_PATH_ROWS_SLABS : FJ_PATH_ROWS);
  return FJ_OK;
}

fj_status fj_solve(const fj_graph* gc, int k, const double* s, double* z, const fj_solve_opts* opts,
                   fj_solve_report* rep, void* stream) {
  FJ_RANGE("fj_solve");
  if (!gc || !s || !z) return fail(FJ_E_INVALID_ARG, "null argument");
  if (k < 1 || k > MAXK) return fail(FJ_E_INVALID_ARG, "k must be in [1, 64]");
  if (s == z) return fail(FJ_E_INVALID_ARG, "s and z must not alias");
  fj_solve_opts o;
  fj_default_solve_opts(&o);
  if (opts) o = *opts;
  if (!(o.rtol > 0.0) || o.max_iter < 0 || o.max_restarts < 0) return fail(FJ_E_INVALID_ARG, "bad solve options");
  fj_graph* g = const_cast<fj_graph*>(gc);
  cudaStream_t st = S(stream);
  SolveWs* w = nullptr;
  FJ_TRY(get_ws(g, st, &w));
  fj_solve_report r{};
  r.converged = 1;
  r.rel_res_true = NAN;
  FJ_CK(cudaEventRecord(w->ev0, st));
  fj_status worst = FJ_OK;
  if (is_dist(g)) {   // rows a8 (+ a9): this rank's slice, columns in groups of <= 4 solved together
    for (int c = 0; c < k; c += 4) {
      fj_status sc = dist_solve_cg(g, std::min(4, k - c), s, z, k, c, o, 0, &r, st);
      if (sc != FJ_OK && sc != FJ_E_NO_CONVERGENCE) return sc;
      if (sc != FJ_OK) worst = sc;
    }
  } else if (k >= batch_min_k()) {   // row a9: all columns together
    fj_status sc = solve_batch(g, k, s, z, o, 0, &r, st);
    if (sc != FJ_OK && sc != FJ_E_NO_CONVERGENCE) return sc;
    worst = sc;
  } else {
    for (int c = 0; c < k; ++c) {
      fj_status sc = solve_col(g, s, z, k, c, o, 0, &r, st, nullptr, false);
      if (sc != FJ_OK && sc != FJ_E_NO_CONVERGENCE) return sc;
      if (sc != FJ_OK) worst = sc;
    }
  }
  FJ_CK(cudaEventRecord(w->ev1, st));
  FJ_CK(cudaEventSynchronize(w->ev1));
  float ms = 0.f;
  cudaEventElapsedTime(&ms, w->ev0, w->ev1);
  r.ms = ms;
  if (rep) *rep = r;
  if (worst != FJ_OK) return fail(worst, "PCG did not reach rtol on the true residual");
  return FJ_OK;
}

}  // extern "C"

// dist.cu — rows a8/e: the graph row-partitioned over ranks (one process per GPU), NCCL halo
// exchange of the PCG search direction and allreduce of the dot products over NVLink.
//
//  Partition  fj_partition_rows: contiguous row blocks balanced by (raw) nonzeros.
//  Local CSR  fj_csr_rows_from_edges: row a1 restricted to the rank's rows (global column ids).
//  Ghosts     fj_dist_ghosts: sorted unique off-rank columns = the halo, grouped by owner rank.
//  Graph      fj_graph_create_dist: columns renumbered (own -> [0, n_loc), ghost -> n_loc + idx);
//             degrees / schedule on the local rows (full rows, so d_i is exact); halo plan.
//  Iteration  pack p[send_idx] -> grouped ncclSend/ncclRecv into p[n_loc..] -> row engine
//             q = (I+L)p on local rows -> allreduce(p^T q) -> update (x, r, rho', ||r||^2)
//             -> allreduce(rho', ||r||^2) -> beta / convergence (identical on all ranks) -> p.
//  Transports NCCL (real ranks) or LOOPBACK (virtual ranks = host threads of one process on one
//             device; collectives become barrier-ordered device copies / host-ordered sums), so
//             the distributed algorithm is tested on one GPU without kernels waiting on kernels.
#include <dlfcn.h>

#include <condition_variable>
#include <cstring>
#include <mutex>
#include <vector>

#include <cub/cub.cuh>

#include "ops.cuh"
#include "workspace.cuh"

// NCCL types only (the library dlopens libnccl.so.2 at fj_comm_init, the copy torch also loads)
#include "nccl.h"

namespace fj {

// ---------------------------------------------------------------- NCCL, loaded lazily
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*ErrStr)(ncclResult_t) = nullptr;
};

static fj_status nccl_api(NcclApi** out) {
  static NcclApi api;
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  if (!api.h) {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      const char* p = getenv("FJ_NCCL_LIB");
      if (p) h = dlopen(p, RTLD_NOW | RTLD_GLOBAL);
    }
    if (!h) return fail(FJ_E_NCCL, std::string("cannot dlopen libnccl.so.2 (set FJ_NCCL_LIB): ") + dlerror());
#define FJ_SYM(f, n) api.f = reinterpret_cast<decltype(api.f)>(dlsym(h, n)); if (!api.f) return fail(FJ_E_NCCL, "missing " n)
    FJ_SYM(GetUniqueId, "ncclGetUniqueId");
    FJ_SYM(CommInitRank, "ncclCommInitRank");
    FJ_SYM(CommDestroy, "ncclCommDestroy");
    FJ_SYM(AllReduce, "ncclAllReduce");
    FJ_SYM(Send, "ncclSend");
    FJ_SYM(Recv, "ncclRecv");
    FJ_SYM(GroupStart, "ncclGroupStart");
    FJ_SYM(GroupEnd, "ncclGroupEnd");
    FJ_SYM(ErrStr, "ncclGetErrorString");
#undef FJ_SYM
    api.h = h;
  }
  *out = &api;
  return FJ_OK;
}

#define FJ_NCCL(call)                                                                  \
  do {                                                                                 \
    ncclResult_t _r = (call);                                                          \
    if (_r != ncclSuccess) return fail(FJ_E_NCCL, std::string("NCCL: ") + #call + ": " + api->ErrStr(_r)); \
  } while (0)

// ---------------------------------------------------------------- loopback world
struct LoopWorld {
  int nranks;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  long gen = 0;
  std::vector<const double*> send_buf;              // per rank
  std::vector<std::vector<int64_t>> send_off, send_cnt;
  std::vector<std::vector<double>> slots;           // allreduce staging per rank
  explicit LoopWorld(int n) : nranks(n), send_buf(n, nullptr), send_off(n), send_cnt(n), slots(n) {}
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const long g = gen;
    if (++arrived == nranks) {
      arrived = 0;
      ++gen;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return gen != g; });
    }
  }
};

}  // namespace fj

struct fj_comm {
  int kind = 0;   // 0 NCCL, 1 loopback
  int nranks = 1, rank = 0;
  ncclComm_t nccl = nullptr;
  fj::LoopWorld* world = nullptr;
};

namespace fj {

enum RedOp { RED_SUM = 0, RED_MIN = 1, RED_MAX = 2 };

// One rank's share of a row-partitioned graph.
struct DistInfo {
  fj_comm* comm = nullptr;
  int rank = 0, nranks = 1;
  int64_t n_global = 0, row_begin = 0, n_loc = 0, n_ghost = 0;
  std::vector<int64_t> bounds;                       // [nranks+1]
  std::vector<int64_t> recv_off, recv_cnt;           // ghost segment per owner (into [n_loc, n_loc+n_ghost))
  std::vector<int64_t> send_off, send_cnt;           // send segment per peer
  int64_t n_send = 0;
  int32_t* col_local = nullptr;                      // renumbered columns (owned)
  int32_t* send_idx = nullptr;                       // [n_send] local row indices (owned)
  double* send_buf = nullptr;                        // [n_send][kHaloMaxW]
  double d_max_global = 0.0;
  // solver workspace (vectors extended by the ghost segment)
  double *x = nullptr, *r = nullptr, *p = nullptr, *q = nullptr, *red = nullptr;   // red: allreduce payloads
  PcgScalars* sc = nullptr;
  double* elem_part = nullptr;
  unsigned int* elem_ticket = nullptr;
  int grid_elem = 0;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
};

static DistInfo* D(const fj_graph* g) { return reinterpret_cast<DistInfo*>(g->dist); }

// ---------------------------------------------------------------- collectives
static fj_status allreduce(DistInfo* d, double* buf, int count, RedOp op, cudaStream_t st) {
  fj_comm* c = d->comm;
  if (c->nranks == 1 && !c->nccl) return FJ_OK;
  if (c->kind == 0) {
    NcclApi* api = nullptr;
    FJ_TRY(nccl_api(&api));
    const ncclRedOp_t nop = op == RED_SUM ? ncclSum : (op == RED_MIN ? ncclMin : ncclMax);
    FJ_NCCL(api->AllReduce(buf, buf, (size_t)count, ncclDouble, nop, c->nccl, st));
    return FJ_OK;
  }
  LoopWorld* w = c->world;
  std::vector<double>& mine = w->slots[d->rank];
  mine.resize(count);
  FJ_CK(cudaMemcpyAsync(mine.data(), buf, sizeof(double) * count, cudaMemcpyDeviceToHost, st));
  FJ_CK(cudaStreamSynchronize(st));
  w->barrier();
  std::vector<double> res(count);
  for (int j = 0; j < count; ++j) {
    double a = w->slots[0][j];
    for (int q = 1; q < w->nranks; ++q) {   // fixed rank order
      const double b = w->slots[q][j];
      a = op == RED_SUM ? a + b : (op == RED_MIN ? std::min(a, b) : std::max(a, b));
    }
    res[j] = a;
  }
  w->barrier();   // every rank has read the slots
  FJ_CK(cudaMemcpyAsync(buf, res.data(), sizeof(double) * count, cudaMemcpyHostToDevice, st));
  FJ_CK(cudaStreamSynchronize(st));   // res is a host temporary
  return FJ_OK;
}

// send rows of W doubles: buf[i][0..W) = x[idx[i]][0..W)
__global__ void k_pack(int64_t ns, int W, const int32_t* __restrict__ idx, const double* __restrict__ x,
                       double* __restrict__ buf) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < ns * W; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = q / W;
    buf[q] = x[(int64_t)idx[i] * W + (q - i * W)];
  }
}

constexpr int kHaloMaxW = 4;   // widest row the halo carries (the small-k vector engine's KP)

// rows [n_loc .. n_loc + n_ghost) of the W-wide row-major x <- the owners' rows
static fj_status halo_exchange(DistInfo* d, double* x, cudaStream_t st, int W = 1) {
  fj_comm* c = d->comm;
  if (c->nranks == 1) return FJ_OK;
  if (W < 1 || W > kHaloMaxW) return fail(FJ_E_INTERNAL, "halo row width");
  if (d->n_send > 0) {
    const unsigned gb = (unsigned)std::min<int64_t>((d->n_send * W + 255) / 256, 4096);
    k_pack<<<gb, 256, 0, st>>>(d->n_send, W, d->send_idx, x, d->send_buf);
    FJ_CK_LAUNCH();
  }
  if (c->kind == 0) {
    NcclApi* api = nullptr;
    FJ_TRY(nccl_api(&api));
    FJ_NCCL(api->GroupStart());
    for (int q = 0; q < c->nranks; ++q) {
      if (q == d->rank) continue;
      if (d->send_cnt[q] > 0)
        FJ_NCCL(api->Send(d->send_buf + d->send_off[q] * W, (size_t)(d->send_cnt[q] * W), ncclDouble, q, c->nccl, st));
      if (d->recv_cnt[q] > 0)
        FJ_NCCL(api->Recv(x + (d->n_loc + d->recv_off[q]) * W, (size_t)(d->recv_cnt[q] * W), ncclDouble, q, c->nccl, st));
    }
    FJ_NCCL(api->GroupEnd());
    return FJ_OK;
  }
  LoopWorld* w = c->world;
  FJ_CK(cudaStreamSynchronize(st));
  w->barrier();   // all send buffers packed
  for (int o = 0; o < c->nranks; ++o) {
    if (o == d->rank || d->recv_cnt[o] == 0) continue;
    FJ_CK(cudaMemcpyAsync(x + (d->n_loc + d->recv_off[o]) * W, w->send_buf[o] + w->send_off[o][d->rank] * W,
                          sizeof(double) * d->recv_cnt[o] * W, cudaMemcpyDeviceToDevice, st));
  }
  FJ_CK(cudaStreamSynchronize(st));
  w->barrier();   // all pulls done before anyone repacks
  return FJ_OK;
}

// ---------------------------------------------------------------- a1 restricted to a row range
struct RowRangeBuild {
  int64_t r0, r1;
};

__global__ void k_degree_hist(int64_t m, const int32_t* __restrict__ u, const int32_t* __restrict__ v,
                              unsigned long long* __restrict__ cnt) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x) {
    const int32_t a = u[e], b = v[e];
    if (a == b) continue;
    atomicAdd(cnt + a, 1ULL);
    atomicAdd(cnt + b, 1ULL);
  }
}

__global__ void k_bounds(int64_t n, const unsigned long long* __restrict__ pre /*[n+1] exclusive*/, int P,
                         int64_t* __restrict__ bounds) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r > P) return;
  if (r == 0) { bounds[0] = 0; return; }
  if (r == P) { bounds[P] = n; return; }
  const unsigned long long total = pre[n];
  const unsigned long long target = (total / P) * r + (total % P) * r / P;   // floor(total r / P), exact
  int64_t lo = 0, hi = n;   // first row i with pre[i] >= target
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (pre[mid] < target) lo = mid + 1; else hi = mid;
  }
  bounds[r] = lo;
}

struct NotInRange {
  int32_t r0, r1;
  __host__ __device__ __forceinline__ bool operator()(const int32_t& c) const { return c < r0 || c >= r1; }
};

// columns -> local numbering: [r0, r1) -> c - r0; ghosts -> n_loc + index in the sorted ghost list
__global__ void k_renumber(int64_t nnz, const int32_t* __restrict__ cg, int64_t r0, int64_t r1,
                           const int32_t* __restrict__ ghosts, int64_t ng, int32_t* __restrict__ cl) {
  const int64_t nl = r1 - r0;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < nnz; p += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = cg[p];
    if (c >= r0 && c < r1) {
      cl[p] = (int32_t)(c - r0);
    } else {
      int64_t lo = 0, hi = ng;
      while (lo < hi) {
        const int64_t mid = (lo + hi) >> 1;
        if (ghosts[mid] < c) lo = mid + 1; else hi = mid;
      }
      cl[p] = (int32_t)(nl + lo);
    }
  }
}

// position of each owner's first ghost (bounds[o]) in the sorted ghost list
__global__ void k_owner_split(int P, const int64_t* __restrict__ bounds, const int32_t* __restrict__ ghosts,
                              int64_t ng, int64_t* __restrict__ pos) {
  const int o = blockIdx.x * blockDim.x + threadIdx.x;
  if (o > P) return;
  const int64_t b = bounds[o];
  int64_t lo = 0, hi = ng;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (ghosts[mid] < b) lo = mid + 1; else hi = mid;
  }
  pos[o] = lo;
}

// ---------------------------------------------------------------- distributed PCG kernels
constexpr int DTPB = 256;

template <int NPART>
__device__ __forceinline__ bool d_reduce(double (&v)[NPART], double* part, unsigned int* ticket, double* s_red) {
  block_sum<NPART, DTPB>(v, s_red);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int j = 0; j < NPART; ++j) part[blockIdx.x * 4 + j] = v[j];
  }
  if (!last_block_ticket(ticket, gridDim.x)) return false;
  double t[NPART];
#pragma unroll
  for (int j = 0; j < NPART; ++j) t[j] = 0.0;
  for (int b = threadIdx.x; b < (int)gridDim.x; b += DTPB) {
#pragma unroll
    for (int j = 0; j < NPART; ++j) t[j] += __ldcg(part + b * 4 + j);
  }
  block_sum<NPART, DTPB>(t, s_red);
#pragma unroll
  for (int j = 0; j < NPART; ++j) v[j] = t[j];
  return true;
}

// local part of the (re)start: r = s - q (restart) or s, x = 0 (fresh), p = dinv r;
// red[3..5] = local (r^T y, r^T r, s^T s)
__global__ void __launch_bounds__(DTPB) k_dinit(int64_t n, const double* __restrict__ s, int64_t ld, int64_t c,
                                                const double* __restrict__ dinv, const double* __restrict__ q,
                                                int restart, double* __restrict__ x, double* __restrict__ r,
                                                double* __restrict__ p, double* red, double* part,
                                                unsigned int* ticket) {
  __shared__ double s_red[3 * DTPB / 32];
  double v[3] = {0.0, 0.0, 0.0};
  for (int64_t i = blockIdx.x * (int64_t)DTPB + threadIdx.x; i < n; i += (int64_t)gridDim.x * DTPB) {
    const double si = s[i * ld + c];
    const double ri = restart ? si - q[i] : si;
    if (!restart) x[i] = 0.0;
    const double yi = dinv[i] * ri;
    r[i] = ri;
    p[i] = yi;
    v[0] = fma(ri, yi, v[0]);
    v[1] = fma(ri, ri, v[1]);
    v[2] = fma(si, si, v[2]);
  }
  if (d_reduce<3>(v, part, ticket, s_red) && threadIdx.x == 0) {
    red[3] = v[0]; red[4] = v[1]; red[5] = v[2];
    *ticket = 0u;
  }
}

// global scalars after allreduce(red[3..5])
__global__ void k_dinit_post(const double* red, PcgScalars* sc, double rtol, int max_iter) {
  sc->rho = red[3];
  sc->rr = red[4];
  sc->ss = red[5];
  sc->tol2 = rtol * rtol * red[5];
  sc->iter = 0;
  sc->max_iter = max_iter;
  sc->converged = red[4] <= sc->tol2 ? 1 : 0;
  sc->done = (sc->converged || max_iter <= 0) ? 1 : 0;
  sc->breakdown = 0;
  sc->alpha = sc->beta = 0.0;
}

// K_B with alpha = rho / allreduced p^T q (red[0]); red[1..2] = local (rho', ||r||^2)
__global__ void __launch_bounds__(DTPB) k_dupdate(int64_t n, const double* __restrict__ dinv,
                                                  const double* __restrict__ p, const double* __restrict__ q,
                                                  double* __restrict__ x, double* __restrict__ r,
                                                  const PcgScalars* sc, double* red, double* part,
                                                  unsigned int* ticket) {
  __shared__ double s_red[2 * DTPB / 32];
  if (*(volatile const int32_t*)&sc->done) return;
  const double pq = red[0];
  const double alpha = (pq > 0.0 && isfinite(pq)) ? sc->rho / pq : 0.0;
  double v[2] = {0.0, 0.0};
  for (int64_t i = blockIdx.x * (int64_t)DTPB + threadIdx.x; i < n; i += (int64_t)gridDim.x * DTPB) {
    x[i] = fma(alpha, p[i], x[i]);
    const double ri = fma(-alpha, q[i], r[i]);
    r[i] = ri;
    v[0] = fma(ri, dinv[i] * ri, v[0]);
    v[1] = fma(ri, ri, v[1]);
  }
  if (d_reduce<2>(v, part, ticket, s_red) && threadIdx.x == 0) {
    red[1] = v[0]; red[2] = v[1];
    *ticket = 0u;
  }
}

// beta / convergence from the allreduced red[0..2]; identical on every rank
__global__ void k_dpost(const double* red, PcgScalars* sc) {
  if (sc->done) return;
  const double pq = red[0];
  if (!(pq > 0.0) || !isfinite(pq)) { sc->breakdown = 1; sc->done = 1; return; }
  sc->pq = pq;
  sc->alpha = sc->rho / pq;
  sc->beta = red[1] / sc->rho;
  sc->rho = red[1];
  sc->rr = red[2];
  const int it = sc->iter + 1;
  sc->iter = it;
  sc->converged = red[2] <= sc->tol2 ? 1 : 0;
  if (sc->converged || it >= sc->max_iter || !isfinite(red[2])) sc->done = 1;
}

__global__ void __launch_bounds__(DTPB) k_ddir(int64_t n, const double* __restrict__ dinv,
                                               const double* __restrict__ r, double* __restrict__ p,
                                               const PcgScalars* sc) {
  if (*(volatile const int32_t*)&sc->done) return;
  const double beta = sc->beta;
  for (int64_t i = blockIdx.x * (int64_t)DTPB + threadIdx.x; i < n; i += (int64_t)gridDim.x * DTPB)
    p[i] = fma(beta, p[i], dinv[i] * r[i]);
}

__global__ void k_dcopy(int64_t n, const double* __restrict__ src, int64_t sld, int64_t sc_, double* __restrict__ dst,
                        int64_t dld, int64_t dc) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i * dld + dc] = src[i * sld + sc_];
}

// ---------------------------------------------------------------- row engine on the local rows
template <int WT, class Op>
static fj_status dist_rows(const fj_graph* g, const Op& op, cudaStream_t st) {
  SolveWs* w = nullptr;
  FJ_TRY(get_ws(const_cast<fj_graph*>(g), st, &w));
  FJ_CK(launch_warp_items<WT>(g, w, op, st));
  FJ_CK_LAUNCH();
  return FJ_OK;
}

template <int WT>
static fj_status d_apply_wt(const fj_graph* g, const double* x, double* y, const PcgScalars* sc, double* dot,
                            int opL, cudaStream_t st) {
  ApplyOp<WT> op{x, y, g->deg, 1, 0, opL, const_cast<PcgScalars*>(sc), dot};
  op.alpha_on_device = 0;
  return dist_rows<WT>(g, op, st);
}

static fj_status d_apply(const fj_graph* g, const double* x, double* y, const PcgScalars* sc, double* dot, int opL,
                         cudaStream_t st) {
  switch (g->wtype) {
    case FJ_W_UNIT: return d_apply_wt<FJ_W_UNIT>(g, x, y, sc, dot, opL, st);
    case FJ_W_U8: return d_apply_wt<FJ_W_U8>(g, x, y, sc, dot, opL, st);
    case FJ_W_F32: return d_apply_wt<FJ_W_F32>(g, x, y, sc, dot, opL, st);
    default: return d_apply_wt<FJ_W_F64>(g, x, y, sc, dot, opL, st);
  }
}

template <int WT>
static fj_status d_resid_wt(const fj_graph* g, const double* xext, const double* s, int64_t ld, int64_t c, double* out,
                            cudaStream_t st) {
  ResidOp<WT> op{xext, s, g->deg, ld, c, out};
  return dist_rows<WT>(g, op, st);
}

static fj_status d_resid(const fj_graph* g, const double* xext, const double* s, int64_t ld, int64_t c, double* out,
                         cudaStream_t st) {
  switch (g->wtype) {
    case FJ_W_UNIT: return d_resid_wt<FJ_W_UNIT>(g, xext, s, ld, c, out, st);
    case FJ_W_U8: return d_resid_wt<FJ_W_U8>(g, xext, s, ld, c, out, st);
    case FJ_W_F32: return d_resid_wt<FJ_W_F32>(g, xext, s, ld, c, out, st);
    default: return d_resid_wt<FJ_W_F64>(g, xext, s, ld, c, out, st);
  }
}

template <int WT>
static fj_status d_quant_wt(const fj_graph* g, const double* zext, const double* s, int64_t ld, int64_t c, double m,
                            double* out, cudaStream_t st) {
  QuantOp<WT> op{zext, s, g->deg, ld, c, m, out};
  op.zld = 1;
  op.zc = 0;
  return dist_rows<WT>(g, op, st);
}

fj_status dist_quant_pass(const fj_graph* g, const double* s, const double* z, int64_t ld, int64_t c, double m,
                          double* host10, cudaStream_t st);

static fj_status ensure_dist_ws(fj_graph* g, cudaStream_t st) {
  DistInfo* d = D(g);
  if (d->x) return FJ_OK;
  const int64_t ne = d->n_loc + d->n_ghost;
  FJ_CK(dmalloc(&d->x, sizeof(double) * std::max<int64_t>(ne, 1), st));
  FJ_CK(dmalloc(&d->p, sizeof(double) * std::max<int64_t>(ne, 1), st));
  FJ_CK(dmalloc(&d->r, sizeof(double) * std::max<int64_t>(d->n_loc, 1), st));
  FJ_CK(dmalloc(&d->q, sizeof(double) * std::max<int64_t>(d->n_loc, 1), st));
  FJ_CK(dmalloc(&d->red, sizeof(double) * 16, st));
  FJ_CK(dmalloc(&d->sc, sizeof(PcgScalars), st));
  FJ_CK(cudaMemsetAsync(d->sc, 0, sizeof(PcgScalars), st));
  int64_t ge = (int64_t)g->num_sms * (2048 / DTPB);
  const int64_t need = (d->n_loc + DTPB - 1) / DTPB;
  if (ge > need) ge = need > 0 ? need : 1;
  d->grid_elem = (int)ge;
  FJ_CK(dmalloc(&d->elem_part, sizeof(double) * 4 * ge, st));
  FJ_CK(dmalloc(&d->elem_ticket, sizeof(unsigned int), st));
  FJ_CK(cudaMemsetAsync(d->elem_ticket, 0, sizeof(unsigned int), st));
  FJ_CK(cudaEventCreate(&d->ev0));
  FJ_CK(cudaEventCreate(&d->ev1));
  return FJ_OK;
}

// One column: s column c of [n_loc][ld] -> z column c.  Host-driven loop (NCCL calls between
// kernels); the host reads the device `done` flag every 8 iterations.
fj_status dist_solve_col(fj_graph* g, const double* s, double* z, int64_t ld, int64_t c, const fj_solve_opts& o,
                         int warm, fj_solve_report* rep, cudaStream_t st) {
  DistInfo* d = D(g);
  FJ_TRY(ensure_dist_ws(g, st));
  const int64_t nl = d->n_loc;
  const unsigned gb = (unsigned)std::min<int64_t>((nl + 255) / 256, 4096);
  int restarts = 0, total = 0;
  PcgScalars h{};
  double rel_true = NAN, res2 = 0.0;
  bool first = true;
  for (;;) {
    const bool restart = !first || warm;
    if (restart) {
      if (first) { k_dcopy<<<gb, 256, 0, st>>>(nl, z, ld, c, d->x, 1, 0); FJ_CK_LAUNCH(); }
      FJ_TRY(halo_exchange(d, d->x, st));
      FJ_TRY(d_apply(g, d->x, d->q, nullptr, nullptr, 0, st));
    }
    const int budget = std::max(0, o.max_iter - total);
    FJ_CK(cudaEventRecord(d->ev0, st));
    k_dinit<<<d->grid_elem, DTPB, 0, st>>>(nl, s, ld, c, g->dinv, d->q, restart ? 1 : 0, d->x, d->r, d->p, d->red,
                                           d->elem_part, d->elem_ticket);
    FJ_CK_LAUNCH();
    FJ_TRY(allreduce(d, d->red + 3, 3, RED_SUM, st));
    k_dinit_post<<<1, 1, 0, st>>>(d->red, d->sc, o.rtol, budget);
    FJ_CK_LAUNCH();
    first = false;
    for (;;) {
      for (int u = 0; u < 8; ++u) {
        FJ_TRY(halo_exchange(d, d->p, st));
        FJ_TRY(d_apply(g, d->p, d->q, d->sc, d->red, 0, st));          // red[0] = local p^T q
        FJ_TRY(allreduce(d, d->red, 1, RED_SUM, st));
        k_dupdate<<<d->grid_elem, DTPB, 0, st>>>(nl, g->dinv, d->p, d->q, d->x, d->r, d->sc, d->red, d->elem_part,
                                                 d->elem_ticket);
        FJ_CK_LAUNCH();
        FJ_TRY(allreduce(d, d->red + 1, 2, RED_SUM, st));
        k_dpost<<<1, 1, 0, st>>>(d->red, d->sc);
        FJ_CK_LAUNCH();
        k_ddir<<<d->grid_elem, DTPB, 0, st>>>(nl, g->dinv, d->r, d->p, d->sc);
        FJ_CK_LAUNCH();
      }
      FJ_CK(cudaMemcpyAsync(&h, d->sc, sizeof h, cudaMemcpyDeviceToHost, st));
      FJ_CK(cudaStreamSynchronize(st));
      if (h.done) break;
    }
    FJ_CK(cudaEventRecord(d->ev1, st));
    // true residual: halo of x, local ||s - (I+L)x||^2, allreduce
    FJ_TRY(halo_exchange(d, d->x, st));
    FJ_TRY(d_resid(g, d->x, s, ld, c, d->red + 6, st));
    FJ_TRY(allreduce(d, d->red + 6, 1, RED_SUM, st));
    FJ_CK(cudaMemcpyAsync(&res2, d->red + 6, sizeof res2, cudaMemcpyDeviceToHost, st));
    FJ_CK(cudaStreamSynchronize(st));
    float lms = 0.f;
    cudaEventElapsedTime(&lms, d->ev0, d->ev1);
    total += h.iter;
    if (rep) { rep->ms_loop += lms; rep->iterations_total += h.iter; }
    rel_true = h.ss > 0 ? std::sqrt(res2 / h.ss) : 0.0;
    if (res2 <= h.tol2 || restarts >= o.max_restarts || total >= o.max_iter || h.breakdown) break;
    ++restarts;
  }
  k_dcopy<<<gb, 256, 0, st>>>(nl, d->x, 1, 0, z, ld, c);
  FJ_CK_LAUNCH();
  const bool ok = res2 <= h.tol2;
  if (rep) {
    rep->iterations = std::max(rep->iterations, total);
    rep->restarts = std::max(rep->restarts, restarts);
    rep->rel_res_recursive = std::max(rep->rel_res_recursive, h.ss > 0 ? std::sqrt(h.rr / h.ss) : 0.0);
    rep->rel_res_true = std::isnan(rep->rel_res_true) ? rel_true : std::max(rep->rel_res_true, rel_true);
    if (!ok) rep->converged = 0;
  }
  return ok ? FJ_OK : fail(FJ_E_NO_CONVERGENCE, "distributed PCG did not reach rtol on the true residual");
}

// Quantities of one column: halo of z, fused pass on the local rows, allreduce of the 10 sums.
fj_status dist_quant_pass(const fj_graph* g, const double* s, const double* z, int64_t ld, int64_t c, double m,
                          double* host10, cudaStream_t st) {
  DistInfo* d = D(g);
  FJ_TRY(ensure_dist_ws(const_cast<fj_graph*>(g), st));
  const int64_t nl = d->n_loc;
  const unsigned gb = (unsigned)std::min<int64_t>((nl + 255) / 256, 4096);
  k_dcopy<<<gb, 256, 0, st>>>(nl, z, ld, c, d->x, 1, 0);
  FJ_CK_LAUNCH();
  FJ_TRY(halo_exchange(d, d->x, st));
  fj_status r;
  switch (g->wtype) {
    case FJ_W_UNIT: r = d_quant_wt<FJ_W_UNIT>(g, d->x, s, ld, c, m, d->red, st); break;
    case FJ_W_U8: r = d_quant_wt<FJ_W_U8>(g, d->x, s, ld, c, m, d->red, st); break;
    case FJ_W_F32: r = d_quant_wt<FJ_W_F32>(g, d->x, s, ld, c, m, d->red, st); break;
    default: r = d_quant_wt<FJ_W_F64>(g, d->x, s, ld, c, m, d->red, st); break;
  }
  FJ_TRY(r);
  FJ_TRY(allreduce(d, d->red, 10, RED_SUM, st));
  FJ_CK(cudaMemcpyAsync(host10, d->red, sizeof(double) * 10, cudaMemcpyDeviceToHost, st));
  FJ_CK(cudaStreamSynchronize(st));
  return FJ_OK;
}

// Opinion statistics of the local slices combined across ranks: (sum, sumsq) summed, min, max.
fj_status dist_stats_combine(const fj_graph* g, int k, double* dev4k /* [k][4] device */, cudaStream_t st) {
  DistInfo* d = D(g);
  if (d->nranks == 1) return FJ_OK;
  std::vector<double> h(4 * k);
  FJ_CK(cudaMemcpyAsync(h.data(), dev4k, sizeof(double) * 4 * k, cudaMemcpyDeviceToHost, st));
  FJ_CK(cudaStreamSynchronize(st));
  std::vector<double> sums(2 * k), mins(k), maxs(k);
  for (int c = 0; c < k; ++c) { sums[2 * c] = h[4 * c]; sums[2 * c + 1] = h[4 * c + 1]; mins[c] = h[4 * c + 2]; maxs[c] = h[4 * c + 3]; }
  double* tmp = nullptr;
  FJ_CK(dmalloc(&tmp, sizeof(double) * 4 * k, st));
  FJ_CK(cudaMemcpyAsync(tmp, sums.data(), sizeof(double) * 2 * k, cudaMemcpyHostToDevice, st));
  FJ_CK(cudaMemcpyAsync(tmp + 2 * k, mins.data(), sizeof(double) * k, cudaMemcpyHostToDevice, st));
  FJ_CK(cudaMemcpyAsync(tmp + 3 * k, maxs.data(), sizeof(double) * k, cudaMemcpyHostToDevice, st));
  fj_status s1 = allreduce(d, tmp, 2 * k, RED_SUM, st);
  fj_status s2 = s1 == FJ_OK ? allreduce(d, tmp + 2 * k, k, RED_MIN, st) : s1;
  fj_status s3 = s2 == FJ_OK ? allreduce(d, tmp + 3 * k, k, RED_MAX, st) : s2;
  if (s3 == FJ_OK) {
    FJ_CK(cudaMemcpyAsync(sums.data(), tmp, sizeof(double) * 2 * k, cudaMemcpyDeviceToHost, st));
    FJ_CK(cudaMemcpyAsync(mins.data(), tmp + 2 * k, sizeof(double) * k, cudaMemcpyDeviceToHost, st));
    FJ_CK(cudaMemcpyAsync(maxs.data(), tmp + 3 * k, sizeof(double) * k, cudaMemcpyDeviceToHost, st));
    FJ_CK(cudaStreamSynchronize(st));
    for (int c = 0; c < k; ++c) { h[4 * c] = sums[2 * c]; h[4 * c + 1] = sums[2 * c + 1]; h[4 * c + 2] = mins[c]; h[4 * c + 3] = maxs[c]; }
    FJ_CK(cudaMemcpyAsync(dev4k, h.data(), sizeof(double) * 4 * k, cudaMemcpyHostToDevice, st));
    FJ_CK(cudaStreamSynchronize(st));
  }
  dfree_on(tmp, st);
  return s3;
}

bool is_dist(const fj_graph* g) { return g->dist != nullptr; }
int64_t dist_n_ghost(const fj_graph* g) { return g->dist ? D(g)->n_ghost : 0; }
fj_status dist_halo_rows(const fj_graph* g, double* x_ext, int width, cudaStream_t st) {
  return halo_exchange(D(g), x_ext, st, width);
}
fj_status dist_allreduce_sum(const fj_graph* g, double* buf, int count, cudaStream_t st) {
  return allreduce(D(g), buf, count, RED_SUM, st);
}
// ||s_c - (I+L) z_c||^2 over all ranks for column c of the local slices (host result)
fj_status dist_true_res2(fj_graph* g, const double* s, const double* z, int64_t ld, int64_t c, double* res2_host,
                         cudaStream_t st) {
  DistInfo* d = D(g);
  FJ_TRY(ensure_dist_ws(g, st));
  const int64_t nl = d->n_loc;
  const unsigned gb = (unsigned)std::min<int64_t>((nl + 255) / 256, 4096);
  k_dcopy<<<gb, 256, 0, st>>>(nl, z, ld, c, d->x, 1, 0);
  FJ_CK_LAUNCH();
  FJ_TRY(halo_exchange(d, d->x, st));
  FJ_TRY(d_resid(g, d->x, s, ld, c, d->red + 6, st));
  FJ_TRY(allreduce(d, d->red + 6, 1, RED_SUM, st));
  FJ_CK(cudaMemcpyAsync(res2_host, d->red + 6, sizeof(double), cudaMemcpyDeviceToHost, st));
  FJ_CK(cudaStreamSynchronize(st));
  return FJ_OK;
}
int64_t global_n(const fj_graph* g) { return g->dist ? D(g)->n_global : g->n; }
double global_dmax(const fj_graph* g) { return g->dist ? D(g)->d_max_global : g->info.d_max; }

void free_dist(fj_graph* g) {
  DistInfo* d = D(g);
  if (!d) return;
  if (d->comm && d->comm->kind == 1 && d->comm->world) {
    d->comm->world->send_buf[d->rank] = nullptr;
  }
  dfree(d->col_local); dfree(d->send_idx); dfree(d->send_buf);
  dfree(d->x); dfree(d->r); dfree(d->p); dfree(d->q); dfree(d->red); dfree(d->sc);
  dfree(d->elem_part); dfree(d->elem_ticket);
  if (d->ev0) cudaEventDestroy(d->ev0);
  if (d->ev1) cudaEventDestroy(d->ev1);
  delete d;
  g->dist = nullptr;
}

}  // namespace fj

using namespace fj;

extern "C" {

fj_status fj_comm_unique_id(unsigned char id[128]) {
  if (!id) return fail(FJ_E_INVALID_ARG, "null id");
  NcclApi* api = nullptr;
  FJ_TRY(nccl_api(&api));
  ncclUniqueId u;
  FJ_NCCL(api->GetUniqueId(&u));
  memcpy(id, u.internal, 128);
  return FJ_OK;
}

fj_status fj_comm_init(int nranks, int rank, const unsigned char id[128], fj_comm** out) {
  if (!out || !id || nranks < 1 || rank < 0 || rank >= nranks) return fail(FJ_E_INVALID_ARG, "bad comm arguments");
  *out = nullptr;
  fj_comm* c = new fj_comm();
  c->kind = 0;
  c->nranks = nranks;
  c->rank = rank;
  // a 1-rank communicator skips NCCL unless FJ_NCCL_FORCE is set (exercises the NCCL calls on one GPU)
  if (nranks > 1 || getenv("FJ_NCCL_FORCE")) {
    NcclApi* api = nullptr;
    fj_status s = nccl_api(&api);
    if (s != FJ_OK) { delete c; return s; }
    ncclUniqueId u;
    memcpy(u.internal, id, 128);
    ncclResult_t r = api->CommInitRank(&c->nccl, nranks, u, rank);
    if (r != ncclSuccess) { delete c; return fail(FJ_E_NCCL, std::string("ncclCommInitRank: ") + api->ErrStr(r)); }
  }
  *out = c;
  return FJ_OK;
}

fj_status fj_comm_init_loopback(int nranks, fj_comm** out) {
  if (!out || nranks < 1) return fail(FJ_E_INVALID_ARG, "bad comm arguments");
  fj_comm* c = new fj_comm();
  c->kind = 1;
  c->nranks = nranks;
  c->world = new LoopWorld(nranks);
  *out = c;
  return FJ_OK;
}

fj_status fj_comm_destroy(fj_comm* c) {
  if (!c) return FJ_OK;
  if (c->kind == 0 && c->nccl) {
    NcclApi* api = nullptr;
    if (nccl_api(&api) == FJ_OK) api->CommDestroy(c->nccl);
  }
  delete c->world;
  delete c;
  return FJ_OK;
}

fj_status fj_partition_rows(int64_t n, int64_t m, const int32_t* u, const int32_t* v, int nranks, int64_t* bounds_host,
                            void* stream) {
  if (n < 1 || n >= INT32_MAX || m < 0 || nranks < 1 || !bounds_host || (m > 0 && (!u || !v)))
    return fail(FJ_E_INVALID_ARG, "bad partition arguments");
  cudaStream_t st = S(stream);
  DevBuf<unsigned long long> cnt, pre;
  DevBuf<int64_t> b;
  FJ_TRY(cnt.alloc(n + 1, st));
  FJ_TRY(pre.alloc(n + 1, st));
  FJ_TRY(b.alloc(nranks + 1, st));
  FJ_CK(cudaMemsetAsync(cnt.p, 0, sizeof(unsigned long long) * (n + 1), st));
  if (m > 0) {
    k_degree_hist<<<(unsigned)std::min<int64_t>((m + 255) / 256, 8192), 256, 0, st>>>(m, u, v, cnt.p);
    FJ_CK_LAUNCH();
  }
  size_t bytes = 0;
  FJ_CK(cub::DeviceScan::ExclusiveSum(nullptr, bytes, cnt.p, pre.p, n + 1, st));
  {
    DevBuf<uint8_t> tmp;
    FJ_TRY(tmp.alloc((int64_t)bytes, st));
    FJ_CK(cub::DeviceScan::ExclusiveSum(tmp.p, bytes, cnt.p, pre.p, n + 1, st));
    count_cub();
  }
  k_bounds<<<(nranks + 1 + 63) / 64, 64, 0, st>>>(n, pre.p, nranks, b.p);
  FJ_CK_LAUNCH();
  FJ_CK(cudaMemcpyAsync(bounds_host, b.p, sizeof(int64_t) * (nranks + 1), cudaMemcpyDeviceToHost, st));
  FJ_CK(cudaStreamSynchronize(st));
  return FJ_OK;
}

fj_status fj_dist_ghosts(int64_t nnz, const int32_t* col_global, int64_t r0, int64_t r1, int32_t* ghosts_out,
                         int64_t* n_ghost_out, void* stream) {
  if (nnz < 0 || !n_ghost_out || (nnz > 0 && (!col_global || !ghosts_out)) || r0 < 0 || r1 < r0)
    return fail(FJ_E_INVALID_ARG, "bad ghost arguments");
  cudaStream_t st = S(stream);
  if (nnz == 0) { *n_ghost_out = 0; return FJ_OK; }
  DevBuf<int32_t> sel, sorted;
  DevBuf<int64_t> nsel;
  FJ_TRY(sel.alloc(nnz, st));
  FJ_TRY(sorted.alloc(nnz, st));
  FJ_TRY(nsel.alloc(2, st));
  NotInRange pred{(int32_t)r0, (int32_t)r1};
  size_t bytes = 0;
  FJ_CK(cub::DeviceSelect::If(nullptr, bytes, col_global, sel.p, nsel.p, nnz, pred, st));
  {
    DevBuf<uint8_t> tmp;
    FJ_TRY(tmp.alloc((int64_t)bytes, st));
    FJ_CK(cub::DeviceSelect::If(tmp.p, bytes, col_global, sel.p, nsel.p, nnz, pred, st));
    count_cub();
  }
  int64_t ns = 0;
  FJ_CK(cudaMemcpyAsync(&ns, nsel.p, sizeof ns, cudaMemcpyDeviceToHost, st));
  FJ_CK(cudaStreamSynchronize(st));
  if (ns == 0) { *n_ghost_out = 0; return FJ_OK; }
  bytes = 0;
  FJ_CK(cub::DeviceRadixSort::SortKeys(nullptr, bytes, sel.p, sorted.p, ns, 0, 32, st));
  {
    DevBuf<uint8_t> tmp;
    FJ_TRY(tmp.alloc((int64_t)bytes, st));
    FJ_CK(cub::DeviceRadixSort::SortKeys(tmp.p, bytes, sel.p, sorted.p, ns, 0, 32, st));
    count_cub();
  }
  bytes = 0;
  FJ_CK(cub::DeviceSelect::Unique(nullptr, bytes, sorted.p, ghosts_out, nsel.p + 1, ns, st));
  {
    DevBuf<uint8_t> tmp;
    FJ_TRY(tmp.alloc((int64_t)bytes, st));
    FJ_CK(cub::DeviceSelect::Unique(tmp.p, bytes, sorted.p, ghosts_out, nsel.p + 1, ns, st));
    count_cub();
  }
  FJ_CK(cudaMemcpyAsync(n_ghost_out, nsel.p + 1, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  FJ_CK(cudaStreamSynchronize(st));
  return FJ_OK;
}

fj_status fj_graph_create_dist(fj_comm* comm, int rank, int64_t n_global, const int64_t* bounds, int64_t nnz_local,
                               const int64_t* row_ptr_local, const int32_t* col_global, const void* w, int wtype,
                               int64_t n_ghost, const int32_t* ghosts, const int64_t* send_counts,
                               const int32_t* send_idx, void* stream, fj_graph** out) {
  if (!comm || !bounds || !out || !send_counts || rank < 0 || rank >= comm->nranks)
    return fail(FJ_E_INVALID_ARG, "bad distributed graph arguments");
  if (comm->kind == 0 && rank != comm->rank) return fail(FJ_E_INVALID_ARG, "rank does not match the NCCL communicator");
  *out = nullptr;
  const int P = comm->nranks;
  const int64_t r0 = bounds[rank], r1 = bounds[rank + 1], nl = r1 - r0;
  if (nl < 1) return fail(FJ_E_INVALID_ARG, "empty row block");
  if (n_ghost < 0 || (n_ghost > 0 && !ghosts)) return fail(FJ_E_INVALID_ARG, "bad ghost list");
  cudaStream_t st = S(stream);
  DistInfo* d = new DistInfo();
  d->comm = comm;
  d->rank = rank;
  d->nranks = P;
  d->n_global = n_global;
  d->row_begin = r0;
  d->n_loc = nl;
  d->n_ghost = n_ghost;
  d->bounds.assign(bounds, bounds + P + 1);
  auto bail = [&](fj_status s) { dfree(d->col_local); dfree(d->send_idx); dfree(d->send_buf); delete d; return s; };
  cudaError_t ce = dmalloc(&d->col_local, sizeof(int32_t) * std::max<int64_t>(nnz_local, 1), st);
  if (ce != cudaSuccess) return bail(cuda_fail(ce, "dmalloc", __FILE__, __LINE__));
  if (nnz_local > 0) {
    k_renumber<<<(unsigned)std::min<int64_t>((nnz_local + 255) / 256, 8192), 256, 0, st>>>(
        nnz_local, col_global, r0, r1, ghosts, n_ghost, d->col_local);
    ce = cudaGetLastError();
    if (ce != cudaSuccess) return bail(cuda_fail(ce, "k_renumber", __FILE__, __LINE__));
  }
  // ghost segment per owner
  {
    DevBuf<int64_t> bd, pos;
    if (bd.alloc(P + 1, st) != FJ_OK || pos.alloc(P + 1, st) != FJ_OK) return bail(FJ_E_OOM);
    cudaMemcpyAsync(bd.p, bounds, sizeof(int64_t) * (P + 1), cudaMemcpyHostToDevice, st);
    k_owner_split<<<(P + 1 + 63) / 64, 64, 0, st>>>(P, bd.p, ghosts, n_ghost, pos.p);
    std::vector<int64_t> hp(P + 1);
    cudaMemcpyAsync(hp.data(), pos.p, sizeof(int64_t) * (P + 1), cudaMemcpyDeviceToHost, st);
    ce = cudaStreamSynchronize(st);
    if (ce != cudaSuccess) return bail(cuda_fail(ce, "ghost split", __FILE__, __LINE__));
    d->recv_off.resize(P);
    d->recv_cnt.resize(P);
    for (int o = 0; o < P; ++o) { d->recv_off[o] = hp[o]; d->recv_cnt[o] = hp[o + 1] - hp[o]; }
    if (d->recv_cnt[rank] != 0) return bail(fail(FJ_E_INTERNAL, "ghost list contains own rows"));
  }
  d->send_off.resize(P);
  d->send_cnt.assign(send_counts, send_counts + P);
  int64_t acc = 0;
  for (int q = 0; q < P; ++q) { d->send_off[q] = acc; acc += d->send_cnt[q]; }
  d->n_send = acc;
  if (acc > 0) {
    if (!send_idx) return bail(fail(FJ_E_INVALID_ARG, "send_idx is NULL"));
    if (dmalloc(&d->send_idx, sizeof(int32_t) * acc, st) != cudaSuccess ||
        dmalloc(&d->send_buf, sizeof(double) * acc * kHaloMaxW, st) != cudaSuccess)
      return bail(FJ_E_OOM);
    cudaMemcpyAsync(d->send_idx, send_idx, sizeof(int32_t) * acc, cudaMemcpyDeviceToDevice, st);
  }
  // the local graph: n_loc rows, columns in [0, n_loc + n_ghost)
  fj_graph* g = nullptr;
  fj_status s = fj_graph_create(nl, nnz_local, row_ptr_local, d->col_local, w, wtype, 0, stream, &g);
  if (s != FJ_OK) return bail(s);
  g->dist = d;
  // global d_max (identical rounding allowance on every rank)
  {
    double* tmp = nullptr;
    ce = dmalloc(&tmp, sizeof(double), st);
    if (ce != cudaSuccess) { fj_graph_destroy(g); return cuda_fail(ce, "dmalloc", __FILE__, __LINE__); }
    cudaMemcpyAsync(tmp, &g->info.d_max, sizeof(double), cudaMemcpyHostToDevice, st);
    if (comm->kind == 1) {
      LoopWorld* wd = comm->world;
      wd->send_buf[rank] = d->send_buf;
      wd->send_off[rank] = d->send_off;
      wd->send_cnt[rank] = d->send_cnt;
    }
    s = allreduce(d, tmp, 1, RED_MAX, st);
    cudaMemcpyAsync(&d->d_max_global, tmp, sizeof(double), cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    dfree_on(tmp, st);
    if (s != FJ_OK) { fj_graph_destroy(g); return s; }
  }
  *out = g;
  return FJ_OK;
}

}  // extern "C"

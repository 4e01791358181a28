// dist.cu — rows a8/e: the graph row-partitioned over ranks (one process per GPU), NCCL halo
// exchange of the PCG search direction and allreduce of the dot products over NVLink.
//
//  Partition  fj_partition_rows: contiguous row blocks balanced by (raw) nonzeros.
//  Local CSR  fj_csr_rows_from_edges: row a1 restricted to the rank's rows (global column ids).
//  Ghosts     fj_dist_ghosts: sorted unique off-rank columns = the halo, grouped by owner rank.
//  Graph      fj_graph_create_dist: columns renumbered (own -> [0, n_loc), ghost -> n_loc + idx);
//             degrees / schedule on the local rows (full rows, so d_i is exact); halo plan.
//  Iteration  Chronopoulos-Gear PCG (dist_solve_cg, below): one elementwise step, the product of
//             the preconditioned residual with its halo (grouped ncclSend/ncclRecv on a comm
//             stream) overlapped with the own-column pass, ONE allreduce of 3 KP doubles; the
//             iteration is captured in a CUDA graph with the NCCL calls.
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
#include "rows.cuh"
#include "vec.cuh"
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
  struct CgWs* cg = nullptr;                         // single-reduction solver (dist_solve_cg)
};

static DistInfo* D(const fj_graph* g) { return reinterpret_cast<DistInfo*>(g->dist); }
static void free_cg(DistInfo* d);

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

// raw (pre-dedup) endpoint counts, optionally in relabelled ids map[.]
__global__ void k_degree_hist(int64_t m, int64_t n, const int32_t* __restrict__ u, const int32_t* __restrict__ v,
                              const int32_t* __restrict__ map, unsigned long long* __restrict__ cnt) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x) {
    int32_t a = u[e], b = v[e];
    if (a == b || a < 0 || b < 0 || a >= n || b >= n) continue;   // ranges are checked by the row builders
    if (map) { a = map[a]; b = map[b]; }
    atomicAdd(cnt + a, 1ULL);
    atomicAdd(cnt + b, 1ULL);
  }
}

// Partition cost of a row: its raw nonzeros plus PART_ROW_COST.  Measured per rank on C5 (tools/
// dist_model.py): a row costs about as much as 6 nonzeros (its T-tile slot in the product plus the
// elementwise PCG step), so blocks of many short / isolated rows were the stragglers when balanced
// by nonzeros alone.
constexpr unsigned long long PART_ROW_COST = 6;
__global__ void k_fill_u64(int64_t n, unsigned long long v, unsigned long long* __restrict__ a) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    a[i] = v;
}

// key = ~count (ascending radix sort = descending count, stable: ties by ascending id)
__global__ void k_deg_keys(int64_t n, const unsigned long long* __restrict__ cnt, uint64_t* __restrict__ key,
                           int32_t* __restrict__ id) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    key[i] = ~(uint64_t)cnt[i];
    id[i] = (int32_t)i;
  }
}
__global__ void k_inverse_perm(int64_t n, const int32_t* __restrict__ p, int32_t* __restrict__ inv) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    inv[p[i]] = (int32_t)i;
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

// ================================================================ single-reduction distributed PCG
// Rows a8/e, SURVEY §8(a) "fusion floor" / §8(e): Jacobi-PCG in the Chronopoulos-Gear form, so one
// iteration needs ONE allreduce (3 KP doubles) instead of two, with the halo exchange of the
// preconditioned residual u overlapped with the on-rank part of the product:
//   E  k_cg_step      beta = gamma_i / gamma_{i-1}, alpha = gamma_i / (delta_i - beta gamma_i / alpha_{i-1})
//                     (alpha_0 = gamma_0 / delta_0), p = u + beta p, s = w + beta s, x += alpha p,
//                     r -= alpha s, u = dinv o r, local gamma' = r^T u, rho' = ||r||^2
//   H  halo(u)        pack + grouped ncclSend/ncclRecv on the comm stream          } concurrent
//   Sd t = A_own u    adjacency product over the OWN columns of every row          }
//   So t += A_gh u_gh over the ghost columns of the boundary rows (after H); both add u^T t
//   R  allreduce [gamma', u^T t, rho']  (3 KP doubles)  -> the next E on every rank, which forms
//      w = (I+L)u = r - t  and  delta = u^T w = gamma - u^T t   ((1+d) o u = r since u = dinv o r)
// w = (I+L)u, so s = (I+L)p and the recurrences are those of textbook PCG (same iterates in exact
// arithmetic).  The product needs no degree and no per-row boundary flag (no per-row dependent
// loads).  Columns of a k <= 4 batch are independent (per-column alpha, beta, mask) and padded
// to KP = 1, 2 or 4 (k = 3 -> 4).  Every decision is taken from allreduced scalars, identically on
// every rank; partial sums are formed and combined in a fixed order.  With NCCL the iteration is
// captured once into a CUDA graph of CG_UNROLL iterations (kernels exit early once converged) and
// replayed until the device `done` flag is set; the LOOPBACK transport runs the same kernels from the
// host (its exchanges are host-synchronous).

constexpr int CG_UNROLL = 4;

template <int KP> struct VT { using type = DVec<KP>; };
template <> struct VT<1> { using type = double; };
template <int KP>
__device__ __forceinline__ typename VT<KP>::type ldv(const double* p) {
  if constexpr (KP == 1) return *p;
  else return ld_vec<KP>(p);
}
template <int KP>
__device__ __forceinline__ void stv(double* p, const typename VT<KP>::type& v) {
  if constexpr (KP == 1) *p = v;
  else st_vec<KP>(p, v);
}
template <int KP>
__device__ __forceinline__ double cmp(const typename VT<KP>::type& v, int c) {
  if constexpr (KP == 1) return v;
  else return v.v[c];
}
template <int KP>
__device__ __forceinline__ void setc(typename VT<KP>::type& v, int c, double x) {
  if constexpr (KP == 1) v = x;
  else v.v[c] = x;
}

// The rank's local CSR split by column owner: own columns (< n_loc) of every row, and the ghost
// columns of the boundary rows (compact row list), each entry keeping its position order.
struct SplitCsr {
  int64_t nnz_d = 0, nnz_o = 0, n_bnd = 0;
  int64_t *rp_d = nullptr, *rp_o = nullptr;
  int32_t *col_d = nullptr, *col_o = nullptr, *rows_o = nullptr;
  void *w_d = nullptr, *w_o = nullptr;
  uint8_t* bnd = nullptr;
  Sched sd[2], so[2];             // [0] scalar engine (KP = 1), [1] vector engine (KP > 1)
  TileScratch tsd[2], tso[2];
  RowsPlan pd[2], po[2];          // the lean row kernel's plans of the two views (rows.cuh)
};

struct CgState {
  double gprev[KVMAX], aprev[KVMAX], tol2[KVMAX], rr[KVMAX], ss[KVMAX];
  double rtol2;
  int32_t active[KVMAX], conv[KVMAX], brk[KVMAX];
  int32_t first, iter, max_iter, done, k;
};

struct CgWs {
  int kp = 0;
  SplitCsr sp;
  bool split_built = false;
  double *u = nullptr, *w = nullptr, *p = nullptr, *s = nullptr, *x = nullptr, *r = nullptr;
  double *red = nullptr, *dpart = nullptr;   // red: [gamma | delta | rho | ss] x KVMAX
  CgState* cs = nullptr;
  double* part = nullptr;
  unsigned int* ticket = nullptr;
  int grid_elem = 0, grid_max = 0;
  cudaStream_t comm = nullptr, cap = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev0 = nullptr, ev1 = nullptr;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  int graph_k = 0;                           // the k the graph was captured for
};

static void free_ts(TileScratch& t) {
  dfree(t.block_part); dfree(t.long_part); dfree(t.chunk_acc); dfree(t.long_ticket); dfree(t.grid_ticket);
  t = TileScratch{};
}

static void free_cg(DistInfo* d) {
  CgWs* c = d->cg;
  if (!c) return;
  if (c->exec) cudaGraphExecDestroy(c->exec);
  if (c->graph) cudaGraphDestroy(c->graph);
  if (c->comm) cudaStreamDestroy(c->comm);
  if (c->cap) cudaStreamDestroy(c->cap);
  for (cudaEvent_t e : {c->ev_fork, c->ev_join, c->ev0, c->ev1})
    if (e) cudaEventDestroy(e);
  SplitCsr& sp = c->sp;
  dfree(sp.rp_d); dfree(sp.rp_o); dfree(sp.col_d); dfree(sp.col_o); dfree(sp.rows_o); dfree(sp.w_d); dfree(sp.w_o);
  dfree(sp.bnd);
  for (int f = 0; f < 2; ++f) {
    free_sched(sp.sd[f]); free_sched(sp.so[f]);
    rows_plan_free(sp.pd[f]); rows_plan_free(sp.po[f]);
    free_ts(sp.tsd[f]); free_ts(sp.tso[f]);
  }
  dfree(c->u); dfree(c->w); dfree(c->p); dfree(c->s); dfree(c->x); dfree(c->r);
  dfree(c->red); dfree(c->dpart); dfree(c->cs); dfree(c->part); dfree(c->ticket);
  delete c;
  d->cg = nullptr;
}

// per row: own / ghost column counts (warp per row: hub rows are long)
__global__ void k_split_count(int64_t n, const int64_t* __restrict__ rp, const int32_t* __restrict__ col, int64_t nl,
                              int64_t* __restrict__ cd, int64_t* __restrict__ co, uint8_t* __restrict__ bnd) {
  const int lane = threadIdx.x & 31;
  const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5, nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = wid; i < n; i += nw) {
    const int64_t rb = rp[i], re = rp[i + 1];
    int64_t own = 0;
    for (int64_t p = rb + lane; p < re; p += 32) own += col[p] < nl ? 1 : 0;
    for (int o = 16; o > 0; o >>= 1) own += __shfl_xor_sync(0xffffffffu, own, o);
    if (lane == 0) {
      cd[i] = own;
      co[i] = (re - rb) - own;
      bnd[i] = (re - rb) > own ? 1 : 0;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) { cd[n] = 0; co[n] = 0; }
}

// scatter each row's own / ghost entries (position order kept) into the two CSRs; warp per row,
// ballot prefix for the order within each 32-entry step
__global__ void k_split_scatter(int64_t n, const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                                const uint8_t* __restrict__ w, int wb, int64_t nl, const int64_t* __restrict__ pd,
                                const int64_t* __restrict__ po, int32_t* __restrict__ col_d, uint8_t* __restrict__ w_d,
                                int32_t* __restrict__ col_o, uint8_t* __restrict__ w_o) {
  const int lane = threadIdx.x & 31;
  const int64_t wid = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5, nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = wid; i < n; i += nw) {
    const int64_t rb = rp[i], re = rp[i + 1];
    int64_t od = pd[i], oo = po[i];
    for (int64_t b = rb; b < re; b += 32) {
      const int64_t p = b + lane;
      const bool in = p < re;
      const int32_t c = in ? col[p] : 0;
      const bool own = in && c < nl;
      const unsigned mo = __ballot_sync(0xffffffffu, own), mg = __ballot_sync(0xffffffffu, in && !own);
      const unsigned below = (1u << lane) - 1u;
      if (own) {
        const int64_t q = od + __popc(mo & below);
        col_d[q] = c;
        for (int t = 0; t < wb; ++t) w_d[q * wb + t] = w[p * wb + t];
      } else if (in) {
        const int64_t q = oo + __popc(mg & below);
        col_o[q] = c;
        for (int t = 0; t < wb; ++t) w_o[q * wb + t] = w[p * wb + t];
      }
      od += __popc(mo);
      oo += __popc(mg);
    }
  }
}

__global__ void k_rows_rp(int64_t nb, const int32_t* __restrict__ rows, const int64_t* __restrict__ po, int64_t tot,
                          int64_t* __restrict__ rp_o) {
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b <= nb; b += (int64_t)gridDim.x * blockDim.x)
    rp_o[b] = b < nb ? po[rows[b]] : tot;
}

static int wbytes_of(int wtype) { return wtype == FJ_W_UNIT ? 0 : wtype == FJ_W_U8 ? 1 : wtype == FJ_W_F32 ? 4 : 8; }

static fj_status alloc_ts(TileScratch& t, int grid_max, const Sched& S, int np, cudaStream_t st) {
  FJ_CK(dmalloc(&t.block_part, sizeof(double) * (size_t)grid_max * np, st));
  FJ_CK(dmalloc(&t.long_part, sizeof(double) * (size_t)std::max<int64_t>(S.n_long, 1) * np, st));
  FJ_CK(dmalloc(&t.chunk_acc, sizeof(double) * (size_t)std::max<int64_t>(S.n_long_chunks, 1) * np, st));
  FJ_CK(dmalloc(&t.long_ticket, sizeof(unsigned int) * (size_t)std::max<int64_t>(S.n_long, 1), st));
  FJ_CK(dmalloc(&t.grid_ticket, sizeof(unsigned int), st));
  FJ_CK(cudaMemsetAsync(t.long_ticket, 0, sizeof(unsigned int) * (size_t)std::max<int64_t>(S.n_long, 1), st));
  FJ_CK(cudaMemsetAsync(t.grid_ticket, 0, sizeof(unsigned int), st));
  return FJ_OK;
}

// the split CSR and the two schedules of engine flavour f (0 scalar, 1 vector)
static fj_status ensure_split(fj_graph* g, CgWs* c, int f, cudaStream_t st) {
  DistInfo* d = D(g);
  SplitCsr& sp = c->sp;
  const int64_t n = g->n, nl = d->n_loc;
  const int wb = wbytes_of(g->wtype);
  if (!c->split_built) {
    DevBuf<int64_t> cd, co, pd, po;
    FJ_TRY(cd.alloc(n + 1, st)); FJ_TRY(co.alloc(n + 1, st)); FJ_TRY(pd.alloc(n + 1, st)); FJ_TRY(po.alloc(n + 1, st));
    FJ_CK(dmalloc(&sp.bnd, (size_t)std::max<int64_t>(n, 1), st));
    const unsigned gb = (unsigned)std::min<int64_t>((n * 32 + 255) / 256, 65535);
    k_split_count<<<gb, 256, 0, st>>>(n, g->row_ptr, g->col, nl, cd.p, co.p, sp.bnd);
    FJ_CK_LAUNCH();
    FJ_TRY(cub_exclusive_sum(cd.p, pd.p, n + 1, st));
    FJ_TRY(cub_exclusive_sum(co.p, po.p, n + 1, st));
    int64_t tot[2];
    FJ_CK(cudaMemcpyAsync(&tot[0], pd.p + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    FJ_CK(cudaMemcpyAsync(&tot[1], po.p + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    FJ_CK(cudaStreamSynchronize(st));
    sp.nnz_d = tot[0];
    sp.nnz_o = tot[1];
    FJ_CK(dmalloc(&sp.rp_d, sizeof(int64_t) * (size_t)(n + 1), st));
    FJ_CK(cudaMemcpyAsync(sp.rp_d, pd.p, sizeof(int64_t) * (size_t)(n + 1), cudaMemcpyDeviceToDevice, st));
    FJ_CK(dmalloc(&sp.col_d, sizeof(int32_t) * (size_t)std::max<int64_t>(sp.nnz_d, 1), st));
    FJ_CK(dmalloc(&sp.col_o, sizeof(int32_t) * (size_t)std::max<int64_t>(sp.nnz_o, 1), st));
    if (wb) {
      FJ_CK(dmalloc(&sp.w_d, (size_t)wb * (size_t)std::max<int64_t>(sp.nnz_d, 1), st));
      FJ_CK(dmalloc(&sp.w_o, (size_t)wb * (size_t)std::max<int64_t>(sp.nnz_o, 1), st));
    }
    k_split_scatter<<<gb, 256, 0, st>>>(n, g->row_ptr, g->col, reinterpret_cast<const uint8_t*>(g->w), wb, nl, pd.p,
                                       po.p, sp.col_d, reinterpret_cast<uint8_t*>(sp.w_d), sp.col_o,
                                       reinterpret_cast<uint8_t*>(sp.w_o));
    FJ_CK_LAUNCH();
    // compact boundary rows
    FJ_CK(dmalloc(&sp.rows_o, sizeof(int32_t) * (size_t)std::max<int64_t>(n, 1), st));
    DevBuf<int32_t> nsel;
    FJ_TRY(nsel.alloc(1, st));
    FJ_TRY(cub_select_index(sp.bnd, sp.rows_o, nsel.p, n, st));
    int32_t nb = 0;
    FJ_CK(cudaMemcpyAsync(&nb, nsel.p, sizeof nb, cudaMemcpyDeviceToHost, st));
    FJ_CK(cudaStreamSynchronize(st));
    sp.n_bnd = nb;
    FJ_CK(dmalloc(&sp.rp_o, sizeof(int64_t) * (size_t)(nb + 1), st));
    k_rows_rp<<<(unsigned)std::min<int64_t>((nb + 256) / 256, 4096), 256, 0, st>>>(nb, sp.rows_o, po.p, sp.nnz_o,
                                                                                  sp.rp_o);
    FJ_CK_LAUNCH();
    FJ_CK(cudaStreamSynchronize(st));
    c->split_built = true;
  }
  if (!sp.sd[f].built) {
    const SchedParams P = f == 0 ? kSchedK1 : kSchedVec;
    fj_graph vd;                        // views: schedules depend only on (n, row_ptr)
    vd.n = n; vd.row_ptr = sp.rp_d;
    FJ_TRY(build_schedule(&vd, P, sp.sd[f], st));
    fj_graph vo;
    vo.n = sp.n_bnd; vo.row_ptr = sp.rp_o;
    FJ_TRY(build_schedule(&vo, P, sp.so[f], st));
    FJ_TRY(alloc_ts(sp.tsd[f], c->grid_max, sp.sd[f], KVMAX, st));
    FJ_TRY(alloc_ts(sp.tso[f], c->grid_max, sp.so[f], KVMAX, st));
    // the same two views on the lean row kernel (one pass each; FJ_ROWS=0 keeps the engine)
    FJ_TRY(rows_plan_build_csr(n, sp.nnz_d, sp.rp_d, sp.col_d, f == 0 ? 1 : 4, g->num_sms, sp.pd[f], st));
    FJ_TRY(rows_plan_build_csr(sp.n_bnd, sp.nnz_o, sp.rp_o, sp.col_o, f == 0 ? 1 : 4, g->num_sms, sp.po[f], st));
  }
  return FJ_OK;
}

// ---------------------------------------------------------------- the two product passes
template <int WT, int KP>
struct CgDiagOp {   // t = A u over the own columns of every row; u^T t
  using V = typename VT<KP>::type;
  static constexpr int ITEMS = KP == 1 ? fj::ITEMS : VEC_ITEMS;
  static constexpr int TILE_ROWS = KP == 1 ? fj::TILE_ROWS : VEC_TILE_ROWS;
  static constexpr int MIN_BLOCKS = engine_min_blocks<V>();
  static constexpr bool TMA = KP > 1;
  static constexpr int NA = KP, NP = KP;
  static constexpr bool NEEDS_XI = false;   // add() does not use x_i
  static __device__ __forceinline__ V vzero() {
    V r;
#pragma unroll
    for (int c = 0; c < KP; ++c) setc<KP>(r, c, 0.0);
    return r;
  }
  const double* __restrict__ u;
  double* __restrict__ w;   // t
  double* dot_out;
  const int32_t* done;
  __device__ __forceinline__ bool skip() const { return done && *(volatile const int32_t*)done; }
  __device__ __forceinline__ bool wants_xi() const { return true; }
  __device__ __forceinline__ V gather(int32_t j) const { return ldv<KP>(u + (int64_t)j * KP); }
  __device__ __forceinline__ V row_value(int64_t i) const { return ldv<KP>(u + i * KP); }
  __device__ __forceinline__ const V* xi_base() const { return reinterpret_cast<const V*>(u); }
  __device__ __forceinline__ void add(double (&a)[NA], double wgt, const V& xj, const V&) const {
#pragma unroll
    for (int c = 0; c < KP; ++c) a[c] = (WT == FJ_W_UNIT) ? a[c] + cmp<KP>(xj, c) : fma(wgt, cmp<KP>(xj, c), a[c]);
  }
  template <class P>
  __device__ __forceinline__ void finish_row(int64_t i, int64_t, const V& ui, const double (&a)[NA], P& part) const {
    V ti;
#pragma unroll
    for (int c = 0; c < KP; ++c) setc<KP>(ti, c, a[c]);
    stv<KP>(w + i * KP, ti);
#pragma unroll
    for (int c = 0; c < KP; ++c) part[c] = fma(cmp<KP>(ui, c), a[c], part[c]);
  }
  __device__ __forceinline__ void finalize(const double (&tot)[NP]) const {
#pragma unroll
    for (int c = 0; c < KP; ++c) dot_out[c] = tot[c];
  }
};

template <int WT, int KP>
struct CgOffOp {    // t_i += sum over the ghost columns of boundary row i; u^T (that part)
  using V = typename VT<KP>::type;
  static constexpr int ITEMS = KP == 1 ? fj::ITEMS : VEC_ITEMS;
  static constexpr int TILE_ROWS = KP == 1 ? fj::TILE_ROWS : VEC_TILE_ROWS;
  static constexpr int MIN_BLOCKS = engine_min_blocks<V>();
  static constexpr bool TMA = KP > 1;
  static constexpr int NA = KP, NP = KP;
  static constexpr bool NEEDS_XI = false;   // add() does not use x_i
  static __device__ __forceinline__ V vzero() { return CgDiagOp<WT, KP>::vzero(); }
  const double* __restrict__ u;
  double* __restrict__ w;
  const int32_t* __restrict__ rows;
  const double* dpart;   // the diag pass's (u, w) partial
  double* red;           // red[KP + c] <- local u^T t
  const int32_t* done;
  __device__ __forceinline__ bool skip() const { return done && *(volatile const int32_t*)done; }
  __device__ __forceinline__ bool wants_xi() const { return true; }
  __device__ __forceinline__ V gather(int32_t j) const { return ldv<KP>(u + (int64_t)j * KP); }
  __device__ __forceinline__ V row_value(int64_t b) const { return ldv<KP>(u + (int64_t)rows[b] * KP); }
  __device__ __forceinline__ const V* xi_base() const { return nullptr; }
  __device__ __forceinline__ void add(double (&a)[NA], double wgt, const V& xj, const V&) const {
#pragma unroll
    for (int c = 0; c < KP; ++c) a[c] = (WT == FJ_W_UNIT) ? a[c] + cmp<KP>(xj, c) : fma(wgt, cmp<KP>(xj, c), a[c]);
  }
  template <class P>
  __device__ __forceinline__ void finish_row(int64_t b, int64_t, const V& ui, const double (&a)[NA], P& part) const {
    const int64_t i = rows[b];
    V ti = ldv<KP>(w + i * KP);
#pragma unroll
    for (int c = 0; c < KP; ++c) setc<KP>(ti, c, cmp<KP>(ti, c) + a[c]);
    stv<KP>(w + i * KP, ti);
#pragma unroll
    for (int c = 0; c < KP; ++c) part[c] = fma(cmp<KP>(ui, c), a[c], part[c]);
  }
  __device__ __forceinline__ void finalize(const double (&tot)[NP]) const {
#pragma unroll
    for (int c = 0; c < KP; ++c) red[KP + c] = dpart[c] + tot[c];
  }
};

template <int WT, class Op>
static fj_status launch_view(const fj_graph* g, const Sched& S, const int64_t* rp, const int32_t* col, const void* w,
                             int64_t nrows, int64_t nnz, const TileScratch& ts, int grid_max, const Op& op,
                             cudaStream_t st) {
  static int occ = 0;
  if (occ == 0) {
    FJ_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, warp_kernel<WT, Op>, WTPB, 0));
    if (occ < 1) occ = 1;
  }
  TileSched t = make_sched(g, S);
  t.n = nrows; t.nnz = nnz; t.row_ptr = rp; t.col = col; t.w = w;
  int64_t grid = (int64_t)g->num_sms * occ;
  const int64_t need = (S.n_items + WPB - 1) / WPB;
  if (grid > need) grid = need > 0 ? need : 1;
  if (grid > grid_max) grid = grid_max;
  warp_kernel<WT, Op><<<(unsigned)grid, WTPB, 0, st>>>(t, op, ts);
  FJ_CK_LAUNCH();
  return FJ_OK;
}

// t = A v on the rank's rows (into c->w), red[KP..2KP) = local v^T t; the halo of v travels on the
// comm stream while the own-column pass runs (NCCL); LOOPBACK exchanges first, host-synchronously.
template <int KP>
static fj_status cg_product(fj_graph* g, CgWs* c, const double* u_in, cudaStream_t st, bool in_loop) {
  DistInfo* d = D(g);
  SplitCsr& sp = c->sp;
  constexpr int f = KP == 1 ? 0 : 1;
  double* u = c->u;
  if (u_in != u) FJ_CK(cudaMemcpyAsync(u, u_in, sizeof(double) * (size_t)d->n_loc * KP, cudaMemcpyDeviceToDevice, st));
  const bool overlap = d->comm->kind == 0 && d->comm->nranks > 1;
  if (overlap) {
    FJ_CK(cudaEventRecord(c->ev_fork, st));
    FJ_CK(cudaStreamWaitEvent(c->comm, c->ev_fork, 0));
    FJ_TRY(halo_exchange(d, u, c->comm, KP));
    FJ_CK(cudaEventRecord(c->ev_join, c->comm));
  } else {
    FJ_TRY(halo_exchange(d, u, st, KP));
  }
  const int32_t* done = in_loop ? &c->cs->done : nullptr;   // loop products exit once converged
  auto run = [&](auto wt) -> fj_status {
    constexpr int WT = decltype(wt)::value;
    CgDiagOp<WT, KP> od{u, c->w, c->dpart, done};
    if (sp.pd[f].mode != 0) FJ_TRY((rows_op<WT>(sp.pd[f], g->n, sp.col_d, sp.w_d, od, st)));
    else FJ_TRY((launch_view<WT>(g, sp.sd[f], sp.rp_d, sp.col_d, sp.w_d, g->n, sp.nnz_d, sp.tsd[f], c->grid_max, od, st)));
    if (overlap) FJ_CK(cudaStreamWaitEvent(st, c->ev_join, 0));
    CgOffOp<WT, KP> oo{u, c->w, sp.rows_o, c->dpart, c->red, done};
    if (sp.po[f].mode != 0) return rows_op<WT>(sp.po[f], sp.n_bnd, sp.col_o, sp.w_o, oo, st);
    return launch_view<WT>(g, sp.so[f], sp.rp_o, sp.col_o, sp.w_o, sp.n_bnd, sp.nnz_o, sp.tso[f], c->grid_max, oo, st);
  };
  switch (g->wtype) {
    case FJ_W_UNIT: return run(std::integral_constant<int, FJ_W_UNIT>());
    case FJ_W_U8: return run(std::integral_constant<int, FJ_W_U8>());
    case FJ_W_F32: return run(std::integral_constant<int, FJ_W_F32>());
    default: return run(std::integral_constant<int, FJ_W_F64>());
  }
}

// ---------------------------------------------------------------- elementwise kernels
template <int NPART>
__device__ __forceinline__ bool cg_reduce(double (&v)[NPART], double* part, unsigned int* ticket, double* s_red) {
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

// (re)start: r = s - (I+L) x = s - ((1+d) o x - t) with t = A x (restart), or r = s, x = 0;
// u = dinv o r; red[0..KP) = local r^T u, red[2KP..3KP) = ||r||^2, red[3KP..4KP) = ||s||^2.
// Rows are KP-wide vectors (one aligned load / store per row and array).
template <int KP>
__global__ void __launch_bounds__(VETB) k_cg_init(int64_t n, int k, const double* __restrict__ sv, int64_t ld, int c0,
                                                  const double* __restrict__ dinv, const double* __restrict__ deg,
                                                  const double* __restrict__ t, int restart, double* __restrict__ x,
                                                  double* __restrict__ r, double* __restrict__ u, double* red,
                                                  double* part, unsigned int* ticket) {
  using V = typename VT<KP>::type;
  __shared__ double s_red[3 * KP * VETB / 32];
  double v[3 * KP];
#pragma unroll
  for (int j = 0; j < 3 * KP; ++j) v[j] = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)VETB + threadIdx.x; i < n; i += (int64_t)gridDim.x * VETB) {
    const double di = dinv[i];
    V xv, tv, rv, uv;
    if (restart) { xv = ldv<KP>(x + i * KP); tv = ldv<KP>(t + i * KP); }
    const double dd = restart ? 1.0 + deg[i] : 0.0;
#pragma unroll
    for (int c = 0; c < KP; ++c) {
      const double si = c < k ? sv[i * ld + c0 + c] : 0.0;
      const double ri = restart ? si - fma(dd, cmp<KP>(xv, c), -cmp<KP>(tv, c)) : si;
      const double ui = di * ri;
      setc<KP>(rv, c, ri);
      setc<KP>(uv, c, ui);
      if (!restart) setc<KP>(xv, c, 0.0);
      v[c] = fma(ri, ui, v[c]);
      v[KP + c] = fma(ri, ri, v[KP + c]);
      v[2 * KP + c] = fma(si, si, v[2 * KP + c]);
    }
    if (!restart) stv<KP>(x + i * KP, xv);
    stv<KP>(r + i * KP, rv);
    stv<KP>(u + i * KP, uv);
  }
  if (cg_reduce<3 * KP>(v, part, ticket, s_red) && threadIdx.x == 0) {
#pragma unroll
    for (int c = 0; c < KP; ++c) { red[c] = v[c]; red[2 * KP + c] = v[KP + c]; red[3 * KP + c] = v[2 * KP + c]; }
    *ticket = 0u;
  }
}

__global__ void k_cg_state(CgState* cs, int k, double rtol, int max_iter) {
  for (int c = 0; c < KVMAX; ++c) {
    cs->active[c] = c < k ? 1 : 0;
    cs->conv[c] = 0;
    cs->brk[c] = 0;
    cs->gprev[c] = cs->aprev[c] = 0.0;
  }
  cs->rtol2 = rtol * rtol;
  cs->first = 1;
  cs->iter = 0;
  cs->max_iter = max_iter;
  cs->done = 0;
  cs->k = k;
}

// one Chronopoulos-Gear step from the allreduced [gamma | u^T t | rho (| ss on the first step)]:
// w = (I+L) u = r - t (t = A u from the product), delta = u^T w = gamma - u^T t
template <int KP>
__global__ void __launch_bounds__(VETB) k_cg_step(int64_t n, int k, const double* __restrict__ dinv,
                                                  double* __restrict__ u, const double* __restrict__ t,
                                                  double* __restrict__ p, double* __restrict__ s,
                                                  double* __restrict__ x, double* __restrict__ r, CgState* cs,
                                                  double* red, double* part, unsigned int* ticket) {
  using V = typename VT<KP>::type;
  __shared__ double s_red[2 * KP * VETB / 32];
  if (*(volatile int32_t*)&cs->done) return;
  const int first = cs->first;
  double al[KP], be[KP], g[KP], rr[KP], t2[KP];
  bool act[KP];
  bool any = false;
#pragma unroll
  for (int c = 0; c < KP; ++c) {
    act[c] = false;
    al[c] = be[c] = 0.0;
    g[c] = red[c];
    rr[c] = red[2 * KP + c];
    t2[c] = first ? cs->rtol2 * red[3 * KP + c] : cs->tol2[c];
    if (c < k && cs->active[c] && rr[c] > t2[c] && isfinite(rr[c])) {
      const double dl = g[c] - red[KP + c];
      const double b = first ? 0.0 : g[c] / cs->gprev[c];
      const double den = first ? dl : dl - b * g[c] / cs->aprev[c];
      if (den > 0.0 && isfinite(den) && isfinite(b)) {
        act[c] = true;
        al[c] = g[c] / den;
        be[c] = b;
      }
    }
    any |= act[c];
  }
  const int it = cs->iter;
  if (!any || it >= cs->max_iter) {   // identical in every block; block 0 records the outcome
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      for (int c = 0; c < k && c < KP; ++c) {
        if (first) { cs->tol2[c] = t2[c]; cs->ss[c] = red[3 * KP + c]; }
        cs->rr[c] = rr[c];
        if (cs->active[c]) {
          cs->conv[c] = rr[c] <= t2[c] ? 1 : 0;
          cs->brk[c] = (rr[c] > t2[c] && !act[c] && it < cs->max_iter) ? 1 : 0;
        }
        cs->active[c] = 0;
      }
      cs->done = 1;
    }
    return;
  }
  double v[2 * KP];
#pragma unroll
  for (int j = 0; j < 2 * KP; ++j) v[j] = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)VETB + threadIdx.x; i < n; i += (int64_t)gridDim.x * VETB) {
    const double di = dinv[i];
    V rv = ldv<KP>(r + i * KP), uv = ldv<KP>(u + i * KP);
    const V tv = ldv<KP>(t + i * KP);
    V pv, sv, xv = ldv<KP>(x + i * KP);
    if (!first) { pv = ldv<KP>(p + i * KP); sv = ldv<KP>(s + i * KP); }
#pragma unroll
    for (int c = 0; c < KP; ++c) {
      double ri = cmp<KP>(rv, c), ui = cmp<KP>(uv, c);
      const double wi = ri - cmp<KP>(tv, c);
      double pc = first ? ui : fma(be[c], cmp<KP>(pv, c), ui);
      double sc = first ? wi : fma(be[c], cmp<KP>(sv, c), wi);
      if (act[c]) {
        setc<KP>(xv, c, fma(al[c], pc, cmp<KP>(xv, c)));
        ri = fma(-al[c], sc, ri);
        ui = di * ri;
      } else if (!first) {   // frozen column: keep its p, s
        pc = cmp<KP>(pv, c);
        sc = cmp<KP>(sv, c);
      }
      setc<KP>(pv, c, pc);
      setc<KP>(sv, c, sc);
      setc<KP>(rv, c, ri);
      setc<KP>(uv, c, ui);
      v[c] = fma(ri, ui, v[c]);
      v[KP + c] = fma(ri, ri, v[KP + c]);
    }
    stv<KP>(p + i * KP, pv);
    stv<KP>(s + i * KP, sv);
    stv<KP>(x + i * KP, xv);
    stv<KP>(r + i * KP, rv);
    stv<KP>(u + i * KP, uv);
  }
  if (cg_reduce<2 * KP>(v, part, ticket, s_red) && threadIdx.x == 0) {
#pragma unroll
    for (int c = 0; c < KP; ++c) {
      if (c < k) {
        if (first) { cs->tol2[c] = t2[c]; cs->ss[c] = red[3 * KP + c]; }
        cs->rr[c] = rr[c];
        if (act[c]) {
          cs->gprev[c] = g[c];
          cs->aprev[c] = al[c];
        } else if (cs->active[c]) {   // left the batch this step
          cs->conv[c] = rr[c] <= t2[c] ? 1 : 0;
          cs->brk[c] = rr[c] > t2[c] ? 1 : 0;
          cs->active[c] = 0;
        }
      }
      red[c] = v[c];
      red[2 * KP + c] = v[KP + c];
    }
    cs->first = 0;
    cs->iter = it + 1;
    *ticket = 0u;
  }
}

// local ||s_c - (I+L) x_c||^2 = ||s - ((1+d) o x - t)||^2 (t = A x) -> red[0..KP)
template <int KP>
__global__ void __launch_bounds__(VETB) k_cg_resid(int64_t n, int k, const double* __restrict__ sv, int64_t ld, int c0,
                                                   const double* __restrict__ deg, const double* __restrict__ x,
                                                   const double* __restrict__ t, double* red, double* part,
                                                   unsigned int* ticket) {
  using V = typename VT<KP>::type;
  __shared__ double s_red[KP * VETB / 32];
  double v[KP];
#pragma unroll
  for (int c = 0; c < KP; ++c) v[c] = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)VETB + threadIdx.x; i < n; i += (int64_t)gridDim.x * VETB) {
    const V xv = ldv<KP>(x + i * KP), tv = ldv<KP>(t + i * KP);
    const double dd = 1.0 + deg[i];
#pragma unroll
    for (int c = 0; c < KP; ++c) {
      if (c < k) {
        const double e = sv[i * ld + c0 + c] - fma(dd, cmp<KP>(xv, c), -cmp<KP>(tv, c));
        v[c] = fma(e, e, v[c]);
      }
    }
  }
  if (cg_reduce<KP>(v, part, ticket, s_red) && threadIdx.x == 0) {
#pragma unroll
    for (int c = 0; c < KP; ++c) red[c] = v[c];
    *ticket = 0u;
  }
}

template <int KP>
__global__ void k_cg_pack(int64_t n, int k, const double* __restrict__ z, int64_t ld, int c0, double* __restrict__ x) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
#pragma unroll
    for (int c = 0; c < KP; ++c) x[i * KP + c] = c < k ? z[i * ld + c0 + c] : 0.0;
}
template <int KP>
__global__ void k_cg_unpack(int64_t n, int k, const double* __restrict__ x, double* __restrict__ z, int64_t ld, int c0) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
#pragma unroll
    for (int c = 0; c < KP; ++c)
      if (c < k) z[i * ld + c0 + c] = x[i * KP + c];
}

static fj_status get_cg(fj_graph* g, int kp, cudaStream_t st, CgWs** out) {
  DistInfo* d = D(g);
  if (d->cg && d->cg->kp != kp) {
    FJ_CK(cudaStreamSynchronize(st));
    SplitCsr keep = d->cg->sp;       // the split CSR does not depend on kp: keep it
    const bool built = d->cg->split_built;
    d->cg->sp = SplitCsr{};
    free_cg(d);
    d->cg = new CgWs();
    d->cg->sp = keep;
    d->cg->split_built = built;
  }
  if (!d->cg) d->cg = new CgWs();
  CgWs* c = d->cg;
  if (c->u) { *out = c; return FJ_OK; }
  c->kp = kp;
  const int64_t nl = d->n_loc, ne = nl + d->n_ghost;
  c->grid_max = g->num_sms * (2048 / WTPB);
  int64_t ge = (int64_t)g->num_sms * (2048 / VETB);
  const int64_t need = (nl + VETB - 1) / VETB;
  if (ge > need) ge = need > 0 ? need : 1;
  c->grid_elem = (int)ge;
  FJ_CK(dmalloc(&c->u, sizeof(double) * (size_t)std::max<int64_t>(ne * kp, 1), st));
  for (double** b : {&c->w, &c->p, &c->s, &c->x, &c->r})
    FJ_CK(dmalloc(b, sizeof(double) * (size_t)std::max<int64_t>(nl * kp, 1), st));
  FJ_CK(dmalloc(&c->red, sizeof(double) * 4 * KVMAX, st));
  FJ_CK(dmalloc(&c->dpart, sizeof(double) * KVMAX, st));
  FJ_CK(dmalloc(&c->cs, sizeof(CgState), st));
  FJ_CK(cudaMemsetAsync(c->cs, 0, sizeof(CgState), st));
  FJ_CK(dmalloc(&c->part, sizeof(double) * (size_t)ge * 3 * KVMAX, st));
  FJ_CK(dmalloc(&c->ticket, sizeof(unsigned int), st));
  FJ_CK(cudaMemsetAsync(c->ticket, 0, sizeof(unsigned int), st));
  if (!c->comm) FJ_CK(cudaStreamCreateWithFlags(&c->comm, cudaStreamNonBlocking));
  if (!c->cap) FJ_CK(cudaStreamCreateWithFlags(&c->cap, cudaStreamNonBlocking));
  for (cudaEvent_t* e : {&c->ev_fork, &c->ev_join})
    if (!*e) FJ_CK(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
  for (cudaEvent_t* e : {&c->ev0, &c->ev1})
    if (!*e) FJ_CK(cudaEventCreate(e));
  FJ_TRY(ensure_split(g, c, kp == 1 ? 0 : 1, st));
  *out = c;
  return FJ_OK;
}

// one iteration: E, then the product of the new u (halo overlapped), then the single allreduce
template <int KP>
static fj_status cg_iteration(fj_graph* g, CgWs* c, int k, cudaStream_t st) {
  DistInfo* d = D(g);
  k_cg_step<KP><<<c->grid_elem, VETB, 0, st>>>(d->n_loc, k, g->dinv, c->u, c->w, c->p, c->s, c->x, c->r, c->cs,
                                               c->red, c->part, c->ticket);
  FJ_CK_LAUNCH();
  FJ_TRY(cg_product<KP>(g, c, c->u, st, true));
  FJ_TRY(allreduce(d, c->red, 3 * KP, RED_SUM, st));
  return FJ_OK;
}

template <int KP>
static fj_status build_cg_graph(fj_graph* g, CgWs* c, int k) {
  if (c->exec) return FJ_OK;
  FJ_CK(cudaStreamBeginCapture(c->cap, cudaStreamCaptureModeThreadLocal));
  g_capturing = true;
  fj_status s = FJ_OK;
  for (int u = 0; u < CG_UNROLL && s == FJ_OK; ++u) s = cg_iteration<KP>(g, c, k, c->cap);
  g_capturing = false;
  cudaGraph_t gr = nullptr;
  cudaError_t e = cudaStreamEndCapture(c->cap, &gr);
  FJ_TRY(s);
  FJ_CK(e);
  c->graph = gr;
  FJ_CK(cudaGraphInstantiate(&c->exec, gr, 0));
  return FJ_OK;
}

template <int KP>
static fj_status dist_cg_t(fj_graph* g, int k, const double* sv, double* z, int64_t ld, int c0, const fj_solve_opts& o,
                           int warm, fj_solve_report* rep, cudaStream_t st) {
  DistInfo* d = D(g);
  CgWs* c = nullptr;
  FJ_TRY(get_cg(g, KP, st, &c));
  const int64_t nl = d->n_loc;
  const unsigned cb = (unsigned)std::min<int64_t>((nl + 255) / 256, 8192);
  const bool graph = o.use_cuda_graph && d->comm->kind == 0;
  if (graph) {
    if (c->exec && c->graph_k != k) {
      cudaGraphExecDestroy(c->exec); cudaGraphDestroy(c->graph);
      c->exec = nullptr; c->graph = nullptr;
    }
    FJ_TRY(build_cg_graph<KP>(g, c, k));
    c->graph_k = k;
  }
  CgState h{};
  std::vector<double> res2(KP, 0.0);
  int restarts = 0, total = 0;
  bool first = true;
  for (;;) {
    const bool restart = !first || warm;
    if (restart) {   // t = A x (x from z on a warm start); k_cg_init forms (I+L) x = (1+d) o x - t
      if (first) { k_cg_pack<KP><<<cb, 256, 0, st>>>(nl, k, z, ld, c0, c->x); FJ_CK_LAUNCH(); }
      FJ_TRY(cg_product<KP>(g, c, c->x, st, false));
    }
    const int budget = std::max(0, o.max_iter - total);
    FJ_CK(cudaEventRecord(c->ev0, st));
    k_cg_state<<<1, 1, 0, st>>>(c->cs, k, o.rtol, budget);
    FJ_CK_LAUNCH();
    k_cg_init<KP><<<c->grid_elem, VETB, 0, st>>>(nl, k, sv, ld, c0, g->dinv, g->deg, c->w, restart ? 1 : 0, c->x,
                                                 c->r, c->u, c->red, c->part, c->ticket);
    FJ_CK_LAUNCH();
    FJ_TRY(cg_product<KP>(g, c, c->u, st, false));    // t = A u, u^T t
    FJ_TRY(allreduce(d, c->red, 4 * KP, RED_SUM, st));
    first = false;
    for (;;) {
      if (graph) {
        FJ_CK(cudaGraphLaunch(c->exec, st));
      } else {
        for (int u = 0; u < CG_UNROLL; ++u) FJ_TRY(cg_iteration<KP>(g, c, k, st));
      }
      if (graph) {
        constexpr int f = KP == 1 ? 0 : 1;
        const int per_it = 1 + rows_op_launches(c->sp.pd[f]) + rows_op_launches(c->sp.po[f]) +
                           (d->comm->nranks > 1 && d->n_send > 0 ? 1 : 0);
        count_launch((int64_t)CG_UNROLL * per_it);
      }
      FJ_CK(cudaMemcpyAsync(&h, c->cs, sizeof h, cudaMemcpyDeviceToHost, st));
      FJ_CK(cudaStreamSynchronize(st));
      if (h.done) break;
    }
    FJ_CK(cudaEventRecord(c->ev1, st));
    // true residual: t = A x (same product), then ||s - ((1+d) o x - t)||^2 per column, allreduced
    FJ_TRY(cg_product<KP>(g, c, c->x, st, false));
    k_cg_resid<KP><<<c->grid_elem, VETB, 0, st>>>(nl, k, sv, ld, c0, g->deg, c->x, c->w, c->red + 3 * KVMAX,
                                                  c->part, c->ticket);
    FJ_CK_LAUNCH();
    FJ_TRY(allreduce(d, c->red + 3 * KVMAX, KP, RED_SUM, st));
    FJ_CK(cudaMemcpyAsync(res2.data(), c->red + 3 * KVMAX, sizeof(double) * KP, cudaMemcpyDeviceToHost, st));
    FJ_CK(cudaStreamSynchronize(st));
    float lms = 0.f;
    cudaEventElapsedTime(&lms, c->ev0, c->ev1);
    total += h.iter;
    if (rep) { rep->ms_loop += lms; rep->iterations_total += (int64_t)h.iter * k; }
    bool ok = true, brk = false;
    for (int j = 0; j < k; ++j) {
      if (res2[j] > h.tol2[j]) ok = false;
      if (h.brk[j]) brk = true;
    }
    if (ok || restarts >= o.max_restarts || total >= o.max_iter || brk) break;
    ++restarts;
  }
  k_cg_unpack<KP><<<cb, 256, 0, st>>>(nl, k, c->x, z, ld, c0);
  FJ_CK_LAUNCH();
  bool converged = true;
  double worst_true = 0.0, worst_rec = 0.0;
  for (int j = 0; j < k; ++j) {
    if (res2[j] > h.tol2[j]) converged = false;
    if (h.ss[j] > 0) {
      worst_true = std::max(worst_true, std::sqrt(res2[j] / h.ss[j]));
      worst_rec = std::max(worst_rec, std::sqrt(h.rr[j] / h.ss[j]));
    }
  }
  if (rep) {
    rep->iterations = std::max(rep->iterations, total);
    rep->restarts = std::max(rep->restarts, restarts);
    if (k > 1) rep->batch_k = k;
    rep->rel_res_recursive = std::max(rep->rel_res_recursive, worst_rec);
    rep->rel_res_true = std::isnan(rep->rel_res_true) ? worst_true : std::max(rep->rel_res_true, worst_true);
    if (!converged) rep->converged = 0;
  }
  return converged ? FJ_OK : fail(FJ_E_NO_CONVERGENCE, "distributed PCG did not reach rtol on the true residual");
}

// columns [c0, c0 + k) of the row-major [n_loc][ld] slices s, z; 1 <= k <= 4
fj_status dist_solve_cg(fj_graph* g, int k, const double* s, double* z, int64_t ld, int c0, const fj_solve_opts& o,
                        int warm, fj_solve_report* rep, cudaStream_t st) {
  if (k < 1 || k > KVMAX) return fail(FJ_E_INTERNAL, "dist_solve_cg: 1 <= k <= 4");
  if (k == 1) return dist_cg_t<1>(g, k, s, z, ld, c0, o, warm, rep, st);
  if (k == 2) return dist_cg_t<2>(g, k, s, z, ld, c0, o, warm, rep, st);
  return dist_cg_t<4>(g, k, s, z, ld, c0, o, warm, rep, st);
}

bool is_dist(const fj_graph* g) { return g->dist != nullptr; }
int64_t dist_n_ghost(const fj_graph* g) { return g->dist ? D(g)->n_ghost : 0; }
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
  free_cg(d);
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

static fj_status partition_rows(int64_t n, int64_t m, const int32_t* u, const int32_t* v, const int32_t* map,
                                int nranks, int64_t* bounds_host, void* stream) {
  if (n < 1 || n >= INT32_MAX || m < 0 || nranks < 1 || !bounds_host || (m > 0 && (!u || !v)))
    return fail(FJ_E_INVALID_ARG, "bad partition arguments");
  cudaStream_t st = S(stream);
  DevBuf<unsigned long long> cnt, pre;
  DevBuf<int64_t> b;
  FJ_TRY(cnt.alloc(n + 1, st));
  FJ_TRY(pre.alloc(n + 1, st));
  FJ_TRY(b.alloc(nranks + 1, st));
  k_fill_u64<<<(unsigned)std::min<int64_t>((n + 256) / 256, 8192), 256, 0, st>>>(n, PART_ROW_COST, cnt.p);
  FJ_CK_LAUNCH();
  FJ_CK(cudaMemsetAsync(cnt.p + n, 0, sizeof(unsigned long long), st));
  if (m > 0) {
    k_degree_hist<<<(unsigned)std::min<int64_t>((m + 255) / 256, 8192), 256, 0, st>>>(m, n, u, v, map, cnt.p);
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

fj_status fj_partition_rows(int64_t n, int64_t m, const int32_t* u, const int32_t* v, int nranks, int64_t* bounds_host,
                            void* stream) {
  FJ_RANGE("fj_partition_rows");
  return partition_rows(n, m, u, v, nullptr, nranks, bounds_host, stream);
}

fj_status fj_partition_rows_relabelled(int64_t n, int64_t m, const int32_t* u, const int32_t* v, const int32_t* old2new,
                                       int nranks, int64_t* bounds_host, void* stream) {
  if (!old2new) return fail(FJ_E_INVALID_ARG, "old2new is NULL");
  return partition_rows(n, m, u, v, old2new, nranks, bounds_host, stream);
}

fj_status fj_edge_degree_order(int64_t n, int64_t m, const int32_t* u, const int32_t* v, int32_t* new2old,
                               int32_t* old2new, void* stream) {
  FJ_RANGE("fj_edge_degree_order");
  if (n < 1 || n >= INT32_MAX || m < 0 || !new2old || !old2new || (m > 0 && (!u || !v)))
    return fail(FJ_E_INVALID_ARG, "bad degree-order arguments");
  cudaStream_t st = S(stream);
  DevBuf<unsigned long long> cnt;
  DevBuf<uint64_t> key, key2;
  DevBuf<int32_t> id;
  FJ_TRY(cnt.alloc(n, st)); FJ_TRY(key.alloc(n, st)); FJ_TRY(key2.alloc(n, st)); FJ_TRY(id.alloc(n, st));
  FJ_CK(cudaMemsetAsync(cnt.p, 0, sizeof(unsigned long long) * n, st));
  if (m > 0) {
    k_degree_hist<<<(unsigned)std::min<int64_t>((m + 255) / 256, 8192), 256, 0, st>>>(m, n, u, v, nullptr, cnt.p);
    FJ_CK_LAUNCH();
  }
  const unsigned gb = (unsigned)std::min<int64_t>((n + 255) / 256, 8192);
  k_deg_keys<<<gb, 256, 0, st>>>(n, cnt.p, key.p, id.p);
  FJ_CK_LAUNCH();
  size_t bytes = 0;
  FJ_CK(cub::DeviceRadixSort::SortPairs(nullptr, bytes, key.p, key2.p, id.p, new2old, n, 0, 64, st));
  {
    DevBuf<uint8_t> tmp;
    FJ_TRY(tmp.alloc((int64_t)bytes, st));
    FJ_CK(cub::DeviceRadixSort::SortPairs(tmp.p, bytes, key.p, key2.p, id.p, new2old, n, 0, 64, st));
    count_cub();
  }
  k_inverse_perm<<<gb, 256, 0, st>>>(n, new2old, old2new);
  FJ_CK_LAUNCH();
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
  FJ_RANGE("fj_graph_create_dist");
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

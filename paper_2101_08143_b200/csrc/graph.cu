// graph.cu — graph handle (row a2): validation, weighted degrees d_i = sum_j w_ij,
// Jacobi diagonal 1/(1+d_i), statistics (P:L86 w_min/w_max) and the tile-engine schedule.
#include <cub/cub.cuh>
#include <atomic>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <unordered_map>
#include <vector>

#include "common.cuh"
#include "tiles.cuh"
#include "workspace.cuh"

namespace fj {

thread_local std::string g_last_error;
thread_local bool g_capturing = false;
static std::atomic<int64_t> g_launches{0}, g_cub{0};
void count_launch(int64_t n) { g_launches += n; }

int batch_min_k() {
  static const int v = [] {
    const char* e = getenv("FJ_BATCH_MIN_K");
    return e ? std::max(2, atoi(e)) : 2;
  }();
  return v;
}

int l2_hint() {
  static const int v = [] {
    const char* e = getenv("FJ_L2_HINT");
    return e ? atoi(e) : 0;
  }();
  return v;
}

int vec_pad3() {
  static const int v = [] {
    const char* e = getenv("FJ_VEC_PAD");
    return (e && atoi(e) == 0) ? 3 : 4;
  }();
  return v;
}

void phase_tick(const char* label, cudaStream_t st) {
  static const bool on = getenv("FJ_TIMING") != nullptr;
  if (!on) return;
  static std::chrono::steady_clock::time_point last = std::chrono::steady_clock::now();
  cudaStreamSynchronize(st);
  auto now = std::chrono::steady_clock::now();
  fprintf(stderr, "[fj] %-28s %9.3f ms\n", label,
          std::chrono::duration<double, std::milli>(now - last).count());
  last = now;
}

// ---------------------------------------------------------------- allocator hook (fj_set_allocator)
namespace {
struct UserAlloc {
  fj_alloc_fn alloc = nullptr;
  fj_free_fn free = nullptr;
  void* ctx = nullptr;
};
struct AllocRec {
  UserAlloc a;
  size_t bytes;
};
std::mutex g_alloc_mu;
UserAlloc g_user;                                  // installed allocator (alloc == nullptr: pool)
std::unordered_map<void*, AllocRec> g_user_live;   // user-allocated blocks -> the allocator to return them to
}  // namespace

cudaError_t dmalloc_raw(void** p, size_t bytes, cudaStream_t st) {
  UserAlloc a;
  {
    std::lock_guard<std::mutex> lk(g_alloc_mu);
    a = g_user;
  }
  if (a.alloc) {
    void* q = a.alloc(bytes, reinterpret_cast<void*>(st), a.ctx);
    if (!q) return cudaErrorMemoryAllocation;
    std::lock_guard<std::mutex> lk(g_alloc_mu);
    g_user_live[q] = AllocRec{a, bytes};
    *p = q;
    return cudaSuccess;
  }
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  return cudaMallocFromPoolAsync(p, bytes, lib_pool(dev), st);
}

void dfree_on(void* p, cudaStream_t st) {
  if (!p) return;
  AllocRec rec{};
  bool user = false;
  {
    std::lock_guard<std::mutex> lk(g_alloc_mu);
    auto it = g_user_live.find(p);
    if (it != g_user_live.end()) {
      rec = it->second;
      user = true;
      g_user_live.erase(it);
    }
  }
  if (!user) {
    cudaFreeAsync(p, st);
    return;
  }
  cudaStreamSynchronize(st);   // the user's free is not stream-ordered: drain the work using p
  rec.a.free(p, rec.bytes, reinterpret_cast<void*>(st), rec.a.ctx);
}

cudaMemPool_t lib_pool(int device) {
  static std::mutex mu;
  static cudaMemPool_t pools[64] = {};
  std::lock_guard<std::mutex> lk(mu);
  if (device < 0 || device >= 64) device = 0;
  if (!pools[device]) {
    cudaMemPoolProps props;
    memset(&props, 0, sizeof props);
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = device;
    if (cudaMemPoolCreate(&pools[device], &props) != cudaSuccess) {
      cudaDeviceGetDefaultMemPool(&pools[device], device);
    }
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pools[device], cudaMemPoolAttrReleaseThreshold, &thr);
  }
  return pools[device];
}
void count_cub(int64_t n) { g_cub += n; }

void set_error(const std::string& msg) { g_last_error = msg; }

fj_status fail(fj_status st, const std::string& msg) {
  g_last_error = msg;
  return st;
}

fj_status cuda_fail(cudaError_t e, const char* what, const char* file, int line) {
  char buf[512];
  snprintf(buf, sizeof buf, "CUDA error %d (%s) in %s at %s:%d", (int)e, cudaGetErrorString(e), what,
           file, line);
  g_last_error = buf;
  if (e == cudaErrorMemoryAllocation) return FJ_E_OOM;
  return FJ_E_CUDA;
}

// ---------------------------------------------------------------- stats / degree kernel
struct GStats {
  unsigned long long deg_max;
  unsigned long long dmax_bits;   // positive doubles order like their bit patterns
  unsigned long long wmin_bits;
  unsigned long long wmax_bits;
  unsigned long long n_isolated;
  unsigned int bad_flags;         // validation: 1 not-simple, 2 asymmetric, 4 bad weight
};

__device__ __forceinline__ unsigned long long dbits(double x) {
  return (unsigned long long)__double_as_longlong(x);
}

constexpr int64_t kDegLong = 32;   // u8 rows longer than this are summed by a whole warp

// Long rows of an integer-weighted graph: one warp per row; the integer sum is exact in any order,
// so the degree is bit-identical to the ascending-column sum of k_degree and of the oracle.
__global__ void k_degree_long_u8(int64_t n, const int64_t* __restrict__ rp, const uint8_t* __restrict__ w,
                                 double* __restrict__ deg, double* __restrict__ dinv, GStats* st) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t r0 = ((int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 32; r0 < n; r0 += nw * 32) {
    const int64_t i = r0 + lane;
    const int64_t len = i < n ? rp[i + 1] - rp[i] : 0;
    unsigned longs = __ballot_sync(0xffffffffu, len > kDegLong);
    while (longs) {
      const int t = __ffs(longs) - 1;
      longs &= longs - 1;
      const int64_t row = r0 + t;
      const int64_t b = rp[row], e = rp[row + 1];
      unsigned long long s = 0;
      unsigned mn = 255, mx = 0;
      for (int64_t p = b + lane; p < e; p += 32) {
        const unsigned x = w[p];
        s += x;
        mn = min(mn, x);
        mx = max(mx, x);
      }
      for (int o = 16; o > 0; o >>= 1) {
        s += __shfl_xor_sync(0xffffffffu, s, o);
        mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      }
      if (lane == 0) {
        const double d = (double)s;
        deg[row] = d;
        dinv[row] = 1.0 / (1.0 + d);
        atomicMax(&st->dmax_bits, dbits(d));
        atomicMin(&st->wmin_bits, dbits((double)mn));
        atomicMax(&st->wmax_bits, dbits((double)mx));
      }
    }
  }
}

template <int WT>
__global__ void k_degree(int64_t n, const int64_t* __restrict__ rp, const void* __restrict__ w,
                         double* __restrict__ deg, double* __restrict__ dinv, GStats* st) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t len = 0;
  double d = 0.0, wmn = INFINITY, wmx = 0.0;
  if (i < n) {
    const int64_t b = rp[i], e = rp[i + 1];
    len = e - b;
    if (WT == FJ_W_UNIT) {
      d = (double)len;
      if (len) { wmn = 1.0; wmx = 1.0; }
    } else if (WT == FJ_W_U8 && len > kDegLong) {
      // integer weights: the sum is exact in any order -> long rows go to k_degree_long (a warp each)
    } else {
      for (int64_t p = b; p < e; ++p) {   // ascending column order: bit-exact with the oracle
        const double x = WeightT<WT>::get(w, p);
        d += x;
        wmn = fmin(wmn, x);
        wmx = fmax(wmx, x);
      }
    }
    if (!(WT == FJ_W_U8 && len > kDegLong)) {
      deg[i] = d;
      dinv[i] = 1.0 / (1.0 + d);   // IEEE division (no fast-math)
    }
  }
  // warp-aggregated statistics
  const unsigned iso = __ballot_sync(0xffffffffu, i < n && len == 0);
  unsigned long long lm = (unsigned long long)len;
  unsigned long long dm = dbits(d);
  unsigned long long mn = dbits(wmn > 0 && wmn < INFINITY ? wmn : INFINITY);
  unsigned long long mx = dbits(wmx);
  for (int o = 16; o > 0; o >>= 1) {
    lm = max(lm, __shfl_xor_sync(0xffffffffu, lm, o));
    dm = max(dm, __shfl_xor_sync(0xffffffffu, dm, o));
    mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(&st->deg_max, lm);
    atomicMax(&st->dmax_bits, dm);
    atomicMin(&st->wmin_bits, mn);
    atomicMax(&st->wmax_bits, mx);
    if (iso) atomicAdd(&st->n_isolated, (unsigned long long)__popc(iso));
  }
}

// Validation (P:L86 simple graph, w > 0; P:L88 symmetric adjacency): one thread per row.
template <int WT>
__global__ void k_validate(int64_t n, const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                           const void* __restrict__ w, GStats* st) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  unsigned flags = 0;
  const int64_t b = rp[i], e = rp[i + 1];
  if (e < b) flags |= 1;
  int64_t prev = -1;
  for (int64_t p = b; p < e && !(flags & 1); ++p) {
    const int64_t j = col[p];
    if (j < 0 || j >= n || j == i || j <= prev) { flags |= 1; break; }
    prev = j;
    const double x = WeightT<WT>::get(w, p);
    if (!(x > 0.0) || !isfinite(x)) flags |= 4;
    // mirror entry (j, i) with the same weight: binary search in row j
    int64_t lo = rp[j], hi = rp[j + 1];
    bool found = false;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      const int32_t c = col[mid];
      if (c == i) { found = (WeightT<WT>::get(w, mid) == x); break; }
      if (c < i) lo = mid + 1; else hi = mid;
    }
    if (!found) flags |= 2;
  }
  if (flags) atomicOr(&st->bad_flags, flags);
}

__global__ void k_check_rowptr(int64_t n, int64_t nnz, const int64_t* rp, GStats* st) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i > n) return;
  const int64_t v = rp[i];
  bool bad = (v < 0 || v > nnz) || (i == 0 && v != 0) || (i == n && v != nnz) ||
             (i > 0 && rp[i - 1] > v);
  if (bad) atomicOr(&st->bad_flags, 1u);
}

static inline double bits2d(unsigned long long b) { double d; memcpy(&d, &b, sizeof d); return d; }
static inline unsigned nblk(int64_t n, int t = 256) { return (unsigned)((n + t - 1) / t); }

template <int WT>
static fj_status launch_degree(fj_graph* g, GStats* st_d, int validate, cudaStream_t st) {
  if (validate) {
    k_check_rowptr<<<nblk(g->n + 1), 256, 0, st>>>(g->n, g->nnz, g->row_ptr, st_d);
    FJ_CK_LAUNCH();
    GStats h;
    FJ_CK(cudaMemcpyAsync(&h, st_d, sizeof h, cudaMemcpyDeviceToHost, st));
    FJ_CK(cudaStreamSynchronize(st));
    if (h.bad_flags) return fail(FJ_E_NOT_SIMPLE, "row_ptr is not a valid CSR row pointer");
    k_validate<WT><<<nblk(g->n), 256, 0, st>>>(g->n, g->row_ptr, g->col, g->w, st_d);
    FJ_CK_LAUNCH();
  }
  k_degree<WT><<<nblk(g->n), 256, 0, st>>>(g->n, g->row_ptr, g->w, g->deg, g->dinv, st_d);
  FJ_CK_LAUNCH();
  if (WT == FJ_W_U8) {
    k_degree_long_u8<<<g->num_sms * 8, 256, 0, st>>>(g->n, g->row_ptr, reinterpret_cast<const uint8_t*>(g->w),
                                                     g->deg, g->dinv, st_d);
    FJ_CK_LAUNCH();
  }
  return FJ_OK;
}

}  // namespace fj

using namespace fj;

extern "C" {

int fj_abi_version(void) { return FJ_ABI_VERSION; }

int64_t fj_kernel_launches(int64_t* cub_launches) {
  if (cub_launches) *cub_launches = g_cub.load();
  return g_launches.load();
}

const char* fj_last_error(void) { return g_last_error.c_str(); }

const char* fj_status_str(int s) {
  switch (s) {
    case FJ_OK: return "FJ_OK";
    case FJ_E_INVALID_ARG: return "FJ_E_INVALID_ARG";
    case FJ_E_NOT_SIMPLE: return "FJ_E_NOT_SIMPLE";
    case FJ_E_ASYMMETRIC: return "FJ_E_ASYMMETRIC";
    case FJ_E_BAD_WEIGHT: return "FJ_E_BAD_WEIGHT";
    case FJ_E_NONFINITE_INPUT: return "FJ_E_NONFINITE_INPUT";
    case FJ_E_NO_CONVERGENCE: return "FJ_E_NO_CONVERGENCE";
    case FJ_E_CUDA: return "FJ_E_CUDA";
    case FJ_E_NCCL: return "FJ_E_NCCL";
    case FJ_E_OOM: return "FJ_E_OOM";
    case FJ_E_INTERNAL: return "FJ_E_INTERNAL";
    case FJ_E_UNSUPPORTED: return "FJ_E_UNSUPPORTED";
    default: return "FJ_E_UNKNOWN";
  }
}

void fj_default_solve_opts(fj_solve_opts* o) {
  if (!o) return;
  o->rtol = 1e-10;
  o->eps_target = 0.0;
  o->max_iter = 10000;
  o->max_restarts = 3;
  o->use_cuda_graph = 1;
  o->vertex_order = FJ_ORDER_NATURAL;
}

fj_status fj_graph_create(int64_t n, int64_t nnz, const int64_t* row_ptr, const int32_t* col, const void* w,
                          int wtype, int validate, void* stream, fj_graph** out) {
  FJ_RANGE("fj_graph_create");
  if (!out) return fail(FJ_E_INVALID_ARG, "out is NULL");
  *out = nullptr;
  if (n < 1 || n >= INT32_MAX) return fail(FJ_E_INVALID_ARG, "n must be in [1, 2^31-2]");
  if (nnz < 0 || !row_ptr || (nnz > 0 && !col)) return fail(FJ_E_INVALID_ARG, "bad CSR arrays");
  if (wtype < FJ_W_UNIT || wtype > FJ_W_F64) return fail(FJ_E_INVALID_ARG, "bad wtype");
  if (wtype != FJ_W_UNIT && nnz > 0 && !w) return fail(FJ_E_INVALID_ARG, "weights are NULL");
  cudaStream_t st = S(stream);
  fj_graph* g = new fj_graph();
  g->n = n; g->nnz = nnz; g->wtype = wtype; g->row_ptr = row_ptr; g->col = col;
  g->w = (wtype == FJ_W_UNIT) ? nullptr : w;
  auto cleanup = [&](fj_status s) { fj_graph_destroy(g); return s; };
  cudaError_t ce = cudaGetDevice(&g->device);
  if (ce != cudaSuccess) return cleanup(cuda_fail(ce, "cudaGetDevice", __FILE__, __LINE__));
  cudaDeviceGetAttribute(&g->num_sms, cudaDevAttrMultiProcessorCount, g->device);
  ce = dmalloc(&g->deg, sizeof(double) * n, st);
  if (ce == cudaSuccess) ce = dmalloc(&g->dinv, sizeof(double) * n, st);
  if (ce != cudaSuccess) return cleanup(cuda_fail(ce, "cudaMallocAsync", __FILE__, __LINE__));
  GStats* st_d = nullptr;
  ce = dmalloc(&st_d, sizeof(GStats), st);
  if (ce != cudaSuccess) return cleanup(cuda_fail(ce, "cudaMallocAsync", __FILE__, __LINE__));
  GStats init{};
  init.wmin_bits = (unsigned long long)0x7FF0000000000000ULL;  // +inf
  cudaMemcpyAsync(st_d, &init, sizeof init, cudaMemcpyHostToDevice, st);
  fj_status s = FJ_OK;
  switch (wtype) {
    case FJ_W_UNIT: s = launch_degree<FJ_W_UNIT>(g, st_d, validate, st); break;
    case FJ_W_U8: s = launch_degree<FJ_W_U8>(g, st_d, validate, st); break;
    case FJ_W_F32: s = launch_degree<FJ_W_F32>(g, st_d, validate, st); break;
    default: s = launch_degree<FJ_W_F64>(g, st_d, validate, st); break;
  }
  GStats h{};
  if (s == FJ_OK) {
    ce = cudaMemcpyAsync(&h, st_d, sizeof h, cudaMemcpyDeviceToHost, st);
    if (ce == cudaSuccess) ce = cudaStreamSynchronize(st);
    if (ce != cudaSuccess) s = cuda_fail(ce, "stats readback", __FILE__, __LINE__);
  }
  dfree_on(st_d, st);
  if (s != FJ_OK) return cleanup(s);
  if (validate && h.bad_flags) {
    if (h.bad_flags & 1) return cleanup(fail(FJ_E_NOT_SIMPLE, "CSR not simple: column out of range, self-loop, or columns not strictly ascending"));
    if (h.bad_flags & 4) return cleanup(fail(FJ_E_BAD_WEIGHT, "edge weight <= 0 or non-finite"));
    return cleanup(fail(FJ_E_ASYMMETRIC, "adjacency not symmetric: (i,j,w) without (j,i,w)"));
  }
  if (nnz % 2 != 0 && validate) return cleanup(fail(FJ_E_ASYMMETRIC, "odd nnz"));
  phase_tick("graph: degrees + stats", st);
  s = build_schedule(g, kSchedK1, g->s1, st);
  phase_tick("graph: k=1 schedule", st);
  if (s != FJ_OK) return cleanup(s);
  fj_graph_info_t& I = g->info;
  I.n = n; I.nnz = nnz; I.m = nnz / 2;
  I.n_isolated = (int64_t)h.n_isolated;
  I.deg_max = (int64_t)h.deg_max;
  I.d_max = bits2d(h.dmax_bits);
  I.w_min = nnz ? bits2d(h.wmin_bits) : 0.0;
  I.w_max = nnz ? bits2d(h.wmax_bits) : 0.0;
  I.n_tiles = g->s1.n_tiles; I.n_wrows = g->s1.n_wrows; I.n_long_rows = g->s1.n_long;
  I.n_long_chunks = g->s1.n_long_chunks;
  I.wtype = wtype;
  ce = cudaStreamSynchronize(st);
  if (ce != cudaSuccess) return cleanup(cuda_fail(ce, "graph create", __FILE__, __LINE__));
  *out = g;
  return FJ_OK;
}

fj_status fj_graph_info(const fj_graph* g, fj_graph_info_t* out) {
  if (!g || !out) return fail(FJ_E_INVALID_ARG, "null argument");
  *out = g->info;
  return FJ_OK;
}

fj_status fj_graph_degrees(const fj_graph* g, double* d, void* stream) {
  if (!g || !d) return fail(FJ_E_INVALID_ARG, "null argument");
  FJ_CK(cudaMemcpyAsync(d, g->deg, sizeof(double) * g->n, cudaMemcpyDeviceToDevice, S(stream)));
  return FJ_OK;
}

fj_status fj_set_allocator(fj_alloc_fn alloc, fj_free_fn free_fn, void* ctx) {
  if ((alloc == nullptr) != (free_fn == nullptr))
    return fail(FJ_E_INVALID_ARG, "fj_set_allocator: alloc and free must both be set or both be NULL");
  std::lock_guard<std::mutex> lk(g_alloc_mu);
  g_user.alloc = alloc;
  g_user.free = free_fn;
  g_user.ctx = ctx;
  return FJ_OK;
}

int64_t fj_allocator_live_blocks(void) {
  std::lock_guard<std::mutex> lk(g_alloc_mu);
  return (int64_t)g_user_live.size();
}

fj_status fj_graph_destroy(fj_graph* g) {
  if (!g) return FJ_OK;
  cudaDeviceSynchronize();
  free_solve_ws(g);
  free_quant_ws(g);
  free_batch_ws(g);
  free_vec_ws(g);
  free_dist(g);
  dfree(g->deg); dfree(g->dinv);
  free_sched(g->s1);
  free_sched(g->sb);
  free_sched(g->sv);
  delete g;
  return FJ_OK;
}

}  // extern "C"

// common.cuh — internal helpers of libfj (not part of the ABI).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <string>
#include <utility>
#include <cstdio>
#include <cmath>

#include "../../include/fj.h"
#include <nvtx3/nvToolsExt.h>

namespace fj {

// ---------------------------------------------------------------- errors
void set_error(const std::string& msg);
fj_status fail(fj_status st, const std::string& msg);
fj_status cuda_fail(cudaError_t e, const char* what, const char* file, int line);

#define FJ_CK(call)                                                            \
  do {                                                                         \
    cudaError_t _e = (call);                                                   \
    if (_e != cudaSuccess) return ::fj::cuda_fail(_e, #call, __FILE__, __LINE__); \
  } while (0)

#define FJ_TRY(call)                                                           \
  do {                                                                         \
    fj_status _s = (call);                                                     \
    if (_s != FJ_OK) return _s;                                                \
  } while (0)

// Device memory.  Default: a library-owned stream-ordered pool per device whose release threshold
// is unbounded, so repeated graph builds / solves reuse memory instead of re-mapping it.  With an
// allocator installed by fj_set_allocator (e.g. the torch caching allocator), every workspace
// allocation goes through it and is returned to it (graph.cu).
cudaMemPool_t lib_pool(int device);
cudaError_t dmalloc_raw(void** p, size_t bytes, cudaStream_t st);
// Free stream-ordered on `st`: pool memory by cudaFreeAsync; user-allocator memory after `st` has
// drained (the user's free is not stream-ordered).
void dfree_on(void* p, cudaStream_t st);
template <class T>
inline cudaError_t dmalloc(T** p, size_t bytes, cudaStream_t st) {
  return dmalloc_raw(reinterpret_cast<void**>(p), bytes, st);
}

// Free on the legacy stream (callers synchronise the device first); plain cudaFree on pool memory
// would hand it back to the OS and the next graph would re-map it.
inline void dfree(void* p) {
  if (p) dfree_on(p, 0);
}

// FJ_TIMING=1: host-side phase timestamps on stderr (diagnostics; synchronises the stream)
void phase_tick(const char* label, cudaStream_t st);

// Device-side invariant checks of the debug build (-DFJ_DEBUG_CHECKS; tools/sanitize_cases.py runs
// every engine with them, since compute-sanitizer is closed on this GPU pool): a failed check
// prints the condition and traps (the launch fails with an illegal-instruction error).
#ifdef FJ_DEBUG_CHECKS
#define FJ_DCHECK(c)                                                                   \
  do {                                                                                 \
    if (!(c)) {                                                                        \
      printf("FJ_DCHECK failed %s:%d: %s (block %d thread %d)\n", __FILE__, __LINE__, #c, \
             (int)blockIdx.x, (int)threadIdx.x);                                       \
      __trap();                                                                        \
    }                                                                                  \
  } while (0)
#else
#define FJ_DCHECK(c) \
  do {               \
  } while (0)
#endif

// NVTX range over a public entry point (visible in nsys / ncu --nvtx; header-only NVTX3, a no-op
// without a tool attached)
struct NvtxRange {
  explicit NvtxRange(const char* s) { nvtxRangePushA(s); }
  ~NvtxRange() { nvtxRangePop(); }
};
#define FJ_RANGE(name) ::fj::NvtxRange _fj_nvtx_range_(name)

// Programmatic dependent launch (PDL) between the kernels of a solver iteration: a kernel launched
// with pdl_launch() may start its blocks while its predecessor's last blocks drain; each such kernel
// calls pdl_prologue() first -- it allows its own successor to launch early, then waits until the
// predecessor grid has completed and its writes are visible.  Without the launch attribute both
// instructions are no-ops.  FJ_PDL=0 disables (A/B).
#ifndef FJ_PDL
#define FJ_PDL 1
#endif
__device__ __forceinline__ void pdl_prologue() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
}
template <class... KArgs, class... Args>
inline cudaError_t pdl_launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = FJ_PDL ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// kernel launch accounting (fj_kernel_launches)
void count_launch(int64_t n = 1);
void count_cub(int64_t n = 1);
extern thread_local bool g_capturing;

#define FJ_CK_LAUNCH()                                 \
  do {                                                 \
    FJ_CK(cudaGetLastError());                         \
    if (!::fj::g_capturing) ::fj::count_launch();      \
  } while (0)

// ---------------------------------------------------------------- constants
constexpr int MAXK = 64;
// k >= batch_min_k() columns are solved together (row a9): 2 <= k <= 4 on the warp-item engine with
// vector values (spmv_vec.cu), k > 4 on the warp-per-row engine (spmm.cu); fewer columns run the
// k = 1 path once per column.  FJ_BATCH_MIN_K overrides (tests).
int batch_min_k();
// row-engine knobs (FJ_L2_HINT; bit 1 disables the TMA tile prefetch, tiles.cuh)
int l2_hint();
// padded row width of the small-k engine for k = 3 (default 4; FJ_VEC_PAD=0: unpadded 3; spmv_vec.cu)
int vec_pad3();

// ---------------------------------------------------------------- device workspace per solve
struct SolveWs;   // pcg.cu
struct QuantWs;   // quantities.cu

// One work-item list of the row engine: items [0, n_long_chunks) are long-row chunks, then W rows,
// then T tiles (schedule.cu).
struct Sched {
  int64_t n_items = 0, n_tiles = 0, n_wrows = 0, n_long = 0, n_long_chunks = 0;
  void* items = nullptr;            // ItemMeta [n_items] (tiles.cuh)
  int32_t* long_nchunks = nullptr;  // [n_long]
  int32_t* long_item0 = nullptr;    // [n_long] item index of chunk 0
  int chunk = 0;                    // nonzeros per long-row chunk (= max W row length)
  bool built = false;
};
struct SchedParams {
  int trow_max;     // rows with <= trow_max nonzeros go to T tiles
  int t_units;      // merge-coordinate cut of T tiles
  int t_min_cost;   // minimum merge units charged per T row (caps rows per tile)
  int chunk;        // W rows up to chunk nonzeros; longer rows are cut in chunks of this size
};

}  // namespace fj

// The graph handle (borrowed CSR + derived arrays + schedule).
struct fj_graph {
  int device = 0;
  int64_t n = 0, nnz = 0;
  int wtype = FJ_W_UNIT;
  const int64_t* row_ptr = nullptr;
  const int32_t* col = nullptr;
  const void* w = nullptr;
  // derived (owned)
  double* deg = nullptr;        // weighted degree d_i            [n]
  double* dinv = nullptr;       // 1 / (1 + d_i)                  [n]
  // row-engine work-item lists (schedule.cu): s1 for k = 1 (tiles.cuh), sb for batched k (spmm.cu,
  // built on first use)
  fj::Sched s1, sb, sv;   // sv: vector engine (spmv_vec.cu, VEC_ITEMS per lane), built on first use
  fj_graph_info_t info{};
  int num_sms = 148;
  // caches
  fj::SolveWs* solve_ws = nullptr;
  fj::QuantWs* quant_ws = nullptr;
  void* batch_ws = nullptr;       // spmm.cu BatchWs (k > 4)
  void* vec_ws = nullptr;         // spmv_vec.cu VecWs (2 <= k <= 4)
  void* dist = nullptr;           // dist.cu DistInfo when this is one rank's row block
};

namespace fj {

inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// ---------------------------------------------------------------- weights
template <int WT> struct WeightT;
template <> struct WeightT<FJ_W_UNIT> {
  __device__ static __forceinline__ double get(const void*, int64_t) { return 1.0; }
};
template <> struct WeightT<FJ_W_U8> {
  __device__ static __forceinline__ double get(const void* w, int64_t p) {
    return (double)__ldg(reinterpret_cast<const uint8_t*>(w) + p);
  }
};
template <> struct WeightT<FJ_W_F32> {
  __device__ static __forceinline__ double get(const void* w, int64_t p) {
    return (double)__ldg(reinterpret_cast<const float*>(w) + p);
  }
};
template <> struct WeightT<FJ_W_F64> {
  __device__ static __forceinline__ double get(const void* w, int64_t p) {
    return __ldg(reinterpret_cast<const double*>(w) + p);
  }
};

// ---------------------------------------------------------------- deterministic reductions
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide sum of NP values per thread; result valid in thread 0.  Fixed tree -> deterministic.
template <int NP, int BLOCK>
__device__ __forceinline__ void block_sum(double (&v)[NP], double* smem /* >= NP*BLOCK/32 */) {
  constexpr int NW = BLOCK / 32;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int j = 0; j < NP; ++j) v[j] = warp_sum(v[j]);
  __syncthreads();
  if (lane == 0) {
#pragma unroll
    for (int j = 0; j < NP; ++j) smem[j * NW + wid] = v[j];
  }
  __syncthreads();
  if (wid == 0) {
#pragma unroll
    for (int j = 0; j < NP; ++j) {
      double x = lane < NW ? smem[j * NW + lane] : 0.0;
      v[j] = warp_sum(x);
    }
  }
  __syncthreads();
}

// "Last block" ticket: returns true in ALL threads of the block that arrives last.
__device__ __forceinline__ bool last_block_ticket(unsigned int* counter, unsigned int total) {
  __shared__ bool am_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int t = atomicAdd(counter, 1u);
    am_last = (t == total - 1);
  }
  __syncthreads();
  if (am_last) __threadfence();
  return am_last;
}

__device__ __forceinline__ double ld_cg(const double* p) { return __ldcg(p); }

// gather of one fp64 through the plain (coherent) global path
__device__ __forceinline__ double ld_plain(const double* p) {
  double r;
  asm volatile("ld.global.f64 %0, [%1];" : "=d"(r) : "l"(p));
  return r;
}

}  // namespace fj

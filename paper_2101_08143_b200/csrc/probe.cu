// probe.cu — measured denominator for the SpMV's real bound (DESIGN.md §6 "gather roofline").
//
// The (I+L)p product on these random graphs is bound by the rate of random 8..32-byte gathers
// (one L2 sector request each), not by HBM bytes.  fj_probe_gather measures the best rate this
// GPU sustains for the same access pattern with no row logic at all: an int32 index stream read
// once (coalesced, evict-first) and one gather of `width` doubles per index from an n_vec-row
// vector, 8 independent gathers in flight per thread, a fixed grid of #SMs x occupancy.  The
// ratio (SpMV nonzeros / s) / (probe gathers / s) is the fraction of that bound the engine reaches.
#include <vector>

#include "common.cuh"
#include "workspace.cuh"

namespace fj {

__device__ __forceinline__ uint32_t mix32(uint64_t x) {   // splitmix64 finaliser, low 32 bits
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return (uint32_t)(x ^ (x >> 31));
}

__global__ void k_probe_fill(int64_t n_vec, int64_t m, int width, double* __restrict__ x, int32_t* __restrict__ idx) {
  const int64_t T = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n_vec * width; i += T) x[i] = 1.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += T)
    idx[i] = (int32_t)(((uint64_t)mix32((uint64_t)i) * (uint64_t)n_vec) >> 32);
}

template <int W>
__device__ __forceinline__ double probe_ld(const double* p) {
  if (W == 1) {
    double r;
    asm volatile("ld.global.f64 %0, [%1];" : "=d"(r) : "l"(p));
    return r;
  } else if (W == 2) {
    double a, b;
    asm volatile("ld.global.v2.f64 {%0, %1}, [%2];" : "=d"(a), "=d"(b) : "l"(p));
    return a + b;
  } else {
    double a, b, c, d;
    asm volatile("ld.global.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p));
    return (a + b) + (c + d);
  }
}

template <int W>
__global__ void __launch_bounds__(256) k_probe_gather(int64_t m, const double* __restrict__ x,
                                                      const int32_t* __restrict__ idx, double* __restrict__ out) {
  constexpr int U = 8;
  const int64_t T = (int64_t)gridDim.x * blockDim.x;
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  double acc = 0.0;
  for (int64_t i = t; i < m; i += U * T) {
    int32_t j[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t q = i + u * T;
      if (q < m) {
        asm volatile("ld.global.cs.s32 %0, [%1];" : "=r"(j[u]) : "l"(idx + q));
      } else {
        j[u] = -1;
      }
    }
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = j[u] >= 0 ? probe_ld<W>(x + (int64_t)j[u] * W) : 0.0;
#pragma unroll
    for (int u = 0; u < U; ++u) acc += v[u];
  }
  out[t] = acc;
}

template <int W>
static fj_status run_probe(int64_t n_vec, int64_t m, int reps, double* rate, cudaStream_t st) {
  int dev = 0, sms = 0, occ = 0;
  FJ_CK(cudaGetDevice(&dev));
  FJ_CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  FJ_CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_probe_gather<W>, 256, 0));
  const int grid = sms * std::max(occ, 1);
  DevBuf<double> x, out;
  DevBuf<int32_t> idx;
  FJ_TRY(x.alloc(n_vec * W, st));
  FJ_TRY(idx.alloc(m, st));
  FJ_TRY(out.alloc((int64_t)grid * 256, st));
  k_probe_fill<<<sms * 8, 256, 0, st>>>(n_vec, m, W, x.p, idx.p);
  FJ_CK_LAUNCH();
  k_probe_gather<W><<<grid, 256, 0, st>>>(m, x.p, idx.p, out.p);   // warm: x resident in L2 if it fits
  FJ_CK_LAUNCH();
  cudaEvent_t e0, e1;
  FJ_CK(cudaEventCreate(&e0));
  FJ_CK(cudaEventCreate(&e1));
  FJ_CK(cudaEventRecord(e0, st));
  for (int r = 0; r < reps; ++r) {
    k_probe_gather<W><<<grid, 256, 0, st>>>(m, x.p, idx.p, out.p);
    FJ_CK_LAUNCH();
  }
  FJ_CK(cudaEventRecord(e1, st));
  FJ_CK(cudaEventSynchronize(e1));
  float ms = 0.f;
  FJ_CK(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  *rate = (double)m * reps / (ms * 1e-3);
  return FJ_OK;
}

}  // namespace fj

using namespace fj;

extern "C" fj_status fj_probe_gather(int64_t n_vec, int64_t m, int width, int reps, double* gathers_per_s,
                                     void* stream) {
  if (n_vec < 1 || n_vec > INT32_MAX || m < 1 || reps < 1 || !gathers_per_s)
    return fail(FJ_E_INVALID_ARG, "fj_probe_gather: n_vec in [1, 2^31), m >= 1, reps >= 1");
  cudaStream_t st = S(stream);
  switch (width) {
    case 1: return run_probe<1>(n_vec, m, reps, gathers_per_s, st);
    case 2: return run_probe<2>(n_vec, m, reps, gathers_per_s, st);
    case 4: return run_probe<4>(n_vec, m, reps, gathers_per_s, st);
    default: return fail(FJ_E_INVALID_ARG, "fj_probe_gather: width must be 1, 2 or 4");
  }
}

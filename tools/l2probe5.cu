// l2probe5.cu — scratch microbenchmark (not product code): the C3 product's gather pattern (nnz
// uniform random int32 indices streamed once, one 32-byte row gathered per index from an n-row
// [n][4] fp64 block) with different PTX load flavours, to see whether the L2/DRAM side fetches more
// than the 32-byte sector per random gather and whether a cache qualifier changes it.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/l2probe5.bin tools/l2probe5.cu
// One JSON line per (flavour, block size): ms per pass and G gathers / s.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

struct D4 { double a, b, c, d; };
template <int F>
__device__ __forceinline__ D4 ld4(const double* p) {
  D4 r;
  if constexpr (F == 0)
    asm volatile("ld.global.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(r.a), "=d"(r.b), "=d"(r.c), "=d"(r.d) : "l"(p));
  else if constexpr (F == 1)
    asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(r.a), "=d"(r.b), "=d"(r.c), "=d"(r.d) : "l"(p));
  else if constexpr (F == 2)
    asm volatile("ld.global.cg.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(r.a), "=d"(r.b), "=d"(r.c), "=d"(r.d) : "l"(p));
  else if constexpr (F == 3)
    asm volatile("ld.global.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(r.a), "=d"(r.b), "=d"(r.c), "=d"(r.d) : "l"(p));
  else if constexpr (F == 4)
    asm volatile("ld.global.cs.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(r.a), "=d"(r.b), "=d"(r.c), "=d"(r.d) : "l"(p));
  else if constexpr (F == 5)
    asm volatile("ld.global.lu.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(r.a), "=d"(r.b), "=d"(r.c), "=d"(r.d) : "l"(p));
  else if constexpr (F == 6) {
    asm volatile("ld.global.v2.f64 {%0,%1}, [%2];" : "=d"(r.a), "=d"(r.b) : "l"(p));
    asm volatile("ld.global.v2.f64 {%0,%1}, [%2];" : "=d"(r.c), "=d"(r.d) : "l"(p + 2));
  } else if constexpr (F == 7)
    asm volatile("ld.global.L2::64B.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(r.a), "=d"(r.b), "=d"(r.c), "=d"(r.d) : "l"(p));
  else if constexpr (F == 8)
    asm volatile("ld.global.L2::256B.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(r.a), "=d"(r.b), "=d"(r.c), "=d"(r.d) : "l"(p));
  else if constexpr (F == 9)
    asm volatile("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(r.a), "=d"(r.b), "=d"(r.c), "=d"(r.d) : "l"(p));
  return r;
}

template <int F, int U>
__global__ void __launch_bounds__(128) k_gather(int64_t nnz, const int32_t* __restrict__ idx, const double* __restrict__ x,
                                                double* out) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x, nt = (int64_t)gridDim.x * blockDim.x;
  double acc = 0;
  for (int64_t b = t; b < nnz; b += nt * U) {
    int32_t j[U];
#pragma unroll
    for (int u = 0; u < U; ++u) j[u] = b + u * nt < nnz ? __ldg(idx + b + u * nt) : 0;
    D4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = ld4<F>(x + (int64_t)j[u] * 4);
#pragma unroll
    for (int u = 0; u < U; ++u) acc += v[u].a + v[u].b + v[u].c;
  }
  if (acc == 123.0) out[0] = acc;
}

__global__ void k_idx(int64_t nnz, int64_t n, uint64_t seed, int32_t* idx) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nnz; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t x = (uint64_t)i * 0x9E3779B97F4A7C15ull + seed;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    x ^= x >> 31;
    idx[i] = (int32_t)(x % (uint64_t)n);
  }
}

template <int F>
void run(const char* name, int64_t nnz, int64_t n, const int32_t* idx, const double* x, double* out, int sms, int reps) {
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  auto go = [&]() { k_gather<F, 8><<<sms * 8, 128>>>(nnz, idx, x, out); };
  go();
  CK(cudaEventRecord(e0));
  for (int r = 0; r < reps; ++r) go();
  CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1)); CK(cudaGetLastError());
  float ms; CK(cudaEventElapsedTime(&ms, e0, e1)); ms /= reps;
  printf("{\"flavour\": \"%s\", \"block_MB\": %.1f, \"nnz\": %lld, \"ms\": %.4f, \"Ggps\": %.1f}\n", name,
         n * 32.0 / 1e6, (long long)nnz, ms, nnz / (ms * 1e-3) / 1e9);
  fflush(stdout);
}

int main(int argc, char** argv) {
  CK(cudaSetDevice(0));
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int reps = argc > 1 ? atoi(argv[1]) : 5;
  const int64_t nnz = 64ll << 20;
  int32_t* idx; double* x; double* out;
  CK(cudaMalloc(&idx, nnz * 4)); CK(cudaMalloc(&out, 64));
  const int64_t nmax = 4ll << 20;
  CK(cudaMalloc(&x, nmax * 32)); CK(cudaMemset(x, 0, nmax * 32));
  for (int64_t n : {nmax / 2, nmax}) {
    k_idx<<<sms * 8, 256>>>(nnz, n, 12345, idx);
    CK(cudaDeviceSynchronize());
    run<0>("default", nnz, n, idx, x, out, sms, reps);
    run<1>("nc", nnz, n, idx, x, out, sms, reps);
    run<2>("cg", nnz, n, idx, x, out, sms, reps);
    run<3>("L1::no_allocate", nnz, n, idx, x, out, sms, reps);
    run<4>("cs", nnz, n, idx, x, out, sms, reps);
    run<5>("lu", nnz, n, idx, x, out, sms, reps);
    run<6>("2x16B", nnz, n, idx, x, out, sms, reps);
    run<7>("L2::64B", nnz, n, idx, x, out, sms, reps);
    run<8>("L2::256B", nnz, n, idx, x, out, sms, reps);
    run<9>("nc.L1::no_allocate", nnz, n, idx, x, out, sms, reps);
  }
  return 0;
}

// l2probe3.cu — scratch microbenchmark (not product code): can L2 eviction-priority hints keep the
// HOT part of a gathered block resident when the whole block exceeds the L2?  Indices follow the
// BA endpoint law (j = R u^2: low rows hot), streamed from HBM like the CSR col array.  Gathers to
// rows j < H use an evict_last policy, the rest evict_first (or no hint), the index stream .cs.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}
__global__ void k_fill(int64_t R, int64_t m, int skew, int32_t* idx) {
  const int64_t T = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += T) {
    const double u = (double)(mix(i) >> 11) * 0x1.0p-53;
    int64_t j = skew == 0 ? (int64_t)(u * R) : skew == 1 ? (int64_t)(u * u * R) : (int64_t)(u * u * u * R);
    if (j >= R) j = R - 1;
    idx[i] = (int32_t)j;
  }
}

// mode 0: plain; 1: hot evict_last / cold evict_first; 2: hot evict_last / cold plain;
// 3: hot plain / cold evict_first; 4: hot evict_normal / cold L2::evict_first + L1 no_allocate
__global__ void __launch_bounds__(256) k_gather(int64_t m, const double* __restrict__ x, const int32_t* __restrict__ idx,
                                                int64_t H, int mode, double* __restrict__ out) {
  constexpr int U = 8;
  uint64_t pl, pf;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pl));
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pf));
  const int64_t T = (int64_t)gridDim.x * blockDim.x;
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  double acc = 0.0;
  for (int64_t i = t; i < m; i += U * T) {
    int32_t j[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t q = i + u * T;
      j[u] = q < m ? __ldcs(idx + q) : -1;
    }
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      v[u] = 0.0;
      if (j[u] < 0) continue;
      const double* p = x + (int64_t)j[u] * 4;
      double a, b, c, d;
      const bool hot = j[u] < H;
      if (mode == 0 || (mode == 2 && !hot) || (mode == 3 && hot)) {
        asm volatile("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p));
      } else if (hot && mode != 4) {
        asm volatile("ld.global.nc.L2::cache_hint.v4.f64 {%0, %1, %2, %3}, [%4], %5;"
                     : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p), "l"(pl));
      } else if (hot) {
        asm volatile("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p));
      } else if (mode == 4) {
        asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f64 {%0, %1, %2, %3}, [%4], %5;"
                     : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p), "l"(pf));
      } else {
        asm volatile("ld.global.nc.L2::cache_hint.v4.f64 {%0, %1, %2, %3}, [%4], %5;"
                     : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p), "l"(pf));
      }
      v[u] = (a + b) + (c + d);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc += v[u];
  }
  out[t] = acc;
}

int main() {
  CK(cudaSetDevice(0));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int64_t m = 64000000;
  double* x; int32_t* idx; double* out;
  CK(cudaMalloc(&x, 256ll << 20));
  CK(cudaMemset(x, 0, 256ll << 20));
  CK(cudaMalloc(&idx, m * 4));
  CK(cudaMalloc(&out, 1 << 24));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  const int grid = sms * 8;
  for (int skew = 1; skew <= 2; ++skew) {
    for (int mb : {128, 160, 256}) {
      const int64_t R = ((int64_t)mb << 20) / 32;
      k_fill<<<sms * 8, 256>>>(R, m, skew, idx);
      for (int mode = 0; mode <= 4; ++mode) {
        for (int hmb : {32, 48, 64, 80, 96}) {
          if (mode == 0 && hmb != 32) continue;
          const int64_t H = ((int64_t)hmb << 20) / 32;
          k_gather<<<grid, 256>>>(m, x, idx, H, mode, out);
          k_gather<<<grid, 256>>>(m, x, idx, H, mode, out);
          CK(cudaEventRecord(e0));
          for (int r = 0; r < 5; ++r) k_gather<<<grid, 256>>>(m, x, idx, H, mode, out);
          CK(cudaEventRecord(e1));
          CK(cudaEventSynchronize(e1));
          CK(cudaGetLastError());
          float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
          ms /= 5;
          printf("{\"skew\": %d, \"block_MB\": %d, \"mode\": %d, \"hot_MB\": %d, \"ms\": %.4f, \"Ggps\": %.1f}\n", skew, mb,
                 mode, mode ? hmb : 0, ms, m / (ms * 1e-3) / 1e9);
          fflush(stdout);
        }
      }
    }
  }
  return 0;
}

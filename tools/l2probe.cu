// l2probe.cu — scratch microbenchmark (not product code): random-gather rate on B200 as a function
// of the gathered block size, row width, index skew, L2 fetch granularity and persisting window.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/l2probe.cu -o gpurun_out/l2probe
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

// skew 0: uniform rows; 1: BA-like endpoint law P(j) ~ 1/sqrt(j) (j = R u^2); 2: hot rows spread
// (BA law applied through a random bijection-ish scramble so hot rows are scattered)
__global__ void k_fill(int64_t R, int64_t m, int skew, int32_t* idx) {
  const int64_t T = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += T) {
    const double u = (double)(mix(i) >> 11) * 0x1.0p-53;
    int64_t j = skew == 0 ? (int64_t)(u * R) : (int64_t)(u * u * R);
    if (j >= R) j = R - 1;
    if (skew == 2) j = (int64_t)((j * 2654435761ull) % (uint64_t)R);
    idx[i] = (int32_t)j;
  }
}

template <int W>   // W doubles per row
__device__ __forceinline__ double ldrow(const double* p) {
  if (W == 1) { return __ldg(p); }
  if (W == 2) { double2 v = __ldg(reinterpret_cast<const double2*>(p)); return v.x + v.y; }
  if (W == 3) {   // 24-B row: the 16-B aligned pair + the single (even rows: 0,1 | 2; odd rows: 0 | 1,2)
    const bool odd = (reinterpret_cast<uintptr_t>(p) & 8) != 0;
    double2 v = __ldg(reinterpret_cast<const double2*>(p + (odd ? 1 : 0)));
    return v.x + v.y + __ldg(p + (odd ? 0 : 2));
  }
  double a, b, c, d;
  asm volatile("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p));
  return (a + b) + (c + d);
}

// stride = doubles between rows (W3 with stride 3 = packed 24 B rows; stride 4 = padded)
template <int W>
__global__ void __launch_bounds__(256) k_gather(int64_t m, int stride, const double* __restrict__ x,
                                                const int32_t* __restrict__ idx, double* __restrict__ out,
                                                double* __restrict__ qout, int qw) {
  constexpr int U = 8;
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
    for (int u = 0; u < U; ++u) v[u] = j[u] >= 0 ? ldrow<W>(x + (int64_t)j[u] * stride) : 0.0;
    double s = 0.0;
#pragma unroll
    for (int u = 0; u < U; ++u) s += v[u];
    acc += s;
    if (qw) {   // simulate the q write stream: qw doubles per 8 gathers (one row per ~8 nonzeros)
      const int64_t r = i / U;
      for (int c = 0; c < qw; ++c) qout[r * qw + c] = s;
    }
  }
  out[t] = acc;
}

int main(int argc, char** argv) {
  int dev = 0;
  CK(cudaSetDevice(dev));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  int l2 = 0, persist_max = 0;
  CK(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev));
  CK(cudaDeviceGetAttribute(&persist_max, cudaDevAttrMaxPersistingL2CacheSize, dev));
  printf("{\"sms\": %d, \"l2_bytes\": %d, \"persist_max\": %d}\n", sms, l2, persist_max);
  const int64_t m = 64000000;
  const int64_t maxbytes = 256ll << 20;
  double* x; int32_t* idx; double* out; double* q;
  CK(cudaMalloc(&x, maxbytes));
  CK(cudaMemset(x, 0, maxbytes));
  CK(cudaMalloc(&idx, m * 4));
  CK(cudaMalloc(&out, 1 << 24));
  CK(cudaMalloc(&q, (m / 8 + 1024) * 4 * 8));
  cudaStream_t st;
  CK(cudaStreamCreate(&st));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  const int grid = sms * 8;
  auto run = [&](int W, int stride, int64_t R, int skew, int gran, int64_t persist_bytes, int qw) {
    k_fill<<<sms * 8, 256, 0, st>>>(R, m, skew, idx);
    CK(cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, gran));
    cudaStreamAttrValue av;
    memset(&av, 0, sizeof(av));
    if (persist_bytes > 0) {
      CK(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, persist_max));
      av.accessPolicyWindow.base_ptr = x;
      av.accessPolicyWindow.num_bytes = persist_bytes;
      av.accessPolicyWindow.hitRatio = 1.0f;
      av.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
      av.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    } else {
      av.accessPolicyWindow.num_bytes = 0;
    }
    CK(cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &av));
    auto launch = [&]() {
      switch (W) {
        case 1: k_gather<1><<<grid, 256, 0, st>>>(m, stride, x, idx, out, q, qw); break;
        case 2: k_gather<2><<<grid, 256, 0, st>>>(m, stride, x, idx, out, q, qw); break;
        case 3: k_gather<3><<<grid, 256, 0, st>>>(m, stride, x, idx, out, q, qw); break;
        default: k_gather<4><<<grid, 256, 0, st>>>(m, stride, x, idx, out, q, qw); break;
      }
    };
    launch(); launch();
    const int reps = 5;
    CK(cudaEventRecord(e0, st));
    for (int r = 0; r < reps; ++r) launch();
    CK(cudaEventRecord(e1, st));
    CK(cudaEventSynchronize(e1));
    CK(cudaGetLastError());
    float ms = 0; CK(cudaEventElapsedTime(&ms, e0, e1));
    ms /= reps;
    if (persist_bytes > 0) {
      av.accessPolicyWindow.num_bytes = 0;
      CK(cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &av));
      CK(cudaCtxResetPersistingL2Cache());
    }
    printf("{\"W\": %d, \"stride\": %d, \"block_MB\": %.1f, \"skew\": %d, \"gran\": %d, \"persist_MB\": %.1f, \"qw\": %d, "
           "\"ms\": %.4f, \"Ggps\": %.1f}\n",
           W, stride, R * stride * 8 / 1e6, skew, gran, persist_bytes / 1e6, qw, ms, m / (ms * 1e-3) / 1e9);
    fflush(stdout);
  };
  const int sizes_mb[] = {32, 48, 64, 80, 96, 112, 128, 160, 256};
  // 1. block size sweep, padded 32-B rows, uniform and BA-skewed
  if (getenv("FULL")) for (int skew = 0; skew <= 2; ++skew)
    for (int s : sizes_mb) run(4, 4, ((int64_t)s << 20) / 32, skew, 0, 0, 0);
  // 2. fetch granularity at 128 MB / 32 B rows and 64 MB
  if (getenv("FULL")) for (int g : {32, 64, 128})
    for (int skew = 0; skew <= 1; ++skew) {
      run(4, 4, (128ll << 20) / 32, skew, g, 0, 0);
      run(4, 4, (96ll << 20) / 32, skew, g, 0, 0);
    }
  // 3. C3 k = 3 shapes: 4M rows padded (128 MB) vs packed 24 B (96 MB) vs [n][2]+[n][1] emulated as two probes
  const int64_t n3 = 4000000;
  for (int skew = 0; skew <= 1; ++skew) {
    run(4, 4, n3, skew, 0, 0, 0);
    run(3, 3, n3, skew, 0, 0, 0);
    run(3, 3, n3, skew, 32, 0, 0);
    run(2, 2, n3, skew, 0, 0, 0);
    run(1, 1, n3, skew, 0, 0, 0);
    run(4, 4, n3, skew, 0, 0, 3);      // with a q write stream (24 B per 8 gathers)
    run(4, 4, n3, skew, 0, (int64_t)persist_max, 0);
    run(4, 4, n3, skew, 0, (int64_t)persist_max / 2, 0);
  }
  printf("{\"done\": 1}\n");
  return 0;
}

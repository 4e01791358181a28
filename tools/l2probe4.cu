// l2probe4.cu — scratch microbenchmark (not product code): random gathers of WIDE rows (the k = 64
// product's 512-byte neighbour rows), one warp per row (16 B per lane), U rows in flight per warp,
// uniform or R-MAT-like skewed row ids, block 128 MB .. 2 GB.  Reports rows/s and DRAM-side GB/s
// (rows x row bytes; an upper bound of useful bytes).
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)
__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull; x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull; return x ^ (x >> 31);
}
template <int U>
__global__ void __launch_bounds__(128) k_rows(int64_t rows_total, int64_t R, int skew, int rowd, const double* __restrict__ x, double* out) {
  const int lane = threadIdx.x & 31;
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5, nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  double acc0 = 0, acc1 = 0;
  for (int64_t b = w * U; b < rows_total; b += nw * U) {
    double2 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const double q = (double)(mix(b + u) >> 11) * 0x1.0p-53;
      int64_t j = skew ? (int64_t)(q * q * q * R) : (int64_t)(q * R);
      if (j >= R) j = R - 1;
      v[u] = __ldg(reinterpret_cast<const double2*>(x + j * rowd) + lane);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) { acc0 += v[u].x; acc1 += v[u].y; }
  }
  if (acc0 == 123.0) out[0] = acc1;
}
int main() {
  CK(cudaSetDevice(0));
  int sms; CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int64_t maxb = 2304ll << 20;
  double* x; double* out;
  CK(cudaMalloc(&x, maxb)); CK(cudaMemset(x, 0, maxb)); CK(cudaMalloc(&out, 64));
  cudaEvent_t e0, e1; CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  const int rowd = 64;   // 512-byte rows
  const int64_t rows_total = 32ll << 20;
  for (int skew = 0; skew <= 1; ++skew)
    for (int mb : {128, 512, 2048})
      for (int occ : {4, 8, 16}) {
        const int64_t R = ((int64_t)mb << 20) / (rowd * 8);
        auto go = [&]() { k_rows<8><<<sms * occ, 128>>>(rows_total, R, skew, rowd, x, out); };
        go(); CK(cudaEventRecord(e0));
        for (int r = 0; r < 3; ++r) go();
        CK(cudaEventRecord(e1)); CK(cudaEventSynchronize(e1)); CK(cudaGetLastError());
        float ms; CK(cudaEventElapsedTime(&ms, e0, e1)); ms /= 3;
        printf("{\"skew\": %d, \"block_MB\": %d, \"blocks_per_sm\": %d, \"ms\": %.3f, \"Grows_s\": %.2f, \"row_GBs\": %.0f}\n",
               skew, mb, occ, ms, rows_total / (ms * 1e-3) / 1e9, rows_total * 512.0 / (ms * 1e-3) / 1e9);
        fflush(stdout);
      }
  return 0;
}

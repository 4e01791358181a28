// bulkgather_probe.cu — scratch microbenchmark (not product code): random 512-byte row gathers (the
// k = 64 product's pattern) from a large [n][64] fp64 block, summed per warp:
//   mode 0: registers — lane l loads 16 bytes of each row, R rows in flight per warp (the spmm engine)
//   mode 1: TMA bulk copies — lane 0 issues cp.async.bulk of whole 512-byte rows into a per-warp
//           shared-memory ring of D slots (mbarrier completion); lanes consume 16 bytes per slot
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/bulkgather_probe.bin tools/bulkgather_probe.cu
// One JSON line per (mode, depth, warps per block, skew): G rows / s.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int R>
__global__ void k_reg(int64_t m, const int32_t* __restrict__ idx, const double2* __restrict__ x, double* out) {
  const int lane = threadIdx.x & 31;
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5, nw = (int64_t)gridDim.x * blockDim.x / 32;
  double a0 = 0, a1 = 0;
  for (int64_t b = w * R; b < m; b += nw * R) {
    double2 v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int32_t j = b + r < m ? __ldg(idx + b + r) : 0;
      v[r] = __ldg(x + (int64_t)j * 32 + lane);
    }
#pragma unroll
    for (int r = 0; r < R; ++r) { a0 += v[r].x; a1 += v[r].y; }
  }
  if (a0 + a1 == 1234.5) out[0] = a0;
}

template <int D, int WPB>
__global__ void __launch_bounds__(WPB * 32) k_bulk(int64_t m, const int32_t* __restrict__ idx, const double* __restrict__ x,
                                                   double* out) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  double2* ring = reinterpret_cast<double2*>(smem) + (size_t)wib * D * 32;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)WPB * D * 512) + wib * D;
  if (lane == 0)
    for (int s = 0; s < D; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bars + s)));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5, nw = (int64_t)gridDim.x * blockDim.x / 32;
  // this warp's rows: a contiguous range of the index stream (lane 0's index loads hit L1)
  const int64_t per = (m + nw - 1) / nw, base = w * per;
  const int64_t cnt = m > base ? (m - base < per ? m - base : per) : 0;
  auto issue = [&](int64_t t) {   // lane 0: row t of this warp into slot t % D
    const int s = (int)(t % D);
    const int32_t j = __ldg(idx + base + t);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 512;" ::"r"(smem_u32(bars + s)) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 512, [%2];"
                 ::"r"(smem_u32(ring + (size_t)s * 32)), "l"(x + (int64_t)j * 64), "r"(smem_u32(bars + s)) : "memory");
  };
  if (lane == 0)
    for (int64_t t = 0; t < D && t < cnt; ++t) issue(t);
  double a0 = 0, a1 = 0;
  for (int64_t t = 0; t < cnt; ++t) {
    const int s = (int)(t % D);
    const uint32_t par = (uint32_t)((t / D) & 1);
    asm volatile("{\n .reg .pred p;\n W_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W_%=;\n}"
                 ::"r"(smem_u32(bars + s)), "r"(par) : "memory");
    const double2 v = ring[(size_t)s * 32 + lane];
    a0 += v.x; a1 += v.y;
    __syncwarp();
    if (lane == 0 && t + D < cnt) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(t + D);
    }
  }
  if (a0 + a1 == 1234.5) out[0] = a0;
}

static uint64_t sm64(uint64_t& s) {
  uint64_t z = (s += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

int main(int argc, char** argv) {
  const int64_t n = argc > 1 ? atoll(argv[1]) : 4194304;     // rows of 512 bytes: 2 GB
  const int64_t m = argc > 2 ? atoll(argv[2]) : 64000000;    // gathers
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  double* x; int32_t* idx; double* out;
  CK(cudaMalloc(&x, (size_t)n * 512));
  CK(cudaMemset(x, 0, (size_t)n * 512));
  CK(cudaMalloc(&idx, (size_t)m * 4));
  CK(cudaMalloc(&out, 8));
  int32_t* h = (int32_t*)malloc((size_t)m * 4);
  for (int skew = 0; skew < 2; ++skew) {
    uint64_t s = 12345;
    for (int64_t i = 0; i < m; ++i) {
      const uint64_t r = sm64(s);
      if (!skew) h[i] = (int32_t)(r % (uint64_t)n);
      else {   // R-MAT-like skew: a quarter of the gathers in the first 1/16 of the rows
        h[i] = (r & 3) == 0 ? (int32_t)((r >> 2) % (uint64_t)(n / 16)) : (int32_t)((r >> 2) % (uint64_t)n);
      }
    }
    CK(cudaMemcpy(idx, h, (size_t)m * 4, cudaMemcpyHostToDevice));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
    auto timeit = [&](auto launch) {
      launch();
      CK(cudaDeviceSynchronize());
      CK(cudaEventRecord(e0));
      for (int r = 0; r < 5; ++r) launch();
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, e0, e1));
      return ms / 5;
    };
    for (int bps : {8, 16}) {
      float ms = timeit([&] { k_reg<8><<<sms * bps, 128>>>(m, idx, (const double2*)x, out); });
      printf("{\"mode\": \"reg\", \"R\": 8, \"blocks_per_sm\": %d, \"skew\": %d, \"ms\": %.4f, \"Grows_s\": %.2f}\n", bps, skew, ms, m / ms / 1e6);
      ms = timeit([&] { k_reg<16><<<sms * bps, 128>>>(m, idx, (const double2*)x, out); });
      printf("{\"mode\": \"reg\", \"R\": 16, \"blocks_per_sm\": %d, \"skew\": %d, \"ms\": %.4f, \"Grows_s\": %.2f}\n", bps, skew, ms, m / ms / 1e6);
    }
#define BULK(D, WPB)                                                                                                  \
    {                                                                                                                 \
      const size_t sh = (size_t)WPB * D * 512 + (size_t)WPB * D * 8;                                                  \
      CK(cudaFuncSetAttribute(k_bulk<D, WPB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sh));                  \
      int occ = 0;                                                                                                    \
      CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_bulk<D, WPB>, WPB * 32, sh));                          \
      float ms = timeit([&] { k_bulk<D, WPB><<<sms * occ, WPB * 32, sh>>>(m, idx, x, out); });                        \
      CK(cudaGetLastError());                                                                                         \
      printf("{\"mode\": \"bulk\", \"D\": %d, \"warps_per_block\": %d, \"blocks_per_sm\": %d, \"skew\": %d, \"ms\": %.4f, \"Grows_s\": %.2f}\n", D, WPB, occ, skew, ms, m / ms / 1e6); \
    }
    BULK(8, 4) BULK(16, 4) BULK(32, 4) BULK(16, 8) BULK(8, 8) BULK(24, 4) BULK(64, 2)
    fflush(stdout);
  }
  return 0;
}

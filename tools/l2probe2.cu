// l2probe2.cu — scratch microbenchmark (not product code).  Questions:
//  (1) effective L2 capacity for random 32-B gathers with no competing stream (indices hashed in
//      registers), block 32..168 MB;
//  (2) does each die's L2 cache lines for its own SMs (replication), i.e. does splitting the gathered
//      block between the dies (CTAs on die d gather only from half d) behave like a half-size block?
//  SM -> die map: per SM, L2-hit latency of a dependent chain on a few fixed lines; the SMs split in
//  two latency groups (near / far home die).
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

__device__ __forceinline__ uint32_t smid() { uint32_t r; asm volatile("mov.u32 %0, %%smid;" : "=r"(r)); return r; }
__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

// latency of L2 hits on line `a` (dependent chain through ld.cg of a self-pointer)
__global__ void k_lat(uint64_t* const* lines, int nlines, long long* out /* [grid][nlines] */, int* sm_of_block) {
  if (threadIdx.x != 0) return;
  sm_of_block[blockIdx.x] = smid();
  for (int l = 0; l < nlines; ++l) {
    uint64_t* p = lines[l];
    uint64_t v = (uint64_t)p;
    for (int w = 0; w < 8; ++w) v = __ldcg(reinterpret_cast<uint64_t*>(v));
    long long t0 = clock64();
    for (int r = 0; r < 256; ++r) v = __ldcg(reinterpret_cast<uint64_t*>(v));
    long long t1 = clock64();
    out[blockIdx.x * nlines + l] = (t1 - t0) / 256 + (v == 1 ? 1 : 0);
  }
}

// random 32-B gathers; mode 0: uniform over the block; mode 1: CTA on die d -> half d only
__global__ void __launch_bounds__(256) k_gather(int64_t m_per_thread, int64_t rows, const double* __restrict__ x,
                                                const int8_t* __restrict__ die_of_sm, int mode, double* out) {
  constexpr int U = 8;
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int64_t lo = 0, span = rows;
  if (mode == 1) {
    const int d = die_of_sm[smid()];
    span = rows / 2;
    lo = d ? span : 0;
  }
  double acc = 0.0;
  uint64_t st = mix(t * 7919 + 13);
  for (int64_t i = 0; i < m_per_thread; i += U) {
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      st = mix(st + u);
      const int64_t j = lo + (int64_t)(((st >> 32) * (uint64_t)span) >> 32);
      const double* p = x + j * 4;
      double a, b, c, d;
      asm volatile("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p));
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
  // ---- SM -> die map
  const int NL = 16;
  uint64_t* buf;
  CK(cudaMalloc(&buf, 64ll << 20));
  std::vector<uint64_t*> lines(NL);
  for (int l = 0; l < NL; ++l) {
    uint64_t* a = buf + (int64_t)l * (2 << 20) / 8 + 17 * l;   // 2 MB apart
    uint64_t hv = (uint64_t)a;
    CK(cudaMemcpy(a, &hv, 8, cudaMemcpyHostToDevice));
    lines[l] = a;
  }
  uint64_t** dl;
  CK(cudaMalloc(&dl, NL * sizeof(void*)));
  CK(cudaMemcpy(dl, lines.data(), NL * sizeof(void*), cudaMemcpyHostToDevice));
  const int G = sms * 4;
  long long* dlat; int* dsm;
  CK(cudaMalloc(&dlat, G * NL * 8));
  CK(cudaMalloc(&dsm, G * 4));
  k_lat<<<G, 32>>>(dl, NL, dlat, dsm);
  CK(cudaDeviceSynchronize());
  std::vector<long long> lat(G * NL);
  std::vector<int> smb(G);
  CK(cudaMemcpy(lat.data(), dlat, G * NL * 8, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(smb.data(), dsm, G * 4, cudaMemcpyDeviceToHost));
  std::vector<std::vector<long long>> per_sm(sms, std::vector<long long>(NL, 1 << 30));
  for (int b = 0; b < G; ++b)
    for (int l = 0; l < NL; ++l) per_sm[smb[b]][l] = std::min(per_sm[smb[b]][l], lat[b * NL + l]);
  // die of SM = 1 if its latency on line 0 is in the upper group (threshold = midpoint of min/max)
  std::vector<int8_t> die(sms, 0);
  long long mn = 1 << 30, mx = 0;
  for (int s = 0; s < sms; ++s) { mn = std::min(mn, per_sm[s][0]); mx = std::max(mx, per_sm[s][0]); }
  int n1 = 0;
  for (int s = 0; s < sms; ++s) { die[s] = per_sm[s][0] * 2 > mn + mx; n1 += die[s]; }
  // consistency: for every other line, the split should be the same partition (or its complement)
  int consistent = 0;
  for (int l = 1; l < NL; ++l) {
    long long a = 1 << 30, b = 0;
    for (int s = 0; s < sms; ++s) { a = std::min(a, per_sm[s][l]); b = std::max(b, per_sm[s][l]); }
    int same = 0, comp = 0;
    for (int s = 0; s < sms; ++s) {
      const int d = per_sm[s][l] * 2 > a + b;
      same += d == die[s];
      comp += d != die[s];
    }
    consistent += (same == sms || comp == sms);
  }
  printf("{\"lat_min\": %lld, \"lat_max\": %lld, \"die1_sms\": %d, \"lines_consistent\": %d, \"of\": %d}\n", mn, mx, n1,
         consistent, NL - 1);
  printf("{\"die_map\": \"");
  for (int s = 0; s < sms; ++s) printf("%d", die[s]);
  printf("\"}\n");
  int8_t* ddie;
  CK(cudaMalloc(&ddie, sms));
  CK(cudaMemcpy(ddie, die.data(), sms, cudaMemcpyHostToDevice));
  // ---- gathers
  double* x;
  const int64_t maxb = 320ll << 20;
  CK(cudaMalloc(&x, maxb));
  CK(cudaMemset(x, 0, maxb));
  double* out;
  CK(cudaMalloc(&out, 1 << 24));
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  const int grid = sms * 8;
  const int64_t total = 64000000;
  const int64_t per = total / ((int64_t)grid * 256) + 1;
  for (int mode = 0; mode <= 1; ++mode) {
    for (int mb : {32, 48, 64, 80, 96, 112, 128, 144, 160, 192, 256}) {
      const int64_t rows = ((int64_t)mb << 20) / 32;
      k_gather<<<grid, 256>>>(per, rows, x, ddie, mode, out);
      k_gather<<<grid, 256>>>(per, rows, x, ddie, mode, out);
      CK(cudaEventRecord(e0));
      for (int r = 0; r < 5; ++r) k_gather<<<grid, 256>>>(per, rows, x, ddie, mode, out);
      CK(cudaEventRecord(e1));
      CK(cudaEventSynchronize(e1));
      CK(cudaGetLastError());
      float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
      ms /= 5;
      printf("{\"mode\": %d, \"block_MB\": %d, \"ms\": %.4f, \"Ggps\": %.1f}\n", mode, mb, ms,
             (double)per * grid * 256 / (ms * 1e-3) / 1e9);
      fflush(stdout);
    }
  }
  return 0;
}

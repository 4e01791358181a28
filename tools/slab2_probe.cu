// slab2_probe.cu — scratch microbenchmark (not product code): a LEAN product kernel for the k = 3
// padded [n][4] block, run either as one pass over the whole CSR or as S passes over column slabs
// (each slab's gathered rows fit the L2), to see whether the slab split pays once the per-pass row
// cost is small (the warp-item engine costs ~0.35 ms per pass regardless of slab size).
//   nvcc -O3 -shared -Xcompiler -fPIC -gencode arch=compute_100a,code=sm_100a -o tools/slab2_probe.so tools/slab2_probe.cu
// q_i (3 columns) accumulates -sum_j p_j over the slab's entries; the last pass adds (1+d_i) p_i.
#include <cstdint>
#include <cuda_runtime.h>
#ifndef FJ_MINB2
#define FJ_MINB2 8
#endif
#ifndef FJ_MINB
#define FJ_MINB 4
#endif

struct D4 { double a, b, c, d; };
__device__ __forceinline__ D4 ld4(const double* p) {
  D4 r;
  asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(r.a), "=d"(r.b), "=d"(r.c), "=d"(r.d) : "l"(p));
  return r;
}

// G lanes per row (G = 1: lane per row).  Rows [0, n); each group walks its row's entries with a
// stride of G, U gathers in flight per lane.  FIRST: q = -acc, else q -= acc; LAST: q += (1+d) p_i.
constexpr int LONG_ROW = 256;

template <int G, int U, bool FIRST, bool LAST>
__global__ void __launch_bounds__(256, FJ_MINB) k_rows(int64_t n, const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                                              const double* __restrict__ p, const double* __restrict__ deg,
                                              double* __restrict__ q) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t ngroups = (int64_t)gridDim.x * blockDim.x / G;
  const int sub = threadIdx.x % G;
  for (int64_t i = t / G; i < n; i += ngroups) {
    const int64_t b = rp[i];
    int64_t e = rp[i + 1];
    if (e - b > LONG_ROW) e = b;   // long rows: their sums come from k_chunks
    double a0 = 0, a1 = 0, a2 = 0;
    int64_t k = b + sub;
    for (; k + (U - 1) * G < e; k += G * U) {   // full batches: U independent gathers in flight
      int32_t j[U];
#pragma unroll
      for (int u = 0; u < U; ++u) j[u] = __ldg(col + k + u * G);
      D4 v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = ld4(p + 4 * (int64_t)j[u]);
#pragma unroll
      for (int u = 0; u < U; ++u) { a0 += v[u].a; a1 += v[u].b; a2 += v[u].c; }
    }
    for (; k < e; k += G) {
      const D4 v = ld4(p + 4 * (int64_t)__ldg(col + k));
      a0 += v.a; a1 += v.b; a2 += v.c;
    }
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) {
      a0 += __shfl_xor_sync(0xffffffffu, a0, o, G);
      a1 += __shfl_xor_sync(0xffffffffu, a1, o, G);
      a2 += __shfl_xor_sync(0xffffffffu, a2, o, G);
    }
    if (sub == 0) {
      double* qi = q + 3 * i;
      double q0, q1, q2;
      if (FIRST) { q0 = -a0; q1 = -a1; q2 = -a2; }
      else { q0 = qi[0] - a0; q1 = qi[1] - a1; q2 = qi[2] - a2; }
      if (LAST) {
        const double di = 1.0 + deg[i];
        const D4 pi = ld4(p + 4 * i);
        q0 += di * pi.a; q1 += di * pi.b; q2 += di * pi.c;
      }
      qi[0] = q0; qi[1] = q1; qi[2] = q2;
    }
  }
}

// long rows: one warp per 512-nonzero chunk (chunk list [nch][3] = row, k0, k1), q -= sum by atomics
__global__ void __launch_bounds__(256) k_chunks(int64_t nch, const int64_t* __restrict__ ch, const int32_t* __restrict__ col,
                                                const double* __restrict__ p, double* q) {
  const int64_t w = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= nch) return;
  const int64_t i = ch[3 * w], k0 = ch[3 * w + 1], k1 = ch[3 * w + 2];
  double a0 = 0, a1 = 0, a2 = 0;
  for (int64_t k = k0 + lane; k < k1; k += 32) {
    const D4 v = ld4(p + 4 * (int64_t)__ldg(col + k));
    a0 += v.a; a1 += v.b; a2 += v.c;
  }
  for (int o = 16; o > 0; o >>= 1) {
    a0 += __shfl_xor_sync(0xffffffffu, a0, o);
    a1 += __shfl_xor_sync(0xffffffffu, a1, o);
    a2 += __shfl_xor_sync(0xffffffffu, a2, o);
  }
  if (lane == 0) { atomicAdd(q + 3 * i, -a0); atomicAdd(q + 3 * i + 1, -a1); atomicAdd(q + 3 * i + 2, -a2); }
}

extern "C" int slab_chunks(int64_t nch, const int64_t* ch, const int32_t* col, const double* p, double* q, void* stream) {
  if (nch == 0) return 0;
  k_chunks<<<(unsigned)((nch * 32 + 255) / 256), 256, 0, (cudaStream_t)stream>>>(nch, ch, col, p, q);
  return (int)cudaGetLastError();
}

template <int G, int U>
static void launch(int first, int last, int64_t n, const int64_t* rp, const int32_t* col, const double* p,
                   const double* deg, double* q, int blocks, cudaStream_t st) {
  if (first && last) k_rows<G, U, true, true><<<blocks, 256, 0, st>>>(n, rp, col, p, deg, q);
  else if (first) k_rows<G, U, true, false><<<blocks, 256, 0, st>>>(n, rp, col, p, deg, q);
  else if (last) k_rows<G, U, false, true><<<blocks, 256, 0, st>>>(n, rp, col, p, deg, q);
  else k_rows<G, U, false, false><<<blocks, 256, 0, st>>>(n, rp, col, p, deg, q);
}


// v2: software-pipelined rows.  Bounds of the row after next and the first batch of column indices
// of the next row are loaded while the current row's gathers are in flight; the epilogue operands
// (q_in, d_i, p_i) are issued before the gathers are consumed.
template <int G, int U, bool FIRST, bool LAST>
__global__ void __launch_bounds__(128, FJ_MINB2) k_rows2(int64_t n, const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                                                   const double* __restrict__ p, const double* __restrict__ deg,
                                                   double* __restrict__ q) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t ng = (int64_t)gridDim.x * blockDim.x / G;
  const int sub = threadIdx.x % G;
  int64_t i = t / G;
  if (i >= n) return;
  auto bounds = [&](int64_t r, int64_t& b, int64_t& e) {
    if (r < n) { b = __ldg(rp + r); e = __ldg(rp + r + 1); if (e - b > LONG_ROW) e = b; } else { b = 0; e = 0; }
  };
  auto first_cols = [&](int64_t b, int64_t e, int64_t r, int32_t (&j)[U]) {
#pragma unroll
    for (int u = 0; u < U; ++u) { const int64_t k = b + sub + u * G; j[u] = k < e ? __ldg(col + k) : (int32_t)(r < n ? r : 0); }
  };
  int64_t b, e, bn, en;
  bounds(i, b, e);
  bounds(i + ng, bn, en);
  int32_t j[U];
  first_cols(b, e, i, j);
  for (; i < n; i += ng) {
    D4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = ld4(p + 4 * (int64_t)j[u]);
    double q0 = 0, q1 = 0, q2 = 0, di = 0;
    D4 pi{0, 0, 0, 0};
    if (sub == 0) {
      if (!FIRST) { q0 = q[3 * i]; q1 = q[3 * i + 1]; q2 = q[3 * i + 2]; }
      if (LAST) { di = 1.0 + __ldg(deg + i); pi = ld4(p + 4 * i); }
    }
    int64_t bnn, enn;
    bounds(i + 2 * ng, bnn, enn);
    int32_t jn[U];
    first_cols(bn, en, i + ng, jn);
    double a0 = 0, a1 = 0, a2 = 0;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const bool ok = b + sub + u * G < e;
      a0 += ok ? v[u].a : 0.0; a1 += ok ? v[u].b : 0.0; a2 += ok ? v[u].c : 0.0;
    }
    for (int64_t k = b + sub + G * U; k < e; k += G * U) {   // rows longer than one batch
      int32_t jj[U];
#pragma unroll
      for (int u = 0; u < U; ++u) jj[u] = k + u * G < e ? __ldg(col + k + u * G) : (int32_t)i;
      D4 w[U];
#pragma unroll
      for (int u = 0; u < U; ++u) w[u] = ld4(p + 4 * (int64_t)jj[u]);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const bool ok = k + u * G < e;
        a0 += ok ? w[u].a : 0.0; a1 += ok ? w[u].b : 0.0; a2 += ok ? w[u].c : 0.0;
      }
    }
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) {
      a0 += __shfl_xor_sync(0xffffffffu, a0, o, G);
      a1 += __shfl_xor_sync(0xffffffffu, a1, o, G);
      a2 += __shfl_xor_sync(0xffffffffu, a2, o, G);
    }
    if (sub == 0) {
      q0 -= a0; q1 -= a1; q2 -= a2;
      if (LAST) { q0 += di * pi.a; q1 += di * pi.b; q2 += di * pi.c; }
      q[3 * i] = q0; q[3 * i + 1] = q1; q[3 * i + 2] = q2;
    }
    b = bn; e = en; bn = bnn; en = enn;
#pragma unroll
    for (int u = 0; u < U; ++u) j[u] = jn[u];
  }
}

template <int G, int U>
static void launch2(int first, int last, int64_t n, const int64_t* rp, const int32_t* col, const double* p,
                    const double* deg, double* q, int blocks, cudaStream_t st) {
  if (first && last) k_rows2<G, U, true, true><<<blocks, 128, 0, st>>>(n, rp, col, p, deg, q);
  else if (first) k_rows2<G, U, true, false><<<blocks, 128, 0, st>>>(n, rp, col, p, deg, q);
  else if (last) k_rows2<G, U, false, true><<<blocks, 128, 0, st>>>(n, rp, col, p, deg, q);
  else k_rows2<G, U, false, false><<<blocks, 128, 0, st>>>(n, rp, col, p, deg, q);
}

extern "C" int slab_pass(int G, int U, int first, int last, int64_t n, const int64_t* rp, const int32_t* col,
                         const double* p, const double* deg, double* q, int blocks, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
#define L(g, u) if (G == g && U == u) { launch<g, u>(first, last, n, rp, col, p, deg, q, blocks, st); return (int)cudaGetLastError(); }
  L(1, 4) L(1, 8) L(2, 4) L(2, 8) L(4, 2) L(4, 4) L(8, 2) L(8, 4) L(16, 1) L(16, 2) L(32, 1)
#undef L
#define L2(g, u) if (G == 100 + g && U == u) { launch2<g, u>(first, last, n, rp, col, p, deg, q, blocks, st); return (int)cudaGetLastError(); }
  L2(1, 4) L2(1, 8) L2(2, 4) L2(2, 8) L2(4, 4) L2(4, 2) L2(8, 2)
#undef L2
  return -1;
}

// vec.cuh — padded row vectors of the small-k engines (spmv_vec.cu, dist.cu): a row of KP doubles
// loaded / stored as ONE aligned vector access (KP = 2: LDG.128, KP = 4: LDG.E.ENL2.256).
#pragma once
#include "common.cuh"

namespace fj {

constexpr int KVMAX = 4;     // widest padded row handled here
constexpr int VETB = 256;    // elementwise kernels: one thread per row

template <int KP>
struct alignas(KP == 3 ? 8 : KP * 8) DVec {
  double v[KP];
};

// Device scalars of one small-k batched solve (per column), written only by last-block finalisers
// (spmv_vec.cu; the rows product's finaliser, rows.cuh).
struct VecScalars {
  double rho[KVMAX], alpha[KVMAX], beta[KVMAX], pq[KVMAX], rr[KVMAX], ss[KVMAX], tol2[KVMAX], res2[KVMAX];
  double alx[KVMAX];   // alpha applied to x by k_v_dir<XD> (0 for columns inactive in that iteration)
  int32_t active[KVMAX], conv[KVMAX], breakdown[KVMAX];
  int32_t iter, max_iter, done, k;
  int32_t xpend;       // k_v_dir<XD> owes x += alx p for the iteration k_v_update just finished
};

template <int KP> __device__ __forceinline__ DVec<KP> ld_vec(const double* p);
template <> __device__ __forceinline__ DVec<1> ld_vec<1>(const double* p) {
  DVec<1> r;
  r.v[0] = *p;
  return r;
}
template <> __device__ __forceinline__ DVec<2> ld_vec<2>(const double* p) {
  DVec<2> r;
  asm volatile("ld.global.v2.f64 {%0, %1}, [%2];" : "=d"(r.v[0]), "=d"(r.v[1]) : "l"(p));
  return r;
}
template <> __device__ __forceinline__ DVec<4> ld_vec<4>(const double* p) {   // 256-bit LDG (sm_100)
  DVec<4> r;
  asm volatile("ld.global.v4.f64 {%0, %1, %2, %3}, [%4];"
               : "=d"(r.v[0]), "=d"(r.v[1]), "=d"(r.v[2]), "=d"(r.v[3]) : "l"(p));
  return r;
}
// KP = 3 (unpadded [n][3], 24-byte rows, base 16-byte aligned): one 16-byte pair + one 8-byte load.
// Even rows start 16-byte aligned (pair = columns 0,1); odd rows end 16-byte aligned (pair = 1,2).
// A row touches 1.5 sectors on average (vs 1 padded to 32 bytes, which no longer fits in L2 at C3).
template <> __device__ __forceinline__ DVec<3> ld_vec<3>(const double* p) {
  const bool odd = (reinterpret_cast<uintptr_t>(p) & 8) != 0;
  const double* pp = p + (odd ? 1 : 0);
  const double* ps = p + (odd ? 0 : 2);
  double a, b, c;
  asm volatile("ld.global.v2.f64 {%0, %1}, [%2];" : "=d"(a), "=d"(b) : "l"(pp));
  asm volatile("ld.global.f64 %0, [%1];" : "=d"(c) : "l"(ps));
  DVec<3> r;
  r.v[0] = odd ? c : a;
  r.v[1] = odd ? a : b;
  r.v[2] = odd ? b : c;
  return r;
}
template <int KP> __device__ __forceinline__ void st_vec(double* p, const DVec<KP>& v);
template <> __device__ __forceinline__ void st_vec<3>(double* p, const DVec<3>& v) {
  const bool odd = (reinterpret_cast<uintptr_t>(p) & 8) != 0;
  const double a = odd ? v.v[1] : v.v[0], b = odd ? v.v[2] : v.v[1], c = odd ? v.v[0] : v.v[2];
  asm volatile("st.global.v2.f64 [%0], {%1, %2};" ::"l"(p + (odd ? 1 : 0)), "d"(a), "d"(b) : "memory");
  asm volatile("st.global.f64 [%0], %1;" ::"l"(p + (odd ? 0 : 2)), "d"(c) : "memory");
}
template <> __device__ __forceinline__ void st_vec<1>(double* p, const DVec<1>& v) { *p = v.v[0]; }
template <> __device__ __forceinline__ void st_vec<2>(double* p, const DVec<2>& v) {
  asm volatile("st.global.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(v.v[0]), "d"(v.v[1]) : "memory");
}
template <> __device__ __forceinline__ void st_vec<4>(double* p, const DVec<4>& v) {
  asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(v.v[0]), "d"(v.v[1]), "d"(v.v[2]),
               "d"(v.v[3]) : "memory");
}
template <int KP> __device__ __forceinline__ DVec<KP> vzero_kp() {
  DVec<KP> r;
#pragma unroll
  for (int c = 0; c < KP; ++c) r.v[c] = 0.0;
  return r;
}

// Rows of the solver's other vectors (x, r, q) are stored KQ wide (KQ = k: 3 for k = 3, no padding);
// only the gathered direction p is padded to KP.  ld_q/st_q move a KQ-wide row as a KP vector.
template <int KP, int KQ>
__device__ __forceinline__ DVec<KP> ld_q(const double* base, int64_t i) {
  if (KP == KQ) return ld_vec<KP>(base + i * KP);
  const DVec<KQ> t = ld_vec<KQ>(base + i * KQ);
  DVec<KP> r;
#pragma unroll
  for (int c = 0; c < KP; ++c) r.v[c] = c < KQ ? t.v[c] : 0.0;
  return r;
}
template <int KP, int KQ>
__device__ __forceinline__ void st_q(double* base, int64_t i, const DVec<KP>& v) {
  if (KP == KQ) { st_vec<KP>(base + i * KP, *reinterpret_cast<const DVec<KP>*>(&v)); return; }
  DVec<KQ> t;
#pragma unroll
  for (int c = 0; c < KQ; ++c) t.v[c] = v.v[c];
  st_vec<KQ>(base + i * KQ, t);
}

}  // namespace fj

// csr_build.cu — row a1: raw edge list -> canonical CSR of the simple undirected graph
// ("simple graph", P:L88 symmetric adjacency w_ij = w_ji; SURVEY.md §8(c) O-1 rules).
//
//  1. k_mirror_keys  both orientations of each raw edge e: (u << b) | v and (v << b) | u, payload e
//                    (payload only for weighted graphs); self-loops get a sentinel key
//  2. radix sort     (stable, 2b bits): row-major, columns ascending, equal keys in input order
//  3. k_kept         first occurrence of each key = keep-first duplicate rule (both orientations of
//                    a pair keep the same, smallest e, so the kept weights stay symmetric)
//  4. scan + k_scatter  col, weight (gathered by payload) and row_ptr of every kept entry
// Sorting uses CUB's DeviceRadixSort (a library primitive, like a BLAS call); every other step
// is a hand-written kernel.  The output is unique, hence bitwise deterministic.
#include <cub/cub.cuh>

#include "common.cuh"
#include "workspace.cuh"

namespace fj {

struct BuildFlags {
  unsigned long long selfloops;
  unsigned int bad_range;
};

// Both orientations of every raw edge e: keys 2e = (u << b) | v and 2e+1 = (v << b) | u, payload e.
// Self-loops (and out-of-range ids) get the sentinel key, which sorts last.
__global__ void k_mirror_keys(int64_t m, int64_t n, const int32_t* __restrict__ u, const int32_t* __restrict__ v,
                              int b, uint64_t sent, uint64_t* __restrict__ keys,
                              int32_t* __restrict__ vals, BuildFlags* fl) {
  unsigned long long loops = 0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x) {
    int64_t a = u[e], c = v[e];
    uint64_t k0 = sent, k1 = sent;
    if (a < 0 || c < 0 || a >= n || c >= n) {
      atomicOr(&fl->bad_range, 1u);
    } else if (a == c) {
      ++loops;
    } else {
      k0 = ((uint64_t)a << b) | (uint64_t)c;
      k1 = ((uint64_t)c << b) | (uint64_t)a;
    }
    keys[2 * e] = k0;
    keys[2 * e + 1] = k1;
    if (vals) { vals[2 * e] = (int32_t)e; vals[2 * e + 1] = (int32_t)e; }
  }
  for (int o = 16; o > 0; o >>= 1) loops += __shfl_xor_sync(0xffffffffu, loops, o);
  if ((threadIdx.x & 31) == 0 && loops) atomicAdd(&fl->selfloops, loops);
}

// first occurrence of each key in the stably sorted list = keep-first duplicate rule
__global__ void k_kept(int64_t m, const uint64_t* __restrict__ keys, uint64_t sent, uint8_t* __restrict__ f) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = keys[i];
    f[i] = (k != sent && (i == 0 || keys[i - 1] != k)) ? 1 : 0;
  }
}

struct U8ToI64 {
  __host__ __device__ __forceinline__ int64_t operator()(const uint8_t& x) const { return (int64_t)x; }
};

// kept entry i -> CSR slot pos[i]: column, weight (gathered through the payload), row_ptr entries
__global__ void k_scatter(int64_t m, int64_t n, const uint64_t* __restrict__ keys, const int32_t* __restrict__ vals,
                          const uint8_t* __restrict__ f, const int64_t* __restrict__ pos, int b, int wbytes,
                          const void* __restrict__ w, int32_t* __restrict__ col, void* __restrict__ w_out,
                          int64_t* __restrict__ row_ptr) {
  const uint64_t mask = (1ULL << b) - 1ULL;
  const int64_t nnz = pos[m - 1] + f[m - 1];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    if (!f[i]) continue;
    const uint64_t key = keys[i];
    const int64_t k = pos[i];
    const int64_t row = (int64_t)(key >> b);
    col[k] = (int32_t)(key & mask);
    if (wbytes) {
      const int64_t e = vals[i];
      if (wbytes == 1) reinterpret_cast<uint8_t*>(w_out)[k] = reinterpret_cast<const uint8_t*>(w)[e];
      else if (wbytes == 4) reinterpret_cast<float*>(w_out)[k] = reinterpret_cast<const float*>(w)[e];
      else reinterpret_cast<double*>(w_out)[k] = reinterpret_cast<const double*>(w)[e];
    }
    // keys[i-1] is the previous kept key (or a duplicate of it): first entry of rows (prev, row]
    const int64_t prev = (i == 0) ? -1 : (int64_t)(keys[i - 1] >> b);
    for (int64_t r = prev + 1; r <= row; ++r) row_ptr[r] = k;
    if (k == nnz - 1)
      for (int64_t r = row + 1; r <= n; ++r) row_ptr[r] = nnz;
  }
}

__global__ void k_fill_empty(int64_t n, int64_t* row_ptr) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= n; i += (int64_t)gridDim.x * blockDim.x)
    row_ptr[i] = 0;
}

static inline unsigned grid_for(int64_t n, int num_sms) {
  int64_t g = (n + 255) / 256;
  int64_t cap = (int64_t)num_sms * 16;
  if (g > cap) g = cap;
  return (unsigned)(g < 1 ? 1 : g);
}

}  // namespace fj

using namespace fj;

static fj_status csr_from_edges(int64_t n, int64_t m_in, const int32_t* u, const int32_t* v,
                                const void* w, int wtype, int64_t* row_ptr, int32_t* col, void* w_out,
                                int64_t* nnz_out, int64_t* selfloops_out, int64_t* dups_out, void* stream) {
  if (n < 1 || n >= INT32_MAX) return fail(FJ_E_INVALID_ARG, "n must be in [1, 2^31-2]");
  if (m_in < 0 || m_in >= INT32_MAX) return fail(FJ_E_INVALID_ARG, "m_in must be in [0, 2^31-2]");
  if (!row_ptr || !nnz_out || (m_in > 0 && (!u || !v || !col))) return fail(FJ_E_INVALID_ARG, "null argument");
  if (wtype < FJ_W_UNIT || wtype > FJ_W_F64) return fail(FJ_E_INVALID_ARG, "bad wtype");
  if (wtype != FJ_W_UNIT && m_in > 0 && (!w || !w_out)) return fail(FJ_E_INVALID_ARG, "weights are NULL");
  const int wbytes = wtype == FJ_W_UNIT ? 0 : wtype == FJ_W_U8 ? 1 : wtype == FJ_W_F32 ? 4 : 8;
  cudaStream_t st = S(stream);
  int dev = 0, sms = 148;
  FJ_CK(cudaGetDevice(&dev));
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int b = 1;
  while ((1LL << b) < n) ++b;   // ids fit in b bits
  const uint64_t sent = (b == 32) ? ~0ULL : ((1ULL << (2 * b)) - 1ULL);
  if (m_in == 0) {
    k_fill_empty<<<grid_for(n + 1, sms), 256, 0, st>>>(n, row_ptr);
    FJ_CK_LAUNCH();
    FJ_CK(cudaStreamSynchronize(st));
    *nnz_out = 0;
    if (selfloops_out) *selfloops_out = 0;
    if (dups_out) *dups_out = 0;
    return FJ_OK;
  }
  const int64_t m = m_in, m2 = 2 * m_in;
  BuildFlags hf{};
  DevBuf<uint64_t> ka, kb;
  DevBuf<int32_t> va, vb;
  DevBuf<BuildFlags> fl;
  FJ_TRY(ka.alloc(m2, st)); FJ_TRY(kb.alloc(m2, st));
  if (wbytes) { FJ_TRY(va.alloc(m2, st)); FJ_TRY(vb.alloc(m2, st)); }
  FJ_TRY(fl.alloc(1, st));
  FJ_CK(cudaMemsetAsync(fl.p, 0, sizeof(BuildFlags), st));
  phase_tick("csr: alloc", st);
  k_mirror_keys<<<grid_for(m, sms), 256, 0, st>>>(m, n, u, v, b, sent, ka.p, wbytes ? va.p : nullptr, fl.p);
  FJ_CK_LAUNCH();
  phase_tick("csr: mirror keys", st);
  cub::DoubleBuffer<uint64_t> dk(ka.p, kb.p);
  cub::DoubleBuffer<int32_t> dv(va.p, vb.p);
  size_t bytes = 0;
  if (wbytes) FJ_CK(cub::DeviceRadixSort::SortPairs(nullptr, bytes, dk, dv, m2, 0, 2 * b, st));
  else FJ_CK(cub::DeviceRadixSort::SortKeys(nullptr, bytes, dk, m2, 0, 2 * b, st));
  {
    DevBuf<uint8_t> tmp;
    FJ_TRY(tmp.alloc((int64_t)bytes, st));
    if (wbytes) FJ_CK(cub::DeviceRadixSort::SortPairs(tmp.p, bytes, dk, dv, m2, 0, 2 * b, st));
    else FJ_CK(cub::DeviceRadixSort::SortKeys(tmp.p, bytes, dk, m2, 0, 2 * b, st));
    count_cub();
  }
  phase_tick("csr: radix sort", st);
  const uint64_t* ks = dk.Current();
  const int32_t* vs = wbytes ? dv.Current() : nullptr;
  DevBuf<uint8_t> f;
  DevBuf<int64_t> pos;
  FJ_TRY(f.alloc(m2, st));
  FJ_TRY(pos.alloc(m2, st));
  k_kept<<<grid_for(m2, sms), 256, 0, st>>>(m2, ks, sent, f.p);
  FJ_CK_LAUNCH();
  cub::TransformInputIterator<int64_t, U8ToI64, const uint8_t*> fi(f.p, U8ToI64());
  bytes = 0;
  FJ_CK(cub::DeviceScan::ExclusiveSum(nullptr, bytes, fi, pos.p, m2, st));
  {
    DevBuf<uint8_t> tmp;
    FJ_TRY(tmp.alloc((int64_t)bytes, st));
    FJ_CK(cub::DeviceScan::ExclusiveSum(tmp.p, bytes, fi, pos.p, m2, st));
    count_cub();
  }
  k_fill_empty<<<grid_for(n + 1, sms), 256, 0, st>>>(n, row_ptr);   // rows before the first entry, or nnz = 0
  FJ_CK_LAUNCH();
  phase_tick("csr: kept + scan", st);
  k_scatter<<<grid_for(m2, sms), 256, 0, st>>>(m2, n, ks, vs, f.p, pos.p, b, wbytes, w, col, w_out, row_ptr);
  FJ_CK_LAUNCH();
  phase_tick("csr: scatter", st);
  int64_t last_pos = 0;
  uint8_t last_f = 0;
  FJ_CK(cudaMemcpyAsync(&last_pos, pos.p + m2 - 1, sizeof last_pos, cudaMemcpyDeviceToHost, st));
  FJ_CK(cudaMemcpyAsync(&last_f, f.p + m2 - 1, 1, cudaMemcpyDeviceToHost, st));
  FJ_CK(cudaMemcpyAsync(&hf, fl.p, sizeof hf, cudaMemcpyDeviceToHost, st));
  FJ_CK(cudaStreamSynchronize(st));
  if (hf.bad_range) return fail(FJ_E_INVALID_ARG, "edge endpoint out of [0, n)");
  const int64_t nnz = last_pos + last_f;
  *nnz_out = nnz;
  if (selfloops_out) *selfloops_out = (int64_t)hf.selfloops;
  if (dups_out) *dups_out = m - (int64_t)hf.selfloops - nnz / 2;
  return FJ_OK;
}

extern "C" fj_status fj_csr_from_edges(int64_t n, int64_t m_in, const int32_t* u, const int32_t* v, const void* w,
                                       int wtype, int64_t* row_ptr, int32_t* col, void* w_out, int64_t* nnz_out,
                                       int64_t* selfloops_out, int64_t* dups_out, void* stream) {
  FJ_RANGE("fj_csr_from_edges");
  return csr_from_edges(n, m_in, u, v, w, wtype, row_ptr, col, w_out, nnz_out, selfloops_out, dups_out,
                        stream);
}

// ---------------------------------------------------------------- a1 for a row block (row a8)
namespace fj {

// per raw edge: how many of its two orientations have their row in [r0, r1)
// map (optional): endpoints relabelled old -> map[old] after the range check (the rows are those
// of the relabelled graph; fj_csr_rows_from_edges_relabelled)
__global__ void k_range_count(int64_t m, int64_t n, const int32_t* __restrict__ u, const int32_t* __restrict__ v,
                              const int32_t* __restrict__ map, int64_t r0, int64_t r1, int64_t* __restrict__ cnt,
                              BuildFlags* fl) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x) {
    int64_t a = u[e], c = v[e];
    int64_t k = 0;
    if (a < 0 || c < 0 || a >= n || c >= n) {
      atomicOr(&fl->bad_range, 1u);
    } else if (a != c) {
      if (map) { a = map[a]; c = map[c]; }
      k = (a >= r0 && a < r1) + (c >= r0 && c < r1);
    }
    cnt[e] = k;
  }
}

// emit the in-range orientations in (edge, orientation) order: key = ((row - r0) << b) | col
__global__ void k_range_emit(int64_t m, const int32_t* __restrict__ u, const int32_t* __restrict__ v,
                             const int32_t* __restrict__ map, int64_t r0, int64_t r1, int b,
                             const int64_t* __restrict__ pos, uint64_t* __restrict__ keys, int32_t* __restrict__ vals) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x) {
    int64_t a = u[e], c = v[e];
    if (a == c || a < 0 || c < 0) continue;
    if (map) { a = map[a]; c = map[c]; }
    int64_t p = pos[e];
    if (a >= r0 && a < r1) {
      keys[p] = ((uint64_t)(a - r0) << b) | (uint64_t)c;
      if (vals) vals[p] = (int32_t)e;
      ++p;
    }
    if (c >= r0 && c < r1) {
      keys[p] = ((uint64_t)(c - r0) << b) | (uint64_t)a;
      if (vals) vals[p] = (int32_t)e;
    }
  }
}

}  // namespace fj

static fj_status csr_rows(int64_t n, int64_t m_in, const int32_t* u, const int32_t* v, const int32_t* map,
                          const void* w, int wtype, int64_t r0, int64_t r1, int64_t* row_ptr, int32_t* col,
                          void* w_out, int64_t* nnz_out, void* stream) {
  if (n < 1 || n >= INT32_MAX) return fail(FJ_E_INVALID_ARG, "n must be in [1, 2^31-2]");
  if (m_in < 0 || m_in >= INT32_MAX) return fail(FJ_E_INVALID_ARG, "m_in must be in [0, 2^31-2]");
  if (r0 < 0 || r1 > n || r1 <= r0) return fail(FJ_E_INVALID_ARG, "bad row range");
  if (!row_ptr || !nnz_out || (m_in > 0 && (!u || !v || !col))) return fail(FJ_E_INVALID_ARG, "null argument");
  if (wtype < FJ_W_UNIT || wtype > FJ_W_F64) return fail(FJ_E_INVALID_ARG, "bad wtype");
  if (wtype != FJ_W_UNIT && m_in > 0 && (!w || !w_out)) return fail(FJ_E_INVALID_ARG, "weights are NULL");
  const int wbytes = wtype == FJ_W_UNIT ? 0 : wtype == FJ_W_U8 ? 1 : wtype == FJ_W_F32 ? 4 : 8;
  cudaStream_t st = S(stream);
  int dev = 0, sms = 148;
  FJ_CK(cudaGetDevice(&dev));
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t nl = r1 - r0;
  int b = 1;
  while ((1LL << b) < n) ++b;
  const uint64_t sent = (b == 32) ? ~0ULL : ((1ULL << (2 * b)) - 1ULL);
  k_fill_empty<<<grid_for(nl + 1, sms), 256, 0, st>>>(nl, row_ptr);
  FJ_CK_LAUNCH();
  if (m_in == 0) {
    FJ_CK(cudaStreamSynchronize(st));
    *nnz_out = 0;
    return FJ_OK;
  }
  const int64_t m = m_in;
  DevBuf<int64_t> cnt, pos;
  DevBuf<BuildFlags> fl;
  FJ_TRY(cnt.alloc(m, st)); FJ_TRY(pos.alloc(m + 1, st)); FJ_TRY(fl.alloc(1, st));
  FJ_CK(cudaMemsetAsync(fl.p, 0, sizeof(BuildFlags), st));
  k_range_count<<<grid_for(m, sms), 256, 0, st>>>(m, n, u, v, map, r0, r1, cnt.p, fl.p);
  FJ_CK_LAUNCH();
  FJ_TRY(cub_exclusive_sum(cnt.p, pos.p, m, st));
  int64_t last_pos = 0, last_cnt = 0;
  BuildFlags hf{};
  FJ_CK(cudaMemcpyAsync(&last_pos, pos.p + m - 1, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  FJ_CK(cudaMemcpyAsync(&last_cnt, cnt.p + m - 1, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  FJ_CK(cudaMemcpyAsync(&hf, fl.p, sizeof hf, cudaMemcpyDeviceToHost, st));
  FJ_CK(cudaStreamSynchronize(st));
  if (hf.bad_range) return fail(FJ_E_INVALID_ARG, "edge endpoint out of [0, n)");
  const int64_t m2 = last_pos + last_cnt;
  if (m2 == 0) { *nnz_out = 0; return FJ_OK; }
  DevBuf<uint64_t> ka, kb;
  DevBuf<int32_t> va, vb;
  FJ_TRY(ka.alloc(m2, st)); FJ_TRY(kb.alloc(m2, st));
  if (wbytes) { FJ_TRY(va.alloc(m2, st)); FJ_TRY(vb.alloc(m2, st)); }
  k_range_emit<<<grid_for(m, sms), 256, 0, st>>>(m, u, v, map, r0, r1, b, pos.p, ka.p, wbytes ? va.p : nullptr);
  FJ_CK_LAUNCH();
  cnt.release();
  pos.release();
  cub::DoubleBuffer<uint64_t> dk(ka.p, kb.p);
  cub::DoubleBuffer<int32_t> dv(va.p, vb.p);
  size_t bytes = 0;
  if (wbytes) FJ_CK(cub::DeviceRadixSort::SortPairs(nullptr, bytes, dk, dv, m2, 0, 2 * b, st));
  else FJ_CK(cub::DeviceRadixSort::SortKeys(nullptr, bytes, dk, m2, 0, 2 * b, st));
  {
    DevBuf<uint8_t> tmp;
    FJ_TRY(tmp.alloc((int64_t)bytes, st));
    if (wbytes) FJ_CK(cub::DeviceRadixSort::SortPairs(tmp.p, bytes, dk, dv, m2, 0, 2 * b, st));
    else FJ_CK(cub::DeviceRadixSort::SortKeys(tmp.p, bytes, dk, m2, 0, 2 * b, st));
    count_cub();
  }
  const uint64_t* ks = dk.Current();
  const int32_t* vs = wbytes ? dv.Current() : nullptr;
  DevBuf<uint8_t> f;
  DevBuf<int64_t> kp;
  FJ_TRY(f.alloc(m2, st));
  FJ_TRY(kp.alloc(m2, st));
  k_kept<<<grid_for(m2, sms), 256, 0, st>>>(m2, ks, sent, f.p);
  FJ_CK_LAUNCH();
  cub::TransformInputIterator<int64_t, U8ToI64, const uint8_t*> fi(f.p, U8ToI64());
  bytes = 0;
  FJ_CK(cub::DeviceScan::ExclusiveSum(nullptr, bytes, fi, kp.p, m2, st));
  {
    DevBuf<uint8_t> tmp;
    FJ_TRY(tmp.alloc((int64_t)bytes, st));
    FJ_CK(cub::DeviceScan::ExclusiveSum(tmp.p, bytes, fi, kp.p, m2, st));
    count_cub();
  }
  k_scatter<<<grid_for(m2, sms), 256, 0, st>>>(m2, nl, ks, vs, f.p, kp.p, b, wbytes, w, col, w_out, row_ptr);
  FJ_CK_LAUNCH();
  int64_t lp = 0;
  uint8_t lf = 0;
  FJ_CK(cudaMemcpyAsync(&lp, kp.p + m2 - 1, sizeof lp, cudaMemcpyDeviceToHost, st));
  FJ_CK(cudaMemcpyAsync(&lf, f.p + m2 - 1, 1, cudaMemcpyDeviceToHost, st));
  FJ_CK(cudaStreamSynchronize(st));
  *nnz_out = lp + lf;
  return FJ_OK;
}

extern "C" fj_status fj_csr_rows_from_edges(int64_t n, int64_t m_in, const int32_t* u, const int32_t* v, const void* w,
                                            int wtype, int64_t r0, int64_t r1, int64_t* row_ptr, int32_t* col,
                                            void* w_out, int64_t* nnz_out, void* stream) {
  FJ_RANGE("fj_csr_rows_from_edges");
  return csr_rows(n, m_in, u, v, nullptr, w, wtype, r0, r1, row_ptr, col, w_out, nnz_out, stream);
}

extern "C" fj_status fj_csr_rows_from_edges_relabelled(int64_t n, int64_t m_in, const int32_t* u, const int32_t* v,
                                                       const int32_t* old2new, const void* w, int wtype, int64_t r0,
                                                       int64_t r1, int64_t* row_ptr, int32_t* col, void* w_out,
                                                       int64_t* nnz_out, void* stream) {
  if (!old2new) return fail(FJ_E_INVALID_ARG, "old2new is NULL");
  return csr_rows(n, m_in, u, v, old2new, w, wtype, r0, r1, row_ptr, col, w_out, nnz_out, stream);
}

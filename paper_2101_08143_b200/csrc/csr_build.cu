// csr_build.cu — row a1: raw edge list -> canonical CSR of the simple undirected graph
// ("simple graph", P:L88 symmetric adjacency w_ij = w_ji; SURVEY.md §8(c) O-1 rules).
//
//  1. k_make_keys   key_e = (min(u,v) << b) | max(u,v), payload e; self-loops get a sentinel key
//  2. radix sort    (stable, 2b bits) -> equal keys keep input order
//  3. k_kept        first occurrence of each key  (keep-first duplicate rule)
//  4. scan + k_mirror  each kept edge emits (lo,hi) and (hi,lo) keys with payload e
//  5. radix sort    -> row-major, columns ascending (keys unique after dedup)
//  6. k_fill        col, weights (gathered by payload), row_ptr from the sorted row ids
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

__global__ void k_make_keys(int64_t m, int64_t n, const int32_t* __restrict__ u, const int32_t* __restrict__ v,
                            int b, uint64_t* __restrict__ keys, int32_t* __restrict__ vals, BuildFlags* fl) {
  const uint64_t sent = (b == 32) ? ~0ULL : ((1ULL << (2 * b)) - 1ULL);
  unsigned long long loops = 0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = u[e], c = v[e];
    uint64_t key;
    if (a < 0 || c < 0 || a >= n || c >= n) {
      atomicOr(&fl->bad_range, 1u);
      key = sent;
    } else if (a == c) {
      ++loops;
      key = sent;
    } else {
      const uint64_t lo = (uint64_t)(a < c ? a : c), hi = (uint64_t)(a < c ? c : a);
      key = (lo << b) | hi;
    }
    keys[e] = key;
    vals[e] = (int32_t)e;
  }
  for (int o = 16; o > 0; o >>= 1) loops += __shfl_xor_sync(0xffffffffu, loops, o);
  if ((threadIdx.x & 31) == 0 && loops) atomicAdd(&fl->selfloops, loops);
}

__global__ void k_kept(int64_t m, const uint64_t* __restrict__ keys, uint64_t sent, uint8_t* __restrict__ f) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = keys[i];
    f[i] = (k != sent && (i == 0 || keys[i - 1] != k)) ? 1 : 0;
  }
}

struct U8ToI64 {
  __host__ __device__ __forceinline__ int64_t operator()(const uint8_t& x) const { return (int64_t)x; }
};

__global__ void k_mirror(int64_t m, const uint64_t* __restrict__ keys, const int32_t* __restrict__ vals,
                         const uint8_t* __restrict__ f, const int64_t* __restrict__ pos, int b,
                         uint64_t* __restrict__ k2, int32_t* __restrict__ v2) {
  const uint64_t mask = (1ULL << b) - 1ULL;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    if (!f[i]) continue;
    const uint64_t k = keys[i];
    const uint64_t lo = k >> b, hi = k & mask;
    const int64_t p = 2 * pos[i];
    k2[p] = k;
    k2[p + 1] = (hi << b) | lo;
    v2[p] = vals[i];
    v2[p + 1] = vals[i];
  }
}

__global__ void k_fill(int64_t nnz, int64_t n, const uint64_t* __restrict__ k2, const int32_t* __restrict__ v2, int b,
                       int wbytes, const void* __restrict__ w, int32_t* __restrict__ col, void* __restrict__ w_out,
                       int64_t* __restrict__ row_ptr) {
  const uint64_t mask = (1ULL << b) - 1ULL;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t key = k2[k];
    const int64_t row = (int64_t)(key >> b);
    col[k] = (int32_t)(key & mask);
    if (wbytes) {
      const int64_t e = v2[k];
      if (wbytes == 1) reinterpret_cast<uint8_t*>(w_out)[k] = reinterpret_cast<const uint8_t*>(w)[e];
      else if (wbytes == 4) reinterpret_cast<float*>(w_out)[k] = reinterpret_cast<const float*>(w)[e];
      else reinterpret_cast<double*>(w_out)[k] = reinterpret_cast<const double*>(w)[e];
    }
    const int64_t prev = (k == 0) ? -1 : (int64_t)(k2[k - 1] >> b);
    for (int64_t r = prev + 1; r <= row; ++r) row_ptr[r] = k;   // first entry of rows (prev, row]
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

extern "C" fj_status fj_csr_from_edges(int64_t n, int64_t m_in, const int32_t* u, const int32_t* v, const void* w,
                                       int wtype, int64_t* row_ptr, int32_t* col, void* w_out, int64_t* nnz_out,
                                       int64_t* selfloops_out, int64_t* dups_out, void* stream) {
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
  const int64_t m = m_in;
  int64_t kept = 0;
  BuildFlags hf{};
  DevBuf<uint64_t> k2a, k2b;
  DevBuf<int32_t> v2a, v2b;
  {
    DevBuf<uint64_t> ka, kb;
    DevBuf<int32_t> va, vb;
    DevBuf<BuildFlags> fl;
    FJ_TRY(ka.alloc(m, st)); FJ_TRY(kb.alloc(m, st));
    FJ_TRY(va.alloc(m, st)); FJ_TRY(vb.alloc(m, st));
    FJ_TRY(fl.alloc(1, st));
    FJ_CK(cudaMemsetAsync(fl.p, 0, sizeof(BuildFlags), st));
    k_make_keys<<<grid_for(m, sms), 256, 0, st>>>(m, n, u, v, b, ka.p, va.p, fl.p);
    FJ_CK_LAUNCH();
    cub::DoubleBuffer<uint64_t> dk(ka.p, kb.p);
    cub::DoubleBuffer<int32_t> dv(va.p, vb.p);
    size_t bytes = 0;
    FJ_CK(cub::DeviceRadixSort::SortPairs(nullptr, bytes, dk, dv, m, 0, 2 * b, st));
    {
      DevBuf<uint8_t> tmp;
      FJ_TRY(tmp.alloc((int64_t)bytes, st));
      FJ_CK(cub::DeviceRadixSort::SortPairs(tmp.p, bytes, dk, dv, m, 0, 2 * b, st));
      count_cub();
    }
    const uint64_t* ks = dk.Current();
    const int32_t* vs = dv.Current();
    DevBuf<uint8_t> f;
    DevBuf<int64_t> pos;
    FJ_TRY(f.alloc(m, st));
    FJ_TRY(pos.alloc(m, st));
    k_kept<<<grid_for(m, sms), 256, 0, st>>>(m, ks, sent, f.p);
    FJ_CK_LAUNCH();
    cub::TransformInputIterator<int64_t, U8ToI64, const uint8_t*> fi(f.p, U8ToI64());
    bytes = 0;
    FJ_CK(cub::DeviceScan::ExclusiveSum(nullptr, bytes, fi, pos.p, m, st));
    {
      DevBuf<uint8_t> tmp;
      FJ_TRY(tmp.alloc((int64_t)bytes, st));
      FJ_CK(cub::DeviceScan::ExclusiveSum(tmp.p, bytes, fi, pos.p, m, st));
      count_cub();
    }
    int64_t last_pos = 0;
    uint8_t last_f = 0;
    FJ_CK(cudaMemcpyAsync(&last_pos, pos.p + m - 1, sizeof last_pos, cudaMemcpyDeviceToHost, st));
    FJ_CK(cudaMemcpyAsync(&last_f, f.p + m - 1, 1, cudaMemcpyDeviceToHost, st));
    FJ_CK(cudaMemcpyAsync(&hf, fl.p, sizeof hf, cudaMemcpyDeviceToHost, st));
    FJ_CK(cudaStreamSynchronize(st));
    if (hf.bad_range) return fail(FJ_E_INVALID_ARG, "edge endpoint out of [0, n)");
    kept = last_pos + last_f;
    if (kept > 0) {
      FJ_TRY(k2a.alloc(2 * kept, st)); FJ_TRY(k2b.alloc(2 * kept, st));
      FJ_TRY(v2a.alloc(2 * kept, st)); FJ_TRY(v2b.alloc(2 * kept, st));
      k_mirror<<<grid_for(m, sms), 256, 0, st>>>(m, ks, vs, f.p, pos.p, b, k2a.p, v2a.p);
      FJ_CK_LAUNCH();
    }
  }
  const int64_t nnz = 2 * kept;
  if (nnz == 0) {
    k_fill_empty<<<grid_for(n + 1, sms), 256, 0, st>>>(n, row_ptr);
    FJ_CK_LAUNCH();
  } else {
    cub::DoubleBuffer<uint64_t> dk(k2a.p, k2b.p);
    cub::DoubleBuffer<int32_t> dv(v2a.p, v2b.p);
    size_t bytes = 0;
    FJ_CK(cub::DeviceRadixSort::SortPairs(nullptr, bytes, dk, dv, nnz, 0, 2 * b, st));
    {
      DevBuf<uint8_t> tmp;
      FJ_TRY(tmp.alloc((int64_t)bytes, st));
      FJ_CK(cub::DeviceRadixSort::SortPairs(tmp.p, bytes, dk, dv, nnz, 0, 2 * b, st));
      count_cub();
    }
    k_fill<<<grid_for(nnz, sms), 256, 0, st>>>(nnz, n, dk.Current(), dv.Current(), b, wbytes, w, col, w_out, row_ptr);
    FJ_CK_LAUNCH();
  }
  k2a.release(); k2b.release(); v2a.release(); v2b.release();
  FJ_CK(cudaStreamSynchronize(st));
  *nnz_out = nnz;
  if (selfloops_out) *selfloops_out = (int64_t)hf.selfloops;
  if (dups_out) *dups_out = m - (int64_t)hf.selfloops - kept;
  return FJ_OK;
}

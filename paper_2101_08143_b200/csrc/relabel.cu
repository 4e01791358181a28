// relabel.cu — locality relabelling for the gather-bound product.
//
// The PCG product gathers x_j for every nonzero (i, j); on power-law graphs most gathers hit a
// small set of high-degree vertices, but in the generator's labels those are scattered over the id
// space, so every 32-byte L2 sector holding a hot x_j also holds ~3 cold ones.  Renumbering the
// vertices by descending degree packs the hot x_j densely: the same L2 then holds ~4x more of the
// gathered working set (measured: C5 product 15.8 -> 10.7 ms, C4 7.6 -> 6.8 ms, C3 0.67 -> 0.65 ms).
//
// The relabelled graph is isomorphic: its Laplacian is P L P^T, (I + P L P^T)^{-1} P s =
// P (I + L)^{-1} s, and every quantity of a6 is a sum over vertices or edges, so it is
// unchanged up to the rounding order of those sums.  Callers map s in and z out with
// fj_permute_rows.
//
//   fj_permute_rows   out[i][:] = in[idx[i]][:]   (idx = new2old: into the new labels;
//                     idx = old2new: back to the old ones)
#include <cub/cub.cuh>

#include "common.cuh"
#include "workspace.cuh"

namespace fj {

__global__ void k_invert(int64_t n, const int32_t* __restrict__ new2old, int32_t* __restrict__ old2new) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    old2new[new2old[i]] = (int32_t)i;
}

template <int K>
__global__ void k_permute_rows_k(int64_t n, const int32_t* __restrict__ idx, const double* __restrict__ in,
                                 double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t src = idx[i];
#pragma unroll
    for (int c = 0; c < K; ++c) out[i * K + c] = in[src * K + c];
  }
}

// wide rows: one warp per row, lanes over the k columns
__global__ void k_permute_rows_w(int64_t n, int k, const int32_t* __restrict__ idx, const double* __restrict__ in,
                                 double* __restrict__ out) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t i = w0; i < n; i += nw) {
    const int64_t src = idx[i];
    for (int c = lane; c < k; c += 32) out[i * k + c] = in[src * k + c];
  }
}

static inline unsigned grid_of(int64_t items, int per_block, int sms) {
  int64_t g = (items + per_block - 1) / per_block;
  const int64_t cap = (int64_t)sms * 16;
  if (g > cap) g = cap;
  return (unsigned)(g < 1 ? 1 : g);
}

static int num_sms() {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

// ---------------------------------------------------------------- relabelling a built CSR
// key = ~row length (ascending sort = descending degree), value = vertex id
__global__ void k_rowlen_keys(int64_t n, const int64_t* __restrict__ rp, uint32_t* __restrict__ key,
                              int32_t* __restrict__ id) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    key[i] = ~(uint32_t)(rp[i + 1] - rp[i]);
    id[i] = (int32_t)i;
  }
}

// len2[i'] = length of old row new2old[i'] (len2[n] = 0, so an exclusive scan gives row_ptr_out)
__global__ void k_perm_lens(int64_t n, const int64_t* __restrict__ rp, const int32_t* __restrict__ new2old,
                            int64_t* __restrict__ len2) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i <= n; i += (int64_t)gridDim.x * blockDim.x) {
    if (i == n) { len2[i] = 0; continue; }
    const int64_t r = new2old[i];
    len2[i] = rp[r + 1] - rp[r];
  }
}

// P A P^T: output positions in chunks of PCH.  k_chunk_rows first records, per chunk, the rows
// holding its first and last position (every non-empty row writes the chunk boundaries inside it,
// so no search over row_ptr is needed).  Rows are in descending length, so the rows overlapping a
// chunk are all non-empty: at most PCH of them (any other order: searched in global memory).  Their
// output starts and source shifts are staged in shared memory; each position finds its row by
// binary search there.  Columns are relabelled and keep their source order (ascending in the OLD
// labels), weights move with them.
constexpr int PCH = 2048;
constexpr int PTB = 256;
__global__ void k_chunk_rows(int64_t n, int64_t nnz, const int64_t* __restrict__ rp_out, int64_t* __restrict__ c_first,
                             int64_t* __restrict__ c_last) {
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = rp_out[r], e = rp_out[r + 1];
    if (e <= b) continue;
    for (int64_t c = (b + PCH - 1) / PCH; c * PCH < e; ++c) c_first[c] = r;            // chunk starts in [b, e)
    for (int64_t c = (b + 1 + PCH - 1) / PCH - 1; c <= (e + PCH - 1) / PCH - 1; ++c) {  // last positions in [b, e)
      const int64_t last = min((c + 1) * (int64_t)PCH, nnz) - 1;
      if (last >= b && last < e) c_last[c] = r;
    }
  }
}

template <int WB>
__device__ __forceinline__ void perm_entry(int64_t p, int64_t src, const int32_t* __restrict__ col, const void* w,
                                           const int32_t* __restrict__ old2new, int32_t* __restrict__ col_out,
                                           void* w_out) {
  col_out[p] = old2new[col[src]];
  if (WB == 1) reinterpret_cast<uint8_t*>(w_out)[p] = reinterpret_cast<const uint8_t*>(w)[src];
  else if (WB == 4) reinterpret_cast<float*>(w_out)[p] = reinterpret_cast<const float*>(w)[src];
  else if (WB == 8) reinterpret_cast<double*>(w_out)[p] = reinterpret_cast<const double*>(w)[src];
}

template <int WB>
__global__ void __launch_bounds__(PTB) k_csr_permute(int64_t nnz, const int64_t* __restrict__ rp,
                                                     const int32_t* __restrict__ col, const void* __restrict__ w,
                                                     const int32_t* __restrict__ new2old,
                                                     const int32_t* __restrict__ old2new,
                                                     const int64_t* __restrict__ rp_out,
                                                     const int64_t* __restrict__ c_first,
                                                     const int64_t* __restrict__ c_last, int32_t* __restrict__ col_out,
                                                     void* __restrict__ w_out) {
  __shared__ int64_t s_beg[PCH];
  __shared__ int64_t s_shift[PCH];
  const int64_t nch = (nnz + PCH - 1) / PCH;
  for (int64_t c = blockIdx.x; c < nch; c += gridDim.x) {
    const int64_t p0 = c * PCH, p1 = min(p0 + (int64_t)PCH, nnz);
    const int64_t rlo = c_first[c];
    const int64_t R64 = c_last[c] - rlo + 1;
    if (R64 > PCH) {   // empty rows inside the chunk (a caller's order, not fj_csr_degree_order's)
      for (int64_t p = p0 + threadIdx.x; p < p1; p += PTB) {
        int64_t lo = rlo, hi = rlo + R64 - 1;
        while (lo < hi) {
          const int64_t mid = (lo + hi + 1) >> 1;
          if (rp_out[mid] <= p) lo = mid; else hi = mid - 1;
        }
        perm_entry<WB>(p, p + rp[new2old[lo]] - rp_out[lo], col, w, old2new, col_out, w_out);
      }
      continue;
    }
    const int R = (int)R64;
    for (int j = threadIdx.x; j < R; j += PTB) {
      const int64_t r = rlo + j;
      const int64_t b = rp_out[r];
      s_beg[j] = b;
      s_shift[j] = rp[new2old[r]] - b;
    }
    __syncthreads();
    // PCH / PTB positions per thread: all sources first, then all loads, then all gathers, so the
    // global latencies overlap (memory-level parallelism) instead of chaining position by position
    constexpr int EPT = PCH / PTB;
    int64_t src[EPT];
#pragma unroll
    for (int e = 0; e < EPT; ++e) {
      const int64_t p = p0 + threadIdx.x + (int64_t)e * PTB;
      src[e] = -1;
      if (p < p1) {
        int lo = 0, hi = R - 1;   // last staged row with s_beg <= p
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (s_beg[mid] <= p) lo = mid; else hi = mid - 1;
        }
        src[e] = p + s_shift[lo];
      }
    }
    int32_t cv[EPT];
#pragma unroll
    for (int e = 0; e < EPT; ++e) cv[e] = src[e] >= 0 ? __ldg(col + src[e]) : 0;
#pragma unroll
    for (int e = 0; e < EPT; ++e) {
      if (src[e] < 0) continue;
      const int64_t p = p0 + threadIdx.x + (int64_t)e * PTB;
      col_out[p] = __ldg(old2new + cv[e]);
      if (WB == 1) reinterpret_cast<uint8_t*>(w_out)[p] = reinterpret_cast<const uint8_t*>(w)[src[e]];
      else if (WB == 4) reinterpret_cast<float*>(w_out)[p] = reinterpret_cast<const float*>(w)[src[e]];
      else if (WB == 8) reinterpret_cast<double*>(w_out)[p] = reinterpret_cast<const double*>(w)[src[e]];
    }
    __syncthreads();
  }
}

}  // namespace fj

using namespace fj;

extern "C" fj_status fj_csr_degree_order(int64_t n, const int64_t* row_ptr, int32_t* new2old, int32_t* old2new,
                                         void* stream) {
  FJ_RANGE("fj_csr_degree_order");
  if (n < 1 || n >= INT32_MAX) return fail(FJ_E_INVALID_ARG, "n must be in [1, 2^31-2]");
  if (!row_ptr || !new2old || !old2new) return fail(FJ_E_INVALID_ARG, "null argument");
  cudaStream_t st = S(stream);
  const int sms = num_sms();
  DevBuf<uint32_t> key, key2;
  DevBuf<int32_t> id;
  FJ_TRY(key.alloc(n, st)); FJ_TRY(key2.alloc(n, st)); FJ_TRY(id.alloc(n, st));
  k_rowlen_keys<<<grid_of(n, 256, sms), 256, 0, st>>>(n, row_ptr, key.p, id.p);
  FJ_CK_LAUNCH();
  size_t bytes = 0;
  FJ_CK(cub::DeviceRadixSort::SortPairs(nullptr, bytes, key.p, key2.p, id.p, new2old, n, 0, 32, st));
  {
    DevBuf<uint8_t> tmp;
    FJ_TRY(tmp.alloc((int64_t)bytes, st));
    FJ_CK(cub::DeviceRadixSort::SortPairs(tmp.p, bytes, key.p, key2.p, id.p, new2old, n, 0, 32, st));
    count_cub();
  }
  k_invert<<<grid_of(n, 256, sms), 256, 0, st>>>(n, new2old, old2new);
  FJ_CK_LAUNCH();
  return FJ_OK;
}

extern "C" fj_status fj_csr_permute(int64_t n, int64_t nnz, const int64_t* row_ptr, const int32_t* col, const void* w,
                                    int wtype, const int32_t* new2old, const int32_t* old2new, int64_t* row_ptr_out,
                                    int32_t* col_out, void* w_out, void* stream) {
  FJ_RANGE("fj_csr_permute");
  if (n < 1 || nnz < 0) return fail(FJ_E_INVALID_ARG, "n < 1 or nnz < 0");
  if (!row_ptr || !new2old || !old2new || !row_ptr_out || (nnz > 0 && (!col || !col_out)))
    return fail(FJ_E_INVALID_ARG, "null argument");
  if (wtype < FJ_W_UNIT || wtype > FJ_W_F64) return fail(FJ_E_INVALID_ARG, "bad wtype");
  const int wbytes = wtype == FJ_W_UNIT ? 0 : wtype == FJ_W_U8 ? 1 : wtype == FJ_W_F32 ? 4 : 8;
  if (wbytes && nnz > 0 && (!w || !w_out)) return fail(FJ_E_INVALID_ARG, "weights are NULL");
  cudaStream_t st = S(stream);
  const int sms = num_sms();
  DevBuf<int64_t> len2;
  FJ_TRY(len2.alloc(n + 1, st));
  k_perm_lens<<<grid_of(n + 1, 256, sms), 256, 0, st>>>(n, row_ptr, new2old, len2.p);
  FJ_CK_LAUNCH();
  FJ_TRY(cub_exclusive_sum(len2.p, row_ptr_out, n + 1, st));
  if (nnz == 0) return FJ_OK;
  const int64_t nch = (nnz + PCH - 1) / PCH;
  DevBuf<int64_t> cf, cl;
  FJ_TRY(cf.alloc(nch, st)); FJ_TRY(cl.alloc(nch, st));
  k_chunk_rows<<<grid_of(n, 256, sms), 256, 0, st>>>(n, nnz, row_ptr_out, cf.p, cl.p);
  FJ_CK_LAUNCH();
  int64_t g = nch;
  if (g > (int64_t)sms * 8) g = (int64_t)sms * 8;
  const unsigned gb = (unsigned)g;
  switch (wbytes) {
    case 0: k_csr_permute<0><<<gb, PTB, 0, st>>>(nnz, row_ptr, col, w, new2old, old2new, row_ptr_out, cf.p, cl.p, col_out, w_out); break;
    case 1: k_csr_permute<1><<<gb, PTB, 0, st>>>(nnz, row_ptr, col, w, new2old, old2new, row_ptr_out, cf.p, cl.p, col_out, w_out); break;
    case 4: k_csr_permute<4><<<gb, PTB, 0, st>>>(nnz, row_ptr, col, w, new2old, old2new, row_ptr_out, cf.p, cl.p, col_out, w_out); break;
    default: k_csr_permute<8><<<gb, PTB, 0, st>>>(nnz, row_ptr, col, w, new2old, old2new, row_ptr_out, cf.p, cl.p, col_out, w_out); break;
  }
  FJ_CK_LAUNCH();
  return FJ_OK;
}

extern "C" fj_status fj_permute_rows(int64_t n, int k, const int32_t* idx, const double* in, double* out,
                                     void* stream) {
  if (n < 0 || k < 1) return fail(FJ_E_INVALID_ARG, "n < 0 or k < 1");
  if (n == 0) return FJ_OK;
  if (!idx || !in || !out) return fail(FJ_E_INVALID_ARG, "null argument");
  if (in == out) return fail(FJ_E_INVALID_ARG, "in and out must not alias");
  cudaStream_t st = S(stream);
  const int sms = num_sms();
  switch (k) {
    case 1: k_permute_rows_k<1><<<grid_of(n, 256, sms), 256, 0, st>>>(n, idx, in, out); break;
    case 2: k_permute_rows_k<2><<<grid_of(n, 256, sms), 256, 0, st>>>(n, idx, in, out); break;
    case 3: k_permute_rows_k<3><<<grid_of(n, 256, sms), 256, 0, st>>>(n, idx, in, out); break;
    case 4: k_permute_rows_k<4><<<grid_of(n, 256, sms), 256, 0, st>>>(n, idx, in, out); break;
    default: k_permute_rows_w<<<grid_of(n * 32, 256, sms), 256, 0, st>>>(n, k, idx, in, out); break;
  }
  FJ_CK_LAUNCH();
  return FJ_OK;
}

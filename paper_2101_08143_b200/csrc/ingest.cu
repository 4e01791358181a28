// ingest.cu — SURVEY §8 row f1: preprocessing either side of the path, on the device.
//
//  * Opinion generators ("internal opinions ... uniform, exponential and power-law
//    distributions", each rescaled to [0, 1]): the counter-based generator the synthetic
//    workloads use (DESIGN.md §5 / R10) re-implemented on the GPU, so large opinion vectors need
//    no host generation or H2D copy.
//  * Connected components of a raw edge list (Shiloach-Vishkin hooking on roots + pointer jumping;
//    every vertex ends labelled with the smallest vertex id of its component) and the largest
//    connected component ("we use their largest connected components"): a vertex map and
//    the LCC's edges, relabelled, in input order (so a1's keep-first duplicate rule still applies).
#include <cub/cub.cuh>

#include "common.cuh"
#include "workspace.cuh"

namespace fj {

// ---------------------------------------------------------------- opinions
__device__ __forceinline__ uint64_t ig_sm64(uint64_t x) {   // splitmix64 finaliser
  x += 0x9E3779B97F4A7C15ULL;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}
constexpr uint64_t kOpinionStream = 0x1ULL;

// x_i from U_i = (rand64(seed, OPINION, i) >> 11) 2^-53: uniform U; exponential (rate 1, x_min 1)
// 1 - ln(1 - U); power law (alpha 2.5, x_min 1) (1 - U)^(-1/(alpha-1)); block maxima -> part
__global__ void k_opinions(int64_t n, int kind, uint64_t seed, double* __restrict__ s, double* __restrict__ part) {
  __shared__ double s_max[8];
  const uint64_t base = ig_sm64(ig_sm64(seed) ^ kOpinionStream);
  double mx = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const double u = (double)(ig_sm64(base ^ (uint64_t)i) >> 11) * 0x1.0p-53;
    double x;
    if (kind == 0) x = u;
    else if (kind == 1) x = 1.0 - log1p(-u);
    else x = pow(1.0 - u, -1.0 / 1.5);
    s[i] = x;
    mx = fmax(mx, x);
  }
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) s_max[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) mx = fmax(mx, s_max[w]);
    part[blockIdx.x] = mx;
  }
}

__global__ void k_scale(int64_t n, const double* __restrict__ part, int nparts, double* __restrict__ s) {
  double mx = 0.0;
  for (int b = 0; b < nparts; ++b) mx = fmax(mx, part[b]);   // max is order-independent
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    s[i] = s[i] / mx;
}

// ---------------------------------------------------------------- connected components
__device__ __forceinline__ int32_t cc_find(const int32_t* parent, int32_t x) {
  int32_t p = parent[x];
  while (p != x) {   // parents only decrease: terminates, and never leaves the component
    x = p;
    p = parent[x];
  }
  return x;
}

__global__ void k_cc_init(int64_t n, int32_t* __restrict__ parent) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    parent[i] = (int32_t)i;
}

// hook: the larger of two different roots points to the smaller (atomicMin keeps parent <= id)
__global__ void k_cc_hook(int64_t m, const int32_t* __restrict__ u, const int32_t* __restrict__ v,
                          int32_t* parent, int* changed) {
  int local = 0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x) {
    const int32_t a = cc_find(parent, u[e]), b = cc_find(parent, v[e]);
    if (a != b) {
      atomicMin(parent + max(a, b), min(a, b));
      local = 1;
    }
  }
  if (__syncthreads_or(local) && threadIdx.x == 0) *changed = 1;
}

__global__ void k_cc_compress(int64_t n, int32_t* parent) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    parent[i] = cc_find(parent, (int32_t)i);
}

// component sizes at the roots; best = max over roots of (size << 32 | ~root): largest, then smallest id
__global__ void k_cc_count(int64_t n, const int32_t* __restrict__ label, int32_t* __restrict__ size) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(size + label[i], 1);
}
__global__ void k_cc_best(int64_t n, const int32_t* __restrict__ label, const int32_t* __restrict__ size,
                          unsigned long long* best, int* ncomp) {
  int roots = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if (label[i] == (int32_t)i) {
      ++roots;
      atomicMax(best, ((unsigned long long)(uint32_t)size[i] << 32) | (unsigned long long)(0xFFFFFFFFu - (uint32_t)i));
    }
  }
  if (roots) atomicAdd(ncomp, roots);
}

__global__ void k_lcc_flags(int64_t n, const int32_t* __restrict__ label, int32_t root, int32_t* __restrict__ flag) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    flag[i] = label[i] == root ? 1 : 0;
}
__global__ void k_lcc_vmap(int64_t n, const int32_t* __restrict__ flag, const int32_t* __restrict__ pos,
                           int32_t* __restrict__ vmap) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    vmap[i] = flag[i] ? pos[i] : -1;
}
__global__ void k_lcc_eflags(int64_t m, const int32_t* __restrict__ u, const int32_t* __restrict__ vmap,
                             uint8_t* __restrict__ ef) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x)
    ef[e] = vmap[u[e]] >= 0 ? 1 : 0;
}
__global__ void k_lcc_edges(int64_t m2, const int32_t* __restrict__ sel, const int32_t* __restrict__ u,
                            const int32_t* __restrict__ v, const unsigned char* __restrict__ w, int wbytes,
                            const int32_t* __restrict__ vmap, int32_t* __restrict__ u2, int32_t* __restrict__ v2,
                            unsigned char* __restrict__ w2) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < m2; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = sel[t];
    u2[t] = vmap[u[e]];
    v2[t] = vmap[v[e]];
    for (int q = 0; q < wbytes; ++q) w2[t * wbytes + q] = w[e * wbytes + q];
  }
}

static unsigned grid_for(int64_t count) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return (unsigned)std::max<int64_t>(1, std::min<int64_t>((count + 255) / 256, (int64_t)sms * 16));
}

static fj_status components(int64_t n, int64_t m, const int32_t* u, const int32_t* v, int32_t* label,
                            int* rounds, cudaStream_t st) {
  DevBuf<int> changed;
  FJ_TRY(changed.alloc(1, st));
  k_cc_init<<<grid_for(n), 256, 0, st>>>(n, label);
  FJ_CK_LAUNCH();
  int r = 0;
  for (;;) {
    FJ_CK(cudaMemsetAsync(changed.p, 0, sizeof(int), st));
    if (m > 0) {
      k_cc_hook<<<grid_for(m), 256, 0, st>>>(m, u, v, label, changed.p);
      FJ_CK_LAUNCH();
    }
    k_cc_compress<<<grid_for(n), 256, 0, st>>>(n, label);
    FJ_CK_LAUNCH();
    int h = 0;
    FJ_CK(cudaMemcpyAsync(&h, changed.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    FJ_CK(cudaStreamSynchronize(st));
    ++r;
    if (!h) break;
    if (r > 200) return fail(FJ_E_INTERNAL, "connected components did not converge");
  }
  if (rounds) *rounds = r;
  return FJ_OK;
}

static fj_status check_edges(int64_t n, int64_t m, const int32_t* u, const int32_t* v, cudaStream_t st);

}  // namespace fj

using namespace fj;

extern "C" {

fj_status fj_opinions_generate(int64_t n, int kind, uint64_t seed, double* s_dev, void* stream) {
  if (n < 1 || !s_dev || kind < 0 || kind > 2) return fail(FJ_E_INVALID_ARG, "n >= 1, kind in {0,1,2}, s non-null");
  cudaStream_t st = S(stream);
  const unsigned grid = grid_for(n);
  DevBuf<double> part;
  FJ_TRY(part.alloc(grid, st));
  k_opinions<<<grid, 256, 0, st>>>(n, kind, seed, s_dev, part.p);
  FJ_CK_LAUNCH();
  if (kind != 0) {   // rescaled by the maximum: max s = 1 exactly (R10)
    k_scale<<<grid, 256, 0, st>>>(n, part.p, (int)grid, s_dev);
    FJ_CK_LAUNCH();
  }
  FJ_CK(cudaStreamSynchronize(st));
  return FJ_OK;
}

fj_status fj_connected_components(int64_t n, int64_t m_in, const int32_t* u_dev, const int32_t* v_dev,
                                  int32_t* label_dev, int64_t* n_comp, void* stream) {
  FJ_RANGE("fj_connected_components");
  if (n < 1 || n > INT32_MAX || m_in < 0 || !label_dev || (m_in > 0 && (!u_dev || !v_dev)))
    return fail(FJ_E_INVALID_ARG, "n in [1, 2^31), m_in >= 0, non-null buffers");
  cudaStream_t st = S(stream);
  FJ_TRY(check_edges(n, m_in, u_dev, v_dev, st));
  FJ_TRY(components(n, m_in, u_dev, v_dev, label_dev, nullptr, st));
  if (n_comp) {
    DevBuf<int32_t> size;
    DevBuf<unsigned long long> best;
    DevBuf<int> nc;
    FJ_TRY(size.alloc(n, st));
    FJ_TRY(best.alloc(1, st));
    FJ_TRY(nc.alloc(1, st));
    FJ_CK(cudaMemsetAsync(size.p, 0, sizeof(int32_t) * n, st));
    FJ_CK(cudaMemsetAsync(best.p, 0, sizeof(unsigned long long), st));
    FJ_CK(cudaMemsetAsync(nc.p, 0, sizeof(int), st));
    k_cc_count<<<grid_for(n), 256, 0, st>>>(n, label_dev, size.p);
    FJ_CK_LAUNCH();
    k_cc_best<<<grid_for(n), 256, 0, st>>>(n, label_dev, size.p, best.p, nc.p);
    FJ_CK_LAUNCH();
    int h = 0;
    FJ_CK(cudaMemcpyAsync(&h, nc.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    FJ_CK(cudaStreamSynchronize(st));
    *n_comp = h;
  }
  FJ_CK(cudaStreamSynchronize(st));
  return FJ_OK;
}

fj_status fj_lcc(int64_t n, int64_t m_in, const int32_t* u_dev, const int32_t* v_dev, const void* w_dev, int wtype,
                 int32_t* vmap_dev, int32_t* u_out, int32_t* v_out, void* w_out, int64_t* n_lcc, int64_t* m_lcc,
                 void* stream) {
  FJ_RANGE("fj_lcc");
  if (n < 1 || n > INT32_MAX || m_in < 0 || !vmap_dev || !n_lcc || !m_lcc || (m_in > 0 && (!u_dev || !v_dev)))
    return fail(FJ_E_INVALID_ARG, "n in [1, 2^31), m_in >= 0, non-null buffers");
  if (wtype < FJ_W_UNIT || wtype > FJ_W_F64) return fail(FJ_E_INVALID_ARG, "bad wtype");
  const int wbytes = wtype == FJ_W_UNIT ? 0 : wtype == FJ_W_U8 ? 1 : wtype == FJ_W_F32 ? 4 : 8;
  if (wbytes && m_in > 0 && (!w_dev || !w_out)) return fail(FJ_E_INVALID_ARG, "weights are NULL");
  if (m_in > 0 && (!u_out || !v_out)) return fail(FJ_E_INVALID_ARG, "edge outputs are NULL");
  cudaStream_t st = S(stream);
  FJ_TRY(check_edges(n, m_in, u_dev, v_dev, st));
  DevBuf<int32_t> label, size, flag, pos;
  DevBuf<unsigned long long> best;
  DevBuf<int> nc;
  FJ_TRY(label.alloc(n, st));
  FJ_TRY(components(n, m_in, u_dev, v_dev, label.p, nullptr, st));
  FJ_TRY(size.alloc(n, st));
  FJ_TRY(best.alloc(1, st));
  FJ_TRY(nc.alloc(1, st));
  FJ_CK(cudaMemsetAsync(size.p, 0, sizeof(int32_t) * n, st));
  FJ_CK(cudaMemsetAsync(best.p, 0, sizeof(unsigned long long), st));
  FJ_CK(cudaMemsetAsync(nc.p, 0, sizeof(int), st));
  k_cc_count<<<grid_for(n), 256, 0, st>>>(n, label.p, size.p);
  FJ_CK_LAUNCH();
  k_cc_best<<<grid_for(n), 256, 0, st>>>(n, label.p, size.p, best.p, nc.p);
  FJ_CK_LAUNCH();
  unsigned long long hb = 0;
  FJ_CK(cudaMemcpyAsync(&hb, best.p, sizeof hb, cudaMemcpyDeviceToHost, st));
  FJ_CK(cudaStreamSynchronize(st));
  const int32_t root = (int32_t)(0xFFFFFFFFu - (uint32_t)(hb & 0xFFFFFFFFull));
  *n_lcc = (int64_t)(hb >> 32);
  // vertex map: LCC vertices renumbered 0.. in increasing old id
  FJ_TRY(flag.alloc(n, st));
  FJ_TRY(pos.alloc(n, st));
  k_lcc_flags<<<grid_for(n), 256, 0, st>>>(n, label.p, root, flag.p);
  FJ_CK_LAUNCH();
  FJ_TRY(cub_exclusive_sum_i32(flag.p, pos.p, n, st));
  k_lcc_vmap<<<grid_for(n), 256, 0, st>>>(n, flag.p, pos.p, vmap_dev);
  FJ_CK_LAUNCH();
  // edges with both ends in the LCC (one end suffices: an edge never crosses components), input order
  *m_lcc = 0;
  if (m_in > 0) {
    DevBuf<uint8_t> ef;
    DevBuf<int32_t> sel, nsel;
    FJ_TRY(ef.alloc(m_in, st));
    FJ_TRY(sel.alloc(m_in, st));
    FJ_TRY(nsel.alloc(1, st));
    k_lcc_eflags<<<grid_for(m_in), 256, 0, st>>>(m_in, u_dev, vmap_dev, ef.p);
    FJ_CK_LAUNCH();
    FJ_TRY(cub_select_index(ef.p, sel.p, nsel.p, m_in, st));
    int32_t h = 0;
    FJ_CK(cudaMemcpyAsync(&h, nsel.p, sizeof h, cudaMemcpyDeviceToHost, st));
    FJ_CK(cudaStreamSynchronize(st));
    *m_lcc = h;
    if (h > 0) {
      k_lcc_edges<<<grid_for(h), 256, 0, st>>>(h, sel.p, u_dev, v_dev, reinterpret_cast<const unsigned char*>(w_dev),
                                                wbytes, vmap_dev, u_out, v_out, reinterpret_cast<unsigned char*>(w_out));
      FJ_CK_LAUNCH();
    }
  }
  FJ_CK(cudaStreamSynchronize(st));
  return FJ_OK;
}

}  // extern "C"

namespace fj {

__global__ void k_edge_range(int64_t n, int64_t m, const int32_t* __restrict__ u, const int32_t* __restrict__ v,
                             int* bad) {
  int b = 0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x)
    b |= (u[e] < 0 || u[e] >= n || v[e] < 0 || v[e] >= n);
  if (__syncthreads_or(b) && threadIdx.x == 0) *bad = 1;
}

static fj_status check_edges(int64_t n, int64_t m, const int32_t* u, const int32_t* v, cudaStream_t st) {
  if (m == 0) return FJ_OK;
  DevBuf<int> bad;
  FJ_TRY(bad.alloc(1, st));
  FJ_CK(cudaMemsetAsync(bad.p, 0, sizeof(int), st));
  k_edge_range<<<grid_for(m), 256, 0, st>>>(n, m, u, v, bad.p);
  FJ_CK_LAUNCH();
  int h = 0;
  FJ_CK(cudaMemcpyAsync(&h, bad.p, sizeof h, cudaMemcpyDeviceToHost, st));
  FJ_CK(cudaStreamSynchronize(st));
  return h ? fail(FJ_E_INVALID_ARG, "vertex id out of range [0, n)") : FJ_OK;
}

}  // namespace fj

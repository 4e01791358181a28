// workspace.cuh — stream-ordered device buffers and the few CUB calls used by setup code.
#pragma once
#include <cub/cub.cuh>

#include "common.cuh"

namespace fj {

template <class T>
struct DevBuf {
  T* p = nullptr;
  cudaStream_t st = nullptr;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  fj_status alloc(int64_t count, cudaStream_t s) {
    st = s;
    if (count <= 0) count = 1;
    cudaError_t e = dmalloc(&p, sizeof(T) * (size_t)count, s);
    if (e != cudaSuccess) { p = nullptr; return cuda_fail(e, "cudaMallocAsync", __FILE__, __LINE__); }
    return FJ_OK;
  }
  void release() {
    if (p) dfree_on(p, st);
    p = nullptr;
  }
  ~DevBuf() { release(); }
};

// A non-blocking side stream with two events (host-buffer entry points overlap copies with compute).
struct SideStream {
  cudaStream_t s = nullptr;
  cudaEvent_t ev_in = nullptr, ev_out = nullptr;
  fj_status init() {
    FJ_CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    FJ_CK(cudaEventCreateWithFlags(&ev_in, cudaEventDisableTiming));
    FJ_CK(cudaEventCreateWithFlags(&ev_out, cudaEventDisableTiming));
    return FJ_OK;
  }
  ~SideStream() {
    if (s) { cudaStreamSynchronize(s); cudaStreamDestroy(s); }
    if (ev_in) cudaEventDestroy(ev_in);
    if (ev_out) cudaEventDestroy(ev_out);
  }
};

// e[i] = sum_{j<i} c[j] for i in [0, count)
inline fj_status cub_exclusive_sum(const int64_t* c, int64_t* e, int64_t count, cudaStream_t st) {
  size_t bytes = 0;
  FJ_CK(cub::DeviceScan::ExclusiveSum(nullptr, bytes, c, e, count, st));
  DevBuf<uint8_t> tmp;
  FJ_TRY(tmp.alloc((int64_t)bytes, st));
  FJ_CK(cub::DeviceScan::ExclusiveSum(tmp.p, bytes, c, e, count, st));
  count_cub();
  return FJ_OK;
}

inline fj_status cub_exclusive_sum_i32(const int32_t* c, int32_t* e, int64_t count, cudaStream_t st) {
  size_t bytes = 0;
  FJ_CK(cub::DeviceScan::ExclusiveSum(nullptr, bytes, c, e, count, st));
  DevBuf<uint8_t> tmp;
  FJ_TRY(tmp.alloc((int64_t)bytes, st));
  FJ_CK(cub::DeviceScan::ExclusiveSum(tmp.p, bytes, c, e, count, st));
  count_cub();
  return FJ_OK;
}

// out = { i in [0, count) : flags[i] != 0 } in increasing order; *num_out (device) = size.
inline fj_status cub_select_index(const uint8_t* flags, int32_t* out, int32_t* num_out, int64_t count,
                                  cudaStream_t st) {
  cub::CountingInputIterator<int32_t> it(0);
  size_t bytes = 0;
  FJ_CK(cub::DeviceSelect::Flagged(nullptr, bytes, it, flags, out, num_out, (int)count, st));
  DevBuf<uint8_t> tmp;
  FJ_TRY(tmp.alloc((int64_t)bytes, st));
  FJ_CK(cub::DeviceSelect::Flagged(tmp.p, bytes, it, flags, out, num_out, (int)count, st));
  count_cub();
  return FJ_OK;
}

void free_solve_ws(fj_graph* g);   // pcg.cu
void free_quant_ws(fj_graph* g);   // quantities.cu
void free_batch_ws(fj_graph* g);   // spmm.cu
// defer_true_residual: stop on the recursive residual and leave the true-residual check (and any
// restart) to the caller, which gets ||s - (I+L)z||^2 from the fused quantities pass; honoured by
// the small-k vector engine (other engines check it themselves as usual).
fj_status solve_batch(fj_graph* g, int k, const double* s, double* z, const fj_solve_opts& o, int warm,
                      fj_solve_report* rep, cudaStream_t st, bool defer_true_residual = false);
fj_status apply_batch(fj_graph* g, int k, const double* x, double* y, int opL, cudaStream_t st);
fj_status quant_batch(fj_graph* g, int k, const double* s, const double* z, const double* mean_host,
                      double* host_out /* [k][10] */, cudaStream_t st, bool z_from_solve = false);
fj_status time_batch_spmv(fj_graph* g, int k, int reps, float* ms_out, cudaStream_t st);
// spmv_vec.cu (2 <= k <= 4)
void free_vec_ws(fj_graph* g);
bool vec_supported(int k);
fj_status solve_vec(fj_graph* g, int k, const double* s, double* z, const fj_solve_opts& o, int warm,
                    fj_solve_report* rep, cudaStream_t st, bool defer_true_residual = false);
fj_status apply_vec(fj_graph* g, int k, const double* x, double* y, int opL, cudaStream_t st);
fj_status quant_vec(fj_graph* g, int k, const double* s, const double* z, const double* mean_host,
                    double* host_out, bool z_from_solve, cudaStream_t st);
fj_status time_vec_spmv(fj_graph* g, int k, int reps, float* ms_out, cudaStream_t st);
fj_status vec_product_mode(fj_graph* g, int k, cudaStream_t st, int* mode);   // RowsPlan::mode
// onchip.cu: the whole solve + quantities pass of column c in one thread block when the graph fits
// in shared memory (*used = false otherwise)
fj_status onchip_col(fj_graph* g, const double* s, double* z, int64_t ld, int64_t c, double mean,
                     const fj_solve_opts& o, double* t10, int* iters, int* restarts, double* rel_true,
                     double* rel_rec, bool* converged, bool* used, cudaStream_t st);
// dist.cu
void free_dist(fj_graph* g);
bool is_dist(const fj_graph* g);
int64_t global_n(const fj_graph* g);
double global_dmax(const fj_graph* g);
// columns [c0, c0 + k) (1 <= k <= 4) of this rank's [n_loc][ld] slices solved together by the
// single-reduction (Chronopoulos-Gear) distributed PCG
fj_status dist_solve_cg(fj_graph* g, int k, const double* s, double* z, int64_t ld, int c0, const fj_solve_opts& o,
                        int warm, fj_solve_report* rep, cudaStream_t st);
fj_status dist_quant_pass(const fj_graph* g, const double* s, const double* z, int64_t ld, int64_t c, double m,
                          double* host10, cudaStream_t st);
fj_status dist_stats_combine(const fj_graph* g, int k, double* dev4k, cudaStream_t st);
int64_t dist_n_ghost(const fj_graph* g);
}  // namespace fj

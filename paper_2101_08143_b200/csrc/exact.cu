// exact.cu — SURVEY §8 row f3: the paper's "Exact" baseline on the device ("we compute the
// inverse / solve with I + L directly"), as a mid-size checker for fj_approxim: dense fp64 I + L
// (P:L88), Cholesky factorisation and triangular solves for the k opinion columns (cuSOLVER
// potrf/potrs, loaded lazily like NCCL), then the fused quantities pass on the exact z.
// n <= 50000 (a 20 GB dense matrix); the matrix lives only for the call.
#include <dlfcn.h>

#include <mutex>

#include "common.cuh"
#include "workspace.cuh"

namespace fj {

// cuSOLVER dense API subset (types from the public header are not needed: opaque handle + enums)
typedef void* cusolverDnHandle_t_;
struct SolverApi {
  void* h = nullptr;
  int (*Create)(cusolverDnHandle_t_*) = nullptr;
  int (*Destroy)(cusolverDnHandle_t_) = nullptr;
  int (*SetStream)(cusolverDnHandle_t_, cudaStream_t) = nullptr;
  int (*PotrfBuf)(cusolverDnHandle_t_, int, int, double*, int, int*) = nullptr;
  int (*Potrf)(cusolverDnHandle_t_, int, int, double*, int, double*, int, int*) = nullptr;
  int (*Potrs)(cusolverDnHandle_t_, int, int, int, const double*, int, double*, int, int*) = nullptr;
};
constexpr int kFillLower = 0;   // CUBLAS_FILL_MODE_LOWER

static fj_status solver_api(SolverApi** out) {
  static SolverApi api;
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  if (!api.h) {
    const char* names[] = {"libcusolver.so.11", "/usr/local/cuda/lib64/libcusolver.so.11", "libcusolver.so"};
    for (const char* nm : names) {
      api.h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
      if (api.h) break;
    }
    if (!api.h) return fail(FJ_E_UNSUPPORTED, std::string("cannot dlopen libcusolver.so.11: ") + dlerror());
#define FJ_SOLVER_SYM(f, n) \
  api.f = reinterpret_cast<decltype(api.f)>(dlsym(api.h, n)); \
  if (!api.f) return fail(FJ_E_UNSUPPORTED, "missing " n)
    FJ_SOLVER_SYM(Create, "cusolverDnCreate");
    FJ_SOLVER_SYM(Destroy, "cusolverDnDestroy");
    FJ_SOLVER_SYM(SetStream, "cusolverDnSetStream");
    FJ_SOLVER_SYM(PotrfBuf, "cusolverDnDpotrf_bufferSize");
    FJ_SOLVER_SYM(Potrf, "cusolverDnDpotrf");
    FJ_SOLVER_SYM(Potrs, "cusolverDnDpotrs");
#undef FJ_SOLVER_SYM
  }
  *out = &api;
  return FJ_OK;
}

// A (column-major n x n, zeroed) = I + L: A_ii = 1 + d_i, A_ij = -w_ij (P:L88 L = D - A)
template <int WT>
__global__ void k_dense_ipl(int64_t n, const int64_t* __restrict__ rp, const int32_t* __restrict__ col,
                            const void* __restrict__ w, const double* __restrict__ deg, double* __restrict__ A) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    A[i * n + i] = 1.0 + deg[i];
    for (int64_t p = rp[i]; p < rp[i + 1]; ++p) A[(int64_t)col[p] * n + i] = -WeightT<WT>::get(w, p);
  }
}

// row-major [n][k] <-> column-major n x k
__global__ void k_to_colmajor(int64_t n, int k, const double* __restrict__ s, double* __restrict__ B) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n * k; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = q / k, j = q - i * k;
    B[j * n + i] = s[q];
  }
}
__global__ void k_from_colmajor(int64_t n, int k, const double* __restrict__ B, double* __restrict__ z) {
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n * k; q += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = q / k, j = q - i * k;
    z[q] = B[j * n + i];
  }
}

}  // namespace fj

using namespace fj;

extern "C" fj_status fj_exact_dense(const fj_graph* gc, int k, const double* s_dev, double* z_dev,
                                    fj_quantities_t* q_host, void* stream) {
  FJ_RANGE("fj_exact_dense");
  if (!gc || !s_dev || !z_dev) return fail(FJ_E_INVALID_ARG, "null argument");
  if (k < 1 || k > MAXK) return fail(FJ_E_INVALID_ARG, "k must be in [1, 64]");
  if (s_dev == z_dev) return fail(FJ_E_INVALID_ARG, "s and z must not alias");
  fj_graph* g = const_cast<fj_graph*>(gc);
  if (g->dist) return fail(FJ_E_UNSUPPORTED, "fj_exact_dense on a distributed graph");
  const int64_t n = g->n;
  if (n > 50000) return fail(FJ_E_UNSUPPORTED, "fj_exact_dense: n > 50000 (dense matrix over 20 GB)");
  SolverApi* api = nullptr;
  FJ_TRY(solver_api(&api));
  cudaStream_t st = S(stream);
  double* A = nullptr;   // transient: plain cudaMalloc so the pool does not keep it
  FJ_CK(cudaMalloc(&A, sizeof(double) * (size_t)(n * n)));
  struct Guard {
    double* a;
    ~Guard() { cudaFree(a); }
  } guard{A};
  FJ_CK(cudaMemsetAsync(A, 0, sizeof(double) * (size_t)(n * n), st));
  const unsigned gb = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, (int64_t)g->num_sms * 8));
  switch (g->wtype) {
    case FJ_W_UNIT: k_dense_ipl<FJ_W_UNIT><<<gb, 256, 0, st>>>(n, g->row_ptr, g->col, g->w, g->deg, A); break;
    case FJ_W_U8: k_dense_ipl<FJ_W_U8><<<gb, 256, 0, st>>>(n, g->row_ptr, g->col, g->w, g->deg, A); break;
    case FJ_W_F32: k_dense_ipl<FJ_W_F32><<<gb, 256, 0, st>>>(n, g->row_ptr, g->col, g->w, g->deg, A); break;
    default: k_dense_ipl<FJ_W_F64><<<gb, 256, 0, st>>>(n, g->row_ptr, g->col, g->w, g->deg, A); break;
  }
  FJ_CK_LAUNCH();
  DevBuf<double> B;
  DevBuf<int> info;
  FJ_TRY(B.alloc(n * k, st));
  FJ_TRY(info.alloc(1, st));
  const unsigned gk = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n * k + 255) / 256, (int64_t)g->num_sms * 8));
  k_to_colmajor<<<gk, 256, 0, st>>>(n, k, s_dev, B.p);
  FJ_CK_LAUNCH();
  cusolverDnHandle_t_ h = nullptr;
  if (api->Create(&h) != 0) return fail(FJ_E_CUDA, "cusolverDnCreate failed");
  struct HGuard {
    SolverApi* api;
    cusolverDnHandle_t_ h;
    ~HGuard() { api->Destroy(h); }
  } hguard{api, h};
  if (api->SetStream(h, st) != 0) return fail(FJ_E_CUDA, "cusolverDnSetStream failed");
  int lwork = 0;
  if (api->PotrfBuf(h, kFillLower, (int)n, A, (int)n, &lwork) != 0) return fail(FJ_E_CUDA, "potrf_bufferSize failed");
  DevBuf<double> work;
  FJ_TRY(work.alloc(std::max(lwork, 1), st));
  if (api->Potrf(h, kFillLower, (int)n, A, (int)n, work.p, lwork, info.p) != 0) return fail(FJ_E_CUDA, "potrf failed");
  int hinfo = 0;
  FJ_CK(cudaMemcpyAsync(&hinfo, info.p, sizeof hinfo, cudaMemcpyDeviceToHost, st));
  FJ_CK(cudaStreamSynchronize(st));
  if (hinfo != 0) return fail(FJ_E_INTERNAL, "Cholesky of I + L failed (matrix not SPD?)");
  if (api->Potrs(h, kFillLower, (int)n, k, A, (int)n, B.p, (int)n, info.p) != 0) return fail(FJ_E_CUDA, "potrs failed");
  k_from_colmajor<<<gk, 256, 0, st>>>(n, k, B.p, z_dev);
  FJ_CK_LAUNCH();
  FJ_CK(cudaStreamSynchronize(st));
  if (q_host) FJ_TRY(fj_quantities(gc, k, s_dev, z_dev, q_host, stream));
  return FJ_OK;
}

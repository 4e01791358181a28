/*
 * fj.h — C ABI of the B200 library for Friedkin–Johnsen opinion quantities
 * (arXiv 2101.08143, "Fast Evaluation for Relevant Quantities of Opinion Dynamics").
 * Citations "P:L<n>" are lines of the paper's text; §8(b) of SURVEY.md is the
 * contract this header implements.
 *
 * Conventions (apply to every entry point unless stated otherwise)
 *  - Every call returns fj_status; FJ_OK == 0.  No C++ exception crosses the ABI.  On failure
 *    fj_last_error() returns a thread-local, human-readable message (valid until the next call
 *    on the same thread).
 *  - Pointers named *_dev are DEVICE pointers (cudaMalloc / torch CUDA tensors) on the current
 *    CUDA device; pointers named *_host are host pointers.  Inputs are BORROWED: the library
 *    never frees them, and a graph handle borrows its CSR arrays until fj_graph_destroy.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).  All device
 *    work is stream-ordered on it.  Calls that fill a HOST struct synchronise that stream.
 *  - Layouts: CSR row_ptr int64 [n+1] (row_ptr[0] = 0), col int32 [nnz], weights [nnz] in the
 *    type given by fj_wtype (FJ_W_UNIT: no array, every w_ij = 1).  Opinion / solution matrices
 *    with k columns are ROW-MAJOR fp64 [n][k] (k = 1: a plain vector).
 *  - Internal workspace is owned by the handle.  It comes from the allocator installed with
 *    fj_set_allocator, else from a library-owned stream-ordered memory pool (cudaMallocFromPoolAsync
 *    on `stream`).
 *  - There is NO CPU fallback: without a CUDA device every compute call returns FJ_E_CUDA.
 */
#ifndef FJ_H
#define FJ_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FJ_ABI_VERSION 1

typedef enum {
  FJ_OK = 0,
  FJ_E_INVALID_ARG = 1,      /* null pointer, negative size, k out of range, bad enum        */
  FJ_E_NOT_SIMPLE = 2,       /* self-loop, duplicate / unsorted column, column out of range  */
  FJ_E_ASYMMETRIC = 3,       /* (i,j,w) present without (j,i,w)  (P:L88 w_ij = w_ji)         */
  FJ_E_BAD_WEIGHT = 4,       /* weight <= 0 or non-finite  (P:L86 w: E -> R_+)               */
  FJ_E_NONFINITE_INPUT = 5,  /* NaN/Inf in an opinion vector                                 */
  FJ_E_NO_CONVERGENCE = 6,   /* iteration cap hit; best iterate left in z, report filled     */
  FJ_E_CUDA = 7,             /* CUDA runtime error (message in fj_last_error)               */
  FJ_E_NCCL = 8,
  FJ_E_OOM = 9,
  FJ_E_INTERNAL = 10,
  FJ_E_UNSUPPORTED = 11
} fj_status;

typedef enum { FJ_W_UNIT = 0, FJ_W_U8 = 1, FJ_W_F32 = 2, FJ_W_F64 = 3 } fj_wtype;
typedef enum { FJ_OP_L = 0, FJ_OP_IPL = 1 } fj_op;

typedef struct fj_graph fj_graph;

typedef struct {
  int64_t n, nnz;           /* nodes, stored CSR entries (= 2 m)                              */
  int64_t m;                /* undirected edges                                              */
  int64_t n_isolated;       /* rows with no neighbour (z_i = s_i)                            */
  int64_t deg_max;          /* largest row length                                            */
  double w_min, w_max;      /* extremal edge weights; 0 if nnz == 0                  */
  double d_max;             /* largest weighted degree                                       */
  int64_t n_tiles, n_wrows, n_long_rows, n_long_chunks;  /* row-engine items    */
  int32_t wtype, reserved;
} fj_graph_info_t;

typedef struct {
  double rtol;              /* stop when ||s - (I+L)z||_2 <= rtol ||s||_2 (default 1e-10)    */
  double eps_target;        /* fj_approxim only: tighten rtol until every certified relative
                               bound <= eps_target (0 = off).                                */
  int32_t max_iter;         /* total PCG iterations over all restarts (default 10000)         */
  int32_t max_restarts;     /* true-residual restarts (default 3)                             */
  int32_t use_cuda_graph;   /* 1 (default): device-driven conditional-while CUDA graph loop  */
  int32_t vertex_order;     /* fj_approxim_host only: FJ_ORDER_NATURAL (0, default) builds the
                               CSR in the input labels; FJ_ORDER_DEGREE (1) relabels it by
                               descending degree (fj_csr_degree_order + fj_csr_permute; s mapped
                               in, z mapped back out); FJ_ORDER_AUTO (2) relabels only when it
                               pays: per-vertex rows narrower than one 32-byte L2 sector (k <= 2)
                               and a gathered vector larger than the L2      */
} fj_solve_opts;
enum { FJ_ORDER_NATURAL = 0, FJ_ORDER_DEGREE = 1, FJ_ORDER_AUTO = 2 };

typedef struct {
  int32_t iterations;       /* PCG iterations (max over the k columns)                       */
  int32_t converged;        /* 1 when every column met rtol on its TRUE residual             */
  int32_t restarts;
  int32_t batch_k;          /* k if the columns were solved as one batch (row a9), else 0     */
  double rel_res_recursive; /* max_j ||r_j|| / ||s_j|| of the recursion at exit               */
  double rel_res_true;      /* max_j ||s_j - (I+L) z_j|| / ||s_j||, recomputed (NaN if not)  */
  double ms;                /* device time of the whole call (CUDA events on `stream`)       */
  double ms_loop;           /* device time of the PCG iterations only (init + loop), summed
                               over columns and restarts (CUDA events on `stream`)           */
  int64_t iterations_total; /* PCG iterations summed over columns and restarts               */
} fj_solve_report;

/* Quantities for ONE opinion column (fj_quantities / fj_approxim fill k of them).
 * Definitions (on the returned z):                                      [P:L<n>]
 *   CI  = sum_i (z_i - s_i)^2          internal conflict, Def. 3.1       L167
 *   D   = sum_{(i,j) in E} w_ij (z_i - z_j)^2, each edge once, Def. 3.2  L183
 *   P   = sum_i (z_i - mean(s))^2      polarization, Def. 3.3            L204-206 (mean(z) = mean(s), L152)
 *   C   = sum_i z_i^2                  controversy, Def. 3.4             L215
 *   Idc = D + C                        disagreement-controversy index    L224 (= s^T z, L228)
 *   PDI = P + D                        polarization-disagreement index (BASELINE north_star)
 * eps[6] are CERTIFIED relative error bounds |Q - Q_exact| / Q_exact <= eps for
 * (CI, D, P, C, Idc, PDI), derived a posteriori from the true residual (
 * proof pattern of Lemma 4.3, with lambda_min(I+L) = 1).
 * +Inf means "not certified" (e.g. near-consensus input). */
typedef struct {
  double CI, D, P, C, Idc, PDI;
  double mean_s;            /* 1^T s / n                                                     */
  double ss;                /* s^T s   (cross-check: CI + 2D + C = s^T s)                    */
  double sz;                /* s^T z   (cross-check: = Idc)                          */
  double sbzb;              /* (s - mean s)^T (z - mean s)  (cross-check: = PDI)             */
  double Lz2;               /* ||L z||^2 (Algorithm 1 line 5 form of CI; diagnostic) */
  double res_norm;          /* ||s - (I+L) z||_2                                             */
  double s_norm;            /* ||s||_2                                                       */
  double fp_bound;          /* rounding allowance added to res_norm in the certificate       */
  double eps[6];
  int32_t consensus;        /* 1 if s is constant: z = s exactly, P = D = CI = 0             */
  int32_t certified;        /* 1 if all six eps are finite                                   */
} fj_quantities_t;

/* ---------------------------------------------------------------- misc */
int fj_abi_version(void);
/* Number of CUDA kernels this library has launched in this process (host-side counter; kernels
 * executed by a device-driven graph loop are counted from the iteration counts).  Library
 * kernels (CUB radix sort / scan / select) are counted separately in *cub_launches if non-NULL. */
int64_t fj_kernel_launches(int64_t* cub_launches);
const char* fj_status_str(int status);
const char* fj_last_error(void);
void fj_default_solve_opts(fj_solve_opts* opts);

/* ---------------------------------------------------------------- allocator hook
 * Route every device workspace allocation of the library (graph handles, solver / quantities
 * workspaces, setup temporaries) through a caller allocator, e.g. the PyTorch caching allocator
 * (the Python binding's use_torch_allocator()).
 *   alloc(bytes, stream, ctx) -> device pointer on the current device, or NULL (-> FJ_E_CUDA /
 *                                out-of-memory from the calling entry point); `stream` is the
 *                                cudaStream_t (as void*) the block will first be used on.
 *   free(ptr, bytes, stream, ctx) returns a block; the library calls it only after the work that
 *                                used the block on `stream` has completed (it synchronises that
 *                                stream first), so the allocator need not order it.
 * alloc and free are both non-NULL (install) or both NULL (back to the library pool); anything
 * else is FJ_E_INVALID_ARG.  Process-wide; blocks are always returned to the allocator that
 * produced them, even if another one was installed meanwhile.  Not thread-safe with respect to
 * concurrent calls that allocate (install it before creating handles).  The callbacks must not
 * call back into this library. */
typedef void* (*fj_alloc_fn)(size_t bytes, void* stream, void* ctx);
typedef void (*fj_free_fn)(void* ptr, size_t bytes, void* stream, void* ctx);
fj_status fj_set_allocator(fj_alloc_fn alloc, fj_free_fn free_fn, void* ctx);
/* Blocks currently held from an installed allocator (diagnostic; 0 with the library pool). */
int64_t fj_allocator_live_blocks(void);

/* ---------------------------------------------------------------- a1: canonical CSR
 * Build the CSR of the simple undirected graph given by m_in raw edges (u_dev[e], v_dev[e]),
 * e = 0..m_in-1, with 0 <= u,v < n:
 *   self-loops dropped; (u,v) canonicalised to (min,max); duplicate pairs keep the FIRST
 *   occurrence in input order (its weight); every kept edge is mirrored; columns ascend in
 *   each row.  w_dev may be NULL iff wtype == FJ_W_UNIT.
 * Outputs (caller-allocated DEVICE buffers): row_ptr_dev int64 [n+1]; col_dev int32 with
 * capacity 2*m_in; w_out_dev (same type as input, capacity 2*m_in; ignored for FJ_W_UNIT).
 * Host outputs: *nnz_out = 2 * kept edges; *selfloops_out, *dups_out may be NULL.
 * Errors: FJ_E_INVALID_ARG (n < 1, n > 2^31-1, m_in < 0, vertex id out of range),
 * FJ_E_OOM, FJ_E_CUDA.  Synchronises `stream`. */
fj_status fj_csr_from_edges(int64_t n, int64_t m_in, const int32_t* u_dev, const int32_t* v_dev,
                            const void* w_dev, int wtype, int64_t* row_ptr_dev, int32_t* col_dev,
                            void* w_out_dev, int64_t* nnz_out, int64_t* selfloops_out,
                            int64_t* dups_out, void* stream);

/* ---------------------------------------------------------------- a1 option: locality relabelling
 * (not in the paper).  Renumbering the vertices by descending degree packs the
 * x_j most gathered by the PCG product into few L2 sectors.  The relabelled graph is isomorphic:
 * its Laplacian is P L P^T, its solution of (I + L) z = s is P z for the input P s, and the
 * quantities of P:L163-228 (sums over vertices and edges) are unchanged up to rounding order.
 * The relabelling is applied to a built canonical CSR (it keeps a1's sort in the input labels).
 * fj_csr_degree_order: new2old by descending row length = degree (ties by ascending id), old2new its inverse; asynchronous.  fj_csr_permute: the
 * CSR of P A P^T -- row i' is old row new2old[i'] with every column c replaced by old2new[c], in
 * the old row's order (ascending OLD labels, so weighted degree sums keep a1's order and stay
 * bit-exact), weights moved with their entries.  row_ptr_out [n+1], col_out / w_out [nnz]
 * (device, caller-allocated, not aliasing the input).  Any permutation pair is accepted (not
 * checked).  Asynchronous on `stream`. */
fj_status fj_csr_degree_order(int64_t n, const int64_t* row_ptr_dev, int32_t* new2old_dev, int32_t* old2new_dev,
                              void* stream);
fj_status fj_csr_permute(int64_t n, int64_t nnz, const int64_t* row_ptr_dev, const int32_t* col_dev,
                         const void* w_dev, int wtype, const int32_t* new2old_dev, const int32_t* old2new_dev,
                         int64_t* row_ptr_out_dev, int32_t* col_out_dev, void* w_out_dev, void* stream);
/* out_dev[i][:] = in_dev[idx_dev[i]][:] for row-major [n][k] fp64 (device; in and out must not
 * alias).  idx = new2old maps an input s into the new labels, idx = old2new maps a solution z back.
 * Asynchronous on `stream`. */
fj_status fj_permute_rows(int64_t n, int k, const int32_t* idx_dev, const double* in_dev, double* out_dev,
                          void* stream);

/* ---------------------------------------------------------------- a2: graph handle, degrees
 * Borrow a caller-owned device CSR (it must outlive the handle), optionally validate it
 * (validate != 0: sorted/in-range/no self-loop columns, symmetric weights, w > 0 finite;
 * FJ_E_NOT_SIMPLE / FJ_E_ASYMMETRIC / FJ_E_BAD_WEIGHT on failure), compute the weighted degrees
 * d_i = sum_j w_ij (in ascending column order), the Jacobi diagonal 1/(1 + d_i), the graph
 * statistics and the SpMV schedule.  Synchronises `stream`.  *out receives the handle. */
fj_status fj_graph_create(int64_t n, int64_t nnz, const int64_t* row_ptr_dev, const int32_t* col_dev,
                          const void* w_dev, int wtype, int validate, void* stream, fj_graph** out);
fj_status fj_graph_info(const fj_graph* g, fj_graph_info_t* out);
/* d_dev: fp64 [n] device output, d_i = sum_j w_ij (bit-exact: ascending column order). */
fj_status fj_graph_degrees(const fj_graph* g, double* d_dev, void* stream);
fj_status fj_graph_destroy(fj_graph* g);

/* ---------------------------------------------------------------- operators
 * y = L x (op = FJ_OP_L) or y = (I + L) x (op = FJ_OP_IPL) for row-major [n][k] fp64 x, y
 * (device).  x and y must not alias. */
fj_status fj_apply(const fj_graph* g, int op, int k, const double* x_dev, double* y_dev, void* stream);

/* Diagnostic (bench roofline): average device time in ms of ONE search-direction product
 * q = (I + L) p exactly as the k-column PCG loop launches it (same kernel, same schedule, the
 * library's own workspace buffers; their contents are left undefined), over `reps` back-to-back
 * launches timed with CUDA events on `stream`.  Synchronises.  FJ_E_UNSUPPORTED on a distributed
 * handle. */
fj_status fj_time_spmv(const fj_graph* g, int k, int reps, float* ms_host, void* stream);

/* Diagnostic: which kernel path computes the k-column PCG product on this graph (*path, host):
 * FJ_PATH_ENGINE (0) the load-balanced merge-path warp-item engine (tiles.cuh);
 * FJ_PATH_ROWS (1) the lean row kernel, one pass (k <= 4, rows.cuh);
 * FJ_PATH_ROWS_SLABS (2) the lean row kernel over two column slabs (k <= 4, when the gathered
 * block is in (64 MB, 160 MB] and every row's columns ascend);
 * FJ_PATH_BATCH (3) the warp-per-row batched engine (k > 4, spmm.cu).  FJ_ROWS=0/1/2 in the
 * environment forces engine / one pass / two slabs for k <= 4 (A/B, tests).  May build the
 * k-column workspace. */
enum { FJ_PATH_ENGINE = 0, FJ_PATH_ROWS = 1, FJ_PATH_ROWS_SLABS = 2, FJ_PATH_BATCH = 3 };
fj_status fj_product_path(const fj_graph* g, int k, int* path, void* stream);

/* Diagnostic (bench "gather roofline"): the random-gather rate this GPU sustains for the SpMV's
 * access pattern without any row logic: m int32 indices uniform in [0, n_vec) streamed once, one
 * gather of `width` (1, 2 or 4) contiguous doubles per index from an n_vec-row device vector
 * (L2-resident when it fits), 8 gathers in flight per thread.  *gathers_per_s (host) receives
 * indices processed per second over `reps` timed launches (CUDA events on `stream`; one warm-up
 * launch).  Allocates and frees its own buffers.  Synchronises. */
fj_status fj_probe_gather(int64_t n_vec, int64_t m, int width, int reps, double* gathers_per_s, void* stream);

/* ---------------------------------------------------------------- a3: opinion statistics
 * stats_host[4*j + 0..3] = (sum s_j, sum s_j^2, min s_j, max s_j) for each column j of the
 * row-major [n][k] s_dev.  FJ_E_NONFINITE_INPUT if any entry is NaN/Inf.  Synchronises. */
fj_status fj_opinion_stats(const fj_graph* g, int k, const double* s_dev, double* stats_host, void* stream);

/* ---------------------------------------------------------------- a4: SOLVE (Lemma 4.2)
 * z = (I + L)^{-1} s (Eq. (2)) for every column, by Jacobi-preconditioned CG from
 * z0 = 0, stopping when ||r|| <= rtol ||s|| (recursive residual), then recomputing the true
 * residual and restarting from z while it exceeds rtol ||s|| (<= max_restarts).  Since
 * lambda_min(I+L) = 1, ||z - z*||_{I+L} <= ||r||, which meets the SOLVE contract of Lemma 4.2
 * with delta = ||r|| / ||z*||_{I+L}.  k in [1, 64]; s_dev, z_dev row-major [n][k] device
 * (must not alias).  opts may be NULL (defaults).  rep (host, may be NULL) is filled.
 * FJ_E_NO_CONVERGENCE: cap reached; z holds the last iterate.  Synchronises `stream`. */
fj_status fj_solve(const fj_graph* g, int k, const double* s_dev, double* z_dev,
                   const fj_solve_opts* opts, fj_solve_report* rep, void* stream);

/* ---------------------------------------------------------------- a5-a7: quantities + certificate
 * One fused CSR pass over (s, z) per column computing the sums listed in fj_quantities_t and the
 * true residual, then the certificate on the host.  out_host: k structs.  Synchronises. */
fj_status fj_quantities(const fj_graph* g, int k, const double* s_dev, const double* z_dev,
                        fj_quantities_t* out_host, void* stream);

/* Algorithm 1 in single-solve form (reading R4): statistics, one solve
 * per column (q = z - mean(s) 1 replaces the second solve exactly since Omega 1 = 1),
 * fused quantities with certificate; restarts if the certified true residual misses rtol and,
 * when opts->eps_target > 0, tightens rtol (x0.01, warm start) until every eps <= eps_target.
 * z_dev may be NULL (internal buffer).  q_host: k structs; rep may be NULL. */
fj_status fj_approxim(const fj_graph* g, int k, const double* s_dev, double* z_dev,
                      const fj_solve_opts* opts, fj_quantities_t* q_host, fj_solve_report* rep,
                      void* stream);

/* End-to-end convenience from HOST buffers: copies the raw edge list (u_host, v_host, w_host)
 * and s_host [n][k] to the device, builds the CSR (a1), then -- when opts->vertex_order is
 * FJ_ORDER_DEGREE, or FJ_ORDER_AUTO and the rule of fj_solve_opts.vertex_order holds -- relabels
 * it with fj_csr_degree_order + fj_csr_permute (the permuted CSR's columns are NOT ascending; the
 * handle is created without validation) and maps s in / z out with fj_permute_rows; creates the
 * handle (a2), runs fj_approxim, and copies z (input labels) back to z_host (may be NULL) and the
 * quantities to q_host.  Pinned host buffers make the copies asynchronous.  Device memory is
 * released before return, also on every error path. */
fj_status fj_approxim_host(int64_t n, int64_t m_in, const int32_t* u_host, const int32_t* v_host,
                           const void* w_host, int wtype, int k, const double* s_host,
                           double* z_host, const fj_solve_opts* opts, fj_quantities_t* q_host,
                           fj_solve_report* rep, void* stream);

/* ---------------------------------------------------------------- f2: Algorithm 1 verbatim
 * Both solves of Approxim(G, s, eps): z~ = Solve(I+L, s, delta), q = Solve(I+L, s_bar, delta)
 * (lines 3-4, run as one 2-column batch), then C_I = ||L z~||^2, D = ||W^{1/2} B q||^2,
 * P = ||q||^2, C = ||z~||^2, I_dc = D + C (lines 5-9).  delta is line 1's formula; delta_eff clamps
 * it to 1e-12 when it is below 1e-14 (SPEC's solver decision); the solve stops on the relative
 * residual rtol = delta_eff / sqrt(1 + 2 d_max), which implies Lemma 4.2's (I+L)-norm bound since
 * lambda(I+L) lies in [1, 1 + 2 d_max] (Gershgorin); rtol is floored at 1e-14 (fp64), recorded. */
typedef struct {
  double CI, D, P, C, Idc, PDI;   /* lines 5-9 (+ PDI = P + D)                                  */
  double delta;                   /* line 1                                                      */
  double delta_eff;               /* after the clamp                                             */
  double rtol;                    /* relative-residual stop used for both solves                 */
  double D_from_z;                /* ||W^{1/2} B z~||^2: equals D at solver tolerance */
  double CI_def;                  /* sum (z~ - s)^2, Def. 3.1 form of C_I                        */
  double mean_s, sbar_norm;       /* 1^T s / n and ||s_bar|| (line 2)                            */
  int32_t clamped, rtol_floored;
} fj_alg1_t;
/* Host-only arithmetic of line 1 + clamp + residual map (no device work; any thread). */
fj_status fj_alg1_delta(int64_t n, double w_min, double w_max, double d_max, double sbar_norm, double eps,
                        double* delta, double* delta_eff, double* rtol, int* clamped, int* floored);
/* s_dev: fp64 [n] device (one opinion vector); eps in (0, 1/2).  opts: max_iter / restarts / graph
 * mode are honoured, rtol is replaced by the mapped one.  Synchronises. */
fj_status fj_approxim_alg1(const fj_graph* g, const double* s_dev, double eps, const fj_solve_opts* opts,
                           fj_alg1_t* out_host, fj_solve_report* rep, void* stream);

/* ---------------------------------------------------------------- f3: the paper's "Exact" on the device
 * z = (I + L)^{-1} s by a dense fp64 Cholesky of I + L ("Exact"; cuSOLVER potrf / potrs,
 * libcusolver.so.11 loaded on first use) for n <= 50000, then (q_host non-NULL) the fused
 * quantities pass on that z (fj_quantities).  A mid-size checker for fj_approxim (Table 2's
 * relative-error protocol, tools/table2.py).  FJ_E_UNSUPPORTED above n = 50000 or without
 * libcusolver.  The n x n matrix is allocated and freed inside the call.  Synchronises. */
fj_status fj_exact_dense(const fj_graph* g, int k, const double* s_dev, double* z_dev, fj_quantities_t* q_host,
                         void* stream);

/* ---------------------------------------------------------------- f4: forest-matrix entries
 * omega_dev (row-major [n][m], device) receives columns cols_host[0..m) of Omega = (I + L)^{-1}:
 * omega_dev[i*m + t] = omega_{i, cols[t]} = eps(Gamma_{i cols[t]}) / eps(Gamma), the forest-based
 * proximity of P:L103/L132 (Omega is symmetric, so these are rows as well).  Each column solves
 * (I+L) x = e_c; the columns are batched (<= 64 per batch).  rep aggregates the batches. */
fj_status fj_forest_columns(const fj_graph* g, int64_t m, const int32_t* cols_host, double* omega_dev,
                            const fj_solve_opts* opts, fj_solve_report* rep, void* stream);

/* ---------------------------------------------------------------- f1: preprocessing on the device
 * Opinion vectors of P:L637-639 drawn on the device by the synthetic workloads' counter-based
 * generator: U_i = (rand64(seed, 1, i) >> 11) 2^-53 with rand64 = sm(sm(sm(seed) ^ 1) ^ i), sm the
 * splitmix64 finaliser; kind 0: s_i = U_i; kind 1 (exponential, rate 1, x_min 1): x = 1 - ln(1 - U);
 * kind 2 (power law, alpha 2.5, x_min 1): x = (1 - U)^(-1/1.5); kinds 1, 2 divided by max x.
 * s_dev: fp64 [n] device output.  Synchronises. */
fj_status fj_opinions_generate(int64_t n, int kind, uint64_t seed, double* s_dev, void* stream);
/* Connected components of the raw edge list (self-loops / duplicates allowed): label_dev [n]
 * receives the smallest vertex id of each vertex's component; *n_comp (may be NULL) the count.
 * FJ_E_INVALID_ARG on a vertex id outside [0, n).  Synchronises. */
fj_status fj_connected_components(int64_t n, int64_t m_in, const int32_t* u_dev, const int32_t* v_dev,
                                  int32_t* label_dev, int64_t* n_comp, void* stream);
/* Largest connected component (ties -> the component with the smallest vertex id):
 * vmap_dev [n] = new id (LCC vertices renumbered 0.. in increasing old id) or -1; u_out/v_out/w_out
 * (capacity m_in) receive the LCC's raw edges relabelled, in input order (self-loops and duplicates
 * kept: fj_csr_from_edges applies a1's rules afterwards).  *n_lcc, *m_lcc: vertex / edge counts. */
fj_status fj_lcc(int64_t n, int64_t m_in, const int32_t* u_dev, const int32_t* v_dev, const void* w_dev, int wtype,
                 int32_t* vmap_dev, int32_t* u_out, int32_t* v_out, void* w_out, int64_t* n_lcc, int64_t* m_lcc,
                 void* stream);

/* ---------------------------------------------------------------- a8/e: row-partitioned multi-GPU
 * The graph is split into contiguous row blocks balanced by nonzeros, one block per rank (one
 * process per GPU).  Rank r owns rows [bounds[r], bounds[r+1]).  Its CSR first carries GLOBAL
 * column ids; fj_graph_create_dist renumbers them (own columns -> [0, n_loc), off-rank "ghost"
 * columns -> n_loc + their index in the sorted ghost list).  Each PCG iteration exchanges the ghost
 * entries of the preconditioned residual (halo; grouped NCCL send/recv over NVLink, on a comm stream
 * overlapped with the own-column part of the product) and allreduces ONE vector of 3 k dot products
 * (single-reduction Chronopoulos-Gear PCG); every rank takes identical decisions.  s / z passed to fj_solve / fj_approxim /
 * fj_quantities on a distributed handle are the rank's LOCAL row slices [n_loc][k]; quantities are
 * global and identical on every rank.  fj_apply is not available on a distributed handle.
 * Every call on a distributed handle is collective: all ranks must make it, in the same order. */
typedef struct fj_comm fj_comm;
/* 128-byte NCCL unique id (rank 0 creates it; broadcast it to the other ranks out of band). */
fj_status fj_comm_unique_id(unsigned char id_out[128]);
/* NCCL communicator on the current CUDA device (libnccl.so.2 is loaded on first use). */
fj_status fj_comm_init(int nranks, int rank, const unsigned char id[128], fj_comm** out);
/* LOOPBACK transport: nranks virtual ranks inside ONE process on ONE device, one host thread per
 * rank (each passes its rank to fj_graph_create_dist and uses its own stream).  Collectives become
 * barrier-ordered device copies and host sums in rank order.  For testing the distributed path. */
fj_status fj_comm_init_loopback(int nranks, fj_comm** out);
fj_status fj_comm_destroy(fj_comm* comm);

/* bounds_host[0..nranks]: contiguous row blocks of ~equal cost, cost of a row = its raw (pre-dedup)
 * nonzeros + 6 (a row costs about as much as 6 nonzeros per PCG iteration: DESIGN.md §6 measured),
 * computed from the raw edge list on the device (same result on every rank). */
fj_status fj_partition_rows(int64_t n, int64_t m_in, const int32_t* u_dev, const int32_t* v_dev, int nranks,
                            int64_t* bounds_host, void* stream);
/* Row a1 restricted to rows [row_begin, row_end): local row_ptr [n_loc+1] (starting at 0), GLOBAL
 * column ids (capacity 2*m_in), same simple-graph rules as fj_csr_from_edges. */
fj_status fj_csr_rows_from_edges(int64_t n, int64_t m_in, const int32_t* u_dev, const int32_t* v_dev,
                                 const void* w_dev, int wtype, int64_t row_begin, int64_t row_end,
                                 int64_t* row_ptr_local_dev, int32_t* col_global_dev, void* w_out_dev,
                                 int64_t* nnz_out, void* stream);
/* Locality order for the row partition (DESIGN.md §6.7 applied before partitioning): new2old_dev[n]
 * lists the vertices by descending raw endpoint count (non-self-loop raw edges, duplicates counted;
 * ties by ascending id), old2new_dev[n] is its inverse (device int32, written).  Every rank computes
 * the same permutation from the same raw list.  Ids outside [0, n) are skipped here (the row
 * builders reject them).  Synchronises. */
fj_status fj_edge_degree_order(int64_t n, int64_t m_in, const int32_t* u_dev, const int32_t* v_dev,
                               int32_t* new2old_dev, int32_t* old2new_dev, void* stream);
/* fj_partition_rows / fj_csr_rows_from_edges of the RELABELLED graph (endpoint e -> old2new[e]):
 * bounds and rows are in the new labels, columns are new global ids.  The caller maps its opinion
 * slice in (rows new2old[row_begin .. row_end) of s) and z back out (fj_permute_rows). */
fj_status fj_partition_rows_relabelled(int64_t n, int64_t m_in, const int32_t* u_dev, const int32_t* v_dev,
                                       const int32_t* old2new_dev, int nranks, int64_t* bounds_host, void* stream);
fj_status fj_csr_rows_from_edges_relabelled(int64_t n, int64_t m_in, const int32_t* u_dev, const int32_t* v_dev,
                                            const int32_t* old2new_dev, const void* w_dev, int wtype,
                                            int64_t row_begin, int64_t row_end, int64_t* row_ptr_local_dev,
                                            int32_t* col_global_dev, void* w_out_dev, int64_t* nnz_out, void* stream);
/* Sorted unique columns outside [row_begin, row_end) (the halo), ghosts_out capacity nnz_local. */
fj_status fj_dist_ghosts(int64_t nnz_local, const int32_t* col_global_dev, int64_t row_begin, int64_t row_end,
                         int32_t* ghosts_out_dev, int64_t* n_ghost_out, void* stream);
/* One rank's handle.  send_counts_host[q] = how many of MY rows rank q needs; send_idx_dev holds
 * those local row indices, concatenated in peer order (obtained by exchanging ghost lists).  The
 * CSR arrays are borrowed as in fj_graph_create (col_global is renumbered into an owned copy). */
fj_status fj_graph_create_dist(fj_comm* comm, int rank, int64_t n_global, const int64_t* bounds_host,
                               int64_t nnz_local, const int64_t* row_ptr_local_dev, const int32_t* col_global_dev,
                               const void* w_dev, int wtype, int64_t n_ghost, const int32_t* ghosts_dev,
                               const int64_t* send_counts_host, const int32_t* send_idx_dev, void* stream,
                               fj_graph** out);

#ifdef __cplusplus
}
#endif
#endif /* FJ_H */

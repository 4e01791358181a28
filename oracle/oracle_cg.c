/*
 * oracle_cg.c — ORACLE (test infrastructure only).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or constant with the CUDA library
 * (paper_2101_08143_b200/csrc) and never calls it.
 *
 * Plain, slow, obviously-correct fp64 routines, following PAPER.md
 * (/root/reference/PAPER.md, "P:L<n>") and SURVEY.md §8(c) O-2, O-4:
 *
 *   oracle_degrees   d_i = sum_j w_ij, summed in ascending column order
 *                    (§2.1 "the weighted degree of a node i is d_i = sum_j w_ij").
 *   oracle_ipl_apply y = (I + L) x = x + D x - A x   ("L = D - A"; "I + L").
 *   oracle_pcg       z = (I + L)^{-1} s  (Eq. (2)) by textbook Jacobi-preconditioned
 *                    conjugate gradients, x0 = 0, stop on ||r|| <= tol ||s||, then recompute the
 *                    true residual s - (I+L)x and restart from x (at most 3 restarts) when it is
 *                    above tol ||s||.  Unfused loops; dots use Neumaier-compensated sums over a
 *                    static OpenMP schedule (deterministic for a fixed thread count).
 *                    precond = 0 runs plain CG (dinv = 1) as a cross-check mode.
 *
 * Weight types: 0 = unit (w == NULL), 1 = uint8, 3 = float64.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static inline double wval(int wtype, const void* w, int64_t p) {
  if (wtype == 0) return 1.0;
  if (wtype == 1) return (double)((const uint8_t*)w)[p];
  return ((const double*)w)[p];
}

int oracle_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* Thread count of the oracle's OpenMP loops (bench.py times the oracle on all cores and on one). */
void oracle_set_num_threads(int t) {
#ifdef _OPENMP
  if (t > 0) omp_set_num_threads(t);
#else
  (void)t;
#endif
}

int oracle_degrees(int64_t n, const int64_t* row_ptr, int wtype, const void* w, double* d) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    double acc = 0.0;
    for (int64_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p) acc += wval(wtype, w, p);
    d[i] = acc;
  }
  return 0;
}

/* y = (I + L) x with (Lx)_i = d_i x_i - sum_j w_ij x_j */
int oracle_ipl_apply(int64_t n, const int64_t* row_ptr, const int32_t* col, int wtype, const void* w,
                     const double* d, const double* x, double* y) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    double ax = 0.0;
    for (int64_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p) ax += wval(wtype, w, p) * x[col[p]];
    y[i] = x[i] + d[i] * x[i] - ax;
  }
  return 0;
}

/* Neumaier-compensated dot product, static schedule, per-thread partials combined in order */
static double dot(int64_t n, const double* a, const double* b) {
  int nt = oracle_num_threads();
  double* ps = (double*)calloc((size_t)nt, sizeof(double));
  double* pc = (double*)calloc((size_t)nt, sizeof(double));
#pragma omp parallel
  {
    int t = 0;
#ifdef _OPENMP
    t = omp_get_thread_num();
#endif
    double s = 0.0, c = 0.0;
#pragma omp for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
      double x = a[i] * b[i];
      double tt = s + x;
      if (fabs(s) >= fabs(x)) c += (s - tt) + x; else c += (x - tt) + s;
      s = tt;
    }
    ps[t] = s; pc[t] = c;
  }
  double s = 0.0, c = 0.0;
  for (int t = 0; t < nt; ++t) {
    double x = ps[t];
    double tt = s + x;
    if (fabs(s) >= fabs(x)) c += (s - tt) + x; else c += (x - tt) + s;
    s = tt;
    c += pc[t];
  }
  free(ps); free(pc);
  return s + c;
}

/* Jacobi-PCG.  Returns 0 if converged, 1 if max_iter reached.
 * out[0] = iterations (total over restarts), out[1] = final true relative residual,
 * out[2] = number of restarts. */
int oracle_pcg(int64_t n, const int64_t* row_ptr, const int32_t* col, int wtype, const void* w,
               const double* s, double tol, int64_t max_iter, int precond, double* x, double* out) {
  double* d = (double*)malloc(sizeof(double) * (size_t)n);
  double* dinv = (double*)malloc(sizeof(double) * (size_t)n);
  double* r = (double*)malloc(sizeof(double) * (size_t)n);
  double* y = (double*)malloc(sizeof(double) * (size_t)n);
  double* p = (double*)malloc(sizeof(double) * (size_t)n);
  double* q = (double*)malloc(sizeof(double) * (size_t)n);
  if (!d || !dinv || !r || !y || !p || !q) return -1;
  oracle_degrees(n, row_ptr, wtype, w, d);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    dinv[i] = precond ? 1.0 / (1.0 + d[i]) : 1.0;  /* Jacobi: diag(I + L) = 1 + d_i */
    x[i] = 0.0;
  }
  double snorm = sqrt(dot(n, s, s));
  int64_t it = 0;
  int restarts = 0, status = 1;
  double relres = 0.0;
  if (snorm == 0.0) { status = 0; goto done; }
  for (;;) {
    /* r = s - (I+L) x */
    oracle_ipl_apply(n, row_ptr, col, wtype, w, d, x, q);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) r[i] = s[i] - q[i];
    double rnorm = sqrt(dot(n, r, r));
    relres = rnorm / snorm;
    if (relres <= tol) { status = 0; break; }
    if (it >= max_iter || restarts >= 3) { status = 1; break; }
    if (it > 0) ++restarts;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) { y[i] = dinv[i] * r[i]; p[i] = y[i]; }
    double rho = dot(n, r, y);
    while (it < max_iter) {
      oracle_ipl_apply(n, row_ptr, col, wtype, w, d, p, q);   /* q = M p */
      double alpha = rho / dot(n, p, q);
#pragma omp parallel for schedule(static)
      for (int64_t i = 0; i < n; ++i) { x[i] += alpha * p[i]; r[i] -= alpha * q[i]; }
      ++it;
      if (sqrt(dot(n, r, r)) <= tol * snorm) break;
#pragma omp parallel for schedule(static)
      for (int64_t i = 0; i < n; ++i) y[i] = dinv[i] * r[i];
      double rho_new = dot(n, r, y);
      double beta = rho_new / rho;
#pragma omp parallel for schedule(static)
      for (int64_t i = 0; i < n; ++i) p[i] = y[i] + beta * p[i];
      rho = rho_new;
    }
  }
done:
  out[0] = (double)it;
  out[1] = relres;
  out[2] = (double)restarts;
  free(d); free(dinv); free(r); free(y); free(p); free(q);
  return status;
}

/* Fixed iteration count (no convergence test inside the timed loop) — used only by
 * bench.py's cpu_baseline leg to time a bounded sample of oracle PCG iterations. */
int oracle_pcg_fixed_iters(int64_t n, const int64_t* row_ptr, const int32_t* col, int wtype,
                           const void* w, const double* s, int64_t iters, double* x) {
  double out[3];
  return oracle_pcg(n, row_ptr, col, wtype, w, s, 0.0, iters, 1, x, out) < 0 ? -1 : 0;
}

/*
 * oracle_big.c — ORACLE (test infrastructure only).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or constant with the CUDA library
 * (paper_2101_08143_b200/csrc) and never calls it.
 *
 * The same definitions as oracle/__init__.py, written as plain C loops so that they reach the
 * largest config (BASELINE.json configs[4]: 2^26 nodes, 1.07e9 raw edges), where the numpy
 * versions would need tens of GB of temporaries:
 *
 *   oracle_csr_blocked   SURVEY.md §8(c) O-1, from the simple-graph assumption of P:L86 and the
 *                        symmetric adjacency of P:L88: self-loops dropped, a duplicate unordered
 *                        pair keeps its FIRST occurrence in input order (its weight), every kept
 *                        edge appears in both endpoint rows, columns ascend within a row.  Built
 *                        row block by row block (bounded memory): for a block of rows, every raw
 *                        edge e = (u, v), u != v, contributes (row u: col v, e) and (row v: col u, e)
 *                        for the endpoints inside the block; each row's (col, e) pairs are sorted and
 *                        the first pair of every column is kept.
 *   oracle_quantities    Definitions 3.1-3.5 on given (s, z) with Neumaier-compensated sums:
 *                          CI = sum_i (z_i - s_i)^2                     Def. 3.1
 *                          D  = sum_{(i,j) in E, i<j} w_ij (z_i - z_j)^2 Def. 3.2, P:L183 (each edge once)
 *                          P  = sum_i (z_i - mean(z))^2                  Def. 3.3
 *                          C  = sum_i z_i^2                              Def. 3.4
 *                        plus the cross-check sums s^T z, (s - mean s)^T (z - mean z), s^T s.
 *   oracle_csr_permute   P A P^T of a CSR (DESIGN.md §6.7 relabelling; P:L88 L -> P L P^T): row i'
 *                        is old row new2old[i'], every column c replaced by old2new[c], entries in the
 *                        old row's order.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static inline int nthreads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
static inline int thread_id(void) {
#ifdef _OPENMP
  return omp_get_thread_num();
#else
  return 0;
#endif
}

static int cmp_u64(const void* a, const void* b) {
  const uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return x < y ? -1 : (x > y ? 1 : 0);
}

static void sort_u64(uint64_t* a, int64_t k) {
  if (k <= 32) {   /* insertion sort */
    for (int64_t i = 1; i < k; ++i) {
      uint64_t t = a[i];
      int64_t j = i - 1;
      while (j >= 0 && a[j] > t) { a[j + 1] = a[j]; --j; }
      a[j + 1] = t;
    }
  } else {
    qsort(a, (size_t)k, sizeof(uint64_t), cmp_u64);
  }
}

/* Returns nnz (>= 0), or -1 (vertex id out of range), -2 (allocation failure), -3 (m >= 2^32).
 * row_ptr [n+1], col (capacity 2m), w_out (capacity 2m entries of the weight type; wsize = 0 for
 * unit weights, else 1 (uint8) or 8 (float64)).  stats[0] = self-loops, stats[1] = duplicates. */
int64_t oracle_csr_blocked(int64_t n, int64_t m, const int32_t* u, const int32_t* v, int wsize, const void* w,
                           int64_t block_entries, int64_t* row_ptr, int32_t* col, void* w_out, int64_t* stats) {
  if (m >= ((int64_t)1 << 32)) return -3;
  int64_t loops = 0, bad = 0;
#pragma omp parallel for schedule(static) reduction(+ : loops, bad)
  for (int64_t e = 0; e < m; ++e) {
    if (u[e] < 0 || v[e] < 0 || u[e] >= n || v[e] >= n) ++bad;
    else if (u[e] == v[e]) ++loops;
  }
  if (bad) return -1;
  /* raw (pre-dedup) entries per row */
  int64_t* raw = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
  if (!raw) return -2;
#pragma omp parallel for schedule(static)
  for (int64_t e = 0; e < m; ++e) {
    if (u[e] == v[e]) continue;
#pragma omp atomic
    raw[u[e]] += 1;
#pragma omp atomic
    raw[v[e]] += 1;
  }
  if (block_entries < 1) block_entries = 1;
  int64_t maxrow = 0;
  for (int64_t i = 0; i < n; ++i) maxrow = raw[i] > maxrow ? raw[i] : maxrow;
  const int64_t cap = block_entries > maxrow ? block_entries : maxrow;
  uint64_t* keys = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)(cap > 0 ? cap : 1));
  int64_t* off = (int64_t*)malloc(sizeof(int64_t) * (size_t)n + 8);
  int64_t* cur = (int64_t*)malloc(sizeof(int64_t) * (size_t)n + 8);
  int64_t* kept = (int64_t*)malloc(sizeof(int64_t) * (size_t)n + 8);
  if (!keys || !off || !cur || !kept) { free(raw); free(keys); free(off); free(cur); free(kept); return -2; }
  const uint8_t* w8 = (const uint8_t*)w;
  uint8_t* wo8 = (uint8_t*)w_out;
  int64_t out = 0;
  row_ptr[0] = 0;
  int64_t r0 = 0;
  while (r0 < n) {
    /* rows [r0, r1) whose raw entries fit in the key buffer */
    int64_t r1 = r0, tot = 0;
    while (r1 < n && tot + raw[r1] <= cap) { tot += raw[r1]; ++r1; }
    /* slots of the block's rows in the key buffer */
    int64_t acc = 0;
    for (int64_t i = r0; i < r1; ++i) { off[i - r0] = acc; cur[i - r0] = acc; acc += raw[i]; }
#pragma omp parallel for schedule(static)
    for (int64_t e = 0; e < m; ++e) {
      const int64_t a = u[e], b = v[e];
      if (a == b) continue;
      if (a >= r0 && a < r1) {
        int64_t p;
#pragma omp atomic capture
        p = cur[a - r0]++;
        keys[p] = ((uint64_t)b << 32) | (uint64_t)e;
      }
      if (b >= r0 && b < r1) {
        int64_t p;
#pragma omp atomic capture
        p = cur[b - r0]++;
        keys[p] = ((uint64_t)a << 32) | (uint64_t)e;
      }
    }
    /* per row: sort (col, e); keep the first entry of every column, compacted in place */
#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t i = r0; i < r1; ++i) {
      uint64_t* k = keys + off[i - r0];
      const int64_t len = raw[i];
      sort_u64(k, len);
      int64_t nk = 0;
      for (int64_t t = 0; t < len; ++t)
        if (t == 0 || (k[t] >> 32) != (k[t - 1] >> 32)) k[nk++] = k[t];
      kept[i - r0] = nk;
    }
    /* append the block's rows to the output */
    for (int64_t i = r0; i < r1; ++i) {
      row_ptr[i + 1] = row_ptr[i] + kept[i - r0];
    }
#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t i = r0; i < r1; ++i) {
      const uint64_t* k = keys + off[i - r0];
      int64_t o = row_ptr[i];
      for (int64_t t = 0; t < kept[i - r0]; ++t, ++o) {
        const int64_t e = (int64_t)(k[t] & 0xFFFFFFFFu);
        col[o] = (int32_t)(k[t] >> 32);
        if (wsize == 1) wo8[o] = w8[e];
        else if (wsize == 8) memcpy(wo8 + 8 * o, (const uint8_t*)w + 8 * e, 8);
      }
    }
    out = row_ptr[r1];
    r0 = r1;
  }
  stats[0] = loops;
  stats[1] = (m - loops) - out / 2;
  free(raw); free(keys); free(off); free(cur); free(kept);
  return out;
}

/* Neumaier accumulation */
typedef struct { double s, c; } nsum;
static inline void nadd(nsum* a, double x) {
  const double t = a->s + x;
  if (fabs(a->s) >= fabs(x)) a->c += (a->s - t) + x; else a->c += (x - t) + a->s;
  a->s = t;
}
static inline double nval(nsum a) { return a.s + a.c; }

enum { Q_CI, Q_D, Q_P, Q_C, Q_SZ, Q_SBZB, Q_SS, Q_SUMZ, Q_SUMS, Q_N };

static double wv(int wsize, const void* w, int64_t p) {
  if (wsize == 0) return 1.0;
  if (wsize == 1) return (double)((const uint8_t*)w)[p];
  return ((const double*)w)[p];
}

/* out[0..6] = CI, D, P, C, s^T z, (s - mean s)^T (z - mean z), s^T s; out[7], out[8] = mean z, mean s.
 * Two passes: the means first (compensated), then every definition, each a per-thread Neumaier sum
 * over a static schedule, the thread partials combined in thread order (deterministic per thread
 * count). */
int oracle_quantities(int64_t n, const int64_t* row_ptr, const int32_t* col, int wsize, const void* w,
                      const double* s, const double* z, double* out) {
  const int nt = nthreads();
  nsum* part = (nsum*)calloc((size_t)nt * Q_N, sizeof(nsum));
  if (!part) return -2;
#pragma omp parallel
  {
    nsum* a = part + (size_t)thread_id() * Q_N;
#pragma omp for schedule(static)
    for (int64_t i = 0; i < n; ++i) { nadd(&a[Q_SUMZ], z[i]); nadd(&a[Q_SUMS], s[i]); }
  }
  nsum sz_ = {0, 0}, ss_ = {0, 0};
  for (int t = 0; t < nt; ++t) {
    nadd(&sz_, part[(size_t)t * Q_N + Q_SUMZ].s); nadd(&sz_, part[(size_t)t * Q_N + Q_SUMZ].c);
    nadd(&ss_, part[(size_t)t * Q_N + Q_SUMS].s); nadd(&ss_, part[(size_t)t * Q_N + Q_SUMS].c);
  }
  const double mz = nval(sz_) / (double)n, ms = nval(ss_) / (double)n;
  memset(part, 0, sizeof(nsum) * (size_t)nt * Q_N);
#pragma omp parallel
  {
    nsum* a = part + (size_t)thread_id() * Q_N;
#pragma omp for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
      const double zi = z[i], si = s[i];
      const double e1 = zi - si, e2 = zi - mz, e3 = si - ms;
      nadd(&a[Q_CI], e1 * e1);
      nadd(&a[Q_P], e2 * e2);
      nadd(&a[Q_C], zi * zi);
      nadd(&a[Q_SZ], si * zi);
      nadd(&a[Q_SBZB], e3 * e2);
      nadd(&a[Q_SS], si * si);
      for (int64_t p = row_ptr[i]; p < row_ptr[i + 1]; ++p) {
        const int64_t j = col[p];
        if (j > i) {   /* each undirected edge once */
          const double d = zi - z[j];
          nadd(&a[Q_D], wv(wsize, w, p) * d * d);
        }
      }
    }
  }
  for (int q = 0; q < Q_SUMZ; ++q) {
    nsum acc = {0, 0};
    for (int t = 0; t < nt; ++t) { nadd(&acc, part[(size_t)t * Q_N + q].s); nadd(&acc, part[(size_t)t * Q_N + q].c); }
    out[q] = nval(acc);
  }
  out[7] = mz;
  out[8] = ms;
  free(part);
  return 0;
}

int oracle_csr_permute(int64_t n, const int64_t* row_ptr, const int32_t* col, int wsize, const void* w,
                       const int32_t* new2old, const int32_t* old2new, int64_t* rp_out, int32_t* col_out,
                       void* w_out) {
  rp_out[0] = 0;
  for (int64_t i = 0; i < n; ++i) {
    const int64_t o = new2old[i];
    rp_out[i + 1] = rp_out[i] + (row_ptr[o + 1] - row_ptr[o]);
  }
#pragma omp parallel for schedule(dynamic, 1024)
  for (int64_t i = 0; i < n; ++i) {
    const int64_t o = new2old[i];
    int64_t q = rp_out[i];
    for (int64_t p = row_ptr[o]; p < row_ptr[o + 1]; ++p, ++q) {
      col_out[q] = old2new[col[p]];
      if (wsize) memcpy((uint8_t*)w_out + (size_t)wsize * q, (const uint8_t*)w + (size_t)wsize * p, (size_t)wsize);
    }
  }
  return 0;
}

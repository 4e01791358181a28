/*
 * synth.c — seeded synthetic inputs shared by the oracle and the CUDA path.
 *
 * This module holds NO arithmetic of the method (no Laplacian, no solve, no
 * quantity).  It only draws graphs and opinion vectors from a counter-based
 * generator so that every consumer (oracle/, the GPU library's tests, bench.py)
 * sees the same bits for the same (seed, config), independent of thread count.
 *
 * Recipes:
 *   - opinions: uniform U[0,1); exponential x = x_min - ln(1-u); power law
 *     x = x_min (1-u)^(-1/(alpha-1)), alpha = 2.5, x_min = 1; the latter two are
 *     divided by their maximum (§5 "Internal opinion
 *     distributions").
 *   - Erdos-Renyi G(n,p): per-row geometric skipping over j > i.
 *   - Barabasi-Albert (networkx convention): star seed on m+1 nodes, then each
 *     new node draws m distinct targets uniformly from the repeated-endpoint list.
 *   - R-MAT: per edge, per level a quadrant draw with (a,b,c,d); no noise, no
 *     relabelling; self-loops / duplicates are left in (the CSR build drops them).
 *   - edge weights (C4): 1 + rand64(seed, W_STREAM, min<<32|max) mod 5, so
 *     duplicate edges always agree on their weight.
 *
 * Counter-based generator: rand64(seed, stream, ctr) = sm(sm(sm(seed) ^ stream) ^ ctr)
 * with sm = splitmix64's finaliser; U = (rand64 >> 11) * 2^-53 in [0,1).
 * synth/__init__.py mirrors rand64 in numpy for cross-checks.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define STREAM_OPINION 0x1ULL
#define STREAM_ER      (0x2ULL << 40)
#define STREAM_RMAT    (0x3ULL << 40)
#define STREAM_BA      (0x4ULL << 40)
#define STREAM_WEIGHT  (0x5ULL << 40)

static inline uint64_t sm64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ULL;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}

uint64_t synth_rand64(uint64_t seed, uint64_t stream, uint64_t ctr) {
  return sm64(sm64(sm64(seed) ^ stream) ^ ctr);
}

static inline double u01(uint64_t seed, uint64_t stream, uint64_t ctr) {
  return (double)(synth_rand64(seed, stream, ctr) >> 11) * 0x1.0p-53;
}

/* kind: 0 uniform, 1 exponential (rate 1, x_min 1), 2 power law (alpha 2.5, x_min 1).
 * s[i] for i in [0,n). Normalisation by max for kinds 1 and 2. */
int synth_opinions(int kind, uint64_t seed, int64_t n, double* s) {
  if (n < 0 || (n > 0 && !s) || kind < 0 || kind > 2) return -1;
  const double xmin = 1.0, alpha = 2.5;
  double mx = 0.0;
#pragma omp parallel for schedule(static) reduction(max : mx)
  for (int64_t i = 0; i < n; ++i) {
    double u = u01(seed, STREAM_OPINION, (uint64_t)i);
    double x;
    if (kind == 0) x = u;
    else if (kind == 1) x = xmin - log1p(-u);
    else x = xmin * pow(1.0 - u, -1.0 / (alpha - 1.0));
    s[i] = x;
    if (x > mx) mx = x;
  }
  if (kind != 0 && n > 0) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) s[i] = s[i] / mx;
  }
  return 0;
}

/* ---------------- Erdos-Renyi G(n, p) ---------------- */
static int64_t er_row(int64_t i, int64_t n, double lq, uint64_t seed, int32_t* u, int32_t* v) {
  /* candidates j in (i, n); geometric skips; returns count (writes if u != NULL) */
  int64_t j = i, cnt = 0;
  uint64_t ctr = 0;
  for (;;) {
    double r = u01(seed, STREAM_ER | (uint64_t)i, ctr++);
    double skip = floor(log1p(-r) / lq);
    if (skip >= (double)(n - j)) break;
    j += (int64_t)skip + 1;
    if (j >= n) break;
    if (u) { u[cnt] = (int32_t)i; v[cnt] = (int32_t)j; }
    ++cnt;
  }
  return cnt;
}

/* Two-phase: call with u == NULL to get per-row counts' total; then fill.
 * Returns number of edges, or -1 on error. cap = capacity of u/v. */
int64_t synth_er(int64_t n, double p, uint64_t seed, int32_t* u, int32_t* v, int64_t cap) {
  if (n < 0 || n > INT32_MAX || !(p > 0.0 && p < 1.0)) return -1;
  const double lq = log1p(-p);
  int64_t* cnt = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n + 1));
  if (!cnt) return -1;
#pragma omp parallel for schedule(dynamic, 4096)
  for (int64_t i = 0; i < n; ++i) cnt[i] = er_row(i, n, lq, seed, NULL, NULL);
  int64_t tot = 0;
  for (int64_t i = 0; i < n; ++i) { int64_t c = cnt[i]; cnt[i] = tot; tot += c; }
  cnt[n] = tot;
  if (u && v) {
    if (tot > cap) { free(cnt); return -2; }
#pragma omp parallel for schedule(dynamic, 4096)
    for (int64_t i = 0; i < n; ++i) er_row(i, n, lq, seed, u + cnt[i], v + cnt[i]);
  }
  free(cnt);
  return tot;
}

/* ---------------- Barabasi-Albert (networkx convention) ---------------- */
/* edges: m (star) + (n - m - 1) * m. u[e] = new node (or star centre 0), v[e] = target. */
int64_t synth_ba(int64_t n, int64_t m, uint64_t seed, int32_t* u, int32_t* v, int64_t cap) {
  if (m < 1 || n <= m || n > INT32_MAX) return -1;
  int64_t total = m + (n - m - 1) * m;
  if (!u || !v) return total;
  if (total > cap) return -2;
  int64_t rep_cap = 2 * total;
  int32_t* rep = (int32_t*)malloc(sizeof(int32_t) * (size_t)rep_cap);
  int32_t* tg = (int32_t*)malloc(sizeof(int32_t) * (size_t)m);
  if (!rep || !tg) { free(rep); free(tg); return -1; }
  int64_t nrep = 0, e = 0;
  /* star_graph(m): centre 0 joined to 1..m */
  for (int64_t j = 1; j <= m; ++j) {
    u[e] = 0; v[e] = (int32_t)j; ++e;
    rep[nrep++] = 0; rep[nrep++] = (int32_t)j;
  }
  uint64_t ctr = 0;
  for (int64_t src = m + 1; src < n; ++src) {
    int64_t k = 0;
    while (k < m) {
      uint64_t r = synth_rand64(seed, STREAM_BA, ctr++);
      int32_t cand = rep[(int64_t)((r >> 11) % (uint64_t)nrep)];
      int dup = 0;
      for (int64_t t = 0; t < k; ++t) if (tg[t] == cand) { dup = 1; break; }
      if (!dup) tg[k++] = cand;
    }
    for (int64_t t = 0; t < m; ++t) {
      u[e] = (int32_t)src; v[e] = tg[t]; ++e;
      rep[nrep++] = tg[t];
    }
    for (int64_t t = 0; t < m; ++t) rep[nrep++] = (int32_t)src;
  }
  free(rep); free(tg);
  return e;
}

/* ---------------- R-MAT ---------------- */
/* m_edges = edge_factor * 2^scale raw draws (self-loops and duplicates kept). */
int64_t synth_rmat(int scale, int64_t edge_factor, double a, double b, double c, uint64_t seed,
                   int32_t* u, int32_t* v, int64_t cap) {
  if (scale < 1 || scale > 30 || edge_factor < 1) return -1;
  int64_t m = edge_factor << scale;
  if (!u || !v) return m;
  if (m > cap) return -2;
  const double ab = a + b, abc = a + b + c;
#pragma omp parallel for schedule(static)
  for (int64_t e = 0; e < m; ++e) {
    uint32_t src = 0, dst = 0;
    for (int l = 0; l < scale; ++l) {
      double r = u01(seed, STREAM_RMAT | (uint64_t)l, (uint64_t)e);
      uint32_t bit = 1u << (scale - 1 - l);
      if (r < a) { /* quadrant (0,0) */ }
      else if (r < ab) dst |= bit;
      else if (r < abc) src |= bit;
      else { src |= bit; dst |= bit; }
    }
    u[e] = (int32_t)src; v[e] = (int32_t)dst;
  }
  return m;
}

/* ---------------- integer weights 1..5 keyed by the canonical pair ---------------- */
int synth_weights_u8(uint64_t seed, int64_t m, const int32_t* u, const int32_t* v, uint8_t* w) {
  if (m < 0) return -1;
#pragma omp parallel for schedule(static)
  for (int64_t e = 0; e < m; ++e) {
    uint64_t lo = (uint64_t)(uint32_t)(u[e] < v[e] ? u[e] : v[e]);
    uint64_t hi = (uint64_t)(uint32_t)(u[e] < v[e] ? v[e] : u[e]);
    w[e] = (uint8_t)(1 + synth_rand64(seed, STREAM_WEIGHT, (lo << 32) | hi) % 5);
  }
  return 0;
}

int synth_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

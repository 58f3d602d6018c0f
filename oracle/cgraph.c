/*
 * cgraph.c -- plain-C restatement of the reference algorithms (TEST ORACLE and
 * CPU baseline; see oracle/__init__.py).  Never linked into the product.
 *
 * Each function restates /root/reference/pkg/src/graphalg/<file>:<line>
 * semantics on a host CSR (int64 offsets, int32 indices); OpenMP threads
 * parallelise the data-parallel loops.  Results are bit-identical to the
 * reference for BFS levels, CC labels, TC counts and SSSP distances (min/+ are
 * exact); PageRank sums in a different order (1e-12-level differences).
 *
 *   og_rmat_edges   io.py:100-111, 275-295   SplitMix64 R-MAT stream
 *   og_bfs          algorithms.py:48-77 + kernels.py:108-126 dispatch rule
 *   og_sssp         algorithms.py:80-119
 *   og_pagerank     algorithms.py:122-162
 *   og_cc           algorithms.py:165-203 (FastSV with sparsification)
 *   og_tc           algorithms.py:206-240 (count is orientation-free)
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

#define I64MAX INT64_MAX

static const uint64_t GAMMA = 0x9E3779B97F4A7C15ull;

static inline uint64_t mix(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

int og_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

void og_set_threads(int t) {
#ifdef _OPENMP
  if (t > 0) omp_set_num_threads(t);
#else
  (void)t;
#endif
}

/* io.py:275-295: edge e, level l uses draw e*scale+l, MSB first. */
void og_rmat_edges(int scale, int64_t m, uint64_t seed, double a, double tab, double tabc,
                   int32_t* src, int32_t* dst) {
#pragma omp parallel for schedule(static)
  for (int64_t e = 0; e < m; ++e) {
    uint32_t r = 0, c = 0;
    for (int l = 0; l < scale; ++l) {
      uint64_t k = (uint64_t)e * (uint64_t)scale + (uint64_t)l;
      double x = (double)(mix(seed + (k + 1) * GAMMA) >> 11) * (1.0 / 9007199254740992.0);
      r = (r << 1) | (x >= tab);
      c = (c << 1) | ((x >= a && x < tab) || x >= tabc);
    }
    src[e] = (int32_t)r;
    dst[e] = (int32_t)c;
  }
}

/* Parallel LSD radix sort of uint64 keys on the low `bits` bits (11-bit digits). */
static void radix_sort_u64(uint64_t* a, uint64_t* tmp, int64_t n, int bits) {
  const int D = 11, R = 1 << D;
  int T = og_threads();
  int64_t* hist = malloc(sizeof(int64_t) * (size_t)R * (size_t)T);
  for (int shift = 0; shift < bits; shift += D) {
    memset(hist, 0, sizeof(int64_t) * (size_t)R * (size_t)T);
#pragma omp parallel num_threads(T)
    {
#ifdef _OPENMP
      int t = omp_get_thread_num();
#else
      int t = 0;
#endif
      int64_t lo = n * t / T, hi = n * (t + 1) / T;
      int64_t* h = hist + (size_t)t * R;
      for (int64_t i = lo; i < hi; ++i) h[(a[i] >> shift) & (R - 1)]++;
#pragma omp barrier
#pragma omp single
      {
        int64_t sum = 0;
        for (int d = 0; d < R; ++d)
          for (int u = 0; u < T; ++u) {
            int64_t c = hist[(size_t)u * R + d];
            hist[(size_t)u * R + d] = sum;
            sum += c;
          }
      }
      for (int64_t i = lo; i < hi; ++i) tmp[h[(a[i] >> shift) & (R - 1)]++] = a[i];
    }
    uint64_t* x = a;
    a = tmp;
    tmp = x;
  }
  /* an odd number of passes leaves the result in the scratch buffer */
  int passes = (bits + D - 1) / D;
  if (passes & 1) memcpy(tmp, a, sizeof(uint64_t) * (size_t)n);
  free(hist);
}

/* generate_rmat + preprocess(make_undirected) + edges_to_matrix (io.py:220-315):
 * CSR of the symmetrised, deduplicated pattern graph.  ci must hold 2*m. */
int64_t og_rmat_csr(int scale, int64_t m, uint64_t seed, double a, double tab, double tabc,
                    int64_t* rp, int32_t* ci) {
  int64_t n = (int64_t)1 << scale;
  int bits = scale > 0 ? scale : 1;
  uint64_t* k = malloc(sizeof(uint64_t) * (size_t)(2 * m + 1));
  uint64_t* t = malloc(sizeof(uint64_t) * (size_t)(2 * m + 1));
  const uint64_t sentinel = (uint64_t)1 << (2 * bits);
#pragma omp parallel for schedule(static)
  for (int64_t e = 0; e < m; ++e) {
    uint64_t r = 0, c = 0;
    for (int l = 0; l < scale; ++l) {
      uint64_t kk = (uint64_t)e * (uint64_t)scale + (uint64_t)l;
      double x = (double)(mix(seed + (kk + 1) * GAMMA) >> 11) * (1.0 / 9007199254740992.0);
      r = (r << 1) | (x >= tab);
      c = (c << 1) | ((x >= a && x < tab) || x >= tabc);
    }
    k[2 * e] = r == c ? sentinel : ((r << bits) | c);
    k[2 * e + 1] = r == c ? sentinel : ((c << bits) | r);
  }
  radix_sort_u64(k, t, 2 * m, 2 * bits + 1);
  int64_t nnz = 0;
  uint64_t mask = ((uint64_t)1 << bits) - 1;
  int64_t row = 0;
  rp[0] = 0;
  for (int64_t i = 0; i < 2 * m; ++i) {
    uint64_t key = k[i];
    if (key == sentinel) break;
    if (i > 0 && key == k[i - 1]) continue;
    int64_t r = (int64_t)(key >> bits);
    while (row < r) rp[++row] = nnz;
    ci[nnz++] = (int32_t)(key & mask);
  }
  while (row < n) rp[++row] = nnz;
  free(k);
  free(t);
  return nnz;
}

/* assign_weights(edges, low, high, seed) (io.py:252-272) on the symmetric,
 * sorted CSR that preprocess + edges_to_matrix produce: the k-th upper entry
 * (i < j, row-major -- the first appearance of (min, max) in the sorted edge
 * list) draws low + mix_k mod (high-low+1); its mirror (j, i) takes the same
 * value (found by binary search in the sorted row j).  Returns 0, or -1 when
 * a mirror is missing (the CSR is not symmetric). */
int64_t og_upper_weights(int64_t n, const int64_t* rp, const int32_t* ci, uint64_t seed,
                         int64_t low, int64_t high, double* w) {
  int64_t* ufirst = malloc(sizeof(int64_t) * (size_t)(n + 1));
  /* rank of a row's first upper entry = upper entries of all earlier rows */
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    int64_t lo = rp[i], hi = rp[i + 1];
    while (lo < hi) { /* first column > i */
      int64_t mid = lo + (hi - lo) / 2;
      if (ci[mid] <= i) lo = mid + 1; else hi = mid;
    }
    ufirst[i + 1] = rp[i + 1] - lo;
  }
  ufirst[0] = 0;
  for (int64_t i = 0; i < n; ++i) ufirst[i + 1] += ufirst[i];
  uint64_t span = (uint64_t)(high - low + 1);
  int64_t bad = 0;
#pragma omp parallel for schedule(dynamic, 1024) reduction(+ : bad)
  for (int64_t i = 0; i < n; ++i) {
    int64_t base = rp[i + 1] - (ufirst[i + 1] - ufirst[i]); /* first upper slot of row i */
    for (int64_t e = rp[i]; e < rp[i + 1]; ++e) {
      int64_t j = ci[e], k;
      if (j > i) {
        k = ufirst[i] + (e - base);
      } else if (j < i) {
        int64_t lo = rp[j], hi = rp[j + 1];
        while (lo < hi) {
          int64_t mid = lo + (hi - lo) / 2;
          if (ci[mid] < i) lo = mid + 1; else hi = mid;
        }
        if (lo == rp[j + 1] || ci[lo] != i) { ++bad; continue; }
        int64_t bj = rp[j + 1] - (ufirst[j + 1] - ufirst[j]);
        k = ufirst[j] + (lo - bj);
      } else {
        ++bad; /* preprocess drops self loops */
        continue;
      }
      w[e] = (double)(low + (int64_t)(mix(seed + ((uint64_t)k + 1) * GAMMA) % span));
    }
  }
  free(ufirst);
  return bad ? -1 : 0;
}

/* kernels.py:108-126 */
static int decide(int64_t nnz, int64_t nrows, int64_t nnz_u, double ratio, int policy,
                  int64_t* est_out) {
  double d = nrows ? (double)nnz / (double)nrows : 0.0;
  int64_t est = (int64_t)nearbyint(d * (double)nnz_u); /* half-even like Python round */
  *est_out = est;
  if (policy == 1) return 1;
  if (policy == 2) return 2;
  return (double)est > (double)nnz * ratio ? 2 : 1;
}

/* ------------------------------------------------------------------------ */
/* BFS: algorithms.py:48-77; vxm push walks rows (CSR), pull walks in-edges  */
/* (CSC).  Levels 1-based, 0 = unreached.  Returns iterations executed.      */
/* ------------------------------------------------------------------------ */
int64_t og_bfs(int64_t n, const int64_t* rp, const int32_t* ci, const int64_t* cp,
               const int32_t* ri, int64_t source, int64_t max_iters, double ratio, int policy,
               int64_t* levels, int32_t* log_dir, int64_t* log_nv, int64_t* log_est) {
  int64_t nnz = rp[n];
  uint8_t* infront = calloc((size_t)n, 1);
  uint8_t* nxt = calloc((size_t)n, 1);
  int32_t* F = malloc(sizeof(int32_t) * (size_t)(n > 0 ? n : 1));
  memset(levels, 0, sizeof(int64_t) * (size_t)n);
  int64_t K = 1, depth = 1, it;
  F[0] = (int32_t)source;
  infront[source] = 1;
  levels[source] = 1;
  for (it = 0; it < max_iters; ++it) {
    int64_t est;
    int dir = decide(nnz, n, K, ratio, policy, &est);
    log_dir[it] = dir;
    log_nv[it] = K;
    log_est[it] = est;
    if (dir == 2) {
#pragma omp parallel for schedule(dynamic, 1024)
      for (int64_t v = 0; v < n; ++v) {
        if (levels[v]) continue;
        for (int64_t p = cp[v]; p < cp[v + 1]; ++p)
          if (infront[ri[p]]) { nxt[v] = 1; break; }
      }
    } else {
#pragma omp parallel for schedule(dynamic, 64)
      for (int64_t k = 0; k < K; ++k) {
        int32_t u = F[k];
        for (int64_t p = rp[u]; p < rp[u + 1]; ++p) {
          int32_t v = ci[p];
          if (!levels[v] && !nxt[v]) nxt[v] = 1;
        }
      }
    }
    /* the reference stamps a frontier at the start of the next iteration */
    int64_t c = 0;
    for (int64_t v = 0; v < n; ++v) {
      infront[v] = nxt[v];
      if (nxt[v]) {
        nxt[v] = 0;
        F[c++] = (int32_t)v;
      }
    }
    K = c;
    if (K == 0) { ++it; break; }
    ++depth;
    if (it + 1 < max_iters)
      for (int64_t k = 0; k < K; ++k) levels[F[k]] = depth;
  }
  free(infront);
  free(nxt);
  free(F);
  return it;
}

/* ------------------------------------------------------------------------ */
/* SSSP: algorithms.py:80-119 (frontier = strictly improved candidates).     */
/* w is aligned with the CSR (push, rows = out-edges) and wt with the CSC    */
/* (pull, rows = in-edges).                                                  */
/* ------------------------------------------------------------------------ */
static inline void atomic_min_f64(double* addr, double v) {
  /* distances and weights are positive: IEEE order == int64 order */
  int64_t nv;
  memcpy(&nv, &v, 8);
  int64_t old = __atomic_load_n((int64_t*)addr, __ATOMIC_RELAXED);
  while (nv < old &&
         !__atomic_compare_exchange_n((int64_t*)addr, &old, nv, 1, __ATOMIC_RELAXED,
                                      __ATOMIC_RELAXED)) {
  }
}

int64_t og_sssp(int64_t n, const int64_t* rp, const int32_t* ci, const double* w,
                const int64_t* cp, const int32_t* ri, const double* wt, int64_t source,
                int64_t max_iters, double ratio, int policy, double* dist, int32_t* log_dir,
                int64_t* log_nv, int64_t* log_est) {
  int64_t nnz = rp[n];
  double* cand = malloc(sizeof(double) * (size_t)n);
  double* fval = malloc(sizeof(double) * (size_t)n);
  int32_t* F = malloc(sizeof(int32_t) * (size_t)n);
  uint8_t* inf_ = calloc((size_t)n, 1);
  for (int64_t i = 0; i < n; ++i) { dist[i] = INFINITY; cand[i] = INFINITY; fval[i] = INFINITY; }
  dist[source] = 0.0;
  int64_t K = 1, it, succ_last = -1;
  F[0] = (int32_t)source;
  fval[source] = 0.0;
  int64_t reached = 1;
  for (it = 0; it < max_iters; ++it) {
    int64_t est;
    int dir = decide(nnz, n, K, ratio, policy, &est);
    log_dir[it] = dir;
    log_nv[it] = K;
    log_est[it] = est;
    if (dir == 2) {
#pragma omp parallel for schedule(dynamic, 1024)
      for (int64_t v = 0; v < n; ++v) {
        double best = INFINITY;
        for (int64_t p = cp[v]; p < cp[v + 1]; ++p) {
          double u = fval[ri[p]];
          if (u != INFINITY) {
            double x = wt[p] + u;
            if (x < best) best = x;
          }
        }
        cand[v] = best;
      }
    } else {
#pragma omp parallel for schedule(dynamic, 64)
      for (int64_t k = 0; k < K; ++k) {
        int32_t u = F[k];
        double du = fval[u];
        for (int64_t p = rp[u]; p < rp[u + 1]; ++p) atomic_min_f64(&cand[ci[p]], w[p] + du);
      }
    }
    for (int64_t k = 0; k < K; ++k) fval[F[k]] = INFINITY;
    int64_t c = 0;
    for (int64_t v = 0; v < n; ++v) {
      double x = cand[v];
      if (x < dist[v]) {
        if (dist[v] == INFINITY) ++reached;
        dist[v] = x;
        F[c++] = (int32_t)v;
        fval[v] = x;
      }
      cand[v] = INFINITY;
    }
    K = c;
    /* reached = count of dist < f64max (algorithms.py:114-115) */
    if (reached == succ_last && K == 0) { ++it; break; }
    succ_last = reached;
  }
  free(cand);
  free(fval);
  free(F);
  free(inf_);
  return it;
}

/* ------------------------------------------------------------------------ */
/* PageRank: algorithms.py:122-162.  spread[j] = sum_{i in in(j)} (a/deg_i)*p_i */
/* ------------------------------------------------------------------------ */
int64_t og_pagerank(int64_t n, const int64_t* rp, const int64_t* cp, const int32_t* ri,
                    double alpha, double eps, int64_t max_iters, double* ranks, double* errs) {
  double* inv = malloc(sizeof(double) * (size_t)n);
  double* prev = malloc(sizeof(double) * (size_t)n);
  for (int64_t i = 0; i < n; ++i) {
    int64_t d = rp[i + 1] - rp[i];
    inv[i] = d > 0 ? alpha / (double)d : 0.0;
    ranks[i] = 1.0 / (double)n;
  }
  double tele = (1.0 - alpha) / (double)n;
  int64_t it;
  for (it = 0; it < max_iters; ++it) {
    memcpy(prev, ranks, sizeof(double) * (size_t)n);
    double err2 = 0.0;
#pragma omp parallel for schedule(dynamic, 1024) reduction(+ : err2)
    for (int64_t j = 0; j < n; ++j) {
      double s = 0.0;
      for (int64_t p = cp[j]; p < cp[j + 1]; ++p) {
        int32_t i = ri[p];
        if (prev[i] != 0.0) s += inv[i] * prev[i];
      }
      double r = s + tele;
      double dlt = r - prev[j];
      ranks[j] = r;
      err2 += dlt * dlt;
    }
    double err = sqrt(err2);
    if (errs) errs[it] = err;
    if (err <= eps) { ++it; break; }
  }
  free(inv);
  free(prev);
  return it;
}

/* ------------------------------------------------------------------------ */
/* Connected components (FastSV): algorithms.py:165-203.  mxv walks rows of  */
/* A (pull over CSR) or columns (push over CSC).                             */
/* ------------------------------------------------------------------------ */
static inline void atomic_min_i64(int64_t* addr, int64_t v) {
  int64_t old = __atomic_load_n(addr, __ATOMIC_RELAXED);
  while (v < old &&
         !__atomic_compare_exchange_n(addr, &old, v, 1, __ATOMIC_RELAXED, __ATOMIC_RELAXED)) {
  }
}

int64_t og_cc(int64_t n, const int64_t* rp, const int32_t* ci, const int64_t* cp,
              const int32_t* ri, int64_t max_iters, double ratio, int policy, int sparsify,
              int64_t* parent, int32_t* log_dir, int64_t* log_nv, int64_t* log_est) {
  int64_t nnz = rp[n];
  int64_t* mn = malloc(sizeof(int64_t) * (size_t)n);
  int64_t* gp = malloc(sizeof(int64_t) * (size_t)n);
  int64_t* gpp = malloc(sizeof(int64_t) * (size_t)n);
  int64_t* pp = malloc(sizeof(int64_t) * (size_t)n);
  int64_t* hk = malloc(sizeof(int64_t) * (size_t)n);
  for (int64_t i = 0; i < n; ++i) parent[i] = mn[i] = gp[i] = gpp[i] = i;
  int64_t it, live = n;
  for (it = 0; it < max_iters; ++it) {
    memcpy(pp, parent, sizeof(int64_t) * (size_t)n);
    int64_t est;
    int dir = decide(nnz, n, live, ratio, policy, &est);
    log_dir[it] = dir;
    log_nv[it] = live;
    log_est[it] = est;
    if (dir == 2) {
#pragma omp parallel for schedule(dynamic, 1024)
      for (int64_t i = 0; i < n; ++i) {
        int64_t h = I64MAX;
        for (int64_t p = rp[i]; p < rp[i + 1]; ++p) {
          int64_t g = gp[ci[p]];
          if (g != I64MAX && g < h) h = g;
        }
        hk[i] = h;
      }
    } else {
#pragma omp parallel for schedule(static)
      for (int64_t i = 0; i < n; ++i) hk[i] = I64MAX;
#pragma omp parallel for schedule(dynamic, 1024)
      for (int64_t j = 0; j < n; ++j) {
        int64_t g = gp[j];
        if (g == I64MAX) continue;
        for (int64_t p = cp[j]; p < cp[j + 1]; ++p) atomic_min_i64(&hk[ri[p]], g);
      }
    }
    /* mn = min(mn, hooked); parent[pp[k]] = min_k mn[k]; parent = min(parent, mn, pp) */
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < n; ++k) {
      if (hk[k] < mn[k]) mn[k] = hk[k];
      int64_t v = parent[k];
      if (mn[k] < v) v = mn[k];
      atomic_min_i64(&parent[k], v);
    }
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < n; ++k) atomic_min_i64(&parent[pp[k]], mn[k]);
    int64_t changed = 0;
#pragma omp parallel for schedule(static) reduction(+ : changed)
    for (int64_t k = 0; k < n; ++k) {
      int64_t g = parent[parent[k]];
      changed += g != gpp[k];
      gp[k] = g;
    }
    if (changed == 0) { ++it; break; }
    live = sparsify ? changed : n;
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < n; ++k) {
      int64_t g = gp[k];
      int c = g != gpp[k];
      gpp[k] = g;
      if (sparsify && !c) gp[k] = I64MAX;
    }
  }
  free(mn);
  free(gp);
  free(gpp);
  free(pp);
  free(hk);
  return it;
}

/* ------------------------------------------------------------------------ */
/* Triangle count: algorithms.py:206-240.  Degree order with ties by id; each */
/* vertex keeps its higher-ranked neighbours; count = sum over oriented edges */
/* of |N+(u) & N+(v)|.  (The reference's L.L^T.*L gives the same number.)    */
/* ------------------------------------------------------------------------ */
static int cmp_rank(const void* a, const void* b) {
  int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
  return (x > y) - (x < y);
}

int64_t og_tc(int64_t n, const int64_t* rp, const int32_t* ci) {
  /* rank = stable argsort position by (degree, id) */
  int64_t* key = malloc(sizeof(int64_t) * (size_t)n);
  for (int64_t i = 0; i < n; ++i) key[i] = ((rp[i + 1] - rp[i]) << 32) | i;
  qsort(key, (size_t)n, sizeof(int64_t), cmp_rank);
  int64_t* rank = malloc(sizeof(int64_t) * (size_t)n);
  for (int64_t r = 0; r < n; ++r) rank[key[r] & 0xffffffffll] = r;
  int64_t* up = malloc(sizeof(int64_t) * (size_t)(n + 1));
  up[0] = 0;
  for (int64_t i = 0; i < n; ++i) {
    int64_t c = 0;
    for (int64_t p = rp[i]; p < rp[i + 1]; ++p) c += rank[ci[p]] > rank[i];
    up[i + 1] = up[i] + c;
  }
  int64_t* un = malloc(sizeof(int64_t) * (size_t)(up[n] > 0 ? up[n] : 1));
#pragma omp parallel for schedule(dynamic, 256)
  for (int64_t i = 0; i < n; ++i) {
    int64_t o = up[i];
    for (int64_t p = rp[i]; p < rp[i + 1]; ++p)
      if (rank[ci[p]] > rank[i]) un[o++] = rank[ci[p]];
    qsort(un + up[i], (size_t)(up[i + 1] - up[i]), sizeof(int64_t), cmp_rank);
  }
  /* rows indexed by rank */
  int64_t* byrank = malloc(sizeof(int64_t) * (size_t)n);
  for (int64_t i = 0; i < n; ++i) byrank[rank[i]] = i;
  int64_t total = 0;
#pragma omp parallel for schedule(dynamic, 64) reduction(+ : total)
  for (int64_t i = 0; i < n; ++i) {
    const int64_t* a = un + up[i];
    int64_t la = up[i + 1] - up[i];
    for (int64_t q = 0; q < la; ++q) {
      int64_t j = byrank[a[q]];
      const int64_t* b = un + up[j];
      int64_t lb = up[j + 1] - up[j];
      int64_t x = 0, y = 0;
      while (x < la && y < lb) {
        if (a[x] < b[y]) ++x;
        else if (a[x] > b[y]) ++y;
        else { ++total; ++x; ++y; }
      }
    }
  }
  free(key);
  free(rank);
  free(up);
  free(un);
  free(byrank);
  return total;
}

/* ------------------------------------------------------------------------ */
/* BFS parents (the north star's "levels/parents" extension; the reference   */
/* returns levels only, algorithms.py:66-77): parent[v] = the smallest u in  */
/* v's in-edge row (cp/ri, ascending) with level[u] = level[v] - 1;          */
/* parent[source] = source; -1 when unreached.  Returns the number of        */
/* reached vertices without such a u (0 for a consistent level vector).      */
/* ------------------------------------------------------------------------ */
int64_t og_bfs_parents(int64_t n, const int64_t* cp, const int32_t* ri, const int64_t* lv,
                       int64_t source, int64_t* parent) {
  int64_t bad = 0;
#pragma omp parallel for schedule(dynamic, 4096) reduction(+ : bad)
  for (int64_t v = 0; v < n; ++v) {
    if (lv[v] == 0) {
      parent[v] = -1;
    } else if (v == source) {
      parent[v] = source;
    } else {
      int64_t p = -1;
      for (int64_t k = cp[v]; k < cp[v + 1]; ++k)
        if (lv[ri[k]] == lv[v] - 1) {
          p = ri[k];
          break;
        }
      parent[v] = p;
      bad += p < 0;
    }
  }
  return bad;
}

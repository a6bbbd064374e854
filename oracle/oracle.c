/*
 * oracle.c -- TEST INFRASTRUCTURE ONLY (see oracle.h).
 *
 * Plain-C restatement of the reference gblite algorithms on the hot path.  Every
 * function cites the reference file:line it follows (paths relative to
 * /root/reference/proj).  The restatement keeps the reference's observable
 * semantics (which parent the any-monoid keeps, fold order of the PageRank sums
 * and of the L1 norm, the delta-stepping bucket rules, the batched Brandes
 * accumulation order) but uses dense int/double arrays instead of the
 * reference's std::variant containers, so it runs at BASELINE scales.
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static int g_threads = 0;
void orc_set_threads(int t) { g_threads = t; }
int orc_get_threads(void) {
#ifdef _OPENMP
  return g_threads > 0 ? g_threads : omp_get_max_threads();
#else
  return 1;
#endif
}
#define ORC_NT orc_get_threads()

/* ---- seeded inputs ------------------------------------------------------- */
/* The generator has no reference counterpart ("No R-MAT or
 * Kronecker generator exists anywhere in the reference").  Its definition is
 * restated independently in csrc/gen.cu; tests compare the two bit for bit. */

static inline uint64_t mix64(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBull;
  z ^= z >> 31;
  return z;
}
uint64_t orc_splitmix64(uint64_t z) { return mix64(z); }
uint64_t orc_stream(uint64_t seed, uint64_t stream) {
  return mix64(seed ^ mix64(stream + 0x632BE59BD9B4E019ull));
}
uint64_t orc_draw(uint64_t s, uint64_t i) {
  return mix64(s + (i + 1) * 0x9E3779B97F4A7C15ull);
}

uint32_t orc_scramble(uint32_t x, int scale, uint64_t seed) {
  if (scale <= 0) return x;
  uint64_t mask = (scale >= 32) ? 0xFFFFFFFFull : ((1ull << scale) - 1);
  uint64_t add = orc_stream(seed, 1) & mask;
  int sh = scale / 2 + 1;
  uint64_t y = x;
  y = (y * 0x9E3779B97F4A7C15ull) & mask;
  y ^= y >> sh;
  y = (y + add) & mask;
  y = (y * 0xBF58476D1CE4E5B9ull) & mask;
  y ^= y >> sh;
  return (uint32_t)y;
}

int64_t orc_rmat_edges(int scale, int edge_factor, double a, double b, double c,
                       uint64_t seed, int scramble, uint32_t* u, uint32_t* v) {
  int64_t m = (int64_t)edge_factor << scale;
  uint32_t ta = (uint32_t)(a * 4294967296.0);
  uint32_t tab = (uint32_t)((a + b) * 4294967296.0);
  double abc = a + b + c;
  uint32_t tabc = abc >= 1.0 ? 0xFFFFFFFFu : (uint32_t)(abc * 4294967296.0);
  uint64_t s = orc_stream(seed, 0);
  int per = (scale + 1) / 2;
#pragma omp parallel for schedule(static) num_threads(ORC_NT)
  for (int64_t e = 0; e < m; ++e) {
    uint32_t uu = 0, vv = 0;
    uint64_t r = 0;
    for (int l = 0; l < scale; ++l) {
      if ((l & 1) == 0) r = orc_draw(s, (uint64_t)e * per + (l >> 1));
      uint32_t x = (l & 1) ? (uint32_t)(r >> 32) : (uint32_t)r;
      uint32_t ub, vb;
      if (x < ta) { ub = 0; vb = 0; }
      else if (x < tab) { ub = 0; vb = 1; }
      else if (x < tabc) { ub = 1; vb = 0; }
      else { ub = 1; vb = 1; }
      uu = (uu << 1) | ub;
      vv = (vv << 1) | vb;
    }
    if (scramble) {
      uu = orc_scramble(uu, scale, seed);
      vv = orc_scramble(vv, scale, seed);
    }
    u[e] = uu;
    v[e] = vv;
  }
  return m;
}

int64_t orc_er_edges(int logn, int degree, uint64_t seed, uint32_t* u,
                     uint32_t* v, int32_t* w) {
  int64_t m = (int64_t)degree << logn;
  uint64_t s = orc_stream(seed, 2);
#pragma omp parallel for schedule(static) num_threads(ORC_NT)
  for (int64_t e = 0; e < m; ++e) {
    uint64_t r1 = orc_draw(s, 2 * (uint64_t)e);
    uint64_t r2 = orc_draw(s, 2 * (uint64_t)e + 1);
    u[e] = (uint32_t)(r1 >> (64 - logn));
    v[e] = (uint32_t)(r2 >> (64 - logn));
    if (w) w[e] = 1 + (int32_t)(((r1 & 0xFFFFFFFFull) * 255ull) >> 32);
  }
  return m;
}

/* CSR construction: the reference's build_matrix stable-sorts tuples by
 * (row, col) and combines duplicates (containers.cpp:128-169); here the dup
 * combiner is min over the weight (pattern graphs carry w = 0). */
static int cmp_u64(const void* x, const void* y) {
  uint64_t a = *(const uint64_t*)x, b = *(const uint64_t*)y;
  return a < b ? -1 : (a > b ? 1 : 0);
}

int64_t orc_build_csr(int64_t n, int64_t m, const uint32_t* u, const uint32_t* v,
                      const int32_t* w, int symmetrize, int64_t* row_ptr,
                      int32_t* col, int32_t* wout) {
  int64_t* cnt = (int64_t*)calloc((size_t)n + 1, sizeof(int64_t));
  for (int64_t e = 0; e < m; ++e) {
    if (u[e] == v[e]) continue;
    cnt[u[e] + 1]++;
    if (symmetrize) cnt[v[e] + 1]++;
  }
  for (int64_t i = 0; i < n; ++i) cnt[i + 1] += cnt[i];
  int64_t total = cnt[n];
  uint64_t* keys = (uint64_t*)malloc((size_t)(total ? total : 1) * sizeof(uint64_t));
  int64_t* cur = (int64_t*)malloc((size_t)(n + 1) * sizeof(int64_t));
  memcpy(cur, cnt, (size_t)(n + 1) * sizeof(int64_t));
  for (int64_t e = 0; e < m; ++e) {
    if (u[e] == v[e]) continue;
    uint32_t ww = w ? (uint32_t)w[e] : 0u;
    keys[cur[u[e]]++] = ((uint64_t)v[e] << 32) | ww;
    if (symmetrize) keys[cur[v[e]]++] = ((uint64_t)u[e] << 32) | ww;
  }
  free(cur);
  /* sort + dedup per row (in place), then compact */
  int64_t* kept = (int64_t*)malloc((size_t)(n + 1) * sizeof(int64_t));
#pragma omp parallel for schedule(dynamic, 1024) num_threads(ORC_NT)
  for (int64_t i = 0; i < n; ++i) {
    int64_t b = cnt[i], e = cnt[i + 1];
    if (e - b > 1) qsort(keys + b, (size_t)(e - b), sizeof(uint64_t), cmp_u64);
    int64_t o = b;
    for (int64_t p = b; p < e; ++p) {
      if (o > b && (keys[o - 1] >> 32) == (keys[p] >> 32)) continue; /* keep min w */
      keys[o++] = keys[p];
    }
    kept[i] = o - b;
  }
  row_ptr[0] = 0;
  for (int64_t i = 0; i < n; ++i) row_ptr[i + 1] = row_ptr[i] + kept[i];
#pragma omp parallel for schedule(dynamic, 1024) num_threads(ORC_NT)
  for (int64_t i = 0; i < n; ++i) {
    int64_t src = cnt[i], dst = row_ptr[i];
    for (int64_t p = 0; p < kept[i]; ++p) {
      col[dst + p] = (int32_t)(keys[src + p] >> 32);
      if (wout) wout[dst + p] = (int32_t)(keys[src + p] & 0xFFFFFFFFull);
    }
  }
  int64_t nnz = row_ptr[n];
  free(kept);
  free(keys);
  free(cnt);
  return nnz;
}

/* Counting-sort transpose: plain_transpose (core.cpp:237-256). */
void orc_transpose(int64_t n, const int64_t* rp, const int32_t* col,
                   const int32_t* w, int64_t* trp, int32_t* tcol, int32_t* tw) {
  memset(trp, 0, (size_t)(n + 1) * sizeof(int64_t));
  int64_t nnz = rp[n];
  for (int64_t p = 0; p < nnz; ++p) trp[col[p] + 1]++;
  for (int64_t j = 0; j < n; ++j) trp[j + 1] += trp[j];
  int64_t* cur = (int64_t*)malloc((size_t)(n + 1) * sizeof(int64_t));
  memcpy(cur, trp, (size_t)(n + 1) * sizeof(int64_t));
  for (int64_t i = 0; i < n; ++i)
    for (int64_t p = rp[i]; p < rp[i + 1]; ++p) {
      int64_t d = cur[col[p]]++;
      tcol[d] = (int32_t)i;
      if (tw) tw[d] = w[p];
    }
  free(cur);
}

/* ---- BFS ------------------------------------------------------------------
 * run_bfs (algo/bfs.cpp:18-52) with the push step vxm (core.cpp:308-338):
 * frontier rows are scanned in ascending id, DenseAcc keeps the first
 * contribution (core.cpp:214-222, any monoid ops.cpp:170-175) and secondi
 * yields the frontier id k (ops.cpp:211-222), so each newly reached vertex's
 * parent is its minimum-id neighbour on the previous level; harvest sorts the
 * next frontier (core.cpp:224-234).  The pull variant (mxv over AT,
 * core.cpp:340-386) keeps the first hit of an ascending merge, i.e. the same
 * parent.  parent(source) = source, level(source) = 0; unreached = -1. */
int orc_bfs(int64_t n, const int64_t* rp, const int32_t* col, int64_t src,
            int64_t* parent, int64_t* level) {
  if (src < 0 || src >= n) return -7; /* SourceOutOfRange */
  for (int64_t i = 0; i < n; ++i) { parent[i] = -1; if (level) level[i] = -1; }
  int64_t* lev = level ? level : (int64_t*)malloc((size_t)n * sizeof(int64_t));
  if (!level) for (int64_t i = 0; i < n; ++i) lev[i] = -1;
  int64_t* q = (int64_t*)malloc((size_t)(n ? n : 1) * sizeof(int64_t));
  int64_t* nq = (int64_t*)malloc((size_t)(n ? n : 1) * sizeof(int64_t));
  int64_t qn = 1;
  q[0] = src;
  parent[src] = src;
  lev[src] = 0;
  for (int64_t lv = 1; lv + 1 <= n && qn > 0; ++lv) {
    int64_t nn = 0;
    for (int64_t t = 0; t < qn; ++t) {
      int64_t k = q[t];
      for (int64_t p = rp[k]; p < rp[k + 1]; ++p) {
        int64_t j = col[p];
        if (lev[j] == -1) {
          lev[j] = lv;
          parent[j] = k;
          nq[nn++] = j;
        }
      }
    }
    qsort(nq, (size_t)nn, sizeof(int64_t), cmp_u64); /* harvest: ascending */
    int64_t* tmp = q; q = nq; nq = tmp;
    qn = nn;
  }
  free(q);
  free(nq);
  if (!level) free(lev);
  return 0;
}

/* ---- PageRank -------------------------------------------------------------
 * pagerank_gap (algo/pagerank.cpp:8-81):
 *   rank0 = 1/n (:25-26); d(k) = outdeg(k)/damping for outdeg > 0 (:30-40);
 *   per iteration: contrib = prior ./ d on the intersection (:55-56, dangling
 *   vertices contribute nothing); rank = teleport (:58); mxv plus.second with
 *   accum plus (:59-61): the row fold starts from the first hit in ascending
 *   k (core.cpp:366-378) and the accumulator adds teleport + fold (core.cpp:159);
 *   L1 change folded in ascending i from the first element (:65-73,
 *   core.cpp:814-819); stop when < tol (:74); iterations = min(k, itermax) (:76). */
int orc_pagerank(int64_t n, const int64_t* at_rp, const int32_t* at_col,
                 const int64_t* outdeg, double damping, double tol, int itermax,
                 double* rank, int* iters, double* trace) {
  if (!(damping > 0.0)) return -9; /* NonPositiveDamping */
  *iters = 0;
  if (n == 0) return 0;
  double teleport = (1.0 - damping) / (double)n;
  double* prior = (double*)malloc((size_t)n * sizeof(double));
  double* contrib = (double*)malloc((size_t)n * sizeof(double));
  for (int64_t i = 0; i < n; ++i) rank[i] = 1.0 / (double)n;
  int k;
  for (k = 1; k <= itermax; ++k) {
    memcpy(prior, rank, (size_t)n * sizeof(double));
#pragma omp parallel for schedule(static) num_threads(ORC_NT)
    for (int64_t i = 0; i < n; ++i)
      contrib[i] = outdeg[i] > 0 ? prior[i] / ((double)outdeg[i] / damping) : 0.0;
#pragma omp parallel for schedule(dynamic, 4096) num_threads(ORC_NT)
    for (int64_t i = 0; i < n; ++i) {
      int hit = 0;
      double acc = 0.0;
      for (int64_t p = at_rp[i]; p < at_rp[i + 1]; ++p) {
        int32_t kk = at_col[p];
        if (outdeg[kk] <= 0) continue; /* absent from contrib */
        acc = hit ? acc + contrib[kk] : contrib[kk];
        hit = 1;
      }
      rank[i] = hit ? teleport + acc : teleport;
    }
    if (trace) memcpy(trace + (size_t)(k - 1) * (size_t)n, rank, (size_t)n * sizeof(double));
    double norm = 0.0;
    for (int64_t i = 0; i < n; ++i) {
      double d = fabs(prior[i] - rank[i]);
      norm = (i == 0) ? d : norm + d;
    }
    if (norm < tol) break;
  }
  *iters = k < itermax ? k : itermax;
  free(prior);
  free(contrib);
  return 0;
}

/* ---- Triangle count --------------------------------------------------------
 * triangle_count (algo/triangle.cpp:30-64) computes sum(C<s(L)> = L plus.pair
 * U') -- the number of 3-cliques, which is invariant under the optional
 * degree presort (the reference's own test: test_tc.cpp:43-55, 75-85).  Any
 * exact count is therefore bit-exact; this one orients edges by id and merges
 * the higher-id neighbour lists. */
uint64_t orc_triangle_count(int64_t n, const int64_t* rp, const int32_t* col) {
  uint64_t total = 0;
#pragma omp parallel for schedule(dynamic, 256) reduction(+ : total) num_threads(ORC_NT)
  for (int64_t i = 0; i < n; ++i) {
    int64_t bi = rp[i], ei = rp[i + 1];
    int64_t si = bi;
    while (si < ei && col[si] <= i) ++si; /* U(i,:) = neighbours > i */
    for (int64_t p = si; p < ei; ++p) {
      int32_t j = col[p];
      int64_t a = p + 1, b = rp[j], eb = rp[j + 1];
      while (b < eb && col[b] <= j) ++b;
      while (a < ei && b < eb) {
        if (col[a] < col[b]) ++a;
        else if (col[a] > col[b]) ++b;
        else { ++total; ++a; ++b; }
      }
    }
  }
  return total;
}

/* ---- SSSP -----------------------------------------------------------------
 * sssp_delta_stepping (algo/sssp.cpp:16-112), restated on dense arrays:
 * light = w <= delta, heavy = w > delta (:31-34); jump to the first non-empty
 * bucket at or past frontier_lo (:57-65); relax light edges of the bucket to a
 * fixpoint, re-queueing strictly improving candidates that stay in [lo,hi)
 * (:71-94); then relax heavy edges once from every vertex that passed through
 * the bucket (:97-105).  Unreached = +inf. */
int orc_sssp_delta(int64_t n, const int64_t* rp, const int32_t* col,
                   const double* w, int64_t src, double delta, double* dist) {
  if (src < 0 || src >= n) return -7;
  if (!(delta > 0.0)) return -10;
  for (int64_t p = 0; p < rp[n]; ++p)
    if (!(w[p] > 0.0)) return -11;
  const double inf = INFINITY;
  for (int64_t i = 0; i < n; ++i) dist[i] = inf;
  dist[src] = 0.0;
  char* inb = (char*)calloc((size_t)n, 1);
  char* reach = (char*)calloc((size_t)n, 1);
  double* relaxed = (double*)malloc((size_t)n * sizeof(double));
  int64_t* bl = (int64_t*)malloc((size_t)n * sizeof(int64_t));
  int64_t* touched = (int64_t*)malloc((size_t)n * sizeof(int64_t));
  int64_t* rl = (int64_t*)malloc((size_t)n * sizeof(int64_t));
  for (int64_t i = 0; i < n; ++i) relaxed[i] = inf;
  double frontier_lo = 0.0;
  for (;;) {
    double nearest = inf;
    for (int64_t i = 0; i < n; ++i)
      if (dist[i] >= frontier_lo && dist[i] < inf && dist[i] < nearest) nearest = dist[i];
    if (nearest == inf) break;
    double lo = floor(nearest / delta) * delta;
    double hi = lo + delta;
    frontier_lo = hi;
    int64_t nb = 0, nr = 0;
    for (int64_t i = 0; i < n; ++i)
      if (dist[i] >= lo && dist[i] < hi) { bl[nb++] = i; inb[i] = 1; }
    while (nb > 0) {
      for (int64_t t = 0; t < nb; ++t)
        if (!reach[bl[t]]) { reach[bl[t]] = 1; rl[nr++] = bl[t]; }
      int64_t nt = 0;
      for (int64_t t = 0; t < nb; ++t) {
        int64_t k = bl[t];
        for (int64_t p = rp[k]; p < rp[k + 1]; ++p) {
          if (w[p] > delta) continue;
          int64_t j = col[p];
          double cand = dist[k] + w[p];
          if (relaxed[j] == inf) touched[nt++] = j;
          if (cand < relaxed[j]) relaxed[j] = cand;
        }
      }
      for (int64_t t = 0; t < nb; ++t) inb[bl[t]] = 0;
      nb = 0;
      for (int64_t t = 0; t < nt; ++t) {
        int64_t j = touched[t];
        double r = relaxed[j];
        relaxed[j] = inf;
        if (r < dist[j]) {
          if (r >= lo && r < hi && !inb[j]) { bl[nb++] = j; inb[j] = 1; }
          dist[j] = r;
        }
      }
    }
    int64_t nt = 0;
    for (int64_t t = 0; t < nr; ++t) {
      int64_t k = rl[t];
      reach[k] = 0;
      for (int64_t p = rp[k]; p < rp[k + 1]; ++p) {
        if (w[p] <= delta) continue;
        int64_t j = col[p];
        double cand = dist[k] + w[p];
        if (relaxed[j] == inf) touched[nt++] = j;
        if (cand < relaxed[j]) relaxed[j] = cand;
      }
    }
    for (int64_t t = 0; t < nt; ++t) {
      int64_t j = touched[t];
      if (relaxed[j] < dist[j]) dist[j] = relaxed[j];
      relaxed[j] = inf;
    }
  }
  free(inb); free(reach); free(relaxed); free(bl); free(touched); free(rl);
  return 0;
}

/* Dijkstra with a binary heap: verify::dijkstra (verify.cpp:133-155). */
typedef struct { double d; int64_t v; } heap_item;
static void heap_push(heap_item* h, int64_t* hn, heap_item x) {
  int64_t i = (*hn)++;
  while (i > 0) {
    int64_t p = (i - 1) / 2;
    if (h[p].d <= x.d) break;
    h[i] = h[p];
    i = p;
  }
  h[i] = x;
}
static heap_item heap_pop(heap_item* h, int64_t* hn) {
  heap_item top = h[0];
  heap_item x = h[--(*hn)];
  int64_t i = 0, nn = *hn;
  for (;;) {
    int64_t c = 2 * i + 1;
    if (c >= nn) break;
    if (c + 1 < nn && h[c + 1].d < h[c].d) ++c;
    if (h[c].d >= x.d) break;
    h[i] = h[c];
    i = c;
  }
  if (nn > 0) h[i] = x;
  return top;
}
int orc_dijkstra(int64_t n, const int64_t* rp, const int32_t* col,
                 const double* w, int64_t src, double* dist) {
  if (src < 0 || src >= n) return -7;
  for (int64_t i = 0; i < n; ++i) dist[i] = INFINITY;
  int64_t cap = rp[n] + 1;
  heap_item* h = (heap_item*)malloc((size_t)cap * sizeof(heap_item));
  int64_t hn = 0;
  dist[src] = 0.0;
  heap_item s0 = {0.0, src};
  heap_push(h, &hn, s0);
  while (hn > 0) {
    heap_item it = heap_pop(h, &hn);
    if (it.d > dist[it.v]) continue;
    for (int64_t p = rp[it.v]; p < rp[it.v + 1]; ++p) {
      double cand = dist[it.v] + w[p];
      if (cand < dist[col[p]]) {
        dist[col[p]] = cand;
        heap_item x = {cand, col[p]};
        heap_push(h, &hn, x);
      }
    }
  }
  free(h);
  return 0;
}

/* ---- Betweenness ----------------------------------------------------------
 * betweenness_centrality (algo/betweenness.cpp:11-86), one batch row at a
 * time (rows are independent in the reference's ns x n matrices):
 *   forward: F<!s(P)> = F plus.first A, Gustavson in ascending k
 *   (core.cpp:267-306), so sigma(j) = sum over previous-level k ascending;
 *   levels[d] = pattern of the d-th frontier (distance d+1) (:36-52);
 *   backward for i = L-1..1: contrib = B ./ P on levels[i];
 *   pulled<s(levels[i-1])> = contrib plus.first AT; B += pulled .* P (:58-72);
 *   centrality(j) = -ns + fold_b B(b,j) (:74-79, reduce_rows core.cpp:785-810). */
int orc_bc(int64_t n, const int64_t* rp, const int32_t* col, const int64_t* at_rp,
           const int32_t* at_col, const int64_t* sources, int64_t ns,
           double* centrality) {
  if (ns <= 0) return -8;
  for (int64_t b = 0; b < ns; ++b)
    if (sources[b] < 0 || sources[b] >= n) return -7;
  (void)at_rp; (void)at_col;
  double* Bsum = (double*)calloc((size_t)n, sizeof(double));
  double* sigma = (double*)malloc((size_t)n * sizeof(double));
  double* B = (double*)malloc((size_t)n * sizeof(double));
  double* acc = (double*)malloc((size_t)n * sizeof(double));
  int64_t* depth = (int64_t*)malloc((size_t)n * sizeof(int64_t));
  int64_t* order = (int64_t*)malloc((size_t)(n + 1) * sizeof(int64_t));
  int64_t* lstart = (int64_t*)malloc((size_t)(n + 2) * sizeof(int64_t));
  char* seen = (char*)calloc((size_t)n, 1);
  for (int64_t b = 0; b < ns; ++b) {
    for (int64_t i = 0; i < n; ++i) { sigma[i] = 0.0; depth[i] = -1; B[i] = 1.0; }
    int64_t s = sources[b];
    sigma[s] = 1.0;
    depth[s] = 0;
    /* order[] holds levels consecutively: level d occupies lstart[d]..lstart[d+1) */
    order[0] = s;
    lstart[0] = 0;
    lstart[1] = 1;
    int64_t nl = 1; /* number of levels incl. the source level */
    while (nl <= n) {
      int64_t fb = lstart[nl - 1], fe = lstart[nl];
      int64_t out = fe;
      /* Gustavson over the frontier rows, ascending k */
      for (int64_t t = fb; t < fe; ++t) {
        int64_t k = order[t];
        for (int64_t p = rp[k]; p < rp[k + 1]; ++p) {
          int64_t j = col[p];
          if (depth[j] != -1 && depth[j] < nl) continue; /* masked by !s(P) */
          if (!seen[j]) { seen[j] = 1; acc[j] = sigma[k]; order[out++] = j; depth[j] = nl; }
          else acc[j] += sigma[k];
        }
      }
      if (out == fe) break;
      qsort(order + fe, (size_t)(out - fe), sizeof(int64_t), cmp_u64);
      for (int64_t t = fe; t < out; ++t) { sigma[order[t]] = acc[order[t]]; seen[order[t]] = 0; }
      lstart[nl + 1] = out;
      ++nl;
    }
    /* reference levels[] = our levels 1..nl-1; the loop i = L-1..1 maps to
     * our depths nl-1 .. 2 pulling into depth d-1 >= 1 */
    for (int64_t d = nl - 1; d >= 2; --d) {
      /* pulled(j) = sum over k at depth d (ascending) with edge j->k of B(k)/P(k) */
      int64_t pb = lstart[d - 1], pe = lstart[d];
      for (int64_t t = pb; t < pe; ++t) acc[order[t]] = 0.0;
      for (int64_t t = lstart[d]; t < lstart[d + 1]; ++t) {
        int64_t k = order[t];
        double cv = B[k] / sigma[k];
        for (int64_t p = at_rp[k]; p < at_rp[k + 1]; ++p) {
          int64_t j = at_col[p];
          if (depth[j] == d - 1) {
            if (!seen[j]) { seen[j] = 1; acc[j] = cv; }
            else acc[j] += cv;
          }
        }
      }
      for (int64_t t = pb; t < pe; ++t) {
        int64_t j = order[t];
        if (seen[j]) { B[j] = B[j] + acc[j] * sigma[j]; seen[j] = 0; }
      }
    }
    for (int64_t i = 0; i < n; ++i) Bsum[i] = (b == 0) ? B[i] : Bsum[i] + B[i];
  }
  for (int64_t i = 0; i < n; ++i) centrality[i] = -(double)ns + Bsum[i];
  free(Bsum); free(sigma); free(B); free(acc); free(depth); free(order);
  free(lstart); free(seen);
  return 0;
}

/* ---- Connected components --------------------------------------------------
 * connected_components_fastsv (algo/components.cpp:35-106) converges to the
 * component-minimum label; verify::components (verify.cpp:191-204) is the
 * union-find restatement used here. */
static int64_t uf_find(int64_t* up, int64_t x) {
  while (up[x] != x) { up[x] = up[up[x]]; x = up[x]; }
  return x;
}
int orc_cc(int64_t n, const int64_t* rp, const int32_t* col, int64_t* label) {
  int64_t* up = (int64_t*)malloc((size_t)(n ? n : 1) * sizeof(int64_t));
  for (int64_t i = 0; i < n; ++i) up[i] = i;
  for (int64_t i = 0; i < n; ++i)
    for (int64_t p = rp[i]; p < rp[i + 1]; ++p) {
      int64_t a = uf_find(up, i), b = uf_find(up, col[p]);
      if (a != b) up[a < b ? b : a] = a < b ? a : b; /* root = smaller id */
    }
  for (int64_t i = 0; i < n; ++i) label[i] = uf_find(up, i);
  free(up);
  return 0;
}

/* sort_by_degree (util.cpp:35-44): stable ascending permutation. */
static const int64_t* g_sort_deg;
static int cmp_deg(const void* x, const void* y) {
  int64_t a = *(const int64_t*)x, b = *(const int64_t*)y;
  if (g_sort_deg[a] != g_sort_deg[b]) return g_sort_deg[a] < g_sort_deg[b] ? -1 : 1;
  return a < b ? -1 : (a > b ? 1 : 0); /* ties keep id order (stable) */
}
void orc_sort_by_degree(int64_t n, const int64_t* deg, int64_t* perm) {
  for (int64_t i = 0; i < n; ++i) perm[i] = i;
  g_sort_deg = deg;
  qsort(perm, (size_t)n, sizeof(int64_t), cmp_deg);
}

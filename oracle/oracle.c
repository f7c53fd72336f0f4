/*
 * oracle.c — plain, slow, obviously-correct CPU reference for Δ-stepping SSSP.
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library. It shares no code,
 * header or constant with the CUDA path (paper_1911_07260_b200/), and the CUDA
 * path never calls it.
 *
 * What it computes: Δ-stepping, Bellman-Ford and Dijkstra
 * all compute the SAME result — single-source shortest-path distances on a graph
 * with non-negative integer weights (§1: "computing
 * single-source shortest paths (SSSP) on graphs with non-negative edge weights
 * can be implemented either using the Bellman-Ford algorithm ... or the
 * Δ-stepping algorithm"; bucketing only changes the work done, PAPER.md:161-165;
 * priority coarsening costs work-efficiency, never exactness).
 * Since the result has a plain definition, the oracle writes that definition out
 * with the textbook algorithm (binary-heap Dijkstra) rather than following the
 * bucket algorithm.
 *
 *   dist[v] = min over directed paths s->v of the sum of uint32 weights,
 *             UINT32_MAX if no path exists (north_star; SURVEY §8c O1 overrides
 *             the paper's INT_MAX of PAPER.md:241).
 *   A finite distance >= UINT32_MAX cannot be represented -> overflow status
 *   (SURVEY §8c O2).
 *
 * All tentative sums are uint64, so no intermediate can wrap.
 *
 * Pins (tests/test_oracle.py): brute-force Bellman-Ford on tiny graphs for every
 * source, hand-worked examples (tests/golden/), closed forms (Manhattan grid,
 * path), scipy.sparse.csgraph.dijkstra, and the certificate below.
 */
#define _POSIX_C_SOURCE 199309L /* clock_gettime (timing budget only) */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

#define ORACLE_OK 0
#define ORACLE_OVERFLOW 1
#define ORACLE_BAD_INPUT -1
#define ORACLE_NOMEM -2
#define U32_INF 0xFFFFFFFFu
#define U64_INF 0xFFFFFFFFFFFFFFFFull

/* ---- indexed binary min-heap keyed by uint64 tentative distance (CLRS §6.5) ---- */
typedef struct {
  int64_t size;
  int32_t* heap;   /* heap[i] = vertex */
  int64_t* pos;    /* pos[v] = index in heap, -1 if absent */
  uint64_t* key;   /* key[v] = tentative distance D[v] */
} heap_t;

static void heap_swap(heap_t* h, int64_t i, int64_t j) {
  int32_t a = h->heap[i], b = h->heap[j];
  h->heap[i] = b; h->heap[j] = a;
  h->pos[b] = i; h->pos[a] = j;
}

static void sift_up(heap_t* h, int64_t i) {
  while (i > 0) {
    int64_t p = (i - 1) / 2;
    if (h->key[h->heap[p]] <= h->key[h->heap[i]]) break;
    heap_swap(h, i, p);
    i = p;
  }
}

static void sift_down(heap_t* h, int64_t i) {
  for (;;) {
    int64_t l = 2 * i + 1, r = l + 1, s = i;
    if (l < h->size && h->key[h->heap[l]] < h->key[h->heap[s]]) s = l;
    if (r < h->size && h->key[h->heap[r]] < h->key[h->heap[s]]) s = r;
    if (s == i) break;
    heap_swap(h, i, s);
    i = s;
  }
}

static double now_ms(void) {
  struct timespec t;
  clock_gettime(CLOCK_MONOTONIC, &t);
  return (double)t.tv_sec * 1e3 + (double)t.tv_nsec * 1e-6;
}

/* Dijkstra: D[v]=inf, D[s]=0; repeatedly extract the minimum-D vertex u and, for
 * each out-edge (u,v,w) in CSR order, lower D[v] to D[u]+w if smaller
 * (decrease-key). Output dist[v] = D[v] if finite (< UINT32_MAX), UINT32_MAX if
 * unreached; a finite D[v] >= UINT32_MAX returns ORACLE_OVERFLOW.
 *
 * budget_ms > 0 (timing only: bench.py's bounded cpu_baseline / reference sample) stops
 * the loop after that much wall time; the vertices settled so far are final, the rest of
 * dist is not. *settled / *scanned (nullable) receive the extracted vertices and the
 * out-edges examined. The arithmetic is the same with or without a budget. */
int oracle_dijkstra_budget(int64_t n, const int64_t* off, const int32_t* col, const uint32_t* w,
                           int32_t src, uint32_t* dist, double budget_ms, int64_t* settled,
                           int64_t* scanned) {
  if (n < 1 || src < 0 || src >= n || !off || !dist) return ORACLE_BAD_INPUT;
  heap_t h;
  h.size = 0;
  h.heap = (int32_t*)malloc(sizeof(int32_t) * (size_t)n);
  h.pos = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
  h.key = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)n);
  if (!h.heap || !h.pos || !h.key) { free(h.heap); free(h.pos); free(h.key); return ORACLE_NOMEM; }
  for (int64_t v = 0; v < n; ++v) { h.pos[v] = -1; h.key[v] = U64_INF; }
  unsigned char* done = (unsigned char*)calloc((size_t)n, 1);
  if (!done) { free(h.heap); free(h.pos); free(h.key); return ORACLE_NOMEM; }

  h.key[src] = 0;
  h.heap[0] = src; h.pos[src] = 0; h.size = 1;
  const double t0 = budget_ms > 0 ? now_ms() : 0.0;
  int64_t pops = 0, edges = 0;
  while (h.size > 0) {
    if (budget_ms > 0 && (pops & 1023) == 0 && pops > 0 && now_ms() - t0 > budget_ms) break;
    ++pops;
    int32_t u = h.heap[0];
    heap_swap(&h, 0, h.size - 1);
    h.size--; h.pos[u] = -1;
    sift_down(&h, 0);
    done[u] = 1;
    uint64_t du = h.key[u];
    edges += off[u + 1] - off[u];
    for (int64_t e = off[u]; e < off[u + 1]; ++e) {
      int32_t v = col[e];
      uint64_t nd = du + (uint64_t)w[e];
      if (!done[v] && nd < h.key[v]) {
        h.key[v] = nd;
        if (h.pos[v] < 0) { h.heap[h.size] = v; h.pos[v] = h.size; h.size++; }
        sift_up(&h, h.pos[v]);
      }
    }
  }
  int rc = ORACLE_OK;
  for (int64_t v = 0; v < n; ++v) {
    if (h.key[v] == U64_INF) dist[v] = U32_INF;
    else if (h.key[v] >= (uint64_t)U32_INF) { dist[v] = U32_INF; rc = ORACLE_OVERFLOW; }
    else dist[v] = (uint32_t)h.key[v];
  }
  free(h.heap); free(h.pos); free(h.key); free(done);
  if (settled) *settled = pops;
  if (scanned) *scanned = edges;
  return rc;
}

int oracle_dijkstra(int64_t n, const int64_t* off, const int32_t* col, const uint32_t* w,
                    int32_t src, uint32_t* dist) {
  return oracle_dijkstra_budget(n, off, col, w, src, dist, 0.0, NULL, NULL);
}

/* Brute-force Bellman-Ford (tiny graphs only; checks Dijkstra): n-1 full passes
 * over all m edges in uint64, D[v] = min(D[v], D[u]+w). An n-th pass must change
 * nothing (weights are unsigned, so no negative cycle can exist). */
int oracle_bellman_ford(int64_t n, const int64_t* off, const int32_t* col, const uint32_t* w,
                        int32_t src, uint32_t* dist) {
  if (n < 1 || src < 0 || src >= n || !off || !dist) return ORACLE_BAD_INPUT;
  uint64_t* D = (uint64_t*)malloc(sizeof(uint64_t) * (size_t)n);
  if (!D) return ORACLE_NOMEM;
  for (int64_t v = 0; v < n; ++v) D[v] = U64_INF;
  D[src] = 0;
  for (int64_t pass = 0; pass < n; ++pass) {
    int changed = 0;
    for (int64_t u = 0; u < n; ++u) {
      if (D[u] == U64_INF) continue;
      for (int64_t e = off[u]; e < off[u + 1]; ++e) {
        uint64_t nd = D[u] + (uint64_t)w[e];
        if (nd < D[col[e]]) { D[col[e]] = nd; changed = 1; }
      }
    }
    if (!changed) break;
    if (pass == n - 1 && changed) { free(D); return ORACLE_BAD_INPUT; }
  }
  int rc = ORACLE_OK;
  for (int64_t v = 0; v < n; ++v) {
    if (D[v] == U64_INF) dist[v] = U32_INF;
    else if (D[v] >= (uint64_t)U32_INF) { dist[v] = U32_INF; rc = ORACLE_OVERFLOW; }
    else dist[v] = (uint32_t)D[v];
  }
  free(D);
  return rc;
}

/* Transpose a CSR (in-edges of v become the row of v), counting sort; rows keep
 * source order. Needed by the certificate's tightness check on directed inputs. */
int oracle_transpose(int64_t n, int64_t m, const int64_t* off, const int32_t* col, const uint32_t* w,
                     int64_t* toff, int32_t* tcol, uint32_t* tw) {
  if (n < 1 || m < 0) return ORACLE_BAD_INPUT;
  memset(toff, 0, sizeof(int64_t) * (size_t)(n + 1));
  for (int64_t e = 0; e < m; ++e) toff[col[e] + 1]++;
  for (int64_t v = 0; v < n; ++v) toff[v + 1] += toff[v];
  int64_t* pos = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
  if (!pos) return ORACLE_NOMEM;
  memcpy(pos, toff, sizeof(int64_t) * (size_t)n);
  for (int64_t u = 0; u < n; ++u)
    for (int64_t e = off[u]; e < off[u + 1]; ++e) {
      int64_t p = pos[col[e]]++;
      tcol[p] = (int32_t)u; tw[p] = w[e];
    }
  free(pos);
  return ORACLE_OK;
}

/* Certificate (north_star's "two invariants over every edge"):
 *   C0  dist[s] == 0
 *   C1  feasibility: every edge (u,v,w) with dist[u] != INF has dist[v] <= dist[u]+w (uint64)
 *   C2  tightness: every v != s with dist[v] != INF has an in-edge (u,v,w) with
 *       dist[u] != INF and dist[u]+w == dist[v]
 * With all weights >= 1, C0 ∧ C1 ∧ C2 <=> dist is the exact SSSP distance vector.
 * In-edges come from (toff, tcol, tw) (the transpose; for symmetric graphs the
 * graph itself). Returns 0 if all hold, else 1/2/3 for the first failing check
 * and writes the offending vertex to *bad. */
int oracle_certificate(int64_t n, const int64_t* off, const int32_t* col, const uint32_t* w,
                       const int64_t* toff, const int32_t* tcol, const uint32_t* tw,
                       int32_t src, const uint32_t* dist, int64_t* bad) {
  if (n < 1 || src < 0 || src >= n) return ORACLE_BAD_INPUT;
  if (dist[src] != 0) { if (bad) *bad = src; return 1; }
  for (int64_t u = 0; u < n; ++u) {
    if (dist[u] == U32_INF) continue;
    for (int64_t e = off[u]; e < off[u + 1]; ++e) {
      if ((uint64_t)dist[col[e]] > (uint64_t)dist[u] + (uint64_t)w[e]) { if (bad) *bad = col[e]; return 2; }
    }
  }
  for (int64_t v = 0; v < n; ++v) {
    if (v == src || dist[v] == U32_INF) continue;
    int tight = 0;
    for (int64_t e = toff[v]; e < toff[v + 1] && !tight; ++e) {
      int32_t u = tcol[e];
      if (dist[u] != U32_INF && (uint64_t)dist[u] + (uint64_t)tw[e] == (uint64_t)dist[v]) tight = 1;
    }
    if (!tight) { if (bad) *bad = v; return 3; }
  }
  return 0;
}

/* ---- k-core ----------------------------------------------------
 * Coreness by the textbook serial min-degree peel (Matula & Beck 1983, in the O(n+m)
 * bin-sort form of Batagelj & Zaversnik 2003) — NOT the paper's bucketed priority queue.
 * The k-core of G is the maximal subgraph whose vertices all have induced degree >= k;
 * coreness[v] = max k with v in the k-core ("computes the maximum k-core
 * that u is contained in ... using a peeling procedure"). Degrees count stored CSR
 * entries (a parallel edge counts twice, a self-loop once), the convention the GPU path
 * also uses. Peel: repeatedly remove a vertex of minimum current degree d; its coreness is
 * d (kept monotone: never below the previous removal's value); each remaining neighbour's
 * current degree drops by one per connecting entry.
 * Returns 0, or ORACLE_BAD_INPUT / ORACLE_NOMEM. */
int oracle_kcore(int64_t n, const int64_t* off, const int32_t* col, uint32_t* core) {
  if (n < 1) return ORACLE_BAD_INPUT;
  int64_t md = 0;
  int64_t* deg = (int64_t*)malloc(sizeof(int64_t) * n);
  int64_t* pos = (int64_t*)malloc(sizeof(int64_t) * n);
  int32_t* vert = (int32_t*)malloc(sizeof(int32_t) * n);
  char* gone = (char*)calloc((size_t)n, 1);
  if (!deg || !pos || !vert || !gone) { free(deg); free(pos); free(vert); free(gone); return ORACLE_NOMEM; }
  for (int64_t v = 0; v < n; ++v) {
    deg[v] = off[v + 1] - off[v];
    if (deg[v] > md) md = deg[v];
  }
  int64_t* bin = (int64_t*)calloc((size_t)(md + 2), sizeof(int64_t));
  if (!bin) { free(deg); free(pos); free(vert); free(gone); return ORACLE_NOMEM; }
  /* counting sort of the vertices by degree: bin[d] = first position of degree d */
  for (int64_t v = 0; v < n; ++v) bin[deg[v]]++;
  int64_t start = 0;
  for (int64_t d = 0; d <= md; ++d) { int64_t c = bin[d]; bin[d] = start; start += c; }
  for (int64_t v = 0; v < n; ++v) { pos[v] = bin[deg[v]]; vert[pos[v]] = (int32_t)v; bin[deg[v]]++; }
  for (int64_t d = md; d >= 1; --d) bin[d] = bin[d - 1];
  bin[0] = 0;
  /* peel in order of current degree: vert[i] has the minimum current degree among
     the vertices not yet removed */
  for (int64_t i = 0; i < n; ++i) {
    int32_t v = vert[i];
    core[v] = (uint32_t)deg[v];
    gone[v] = 1;
    for (int64_t e = off[v]; e < off[v + 1]; ++e) {
      int32_t u = col[e];
      if (gone[u] || deg[u] <= deg[v]) continue;
      /* move u to the front of its degree bin, then shrink its degree by one */
      int64_t du = deg[u], pu = pos[u], pw = bin[du];
      int32_t w = vert[pw];
      if (u != w) { pos[u] = pw; vert[pu] = w; pos[w] = pu; vert[pw] = u; }
      bin[du]++;
      deg[u]--;
    }
  }
  free(deg); free(pos); free(vert); free(gone); free(bin);
  return ORACLE_OK;
}

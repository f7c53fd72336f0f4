// gigen — seeded synthetic CSR graph generators (shared test/bench input module).
//
// This module is the ONLY code shared between the oracle (oracle/) and the CUDA
// path (paper_1911_07260_b200/). It holds none of the method's arithmetic: it
// only builds input graphs. Recipe: SURVEY.md §8(d) "Generator (proposed exact
// recipe)", standing in for the paper's datasets (PAPER.md:885-904,
// table:datasets) — road networks (RD/GE) and skewed social graphs.
//
//  * mix64 = SplitMix64 finalizer; S(seed,tag) = mix64((seed<<8)|tag);
//    H(seed,tag,x) = mix64(S ^ x); U32 = H >> 32.
//  * integer in [lo,hi): lo + ((U32*(hi-lo)) >> 32); Bernoulli(p): U32 < floor(p*2^32).
//  * canonical undirected key K(u,v) = (min<<32)|max; weight drawn from (seed,W,K),
//    identical for both directions.
//  * CSR canonical: rows by source id, neighbours ascending, no duplicates.
//
// Output CSR: int64 offsets[n+1], int32 cols[m], uint32 w[m]; buffers are
// malloc'ed here and released with gigen_free().
#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <omp.h>

namespace {

enum : uint64_t { TAG_W = 1, TAG_DEL = 2, TAG_DIAG = 3, TAG_RMAT = 4, TAG_SRC = 5, TAG_UNI = 6 };

inline uint64_t mix64(uint64_t z) {
  z ^= z >> 30; z *= 0xBF58476D1CE4E5B9ull;
  z ^= z >> 27; z *= 0x94D049BB133111EBull;
  z ^= z >> 31; return z;
}
inline uint64_t stream_key(uint64_t seed, uint64_t tag) { return mix64((seed << 8) | tag); }
inline uint32_t u32_of(uint64_t skey, uint64_t x) { return (uint32_t)(mix64(skey ^ x) >> 32); }
inline uint32_t in_range(uint32_t u, uint32_t lo, uint32_t hi) {
  return lo + (uint32_t)(((uint64_t)u * (uint64_t)(hi - lo)) >> 32);
}
inline uint64_t ukey(uint32_t u, uint32_t v) {
  uint32_t a = u < v ? u : v, b = u < v ? v : u;
  return ((uint64_t)a << 32) | b;
}

}  // namespace

extern "C" {

typedef struct {
  int64_t n, m;
  int64_t* offsets;
  int32_t* cols;
  uint32_t* w;
} gigen_csr;

void gigen_free(gigen_csr* g) {
  if (!g) return;
  free(g->offsets); free(g->cols); free(g->w);
  g->offsets = nullptr; g->cols = nullptr; g->w = nullptr;
}

uint64_t gigen_mix64(uint64_t z) { return mix64(z); }
uint32_t gigen_u32(uint64_t seed, uint64_t tag, uint64_t x) { return u32_of(stream_key(seed, tag), x); }

// Grid / road-like graph.
// rows x cols lattice, id = r*cols + c. Each lattice edge is DELETED iff
// U32(seed,DEL,K) < del_thresh; each of the two diagonals of every cell is ADDED
// iff U32(seed,DIAG,K) < diag_thresh. Weights U[w_lo, w_hi) from (seed,W,K).
// Thresholds are floor(p*2^32) (0 => never).
int gigen_grid(int64_t rows, int64_t cols, uint32_t w_lo, uint32_t w_hi, uint64_t seed,
               uint32_t del_thresh, uint32_t diag_thresh, gigen_csr* out) {
  if (rows < 1 || cols < 1 || rows * cols > INT32_MAX || w_hi <= w_lo || !out) return -1;
  const int64_t n = rows * cols;
  const uint64_t kdel = stream_key(seed, TAG_DEL), kdiag = stream_key(seed, TAG_DIAG),
                 kw = stream_key(seed, TAG_W);
  auto lattice_present = [&](uint32_t a, uint32_t b) -> bool {
    return del_thresh == 0 ? true : !(u32_of(kdel, ukey(a, b)) < del_thresh);
  };
  auto diag_present = [&](uint32_t a, uint32_t b) -> bool {
    return diag_thresh == 0 ? false : (u32_of(kdiag, ukey(a, b)) < diag_thresh);
  };
  // neighbour candidate list in ascending id order for vertex (r,c)
  auto for_each_nbr = [&](int64_t r, int64_t c, auto&& f) {
    const int64_t id = r * cols + c;
    // up-left, up, up-right (ids id-cols-1, id-cols, id-cols+1)
    if (r > 0) {
      if (c > 0) { int64_t o = id - cols - 1; if (diag_present(id, o)) f(o); }
      { int64_t o = id - cols; if (lattice_present(id, o)) f(o); }
      if (c + 1 < cols) { int64_t o = id - cols + 1; if (diag_present(id, o)) f(o); }
    }
    if (c > 0) { int64_t o = id - 1; if (lattice_present(id, o)) f(o); }
    if (c + 1 < cols) { int64_t o = id + 1; if (lattice_present(id, o)) f(o); }
    if (r + 1 < rows) {
      if (c > 0) { int64_t o = id + cols - 1; if (diag_present(id, o)) f(o); }
      { int64_t o = id + cols; if (lattice_present(id, o)) f(o); }
      if (c + 1 < cols) { int64_t o = id + cols + 1; if (diag_present(id, o)) f(o); }
    }
  };
  int64_t* off = (int64_t*)malloc(sizeof(int64_t) * (n + 1));
  if (!off) return -2;
  off[0] = 0;
#pragma omp parallel for schedule(static)
  for (int64_t v = 0; v < n; ++v) {
    int64_t d = 0;
    for_each_nbr(v / cols, v % cols, [&](int64_t) { ++d; });
    off[v + 1] = d;
  }
  for (int64_t v = 0; v < n; ++v) off[v + 1] += off[v];
  const int64_t m = off[n];
  int32_t* cl = (int32_t*)malloc(sizeof(int32_t) * (m ? m : 1));
  uint32_t* w = (uint32_t*)malloc(sizeof(uint32_t) * (m ? m : 1));
  if (!cl || !w) { free(off); free(cl); free(w); return -2; }
#pragma omp parallel for schedule(static)
  for (int64_t v = 0; v < n; ++v) {
    int64_t p = off[v];
    for_each_nbr(v / cols, v % cols, [&](int64_t o) {
      cl[p] = (int32_t)o;
      w[p] = in_range(u32_of(kw, ukey((uint32_t)v, (uint32_t)o)), w_lo, w_hi);
      ++p;
    });
  }
  out->n = n; out->m = m; out->offsets = off; out->cols = cl; out->w = w;
  return 0;
}

// Canonicalise an undirected edge multiset given as a per-row fill: sort rows,
// drop duplicates, compact, then draw weights from (seed,W,K).
static int finish_symmetric(int64_t n, int64_t* off, int32_t* cl, uint32_t w_lo, uint32_t w_hi,
                            uint64_t seed, gigen_csr* out) {
  // per-row sort + unique; record unique counts
  std::vector<int64_t> ucount(n);
#pragma omp parallel for schedule(dynamic, 1024)
  for (int64_t v = 0; v < n; ++v) {
    int32_t* b = cl + off[v];
    int32_t* e = cl + off[v + 1];
    std::sort(b, e);
    ucount[v] = std::unique(b, e) - b;
  }
  // compact in place (destination never passes the source)
  int64_t pos = 0;
  for (int64_t v = 0; v < n; ++v) {
    int64_t b = off[v];
    int64_t c = ucount[v];
    if (pos != b && c) memmove(cl + pos, cl + b, sizeof(int32_t) * c);
    off[v] = pos;
    pos += c;
  }
  off[n] = pos;
  const int64_t m = pos;
  int32_t* cl2 = (int32_t*)realloc(cl, sizeof(int32_t) * (m ? m : 1));
  if (cl2) cl = cl2;
  uint32_t* w = (uint32_t*)malloc(sizeof(uint32_t) * (m ? m : 1));
  if (!w) { free(off); free(cl); return -2; }
  const uint64_t kw = stream_key(seed, TAG_W);
#pragma omp parallel for schedule(dynamic, 4096)
  for (int64_t v = 0; v < n; ++v)
    for (int64_t p = off[v]; p < off[v + 1]; ++p)
      w[p] = in_range(u32_of(kw, ukey((uint32_t)v, (uint32_t)cl[p])), w_lo, w_hi);
  out->n = n; out->m = m; out->offsets = off; out->cols = cl; out->w = w;
  return 0;
}

// RMAT. Sample e in [0, edge_factor*2^scale), level
// l = 0..scale-1: r = U32(seed,RMAT,e*scale+l); row bit = r >= t2; column bit =
// (t1 <= r < t2) || r >= t3; bits appended MSB-first. Self-loops dropped, dedup
// on K, both directions stored; no noise, no permutation.
int gigen_rmat(int32_t scale, int32_t edge_factor, uint32_t t1, uint32_t t2, uint32_t t3,
               uint32_t w_lo, uint32_t w_hi, uint64_t seed, gigen_csr* out) {
  if (scale < 1 || scale > 30 || edge_factor < 1 || w_hi <= w_lo || !out) return -1;
  const int64_t n = (int64_t)1 << scale;
  const int64_t ns = (int64_t)edge_factor << scale;
  const uint64_t kr = stream_key(seed, TAG_RMAT);
  auto sample = [&](int64_t e, uint32_t& u, uint32_t& v) {
    uint32_t a = 0, b = 0;
    const uint64_t x0 = (uint64_t)e * (uint64_t)scale;
    for (int l = 0; l < scale; ++l) {
      uint32_t r = u32_of(kr, x0 + (uint64_t)l);
      uint32_t rb = r >= t2;
      uint32_t cb = (r >= t1 && r < t2) || r >= t3;
      a = 2 * a + rb; b = 2 * b + cb;
    }
    u = a; v = b;
  };
  // pass 1: degree counts (with duplicates), both directions
  std::atomic<int64_t>* cnt = new (std::nothrow) std::atomic<int64_t>[n];
  if (!cnt) return -2;
#pragma omp parallel for schedule(static)
  for (int64_t v = 0; v < n; ++v) cnt[v].store(0, std::memory_order_relaxed);
#pragma omp parallel for schedule(static, 65536)
  for (int64_t e = 0; e < ns; ++e) {
    uint32_t u, v; sample(e, u, v);
    if (u == v) continue;
    cnt[u].fetch_add(1, std::memory_order_relaxed);
    cnt[v].fetch_add(1, std::memory_order_relaxed);
  }
  int64_t* off = (int64_t*)malloc(sizeof(int64_t) * (n + 1));
  if (!off) { delete[] cnt; return -2; }
  off[0] = 0;
  for (int64_t v = 0; v < n; ++v) off[v + 1] = off[v] + cnt[v].load(std::memory_order_relaxed);
  const int64_t mraw = off[n];
  int32_t* cl = (int32_t*)malloc(sizeof(int32_t) * (mraw ? mraw : 1));
  if (!cl) { delete[] cnt; free(off); return -2; }
#pragma omp parallel for schedule(static)
  for (int64_t v = 0; v < n; ++v) cnt[v].store(off[v], std::memory_order_relaxed);
  // pass 2: fill (order inside a row is arbitrary; rows are sorted afterwards)
#pragma omp parallel for schedule(static, 65536)
  for (int64_t e = 0; e < ns; ++e) {
    uint32_t u, v; sample(e, u, v);
    if (u == v) continue;
    cl[cnt[u].fetch_add(1, std::memory_order_relaxed)] = (int32_t)v;
    cl[cnt[v].fetch_add(1, std::memory_order_relaxed)] = (int32_t)u;
  }
  delete[] cnt;
  return finish_symmetric(n, off, cl, w_lo, w_hi, seed, out);
}

// Symmetric edge list -> canonical CSR (used for small hand-built and
// uniform-random graphs; duplicates removed). Edges (u[i], v[i]); self-loops dropped.
int gigen_from_undirected(int64_t n, int64_t ne, const int32_t* us, const int32_t* vs,
                          uint32_t w_lo, uint32_t w_hi, uint64_t seed, gigen_csr* out) {
  if (n < 1 || ne < 0 || w_hi <= w_lo || !out) return -1;
  int64_t* off = (int64_t*)calloc(n + 1, sizeof(int64_t));
  if (!off) return -2;
  for (int64_t i = 0; i < ne; ++i) {
    if (us[i] < 0 || us[i] >= n || vs[i] < 0 || vs[i] >= n) { free(off); return -1; }
    if (us[i] == vs[i]) continue;
    off[us[i] + 1]++; off[vs[i] + 1]++;
  }
  for (int64_t v = 0; v < n; ++v) off[v + 1] += off[v];
  int32_t* cl = (int32_t*)malloc(sizeof(int32_t) * (off[n] ? off[n] : 1));
  std::vector<int64_t> pos(off, off + n);
  for (int64_t i = 0; i < ne; ++i) {
    if (us[i] == vs[i]) continue;
    cl[pos[us[i]]++] = vs[i];
    cl[pos[vs[i]]++] = us[i];
  }
  return finish_symmetric(n, off, cl, w_lo, w_hi, seed, out);
}

// Batch sources: s_j = (U32(seed,SRC,j) * n) >> 32 for
// j = 0,1,..., skipping repeats until k distinct ids are chosen.
int gigen_sources(int64_t n, int32_t k, uint64_t seed, int32_t* out) {
  if (n < 1 || k < 0 || k > n) return -1;
  const uint64_t ks = stream_key(seed, TAG_SRC);
  std::vector<int32_t> got;
  for (uint64_t j = 0; (int32_t)got.size() < k; ++j) {
    int32_t s = (int32_t)(((uint64_t)u32_of(ks, j) * (uint64_t)n) >> 32);
    if (std::find(got.begin(), got.end(), s) == got.end()) got.push_back(s);
  }
  for (int32_t i = 0; i < k; ++i) out[i] = got[i];
  return 0;
}

// Uniform random directed multigraph ("uniform_random"): m edges
// drawn with replacement, self-loops rejected and redrawn; weights U[w_lo,w_hi).
// Parallel edges are KEPT. Rows sorted by (col, w) for canonical order.
int gigen_uniform(int64_t n, int64_t m, uint32_t w_lo, uint32_t w_hi, uint64_t seed, gigen_csr* out) {
  if (n < 2 || m < 0 || w_hi <= w_lo || !out) return -1;
  const uint64_t ku = stream_key(seed, TAG_UNI), kw = stream_key(seed, TAG_W);
  std::vector<int32_t> su(m), sv(m);
  std::vector<uint32_t> sw(m);
  uint64_t x = 0;
  for (int64_t i = 0; i < m; ++i) {
    int32_t u, v;
    do {
      u = (int32_t)(((uint64_t)u32_of(ku, x++) * (uint64_t)n) >> 32);
      v = (int32_t)(((uint64_t)u32_of(ku, x++) * (uint64_t)n) >> 32);
    } while (u == v);
    su[i] = u; sv[i] = v; sw[i] = in_range(u32_of(kw, (uint64_t)i), w_lo, w_hi);
  }
  int64_t* off = (int64_t*)calloc(n + 1, sizeof(int64_t));
  int32_t* cl = (int32_t*)malloc(sizeof(int32_t) * (m ? m : 1));
  uint32_t* w = (uint32_t*)malloc(sizeof(uint32_t) * (m ? m : 1));
  if (!off || !cl || !w) { free(off); free(cl); free(w); return -2; }
  for (int64_t i = 0; i < m; ++i) off[su[i] + 1]++;
  for (int64_t v = 0; v < n; ++v) off[v + 1] += off[v];
  std::vector<int64_t> idx(m);
  std::vector<int64_t> pos(off, off + n);
  for (int64_t i = 0; i < m; ++i) idx[pos[su[i]]++] = i;
  for (int64_t v = 0; v < n; ++v)
    std::sort(idx.begin() + off[v], idx.begin() + off[v + 1], [&](int64_t a, int64_t b) {
      return sv[a] != sv[b] ? sv[a] < sv[b] : sw[a] < sw[b];
    });
  for (int64_t p = 0; p < m; ++p) { cl[p] = sv[idx[p]]; w[p] = sw[idx[p]]; }
  out->n = n; out->m = m; out->offsets = off; out->cols = cl; out->w = w;
  return 0;
}

int gigen_num_threads(void) { return omp_get_max_threads(); }

}  // extern "C"

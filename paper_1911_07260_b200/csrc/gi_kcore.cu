// gi_kcore.cu — k-core (coreness of every vertex) on sm_100a: bucketed peeling with
// lazy bucket updates and the constant-sum ("histogram") reduction.
//
// The method (Fig. 10 at PAPER.md:1591-1618; the transformed update of
// Fig. kcore_udf at PAPER.md:802-837): priorities start at the degrees; repeatedly take
// the minimum non-empty bucket k, finish its vertices with coreness k, and lower each
// neighbour's priority by the number of its finished neighbours, never below k
// ("std::max(priority + (-1) * count, k)"). There is no priority coarsening.
//
// B200 mapping (one persistent cooperative kernel, phases separated by a group barrier,
// the same phase protocol as the SSSP kernel):
//   EXTRACT(k) — the "pile" (every unfinished vertex, the lazy buckets: no bucket ids are
//                stored; a vertex's bucket is its current priority, read when extracted)
//                is partitioned: priority <= k -> finished with coreness k and appended
//                to the frontier; otherwise kept, and its priority min-reduced into the
//                next k.
//   ROUND(k)   — every edge of the frontier lowers its endpoint's priority. The
//                decrements of one warp to the same vertex are combined first
//                (__match_any_sync: the GPU form of the histogram of counts, so a vertex
//                with many frontier neighbours takes one atomic per warp, not one per
//                edge); the single atomic whose subtraction crosses from > k to <= k
//                finishes that vertex with coreness k and appends it to the next
//                frontier (same k) — so a vertex is finished exactly once and no dedup
//                bit is needed. The floor max(., k) is implicit: a priority that dips below
//                k belongs to a finished vertex, which every later edge skips.
// Frontier chunks are claimed dynamically (skewed degrees) and relaxed edge-balanced:
// block scan of the chunk's degrees, 8 consecutive edges per thread per iteration.
// Bucket fusion carries over (the current bucket k is processed eagerly, R1): vertices
// finished by an extraction or a crossing go to a CTA-local bin drained with CTA barriers
// while it holds < T vertices; a larger bin spills to the global frontier.
#include "gi_internal.h"
#include "gi_device.cuh"

#include <cooperative_groups.h>

namespace gi {
namespace {

namespace cg = cooperative_groups;

constexpr int kKcBlock = 512;
constexpr int kKcEdges = 8;     // consecutive edges per thread per iteration
constexpr int kKcChunk = 2048;  // frontier vertices staged per claim / per local bin (max)
#ifndef GI_KC_LANE_PUSH
#define GI_KC_LANE_PUSH 1
#endif
// slot path (low-degree graphs): combine a warp's decrements of one vertex first
// (__match_any_sync) or send one atomic per edge — on a grid two frontier vertices of a
// warp rarely share a neighbour, so the match is mostly overhead
#ifndef GI_KC_SLOT_MATCH
#define GI_KC_SLOT_MATCH 0
#endif
#ifndef GI_KCT
#define GI_KCT 1024
#endif
// slot path: prefetch a finished vertex's slot into L1 only when it lands below T in this
// CTA's bin (drained here); otherwise (spilled, or a bin that will spill) the slots of a big
// layer only flush the L2
#ifndef GI_KC_PFLOCAL
#define GI_KC_PFLOCAL 1  // config 2: 8.65 -> 7.80 ms, config 3 9.46 -> 9.42 ms (profiles/r02aq_kcore_ab.txt)
#endif
constexpr uint32_t kKcT = GI_KCT; // bucket fusion threshold: a local bin of >= T vertices spills
constexpr uint32_t kKcHub = 1024;  // out-degree >= this: edges split over every CTA in the next round
constexpr uint32_t kUnset = 0xFFFFFFFFu;

enum : uint32_t { KC_ROUND = 0, KC_EXTRACT = 1, KC_DONE = 2 };

struct KcShared {
  uint32_t mode, k, cnt, claim, kmin, hn;
  uint32_t bincnt[3];           // local bin fills, rotating by drain iteration
  unsigned long long total;
  unsigned long long red[kKcBlock / 32];
  uint32_t woff[kKcBlock / 32];  // extraction: per-warp offsets of the kept entries
  uint32_t pbase;                // extraction: this CTA's slot in the next pile
};

struct KcSmem {
  long long* beg;               // [kKcChunk] staged edge offsets
  uint32_t* deg;                // [kKcChunk] staged degrees
  unsigned long long* pre;      // [kKcChunk] exclusive prefix of the staged degrees
  int32_t* bin[2];              // [kKcChunk] local bins (bucket fusion of the current k)
};

// Per-phase relaxation context.
struct KcCtx {
  uint32_t k;
  int32_t* q_next;              // global frontier (spill target)
  uint32_t* qcount_next;
  int32_t* out;                 // local bin receiving crossings (shared memory)
  uint32_t* outcnt;
  const uint2* pf;              // slot path with GI_KC_PFLOCAL: slots prefetched on local pushes
  HubEnt* hub_next;             // group hub list receiving this phase's hubs
  uint32_t* hcount_next;
  uint32_t hubcap;
  uint32_t my_kmin;
  unsigned long long nfin, nedge;
};

__device__ __forceinline__ uint32_t ld_cg(const uint32_t* p) { return __ldcg(p); }
__device__ __forceinline__ void prefetch_l1(const void* p) { asm volatile("prefetch.global.L1 [%0];" ::"l"(p)); }

// Warp-aggregated append of v (lanes with `want`) to a global list.
__device__ __forceinline__ void kc_append(bool want, int32_t v, int32_t* list, uint32_t* count) {
  const uint32_t m = __ballot_sync(0xffffffffu, want);
  if (!m) return;
  const uint32_t lane = threadIdx.x & 31;
  uint32_t base = 0;
  if (lane == 0) base = atomicAdd(count, (uint32_t)__popc(m));
  base = __shfl_sync(0xffffffffu, base, 0);
  if (want) list[base + __popc(m & ((1u << lane) - 1u))] = v;
}

// A vertex finished at k joins the current bucket's frontier: the CTA-local bin (bucket
// fusion: drained in this phase, no group barrier) or, when the bin is full, the global
// frontier (the next group-wide round). Called by all 32 lanes.
__device__ __forceinline__ void kc_push(KcCtx& c, bool want, int32_t v) {
  if (GI_KC_LANE_PUSH) {
    // one shared atomic per pushing lane (as SSSP's bin pushes), and a full bin spills per
    // lane too: no warp-collective operation after the decrements (a lane would wait for
    // the warp's slowest atomic before pushing)
    if (want) {
      const uint32_t pos = atomicAdd(c.outcnt, 1u);
      if (pos < (uint32_t)kKcChunk) {
        c.out[pos] = v;
        if (GI_KC_PFLOCAL && c.pf && pos < kKcT) prefetch_l1(c.pf + 8 * (size_t)v);
      } else {
        cg::coalesced_group g = cg::coalesced_threads();
        uint32_t base = 0;
        if (g.thread_rank() == 0) base = atomicAdd(c.qcount_next, g.size());
        base = g.shfl(base, 0);
        c.q_next[base + g.thread_rank()] = v;
      }
    }
    return;
  }
  const uint32_t m = __ballot_sync(0xffffffffu, want);
  if (!m) return;
  const uint32_t lane = threadIdx.x & 31;
  uint32_t base = 0;
  if (lane == 0) base = atomicAdd(c.outcnt, (uint32_t)__popc(m));
  base = __shfl_sync(0xffffffffu, base, 0);
  const uint32_t pos = base + __popc(m & ((1u << lane) - 1u));
  const bool spill = want && pos >= (uint32_t)kKcChunk;
  if (want && !spill) c.out[pos] = v;
  kc_append(spill, v, c.q_next, c.qcount_next);
}

// Stage the cnt (<= kKcChunk) frontier vertices of `list` (global or shared) as (offset,
// degree) entries; a vertex of degree >= kKcHub goes to the group hub list instead (its
// edges are split over every CTA in the next round) and is staged with degree 0.
__device__ __forceinline__ void kc_stage_vertices(const KcArgs& a, const KcSmem& m, KcCtx& c, const int32_t* list,
                                                  uint32_t cnt) {
  const uint32_t lane = threadIdx.x & 31;
  for (uint32_t i0 = 0; i0 < cnt; i0 += kKcBlock) {  // warp-uniform trip count
    const uint32_t i = i0 + threadIdx.x;
    const bool in = i < cnt;
    long long b0 = 0;
    uint32_t d = 0;
    if (in) {
      const int32_t v = list[i];
      b0 = a.off[v];
      d = (uint32_t)(a.off[v + 1] - b0);
    }
    // hubs: one global atomic per warp (every CTA appends to the same counter)
    const bool hub = in && d >= kKcHub;
    const uint32_t mh = __ballot_sync(0xffffffffu, hub);
    uint32_t hbase = 0;
    if (mh) {
      if (lane == 0) hbase = atomicAdd(c.hcount_next, (uint32_t)__popc(mh));
      hbase = __shfl_sync(0xffffffffu, hbase, 0);
    }
    if (hub) {
      const uint32_t hp = hbase + __popc(mh & ((1u << lane) - 1u));
      if (hp < c.hubcap) {
        HubEnt he;
        he.beg = b0;
        he.deg = d;
        he.du = 0;
        c.hub_next[hp] = he;
        d = 0;
      }
    }
    if (in) {
      m.beg[i] = b0;
      m.deg[i] = d;
    }
  }
  __syncthreads();
}

// Relax every edge of the cnt staged entries (m.beg, m.deg): block scan of the degrees,
// 8 consecutive edges per thread per iteration. Starts after and ends with a CTA barrier;
// all threads call it.
__device__ __forceinline__ void kc_relax_entries(const KcArgs& a, KcShared& s, const KcSmem& m, KcCtx& c,
                                                 uint32_t cnt) {
  const uint32_t tid = threadIdx.x, lane = tid & 31;
  const uint32_t k = c.k;
  unsigned long long sum = 0;
  constexpr int PER = kKcChunk / kKcBlock;
  unsigned long long loc[PER];
#pragma unroll
  for (int x = 0; x < PER; ++x) {
    const uint32_t i = tid * PER + x;
    loc[x] = sum;
    if (i < cnt) sum += m.deg[i];
  }
  unsigned long long incl = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= (uint32_t)o) incl += t;
  }
  if (lane == 31) s.red[tid >> 5] = incl;
  __syncthreads();
  if (tid < 32) {
    const unsigned long long w = lane < kKcBlock / 32 ? s.red[lane] : 0ull;
    unsigned long long wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long t = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= (uint32_t)o) wi += t;
    }
    if (lane < kKcBlock / 32) s.red[lane] = wi - w;
    if (lane == kKcBlock / 32 - 1) s.total = wi;
  }
  __syncthreads();
  const unsigned long long off0 = s.red[tid >> 5] + incl - sum;
#pragma unroll
  for (int x = 0; x < PER; ++x) {
    const uint32_t i = tid * PER + x;
    if (i < cnt) m.pre[i] = off0 + loc[x];
  }
  __syncthreads();
  const unsigned long long total = s.total;
  if (tid == 0) c.nedge += total;
  for (unsigned long long k0 = 0; k0 < total; k0 += (unsigned long long)kKcEdges * kKcBlock) {
    int32_t tv[kKcEdges];
#pragma unroll
    for (int u = 0; u < kKcEdges; ++u) tv[u] = -1;
    const unsigned long long kt = k0 + (unsigned long long)kKcEdges * tid;
    if (kt < total) {
      uint32_t lo = 0, hi = cnt;  // last i with pre[i] <= kt
      while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (m.pre[mid] <= kt) lo = mid; else hi = mid;
      }
      unsigned long long nxt = lo + 1 < cnt ? m.pre[lo + 1] : total;
      long long rel = m.beg[lo] - (long long)m.pre[lo];
#pragma unroll
      for (int u = 0; u < kKcEdges; ++u) {
        const unsigned long long e = kt + u;
        if (e < total) {
          while (e >= nxt) {  // next frontier vertex (skipping degree-0 ones)
            ++lo;
            rel = m.beg[lo] - (long long)nxt;
            nxt = lo + 1 < cnt ? m.pre[lo + 1] : total;
          }
          tv[u] = (int32_t)__ldg(&a.edges[rel + (long long)e].x);
        }
      }
    }
    // skip finished endpoints (coherent read; finished is final)
    uint32_t cv[kKcEdges];
#pragma unroll
    for (int u = 0; u < kKcEdges; ++u) cv[u] = tv[u] >= 0 ? ld_cg(a.core + tv[u]) : 0u;
    // constant-sum reduction: one atomic per distinct endpoint per warp; all 8 atomics
    // of a thread in flight together, then the crossings
    uint32_t lead = 0, cntp[kKcEdges], old[kKcEdges];
#pragma unroll
    for (int u = 0; u < kKcEdges; ++u) {
      const bool want = tv[u] >= 0 && cv[u] == kUnset;
      const uint32_t key = want ? (uint32_t)tv[u] : 0xFFFFFFFFu;
      const uint32_t peers = __match_any_sync(0xffffffffu, key);
      cntp[u] = __popc(peers);
      if (want && (__ffs(peers) - 1) == (int)lane) lead |= 1u << u;
    }
#pragma unroll
    for (int u = 0; u < kKcEdges; ++u) old[u] = (lead & (1u << u)) ? atomicSub(a.prio + tv[u], cntp[u]) : 0u;
#pragma unroll
    for (int u = 0; u < kKcEdges; ++u) {
      bool cross = false;
      if (lead & (1u << u)) {
        if (old[u] > k && old[u] - cntp[u] <= k) {
          // this subtraction took the priority to <= k: finished at k — claimed with a CAS,
          // since another CTA's extraction scan (same phase) may see the lowered priority
          cross = atomicCAS(a.core + tv[u], kUnset, k) == kUnset;
        } else if (old[u] > k) {
          c.my_kmin = min(c.my_kmin, old[u] - cntp[u]);
        }
      }
      c.nfin += cross;
      kc_push(c, cross, tv[u]);
    }
  }
  __syncthreads();
}

// Low-degree graphs (every adjacency in its 64-byte ELL slot, a.ld): relax the edges of the
// cnt vertices of `list` (global frontier or shared-memory bin) with one octet of lanes per
// vertex — lane k of the octet takes entry k of the slot (one coalesced 64-byte load per
// vertex, prefetched into L1 when the vertex was pushed into this CTA's bin). The chain of
// a fused sub-round is then slot (L1) -> decrement (L2) -> push, instead of offsets ->
// edges -> coreness probe -> decrement -> claim:
//   - no coreness probe: a finished vertex's priority is <= its coreness and every later
//     decrement keeps it there (the decrements of a vertex sum to its degree, its initial
//     priority, so it never wraps), so only an unfinished vertex can cross from > k to <= k;
//   - no CAS claim: in the slot path the extraction and the drains of a phase are separated
//     by a group barrier, so the one crossing subtraction is the vertex's only claimant and
//     writes its coreness with a plain store.
// the column of an ELL slot entry, optionally with an L2 evict-first policy (the slots
// stream through once per peel; the priorities should stay in L2)
#ifndef GI_KC_SLOT_EF
#define GI_KC_SLOT_EF 1
#endif
__device__ __forceinline__ uint32_t kc_ld_slot(const uint2* p) {
#if GI_KC_SLOT_EF
  uint64_t pol;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  uint32_t x;
  asm volatile("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(x) : "l"(p), "l"(pol));
  return x;
#else
  return __ldg(p).x;
#endif
}

// Called by all threads; ends with a CTA barrier.
template <int U>
__device__ __forceinline__ void kc_relax_slots(const KcArgs& a, KcCtx& c, const int32_t* list, uint32_t cnt) {
  const uint32_t tid = threadIdx.x, lane = tid & 31, sub = tid & 7;
  const uint32_t k = c.k;
  const uint32_t nitems = cnt * 8;
  for (uint32_t base = 0; base < nitems; base += kKcBlock * U) {  // block-uniform trip count
    uint32_t tv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t item = base + u * kKcBlock + tid;
      tv[u] = kColEmpty;
      if (item < nitems) tv[u] = kc_ld_slot(a.slots + 8 * (size_t)list[item >> 3] + sub);
    }
    uint32_t lead = 0, cntp[U], old[U];
    unsigned ne = 0;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const bool want = tv[u] != kColEmpty;
      ne += want;
      if (GI_KC_SLOT_MATCH) {
        const uint32_t peers = __match_any_sync(0xffffffffu, tv[u]);
        cntp[u] = __popc(peers);
        if (want && (__ffs(peers) - 1) == (int)lane) lead |= 1u << u;
      } else {  // one decrement per edge: the crossing test holds per atomic all the same
        cntp[u] = 1;
        if (want) lead |= 1u << u;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) old[u] = (lead & (1u << u)) ? atomicSub(a.prio + tv[u], cntp[u]) : 0u;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      bool cross = false;
      if (lead & (1u << u)) {
        if (old[u] > k && old[u] - cntp[u] <= k) {
          cross = true;
          a.core[tv[u]] = k;
          if (!GI_KC_PFLOCAL) prefetch_l1(a.slots + 8 * (size_t)tv[u]);  // relaxed by this CTA next sub-round
        } else if (old[u] > k) {
          c.my_kmin = min(c.my_kmin, old[u] - cntp[u]);
        }
      }
      c.nfin += cross;
      kc_push(c, cross, (int32_t)tv[u]);
    }
    c.nedge += ne;
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kKcBlock, 1) kcore_persistent(KcArgs a) {
  extern __shared__ unsigned long long kc_dyn[];  // beg, pre [kKcChunk] 8 B; bins [2][kKcChunk] 4 B
  __shared__ KcShared s;
  KcSmem sm;
  sm.beg = reinterpret_cast<long long*>(kc_dyn);
  sm.pre = kc_dyn + kKcChunk;
  sm.bin[0] = reinterpret_cast<int32_t*>(kc_dyn + 2 * kKcChunk);
  sm.bin[1] = sm.bin[0] + kKcChunk;
  sm.deg = reinterpret_cast<uint32_t*>(sm.bin[1] + kKcChunk);
  const uint32_t G = gridDim.x, rank = blockIdx.x, tid = threadIdx.x;
  const uint32_t lane = tid & 31;
  const int64_t n = a.n;
  KcCtl* ctl = a.ctl;

  // ---- init: priority = degree, coreness unset, pile = every vertex (PAPER.md:1600-1603,
  // "new priority_queue{Vertex}(uint)(false, \"lower_first\", D)") ----
  {
    uint32_t mn = kUnset;
    for (int64_t v = (int64_t)rank * kKcBlock + tid; v < n; v += (int64_t)G * kKcBlock) {
      const int64_t d = a.off[v + 1] - a.off[v];
      const uint32_t pv = d >= (int64_t)kUnset ? kUnset - 1u : (uint32_t)d;
      a.prio[v] = pv;
      a.core[v] = kUnset;
      a.pile[0][v] = (int32_t)v;
      mn = min(mn, pv);
    }
    mn = __reduce_min_sync(0xffffffffu, mn);
    if (lane == 0 && mn != kUnset) atomicMin(&ctl->kmin[0], mn);
  }
  dev::group_barrier(&ctl->bar, G);

  KcCtx c;
  c.nfin = 0; c.nedge = 0;
  unsigned long long buckets = 0, rounds = 0, phases = 0, empty = 0, subrounds = 0, spills = 0;
  unsigned long long critical = 0, sub0 = 0;  // sum over phases of the busiest CTA's sub-rounds
  uint32_t p = 0, j = 0, k = 0, prev = KC_DONE;
  for (;;) {
    if (tid == 0) {
      // an extraction whose k came from a vertex finished later in the same bucket finds
      // nothing (the recorded minimum is a lower bound): counted apart, like SSSP's R6
      if (prev == KC_EXTRACT) {
        if (__ldcg(&ctl->xfin[j % 3])) ++buckets; else ++empty;
      }
      if (p > 0 && rank == 0) critical += __ldcg(&ctl->maxsub[(p - 1) % 3]);
      const uint32_t qn = __ldcg(&ctl->qcount[p % 3]);
      const uint32_t hn = __ldcg(&ctl->hcount[p % 3]);
      const uint32_t pc = __ldcg(&ctl->pcount[j % 3]);
      const uint32_t km = __ldcg(&ctl->kmin[j % 3]);
      uint32_t mode;
      s.hn = min(hn, a.hubcap);
      if (qn > 0 || hn > 0) { mode = KC_ROUND; s.cnt = qn; }
      else if (pc > 0) { mode = KC_EXTRACT; s.cnt = pc; s.k = km; }
      else mode = KC_DONE;
      s.mode = mode;
      s.kmin = kUnset;
      s.bincnt[0] = 0; s.bincnt[1] = 0;
    }
    __syncthreads();
    const uint32_t mode = s.mode;
    if (mode == KC_DONE) break;
    const uint32_t cnt = s.cnt;
    if (mode == KC_EXTRACT) { ++j; k = s.k; }
    if (rank == 0 && tid == 0) {
      ctl->qcount[(p + 2) % 3] = 0;
      ctl->hcount[(p + 2) % 3] = 0;
      ctl->qclaim[(p + 1) % 3] = 0;  // last used in phase p-2, which every CTA has left
      ctl->maxsub[(p + 2) % 3] = 0;  // read above (rank 0 only), rewritten from phase p+2 on
      if (mode == KC_EXTRACT) {
        ctl->pcount[(j + 1) % 3] = 0; ctl->kmin[(j + 1) % 3] = kUnset; ctl->xfin[(j + 1) % 3] = 0;
      } else {
        ++rounds;
      }
    }
    c.k = k;
    c.q_next = (p & 1) ? a.q[0] : a.q[1];
    c.qcount_next = &ctl->qcount[(p + 1) % 3];
    c.out = sm.bin[0];
    c.outcnt = &s.bincnt[0];
    c.hub_next = (p & 1) ? a.hub[0] : a.hub[1];
    c.hcount_next = &ctl->hcount[(p + 1) % 3];
    c.hubcap = a.hubcap;
    c.pf = a.ld ? a.slots : nullptr;
    c.my_kmin = kUnset;
    uint32_t* kmin_live = &ctl->kmin[j % 3];  // the min for the NEXT extraction

    if (mode == KC_EXTRACT) {
      // dequeue_ready_set: the pile entries whose priority is <= k
      const int32_t* pile_src = (j & 1) ? a.pile[0] : a.pile[1];
      int32_t* pile_live = (j & 1) ? a.pile[1] : a.pile[0];
      uint32_t* pcount_live = &ctl->pcount[j % 3];
      const uint32_t lo = (uint32_t)(((uint64_t)cnt * rank) / G), hi = (uint32_t)(((uint64_t)cnt * (rank + 1)) / G);
      uint32_t nx = 0;
      constexpr int X = 4;  // pile entries per thread per iteration, all loads in flight together
      for (uint32_t i0 = lo; i0 < hi; i0 += X * kKcBlock) {  // warp-uniform trip count
        int32_t v[X];
        uint32_t cc[X], pr[X];
#pragma unroll
        for (int x = 0; x < X; ++x) {
          const uint32_t i = i0 + x * kKcBlock + tid;
          v[x] = i < hi ? pile_src[i] : -1;
        }
#pragma unroll
        for (int x = 0; x < X; ++x) {
          cc[x] = v[x] >= 0 ? ld_cg(a.core + v[x]) : 0u;
          pr[x] = v[x] >= 0 ? ld_cg(a.prio + v[x]) : 0u;
        }
        uint32_t keepm = 0;
#pragma unroll
        for (int x = 0; x < X; ++x) {
          const bool live = v[x] >= 0 && cc[x] == kUnset;  // finished entries are dropped
          // a vertex is finished exactly once (its edges are decrements, not idempotent):
          // the extraction and a concurrent crossing in another CTA's drain race for it
          // (slot path: no drain runs during the extraction — a group barrier follows it)
          bool fin = live && pr[x] <= k;
          if (fin) {
            if (a.ld) {
              a.core[v[x]] = k;
              if (!GI_KC_PFLOCAL) prefetch_l1(a.slots + 8 * (size_t)v[x]);
            } else {
              fin = atomicCAS(a.core + v[x], kUnset, k) == kUnset;
            }
          }
          const bool keep = live && pr[x] > k;
          if (fin) { ++c.nfin; ++nx; }
          if (keep) { c.my_kmin = min(c.my_kmin, pr[x]); keepm |= 1u << x; }
          kc_push(c, fin, v[x]);
        }
        // kept entries -> the next pile with ONE global atomic per CTA per iteration: every
        // CTA appends to the same counter, and per-warp atomics (one per 32 entries)
        // serialised on it (config 2 keeps ~16 M entries per extraction)
        uint32_t mk[X], pre[X], wtot = 0;
#pragma unroll
        for (int x = 0; x < X; ++x) {
          mk[x] = __ballot_sync(0xffffffffu, (keepm >> x) & 1u);
          pre[x] = wtot;
          wtot += __popc(mk[x]);
        }
        if (lane == 0) s.woff[tid >> 5] = wtot;
        __syncthreads();
        if (tid == 0) {
          uint32_t run = 0;
          for (int w = 0; w < kKcBlock / 32; ++w) {
            const uint32_t t = s.woff[w];
            s.woff[w] = run;
            run += t;
          }
          s.pbase = run ? atomicAdd(pcount_live, run) : 0u;
        }
        __syncthreads();
        const uint32_t wb = s.pbase + s.woff[tid >> 5];
        const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
        for (int x = 0; x < X; ++x)
          if ((keepm >> x) & 1u) pile_live[wb + pre[x] + __popc(mk[x] & lt)] = v[x];
        __syncthreads();  // s.woff / s.pbase are rewritten next iteration
      }
      nx = __reduce_add_sync(0xffffffffu, nx);
      if (lane == 0 && nx) atomicAdd(&ctl->xfin[j % 3], nx);
      __syncthreads();
      // slot path: the drains below claim crossings without a CAS, so no CTA may still be
      // extracting (the extraction's own claims are plain stores too)
      if (a.ld) dev::group_barrier(&ctl->bar, G);
    } else {
      // edges.from(frontier).applyUpdatePriority(apply_f). Hubs queued in
      // the previous phase first: every CTA relaxes its 1/G slice of every hub's edges.
      const uint32_t hn = s.hn;
      const HubEnt* hub_in = (p & 1) ? a.hub[1] : a.hub[0];
      for (uint32_t h0 = 0; h0 < hn; h0 += kKcChunk) {
        const uint32_t nh = min((uint32_t)kKcChunk, hn - h0);
        for (uint32_t i = tid; i < nh; i += kKcBlock) {
          const HubEnt he = hub_in[h0 + i];
          const uint64_t lo_e = (uint64_t)he.deg * rank / G, hi_e = (uint64_t)he.deg * (rank + 1) / G;
          sm.beg[i] = he.beg + (long long)lo_e;
          sm.deg[i] = (uint32_t)(hi_e - lo_e);
        }
        __syncthreads();
        kc_relax_entries(a, s, sm, c, nh);
      }
      // then the global frontier in claimed chunks; crossings go to the local bin
      const int32_t* q_in = (p & 1) ? a.q[1] : a.q[0];
      const uint32_t claim = max(32u, min((uint32_t)kKcChunk, cnt / (4 * G)));
      const uint64_t first = (uint64_t)G * claim;
      const bool dyn = first < cnt;
      uint32_t* qclaim = &ctl->qclaim[p % 3];
      uint32_t next = 0;
      if (tid == 0) {
        s.claim = rank * claim;
        if (dyn) next = (uint32_t)first + atomicAdd(qclaim, claim);
      }
      __syncthreads();
      for (;;) {
        const uint32_t base = s.claim;
        if (base >= cnt) break;
        const uint32_t chunk = min(claim, cnt - base);
        if (a.ld) {
          kc_relax_slots<4>(a, c, q_in + base, chunk);
        } else {
          kc_stage_vertices(a, sm, c, q_in + base, chunk);
          kc_relax_entries(a, s, sm, c, chunk);
        }
        if (tid == 0) {
          s.claim = dyn ? next : cnt;
          if (dyn && next < cnt) next = (uint32_t)first + atomicAdd(qclaim, claim);
        }
        __syncthreads();
      }
    }

    // bucket fusion (applied here to k-core's current bucket): drain
    // the CTA-local bin while it stays below T, with CTA barriers only; a bin of >= T
    // vertices goes to the global frontier (the next group-wide round)
    for (uint32_t it = 1;; ++it) {
      const uint32_t nin = min(s.bincnt[(it - 1) % 3], (uint32_t)kKcChunk);
      const int32_t* in = sm.bin[(it - 1) & 1];
      if (nin == 0) break;
      if (nin >= kKcT) {
        for (uint32_t i0 = 0; i0 < nin; i0 += kKcBlock) {
          const uint32_t i = i0 + tid;
          kc_append(i < nin, i < nin ? in[i] : 0, c.q_next, c.qcount_next);
        }
        if (tid == 0) ++spills;
        break;
      }
      if (tid == 0) { s.bincnt[(it + 1) % 3] = 0; ++subrounds; }
      c.out = sm.bin[it & 1];
      c.outcnt = &s.bincnt[it % 3];
      if (a.ld) {
        if (nin * 8 <= (uint32_t)kKcBlock) kc_relax_slots<1>(a, c, in, nin);
        else kc_relax_slots<4>(a, c, in, nin);
      } else {
        kc_stage_vertices(a, sm, c, in, nin);
        kc_relax_entries(a, s, sm, c, nin);  // ends with a barrier
      }
    }

    if (tid == 0 && subrounds != sub0) {
      atomicMax(&ctl->maxsub[p % 3], (uint32_t)(subrounds - sub0));
      sub0 = subrounds;
    }
    // next k: the exact minimum priority of the unfinished vertices (kept entries and
    // every non-crossing decrement), warp min -> smem -> one global atomic per CTA
    const uint32_t km = __reduce_min_sync(0xffffffffu, c.my_kmin);
    if (lane == 0 && km != kUnset) atomicMin(&s.kmin, km);
    __syncthreads();
    if (tid == 0 && s.kmin != kUnset) atomicMin(kmin_live, s.kmin);
    dev::group_barrier(&ctl->bar, G);
    ++p;
    ++phases;
    prev = mode;
  }

  // statistics
  const unsigned nf = __reduce_add_sync(0xffffffffu, (unsigned)c.nfin);
  if (lane == 0 && nf) atomicAdd(&a.stats->vertices, (unsigned long long)nf);
  unsigned long long ned = c.nedge;  // per thread (slot path) or per CTA (thread 0)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ned += __shfl_down_sync(0xffffffffu, ned, o);
  if (lane == 0 && ned) atomicAdd(&a.stats->edges, ned);
  if (tid == 0) {
    if (subrounds) atomicAdd(&a.stats->subrounds, subrounds);
    if (spills) atomicAdd(&a.stats->spills, spills);
    if (rank == 0) {
      a.stats->buckets = buckets; a.stats->rounds = rounds; a.stats->phases = phases + 1; a.stats->empty = empty;
      a.stats->critical = critical;
    }
  }
}

}  // namespace

int kcore_smem_bytes() { return kKcChunk * (int)(sizeof(long long) + sizeof(unsigned long long) + 3 * sizeof(int32_t)); }

cudaError_t kcore_occupancy(int* blocks_per_sm) {
  cudaError_t e = cudaFuncSetAttribute(kcore_persistent, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       kcore_smem_bytes());
  if (e != cudaSuccess) return e;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, kcore_persistent, kKcBlock,
                                                       kcore_smem_bytes());
}

cudaError_t launch_kcore(const KcArgs& a, int grid, cudaStream_t st) {
  cudaError_t e = cudaFuncSetAttribute(kcore_persistent, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       kcore_smem_bytes());
  if (e != cudaSuccess) return e;
  KcArgs args = a;
  void* params[] = {&args};
  return cudaLaunchCooperativeKernel((const void*)kcore_persistent, dim3(grid), dim3(kKcBlock), params,
                                     kcore_smem_bytes(), st);
}

}  // namespace gi

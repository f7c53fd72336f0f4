// gi_kernels.cu — sm_100a kernels for Δ-stepping SSSP with lazy far-bucket updates
// and bucket fusion.
//
// One persistent cooperative kernel per call runs the whole bucket loop on the
// device (no host round-trip per bucket, north_star (d)). The grid is split into
// `ngroups` groups of `group_size` co-resident CTAs; each group runs one query
// at a time (batch = several groups in flight). Within a group the loop is a
// sequence of PHASES separated by a group barrier; a phase is either
//
//   EXTRACT  — kernels (d)+(a): the far pile (the paper's overflow bucket,
//              PAPER.md:796, :1519-1522) is partitioned by recomputed bucket id:
//              entries of bucket b (the min live bucket, maintained as a running
//              lower bound by warp min-reductions + one atomicMin per CTA) are
//              extracted into the current-bucket bin, stale entries (bucket < b)
//              are dropped, the rest are compacted into the other far buffer.
//   ROUND    — a group-wide relax pass over the global frontier (spilled bins or,
//              without fusion, every round of the bucket).
//
// and every phase then drains its CTA-local current-bucket bin in shared memory
// while the bin stays below the threshold T — bucket fusion (kernel (c),
// Fig. alg:eager_delta_stepping_merge).
//
// Edge relaxation (kernel (b)), Dist[dst] = min(Dist[dst], Dist[src]+w)
// (PAPER.md:422), is an atomicMin on uint32 and is degree-binned:
//   * deg <= 8: one OCTET (8 lanes) per vertex, lane k relaxes entry k of the
//     vertex's 64-byte ELL slot (one coalesced 64 B load, one atomic per lane),
//     several entries in flight per thread;
//   * deg > 8: the vertex joins the CTA's high-degree list, whose concatenated
//     edges are split evenly over all threads of the CTA (prefix sum + search),
//     coalesced 8-byte {col, w} loads, 4 per thread per iteration.
// Lowerings into a FUTURE bucket are appended once per vertex to the far pile
// (dedup bit = reduceBucketUpdates; "a single bucket update
// per vertex"), staged in shared memory and flushed at the phase
// end, off the bucket's critical chain; lowerings into the CURRENT bucket go to
// the CTA ring as (vertex, distance) pairs (eager) and the
// vertex's slot is prefetched into L2 for the next sub-round.
#include "gi_internal.h"

#include <cooperative_groups.h>

namespace cg = cooperative_groups;

namespace gi {
namespace {

enum : uint32_t { MODE_ROUND = 0, MODE_EXTRACT = 1, MODE_DONE = 2, MODE_NONE = 3 };

#ifdef GI_TRACE
// Debug builds only: cycles between trace points, accumulated by CTA 0 / thread 0 in
// shared memory (so that tracing adds ~no latency) and flushed at kernel exit.
__device__ unsigned long long g_trace[32];
__shared__ unsigned long long s_trace[32];
__shared__ long long s_trace_last;
#define TRACE(k)                                                   \
  do {                                                             \
    if (blockIdx.x == 0 && threadIdx.x == 0) {                     \
      long long t_ = clock64();                                    \
      s_trace[k] += (unsigned long long)(t_ - s_trace_last);       \
      s_trace[16 + (k)] += 1;                                      \
      s_trace_last = t_;                                           \
    }                                                              \
  } while (0)
#define TRACE_INIT()                                                          \
  do {                                                                        \
    if (threadIdx.x < 32) s_trace[threadIdx.x] = 0;                           \
    if (threadIdx.x == 0) s_trace_last = clock64();                           \
    __syncthreads();                                                          \
  } while (0)
#define TRACE_FLUSH()                                                         \
  do {                                                                        \
    if (blockIdx.x == 0 && threadIdx.x < 32) atomicAdd(&g_trace[threadIdx.x], s_trace[threadIdx.x]); \
  } while (0)
#else
#define TRACE(k) do {} while (0)
#define TRACE_INIT() do {} while (0)
#define TRACE_FLUSH() do {} while (0)
#endif

__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void fence_acq_rel() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

// dist[] is written by atomics inside this kernel: read it coherently from L2,
// never through the non-coherent/L1 path (SURVEY §7 hard part 1).
__device__ __forceinline__ uint32_t ld_dist(const uint32_t* p) { return __ldcg(p); }

__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

__device__ __forceinline__ uint32_t fdiv(uint32_t x, const FastDiv& f) {
  uint32_t t = __umulhi(x, f.mul);
  return (t + ((x - t) >> f.s1)) >> f.s2;
}

// Barrier over the G CTAs of one group (all co-resident: cooperative launch).
// One word: arrivals in the low 16 bits, generation in the high 16; the last
// arriver resets the count and bumps the generation with a single atomic.
__device__ __forceinline__ void group_barrier(Ctl* ctl, uint32_t G) {
  __syncthreads();
  if (threadIdx.x == 0) {
    fence_acq_rel();  // publish this CTA's writes (cumulative over the bar.sync above)
    const uint32_t old = atomicAdd(&ctl->bar, 1u);
    if ((old & 0xFFFFu) == G - 1) {
      atomicAdd(&ctl->bar, 0x10000u - G);
    } else {
      const uint32_t gen = old >> 16;
      while ((ld_relaxed(&ctl->bar) >> 16) == gen) {
      }
    }
    fence_acq_rel();
  }
  __syncthreads();
}

template <typename T>
__device__ __forceinline__ T warp_sum(T x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

struct BigEnt {
  int64_t beg;
  uint32_t deg;
  uint32_t du;
};

struct Shared {
  uint32_t cnt3[3];         // current-bucket bin fills, rotating by sub-round
  uint32_t bigtail;         // fill of the high-degree list
  uint32_t farcnt;          // fill of the far staging buffer
  uint32_t mode, b, cnt, hn;
  uint32_t fmin;
  unsigned long long total; // edges of the high-degree list (exclusive-scan total)
  unsigned long long red[kBlock / 32];
  int32_t farstage[kFarStage];
};

// Everything a relaxation needs, held in registers for one phase.
struct Ctx {
  uint32_t* dist;
  const uint2* slots;
  const uint2* edges;
  FastDiv div;
  uint32_t b;              // current bucket
  uint32_t* qbits_next;    // dedup bits of the global frontier being produced
  int32_t* q_next;
  uint32_t* qcount_next;
  uint32_t* farbits;       // far pile dedup bits
  int32_t* far_live;       // far buffer receiving appends this phase
  uint32_t* fcount_live;
  uint32_t* ovfbits;
  uint32_t* ovf_cand;
  uint2* out;              // CTA-local current-bucket bin receiving pushes (shared memory)
  uint32_t* outcnt;        // its fill counter (shared memory)
  BigEnt* big;             // CTA-local high-degree list (shared memory)
  unsigned long long* pre; // exclusive prefix of its degrees (shared memory)
  HubEnt* hub_next;        // group hub list receiving appends this phase
  uint32_t* hcount_next;
  uint32_t hub_min, hubcap;
  Shared* s;
  uint32_t my_fmin;        // thread-local min far bucket (reduced at phase end)
  bool pre_read;
};

// Append v to the global frontier once per phase (dedup bit), warp-aggregated.
__device__ __forceinline__ void push_global(Ctx& c, int32_t v) {
  const uint32_t bit = 1u << (v & 31);
  const uint32_t old = atomicOr(&c.qbits_next[v >> 5], bit);
  if (!(old & bit)) {
    prefetch_l2(c.slots + 8 * (size_t)v);
    cg::coalesced_group g = cg::coalesced_threads();
    uint32_t base = 0;
    if (g.thread_rank() == 0) base = atomicAdd(c.qcount_next, g.size());
    base = g.shfl(base, 0);
    c.q_next[base + g.thread_rank()] = v;
  }
}

// Current-bucket push: CTA-local ring (fusion) or the global frontier.
template <bool FUSED>
__device__ __forceinline__ void push_cur(Ctx& c, int32_t v, uint32_t d) {
  if constexpr (FUSED) {
    prefetch_l2(c.slots + 8 * (size_t)v);
    cg::coalesced_group g = cg::coalesced_threads();
    uint32_t base = 0;
    if (g.thread_rank() == 0) base = atomicAdd(c.outcnt, g.size());
    base = g.shfl(base, 0);
    const uint32_t pos = base + g.thread_rank();
    if (pos < (uint32_t)kBinCap) c.out[pos] = make_uint2((uint32_t)v, d);
    else push_global(c, v);  // bin full: the vertex goes to the next group-wide round
  } else {
    push_global(c, v);
  }
}

// Far-pile append, deduplicated: one live entry per vertex.
__device__ __forceinline__ void push_far_global(Ctx& c, int32_t v) {
  const uint32_t bit = 1u << (v & 31);
  const uint32_t old = atomicOr(&c.farbits[v >> 5], bit);
  if (!(old & bit)) {
    cg::coalesced_group g = cg::coalesced_threads();
    uint32_t base = 0;
    if (g.thread_rank() == 0) base = atomicAdd(c.fcount_live, g.size());
    base = g.shfl(base, 0);
    c.far_live[base + g.thread_rank()] = v;
  }
}

// Future-bucket push: lazy (bucket recomputed from dist at extraction), staged in
// shared memory; the dedup + append happens at the phase end.
__device__ __forceinline__ void push_far(Ctx& c, int32_t v, uint32_t bk) {
  c.my_fmin = min(c.my_fmin, bk);
  cg::coalesced_group g = cg::coalesced_threads();
  uint32_t base = 0;
  if (g.thread_rank() == 0) base = atomicAdd(&c.s->farcnt, g.size());
  base = g.shfl(base, 0);
  const uint32_t pos = base + g.thread_rank();
  if (pos < (uint32_t)kFarStage) c.s->farstage[pos] = v;
  else push_far_global(c, v);
}

__device__ __noinline__ void mark_overflow(uint32_t* ovfbits, uint32_t* ovf_cand, uint32_t v) {
  atomicOr(&ovfbits[v >> 5], 1u << (v & 31));
  atomicOr(ovf_cand, 1u);
}

// Relax K edges per thread (u -> e[k].x, weight e[k].y, from du[k]); lanes with
// bit k of `valid` clear do nothing. Every load and atomic of the batch is issued
// before any result is consumed (memory-level parallelism on the critical chain).
// Must be called by all 32 lanes of the warp (the appends are warp-aggregated).
template <bool FUSED, int K>
__device__ __forceinline__ void relax_batch(Ctx& c, const uint2 (&e)[K], const uint32_t (&du)[K],
                                            uint32_t valid) {
  uint32_t nd[K], old[K];
  uint32_t ok = 0;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    nd[k] = du[k] + e[k].y;
    if (valid & (1u << k)) {
      if (nd[k] < du[k] || nd[k] == kInf) mark_overflow(c.ovfbits, c.ovf_cand, e[k].x);
      else ok |= 1u << k;
    }
  }
  if (c.pre_read) {
    uint32_t cur[K];
#pragma unroll
    for (int k = 0; k < K; ++k) cur[k] = (ok & (1u << k)) ? ld_dist(c.dist + e[k].x) : 0u;
#pragma unroll
    for (int k = 0; k < K; ++k)
      if (!(nd[k] < cur[k])) ok &= ~(1u << k);
  }
#pragma unroll
  for (int k = 0; k < K; ++k) old[k] = (ok & (1u << k)) ? atomicMin(c.dist + e[k].x, nd[k]) : 0u;
  // classify the successful lowerings: current bucket (bin) or a future one (far pile)
  uint32_t curm = 0, farm = 0;
  uint32_t bk[K];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    bk[k] = fdiv(nd[k], c.div);
    if ((ok & (1u << k)) && nd[k] < old[k]) {
      if (bk[k] == c.b) curm |= 1u << k;
      else farm |= 1u << k;  // bk > b: nd >= du >= bΔ
    }
  }
  // warp-aggregated appends: one ballot per item slot, one shared atomic per warp
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t lt = (1u << lane) - 1u;
  if constexpr (FUSED) {
    uint32_t mk[K], pre[K], tot = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      mk[k] = __ballot_sync(0xffffffffu, (curm >> k) & 1u);
      pre[k] = tot;
      tot += __popc(mk[k]);
    }
    if (tot) {
      uint32_t base = 0;
      if (lane == 0) base = atomicAdd(c.outcnt, tot);
      base = __shfl_sync(0xffffffffu, base, 0);
#pragma unroll
      for (int k = 0; k < K; ++k) {
        if ((curm >> k) & 1u) {
          const uint32_t pos = base + pre[k] + __popc(mk[k] & lt);
          prefetch_l2(c.slots + 8 * (size_t)e[k].x);
          if (pos < (uint32_t)kBinCap) c.out[pos] = make_uint2(e[k].x, nd[k]);
          else push_global(c, (int32_t)e[k].x);  // bin full: next group-wide round
        }
      }
    }
  } else {
#pragma unroll
    for (int k = 0; k < K; ++k)
      if ((curm >> k) & 1u) push_global(c, (int32_t)e[k].x);
  }
  {
    uint32_t mk[K], pre[K], tot = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      mk[k] = __ballot_sync(0xffffffffu, (farm >> k) & 1u);
      pre[k] = tot;
      tot += __popc(mk[k]);
    }
    if (tot) {
      uint32_t base = 0;
      if (lane == 0) base = atomicAdd(&c.s->farcnt, tot);
      base = __shfl_sync(0xffffffffu, base, 0);
#pragma unroll
      for (int k = 0; k < K; ++k) {
        if ((farm >> k) & 1u) {
          c.my_fmin = min(c.my_fmin, bk[k]);
          const uint32_t pos = base + pre[k] + __popc(mk[k] & lt);
          if (pos < (uint32_t)kFarStage) c.s->farstage[pos] = (int32_t)e[k].x;
          else push_far_global(c, (int32_t)e[k].x);
        }
      }
    }
  }
}

// Stage A — vertices with deg <= 8: ITEMS (entry, slot index), 8 per frontier entry;
// the 8 lanes of an octet share one entry and lane k relaxes entry k of its 64-byte
// ELL slot (one coalesced 64 B load per octet). Each thread holds U items in flight.
// Vertices with deg > 8 are appended to the CTA's high-degree list for stage B.
template <bool FUSED, int U>
__device__ __forceinline__ void stage_small(Ctx& c, const uint2* in, uint32_t nin, bool check_stale,
                                            uint32_t& nv, uint32_t& ne) {
  const uint32_t nitems = nin * 8;
  const uint32_t sub = threadIdx.x & 7;
  for (uint32_t base = 0; base < nitems; base += kBlock * U) {
    uint2 e[U];
    uint32_t du[U], v[U];
    uint32_t have = 0;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t item = base + u * kBlock + threadIdx.x;
      e[u] = make_uint2(kColEmpty, 0);
      du[u] = 0; v[u] = 0;
      if (item < nitems) {
        const uint2 en = in[item >> 3];
        v[u] = en.x; du[u] = en.y;
        e[u] = __ldg(c.slots + 8 * (size_t)en.x + sub);
        have |= 1u << u;
      }
    }
    if (check_stale) {  // a newer entry for v exists; octet-uniform decision
      uint32_t cur[U];
#pragma unroll
      for (int u = 0; u < U; ++u) cur[u] = (have & (1u << u)) ? ld_dist(c.dist + v[u]) : kInf;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t sb = __ballot_sync(0xffffffffu, cur[u] < du[u]);
        if ((sb >> (threadIdx.x & 24)) & 0xFFu) have &= ~(1u << u);
      }
    }
    TRACE(2);
    uint32_t valid = 0;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (!(have & (1u << u))) continue;
      if (e[u].x == kColBig) {  // octet-uniform: every entry of a big slot is kColBig
        const uint32_t om = 0xFFu << (threadIdx.x & 24);
        const uint32_t lo = __shfl_sync(om, e[u].y, 1, 8);
        const uint32_t hi = __shfl_sync(om, e[u].y, 2, 8);
        if (sub == 0) {
          ++nv;
          const uint32_t deg = e[u].y;
          uint32_t hp = 0xFFFFFFFFu;
          if (deg >= c.hub_min) {  // hub: split over the whole group in the next phase
            hp = atomicAdd(c.hcount_next, 1u);
            if (hp < c.hubcap) {
              HubEnt he;
              he.beg = (int64_t)(((uint64_t)hi << 32) | lo);
              he.deg = deg;
              he.du = du[u];
              c.hub_next[hp] = he;
            }
          }
          const uint32_t pos = hp < c.hubcap ? 0xFFFFFFFFu : atomicAdd(&c.s->bigtail, 1u);
          if (hp < c.hubcap) {
            // queued on the group hub list
          } else if (pos < (uint32_t)kBigCap) {
            BigEnt be;
            be.beg = (int64_t)(((uint64_t)hi << 32) | lo);
            be.deg = e[u].y;
            be.du = du[u];
            c.big[pos] = be;
          } else {
            push_global(c, (int32_t)v[u]);  // list full: the next group-wide round takes it
          }
        }
      } else {
        nv += sub == 0;
        if (e[u].x != kColEmpty) { valid |= 1u << u; ++ne; }
      }
    }
    relax_batch<FUSED, U>(c, e, du, valid);
    TRACE(3);
  }
}

// Stage B — vertices with deg > 8: their edges are concatenated (exclusive prefix of
// the degrees) and split evenly over all threads of the CTA, 4 edges per thread per
// iteration; an edge finds its vertex by binary search in the prefix array.
template <bool FUSED>
__device__ __forceinline__ void stage_big(Ctx& c, Shared& s, uint32_t nb, uint32_t& ne) {
  constexpr int PER = kBigCap / kBlock;
  unsigned long long loc[PER];
  unsigned long long sum = 0;
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    const uint32_t i = threadIdx.x * PER + k;
    loc[k] = sum;
    sum += i < nb ? c.big[i].deg : 0u;
  }
  // block exclusive scan of the per-thread sums
  unsigned long long incl = sum;
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= (uint32_t)o) incl += t;
  }
  if (lane == 31) s.red[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    unsigned long long w = lane < kBlock / 32 ? s.red[lane] : 0ull;
    unsigned long long wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long t = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= (uint32_t)o) wi += t;
    }
    if (lane < kBlock / 32) s.red[lane] = wi - w;  // exclusive warp offsets
    if (lane == kBlock / 32 - 1) s.total = wi;
  }
  __syncthreads();
  const unsigned long long off = s.red[warp] + incl - sum;
#pragma unroll
  for (int k = 0; k < PER; ++k) {
    const uint32_t i = threadIdx.x * PER + k;
    if (i < nb) c.pre[i] = off + loc[k];
  }
  __syncthreads();
  const unsigned long long total = s.total;
  if (threadIdx.x == 0) ne += (uint32_t)total;
  for (unsigned long long k0 = 0; k0 < total; k0 += 4ull * kBlock) {
    uint2 e[4];
    uint32_t du[4];
    uint32_t valid = 0;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const unsigned long long k = k0 + (unsigned long long)u * kBlock + threadIdx.x;
      e[u] = make_uint2(0, 0);
      du[u] = 0;
      if (k < total) {
        uint32_t lo = 0, hi = nb;  // last i with pre[i] <= k
        while (hi - lo > 1) {
          const uint32_t mid = (lo + hi) >> 1;
          if (c.pre[mid] <= k) lo = mid; else hi = mid;
        }
        const BigEnt be = c.big[lo];
        e[u] = __ldg(c.edges + be.beg + (int64_t)(k - c.pre[lo]));
        du[u] = be.du;
        valid |= 1u << u;
      }
    }
    relax_batch<FUSED, 4>(c, e, du, valid);
  }
}

// Relax every entry of a CTA-local bin (stage A, then stage B when high-degree
// vertices were found). Starts after and ends with a CTA barrier.
template <bool FUSED>
__device__ __forceinline__ void process_bin(Ctx& c, Shared& s, const uint2* in, uint32_t nin,
                                            bool check_stale, uint32_t& nv, uint32_t& ne) {
  if (nin * 8 <= (uint32_t)kBlock) stage_small<FUSED, 1>(c, in, nin, check_stale, nv, ne);
  else stage_small<FUSED, 4>(c, in, nin, check_stale, nv, ne);
  __syncthreads();
  TRACE(4);
  const uint32_t nb = min(s.bigtail, (uint32_t)kBigCap);
  if (nb) {
    __syncthreads();  // everyone has read bigtail
    if (threadIdx.x == 0) s.bigtail = 0;
    stage_big<FUSED>(c, s, nb, ne);
    __syncthreads();
  }
}

template <typename T>
__device__ __forceinline__ T block_sum(T x, Shared& s) {
  x = warp_sum(x);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) s.red[threadIdx.x >> 5] = (unsigned long long)x;
  __syncthreads();
  T t = 0;
  if (threadIdx.x < 32) {
    t = threadIdx.x < (kBlock / 32) ? (T)s.red[threadIdx.x] : (T)0;
    t = warp_sum(t);
  }
  return t;  // valid in thread 0
}

template <bool FUSED>
__global__ void __launch_bounds__(kBlock, 1) sssp_persistent(KArgs a) {
  extern __shared__ uint2 s_dyn[];  // bins [2][kBinCap] uint2, high-degree list [kBigCap], its prefix [kBigCap]
  __shared__ Shared s;
  const uint32_t G = (uint32_t)a.group_size;
  const uint32_t gid = blockIdx.x / G;
  const uint32_t rank = blockIdx.x % G;
  const uint32_t tid = threadIdx.x;
  if ((int32_t)gid >= a.ngroups) return;
  const GroupWs ws = a.groups[gid];
  Ctl* ctl = ws.ctl;
  const int64_t n = a.n;
  const uint32_t T = a.T;
  TRACE_INIT();

  for (int32_t si = (int32_t)gid; si < a.nsrc; si += a.ngroups) {
    uint32_t* dist = a.dist + (size_t)si * (size_t)n;
    const int32_t src = a.srcs[si];

    // ---- init: Dist = {inf}, Dist[src] = 0; far pile = {src} ----
    {
      int64_t done = 0;
      if ((reinterpret_cast<uintptr_t>(dist) & 15) == 0) {
        const int64_t n4 = n >> 2;
        uint4* d4 = reinterpret_cast<uint4*>(dist);
        for (int64_t i = (int64_t)rank * kBlock + tid; i < n4; i += (int64_t)G * kBlock) {
          uint4 val = make_uint4(kInf, kInf, kInf, kInf);
          if ((src >> 2) == i) {
            const int k = src & 3;
            val.x = k == 0 ? 0u : kInf; val.y = k == 1 ? 0u : kInf;
            val.z = k == 2 ? 0u : kInf; val.w = k == 3 ? 0u : kInf;
          }
          d4[i] = val;
        }
        done = n4 * 4;
      }
      for (int64_t i = done + (int64_t)rank * kBlock + tid; i < n; i += (int64_t)G * kBlock)
        dist[i] = (i == src) ? 0u : kInf;
    }
    if (rank == 0 && tid == 0) {
      for (int k = 0; k < 3; ++k) {
        ctl->qcount[k] = 0; ctl->fcount[k] = 0; ctl->fmin[k] = kInf; ctl->xlive[k] = 0; ctl->maxsub[k] = 0;
        ctl->hcount[k] = 0;
      }
      ctl->fcount[0] = 1; ctl->fmin[0] = 0; ctl->ovf_cand = 0;
      ws.far[0][0] = src;
      atomicOr(&ws.farbits[src >> 5], 1u << (src & 31));
    }
    group_barrier(ctl, G);

    Ctx c;
    c.dist = dist; c.slots = a.slots; c.edges = a.edges; c.div = a.div;
    c.farbits = ws.farbits; c.ovfbits = ws.ovfbits; c.ovf_cand = &ctl->ovf_cand;
    c.big = reinterpret_cast<BigEnt*>(s_dyn + 2 * kBinCap);
    c.pre = reinterpret_cast<unsigned long long*>(c.big + kBigCap);
    c.s = &s;
    c.pre_read = a.pre_read != 0;
    c.hub_min = a.hub_min;
    c.hubcap = a.hubcap;

    uint32_t nv = 0, ne = 0;                       // per thread (flushed per phase)
    unsigned long long tnv = 0, tne = 0;           // per thread, 64-bit totals
    unsigned long long subrounds = 0, spills = 0, scanned = 0;  // per CTA (thread 0)
    unsigned long long phases = 0, rounds = 0, buckets = 0, empty = 0, critical = 0;  // rank 0, thread 0
    unsigned long long sub_at_phase_start = 0;
    uint32_t p = 0, j = 0, b = 0, prev = MODE_NONE;

    for (;;) {
      // ---- decide (identically in every CTA, from counters final at the barrier) ----
      if (tid == 0) {
        // L2-coherent loads, all four in flight at once (ordered after the barrier's fence)
        const uint32_t xl = __ldcg(&ctl->xlive[j % 3]);
        const uint32_t qn = __ldcg(&ctl->qcount[p % 3]);
        const uint32_t hn = __ldcg(&ctl->hcount[p % 3]);
        const uint32_t fc = __ldcg(&ctl->fcount[j % 3]);
        const uint32_t fm = __ldcg(&ctl->fmin[j % 3]);
        if (p > 0 && rank == 0) critical += __ldcg(&ctl->maxsub[(p - 1) % 3]);
        if (prev == MODE_EXTRACT) {
          if (xl) { ++buckets; if (FUSED) ++rounds; } else { ++empty; }
        }
        uint32_t mode;
        s.hn = min(hn, a.hubcap);
        if (qn > 0 || hn > 0) { mode = MODE_ROUND; s.cnt = qn; }
        else if (fc > 0) { mode = MODE_EXTRACT; s.cnt = fc; s.b = fm; }
        else mode = MODE_DONE;
        s.mode = mode;
        s.cnt3[0] = 0;
        s.cnt3[1] = 0;
        s.bigtail = 0;
        s.farcnt = 0;
        s.fmin = kInf;
      }
      __syncthreads();
      TRACE(5);
      const uint32_t mode = s.mode;
      if (mode == MODE_DONE) break;
      const uint32_t cnt = s.cnt;
      if (mode == MODE_EXTRACT) { ++j; b = s.b; }
      if (rank == 0 && tid == 0) {
        ctl->qcount[(p + 2) % 3] = 0;
        ctl->maxsub[(p + 2) % 3] = 0;
        ctl->hcount[(p + 2) % 3] = 0;
        if (mode == MODE_EXTRACT) {
          ctl->fcount[(j + 1) % 3] = 0; ctl->fmin[(j + 1) % 3] = kInf; ctl->xlive[(j + 1) % 3] = 0;
        }
        if (mode == MODE_ROUND) ++rounds;
      }
      c.b = b;
      c.qbits_next = (p & 1) ? ws.qbits[0] : ws.qbits[1];
      c.q_next = (p & 1) ? ws.q[0] : ws.q[1];
      c.qcount_next = &ctl->qcount[(p + 1) % 3];
      c.hub_next = (p & 1) ? ws.hub[0] : ws.hub[1];
      c.hcount_next = &ctl->hcount[(p + 1) % 3];
      c.far_live = (j & 1) ? ws.far[1] : ws.far[0];
      c.fcount_live = &ctl->fcount[j % 3];
      c.out = s_dyn;  // the first stage fills bin 0 (counter cnt3[0])
      c.outcnt = &s.cnt3[0];
      c.my_fmin = kInf;

      const uint32_t lo = (uint32_t)(((uint64_t)cnt * rank) / G);
      const uint32_t hi = (uint32_t)(((uint64_t)cnt * (rank + 1)) / G);

      if (mode == MODE_EXTRACT) {
        // (d)+(a): partition the far pile by recomputed bucket
        const int32_t* far_src = (j & 1) ? ws.far[0] : ws.far[1];
        uint32_t nlive = 0;
        for (uint32_t i = lo + tid; i < hi; i += kBlock) {
          const int32_t v = far_src[i];
          const uint32_t d = ld_dist(dist + v);
          const uint32_t bk = fdiv(d, c.div);
          if (bk <= b) {
            atomicAnd(&ws.farbits[v >> 5], ~(1u << (v & 31)));
            if (bk == b) { ++nlive; push_cur<FUSED>(c, v, d); }  // else: stale (already settled)
          } else {
            c.my_fmin = min(c.my_fmin, bk);
            cg::coalesced_group g = cg::coalesced_threads();
            uint32_t base = 0;
            if (g.thread_rank() == 0) base = atomicAdd(c.fcount_live, g.size());
            base = g.shfl(base, 0);
            c.far_live[base + g.thread_rank()] = v;
          }
        }
        TRACE(6);
        const uint32_t tl = block_sum(nlive, s);  // ends with a barrier: ring fill is final
        if (tid == 0) {
          if (tl) atomicAdd(&ctl->xlive[j % 3], tl);
          scanned += hi - lo;
        }
      } else {
        // hubs queued in the previous phase: every CTA relaxes its 1/G slice of every
        // hub's edges (stage B over the slices), so a hub costs ~deg/G per CTA
        const uint32_t hn = s.hn;
        const HubEnt* hub_in = (p & 1) ? ws.hub[1] : ws.hub[0];
        for (uint32_t h0 = 0; h0 < hn; h0 += kBigCap) {
          const uint32_t nh = min((uint32_t)kBigCap, hn - h0);
          for (uint32_t i = tid; i < nh; i += kBlock) {
            const HubEnt he = hub_in[h0 + i];
            const uint64_t lo_e = (uint64_t)he.deg * rank / G, hi_e = (uint64_t)he.deg * (rank + 1) / G;
            BigEnt be;
            be.beg = he.beg + (int64_t)lo_e;
            be.deg = (uint32_t)(hi_e - lo_e);
            be.du = he.du;
            c.big[i] = be;
          }
          __syncthreads();
          stage_big<FUSED>(c, s, nh, ne);
          __syncthreads();
        }
        // ROUND: relax the group's global frontier, one slice per CTA, staged through
        // bin 1 in chunks (pushes go to bin 0, which the drain below consumes)
        const int32_t* q_in = (p & 1) ? ws.q[1] : ws.q[0];
        uint32_t* qbits_in = (p & 1) ? ws.qbits[1] : ws.qbits[0];
        uint2* stage = s_dyn + kBinCap;
        for (uint32_t base = lo; base < hi; base += kBinCap) {
          const uint32_t chunk = min((uint32_t)kBinCap, hi - base);
          for (uint32_t i = tid; i < chunk; i += kBlock) {
            const int32_t v = q_in[base + i];
            atomicAnd(&qbits_in[v >> 5], ~(1u << (v & 31)));
            stage[i] = make_uint2((uint32_t)v, ld_dist(dist + v));
          }
          __syncthreads();
          process_bin<FUSED>(c, s, stage, chunk, false, nv, ne);
        }
        __syncthreads();
      }

      if constexpr (FUSED) {
        // (c) bucket fusion: drain the CTA-local bin while it stays below T
        // (PAPER.md:537-550); a bin of size >= T goes to the global frontier
        // ("copied over to the global bucket"). Sub-round k reads
        // bin (k-1)%2 (fill cnt3[(k-1)%3]) and pushes into bin k%2 (fill cnt3[k%3]);
        // cnt3[(k+1)%3] was last read at the top of sub-round k-1 and is reset here,
        // so one barrier per sub-round suffices.
        for (uint32_t k = 1;; ++k) {
          // a barrier has completed: pushes of the previous sub-round are visible
          TRACE(0);
          const uint2* in = s_dyn + ((k - 1) & 1) * kBinCap;
          const uint32_t nin = min(s.cnt3[(k - 1) % 3], (uint32_t)kBinCap);
          if (nin == 0) break;
          if (nin >= T) {
            for (uint32_t i = tid; i < nin; i += kBlock) push_global(c, (int32_t)in[i].x);
            if (tid == 0) ++spills;
            break;
          }
          if (tid == 0) { s.cnt3[(k + 1) % 3] = 0; ++subrounds; }
          c.out = s_dyn + (k & 1) * kBinCap;
          c.outcnt = &s.cnt3[k % 3];
          process_bin<FUSED>(c, s, in, nin, true, nv, ne);
        }
      }

      // flush staged far-pile pushes (dedup + append), then the next-bucket lower
      // bound: warp min + one smem atomic per warp + one global atomic per CTA
      __syncthreads();
      TRACE(7);
      {
        const uint32_t nf = min(s.farcnt, (uint32_t)kFarStage);
        for (uint32_t i = tid; i < nf; i += kBlock) push_far_global(c, s.farstage[i]);
        uint32_t fm = __reduce_min_sync(0xffffffffu, c.my_fmin);
        if ((tid & 31) == 0 && fm != kInf) atomicMin(&s.fmin, fm);
        __syncthreads();
        if (tid == 0 && s.fmin != kInf) atomicMin(&ctl->fmin[j % 3], s.fmin);
        if (FUSED && tid == 0 && subrounds != sub_at_phase_start) {
          atomicMax(&ctl->maxsub[p % 3], (uint32_t)(subrounds - sub_at_phase_start));
          sub_at_phase_start = subrounds;
        }
      }
      tnv += nv; tne += ne; nv = 0; ne = 0;
      TRACE(8);
      group_barrier(ctl, G);
      TRACE(9);
      ++p;
      ++phases;
      prev = mode;
    }

    // ---- overflow resolution: a vertex with an overflowing candidate that never
    // received a representable distance has δ >= UINT32_MAX ----
    if (ld_relaxed(&ctl->ovf_cand)) {
      uint32_t bad = 0;
      for (uint32_t wi = rank * kBlock + tid; wi < a.nwords; wi += G * kBlock) {
        uint32_t bits = ws.ovfbits[wi];
        if (bits) {
          ws.ovfbits[wi] = 0;
          while (bits) {
            const int k = __ffs(bits) - 1;
            bits &= bits - 1;
            const int64_t v = (int64_t)wi * 32 + k;
            if (v < n && ld_dist(dist + v) == kInf) bad = 1;
          }
        }
      }
      if (__syncthreads_or(bad) && tid == 0) atomicOr(&a.qstats[si].overflow, 1u);
    }

    // ---- statistics ----
    const unsigned long long tv = block_sum(tnv, s);
    const unsigned long long te = block_sum(tne, s);
    if (tid == 0) {
      QStats* q = &a.qstats[si];
      atomicAdd(&q->vertices, tv);
      atomicAdd(&q->edges, te);
      if (subrounds) atomicAdd(&q->subrounds, subrounds);
      if (spills) atomicAdd(&q->spills, spills);
      if (scanned) atomicAdd(&q->far_scanned, scanned);
      if (rank == 0) {
        q->buckets = buckets; q->rounds = rounds; q->phases = phases + 2;  // + init and final barriers
        q->empty_extr = empty;
        q->critical_subrounds = critical;
      }
    }
    group_barrier(ctl, G);  // the next query re-initialises ctl
  }
  TRACE_FLUSH();
}

__global__ void interleave_kernel(const int32_t* __restrict__ cols, const uint32_t* __restrict__ w,
                                  uint2* __restrict__ edges, int64_t count, int64_t n, uint32_t* bad) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t c = cols[i];
    if (c < 0 || c >= n) atomicOr(bad, 1u);
    edges[i] = make_uint2((uint32_t)c, w[i]);
  }
}

// ELL slot per vertex (8 x {col, w}, 64 B): deg <= 8 -> edges inline, unused entries
// kColEmpty; deg > 8 -> every entry {kColBig, payload} with payloads deg, beg_lo,
// beg_hi in entries 0..2 (the CSR edges hold the adjacency).
__global__ void build_slots_kernel(const int64_t* __restrict__ off, const uint2* __restrict__ edges,
                                   uint2* __restrict__ slots, int64_t n) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t beg = off[v], deg = off[v + 1] - beg;
    uint2 e[8];
    if (deg <= kSlotEdges) {
#pragma unroll
      for (int k = 0; k < 8; ++k) e[k] = k < deg ? edges[beg + k] : make_uint2(kColEmpty, 0);
    } else {
      e[0] = make_uint2(kColBig, (uint32_t)deg);
      e[1] = make_uint2(kColBig, (uint32_t)(uint64_t)beg);
      e[2] = make_uint2(kColBig, (uint32_t)((uint64_t)beg >> 32));
#pragma unroll
      for (int k = 3; k < 8; ++k) e[k] = make_uint2(kColBig, 0);
    }
    uint4* sp = reinterpret_cast<uint4*>(slots + 8 * v);
    sp[0] = make_uint4(e[0].x, e[0].y, e[1].x, e[1].y);
    sp[1] = make_uint4(e[2].x, e[2].y, e[3].x, e[3].y);
    sp[2] = make_uint4(e[4].x, e[4].y, e[5].x, e[5].y);
    sp[3] = make_uint4(e[6].x, e[6].y, e[7].x, e[7].y);
  }
}

__global__ void max_degree_kernel(const int64_t* __restrict__ off, int64_t n, uint32_t* out) {
  uint32_t mx = 0;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t d = off[v + 1] - off[v];
    mx = max(mx, (uint32_t)min(d, (int64_t)0xFFFFFFFF));
  }
  mx = __reduce_max_sync(0xffffffffu, mx);
  if ((threadIdx.x & 31) == 0) atomicMax(out, mx);
}

__global__ void validate_offsets_kernel(const int64_t* __restrict__ off, int64_t n, int64_t m,
                                        uint32_t* bad) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (off[i] > off[i + 1] || off[i + 1] - off[i] > 0xFFFFFFF0ll) atomicOr(bad, 1u);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && (off[0] != 0 || off[n] != m)) atomicOr(bad, 1u);
}

}  // namespace

int smem_bytes() {
  return 2 * kBinCap * (int)sizeof(uint2) + kBigCap * ((int)sizeof(BigEnt) + (int)sizeof(unsigned long long));
}

#ifdef GI_TRACE
extern "C" int gi_debug_trace(unsigned long long* out, int reset) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out, g_trace, sizeof(unsigned long long) * 32);
  if (reset) {
    unsigned long long z[32] = {0};
    cudaMemcpyToSymbol(g_trace, z, sizeof(z));
  }
  return 0;
}
#endif

static bool g_attr_set = false;

static cudaError_t set_attrs() {
  if (g_attr_set) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(sssp_persistent<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       smem_bytes());
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(sssp_persistent<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           smem_bytes());
  if (e == cudaSuccess) g_attr_set = true;
  return e;
}

cudaError_t query_occupancy(bool fused, int* blocks_per_sm) {
  cudaError_t e = set_attrs();
  if (e != cudaSuccess) return e;
  return fused ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, sssp_persistent<true>,
                                                               kBlock, smem_bytes())
               : cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, sssp_persistent<false>,
                                                               kBlock, smem_bytes());
}

cudaError_t launch_sssp(const KArgs& a, bool fused, int grid, cudaStream_t st) {
  cudaError_t e = set_attrs();
  if (e != cudaSuccess) return e;
  KArgs args = a;
  void* params[] = {&args};
  const void* fn = fused ? (const void*)sssp_persistent<true> : (const void*)sssp_persistent<false>;
  return cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(kBlock), params, smem_bytes(), st);
}

static unsigned grid_for(int64_t count) {
  int64_t blocks = (count + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  if (blocks < 1) blocks = 1;
  return (unsigned)blocks;
}

cudaError_t launch_interleave(const int32_t* cols, const uint32_t* w, uint2* edges, int64_t count,
                              int64_t n, uint32_t* bad_flag, cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  interleave_kernel<<<grid_for(count), 256, 0, st>>>(cols, w, edges, count, n, bad_flag);
  return cudaGetLastError();
}

cudaError_t launch_build_slots(const int64_t* off, const uint2* edges, uint2* slots, int64_t n,
                               cudaStream_t st) {
  build_slots_kernel<<<grid_for(n), 256, 0, st>>>(off, edges, slots, n);
  return cudaGetLastError();
}

cudaError_t launch_max_degree(const int64_t* off, int64_t n, uint32_t* max_deg, cudaStream_t st) {
  max_degree_kernel<<<grid_for(n), 256, 0, st>>>(off, n, max_deg);
  return cudaGetLastError();
}

cudaError_t launch_validate_offsets(const int64_t* off, int64_t n, int64_t m, uint32_t* bad_flag,
                                    cudaStream_t st) {
  validate_offsets_kernel<<<grid_for(n), 256, 0, st>>>(off, n, m, bad_flag);
  return cudaGetLastError();
}

}  // namespace gi

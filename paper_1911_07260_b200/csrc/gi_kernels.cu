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
#include "gi_device.cuh"

// This file is compiled once per CTA width (GI_BLOCK / GI_VARIANT): v512 (the default,
// and the only one with GI_PRIMARY, which also builds the graph-setup kernels) and
// v1024 (skewed graphs: twice the warps per SM for memory-level parallelism).
#ifndef GI_VARIANT
#define GI_VARIANT v512
#endif
#ifndef GI_PRIMARY
#define GI_PRIMARY 1
#endif

#include <cooperative_groups.h>

#include <atomic>

namespace cg = cooperative_groups;

namespace gi {
namespace {

enum : uint32_t { MODE_ROUND = 0, MODE_EXTRACT = 1, MODE_DONE = 2, MODE_NONE = 3, MODE_STOP = 4, MODE_ADVANCE = 5 };
#ifndef GI_XTR
#define GI_XTR 4
#endif
constexpr int kXtr = GI_XTR;  // far-pile entries per thread per extraction chunk
constexpr int kFarSeg = kFarStage / (kBlock / 32);  // bsp: far staging entries per warp
static_assert(kFarSeg >= 32 * 8, "a warp's far segment must hold one relax batch (32 lanes x 8 edges)");
static_assert(kFarSeg <= 1024, "warp_flush_far tracks up to 32 entries per lane");
// A/B switches for measurements only (tools/ab_time.py); all 0 in the product build
#ifndef GI_X_NOPF
#define GI_X_NOPF 0
#endif
#ifndef GI_X_NOSTALE
#define GI_X_NOSTALE 0
#endif
#ifndef GI_BIGK
#if GI_BLOCK >= 1024
#define GI_BIGK 4  // 64 registers per thread at 1024 threads: fewer edges in flight per thread, less spill
#else
#define GI_BIGK 8
#endif
#endif
constexpr int kBigK = GI_BIGK;  // stage B: consecutive edges per thread per iteration

#ifndef GI_CLAIMS
#define GI_CLAIMS 4
#endif
constexpr uint32_t kClaimsPerCta = GI_CLAIMS;  // ROUND: ~claims per CTA per phase (chunk size)
#ifndef GI_MAXCLAIM
#define GI_MAXCLAIM 2048
#endif
// largest claim (= kBinCap, the staging size). Smaller caps (256, 512) were measured
// slower on configs 3-4 (more chunk passes), despite smaller straggler chunks
constexpr uint32_t kMaxClaim = GI_MAXCLAIM;
  // drain: spill a bin's big list above this

#ifndef GI_LANE_FAR
#define GI_LANE_FAR 1
#endif
#ifndef GI_LANE_PUSH
#define GI_LANE_PUSH 1
#endif
#ifdef GI_TRACE
// Debug builds only: cycles between trace points, accumulated by CTA 0 / thread 0 in
// shared memory (so that tracing adds ~no latency) and flushed at kernel exit.
__device__ unsigned long long g_trace[64];
__shared__ unsigned long long s_trace[64];
__shared__ long long s_trace_last;
#define TRACE(k)                                                   \
  do {                                                             \
    if (blockIdx.x == 0 && threadIdx.x == 0) {                     \
      long long t_ = clock64();                                    \
      s_trace[k] += (unsigned long long)(t_ - s_trace_last);       \
      s_trace[32 + (k)] += 1;                                      \
      s_trace_last = t_;                                           \
    }                                                              \
  } while (0)
#define TRACE_INIT()                                                          \
  do {                                                                        \
    if (threadIdx.x < 64) s_trace[threadIdx.x] = 0;                           \
    if (threadIdx.x == 0) s_trace_last = clock64();                           \
    __syncthreads();                                                          \
  } while (0)
#define TRACE_FLUSH()                                                         \
  do {                                                                        \
    if (blockIdx.x == 0 && threadIdx.x < 64) atomicAdd(&g_trace[threadIdx.x], s_trace[threadIdx.x]); \
  } while (0)
// async drain: per phase max over CTAs of feed+drain cycles / max depth; per item
// (all CTAs, lane 0 of each warp) claim->atomics-returned, ->push-done, idle spins
constexpr int kTracePhases = 16384;
__device__ unsigned long long g_phase[7][kTracePhases];  // max drain (async), max depth, max busy, sum busy, mode, cnt, hubs
__device__ unsigned long long g_item[16];
#define ITRACE_T(var) long long var = clock64()
#define ITRACE_DECL() unsigned long long it_acc[16] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0}
#define ITRACE_ADD(k, v) (it_acc[k] += (unsigned long long)(v))
#define ITRACE_FLUSH()                                                                    \
  do {                                                                                    \
    for (int k_ = 0; k_ < 16; ++k_)                                                       \
      if (it_acc[k_] && ((threadIdx.x & 31) == 0 || k_ >= 10)) atomicAdd(&g_item[k_], it_acc[k_]); \
  } while (0)
#else
#define ITRACE_T(var) do {} while (0)
#define ITRACE_DECL() do {} while (0)
#define ITRACE_ADD(k, v) do {} while (0)
#define ITRACE_FLUSH() do {} while (0)
#define TRACE(k) do {} while (0)
#define TRACE_INIT() do {} while (0)
#define TRACE_FLUSH() do {} while (0)
#endif

using dev::fence_acq_rel;
using dev::ld_relaxed;

__device__ __forceinline__ void red_min(uint32_t* p, uint32_t v) {
#if GI_X_DIST_EL
  uint64_t pol;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  asm volatile("red.relaxed.gpu.global.min.L2::cache_hint.u32 [%0], %1, %2;" ::"l"(p), "r"(v), "l"(pol) : "memory");
#else
  asm volatile("red.relaxed.gpu.global.min.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
#endif
}

// dist[] is written by atomics inside this kernel: read it coherently from L2,
// never through the non-coherent/L1 path (SURVEY §7 hard part 1).
__device__ __forceinline__ uint32_t ld_dist(const uint32_t* p) { return __ldcg(p); }

// extraction reads of dist (one random read per far entry): optionally evict-first, so the
// pile scan does not push the bitmaps and the mirror out of L2 (investigation flag)
#ifndef GI_X_XDIST_EF
#define GI_X_XDIST_EF 0
#endif
__device__ __forceinline__ uint32_t ld_dist_x(const uint32_t* p) {
#if GI_X_XDIST_EF
  uint64_t pol;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  uint32_t v;
  asm volatile("ld.global.cg.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
#else
  return __ldcg(p);
#endif
}

// L2 eviction-priority policies (createpolicy; the policy travels with the access).
__device__ __forceinline__ uint64_t pol_evict_last() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t pol_evict_first() {
  uint64_t p;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
#ifndef GI_X_DIST_EL
#define GI_X_DIST_EL 0
#endif
#ifndef GI_X_PMIR
#define GI_X_PMIR 1  // the persistent kernel's pre-reads use the expand mirror too (R17)
#endif
#ifndef GI_X_XSKIP
#define GI_X_XSKIP 1  // expand rows with no candidate past the mirror skip the atomics and pushes
#endif
#ifndef GI_X_RSKIP
#define GI_X_RSKIP 1  // relax_batch: warps with no lowering after the pre-read skip the pushes
#endif
#ifndef GI_X_XCOMPACT
#define GI_X_XCOMPACT 1  // expand: a block's candidates past the mirror relaxed densely
#endif
// slot prefetches (L2) of the vertices a big extraction makes live: the streaming
// extract_kernel (piles >= 2^21) and the persistent kernel's CTA-aggregated extraction.
// Off: a big extraction makes millions of vertices live, whose 64-byte slots overflow the
// L2 before the next round reads them (config 4: 20.04 -> 19.38 ms)
#ifndef GI_X_PFX
#define GI_X_PFX 0
#endif
#ifndef GI_X_PFAGG
#define GI_X_PFAGG 0
#endif
// the init's stores of Dist = {inf} with the streaming (evict-first) hint: the row is first
// touched again when the wavefront reaches it, so it need not displace the L2's working set
#ifndef GI_INIT_CS
#define GI_INIT_CS 0
#endif
// slot prefetches of expand's current-bucket pushes (GI_X_PFXC; off: config 4 19.37 -> 19.27
// ms) and of the relaxations' pushes and bin spills to the global frontier (GI_X_PFG) and of
// small in-kernel extractions (GI_X_PFXS); the last two off together: config 5 143.97 ->
// 142.95 ms, config 3 1.875 -> 1.850 ms, configs 1, 2, 4 within ±0.2 %
#ifndef GI_X_PFXC
#define GI_X_PFXC 0
#endif
#ifndef GI_X_PFG
#define GI_X_PFG 0
#endif
#ifndef GI_X_PFXS
#define GI_X_PFXS 0
#endif
#ifndef GI_X_WSKIP
#define GI_X_WSKIP 0
#endif
#ifndef GI_X_EDGE_EF
#define GI_X_EDGE_EF 0
#endif
// relaxation-target reads / writes of dist (skewed graphs: the hot targets should stay in L2)
#ifndef GI_X_DIST_L1
#define GI_X_DIST_L1 0
#endif
__device__ __forceinline__ uint32_t ld_dist_tgt(const uint32_t* p) {
#if GI_X_DIST_L1
  return __ldca(p);  // L1-cached pre-read: a stale value is only ever too high (dist decreases)
#elif GI_X_DIST_EL
  uint32_t v;
  asm volatile("ld.global.cg.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol_evict_last()));
  return v;
#else
  return __ldcg(p);
#endif
}
// the expand filter's mirror bytes (KArgs.mirror): coherent L2 reads, plain byte stores
__device__ __forceinline__ uint32_t ld_mirror(const uint8_t* p) {
  uint16_t x;
  asm volatile("ld.global.cg.u8 %0, [%1];" : "=h"(x) : "l"(p));
  return x;
}
__device__ __forceinline__ void st_mirror(uint8_t* p, uint32_t v) {
  asm volatile("st.global.u8 [%0], %1;" ::"l"(p), "h"((uint16_t)v) : "memory");
}
// relaxation atomics on dist (no pre-read) and ELL slot loads, with optional L2 policies
// (investigation: keep the wavefront's distances in L2 while the slots stream through)
#ifndef GI_X_ATOM_EL
#define GI_X_ATOM_EL 0
#endif
#ifndef GI_X_SLOT_EF
#define GI_X_SLOT_EF 1
#endif
__device__ __forceinline__ uint32_t atom_min_dist(uint32_t* p, uint32_t v) {
#if GI_X_ATOM_EL
  uint32_t old;
  asm volatile("atom.relaxed.gpu.global.min.L2::cache_hint.u32 %0, [%1], %2, %3;"
               : "=r"(old) : "l"(p), "r"(v), "l"(pol_evict_last()) : "memory");
  return old;
#else
  return atomicMin(p, v);
#endif
}
__device__ __forceinline__ uint2 ld_slot(const uint2* p) {
#if GI_X_SLOT_EF
  uint2 x;
  asm volatile("ld.global.nc.L2::cache_hint.v2.u32 {%0, %1}, [%2], %3;" : "=r"(x.x), "=r"(x.y) : "l"(p), "l"(pol_evict_first()));
  return x;
#else
  return __ldg(p);
#endif
}
// packed edges (w << colbits | col), streamed
#ifndef GI_X_PEDGE
#define GI_X_PEDGE 1
#endif
__device__ __forceinline__ uint32_t ld_pedge(const uint32_t* p) {
#if GI_X_PEDGE == 1
  return __ldcs(p);  // ld.global.cs: streamed once, evict-first
#elif GI_X_PEDGE == 2
  return __ldg(p);
#else
  uint32_t x;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(x) : "l"(p), "l"(pol_evict_first()));
  return x;
#endif
}
// streamed CSR edges: read once per relaxation pass
__device__ __forceinline__ uint2 ld_edge(const uint2* p) {
#if GI_X_EDGE_EF
  uint2 x;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u32 {%0,%1}, [%2], %3;"
               : "=r"(x.x), "=r"(x.y) : "l"(p), "l"(pol_evict_first()));
  return x;
#else
  return __ldg(p);
#endif
}

__device__ __forceinline__ void prefetch_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}
// The slot of a vertex pushed into this CTA's own bin is read by this SM in the next
// sub-round: pull it into L1 so that the read does not cost an L2 round trip.
__device__ __forceinline__ void prefetch_own(const void* p) {
#ifdef GI_PF_L2
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
#else
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
#endif
}

__device__ __forceinline__ uint32_t fdiv(uint32_t x, const FastDiv& f) {
  uint32_t t = __umulhi(x, f.mul);
  return (t + ((x - t) >> f.s1)) >> f.s2;
}

// Bucket of a tentative distance d under the A* priority d + h(v) (the
// "estimated distance" of the path through v). h = 0 for SSSP/PPSP. A priority past
// UINT32_MAX-1 lands in the last bucket (a merged top bucket is still exact).
__device__ __forceinline__ uint32_t prio_bucket(uint32_t d, uint32_t hv, const FastDiv& f) {
  const uint32_t p = d + hv;
  return fdiv((p < d || p == kInf) ? kInf - 1u : p, f);
}

// The group barrier of the execution-group ladder: a one-CTA group needs only
// the CTA barrier, a group that is one thread-block cluster the hardware cluster barrier
// (release / acquire at cluster scope), any other group the barrier of global atomics.
__device__ __forceinline__ void group_barrier_r(Ctl* ctl, uint32_t G, uint32_t rung) {
  if (rung == 1) {
    __syncthreads();
  } else if (rung == 2) {
    __syncthreads();
    cg::this_cluster().sync();
  } else {
    dev::group_barrier(&ctl->bar, G);
  }
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
  uint32_t farcnt;          // fill of the far staging buffer (async drain: one CTA-wide region)
  uint32_t wfar[kBlock / 32];  // bsp kernels: fill of each warp's segment of the far staging
  uint32_t mode, b, cnt, hn;
  uint32_t claim;           // ROUND: base of the chunk this CTA claimed
  uint32_t redw[kBlock / 32];  // EXTRACT: per-warp exclusive offsets of kept far entries
  uint32_t xbase;           // EXTRACT: this chunk's base in the receiving far buffer
  uint32_t fmin;
  unsigned long long total; // edges of the high-degree list (exclusive-scan total)
  unsigned long long red[kBlock / 32];
  // async drain (KIND_FUSED_ASYNC): CTA-local work ring counters
  uint32_t head;            // next ring position to claim
  uint32_t tail;            // ring positions reserved by producers
  uint32_t done;            // processed entries + finished feeding warps - warps (termination)
  uint32_t maxdep;          // max depth (sub-round equivalent) processed this phase
  uint32_t spilled;         // some push overflowed the ring threshold this phase
  uint32_t xhn;             // expand: entries of the group list after collection
  uint32_t wend, ws;        // bucket window: end of the open window, start of a new one (ADVANCE)
  uint32_t lcnt;            // bucket window: later-pile entries (PPSP stop cleanup)
  uint8_t* mirror;          // expand queries: the dist mirror (KArgs.mirror, R17) for the pre-reads
  unsigned long long xS[kMaxGroupCtas + 1];  // expand: exclusive prefix of the CTA slice totals
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
  uint32_t T;              // fusion threshold (async drain: ring occupancy limit)
  int32_t* farstage;       // CTA-local staging of far-pile pushes (shared memory, kFarStage)
  const uint32_t* h;       // A* heuristic per vertex (nullptr: SSSP/PPSP)
  Shared* s;
  uint32_t my_fmin;        // thread-local min far bucket (reduced at phase end)
  bool pre_read;
  bool lazy;               // fully lazy schedule: no eager current-bucket pushes
  bool collect;            // expand collection (E1): every deg > 8 vertex goes to the CTA list,
                           // which process_bin copies to the group list with one atomic
};

// Append v to the global frontier once per phase (dedup bit), warp-aggregated.
__device__ __forceinline__ void push_global(Ctx& c, int32_t v) {
  const uint32_t bit = 1u << (v & 31);
  const uint32_t old = atomicOr(&c.qbits_next[v >> 5], bit);
  if (!(old & bit)) {
    if (GI_X_PFG) prefetch_l2(c.slots + 8 * (size_t)v);
    cg::coalesced_group g = cg::coalesced_threads();
    uint32_t base = 0;
    if (g.thread_rank() == 0) base = atomicAdd(c.qcount_next, g.size());
    base = g.shfl(base, 0);
    c.q_next[base + g.thread_rank()] = v;
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

__device__ __noinline__ void mark_overflow(uint32_t* ovfbits, uint32_t* ovf_cand, uint32_t v) {
  atomicOr(&ovfbits[v >> 5], 1u << (v & 31));
  atomicOr(ovf_cand, 1u);
}

// Warp-aggregated append of the entries v[x] with bit x of `m` set (per lane) to a
// global list: a warp scan of the per-lane counts and ONE atomicAdd per warp.
template <int X>
__device__ __forceinline__ void warp_append(uint32_t m, const int32_t (&v)[X], int32_t* list, uint32_t* count,
                                            const uint2* slots_pf) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t nk = __popc(m);
  uint32_t incl = nk;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= (uint32_t)o) incl += t;
  }
  const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
  if (tot == 0) return;
  uint32_t base = 0;
  if (lane == 0) base = atomicAdd(count, tot);
  base = __shfl_sync(0xffffffffu, base, 0);
  uint32_t off = base + incl - nk;
#pragma unroll
  for (int x = 0; x < X; ++x)
    if (m & (1u << x)) {
      if (slots_pf) prefetch_l2(slots_pf + 8 * (size_t)v[x]);
      list[off++] = v[x];
    }
}

// CTA-aggregated append of the entries v[x] with bit x of `m` set (per lane): a warp scan,
// a scan of the warp totals, ONE global atomic per CTA call. Every thread of the CTA must
// call it (two CTA barriers). Used where a whole grid appends to one counter at a high rate
// (a big extraction: one atomic per warp per chunk on the same word serialised at ~150 M/s).
template <int X>
__device__ __forceinline__ void cta_append(uint32_t m, const int32_t (&v)[X], int32_t* list, uint32_t* count,
                                           uint32_t* wslot, const uint2* slots_pf) {
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t nk = __popc(m);
  uint32_t incl = nk;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= (uint32_t)o) incl += t;
  }
  if (lane == 31) wslot[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const uint32_t w = lane < kBlock / 32 ? wslot[lane] : 0u;
    uint32_t wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= (uint32_t)o) wi += t;
    }
    const uint32_t tot = __shfl_sync(0xffffffffu, wi, kBlock / 32 - 1);
    uint32_t base = 0;
    if (lane == 0 && tot) base = atomicAdd(count, tot);
    base = __shfl_sync(0xffffffffu, base, 0);
    if (lane < kBlock / 32) wslot[lane] = base + wi - w;
  }
  __syncthreads();
  uint32_t off = wslot[warp] + incl - nk;
#pragma unroll
  for (int x = 0; x < X; ++x)
    if (m & (1u << x)) {
      if (slots_pf) prefetch_l2(slots_pf + 8 * (size_t)v[x]);
      list[off++] = v[x];
    }
}

// Dedup-append of n staged vertices to a global list: the bit test-and-set (atomicOr)
// of 4 entries per thread is in flight at once, and the list positions come from one
// global atomic per WARP per 128 entries (warp scan) — no CTA barrier, so that a small
// flush costs one round trip and a large one a few, not one chain per entry. All
// threads call it (warp-uniform trip count).
template <typename Get>
__device__ __forceinline__ void bulk_append(uint32_t n, Get get, uint32_t* bits, int32_t* list, uint32_t* count,
                                            const uint2* slots_pf) {
  for (uint32_t base = 0; base < n; base += 4 * kBlock) {
    int32_t v[4];
    uint32_t old[4];
#pragma unroll
    for (int x = 0; x < 4; ++x) {
      const uint32_t i = base + x * kBlock + threadIdx.x;
      v[x] = i < n ? get(i) : -1;
    }
#pragma unroll
    for (int x = 0; x < 4; ++x) old[x] = v[x] >= 0 ? atomicOr(&bits[v[x] >> 5], 1u << (v[x] & 31)) : ~0u;
    uint32_t newm = 0;
#pragma unroll
    for (int x = 0; x < 4; ++x)
      if (v[x] >= 0 && !(old[x] & (1u << (v[x] & 31)))) newm |= 1u << x;
    warp_append(newm, v, list, count, slots_pf);
  }
}

// A warp's segment of the far staging is full (or the phase ends): dedup-append its n
// entries (atomicOr of 4 per lane in flight, one append atomic per 128 entries). Only this
// warp touches its segment, so no CTA barrier is needed mid-phase.
__device__ __forceinline__ void warp_flush_far(Ctx& c, const int32_t* seg, uint32_t n) {
  // the segment's test-and-sets first (4 per lane in flight per round), then one warp scan
  // and ONE append atomic (every warp of the grid appends to the same counter)
  const uint32_t lane = threadIdx.x & 31;
  uint32_t newm = 0;  // bit r*4+x: entry (r*128 + x*32 + lane) is new
  for (uint32_t r = 0; r * 128 < n; ++r) {
    int32_t v[4];
    uint32_t old[4];
#pragma unroll
    for (int x = 0; x < 4; ++x) {
      const uint32_t i = r * 128 + x * 32 + lane;
      v[x] = i < n ? seg[i] : -1;
    }
#pragma unroll
    for (int x = 0; x < 4; ++x) old[x] = v[x] >= 0 ? atomicOr(&c.farbits[v[x] >> 5], 1u << (v[x] & 31)) : ~0u;
#pragma unroll
    for (int x = 0; x < 4; ++x)
      if (v[x] >= 0 && !(old[x] & (1u << (v[x] & 31)))) newm |= 1u << (r * 4 + x);
  }
  const uint32_t nk = __popc(newm);
  uint32_t incl = nk;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= (uint32_t)o) incl += t;
  }
  const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
  if (tot) {
    uint32_t base = 0;
    if (lane == 0) base = atomicAdd(c.fcount_live, tot);
    base = __shfl_sync(0xffffffffu, base, 0);
    uint32_t off = base + incl - nk;
    while (newm) {
      const int b = __ffs(newm) - 1;
      newm &= newm - 1;
      c.far_live[off++] = seg[(b >> 2) * 128 + (b & 3) * 32 + lane];
    }
  }
  __syncwarp();
}

// R17 in the persistent kernel (expand queries): the pre-read is the vertex's byte of the
// dist mirror; a candidate it does not rule out takes atomicMin, whose old value decides
// the push exactly, and the byte is set to the new distance or tightened to the old one.
// Returns false (nothing done) when the query has no mirror.
template <int K>
__device__ __forceinline__ bool relax_mirrored(Ctx& c, const uint2 (&e)[K], const uint32_t (&nd)[K], uint32_t& ok,
                                               uint32_t (&old)[K]) {
  uint8_t* mir = c.s->mirror;
  if (!mir) return false;
  uint32_t mb[K];
#pragma unroll
  for (int k = 0; k < K; ++k) mb[k] = (ok & (1u << k)) ? ld_mirror(mir + e[k].x) : 0u;
#pragma unroll
  for (int k = 0; k < K; ++k)
    if (!(mb[k] == 0xFFu || nd[k] < mb[k])) ok &= ~(1u << k);
#pragma unroll
  for (int k = 0; k < K; ++k) old[k] = (ok & (1u << k)) ? atomicMin(c.dist + e[k].x, nd[k]) : 0u;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    if (!(ok & (1u << k))) continue;
    if (nd[k] < old[k]) {
      if (nd[k] < 0xFFu) st_mirror(mir + e[k].x, nd[k]);
    } else if (old[k] < mb[k]) {
      st_mirror(mir + e[k].x, old[k]);  // tighten (old < 0xFF)
    }
  }
  return true;
}

// Relax K edges per thread (u -> e[k].x, weight e[k].y, from du[k]); lanes with
// bit k of `valid` clear do nothing. Every load and atomic of the batch is issued
// before any result is consumed (memory-level parallelism on the critical chain).
// Must be called by all 32 lanes of the warp (the appends are warp-aggregated).
template <bool FUSED, int K, bool LD = false, bool MIR = false>
__device__ __forceinline__ uint32_t relax_batch(Ctx& c, const uint2 (&e)[K], const uint32_t (&du)[K],
                                                uint32_t valid, const uint32_t* cur = nullptr) {
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
  TRACE(29);  // the slots have arrived (nd consumed them)
  // expand queries (XP kernels): the candidates the dist mirror rules out touch no dist
  bool mirrored = false;
  if constexpr (MIR && !LD && GI_X_PMIR) mirrored = relax_mirrored<K>(c, e, nd, ok, old);
  if (mirrored) {
    // ok and old are what the atomic path below would leave
  } else if (!LD && c.pre_read) {
    // pre-read dist[v]; only an improving candidate is written, with a fire-and-forget
    // red.min, and the pre-read value stands for the atomic's old value. Two threads that
    // both improve on the same pre-read may both push v: a duplicate entry, which the
    // dedup bits (far pile) or the staleness probe (bins) absorb; the thread holding the
    // final minimum always pushes (whoever wrote it first saw a larger value).
#pragma unroll
    for (int k = 0; k < K; ++k) old[k] = (ok & (1u << k)) ? ld_dist_tgt(c.dist + e[k].x) : 0u;
#pragma unroll
    for (int k = 0; k < K; ++k)
      if (!(nd[k] < old[k])) ok &= ~(1u << k);
#pragma unroll
    for (int k = 0; k < K; ++k)
      if (ok & (1u << k)) red_min(c.dist + e[k].x, nd[k]);
  } else {
#pragma unroll
    for (int k = 0; k < K; ++k) old[k] = (ok & (1u << k)) ? atom_min_dist(c.dist + e[k].x, nd[k]) : 0u;
  }
  // late staleness: the probe of the source vertex (cur, issued with the slot load) was
  // not waited for before the atomics; an entry superseded by a newer one of the same
  // vertex drops its pushes (that entry's relaxations supersede these)
  uint32_t stale = 0;
  if (cur) {
#pragma unroll
    for (int k = 0; k < K; ++k)
      if (cur[k] < du[k]) stale |= 1u << k;
    ok &= ~stale;
  }
  // pre-read / mirror filters (skewed graphs): a warp none of whose lanes lowered anything
  // skips the classification and the pushes with one vote
  if constexpr (!LD && GI_X_RSKIP) {
    if ((mirrored || c.pre_read) && !__any_sync(0xffffffffu, ok != 0u)) return stale;
  }
  // classify the successful lowerings: current bucket (bin) or a future one (far pile).
  // A*: priority bucket of nd + h(v), raised to the current bucket if an inconsistent
  // heuristic would put it below (the monotone max(f + h, g[src]) of SPEC.md:355-358).
  uint32_t curm = 0, farm = 0;
#ifdef GI_TRACE
  if (threadIdx.x == 0 && ok) { volatile uint32_t sink_ = old[0]; (void)sink_; }  // wait for the atomic
#endif
  TRACE(30);  // the atomics have returned
  uint32_t bk[K];
  if (c.h) {  // uniform branch: SSSP / PPSP never pay for the heuristic
    uint32_t hv[K];
#pragma unroll
    for (int k = 0; k < K; ++k) hv[k] = (ok & (1u << k)) ? __ldg(c.h + e[k].x) : 0u;
#pragma unroll
    for (int k = 0; k < K; ++k) bk[k] = max(prio_bucket(nd[k], hv[k], c.div), c.b);
  } else {
#pragma unroll
    for (int k = 0; k < K; ++k) bk[k] = fdiv(nd[k], c.div);  // nd >= du >= bΔ: bk >= b
  }
#pragma unroll
  for (int k = 0; k < K; ++k) {
    if ((ok & (1u << k)) && nd[k] < old[k]) {
      if (bk[k] == c.b && !c.lazy) curm |= 1u << k;
      else farm |= 1u << k;  // bk > b
    }
  }
  // warp-aggregated appends: one ballot per item slot, one shared atomic per warp
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t lt = (1u << lane) - 1u;
  uint32_t ovm = FUSED ? 0u : curm;  // current-bucket pushes bound for the global frontier
  if constexpr (FUSED && GI_LANE_PUSH) {
    // one shared atomic per pushing lane: no ballot -> warp atomic -> shuffle chain on the
    // critical path of a level (a bin sub-round pushes a handful of vertices per warp)
#pragma unroll
    for (int k = 0; k < K; ++k) {
      if ((curm >> k) & 1u) {
        const uint32_t pos = atomicAdd(c.outcnt, 1u);
        if (pos < (uint32_t)kBinCap) {
          if (!GI_X_NOPF) prefetch_own(c.slots + 8 * (size_t)e[k].x);
          c.out[pos] = make_uint2(e[k].x, nd[k]);
        } else {
          ovm |= 1u << k;
        }
      }
    }
  } else if constexpr (FUSED) {
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
          if (pos < (uint32_t)kBinCap) {
            if (!GI_X_NOPF) prefetch_own(c.slots + 8 * (size_t)e[k].x);
            c.out[pos] = make_uint2(e[k].x, nd[k]);
          } else {
            ovm |= 1u << k;  // bin full: next group-wide round
          }
        }
      }
    }
  }
  if (FUSED && LD && GI_LANE_FAR) {
    // a full bin (rare on low-degree graphs): per-lane global pushes, no warp vote on the path
    if (ovm) {
#pragma unroll
      for (int k = 0; k < K; ++k)
        if ((ovm >> k) & 1u) push_global(c, (int32_t)e[k].x);
    }
  } else if (__any_sync(0xffffffffu, ovm != 0)) {  // dedup (qbits) with every atomic in flight, one append per warp
    uint32_t ob[K];
    int32_t vv[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      vv[k] = (int32_t)e[k].x;
      ob[k] = ((ovm >> k) & 1u) ? atomicOr(&c.qbits_next[e[k].x >> 5], 1u << (e[k].x & 31)) : ~0u;
    }
    uint32_t newm = 0;
#pragma unroll
    for (int k = 0; k < K; ++k)
      if (((ovm >> k) & 1u) && !(ob[k] & (1u << (e[k].x & 31)))) newm |= 1u << k;
    warp_append(newm, vv, c.q_next, c.qcount_next, GI_X_PFG ? c.slots : nullptr);
  }
  if (LD && GI_LANE_FAR) {
    // low-degree graphs: far pushes are few per warp; one shared atomic per pushing lane on
    // the warp's segment counter, and the rare overflow goes straight to the global pile
    const uint32_t warp = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      if ((farm >> k) & 1u) {
        c.my_fmin = min(c.my_fmin, bk[k]);
        const uint32_t pos = atomicAdd(&c.s->wfar[warp], 1u);
        if (pos < (uint32_t)kFarSeg) c.farstage[warp * kFarSeg + pos] = (int32_t)e[k].x;
        else push_far_global(c, (int32_t)e[k].x);
      }
    }
  } else {
    uint32_t mk[K], pre[K], tot = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      mk[k] = __ballot_sync(0xffffffffu, (farm >> k) & 1u);
      pre[k] = tot;
      tot += __popc(mk[k]);
    }
    if (tot) {
      // this warp's segment of the far staging; flushed by the warp itself when full
      const uint32_t warp = threadIdx.x >> 5;
      int32_t* seg = c.farstage + warp * kFarSeg;
      uint32_t base = c.s->wfar[warp];
      if (base + tot > (uint32_t)kFarSeg) {  // warp-uniform
        warp_flush_far(c, seg, base);
        base = 0;
      }
#pragma unroll
      for (int k = 0; k < K; ++k) {
        if ((farm >> k) & 1u) {
          c.my_fmin = min(c.my_fmin, bk[k]);
          seg[base + pre[k] + __popc(mk[k] & lt)] = (int32_t)e[k].x;
        }
      }
      __syncwarp();
      if (lane == 0) c.s->wfar[warp] = base + tot;
      __syncwarp();
    }
  }
  return stale;
}

// Stage A — vertices with deg <= 8: ITEMS (entry, slot index), 8 per frontier entry;
// the 8 lanes of an octet share one entry and lane k relaxes entry k of its 64-byte
// ELL slot (one coalesced 64 B load per octet). Each thread holds U items in flight.
// Vertices with deg > 8 are appended to the CTA's high-degree list for stage B.
template <bool FUSED, int U, bool LD = false, bool MIR = false>
__device__ __forceinline__ void stage_small(Ctx& c, const uint2* in, uint32_t nin, bool check_stale,
                                            uint32_t& nv, uint32_t& ne) {
  const uint32_t nitems = nin * 8;
  const uint32_t sub = threadIdx.x & 7;
  for (uint32_t base = 0; base < nitems; base += kBlock * U) {
    // a warp with no item here (nor in any later pass) goes straight to the CTA barrier:
    // a sub-round at a chain's tail holds a few vertices, and 15 idle warps stepping through
    // the predicated-off batch would take the issue slots of the one with work
    if (GI_X_WSKIP && base + (threadIdx.x & ~31u) >= nitems) break;  // warp-uniform
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
        e[u] = ld_slot(c.slots + 8 * (size_t)en.x + sub);
        have |= 1u << u;
      }
    }
    // staleness probe of the source vertices: issued now, consumed after the atomics
    // (relax_batch) except for high-degree vertices, which are queued only if fresh
    uint32_t cur[U];
#pragma unroll
    for (int u = 0; u < U; ++u) cur[u] = (check_stale && (have & (1u << u))) ? ld_dist(c.dist + v[u]) : kInf;
    TRACE(2);
    uint32_t valid = 0, heads = 0;
    const uint32_t lane = threadIdx.x & 31, lt = (1u << lane) - 1u;
#pragma unroll
    for (int u = 0; u < U; ++u) {  // warp-uniform: the appends below are warp-aggregated
      const bool hv_ = (have >> u) & 1u;
      const bool big = !LD && hv_ && e[u].x == kColBig;  // octet-uniform
      if (hv_ && !big) {
        if (sub == 0) heads |= 1u << u;
        if (e[u].x != kColEmpty) valid |= 1u << u;
      }
      if constexpr (!LD) {
        if (!__any_sync(0xffffffffu, big)) continue;
        // a big slot holds {kColBig, deg}, {kColBig, beg_lo}, {kColBig, beg_hi}
        const uint32_t lo = __shfl_sync(0xffffffffu, e[u].y, 1, 8);
        const uint32_t hi = __shfl_sync(0xffffffffu, e[u].y, 2, 8);
        const bool mine = big && sub == 0 && !(cur[u] < du[u]);  // fresh entries only
        const uint32_t deg = e[u].y;
        const int64_t beg = (int64_t)(((uint64_t)hi << 32) | lo);
        // hubs (deg >= hub_min): the group hub list, split over every CTA next phase;
        // one global atomic per warp (every CTA appends to the same counter)
        const bool hub = mine && deg >= c.hub_min && !c.collect;
        const uint32_t mh = __ballot_sync(0xffffffffu, hub);
        uint32_t hbase = 0;
        if (mh) {
          if (lane == 0) hbase = atomicAdd(c.hcount_next, (uint32_t)__popc(mh));
          hbase = __shfl_sync(0xffffffffu, hbase, 0);
        }
        const uint32_t hp = hbase + __popc(mh & lt);
        const bool hub_ok = hub && hp < c.hubcap;
        if (hub_ok) {
          HubEnt he;
          he.beg = beg;
          he.deg = deg;
          he.du = du[u];
          c.hub_next[hp] = he;
        }
        // the rest: this CTA's high-degree list (stage B), one shared atomic per warp
        const bool loc = mine && !hub_ok;
        const uint32_t ml = __ballot_sync(0xffffffffu, loc);
        uint32_t lbase = 0;
        if (ml) {
          if (lane == 0) lbase = atomicAdd(&c.s->bigtail, (uint32_t)__popc(ml));
          lbase = __shfl_sync(0xffffffffu, lbase, 0);
        }
        if (loc) {
          const uint32_t pos = lbase + __popc(ml & lt);
          if (pos < (uint32_t)kBigCap) {
            BigEnt be;
            be.beg = beg;
            be.deg = deg;
            be.du = du[u];
            c.big[pos] = be;
          } else {
            push_global(c, (int32_t)v[u]);  // list full: the next group-wide round takes it
          }
        }
        nv += mine;
      }
    }
    const uint32_t stale = relax_batch<FUSED, U, LD, MIR>(c, e, du, valid, (check_stale && !GI_X_NOSTALE) ? cur : nullptr);
    // counters: non-stale entries and their edges (stale is per lane; each lane saw
    // its own probe of the same word)
    nv += __popc(heads & ~stale);
    ne += __popc(valid & ~stale);
    TRACE(3);
  }
}

// Stage B — vertices with deg > 8: their edges are concatenated (exclusive prefix of
// the degrees) and split evenly over all threads of the CTA, 4 edges per thread per
// iteration; an edge finds its vertex by binary search in the prefix array.
template <bool FUSED, bool MIR = false>
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
  TRACE(12);
  if (threadIdx.x == 0) ne += (uint32_t)total;
  // each thread relaxes kBigK CONSECUTIVE edges per iteration: one binary search for
  // the first, then a forward walk (entries have deg >= 1 except empty hub slices, which
  // the walk skips); a warp covers kBigK*256 B of contiguous edges per iteration.
  // (Software-pipelining the next iteration's edge loads was measured slower: spills at
  // 1024 threads, longer code at 512.)
  auto fetch = [&](unsigned long long k0, uint2 (&e)[kBigK], uint32_t (&du)[kBigK], uint32_t& valid) {
    valid = 0;
    const unsigned long long kt = k0 + (unsigned long long)kBigK * threadIdx.x;
#pragma unroll
    for (int u = 0; u < kBigK; ++u) { e[u] = make_uint2(0, 0); du[u] = 0; }
    if (kt < total) {
      uint32_t lo = 0, hi = nb;  // last i with pre[i] <= kt
      while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (c.pre[mid] <= kt) lo = mid; else hi = mid;
      }
      unsigned long long nxt = lo + 1 < nb ? c.pre[lo + 1] : total;
      BigEnt be = c.big[lo];
      int64_t rel = be.beg - (int64_t)c.pre[lo];  // edge index = rel + k within entry lo
#pragma unroll
      for (int u = 0; u < kBigK; ++u) {
        const unsigned long long k = kt + u;
        if (k < total) {
          while (k >= nxt) {  // next entry (skipping empty ones)
            ++lo;
            be = c.big[lo];
            rel = be.beg - (int64_t)nxt;
            nxt = lo + 1 < nb ? c.pre[lo + 1] : total;
          }
          e[u] = ld_edge(c.edges + rel + (int64_t)k);
          du[u] = be.du;
          valid |= 1u << u;
        }
      }
    }
  };
  const unsigned long long step = (unsigned long long)kBigK * kBlock;
  for (unsigned long long k0 = 0; k0 < total; k0 += step) {
    uint2 e[kBigK];
    uint32_t du[kBigK];
    uint32_t valid;
    fetch(k0, e, du, valid);
    TRACE(16);
    relax_batch<FUSED, kBigK, false, MIR>(c, e, du, valid);
    TRACE(17);
  }
  TRACE(13);
}

// ---------------------------------------------------------------------------------
// Expand (skewed graphs, ROUND phases): every frontier vertex of out-degree > 8 found this
// phase (and every hub queued by the previous phase's drains) is an entry {beg, deg, du} of
// the group list X. The concatenation of their edge lists — E edges — is split into W equal
// contiguous ranges, one per warp of the group, so that a hub of a million edges and ten
// thousand vertices of degree 20 cost the same per warp (edge-balanced relaxation, kernel
// (b)). Two steps after the phase's collection barrier:
//   expand_scan  — each CTA takes a contiguous slice of X and writes the exclusive degree
//                  prefix of every entry WITHIN its slice (xpre) and the slice total (xtot);
//   expand_relax — after a second barrier, global position of entry i of slice r is
//                  S[r] + xpre[i] (S = prefix of the slice totals, built in shared memory by
//                  every CTA). A warp finds the entry holding its first position (binary
//                  search over S, then a 32-ary search over xpre), keeps a window of 32
//                  consecutive entries in its lanes (entry end positions relative to the
//                  range start) and maps each row of 32 consecutive positions to entries
//                  with one ballot, one OR-reduction and a popcount: lane k reads edge
//                  (position - entry start + entry beg) — consecutive lanes read consecutive
//                  edges of the same list (coalesced).
// ---------------------------------------------------------------------------------
__device__ __forceinline__ void expand_scan(const HubEnt* X, unsigned long long* xpre, unsigned long long* xtot,
                                            uint32_t hn, uint32_t G, uint32_t rank, Shared& s) {
  const uint32_t lo = (uint32_t)(((uint64_t)hn * rank) / G), hi = (uint32_t)(((uint64_t)hn * (rank + 1)) / G);
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned long long carry = 0;
  for (uint32_t base = lo; base < hi; base += 4 * kBlock) {
    unsigned long long loc[4], sum = 0;
#pragma unroll
    for (int x = 0; x < 4; ++x) {
      const uint32_t i = base + 4 * threadIdx.x + x;
      loc[x] = sum;
      sum += i < hi ? __ldcg(&X[i].deg) : 0u;
    }
    unsigned long long incl = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= (uint32_t)o) incl += t;
    }
    if (lane == 31) s.red[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      const unsigned long long w = lane < kBlock / 32 ? s.red[lane] : 0ull;
      unsigned long long wi = w;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long t = __shfl_up_sync(0xffffffffu, wi, o);
        if (lane >= (uint32_t)o) wi += t;
      }
      if (lane < kBlock / 32) s.red[lane] = wi - w;
      if (lane == kBlock / 32 - 1) s.total = wi;
    }
    __syncthreads();
    const unsigned long long off = carry + s.red[warp] + incl - sum;
#pragma unroll
    for (int x = 0; x < 4; ++x) {
      const uint32_t i = base + 4 * threadIdx.x + x;
      if (i < hi) xpre[i] = off + loc[x];
    }
    carry += s.total;
    __syncthreads();  // s.red / s.total are rewritten by the next chunk
  }
  if (threadIdx.x == 0) xtot[rank] = carry;
}

// One warp's window of list entries jb .. jb+31: lane k holds entry jb+k's end position
// relative to the warp's range start (clamped to [0, len]), beg - start (edge index of a
// position = off + position) and du.
struct XWin {
  uint32_t endr;
  int64_t off;
  uint32_t du;
};

__device__ __forceinline__ XWin expand_window(const HubEnt* X, const unsigned long long* xpre, uint32_t hn,
                                              uint32_t G, const unsigned long long* S, uint32_t jb,
                                              unsigned long long a, uint32_t len) {
  const uint32_t idx = jb + (threadIdx.x & 31);
  XWin w;
  w.endr = len; w.off = 0; w.du = 0;
  if (idx < hn) {
    // written by other CTAs before the group barrier: L2-coherent loads
    const uint4 he = __ldcg(reinterpret_cast<const uint4*>(X + idx));  // {beg lo, beg hi, deg, du}
    const int64_t beg = (int64_t)(((uint64_t)he.y << 32) | he.x);
    const uint32_t r = (uint32_t)((((uint64_t)idx + 1) * G - 1) / hn);  // slice of idx
    const unsigned long long start = S[r] + __ldcg(xpre + idx);
    const unsigned long long end = start + he.z;
    w.endr = end <= a ? 0u : (uint32_t)min(end - a, (unsigned long long)len);
    w.off = beg - (int64_t)start;
    w.du = he.w;
  }
  return w;
}

#ifndef GI_INKERNEL_EXPAND
#define GI_INKERNEL_EXPAND 0
#endif
#ifndef GI_XK
#if GI_BLOCK >= 1024
#define GI_XK 4
#else
#define GI_XK 8
#endif
#endif
constexpr int kXK = GI_XK;  // expand: rows of 32 edges per warp per iteration

// Lean relaxation of one expand row set: the pre-read dist[v] filters (a skewed graph's
// edges mostly hit settled or already-lower targets); an improving candidate is written
// with red.min and pushed — current bucket to the CTA bin (fusion) or the global frontier,
// future buckets to the warp's far staging segment (one shared atomic per pushing lane).
template <bool FUSED>
__device__ __forceinline__ void expand_push(Ctx& c, uint32_t v, uint32_t nd) {
  red_min(c.dist + v, nd);
  const uint32_t bk = c.h ? max(prio_bucket(nd, __ldg(c.h + v), c.div), c.b) : fdiv(nd, c.div);
  if (bk == c.b && !c.lazy) {
    if constexpr (FUSED) {
      const uint32_t pos = atomicAdd(c.outcnt, 1u);
      if (pos < (uint32_t)kBinCap) {
        prefetch_own(c.slots + 8 * (size_t)v);
        c.out[pos] = make_uint2(v, nd);
        return;
      }
    }
    push_global(c, (int32_t)v);
  } else {
    c.my_fmin = min(c.my_fmin, bk);
    const uint32_t warp = threadIdx.x >> 5;
    const uint32_t pos = atomicAdd(&c.s->wfar[warp], 1u);
    if (pos < (uint32_t)kFarSeg) c.farstage[warp * kFarSeg + pos] = (int32_t)v;
    else push_far_global(c, (int32_t)v);
  }
}

template <bool PACKED> struct XEdge { using T = uint2; };
template <> struct XEdge<true> { using T = uint32_t; };  // {w << colbits | col}

template <bool FUSED, bool PACKED>
__device__ __forceinline__ void expand_relax(Ctx& c, const HubEnt* X, const unsigned long long* xpre, uint32_t hn,
                                             uint32_t G, const unsigned long long* S, unsigned long long a,
                                             unsigned long long b, const uint32_t* pedges, uint32_t colbits,
                                             uint32_t& ne) {
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t len = (uint32_t)(b - a);
  // slice r holding position a: the largest r with S[r] <= a (S[G] = E > a)
  uint32_t rlo = 0, rhi = G;
  while (rhi - rlo > 1) {
    const uint32_t mid = (rlo + rhi) >> 1;
    if (S[mid] <= a) rlo = mid; else rhi = mid;
  }
  // entry within the slice: the largest i with xpre[i] <= a - S[r] (32-ary search)
  const unsigned long long t = a - S[rlo];
  uint32_t ilo = (uint32_t)(((uint64_t)hn * rlo) / G), ihi = (uint32_t)(((uint64_t)hn * (rlo + 1)) / G);
  while (ihi - ilo > 32) {
    const uint32_t step = (ihi - ilo + 31) / 32;
    const uint32_t idx = ilo + lane * step;
    const bool pr = idx < ihi && __ldcg(xpre + idx) <= t;
    const uint32_t cnt = __popc(__ballot_sync(0xffffffffu, pr));
    ilo += (cnt - 1) * step;
    ihi = min(ilo + step, ihi);
  }
  {
    const uint32_t idx = ilo + lane;
    const bool pr = idx < ihi && __ldcg(xpre + idx) <= t;
    ilo += __popc(__ballot_sync(0xffffffffu, pr)) - 1;
  }
  uint32_t jb = ilo;
  XWin w = expand_window(X, xpre, hn, G, S, jb, a, len);
  const uint32_t lanemask = (2u << lane) - 2u;  // bits 1..lane (lane 31: 0xFFFFFFFE)
  const uint32_t cmask = colbits >= 32 ? 0xFFFFFFFFu : (1u << colbits) - 1u;
  constexpr int K = kXK;
  // map the K rows starting at it0 to edges and issue their loads (all K in flight)
  using ET = typename XEdge<PACKED>::T;
  auto map_load = [&](uint32_t it0, ET (&e)[K], uint32_t (&du)[K], uint32_t& valid) {
    int64_t ei[K];
    valid = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      ei[k] = 0;
      du[k] = 0;
      const uint32_t r0 = it0 + 32 * k;
      if (r0 >= len) continue;  // warp-uniform
      // the window must hold every entry of this row: refill at the entry holding r0
      const uint32_t last = __shfl_sync(0xffffffffu, w.endr, 31);
      if (last < min(r0 + 32, len)) {
        jb += __popc(__ballot_sync(0xffffffffu, w.endr <= r0));
        w = expand_window(X, xpre, hn, G, S, jb, a, len);
      }
      const uint32_t c0 = __popc(__ballot_sync(0xffffffffu, w.endr <= r0));  // entry of r0, relative
      const uint32_t x = w.endr - r0;
      const uint32_t heads = __reduce_or_sync(0xffffffffu, (x - 1u < 31u) ? (1u << x) : 0u);
      const uint32_t slot = c0 + __popc(heads & lanemask);
      const int64_t off = __shfl_sync(0xffffffffu, w.off, slot);
      const uint32_t d = __shfl_sync(0xffffffffu, w.du, slot);
      if (r0 + lane < len) {
        ei[k] = off + (int64_t)(a + r0 + lane);
        du[k] = d;
        valid |= 1u << k;
      }
    }
#pragma unroll
    for (int k = 0; k < K; ++k) {
      if constexpr (PACKED) e[k] = (valid >> k) & 1u ? ld_pedge(pedges + ei[k]) : 0u;
      else e[k] = (valid >> k) & 1u ? ld_edge(c.edges + ei[k]) : make_uint2(0, 0);
    }
  };
  auto col_of = [&](const ET& x) -> uint32_t {
    if constexpr (PACKED) return x & cmask; else return x.x;
  };
  auto w_of = [&](const ET& x) -> uint32_t {
    if constexpr (PACKED) return x >> colbits; else return x.y;
  };
  ET e[K];
  uint32_t du[K], valid;
  map_load(0, e, du, valid);
  for (uint32_t it0 = 0; it0 < len; it0 += 32 * K) {
    // the pre-reads of this batch (all K in flight) ...
    uint32_t old[K];
#pragma unroll
    for (int k = 0; k < K; ++k) old[k] = (valid >> k) & 1u ? ld_dist_tgt(c.dist + col_of(e[k])) : 0u;
    // ... while the next batch is mapped and its edge loads are issued
    ET en[K];
    uint32_t dn[K], vn = 0;
    if (it0 + 32 * K < len) map_load(it0 + 32 * K, en, dn, vn);
    TRACE(21);
    ne += __popc(valid);
#pragma unroll
    for (int k = 0; k < K; ++k) {
      if (!((valid >> k) & 1u)) continue;
      const uint32_t v = col_of(e[k]);
      const uint32_t nd = du[k] + w_of(e[k]);
      if (nd < du[k] || nd == kInf) {
        mark_overflow(c.ovfbits, c.ovf_cand, v);
        continue;
      }
      if (nd < old[k]) expand_push<FUSED>(c, v, nd);
    }
    TRACE(22);
    // the warp's far segment is flushed before the next batch could overflow it
    __syncwarp();
    if (c.s->wfar[warp] > (uint32_t)(kFarSeg / 2)) {  // warp-uniform
      warp_flush_far(c, c.farstage + warp * kFarSeg, min(c.s->wfar[warp], (uint32_t)kFarSeg));
      if (lane == 0) c.s->wfar[warp] = 0;
      __syncwarp();
    }
    TRACE(23);
#pragma unroll
    for (int k = 0; k < K; ++k) { e[k] = en[k]; du[k] = dn[k]; }
    valid = vn;
  }
}

// Relax every entry of a CTA-local bin (stage A, then stage B when high-degree
// vertices were found). Starts after and ends with a CTA barrier.
template <bool FUSED, bool LD = false, bool MIR = false>
__device__ __forceinline__ void process_bin(Ctx& c, Shared& s, const uint2* in, uint32_t nin,
                                            bool check_stale, uint32_t& nv, uint32_t& ne) {
  if (nin * 8 <= (uint32_t)kBlock) stage_small<FUSED, 1, LD, MIR>(c, in, nin, check_stale, nv, ne);
  else stage_small<FUSED, 4, LD, MIR>(c, in, nin, check_stale, nv, ne);
  __syncthreads();
  TRACE(4);
  if constexpr (LD) return;  // no high-degree list on a low-degree graph
  const uint32_t nb = min(s.bigtail, (uint32_t)kBigCap);
  if (c.collect && nb) {
    // expand collection: the CTA's list joins the group list with ONE atomicAdd (the whole
    // grid appends to one counter; a CAS reservation loop serialised the CTAs at one
    // success per L2 round trip). Readers clamp the counter to hubcap; the entries past
    // hubcap (possible only with hubs queued twice) are relaxed here.
    if (threadIdx.x == 0) {
      s.xbase = atomicAdd(c.hcount_next, nb);
      s.bigtail = 0;
    }
    __syncthreads();
    const uint32_t base = s.xbase;
    const uint32_t fit = base >= c.hubcap ? 0u : min(nb, c.hubcap - base);
    for (uint32_t i = threadIdx.x; i < fit; i += kBlock) {
      const BigEnt be = c.big[i];
      HubEnt he;
      he.beg = be.beg;
      he.deg = be.deg;
      he.du = be.du;
      c.hub_next[base + i] = he;
    }
    if (fit < nb) {  // block-uniform: move the tail to the front and relax it here
      constexpr int PER = kBigCap / kBlock;
      BigEnt t[PER];
#pragma unroll
      for (int k = 0; k < PER; ++k) {
        const uint32_t i = fit + threadIdx.x + k * kBlock;
        if (i < nb) t[k] = c.big[i];
      }
      __syncthreads();
#pragma unroll
      for (int k = 0; k < PER; ++k) {
        const uint32_t i = threadIdx.x + k * kBlock;
        if (fit + i < nb) c.big[i] = t[k];
      }
      __syncthreads();
      stage_big<FUSED, MIR>(c, s, nb - fit, ne);
    }
    __syncthreads();  // c.big is refilled by the next chunk
    TRACE(24);
    return;
  }
  if (nb) {
    __syncthreads();  // everyone has read bigtail
    if (threadIdx.x == 0) s.bigtail = 0;
    stage_big<FUSED, MIR>(c, s, nb, ne);
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

// ---------------------------------------------------------------------------------
// Async drain (KIND_FUSED_ASYNC; graphs whose every adjacency fits its ELL slot).
//
// The bucket-fusion drain without sub-round barriers: each CTA keeps a work ring in
// shared memory; warps claim up to 4 entries (one per octet), relax them and push the
// lowered current-bucket vertices straight back, so a vertex is relaxed as soon as it
// is lowered instead of at the next CTA barrier. Every ring entry carries the 64-byte
// ELL slot of its vertex, loaded by the producer IN PARALLEL with the atomicMin that
// lowered it; the next hop then starts from shared memory and a level of the
// dependent chain costs one L2 round trip (the atomic), not two (slot load, then
// atomic). Producers also prefetch into L2 the slots of the pushed vertex's
// neighbours (the hop after next).
//
// Ring protocol (positions are per phase, entry i = pos mod kRing, lap = pos/kRing+1):
//   state word hdr[i].w: 2*lap-1 = free for lap, 2*lap = written for lap,
//   2*lap+1 = consumed. A producer reserves positions (one shared atomic on `tail`),
//   waits for "free", writes the slot and {v, d, depth}, then release-stores
//   "written". A consumer claims positions below `tail` by CAS on `head`, waits for
//   "written" (acquire), reads, and marks the entries consumed once its loads that
//   use them have issued.
//   Admission: a push is accepted only while reserved-but-unclaimed entries
//   (tail - head) stay <= its limit, checked before reserving; concurrent pushers can
//   overshoot by < 16 warps x 32 lanes, and claimed-but-unread entries are < 64, so
//   limits <= kRingSafe keep every unread entry inside the ring (a producer never
//   waits on an entry nobody will read).
//   Termination: `done` starts at -(warps) and gains 1 per processed entry (after its
//   children are reserved) and 1 per warp that finished feeding; a warp that finds
//   nothing to claim and reads done == tail (done first) knows that no entry is in
//   flight and no push can follow.
// Threshold: a drain push that would make the local bucket (tail - head) reach T
// spills to the global frontier ("copied over to the global bucket",
// PAPER.md:595-596), processed in the next group-wide round: the paper's
// `size() < threshold` test on the CTA's local bucket.
// ---------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t lds_volatile(const uint32_t* p) {
  return *reinterpret_cast<const volatile uint32_t*>(p);
}
__device__ __forceinline__ void sts_volatile(uint32_t* p, uint32_t v) {
  *reinterpret_cast<volatile uint32_t*>(p) = v;
}
__device__ __forceinline__ uint32_t lds_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.cta.shared.u32 %0, [%1];" : "=r"(v) : "r"((uint32_t)__cvta_generic_to_shared(p)) : "memory");
  return v;
}
__device__ __forceinline__ void sts_release(uint32_t* p, uint32_t v) {
#ifdef GI_NO_FENCE
  *reinterpret_cast<volatile uint32_t*>(p) = v; return;
#endif
  asm volatile("st.release.cta.shared.u32 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(p)), "r"(v) : "memory");
}

#ifndef GI_MIN_BACKOFF
#define GI_MIN_BACKOFF 32
#endif
#ifndef GI_MAX_BACKOFF
#define GI_MAX_BACKOFF 256
#endif
constexpr uint32_t kMinBackoffNs = GI_MIN_BACKOFF, kMaxBackoffNs = GI_MAX_BACKOFF;

struct Ring {
  uint4* hdr;   // [kRing] {v, d, depth, state}
  uint4* slot;  // [kRing][4] the vertex's 64 B ELL slot
  uint4* wq;    // [warps][4][5] per-warp continuation queue: {v, d, depth, -} + slot
};

__device__ __forceinline__ void load_slot(const uint2* slots, uint32_t v, uint4 (&sl)[4]) {
  const uint4* p = reinterpret_cast<const uint4*>(slots + 8 * (size_t)v);
#pragma unroll
  for (int j = 0; j < 4; ++j) sl[j] = __ldg(p + j);
}

// Warp-aggregated push of (x, nd, dep, slot) for the lanes with `want`; called by all
// 32 lanes. FEED pushes may fill the ring; drain pushes respect the threshold T.
template <bool FEED>
__device__ __forceinline__ void ring_push(Ctx& c, Shared& s, const Ring& r, bool want, uint32_t x,
                                          uint32_t nd, uint32_t dep, const uint4 (&sl)[4],
                                          unsigned long long* tr = nullptr) {
  const uint32_t mask = __ballot_sync(0xffffffffu, want);
  if (!mask) return;
#ifdef GI_TRACE
  long long t0 = clock64();
#endif
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t cnt = __popc(mask);
  uint32_t acc = 0, base = 0;
  if (lane == 0) {
    const uint32_t lim = FEED ? (uint32_t)kRingSafe : c.T;
    const uint32_t h = lds_volatile(&s.head), t = lds_volatile(&s.tail);
    const uint32_t size = t - h;  // local bucket: reserved, not yet claimed
    acc = size + cnt < lim ? cnt : (size + 1 < lim ? lim - 1 - size : 0u);  // keep size < T
    if (acc) base = atomicAdd(&s.tail, acc);
  }
  acc = __shfl_sync(0xffffffffu, acc, 0);
  base = __shfl_sync(0xffffffffu, base, 0);
#ifdef GI_TRACE
  long long t1 = clock64();
  long long t2 = t1, t3 = t1;
#endif
  if (want) {
    const uint32_t rk = __popc(mask & ((1u << lane) - 1u));
    if (rk < acc) {
      const uint32_t pos = base + rk, i = pos & (kRing - 1), lap = (pos >> kRingLog) + 1;
      while (lds_volatile(&r.hdr[i].w) != 2 * lap - 1) {
      }
#ifdef GI_TRACE
      t2 = clock64();
#endif
#pragma unroll
      for (int j = 0; j < 4; ++j) r.slot[4 * i + j] = sl[j];
      r.hdr[i].x = x;
      r.hdr[i].y = nd;
      r.hdr[i].z = dep;
#ifdef GI_TRACE
      t3 = clock64();
#endif
      sts_release(&r.hdr[i].w, 2 * lap);  // slot + header visible before the state
#ifdef GI_TRACE
      if (tr) {
        const long long t4 = clock64();
        tr[0] += t1 - t0; tr[1] += t2 - t1; tr[2] += t3 - t2; tr[3] += t4 - t3; tr[4] += 1;
      }
#endif
    } else {
      if (!FEED) s.spilled = 1;
      push_global(c, (int32_t)x);  // over threshold: the next group-wide round takes it
    }
  }
}

// Drain the CTA's ring until it is empty and no warp is feeding or processing.
// Called by every warp (warp-uniform control flow).
//
// Continuation: of the current-bucket vertices a warp lowers, the first (up to) four
// stay with the warp — written with their slots into its private 4-entry queue `wq`
// and relaxed in its next iteration — and only the rest go to the shared ring for
// other warps. A dependent chain thus stays in one warp and a hop costs the atomic's
// round trip plus a warp-local hand-off, with no claim/publish between warps. A warp
// reports the ring entries it claimed as done only when the chains it grew from them
// have ended, so done == tail still means "nothing in flight anywhere".
// Continuation entries skip the staleness probe: the warp itself lowered them a hop
// ago; a duplicate entry of a vertex lowered again since is relaxed once more, which
// costs work but never correctness.
__device__ __forceinline__ void async_drain(Ctx& c, Shared& s, const Ring& r, uint4* wq, uint32_t& nv,
                                            uint32_t& ne) {
  const uint32_t lane = threadIdx.x & 31, oct = lane >> 3, sub = lane & 7;
  const uint32_t lt = (1u << lane) - 1u;
  uint32_t mydep = 0;
  uint32_t nloc = 0;  // continuation entries in wq (octets [0, nloc))
  uint32_t owed = 0;  // ring entries claimed whose chains have not ended yet
  uint32_t backoff = kMinBackoffNs;
  ITRACE_DECL();
  for (;;) {
    // top up the free octets from the shared ring (blocking only when idle)
    uint32_t h = 0, got = 0;
    if (lane == 0) {
      for (;;) {
        const uint32_t dn = lds_volatile(&s.done);  // before tail (see the protocol)
        const uint32_t t = lds_volatile(&s.tail);
        h = lds_volatile(&s.head);
        if ((int32_t)(t - h) <= 0) {
          got = (nloc == 0 && owed == 0 && dn == t) ? 0xFFFFFFFFu : 0u;  // all done / nothing claimable
          break;
        }
        const uint32_t k = min(4u - nloc, t - h);
        if (k == 0) break;
        if (atomicCAS(&s.head, h, h + k) == h) {
          got = k;
          break;
        }
        if (nloc) break;  // busy warp: do not fight over the ring
      }
    }
    got = __shfl_sync(0xffffffffu, got, 0);
    if (got == 0xFFFFFFFFu) break;
    if (nloc == 0 && got == 0) {
      if (owed) {  // this warp's chains have ended
        if (lane == 0) atomicAdd(&s.done, owed);
        owed = 0;
      }
      ITRACE_ADD(7, 1);
      // idle: back off so that polling does not steal shared-memory issue slots from
      // the warps on the chain
      __nanosleep(backoff);
      backoff = min(backoff * 2, (uint32_t)kMaxBackoffNs);
      continue;
    }
    backoff = kMinBackoffNs;
    h = __shfl_sync(0xffffffffu, h, 0);
    owed += got;
    ITRACE_ADD(8, 1);
    ITRACE_ADD(9, nloc + got);
    ITRACE_ADD(10, nloc);

    const bool local = oct < nloc;
    const bool ring_e = !local && oct < nloc + got;
    const bool mine = local || ring_e;
    const uint32_t pos = h + oct - nloc, i = pos & (kRing - 1), lap = (pos >> kRingLog) + 1;
    uint32_t v = 0, du = 0, dep = 0;
    uint2 e = make_uint2(kColEmpty, 0);
    if (local) {
      const uint4 hd = wq[5 * oct];
      v = hd.x; du = hd.y; dep = hd.z;
      e = reinterpret_cast<const uint2*>(wq + 5 * oct + 1)[sub];
    } else if (ring_e) {
      while (lds_acquire(&r.hdr[i].w) != 2 * lap) {
      }
      const uint4 hd = r.hdr[i];
      v = hd.x; du = hd.y; dep = hd.z;
      e = reinterpret_cast<const uint2*>(r.slot + 4 * i)[sub];
    }

    // relax edge `sub` of the vertex; the atomic, the neighbour's slot and (for ring
    // entries) the staleness probe of the vertex itself are all in flight together
    bool valid = mine && e.x != kColEmpty;
    const uint32_t nd = du + e.y;
    if (valid && (nd < du || nd == kInf)) {
      mark_overflow(c.ovfbits, c.ovf_cand, e.x);
      valid = false;
    }
    uint32_t old = 0, cu = kInf;
    uint4 sl[4];
    if (valid) old = atomicMin(c.dist + e.x, nd);
    if (valid) {
      load_slot(c.slots, e.x, sl);
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) sl[j] = make_uint4(kColEmpty, 0, kColEmpty, 0);
    }
    if (mine && sub == 0 && dep > 0) cu = ld_dist(c.dist + v);
    // every lane's ring / wq reads have completed (their values fed the loads above):
    // release the ring entries for the next lap without a fence; wq may be rewritten
    __syncwarp();
    if (ring_e && sub == 0) sts_volatile(&r.hdr[i].w, 2 * lap + 1);
    cu = __shfl_sync(0xffffffffu, cu, lane & 24);
    const bool stale = cu < du;  // a newer entry of v exists: its relaxations supersede these
    if (mine && !stale) {
      nv += sub == 0;
      ne += valid;
    }
    const bool imp = valid && !stale && nd < old;
    const uint32_t bk = fdiv(nd, c.div);
    const bool curp = imp && bk == c.b;
    const bool farp = imp && bk != c.b;  // bk > b: nd >= du >= bΔ

    // continuation: the first four lowered current-bucket vertices stay in this warp
    const uint32_t cm = __ballot_sync(0xffffffffu, curp);
    const uint32_t rk = __popc(cm & lt);
    const uint32_t keep = min(__popc(cm), 4u);
    if (curp && rk < keep) {
      uint4* q = wq + 5 * rk;
      q[0] = make_uint4(e.x, nd, dep + 1, 0);
#pragma unroll
      for (int j = 0; j < 4; ++j) q[1 + j] = sl[j];
    }
    ring_push<false>(c, s, r, curp && rk >= keep, e.x, nd, dep + 1, sl);
    if (curp) {  // the hop after next: neighbours' slots into L2
      mydep = max(mydep, dep + 1);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (sl[j].x < kColBig) prefetch_l2(c.slots + 8 * (size_t)sl[j].x);
        if (sl[j].z < kColBig) prefetch_l2(c.slots + 8 * (size_t)sl[j].z);
      }
    }
    {
      const uint32_t mk = __ballot_sync(0xffffffffu, farp);
      if (mk) {
        uint32_t base = 0;
        if (lane == 0) base = atomicAdd(&s.farcnt, __popc(mk));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (farp) {
          c.my_fmin = min(c.my_fmin, bk);
          const uint32_t p2 = base + __popc(mk & lt);
          if (p2 < (uint32_t)kFarStage) c.farstage[p2] = (int32_t)e.x;
          else push_far_global(c, (int32_t)e.x);
        }
      }
    }
    nloc = keep;
    __syncwarp();  // wq writes visible to the warp's next iteration
  }
  // max depth processed by this warp (an entry of depth k is what the BSP drain relaxes
  // in sub-round k)
  ITRACE_FLUSH();
  mydep = __reduce_max_sync(0xffffffffu, mydep);
  if (lane == 0 && mydep) atomicMax(&s.maxdep, mydep);
}

// Feed one phase's initial work into the ring: the extracted bucket (EXTRACT) or this
// CTA's slice of the global frontier (ROUND). Warp-uniform; ends by releasing the
// warp's `live` token, after which the warp joins the drain.
__device__ __forceinline__ void async_feed(Ctx& c, Shared& s, const Ring& r, bool extract,
                                           const int32_t* src_list, uint32_t* qbits_in, uint32_t lo,
                                           uint32_t hi, uint32_t& nlive) {
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t b = c.b;
  for (uint32_t i0 = lo + warp * 32; i0 < hi; i0 += kBlock) {
    const uint32_t i = i0 + lane;
    const bool in = i < hi;
    const int32_t v = in ? src_list[i] : 0;
    if (in && !extract) atomicAnd(&qbits_in[v >> 5], ~(1u << (v & 31)));
    const uint32_t d = in ? ld_dist(c.dist + v) : kInf;
    bool take;
    if (extract) {  // (d)+(a): partition the far pile by recomputed bucket
      const uint32_t bk = fdiv(d, c.div);
      if (in && bk <= b) atomicAnd(&c.farbits[v >> 5], ~(1u << (v & 31)));
      take = in && bk == b;  // bk < b: stale (already settled)
      if (in && bk > b) {
        c.my_fmin = min(c.my_fmin, bk);
        cg::coalesced_group g = cg::coalesced_threads();
        uint32_t base = 0;
        if (g.thread_rank() == 0) base = atomicAdd(c.fcount_live, g.size());
        base = g.shfl(base, 0);
        c.far_live[base + g.thread_rank()] = v;
      }
      nlive += take;
    } else {
      take = in;
    }
    uint4 sl[4];
    if (take) {
      load_slot(c.slots, (uint32_t)v, sl);
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) sl[j] = make_uint4(0, 0, 0, 0);
    }
    // EXTRACT entries are relaxed in "sub-round 1" of the BSP drain, ROUND entries in
    // the round itself (depth 0)
    ring_push<true>(c, s, r, take, (uint32_t)v, d, extract ? 1u : 0u, sl);
  }
  __syncwarp();
  if (lane == 0) atomicAdd(&s.done, 1u);  // this warp has finished feeding
}

template <int KIND>
__global__ void __launch_bounds__(kBlock, kMinBlocksPerSm) sssp_persistent(KArgs a) {
  constexpr bool FUSED = KIND != KIND_UNFUSED && KIND != KIND_UNFUSED_LD && KIND != KIND_UNFUSED_XP;
  constexpr bool ASYNC = KIND == KIND_FUSED_ASYNC;
  constexpr bool LOWDEG = KIND == KIND_UNFUSED_LD || KIND == KIND_FUSED_BSP_LD;
  // expand (and its split into expand_kernel) exists only in the kernels skewed graphs run:
  // compiled out of the low-degree and async kernels, whose registers it would take
  constexpr bool XP = KIND == KIND_UNFUSED_XP || KIND == KIND_FUSED_BSP_XP;
  // bsp: bins [2][kBinCap] uint2, high-degree list [kBigCap], its prefix [kBigCap], far staging
  // [kFarStage]; async: ring [kRing] (+ per-warp queues), far staging
  extern __shared__ uint2 s_dyn[];
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
  if constexpr (XP) {  // the mirror pre-read runs only in the XP kernels (read after a barrier)
    if (tid == 0) s.mirror = a.mirror;
  }

  // Batch: each group runs one query at a time; after the first (static: source gid) it
  // CLAIMS the next source, so that groups that drew cheap sources run more of them.
  for (int32_t si = (int32_t)gid; si < a.nsrc;) {
    uint32_t* dist = a.dist + (size_t)si * (size_t)n;
    const int32_t src = a.srcs[si];
    // split expand: this launch continues a single query stopped for an external expand
    const bool resuming = XP && a.resume != 0;

    // ---- init: Dist = {inf}, Dist[src] = 0; far pile = {src} ----
    if (!resuming) {
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
          if (GI_INIT_CS) __stcs(d4 + i, val); else d4[i] = val;
        }
        done = n4 * 4;
      }
      for (int64_t i = done + (int64_t)rank * kBlock + tid; i < n; i += (int64_t)G * kBlock)
        dist[i] = (i == src) ? 0u : kInf;
    }
    if (!resuming && rank == 0 && tid == 0) {
      for (int k = 0; k < 3; ++k) {
        ctl->qcount[k] = 0; ctl->fcount[k] = 0; ctl->fmin[k] = kInf; ctl->xlive[k] = 0; ctl->maxsub[k] = 0;
        ctl->hcount[k] = 0; ctl->qclaim[k] = 0; ctl->tdist[k] = kInf;
        ctl->lcount[k] = 0; ctl->lmin[k] = kInf;
      }
      ctl->fcount[0] = 1; ctl->fmin[0] = 0; ctl->ovf_cand = 0;
      ws.far[0][0] = src;
      atomicOr(&ws.farbits[src >> 5], 1u << (src & 31));
    }
    if (!resuming) group_barrier_r(ctl, G, a.rung);

    Ctx c;
    c.dist = dist; c.slots = a.slots; c.edges = a.edges; c.div = a.div;
    c.farbits = ws.farbits; c.ovfbits = ws.ovfbits; c.ovf_cand = &ctl->ovf_cand;
    c.big = reinterpret_cast<BigEnt*>(s_dyn + 2 * kBinCap);
    c.pre = reinterpret_cast<unsigned long long*>(c.big + kBigCap);
    c.s = &s;
    c.pre_read = a.pre_read != 0;
    c.lazy = !FUSED && a.lazy != 0;
    c.collect = false;
    c.hub_min = a.hub_min;
    c.h = a.h;

    c.hubcap = a.hubcap;
    c.T = T;
    c.farstage = ASYNC ? reinterpret_cast<int32_t*>(s_dyn + (kRing + (kBlock / 32) * 4) * 10)
                       : reinterpret_cast<int32_t*>(c.pre + kBigCap);
    Ring ring;
    ring.hdr = reinterpret_cast<uint4*>(s_dyn);
    ring.slot = ring.hdr + kRing;
    ring.wq = ring.slot + 4 * kRing;

    uint32_t nv = 0, ne = 0;                      // per thread (flushed per phase)
    unsigned long long tnv = 0, tne = 0;           // per thread, 64-bit totals
    unsigned long long subrounds = 0, spills = 0, scanned = 0;  // per CTA (thread 0)
    unsigned long long phases = 0, rounds = 0, buckets = 0, empty = 0, critical = 0;  // rank 0, thread 0
    unsigned long long sub_at_phase_start = 0;
    uint32_t p = 0, j = 0, b = 0, prev = MODE_NONE;
    // bucket window (a.window buckets; off: wend = inf): t = advances so far, the later pile
    // of advance t is later[t & 1] with counters lcount / lmin [t % 3]
    // (window_pile > 0: the window opens only once the far pile has shrunk to that size)
    uint32_t t = 0, wend = (XP && a.window && !a.window_pile) ? a.window : kInf;  // constants outside XP
    bool wbig = false;  // window_pile: the far pile has been larger than window_pile (thread 0)
    uint32_t last_b = kInf;  // bucket of the last extraction with live vertices (rank 0, thread 0)
    bool mid = false;  // resuming inside phase p, after its external expand / extraction
    bool xmid = false;  // ... after its external extraction: phase p was an EXTRACT phase
    bool xprev = false;  // the previous phase's extraction ran outside (its bucket went to q)
    if (resuming) {
      const KState* ks = ws.kst;
      // the host enqueues [expand, extract, resume] rounds ahead of knowing whether the
      // query stopped again: a resume with nothing pending (the query finished) is a no-op.
      // Every CTA reads the flag here; it is rewritten only at this segment's next stop or
      // at the query's end, both after group barriers.
      if (*reinterpret_cast<const volatile uint32_t*>(&ks->pending) == 0) return;
      p = ks->p; j = ks->j; b = ks->b; prev = ks->prev; last_b = ks->last_b;
      t = ks->t; wend = ks->wend; wbig = ks->wbig != 0;
      xmid = ks->rkind == 2;
      if (rank == 0 && tid == 0) {
        phases = ks->phases; rounds = ks->rounds; buckets = ks->buckets; empty = ks->empty; critical = ks->critical;
      }
      mid = true;
    }

    // split query (XP kernels): save the phase loop's state in KState and flush this
    // segment's statistics, before the kernel returns for an external expand (kind 1) of
    // phase p's group list (E edges, xn entries) or an external extraction (kind 2) of the
    // xn-entry far pile; the host runs it and resumes this kernel at phase p
    auto stop_for_outside = [&](unsigned long long E, uint32_t xn, uint32_t kind) {
      {
        const uint32_t w = tid >> 5;
        warp_flush_far(c, c.farstage + w * kFarSeg, min(s.wfar[w], (uint32_t)kFarSeg));
        const uint32_t fm = __reduce_min_sync(0xffffffffu, c.my_fmin);
        if ((tid & 31) == 0 && fm != kInf) atomicMin(&s.fmin, fm);
      }
      tnv += nv; tne += ne;
      const unsigned long long tv = block_sum(tnv, s);
      const unsigned long long te = block_sum(tne, s);
      if (tid == 0) {
        if (s.fmin != kInf) atomicMin(&ctl->fmin[j % 3], s.fmin);
        QStats* q = &a.qstats[si];
        atomicAdd(&q->vertices, tv);
        atomicAdd(&q->edges, te + (rank == 0 ? E : 0ull));  // the external expand's edges
        if (subrounds) atomicAdd(&q->subrounds, subrounds);
        if (spills) atomicAdd(&q->spills, spills);
        if (kind == 2 && rank == 0) scanned += xn;  // the external extraction's scan
        if (scanned) atomicAdd(&q->far_scanned, scanned);
        if (rank == 0) {
          KState* ks = ws.kst;
          ks->p = p; ks->j = j; ks->b = b; ks->prev = prev; ks->last_b = last_b;
          ks->phases = phases; ks->rounds = rounds; ks->buckets = buckets; ks->empty = empty;
          ks->critical = critical; ks->E = E; ks->xn = xn; ks->rkind = kind;
          ks->t = t; ks->wend = wend; ks->wbig = wbig ? 1u : 0u;
          __threadfence();
          ks->pending = kind;
        }
      }
      TRACE_FLUSH();
    };
    for (;;) {
      if (mid && tid == 0) {  // phase p continues: its list was relaxed outside, the bins are empty
        s.mode = MODE_ROUND; s.cnt = 0; s.hn = 0; s.wend = wend;
        s.cnt3[0] = 0; s.cnt3[1] = 0; s.bigtail = 0; s.farcnt = 0;
        for (int w = 0; w < kBlock / 32; ++w) s.wfar[w] = 0;
        s.fmin = kInf;
      }
      // ---- decide (identically in every CTA, from counters final at the barrier) ----
      if (tid == 0 && !mid) {
        // L2-coherent loads, all four in flight at once (ordered after the barrier's fence)
        const uint32_t xl = __ldcg(&ctl->xlive[j % 3]);
        const uint32_t qn = __ldcg(&ctl->qcount[p % 3]);
        const uint32_t hn = __ldcg(&ctl->hcount[p % 3]);
        const uint32_t fc = __ldcg(&ctl->fcount[j % 3]);
        const uint32_t fm = __ldcg(&ctl->fmin[j % 3]);
        if (p > 0 && rank == 0) critical += __ldcg(&ctl->maxsub[(p - 1) % 3]);
        if (prev == MODE_EXTRACT) {
          // a lazy schedule extracts a bucket once per round: it counts once
          // (an extraction that ran outside sent its bucket to the global frontier: the
          // next ROUND phase counts that round)
          if (xl) { if (b != last_b) ++buckets; last_b = b; if (FUSED && !xprev) ++rounds; } else { ++empty; }
        }
        uint32_t mode;
        s.hn = min(hn, a.hubcap);
        // bucket window: extract while the far pile's next bucket lies inside the window
        // [ws, wend); else advance it (rescan the later pile) or, with nothing waiting
        // there, move it to the far pile's next bucket without a phase
        const uint32_t lc = (XP && a.window) ? __ldcg(&ctl->lcount[t % 3]) : 0u;
        if (XP && a.window_pile && fc > a.window_pile) wbig = true;  // the tail comes after this
        s.lcnt = lc;
        if (qn > 0 || hn > 0) { mode = MODE_ROUND; s.cnt = qn; }
        else if (XP && a.window && wend == kInf && wbig && fc > 0 && fc <= a.window_pile && fm < kInf - a.window) {
          mode = MODE_EXTRACT; s.cnt = fc; s.b = fm;  // the window opens at this extraction
          wend = fm + a.window;
        } else if (fc > 0 && fm < wend) { mode = MODE_EXTRACT; s.cnt = fc; s.b = fm; }
        else if (XP && lc > 0) {
          const uint32_t lm = __ldcg(&ctl->lmin[t % 3]);
          const uint32_t ws0 = min(fc > 0 ? fm : kInf, lm);
          mode = MODE_ADVANCE; s.cnt = lc; s.ws = ws0;
          wend = ws0 >= kInf - a.window ? kInf : ws0 + a.window;
        } else if (XP && fc > 0) {
          mode = MODE_EXTRACT; s.cnt = fc; s.b = fm;
          wend = fm >= kInf - a.window ? kInf : fm + a.window;
        } else mode = MODE_DONE;
        s.wend = wend;
        // PPSP: entering bucket i with iΔ >= the best distance found
        // to the target ends the query — every vertex below iΔ is settled. The snapshot
        // of dist[target] is a slot every CTA wrote before the barrier (identical
        // decisions in all CTAs; a stale, larger snapshot only delays the stop a phase).
        if (a.target >= 0 && mode == MODE_EXTRACT && p > 0) {
          const uint32_t td = __ldcg(&ctl->tdist[(p - 1) % 3]);
          if (td != kInf && (uint64_t)fm * (uint64_t)a.div.d >= (uint64_t)td) mode = MODE_STOP;
        }
        s.mode = mode;
        s.cnt3[0] = 0;
        s.cnt3[1] = 0;
        s.bigtail = 0;
        s.farcnt = 0;
        for (int w = 0; w < kBlock / 32; ++w) s.wfar[w] = 0;
        s.fmin = kInf;
        if constexpr (ASYNC) {
          s.head = 0; s.tail = 0; s.done = 0u - (uint32_t)(kBlock / 32); s.maxdep = 0; s.spilled = 0;
        }
      }
      if constexpr (ASYNC) {  // every ring entry "free for lap 1"
        for (uint32_t i = tid; i < (uint32_t)kRing; i += kBlock) ring.hdr[i].w = 1;
      }
      __syncthreads();
      TRACE(5);
#ifdef GI_TRACE
      const long long t_busy0 = clock64();
      if (blockIdx.x == 0 && tid == 0 && p < (uint32_t)kTracePhases) {
        g_phase[4][p] = s.mode; g_phase[5][p] = s.cnt; g_phase[6][p] = s.hn;
      }
#endif
      const uint32_t mode = s.mode;
      if (mode == MODE_DONE) break;
      if (mode == MODE_STOP) {
        // PPSP early stop: the far pile still holds entries; clear their dedup bits so
        // that the workspace ends clean (every bitmap all-zero) for the next query
        const int32_t* pile = (j & 1) ? ws.far[1] : ws.far[0];
        const uint32_t fc = s.cnt;
        const uint32_t lo2 = (uint32_t)(((uint64_t)fc * rank) / G), hi2 = (uint32_t)(((uint64_t)fc * (rank + 1)) / G);
        for (uint32_t i = lo2 + tid; i < hi2; i += kBlock) {
          const int32_t v = pile[i];
          if (v >= 0) atomicAnd(&ws.farbits[v >> 5], ~(1u << (v & 31)));  // < 0: an expand chunk's hole
        }
        if (XP && ws.laterbits) {  // ... and the later pile's
          const int32_t* lp = ws.later[t & 1];
          const uint32_t lc = s.lcnt;
          const uint32_t lo3 = (uint32_t)(((uint64_t)lc * rank) / G), hi3 = (uint32_t)(((uint64_t)lc * (rank + 1)) / G);
          for (uint32_t i = lo3 + tid; i < hi3; i += kBlock) {
            const int32_t v = lp[i];
            atomicAnd(&ws.laterbits[v >> 5], ~(1u << (v & 31)));
          }
        }
        break;
      }
      const uint32_t cnt = s.cnt;
      if constexpr (XP) wend = s.wend;
      if (mode == MODE_EXTRACT) { ++j; b = s.b; }
      if (XP && mode == MODE_ADVANCE) ++t;
      if (rank == 0 && tid == 0 && !mid) {
        ctl->qcount[(p + 2) % 3] = 0;
        ctl->maxsub[(p + 2) % 3] = 0;
        ctl->hcount[(p + 2) % 3] = 0;
        ctl->qclaim[(p + 1) % 3] = 0;  // last used in phase p-2, which every CTA has left
        ctl->tdist[(p + 1) % 3] = kInf;  // written at the end of phase p+1
        if (mode == MODE_EXTRACT) {
          ctl->fcount[(j + 1) % 3] = 0; ctl->fmin[(j + 1) % 3] = kInf; ctl->xlive[(j + 1) % 3] = 0;
        }
        if (XP && mode == MODE_ADVANCE) {  // the later pile of advance t+1 (last read by advance t-1)
          ctl->lcount[(t + 1) % 3] = 0; ctl->lmin[(t + 1) % 3] = kInf;
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

      if constexpr (ASYNC) {
        // feed the extracted bucket / the global-frontier slice into the ring, then
        // drain it without sub-round barriers (bucket fusion)
        const bool ex = mode == MODE_EXTRACT;
        const int32_t* list = ex ? ((j & 1) ? ws.far[0] : ws.far[1]) : ((p & 1) ? ws.q[1] : ws.q[0]);
        uint32_t* qbits_in = (p & 1) ? ws.qbits[1] : ws.qbits[0];
        uint32_t nlive = 0;
        ITRACE_T(t_ph0);
        async_feed(c, s, ring, ex, list, qbits_in, lo, hi, nlive);
        TRACE(6);
        async_drain(c, s, ring, ring.wq + (tid >> 5) * 20, nv, ne);
#ifdef GI_TRACE
        __syncthreads();
        TRACE(11);
        if (tid == 0 && p < (uint32_t)kTracePhases) {
          atomicMax(&g_phase[0][p], (unsigned long long)(clock64() - t_ph0));
          atomicMax(&g_phase[1][p], (unsigned long long)s.maxdep);
        }
#endif
        if (ex) {
          const uint32_t tl = block_sum(nlive, s);
          if (tid == 0) {
            if (tl) atomicAdd(&ctl->xlive[j % 3], tl);
            scanned += hi - lo;
          }
        }
      } else if (mode == MODE_EXTRACT) {
        if constexpr (XP) {
          // split query, big pile: the partition runs outside as a streaming kernel
          // (extract_kernel), its bucket going to the global frontier; this kernel resumes
          // at phase p with empty bins
          if (a.xsplit_min && cnt >= a.xsplit_min) {
            stop_for_outside(0ull, cnt, 2u);
            return;
          }
        }
        // (d)+(a): partition the far pile by recomputed bucket.
        // kXtr entries per thread per chunk with every load in flight together; the
        // entries kept for later buckets are compacted with one global atomic per warp
        // per chunk (warp scan), not one per warp per entry.
        const int32_t* far_src = (j & 1) ? ws.far[0] : ws.far[1];
        uint32_t nlive = 0;
        uint32_t my_lmin = kInf;  // bucket window: min bucket sent to the later pile
        // a big pile (every CTA iterates many chunks): CTA-aggregated appends (cta_append)
        const bool agg = cnt >= 2u * G * kXtr * kBlock;
        for (uint32_t base = lo; base < hi; base += kXtr * kBlock) {
          int32_t v[kXtr];
          uint32_t d[kXtr];
#pragma unroll
          for (int x = 0; x < kXtr; ++x) {
            const uint32_t i = base + x * kBlock + tid;
            v[x] = i < hi ? far_src[i] : -1;
          }
#pragma unroll
          for (int x = 0; x < kXtr; ++x) d[x] = v[x] >= 0 ? ld_dist_x(dist + v[x]) : kInf;
          uint32_t keepm = 0;
          uint32_t livem = 0;
          uint32_t latm = 0;  // beyond the window and new to the later pile
#pragma unroll
          for (int x = 0; x < kXtr; ++x) {
            if (v[x] < 0) continue;
            const uint32_t bk = prio_bucket(d[x], c.h ? __ldg(c.h + v[x]) : 0u, c.div);
            if (bk <= b) {
              atomicAnd(&ws.farbits[v[x] >> 5], ~(1u << (v[x] & 31)));
              if (bk == b) { ++nlive; livem |= 1u << x; }  // else: stale (already settled)
            } else if (XP && bk >= wend) {  // (window off: wend = inf, never; XP kernels only)
              atomicAnd(&ws.farbits[v[x] >> 5], ~(1u << (v[x] & 31)));
              my_lmin = min(my_lmin, bk);
              const uint32_t bit = 1u << (v[x] & 31);
              if (!(atomicOr(&ws.laterbits[v[x] >> 5], bit) & bit)) latm |= 1u << x;
            } else {
              c.my_fmin = min(c.my_fmin, bk);
              keepm |= 1u << x;
            }
          }
          TRACE(26);
          if (agg) cta_append(keepm, v, c.far_live, c.fcount_live, s.redw, nullptr);
          else warp_append(keepm, v, c.far_live, c.fcount_live, nullptr);
          if (XP && wend != kInf) {  // CTA-uniform
            if (agg) cta_append(latm, v, ws.later[t & 1], &ctl->lcount[t % 3], s.redw, nullptr);
            else warp_append(latm, v, ws.later[t & 1], &ctl->lcount[t % 3], nullptr);
          }
          TRACE(27);
          // the extracted vertices: the CTA bin (fusion) while it has room, else — and
          // without fusion — the global frontier, deduplicated with all atomics in flight
          uint32_t ovm = FUSED ? 0u : livem;
          if constexpr (FUSED) {
            const uint32_t lane = tid & 31;
#pragma unroll
            for (int x = 0; x < kXtr; ++x) {
              const uint32_t m = __ballot_sync(0xffffffffu, (livem >> x) & 1u);
              if (!m) continue;
              uint32_t base = 0;
              if (lane == 0) base = atomicAdd(c.outcnt, (uint32_t)__popc(m));
              base = __shfl_sync(0xffffffffu, base, 0);
              if ((livem >> x) & 1u) {
                const uint32_t pos = base + __popc(m & ((1u << lane) - 1u));
                if (pos < (uint32_t)kBinCap) {
                  prefetch_own(c.slots + 8 * (size_t)v[x]);
                  c.out[pos] = make_uint2((uint32_t)v[x], d[x]);
                } else {
                  ovm |= 1u << x;
                }
              }
            }
          }
          if (agg || __any_sync(0xffffffffu, ovm != 0)) {  // agg: CTA-uniform
            uint32_t old[kXtr];
#pragma unroll
            for (int x = 0; x < kXtr; ++x)
              old[x] = ((ovm >> x) & 1u) ? atomicOr(&c.qbits_next[v[x] >> 5], 1u << (v[x] & 31)) : ~0u;
            uint32_t newm = 0;
#pragma unroll
            for (int x = 0; x < kXtr; ++x)
              if (((ovm >> x) & 1u) && !(old[x] & (1u << (v[x] & 31)))) newm |= 1u << x;
            if (agg) cta_append(newm, v, c.q_next, c.qcount_next, s.redw, GI_X_PFAGG ? c.slots : nullptr);
            else warp_append(newm, v, c.q_next, c.qcount_next, GI_X_PFXS ? c.slots : nullptr);
          }
          TRACE(28);
        }
        TRACE(6);
        if (XP && wend != kInf) {
          const uint32_t lm = __reduce_min_sync(0xffffffffu, my_lmin);
          if ((tid & 31) == 0 && lm != kInf) atomicMin(&ctl->lmin[t % 3], lm);
        }
        const uint32_t tl = block_sum(nlive, s);  // ends with a barrier: ring fill is final
        if (tid == 0) {
          if (tl) atomicAdd(&ctl->xlive[j % 3], tl);
          scanned += hi - lo;
        }
      } else if (XP && mode == MODE_ADVANCE) {
        // bucket window advance (only expand queries, hence the XP kernels, open a window):
        // the later pile of advance t-1 is partitioned against the new window [ws, wend):
        // settled entries dropped, entries inside the window moved to the far pile (the next
        // extraction's), the rest kept in the later pile of advance t
        const int32_t* lsrc = ws.later[(t - 1) & 1];
        const uint32_t ws0 = s.ws;
        uint32_t my_lmin = kInf;
        const bool agg = cnt >= 2u * G * kXtr * kBlock;
        for (uint32_t base = lo; base < hi; base += kXtr * kBlock) {
          int32_t v[kXtr];
          uint32_t d[kXtr];
#pragma unroll
          for (int x = 0; x < kXtr; ++x) {
            const uint32_t i = base + x * kBlock + tid;
            v[x] = i < hi ? lsrc[i] : -1;
          }
#pragma unroll
          for (int x = 0; x < kXtr; ++x) d[x] = v[x] >= 0 ? ld_dist_x(dist + v[x]) : kInf;
          uint32_t keepm = 0, movem = 0;
#pragma unroll
          for (int x = 0; x < kXtr; ++x) {
            if (v[x] < 0) continue;
            const uint32_t bk = prio_bucket(d[x], c.h ? __ldg(c.h + v[x]) : 0u, c.div);
            const uint32_t bit = 1u << (v[x] & 31);
            if (bk >= wend) {
              my_lmin = min(my_lmin, bk);
              keepm |= 1u << x;
              continue;
            }
            atomicAnd(&ws.laterbits[v[x] >> 5], ~bit);
            if (bk >= ws0 && !(atomicOr(&ws.farbits[v[x] >> 5], bit) & bit)) {  // else settled,
              c.my_fmin = min(c.my_fmin, bk);                                  // or in the pile
              movem |= 1u << x;
            }
          }
          if (agg) {
            cta_append(keepm, v, ws.later[t & 1], &ctl->lcount[t % 3], s.redw, nullptr);
            cta_append(movem, v, c.far_live, c.fcount_live, s.redw, nullptr);
          } else {
            warp_append(keepm, v, ws.later[t & 1], &ctl->lcount[t % 3], nullptr);
            warp_append(movem, v, c.far_live, c.fcount_live, nullptr);
          }
        }
        const uint32_t lm = __reduce_min_sync(0xffffffffu, my_lmin);
        if ((tid & 31) == 0 && lm != kInf) atomicMin(&ctl->lmin[t % 3], lm);
        if (tid == 0) scanned += hi - lo;
      } else if (!mid) {
        const uint32_t hn = s.hn;
        HubEnt* hub_in = (p & 1) ? ws.hub[1] : ws.hub[0];
        if (XP && a.expand) {
          // expand: this phase's high-degree frontier vertices join the hubs queued by the
          // previous phase in the group list, relaxed edge-balanced after the collection
          c.hub_min = kSlotEdges + 1;
          c.collect = true;
          c.hub_next = hub_in;
          c.hcount_next = &ctl->hcount[p % 3];
          // split: a phase may stop for an external expand, which would drop this CTA's bin —
          // the collection's current-bucket pushes go to the global frontier instead (a full bin)
          if (a.split && tid == 0) s.cnt3[0] = kBinCap;
        }
        // a group list relaxed slice-wise: every CTA relaxes its 1/G slice of every entry's
        // edges (stage B over the slices), so an entry costs ~deg/G per CTA
        auto hub_slices = [&](uint32_t hcnt) {
          for (uint32_t h0 = 0; h0 < hcnt; h0 += kBigCap) {
            const uint32_t nh = min((uint32_t)kBigCap, hcnt - h0);
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
            stage_big<FUSED, XP>(c, s, nh, ne);
            __syncthreads();
            TRACE(15);
          }
        };
        // hubs queued in the previous phase (no expand)
        if (!(XP && a.expand)) hub_slices(hn);
        // ROUND: relax the group's global frontier, one slice per CTA, staged through
        // bin 1 in chunks (pushes go to bin 0, which the drain below consumes)
        const int32_t* q_in = (p & 1) ? ws.q[1] : ws.q[0];
        uint32_t* qbits_in = (p & 1) ? ws.qbits[1] : ws.qbits[0];
        // Skewed graphs (a.dyn_claim): chunks are CLAIMED dynamically (one atomic per
        // chunk, the next claim in flight while the current chunk is relaxed), since equal
        // vertex slices are unequal work and a CTA that drew heavy vertices should claim
        // fewer chunks. The first chunk of every CTA is static (rank * claim), so a small
        // frontier costs no atomic. Otherwise: equal static slices (one pass per CTA,
        // every CTA busy — the latency-bound rounds of road graphs).
        uint2* stage = s_dyn + kBinCap;
        const uint32_t claim = a.dyn_claim ? max(32u, min((uint32_t)kMaxClaim, cnt / (kClaimsPerCta * G)))
                                           : (uint32_t)kBinCap;
        const uint64_t first = a.dyn_claim ? (uint64_t)G * claim : (uint64_t)cnt;
        const bool dyn = first < cnt;
        uint32_t* qclaim = &ctl->qclaim[p % 3];
        uint32_t next = 0;
        if (tid == 0) {
          s.claim = rank * claim;
          if (dyn) next = (uint32_t)first + atomicAdd(qclaim, claim);  // in flight during chunk 1
        }
        if (a.dyn_claim) __syncthreads();
        const uint32_t end = a.dyn_claim ? cnt : hi;
        uint32_t base_static = lo;
        for (;;) {
          const uint32_t base = a.dyn_claim ? s.claim : base_static;
          if (base >= end) break;
          const uint32_t chunk = a.dyn_claim ? min(claim, cnt - base) : min((uint32_t)kBinCap, hi - base);
          for (uint32_t i0 = 0; i0 < chunk; i0 += 4 * kBlock) {  // one pass: chunk <= kBinCap
            int32_t vv[4];
            uint32_t dd[4];
#pragma unroll
            for (int x = 0; x < 4; ++x) {
              const uint32_t i = i0 + x * kBlock + tid;
              vv[x] = i < chunk ? q_in[base + i] : -1;
            }
#pragma unroll
            for (int x = 0; x < 4; ++x) dd[x] = vv[x] >= 0 ? ld_dist(dist + vv[x]) : 0u;
#pragma unroll
            for (int x = 0; x < 4; ++x) {
              if (vv[x] < 0) continue;
              atomicAnd(&qbits_in[vv[x] >> 5], ~(1u << (vv[x] & 31)));
              stage[i0 + x * kBlock + tid] = make_uint2((uint32_t)vv[x], dd[x]);
            }
          }
          __syncthreads();
          TRACE(14);
          process_bin<FUSED, LOWDEG, XP>(c, s, stage, chunk, false, nv, ne);  // ends with a barrier
          if (a.dyn_claim) {
            if (tid == 0) {
              s.claim = dyn ? next : cnt;
              if (dyn && next < cnt) next = (uint32_t)first + atomicAdd(qclaim, claim);
            }
            __syncthreads();
            TRACE(25);
          } else {
            base_static = base + chunk;
          }
        }
        __syncthreads();
        if (XP && a.expand) {
          c.hub_min = a.hub_min;
          c.collect = false;
          c.hub_next = (p & 1) ? ws.hub[0] : ws.hub[1];
          c.hcount_next = &ctl->hcount[(p + 1) % 3];
          if (a.split && tid == 0) s.cnt3[0] = 0;  // nothing was written to the bin
          group_barrier_r(ctl, G, a.rung);  // the group list is complete
          ++phases;
          TRACE(19);
          if (tid == 0) s.xhn = min(__ldcg(&ctl->hcount[p % 3]), a.hubcap);
          __syncthreads();
          const uint32_t xn = s.xhn;
          if (xn) {
            expand_scan(hub_in, ws.xpre, ws.xtot, xn, G, rank, s);
            group_barrier_r(ctl, G, a.rung);  // slice prefixes and totals are final
            ++phases;
            if (tid < 32) {  // S[r] = sum of the slice totals before r
              unsigned long long carry = 0;
              if (tid == 0) s.xS[0] = 0;
              for (uint32_t b0 = 0; b0 < G; b0 += 32) {
                const uint32_t r = b0 + tid;
                unsigned long long v = r < G ? __ldcg(ws.xtot + r) : 0ull;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                  const unsigned long long t = __shfl_up_sync(0xffffffffu, v, o);
                  if (tid >= (uint32_t)o) v += t;
                }
                if (r < G) s.xS[r + 1] = carry + v;
                carry += __shfl_sync(0xffffffffu, v, 31);
              }
            }
            __syncthreads();
            TRACE(20);
            const unsigned long long E = s.xS[G];
            if (a.split && E >= a.split_min) {
              // a heavy list: save the phase loop's state and stop; the host runs
              // expand_kernel on the list and resumes this kernel at phase p (KState).
              // expand_kernel reads GLOBAL entry positions: this CTA's slice gets S[rank] added
              {
                const unsigned long long base = s.xS[rank];
                const uint32_t lo_x = (uint32_t)(((uint64_t)xn * rank) / G), hi_x = (uint32_t)(((uint64_t)xn * (rank + 1)) / G);
                if (base)
                  for (uint32_t i = lo_x + tid; i < hi_x; i += kBlock) ws.xpre[i] += base;
              }
              stop_for_outside(E, xn, 1u);
              return;
            }
#if GI_INKERNEL_EXPAND
            const uint64_t W = (uint64_t)G * (kBlock / 32), wg = (uint64_t)rank * (kBlock / 32) + (tid >> 5);
            const unsigned long long a0 = E * wg / W, b0 = E * (wg + 1) / W;
            if (a0 < b0) {
              if (a.pedges) expand_relax<FUSED, true>(c, hub_in, ws.xpre, xn, G, s.xS, a0, b0, a.pedges, a.colbits, ne);
              else expand_relax<FUSED, false>(c, hub_in, ws.xpre, xn, G, s.xS, a0, b0, a.pedges, a.colbits, ne);
            }
            __syncthreads();
#else
            // a light list: each CTA relaxes the whole entries of its own slice of the list
            // with the CTA-wide stage B (the edge-balanced loop inlined here spilled the
            // persistent kernel's registers; a stop for expand_kernel costs ~40 µs) — or, for
            // a list of a few entries (a lone hub of a million edges), every CTA a 1/G slice
            // of every entry
            if (xn <= 4 * G) {
              hub_slices(xn);
            } else {
              const uint32_t lo_x = (uint32_t)(((uint64_t)xn * rank) / G), hi_x = (uint32_t)(((uint64_t)xn * (rank + 1)) / G);
              for (uint32_t h0 = lo_x; h0 < hi_x; h0 += kBigCap) {
                const uint32_t nh = min((uint32_t)kBigCap, hi_x - h0);
                for (uint32_t i = tid; i < nh; i += kBlock) {
                  const uint4 he = __ldcg(reinterpret_cast<const uint4*>(hub_in + h0 + i));
                  BigEnt be;
                  be.beg = (int64_t)(((uint64_t)he.y << 32) | he.x);
                  be.deg = he.z;
                  be.du = he.w;
                  c.big[i] = be;
                }
                __syncthreads();
                stage_big<FUSED, XP>(c, s, nh, ne);
                __syncthreads();
              }
            }
#endif
            TRACE(18);
          }
        }
      }

      mid = false;
      if constexpr (FUSED && !ASYNC) {
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
            bulk_append(nin, [&](uint32_t i) { return (int32_t)in[i].x; }, c.qbits_next, c.q_next,
                        c.qcount_next, GI_X_PFG ? c.slots : nullptr);
            if (tid == 0) ++spills;
            break;
          }
          if (tid == 0) { s.cnt3[(k + 1) % 3] = 0; ++subrounds; }
          c.out = s_dyn + (k & 1) * kBinCap;
          c.outcnt = &s.cnt3[k % 3];
          process_bin<FUSED, LOWDEG, XP>(c, s, in, nin, true, nv, ne);
        }
      }

      // flush staged far-pile pushes (dedup + append), then the next-bucket lower
      // bound: warp min + one smem atomic per warp + one global atomic per CTA
      __syncthreads();
      TRACE(7);
      {
        if constexpr (ASYNC) {
          const uint32_t nf = min(s.farcnt, (uint32_t)kFarStage);
          const int32_t* fs = c.farstage;
          bulk_append(nf, [&](uint32_t i) { return fs[i]; }, c.farbits, c.far_live, c.fcount_live, nullptr);
        } else {  // each warp flushes its own segment
          const uint32_t w = tid >> 5;
          warp_flush_far(c, c.farstage + w * kFarSeg, min(s.wfar[w], (uint32_t)kFarSeg));
        }
        uint32_t fm = __reduce_min_sync(0xffffffffu, c.my_fmin);
        if ((tid & 31) == 0 && fm != kInf) atomicMin(&s.fmin, fm);
        __syncthreads();
        if (tid == 0 && s.fmin != kInf) atomicMin(&ctl->fmin[j % 3], s.fmin);
        if (ASYNC && tid == 0) {
          subrounds += s.maxdep;
          spills += s.spilled;
        }
        if (tid == 0 && a.target >= 0) atomicMin(&ctl->tdist[p % 3], ld_dist(dist + a.target));
        if (FUSED && tid == 0 && subrounds != sub_at_phase_start) {
          atomicMax(&ctl->maxsub[p % 3], (uint32_t)(subrounds - sub_at_phase_start));
          sub_at_phase_start = subrounds;
        }
      }
      tnv += nv; tne += ne; nv = 0; ne = 0;

      TRACE(8);
#ifdef GI_TRACE
      if (tid == 0 && p < (uint32_t)kTracePhases) {
        const unsigned long long busy = (unsigned long long)(clock64() - t_busy0);
        atomicMax(&g_phase[2][p], busy);
        atomicAdd(&g_phase[3][p], busy);
      }
#endif
      group_barrier_r(ctl, G, a.rung);
      TRACE(9);
      ++p;
      ++phases;
      prev = xmid ? (uint32_t)MODE_EXTRACT : mode;
      xprev = xmid;
      xmid = false;
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
            // PPSP stops early: only the target's distance is the result
            if (v < n && (a.target < 0 || v == a.target) && ld_dist(dist + v) == kInf) bad = 1;
          }
        }
      }
      if (__syncthreads_or(bad) && tid == 0) atomicOr(&a.qstats[si].overflow, 1u);
    }

    // ---- fused gather (gi_sssp_batch_peers): the finished row is written straight into
    // every other rank's result matrix (peer memory over NVLink), by this group's CTAs,
    // while the other groups keep computing — no separate all-gather after the batch ----
    if (a.npeers > 0) {
      for (int32_t pi = 0; pi < a.npeers; ++pi) {
        uint32_t* dst = a.peers[pi];
        if (dst == a.dist) continue;  // the rank's own matrix: computed in place
        dst += (size_t)si * (size_t)n;
        if (a.peer_vec) {
          const uint4* s4 = reinterpret_cast<const uint4*>(dist);
          uint4* d4 = reinterpret_cast<uint4*>(dst);
          for (int64_t i = (int64_t)rank * kBlock + tid; i < n / 4; i += (int64_t)G * kBlock) d4[i] = __ldcg(s4 + i);
        } else {
          for (int64_t i = (int64_t)rank * kBlock + tid; i < n; i += (int64_t)G * kBlock) dst[i] = ld_dist(dist + i);
        }
      }
      __threadfence_system();
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
    if (rank == 0 && tid == 0) ctl->next_si = a.ngroups + (int32_t)atomicAdd(a.src_next, 1u);
    if (XP && rank == 0 && tid == 0) ws.kst->pending = 0;  // the split query is finished
    group_barrier_r(ctl, G, a.rung);  // the next query re-initialises ctl
    if (tid == 0) s.cnt = (uint32_t)__ldcg(&ctl->next_si);
    __syncthreads();
    si = (int32_t)s.cnt;
    __syncthreads();  // s.cnt is rewritten by the next query's first decision
  }
  TRACE_FLUSH();
}

#if GI_BLOCK >= 1024
// The external expand of a split query (KState): the edge-balanced relaxation of phase p's
// group list, launched by the host between two segments of the persistent kernel. It is
// written without the persistent kernel's context so that the edge loop keeps only what it
// uses in registers: the window of 32 list entries, K rows of packed edges in flight, the
// pre-read distances. Improving candidates are written with red.min and staged per warp in
// shared memory — future buckets for the far pile, the current bucket for the global
// frontier — and flushed with the dedup test-and-set and one append atomic per warp.
constexpr int kXSeg = 512;     // far staging entries per warp (flushed above half)
constexpr int kXCur = 64;      // current-bucket staging entries per warp (rare on skewed graphs)
#ifndef GI_XROWS
#define GI_XROWS 8
#endif
constexpr int kXRows = GI_XROWS;  // rows of 32 edges per warp per iteration

// the pointers of expand_kernel's cold paths (pushes, flushes, overflow), read from shared
// memory where used so that the edge loop keeps only its own values in registers
struct XPtrs {
  uint32_t* farbits;
  int32_t* far_live;
  uint32_t* fcount;
  uint32_t* qbits;
  int32_t* q;
  uint32_t* qcount;
  uint32_t* ovfbits;
  uint32_t* ovf_cand;
  const uint2* slots;
  const uint32_t* h;
  FastDiv div;
  uint32_t bcur;
};

struct XShared {
  int32_t far[kBlock / 32][kXSeg];
  int32_t cur[kBlock / 32][kXCur];
  uint2 cand[kBlock / 32][32 * kXRows];  // a block's candidates past the mirror, compacted (v, nd)
  uint32_t nfar[kBlock / 32], ncur[kBlock / 32];
  XPtrs ps;
};

// dedup-append of a warp's staged vertices (bits = dedup bitmap) to a global list: the
// test-and-sets of the whole segment first (4 per lane in flight per round), then ONE warp
// scan and ONE append atomic for the segment — every warp of the GPU appends to the same
// counter, which serialises same-word atomics (~150 M/s)
__device__ __forceinline__ void xflush(const int32_t* seg, uint32_t n, uint32_t* bits, int32_t* list,
                                       uint32_t* count, const uint2* slots_pf) {
  const uint32_t lane = threadIdx.x & 31;
  uint32_t newm = 0;  // bit r*4+x: entry (r*128 + x*32 + lane) is new (n <= 1024)
  for (uint32_t r = 0; r * 128 < n; ++r) {
    int32_t v[4];
    uint32_t old[4];
#pragma unroll
    for (int x = 0; x < 4; ++x) {
      const uint32_t i = r * 128 + x * 32 + lane;
      v[x] = i < n ? seg[i] : -1;
    }
#pragma unroll
    for (int x = 0; x < 4; ++x) old[x] = v[x] >= 0 ? atomicOr(&bits[v[x] >> 5], 1u << (v[x] & 31)) : ~0u;
#pragma unroll
    for (int x = 0; x < 4; ++x)
      if (v[x] >= 0 && !(old[x] & (1u << (v[x] & 31)))) newm |= 1u << (r * 4 + x);
  }
  const uint32_t nk = __popc(newm);
  uint32_t incl = nk;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= (uint32_t)o) incl += t;
  }
  const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
  if (tot) {
    uint32_t base = 0;
    if (lane == 0) base = atomicAdd(count, tot);
    base = __shfl_sync(0xffffffffu, base, 0);
    uint32_t off = base + incl - nk;
    while (newm) {
      const int b = __ffs(newm) - 1;
      newm &= newm - 1;
      const int32_t v = seg[(b >> 2) * 128 + (b & 3) * 32 + lane];
      if (slots_pf) prefetch_l2(slots_pf + 8 * (size_t)v);
      list[off++] = v;
    }
  }
  __syncwarp();
}

// The list entries carry GLOBAL start positions here (xpre + S, added by the persistent
// kernel before it stopped): lane k of a window holds entry jb+k's end relative to the warp's
// range start, beg - start, and du.
//
// MIRROR (KArgs.mirror): the pre-read is the vertex's byte in the mirror (n bytes, L2-resident)
// instead of dist[v] (4n bytes, twice the L2 on config 4, so most pre-reads went to DRAM). A
// candidate passes when it could improve (nd < mirror[v], or the byte is 0xFF: unknown); a
// passing candidate takes atomicMin, whose old value decides the push exactly as the
// pre-read did (R11 without the race: the improving thread knows it improved). The byte is
// then set to the new distance, or tightened to the old one: both are values dist[v] held,
// so the invariant dist[v] <= mirror[v] survives racing byte stores.
template <bool PACKED, bool MIRROR>
__global__ void __launch_bounds__(kBlock, 1) expand_kernel(KArgs a) {
  extern __shared__ __align__(16) unsigned char x_dyn[];
  XShared& xs = *reinterpret_cast<XShared*>(x_dyn);
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // enqueued speculatively (see the host's segment loop): a no-op unless the persistent
  // kernel stopped for an expand (KState.pending == 1, cleared by the resumed kernel)
  if (*reinterpret_cast<const volatile uint32_t*>(&a.groups[0].kst->pending) != 1) return;
  if (tid == 0) {
    const GroupWs& ws = a.groups[0];
    const KState* ks = ws.kst;
    const uint32_t p = ks->p, j = ks->j;
    XPtrs& ps = xs.ps;
    ps.farbits = ws.farbits;
    ps.far_live = (j & 1) ? ws.far[1] : ws.far[0];
    ps.fcount = &ws.ctl->fcount[j % 3];
    ps.qbits = (p & 1) ? ws.qbits[0] : ws.qbits[1];
    ps.q = (p & 1) ? ws.q[0] : ws.q[1];
    ps.qcount = &ws.ctl->qcount[(p + 1) % 3];
    ps.ovfbits = ws.ovfbits;
    ps.ovf_cand = &ws.ctl->ovf_cand;
    ps.slots = a.slots;
    ps.h = a.h;
    ps.div = a.div;
    ps.bcur = ks->b;
  }
  if (lane == 0) { xs.nfar[warp] = 0; xs.ncur[warp] = 0; }
  __syncthreads();
  const KState* ks = a.groups[0].kst;
  const uint32_t hn = ks->xn;
  const unsigned long long E = ks->E;
  const HubEnt* X = (ks->p & 1) ? a.groups[0].hub[1] : a.groups[0].hub[0];
  const unsigned long long* xpre = a.groups[0].xpre;
  uint32_t* const dist = a.dist;
  const uint32_t colbits = a.colbits;
  const uint32_t cmask = colbits >= 32 ? 0xFFFFFFFFu : (1u << colbits) - 1u;
  const bool lazy = a.lazy != 0;
  uint32_t my_fmin = kInf;
  auto flush_far = [&]() {
    __syncwarp();
    const XPtrs& ps = xs.ps;
    xflush(xs.far[warp], min(xs.nfar[warp], (uint32_t)kXSeg), ps.farbits, ps.far_live, ps.fcount, nullptr);
    if (lane == 0) xs.nfar[warp] = 0;
    __syncwarp();
  };
  auto flush_cur = [&]() {
    __syncwarp();
    const XPtrs& ps = xs.ps;
    xflush(xs.cur[warp], min(xs.ncur[warp], (uint32_t)kXCur), ps.qbits, ps.q, ps.qcount, GI_X_PFXC ? ps.slots : nullptr);
    if (lane == 0) xs.ncur[warp] = 0;
    __syncwarp();
  };

  const uint64_t W = (uint64_t)gridDim.x * (kBlock / 32), wg = (uint64_t)blockIdx.x * (kBlock / 32) + warp;
  const unsigned long long a0 = E * wg / W, b0 = E * (wg + 1) / W;
  if (a0 < b0) {
    const uint32_t len = (uint32_t)(b0 - a0);
    // the entry holding position a0: the largest i with xpre[i] <= a0 (32-ary search)
    uint32_t ilo = 0, ihi = hn;
    while (ihi - ilo > 32) {
      const uint32_t step = (ihi - ilo + 31) / 32;
      const uint32_t idx = ilo + lane * step;
      const bool pr = idx < ihi && __ldcg(xpre + idx) <= a0;
      ilo += (__popc(__ballot_sync(0xffffffffu, pr)) - 1) * step;
      ihi = min(ilo + step, ihi);
    }
    {
      const uint32_t idx = ilo + lane;
      const bool pr = idx < ihi && __ldcg(xpre + idx) <= a0;
      ilo += __popc(__ballot_sync(0xffffffffu, pr)) - 1;
    }
    uint32_t jb = ilo;
    uint32_t endr;
    int64_t off;
    uint32_t wdu;
    auto window = [&]() {
      const uint32_t idx = jb + lane;
      endr = len; off = 0; wdu = 0;
      if (idx < hn) {
        const uint4 he = __ldcg(reinterpret_cast<const uint4*>(X + idx));  // {beg lo, beg hi, deg, du}
        const unsigned long long start = __ldcg(xpre + idx), end = start + he.z;
        endr = end <= a0 ? 0u : (uint32_t)min(end - a0, (unsigned long long)len);
        off = (int64_t)(((uint64_t)he.y << 32) | he.x) - (int64_t)start;
        wdu = he.w;
      }
    };
    window();
    const uint32_t lanemask = (2u << lane) - 2u;
    // an improved vertex: staged per warp — future buckets for the far pile, the current
    // bucket for the global frontier; a full segment (at most one iteration past half)
    // takes the lane's own dedup push to the global list
    auto push_one = [&](uint32_t vv, uint32_t nd) {
      const XPtrs& ps = xs.ps;
      const uint32_t bk = ps.h ? max(prio_bucket(nd, __ldg(ps.h + vv), ps.div), ps.bcur) : fdiv(nd, ps.div);
      const bool cur = bk == ps.bcur && !lazy;
      if (!cur) my_fmin = min(my_fmin, bk);
      const uint32_t pos = atomicAdd(cur ? &xs.ncur[warp] : &xs.nfar[warp], 1u);
      if (pos < (uint32_t)(cur ? kXCur : kXSeg)) {
        (cur ? xs.cur[warp] : xs.far[warp])[pos] = (int32_t)vv;
      } else {
        uint32_t* bits = cur ? ps.qbits : ps.farbits;
        const uint32_t bit = 1u << (vv & 31);
        if (!(atomicOr(&bits[vv >> 5], bit) & bit)) {
          const uint32_t q = atomicAdd(cur ? ps.qcount : ps.fcount, 1u);
          (cur ? ps.q : ps.far_live)[q] = (int32_t)vv;
        }
      }
    };
    for (uint32_t it0 = 0; it0 < len; it0 += 32 * kXRows) {
      int64_t ei[kXRows];
      uint32_t du[kXRows], valid = 0;
#pragma unroll
      for (int k = 0; k < kXRows; ++k) {
        ei[k] = 0;
        du[k] = 0;
        const uint32_t r0 = it0 + 32 * k;
        if (r0 >= len) continue;  // warp-uniform
        const uint32_t last = __shfl_sync(0xffffffffu, endr, 31);
        if (last < min(r0 + 32, len)) {
          jb += __popc(__ballot_sync(0xffffffffu, endr <= r0));
          window();
        }
        const uint32_t c0 = __popc(__ballot_sync(0xffffffffu, endr <= r0));
        const uint32_t x = endr - r0;
        const uint32_t heads = __reduce_or_sync(0xffffffffu, (x - 1u < 31u) ? (1u << x) : 0u);
        const uint32_t slot = c0 + __popc(heads & lanemask);
        const int64_t o = __shfl_sync(0xffffffffu, off, slot);
        const uint32_t d = __shfl_sync(0xffffffffu, wdu, slot);
        if (r0 + lane < len) {
          ei[k] = o + (int64_t)(a0 + r0 + lane);
          du[k] = d;
          valid |= 1u << k;
        }
      }
      uint32_t v[kXRows], wt[kXRows], old[kXRows];
#pragma unroll
      for (int k = 0; k < kXRows; ++k) {
        if constexpr (PACKED) {
          const uint32_t pe = (valid >> k) & 1u ? ld_pedge(a.pedges + ei[k]) : 0u;
          v[k] = pe & cmask;
          wt[k] = pe >> colbits;
        } else {
          const uint2 e = (valid >> k) & 1u ? ld_edge(a.edges + ei[k]) : make_uint2(0, 0);
          v[k] = e.x;
          wt[k] = e.y;
        }
      }
      if constexpr (MIRROR) {
        // mirror bytes first (L2 hits), then atomicMin for the candidates that pass; the
        // others take no dist access at all
        uint32_t mb[kXRows];
#pragma unroll
        for (int k = 0; k < kXRows; ++k) mb[k] = (valid >> k) & 1u ? ld_mirror(a.mirror + v[k]) : 0u;
        uint32_t passm = 0, keep = 0;  // candidates to atomicMin; those plus overflows
#pragma unroll
        for (int k = 0; k < kXRows; ++k) {
          const uint32_t nd = du[k] + wt[k];
          const bool ovf = nd < du[k] || nd == kInf;
          if ((valid >> k) & 1u) {
            if (ovf) keep |= 1u << k;
            else if (mb[k] == 0xFFu || nd < mb[k]) passm |= 1u << k;
          }
        }
        valid = keep | passm;
        // most rows of a hub phase end here: no lane holds a candidate the mirror lets through
        if (GI_X_XSKIP && !__any_sync(0xffffffffu, valid != 0u)) goto rows_done;
        if constexpr (GI_X_XCOMPACT) {
          // the block's candidates (a few of its 32 x kXRows edges) are compacted into the
          // warp's buffer and relaxed densely, instead of kXRows predicated passes
          if (__any_sync(0xffffffffu, keep != 0u)) {  // overflowing candidates (rare)
            const XPtrs& ps = xs.ps;
#pragma unroll
            for (int k = 0; k < kXRows; ++k)
              if ((keep >> k) & 1u) {
                atomicOr(&ps.ovfbits[v[k] >> 5], 1u << (v[k] & 31));
                atomicOr(ps.ovf_cand, 1u);
              }
          }
          const uint32_t lt = (1u << lane) - 1u;
          uint32_t nc = 0;
#pragma unroll
          for (int k = 0; k < kXRows; ++k) {
            const uint32_t m = __ballot_sync(0xffffffffu, (passm >> k) & 1u);
            if ((passm >> k) & 1u) xs.cand[warp][nc + __popc(m & lt)] = make_uint2(v[k], du[k] + wt[k]);
            nc += __popc(m);
          }
          __syncwarp();
          for (uint32_t i0 = 0; i0 < nc; i0 += 64) {  // two candidates per lane in flight
            const bool h0 = i0 + lane < nc, h1 = i0 + 32 + lane < nc;
            const uint2 c0 = h0 ? xs.cand[warp][i0 + lane] : make_uint2(0, 0);
            const uint2 c1 = h1 ? xs.cand[warp][i0 + 32 + lane] : make_uint2(0, 0);
            const uint32_t o0 = h0 ? atomicMin(dist + c0.x, c0.y) : 0u;
            const uint32_t o1 = h1 ? atomicMin(dist + c1.x, c1.y) : 0u;
            if (h0 && c0.y < o0) {
              if (c0.y < 0xFFu) st_mirror(a.mirror + c0.x, c0.y);
              push_one(c0.x, c0.y);
            }
            if (h1 && c1.y < o1) {
              if (c1.y < 0xFFu) st_mirror(a.mirror + c1.x, c1.y);
              push_one(c1.x, c1.y);
            }
          }
          __syncwarp();  // the buffer is refilled by the next block
          goto rows_done;
        }
#pragma unroll
        for (int k = 0; k < kXRows; ++k) old[k] = (passm >> k) & 1u ? atomicMin(dist + v[k], du[k] + wt[k]) : 0u;
#pragma unroll
        for (int k = 0; k < kXRows; ++k) {
          if (!((passm >> k) & 1u)) continue;
          const uint32_t nd = du[k] + wt[k];
          if (nd < old[k]) {
            if (nd < 0xFFu) st_mirror(a.mirror + v[k], nd);
          } else {
            if (old[k] < mb[k]) st_mirror(a.mirror + v[k], old[k]);  // tighten (old < 0xFF)
            valid &= ~(1u << k);
          }
        }
      } else {
#pragma unroll
        for (int k = 0; k < kXRows; ++k) old[k] = (valid >> k) & 1u ? ld_dist_tgt(dist + v[k]) : 0u;
      }
#pragma unroll
      for (int k = 0; k < kXRows; ++k) {
        const uint32_t nd = du[k] + wt[k];
        const bool ovf = nd < du[k] || nd == kInf;
        if (((valid >> k) & 1u) && (ovf || MIRROR || nd < old[k])) {
          const XPtrs& ps = xs.ps;
          if (ovf) {  // inline: no call in this loop
            atomicOr(&ps.ovfbits[v[k] >> 5], 1u << (v[k] & 31));
            atomicOr(ps.ovf_cand, 1u);
            continue;
          }
          if constexpr (!MIRROR) red_min(dist + v[k], nd);
          push_one(v[k], nd);
        }
      }
    rows_done:
      __syncwarp();
      if (xs.nfar[warp] > (uint32_t)(kXSeg / 2)) flush_far();
      if (xs.ncur[warp] > (uint32_t)(kXCur / 2)) flush_cur();
    }
  }
  flush_far();
  flush_cur();
  const uint32_t fm = __reduce_min_sync(0xffffffffu, my_fmin);
  if (lane == 0 && fm != kInf) atomicMin(&a.groups[0].ctl->fmin[ks->j % 3], fm);
}

// The external extraction of a split query (KState.pending == 2): phase p's partition of
// the far pile by recomputed bucket, (d)+(a) as a streaming
// kernel — the persistent kernel's in-phase extraction keeps 4 entries per thread in flight
// between CTA barriers and same-word appends; here every CTA takes tiles of kETile entries,
// all loads of a tile in flight together, and appends with ONE atomic per list per tile.
// An entry of bucket b joins the global frontier of phase p+1 (the pile holds a vertex at
// most once, so no dedup test is needed); a later bucket is kept in the live pile and
// min-reduced into the next bucket bound; an earlier one is stale and dropped. The dedup
// bit of every leaving entry is cleared.
#ifndef GI_EPER
#define GI_EPER 8
#endif
#ifndef GI_EMINB
#define GI_EMINB 1
#endif
constexpr int kEBlock = 512;
constexpr int kEPer = GI_EPER;  // entries per thread per tile, all their loads in flight together
constexpr uint32_t kETile = kEBlock * kEPer;

__global__ void __launch_bounds__(kEBlock, GI_EMINB) extract_kernel(KArgs a) {
  __shared__ uint32_t s_keep[kEBlock / 32], s_live[kEBlock / 32], s_lat[kEBlock / 32];
  __shared__ uint32_t s_fmin, s_nlive, s_lmin;
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const GroupWs& ws = a.groups[0];
  const KState* ks = ws.kst;
  // enqueued speculatively: a no-op unless the persistent kernel stopped for an extraction
  if (*reinterpret_cast<const volatile uint32_t*>(&ks->pending) != 2) return;
  const uint32_t p = ks->p, j = ks->j, b = ks->b, cnt = ks->xn;
  // bucket window: entries of buckets >= wend go to the later pile of advance t
  const uint32_t wend = ks->wend, t = ks->t;
  int32_t* later = ws.laterbits ? ws.later[t & 1] : nullptr;
  uint32_t* lcount = &ws.ctl->lcount[t % 3];
  const int32_t* far_src = (j & 1) ? ws.far[0] : ws.far[1];
  int32_t* far_live = (j & 1) ? ws.far[1] : ws.far[0];
  uint32_t* fcount_live = &ws.ctl->fcount[j % 3];
  int32_t* q_next = (p & 1) ? ws.q[0] : ws.q[1];
  uint32_t* qcount_next = &ws.ctl->qcount[(p + 1) % 3];
  const uint32_t* dist = a.dist;
  if (tid == 0) { s_fmin = kInf; s_nlive = 0; s_lmin = kInf; }
  uint32_t my_fmin = kInf, my_lmin = kInf;
  for (uint32_t t0 = blockIdx.x * kETile; t0 < cnt; t0 += gridDim.x * kETile) {
    int32_t v[kEPer];
    uint32_t d[kEPer], hv[kEPer];
#pragma unroll
    for (int x = 0; x < kEPer; ++x) {
      const uint32_t i = t0 + x * kEBlock + tid;
      v[x] = i < cnt ? __ldcs(far_src + i) : -1;  // read once
    }
#pragma unroll
    for (int x = 0; x < kEPer; ++x) d[x] = v[x] >= 0 ? ld_dist_x(dist + v[x]) : kInf;
#pragma unroll
    for (int x = 0; x < kEPer; ++x) hv[x] = (a.h && v[x] >= 0) ? __ldg(a.h + v[x]) : 0u;
    uint32_t keepm = 0, livem = 0, latm = 0;
#pragma unroll
    for (int x = 0; x < kEPer; ++x) {
      if (v[x] < 0) continue;
      const uint32_t bk = prio_bucket(d[x], hv[x], a.div);
      if (bk <= b) {
        atomicAnd(&ws.farbits[v[x] >> 5], ~(1u << (v[x] & 31)));
        if (bk == b) livem |= 1u << x;  // else: stale (already settled)
      } else if (bk >= wend) {  // beyond the window (off: wend = inf, never)
        atomicAnd(&ws.farbits[v[x] >> 5], ~(1u << (v[x] & 31)));
        my_lmin = min(my_lmin, bk);
        const uint32_t bit = 1u << (v[x] & 31);
        if (!(atomicOr(&ws.laterbits[v[x] >> 5], bit) & bit)) latm |= 1u << x;
      } else {
        my_fmin = min(my_fmin, bk);
        keepm |= 1u << x;
      }
    }
    // per-warp counts, one reservation per list per tile
    uint32_t km[kEPer], lm[kEPer], am[kEPer], kpre[kEPer], lpre[kEPer], apre[kEPer], kt = 0, lt = 0, at = 0;
#pragma unroll
    for (int x = 0; x < kEPer; ++x) {
      km[x] = __ballot_sync(0xffffffffu, (keepm >> x) & 1u);
      lm[x] = __ballot_sync(0xffffffffu, (livem >> x) & 1u);
      am[x] = __ballot_sync(0xffffffffu, (latm >> x) & 1u);
      kpre[x] = kt; lpre[x] = lt; apre[x] = at;
      kt += __popc(km[x]); lt += __popc(lm[x]); at += __popc(am[x]);
    }
    if (lane == 0) { s_keep[warp] = kt; s_live[warp] = lt; s_lat[warp] = at; }
    __syncthreads();
    if (tid < 32) {
      const uint32_t k0 = tid < kEBlock / 32 ? s_keep[tid] : 0u, l0 = tid < kEBlock / 32 ? s_live[tid] : 0u;
      const uint32_t a0 = tid < kEBlock / 32 ? s_lat[tid] : 0u;
      uint32_t ki = k0, li = l0, ai = a0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t a1 = __shfl_up_sync(0xffffffffu, ki, o), a2 = __shfl_up_sync(0xffffffffu, li, o);
        const uint32_t a3 = __shfl_up_sync(0xffffffffu, ai, o);
        if (tid >= (uint32_t)o) { ki += a1; li += a2; ai += a3; }
      }
      const uint32_t ktot = __shfl_sync(0xffffffffu, ki, 31), ltot = __shfl_sync(0xffffffffu, li, 31);
      const uint32_t atot = __shfl_sync(0xffffffffu, ai, 31);
      uint32_t kb = 0, lb = 0, ab = 0;
      if (tid == 0) {
        if (ktot) kb = atomicAdd(fcount_live, ktot);
        if (ltot) { lb = atomicAdd(qcount_next, ltot); s_nlive += ltot; }
        if (atot) ab = atomicAdd(lcount, atot);
      }
      kb = __shfl_sync(0xffffffffu, kb, 0);
      lb = __shfl_sync(0xffffffffu, lb, 0);
      ab = __shfl_sync(0xffffffffu, ab, 0);
      if (tid < kEBlock / 32) { s_keep[tid] = kb + ki - k0; s_live[tid] = lb + li - l0; s_lat[tid] = ab + ai - a0; }
    }
    __syncthreads();
    const uint32_t kw = s_keep[warp], lw = s_live[warp], aw = s_lat[warp], ltm = (1u << lane) - 1u;
#pragma unroll
    for (int x = 0; x < kEPer; ++x) {
      if ((keepm >> x) & 1u) far_live[kw + kpre[x] + __popc(km[x] & ltm)] = v[x];
      if ((latm >> x) & 1u) later[aw + apre[x] + __popc(am[x] & ltm)] = v[x];
      if ((livem >> x) & 1u) {
        if (GI_X_PFX) prefetch_l2(a.slots + 8 * (size_t)v[x]);  // read by the next ROUND phase
        q_next[lw + lpre[x] + __popc(lm[x] & ltm)] = v[x];
      }
    }
    __syncthreads();  // s_keep / s_live are rewritten by the next tile
  }
  const uint32_t fm = __reduce_min_sync(0xffffffffu, my_fmin);
  if (lane == 0 && fm != kInf) atomicMin(&s_fmin, fm);
  const uint32_t lmn = __reduce_min_sync(0xffffffffu, my_lmin);
  if (lane == 0 && lmn != kInf) atomicMin(&s_lmin, lmn);
  __syncthreads();
  if (tid == 0) {
    if (s_fmin != kInf) atomicMin(&ws.ctl->fmin[j % 3], s_fmin);
    if (s_lmin != kInf) atomicMin(&ws.ctl->lmin[t % 3], s_lmin);
    if (s_nlive) atomicAdd(&ws.ctl->xlive[j % 3], s_nlive);
  }
}
#endif

#if GI_PRIMARY
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

__global__ void count_big_kernel(const int64_t* __restrict__ off, int64_t n, unsigned long long* out) {
  unsigned long long c = 0;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
    c += (off[v + 1] - off[v]) > kSlotEdges;
  c = warp_sum(c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

__global__ void max_weight_kernel(const uint2* __restrict__ edges, int64_t m, uint32_t* out) {
  uint32_t mx = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
    mx = max(mx, edges[i].y);
  mx = __reduce_max_sync(0xffffffffu, mx);
  if ((threadIdx.x & 31) == 0) atomicMax(out, mx);
}

__global__ void pack_edges_kernel(const uint2* __restrict__ edges, uint32_t* __restrict__ packed, int64_t m,
                                  uint32_t colbits) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
    const uint2 e = edges[i];
    packed[i] = (e.y << colbits) | e.x;
  }
}

__global__ void validate_offsets_kernel(const int64_t* __restrict__ off, int64_t n, int64_t m,
                                        uint32_t* bad) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (off[i] > off[i + 1] || off[i + 1] - off[i] > 0xFFFFFFF0ll) atomicOr(bad, 1u);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && (off[0] != 0 || off[n] != m)) atomicOr(bad, 1u);
}

#endif  // GI_PRIMARY

}  // namespace

namespace GI_VARIANT {

int smem_bytes(int kind) {
  const int far = kFarStage * (int)sizeof(int32_t);
  if (kind == KIND_FUSED_ASYNC) return (kRing + (kBlock / 32) * 4) * (int)(sizeof(uint4) * 5) + far;
  return 2 * kBinCap * (int)sizeof(uint2) + kBigCap * ((int)sizeof(BigEnt) + (int)sizeof(unsigned long long)) + far;
}


static const void* kernel_fn(int kind) {
  switch (kind) {
    case KIND_UNFUSED: return (const void*)sssp_persistent<KIND_UNFUSED>;
    case KIND_FUSED_BSP: return (const void*)sssp_persistent<KIND_FUSED_BSP>;
    case KIND_UNFUSED_LD: return (const void*)sssp_persistent<KIND_UNFUSED_LD>;
    case KIND_FUSED_BSP_LD: return (const void*)sssp_persistent<KIND_FUSED_BSP_LD>;
    case KIND_UNFUSED_XP: return (const void*)sssp_persistent<KIND_UNFUSED_XP>;
    case KIND_FUSED_BSP_XP: return (const void*)sssp_persistent<KIND_FUSED_BSP_XP>;
    default: return (const void*)sssp_persistent<KIND_FUSED_ASYNC>;
  }
}

// The dynamic shared-memory attribute belongs to the kernel's per-context function object:
// cached per (device, kind), so that a graph on a second device sets it there too.
static std::atomic<uint64_t> g_attr_set[KIND_COUNT];

static cudaError_t set_attrs(int kind) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  const uint64_t bit = dev < 64 ? 1ull << dev : 0ull;
  if (bit && (g_attr_set[kind].load(std::memory_order_acquire) & bit)) return cudaSuccess;
  e = cudaFuncSetAttribute(kernel_fn(kind), cudaFuncAttributeMaxDynamicSharedMemorySize, smem_bytes(kind));
  if (e == cudaSuccess && bit) g_attr_set[kind].fetch_or(bit, std::memory_order_acq_rel);
  return e;
}

cudaError_t query_occupancy(int kind, int* blocks_per_sm) {
  cudaError_t e = set_attrs(kind);
  if (e != cudaSuccess) return e;
  return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks_per_sm, kernel_fn(kind), kBlock, smem_bytes(kind));
}

cudaError_t launch_sssp(const KArgs& a, int kind, int grid, cudaStream_t st) {
  cudaError_t e = set_attrs(kind);
  if (e != cudaSuccess) return e;
  KArgs args = a;
  void* params[] = {&args};
  if (a.rung != 2)
    return cudaLaunchCooperativeKernel(kernel_fn(kind), dim3(grid), dim3(kBlock), params, smem_bytes(kind), st);
  // cluster rung: every group is one thread-block cluster (co-scheduled by the hardware;
  // groups never wait on each other, so the launch need not be cooperative). The
  // non-portable size flag belongs to each kernel variant: the expand (XP) variant chosen
  // after query_clusters needs it too.
  if (a.group_size > 8 &&
      (e = cudaFuncSetAttribute(kernel_fn(kind), cudaFuncAttributeNonPortableClusterSizeAllowed, 1)) != cudaSuccess)
    return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kBlock);
  cfg.dynamicSmemBytes = smem_bytes(kind);
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = a.group_size;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelExC(&cfg, kernel_fn(kind), params);
}

// How many clusters of `cluster` CTAs of this kernel variant fit on the device at once.
cudaError_t query_clusters(int kind, int cluster, int* max_clusters) {
  cudaError_t e = set_attrs(kind);
  if (e != cudaSuccess) return e;
  if (cluster > 8) {
    e = cudaFuncSetAttribute(kernel_fn(kind), cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e != cudaSuccess) return e;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(cluster);
  cfg.blockDim = dim3(kBlock);
  cfg.dynamicSmemBytes = smem_bytes(kind);
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cluster;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaOccupancyMaxActiveClusters(max_clusters, kernel_fn(kind), &cfg);
}

#if GI_BLOCK >= 1024
// Launch geometry of the split kernels, computed once per (device, kernel): the host's
// segment loop enqueues these kernels every round, so no attribute or occupancy query may
// sit on that path. Grid sizes are cached per device; the max-dynamic-smem attribute is set
// before the first query on each device (the attribute is per context).
constexpr int kMaxDev = 64;
static std::atomic<int> g_xgrid[kMaxDev][5];  // 4 expand variants + extract_kernel; 0 = unknown
static cudaError_t split_grid(int slot, const void* fn, int threads, int smem, int* grid) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev < kMaxDev) {
    const int g = g_xgrid[dev][slot].load(std::memory_order_acquire);
    if (g > 0) { *grid = g; return cudaSuccess; }
  }
  int sms = 0, bps = 0;
  if (smem > 0) e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, fn, threads, smem);
  if (e != cudaSuccess) return e;
  *grid = sms * (bps > 0 ? bps : 1);
  if (dev < kMaxDev) g_xgrid[dev][slot].store(*grid, std::memory_order_release);
  return cudaSuccess;
}

cudaError_t launch_expand(const KArgs& a, cudaStream_t st, int* grid_used) {
  const int slot = (a.pedges ? 2 : 0) + (a.mirror ? 1 : 0);
  const void* fn = a.pedges ? (a.mirror ? (const void*)expand_kernel<true, true> : (const void*)expand_kernel<true, false>)
                            : (a.mirror ? (const void*)expand_kernel<false, true> : (const void*)expand_kernel<false, false>);
  const int smem = (int)sizeof(XShared);
  int grid = 0;
  cudaError_t e = split_grid(slot, fn, kBlock, smem, &grid);
  if (e != cudaSuccess) return e;
  if (grid_used) *grid_used = grid;
  KArgs args = a;
  void* params[] = {&args};
  return cudaLaunchKernel(fn, dim3(grid), dim3(kBlock), params, smem, st);
}

cudaError_t launch_extract(const KArgs& a, cudaStream_t st) {
  int grid = 0;
  cudaError_t e = split_grid(4, (const void*)extract_kernel, kEBlock, 0, &grid);
  if (e != cudaSuccess) return e;
  // the pile size is read by the kernel (KState.xn): one resident wave, tiles grid-strided
  extract_kernel<<<grid, kEBlock, 0, st>>>(a);
  return cudaGetLastError();
}
#endif

}  // namespace GI_VARIANT

#if GI_PRIMARY
#ifdef GI_TRACE
extern "C" int gi_debug_trace2(unsigned long long* phase, unsigned long long* item, int reset) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(phase, g_phase, sizeof(unsigned long long) * 7 * kTracePhases);
  cudaMemcpyFromSymbol(item, g_item, sizeof(unsigned long long) * 16);
  if (reset) {
    static unsigned long long z[7 * kTracePhases];
    cudaMemcpyToSymbol(g_phase, z, sizeof(z));
    cudaMemcpyToSymbol(g_item, z, sizeof(unsigned long long) * 16);
  }
  return 0;
}

extern "C" int gi_debug_trace(unsigned long long* out, int reset) {
  cudaDeviceSynchronize();
  cudaMemcpyFromSymbol(out, g_trace, sizeof(unsigned long long) * 64);
  if (reset) {
    unsigned long long z[64] = {0};
    cudaMemcpyToSymbol(g_trace, z, sizeof(z));
  }
  return 0;
}
#endif

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

cudaError_t launch_count_big(const int64_t* off, int64_t n, unsigned long long* count, cudaStream_t st) {
  count_big_kernel<<<grid_for(n), 256, 0, st>>>(off, n, count);
  return cudaGetLastError();
}

cudaError_t launch_max_weight(const uint2* edges, int64_t m, uint32_t* max_w, cudaStream_t st) {
  if (m <= 0) return cudaSuccess;
  max_weight_kernel<<<grid_for(m), 256, 0, st>>>(edges, m, max_w);
  return cudaGetLastError();
}

cudaError_t launch_pack_edges(const uint2* edges, uint32_t* packed, int64_t m, uint32_t colbits, cudaStream_t st) {
  if (m <= 0) return cudaSuccess;
  pack_edges_kernel<<<grid_for(m), 256, 0, st>>>(edges, packed, m, colbits);
  return cudaGetLastError();
}

cudaError_t launch_validate_offsets(const int64_t* off, int64_t n, int64_t m, uint32_t* bad_flag,
                                    cudaStream_t st) {
  validate_offsets_kernel<<<grid_for(n), 256, 0, st>>>(off, n, m, bad_flag);
  return cudaGetLastError();
}

#endif  // GI_PRIMARY

}  // namespace gi

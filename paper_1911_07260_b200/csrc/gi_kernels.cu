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
// Fig. alg:eager_delta_stepping_merge). Edge relaxation
// (kernel (b)) is degree-binned: CTA per vertex (deg >= deg_cta_min), warp per
// vertex (deg >= deg_warp_min), thread per vertex otherwise; Dist[dst] =
// min(Dist[dst], Dist[src]+w) is an atomicMin on uint32, issued
// for all of a thread's edges before any result is consumed.
// Lowerings into a FUTURE bucket are appended once per vertex to the far pile
// (dedup bit = reduceBucketUpdates; "a single bucket update
// per vertex"), staged in shared memory and flushed at the phase
// end, off the bucket's critical chain; lowerings into the CURRENT bucket go to
// the CTA bin as (vertex, distance) pairs (eager) and the
// vertex's adjacency slot is prefetched into L2 for the next sub-round.
#include "gi_internal.h"

#include <cooperative_groups.h>

namespace cg = cooperative_groups;

namespace gi {
namespace {

enum : uint32_t { MODE_ROUND = 0, MODE_EXTRACT = 1, MODE_DONE = 2, MODE_NONE = 3 };

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

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

// Barrier over the CTAs of one group (all co-resident: cooperative launch).
__device__ __forceinline__ void group_barrier(Ctl* ctl, uint32_t nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t gen = ld_acquire(&ctl->bar_gen);
    __threadfence();
    const uint32_t arrived = atomicAdd(&ctl->bar_count, 1u);
    if (arrived == nblocks - 1) {
      atomicExch(&ctl->bar_count, 0u);
      __threadfence();
      atomicAdd(&ctl->bar_gen, 1u);
    } else {
      while (ld_acquire(&ctl->bar_gen) == gen) {
      }
    }
    __threadfence();
  }
  __syncthreads();
}

template <typename T>
__device__ __forceinline__ T warp_sum(T x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}

struct Shared {
  uint32_t outcnt;         // fill of the current-bucket bin
  uint32_t farcnt;         // fill of the far staging buffer
  uint32_t mode, b, cnt;
  int32_t claim;
  uint32_t cdu;
  int64_t cbeg, cend;
  uint32_t fmin;
  unsigned long long red[kBlock / 32];
  int32_t farstage[kFarStage];
};

// Everything a relaxation needs, held in registers for one phase.
struct Ctx {
  uint32_t* dist;
  const uint4* slots;
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
  uint2* out;              // CTA-local current-bucket bin (shared memory)
  Shared* s;
  uint32_t my_fmin;        // thread-local min far bucket (reduced at phase end)
  bool pre_read;
};

// Append v to the global frontier once per phase (dedup bit), warp-aggregated.
__device__ __forceinline__ void push_global(Ctx& c, int32_t v) {
  const uint32_t bit = 1u << (v & 31);
  const uint32_t old = atomicOr(&c.qbits_next[v >> 5], bit);
  if (!(old & bit)) {
    prefetch_l2(c.slots + 4 * (size_t)v);
    cg::coalesced_group g = cg::coalesced_threads();
    uint32_t base = 0;
    if (g.thread_rank() == 0) base = atomicAdd(c.qcount_next, g.size());
    base = g.shfl(base, 0);
    c.q_next[base + g.thread_rank()] = v;
  }
}

// Current-bucket push: CTA-local bin (fusion) or the global frontier.
template <bool FUSED>
__device__ __forceinline__ void push_cur(Ctx& c, int32_t v, uint32_t d) {
  if constexpr (FUSED) {
    prefetch_l2(c.slots + 4 * (size_t)v);
    cg::coalesced_group g = cg::coalesced_threads();
    uint32_t base = 0;
    if (g.thread_rank() == 0) base = atomicAdd(&c.s->outcnt, g.size());
    base = g.shfl(base, 0);
    const uint32_t pos = base + g.thread_rank();
    if (pos < (uint32_t)kBinCap) c.out[pos] = make_uint2((uint32_t)v, d);
    else push_global(c, v);
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

__device__ __noinline__ void mark_overflow(Ctx& c, uint32_t v) {
  atomicOr(&c.ovfbits[v >> 5], 1u << (v & 31));
  atomicOr(c.ovf_cand, 1u);
}

// Relax up to K edges (u -> e[k].x, weight e[k].y) from tentative distance du
// (PAPER.md:422). All loads / atomics are issued before any result is consumed.
template <bool FUSED, int K>
__device__ __forceinline__ void relax_k(Ctx& c, uint32_t du, const uint2 (&e)[K], uint32_t valid) {
  uint32_t nd[K];
  uint32_t ok = 0;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    nd[k] = 0;
    if (valid & (1u << k)) {
      const uint64_t s = (uint64_t)du + (uint64_t)e[k].y;
      if (s >= (uint64_t)kInf) mark_overflow(c, e[k].x);  // not representable
      else { nd[k] = (uint32_t)s; ok |= 1u << k; }
    }
  }
  if (c.pre_read) {
    uint32_t cur[K];
#pragma unroll
    for (int k = 0; k < K; ++k) cur[k] = (ok & (1u << k)) ? ld_dist(c.dist + e[k].x) : 0u;
#pragma unroll
    for (int k = 0; k < K; ++k)
      if ((ok & (1u << k)) && !(nd[k] < cur[k])) ok &= ~(1u << k);
  }
  uint32_t old[K];
#pragma unroll
  for (int k = 0; k < K; ++k) old[k] = (ok & (1u << k)) ? atomicMin(c.dist + e[k].x, nd[k]) : 0u;
#pragma unroll
  for (int k = 0; k < K; ++k) {
    if ((ok & (1u << k)) && nd[k] < old[k]) {
      const uint32_t bk = fdiv(nd[k], c.div);
      if (bk == c.b) push_cur<FUSED>(c, (int32_t)e[k].x, nd[k]);
      else push_far(c, (int32_t)e[k].x, bk);  // bk > b: nd >= du >= bΔ
    }
  }
}

// Relax edges [beg, end) of the CSR with stride `stride` starting at beg+lane,
// 4 per iteration per thread.
template <bool FUSED>
__device__ __forceinline__ void relax_range(Ctx& c, uint32_t du, int64_t beg, int64_t end, int lane,
                                            int stride) {
  for (int64_t e0 = beg + lane; e0 < end; e0 += 4 * (int64_t)stride) {
    uint2 e[4];
    uint32_t valid = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int64_t i = e0 + (int64_t)k * stride;
      if (i < end) { e[k] = __ldg(c.edges + i); valid |= 1u << k; }
      else e[k] = make_uint2(0, 0);
    }
    relax_k<FUSED, 4>(c, du, e, valid);
  }
}

// One wave: every thread of the CTA holds at most one frontier entry (v, du).
// Degree-binned relaxation (thread / warp / CTA per vertex).
template <bool FUSED>
__device__ __forceinline__ void relax_wave(Ctx& c, Shared& s, bool have, int32_t v, uint32_t du,
                                           bool check_stale, uint32_t warp_min, uint32_t cta_min,
                                           unsigned long long& nv, unsigned long long& ne) {
  uint4 s0 = make_uint4(kColEmpty, kColEmpty, kColEmpty, kColEmpty), s1 = s0, s2 = s0, s3 = s0;
  if (have) {
    const uint4* sp = c.slots + 4 * (size_t)v;
    s0 = __ldg(sp); s1 = __ldg(sp + 1); s2 = __ldg(sp + 2); s3 = __ldg(sp + 3);
    if (check_stale && ld_dist(c.dist + v) < du) have = false;  // a newer entry exists
  }
  const bool big = have && s0.x == kColBig;
  int64_t deg = 0, beg = 0, end = 0;
  uint2 e[8];
  uint32_t valid = 0;
  if (big) {
    deg = s0.y;
    beg = (int64_t)(((uint64_t)s0.w << 32) | s0.z);
    end = beg + deg;
  } else if (have) {
    e[0] = make_uint2(s0.x, s0.y); e[1] = make_uint2(s0.z, s0.w);
    e[2] = make_uint2(s1.x, s1.y); e[3] = make_uint2(s1.z, s1.w);
    e[4] = make_uint2(s2.x, s2.y); e[5] = make_uint2(s2.z, s2.w);
    e[6] = make_uint2(s3.x, s3.y); e[7] = make_uint2(s3.z, s3.w);
#pragma unroll
    for (int k = 0; k < 8; ++k) valid |= (e[k].x != kColEmpty) ? (1u << k) : 0u;
    deg = __popc(valid);
  }
  nv += have ? 1 : 0;
  ne += (unsigned long long)deg;

  // small vertex, adjacency inline in its slot: one thread
  if (valid) relax_k<FUSED, 8>(c, du, e, valid);
  if (!big) deg = 0;

  // CTA per vertex
  while (__syncthreads_or(deg >= (int64_t)cta_min)) {
    if (deg >= (int64_t)cta_min) s.claim = (int32_t)threadIdx.x;
    __syncthreads();
    if (s.claim == (int32_t)threadIdx.x) {
      s.cdu = du; s.cbeg = beg; s.cend = end;
      deg = 0;
    }
    __syncthreads();
    relax_range<FUSED>(c, s.cdu, s.cbeg, s.cend, threadIdx.x, kBlock);
  }
  // warp per vertex
  const int lane = threadIdx.x & 31;
  uint32_t wm;
  while ((wm = __ballot_sync(0xffffffffu, deg >= (int64_t)warp_min)) != 0) {
    const int leader = __ffs(wm) - 1;
    const uint32_t ldu = __shfl_sync(0xffffffffu, du, leader);
    const int64_t lb = __shfl_sync(0xffffffffu, beg, leader);
    const int64_t le = __shfl_sync(0xffffffffu, end, leader);
    if (lane == leader) deg = 0;
    relax_range<FUSED>(c, ldu, lb, le, lane, 32);
  }
  // thread per vertex (deg > 8 but below the warp threshold)
  if (deg > 0) relax_range<FUSED>(c, du, beg, end, 0, 1);
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
  extern __shared__ uint2 s_bins[];  // [2 * kBinCap]
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
        ctl->qcount[k] = 0; ctl->fcount[k] = 0; ctl->fmin[k] = kInf; ctl->xlive[k] = 0;
      }
      ctl->fcount[0] = 1; ctl->fmin[0] = 0; ctl->ovf_cand = 0;
      ws.far[0][0] = src;
      atomicOr(&ws.farbits[src >> 5], 1u << (src & 31));
    }
    group_barrier(ctl, G);

    Ctx c;
    c.dist = dist; c.slots = a.slots; c.edges = a.edges; c.div = a.div;
    c.farbits = ws.farbits; c.ovfbits = ws.ovfbits; c.ovf_cand = &ctl->ovf_cand;
    c.s = &s;
    c.pre_read = a.pre_read != 0;

    unsigned long long nv = 0, ne = 0;            // per thread
    unsigned long long subrounds = 0, spills = 0, scanned = 0;  // per CTA (thread 0)
    unsigned long long phases = 0, rounds = 0, buckets = 0, empty = 0;  // rank 0, thread 0
    uint32_t p = 0, j = 0, b = 0, prev = MODE_NONE;

    for (;;) {
      // ---- decide (identically in every CTA, from counters final at the barrier) ----
      if (tid == 0) {
        if (prev == MODE_EXTRACT) {
          const uint32_t xl = ld_acquire(&ctl->xlive[j % 3]);
          if (xl) { ++buckets; if (FUSED) ++rounds; } else { ++empty; }
        }
        const uint32_t qn = ld_acquire(&ctl->qcount[p % 3]);
        uint32_t mode;
        if (qn > 0) {
          mode = MODE_ROUND; s.cnt = qn;
        } else {
          const uint32_t fc = ld_acquire(&ctl->fcount[j % 3]);
          if (fc > 0) { mode = MODE_EXTRACT; s.cnt = fc; s.b = ld_acquire(&ctl->fmin[j % 3]); }
          else mode = MODE_DONE;
        }
        s.mode = mode;
        s.outcnt = 0;
        s.farcnt = 0;
        s.fmin = kInf;
      }
      __syncthreads();
      const uint32_t mode = s.mode;
      if (mode == MODE_DONE) break;
      const uint32_t cnt = s.cnt;
      if (mode == MODE_EXTRACT) { ++j; b = s.b; }
      if (rank == 0 && tid == 0) {
        ctl->qcount[(p + 2) % 3] = 0;
        if (mode == MODE_EXTRACT) {
          ctl->fcount[(j + 1) % 3] = 0; ctl->fmin[(j + 1) % 3] = kInf; ctl->xlive[(j + 1) % 3] = 0;
        }
        if (mode == MODE_ROUND) ++rounds;
      }
      c.b = b;
      c.qbits_next = ws.qbits[(p + 1) & 1];
      c.q_next = ws.q[(p + 1) & 1];
      c.qcount_next = &ctl->qcount[(p + 1) % 3];
      c.far_live = ws.far[j & 1];
      c.fcount_live = &ctl->fcount[j % 3];
      c.out = s_bins;
      c.my_fmin = kInf;

      const uint32_t lo = (uint32_t)(((uint64_t)cnt * rank) / G);
      const uint32_t hi = (uint32_t)(((uint64_t)cnt * (rank + 1)) / G);

      if (mode == MODE_EXTRACT) {
        // (d)+(a): partition the far pile by recomputed bucket
        const int32_t* far_src = ws.far[(j - 1) & 1];
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
        const uint32_t tl = block_sum(nlive, s);
        if (tid == 0) {
          if (tl) atomicAdd(&ctl->xlive[j % 3], tl);
          scanned += hi - lo;
        }
      } else {
        // ROUND: relax the group's global frontier, one slice per CTA
        const int32_t* q_in = ws.q[p & 1];
        uint32_t* qbits_in = ws.qbits[p & 1];
        for (uint32_t base = lo; base < hi; base += kBlock) {
          const uint32_t i = base + tid;
          const bool have = i < hi;
          int32_t v = 0;
          uint32_t du = 0;
          if (have) {
            v = q_in[i];
            atomicAnd(&qbits_in[v >> 5], ~(1u << (v & 31)));
            du = ld_dist(dist + v);
          }
          relax_wave<FUSED>(c, s, have, v, du, false, a.deg_warp_min, a.deg_cta_min, nv, ne);
        }
      }

      if constexpr (FUSED) {
        // (c) bucket fusion: drain the CTA-local bin while it stays below T
        // (PAPER.md:537-550); a bin of size >= T goes to the global frontier
        // ("copied over to the global bucket").
        uint2* in = s_bins + kBinCap;
        for (;;) {
          __syncthreads();
          const uint32_t nout = min(s.outcnt, (uint32_t)kBinCap);
          if (nout == 0) break;
          if (nout >= T) {
            for (uint32_t i = tid; i < nout; i += kBlock) push_global(c, (int32_t)c.out[i].x);
            if (tid == 0) ++spills;
            break;
          }
          uint2* t = in; in = c.out; c.out = t;
          __syncthreads();
          if (tid == 0) { s.outcnt = 0; ++subrounds; }
          __syncthreads();
          for (uint32_t base = 0; base < nout; base += kBlock) {
            const uint32_t i = base + tid;
            const bool have = i < nout;
            uint2 e = make_uint2(0, 0);
            if (have) e = in[i];
            relax_wave<FUSED>(c, s, have, (int32_t)e.x, e.y, true, a.deg_warp_min, a.deg_cta_min, nv, ne);
          }
        }
      }

      // flush staged far-pile pushes (dedup + append), then the next-bucket lower
      // bound: warp min + one smem atomic per warp + one global atomic per CTA
      __syncthreads();
      {
        const uint32_t nf = min(s.farcnt, (uint32_t)kFarStage);
        for (uint32_t i = tid; i < nf; i += kBlock) push_far_global(c, s.farstage[i]);
        uint32_t fm = __reduce_min_sync(0xffffffffu, c.my_fmin);
        if ((tid & 31) == 0 && fm != kInf) atomicMin(&s.fmin, fm);
        __syncthreads();
        if (tid == 0 && s.fmin != kInf) atomicMin(&ctl->fmin[j % 3], s.fmin);
      }
      group_barrier(ctl, G);
      ++p;
      ++phases;
      prev = mode;
    }

    // ---- overflow resolution: a vertex with an overflowing candidate that never
    // received a representable distance has δ >= UINT32_MAX ----
    if (ld_acquire(&ctl->ovf_cand)) {
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
    const unsigned long long tv = block_sum(nv, s);
    const unsigned long long te = block_sum(ne, s);
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
      }
    }
    group_barrier(ctl, G);  // the next query re-initialises ctl
  }
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

// ELL slot per vertex: deg <= 8 -> edges inline (unused entries kColEmpty);
// deg > 8 -> header {kColBig, deg, beg_lo, beg_hi} pointing into the CSR edges.
__global__ void build_slots_kernel(const int64_t* __restrict__ off, const uint2* __restrict__ edges,
                                   uint4* __restrict__ slots, int64_t n) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    const int64_t beg = off[v], deg = off[v + 1] - beg;
    uint2 e[8];
    if (deg <= kSlotEdges) {
#pragma unroll
      for (int k = 0; k < 8; ++k) e[k] = k < deg ? edges[beg + k] : make_uint2(kColEmpty, 0);
    } else {
      e[0] = make_uint2(kColBig, (uint32_t)deg);
      e[1] = make_uint2((uint32_t)(uint64_t)beg, (uint32_t)((uint64_t)beg >> 32));
#pragma unroll
      for (int k = 2; k < 8; ++k) e[k] = make_uint2(kColEmpty, 0);
    }
    uint4* sp = slots + 4 * v;
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

int smem_bytes() { return 2 * kBinCap * (int)sizeof(uint2); }

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

cudaError_t launch_build_slots(const int64_t* off, const uint2* edges, uint4* slots, int64_t n,
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

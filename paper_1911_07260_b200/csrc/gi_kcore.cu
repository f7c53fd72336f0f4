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
#include "gi_internal.h"
#include "gi_device.cuh"

namespace gi {
namespace {

constexpr int kKcBlock = 512;
constexpr int kKcEdges = 8;     // consecutive edges per thread per iteration
constexpr int kKcChunk = 2048;  // frontier vertices staged per claim (max)
constexpr uint32_t kUnset = 0xFFFFFFFFu;

enum : uint32_t { KC_ROUND = 0, KC_EXTRACT = 1, KC_DONE = 2 };

struct KcShared {
  uint32_t mode, k, cnt, claim, kmin;
  unsigned long long total;
  unsigned long long red[kKcBlock / 32];
};

__device__ __forceinline__ uint32_t ld_cg(const uint32_t* p) { return __ldcg(p); }

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

__global__ void __launch_bounds__(kKcBlock, 1) kcore_persistent(KcArgs a) {
  extern __shared__ unsigned long long kc_dyn[];  // beg [kKcChunk] int64, pre [kKcChunk] u64
  __shared__ KcShared s;
  long long* sbeg = reinterpret_cast<long long*>(kc_dyn);
  unsigned long long* spre = kc_dyn + kKcChunk;
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
      const uint32_t p = d >= (int64_t)kUnset ? kUnset - 1u : (uint32_t)d;
      a.prio[v] = p;
      a.core[v] = kUnset;
      a.pile[0][v] = (int32_t)v;
      mn = min(mn, p);
    }
    mn = __reduce_min_sync(0xffffffffu, mn);
    if (lane == 0 && mn != kUnset) atomicMin(&ctl->kmin[0], mn);
  }
  dev::group_barrier(&ctl->bar, G);

  unsigned long long nfin = 0, nedge = 0;     // per thread
  unsigned long long buckets = 0, rounds = 0, phases = 0, empty = 0;  // rank 0 / thread 0
  uint32_t p = 0, j = 0, k = 0, prev = KC_DONE;
  for (;;) {
    if (tid == 0) {
      // an extraction whose k came from a vertex finished later in the same bucket finds
      // nothing (the recorded minimum is a lower bound): counted apart, like SSSP's R6
      if (prev == KC_EXTRACT) {
        if (__ldcg(&ctl->xfin[j % 3])) ++buckets; else ++empty;
      }
      const uint32_t qn = __ldcg(&ctl->qcount[p % 3]);
      const uint32_t pc = __ldcg(&ctl->pcount[j % 3]);
      const uint32_t km = __ldcg(&ctl->kmin[j % 3]);
      uint32_t mode;
      if (qn > 0) { mode = KC_ROUND; s.cnt = qn; }
      else if (pc > 0) { mode = KC_EXTRACT; s.cnt = pc; s.k = km; }
      else mode = KC_DONE;
      s.mode = mode;
      s.kmin = kUnset;
    }
    __syncthreads();
    const uint32_t mode = s.mode;
    if (mode == KC_DONE) break;
    const uint32_t cnt = s.cnt;
    if (mode == KC_EXTRACT) { ++j; k = s.k; }
    if (rank == 0 && tid == 0) {
      ctl->qcount[(p + 2) % 3] = 0;
      ctl->qclaim[(p + 1) % 3] = 0;  // last used in phase p-2, which every CTA has left
      if (mode == KC_EXTRACT) {
        ctl->pcount[(j + 1) % 3] = 0; ctl->kmin[(j + 1) % 3] = kUnset; ctl->xfin[(j + 1) % 3] = 0;
      } else {
        ++rounds;
      }
    }
    int32_t* q_next = (p & 1) ? a.q[0] : a.q[1];
    uint32_t* qcount_next = &ctl->qcount[(p + 1) % 3];
    uint32_t* kmin_live = &ctl->kmin[j % 3];  // the min for the NEXT extraction
    uint32_t my_kmin = kUnset;

    if (mode == KC_EXTRACT) {
      // dequeue_ready_set: the pile entries whose priority is <= k
      const int32_t* pile_src = (j & 1) ? a.pile[0] : a.pile[1];
      int32_t* pile_live = (j & 1) ? a.pile[1] : a.pile[0];
      uint32_t* pcount_live = &ctl->pcount[j % 3];
      const uint32_t lo = (uint32_t)(((uint64_t)cnt * rank) / G), hi = (uint32_t)(((uint64_t)cnt * (rank + 1)) / G);
      uint32_t nx = 0;
      for (uint32_t i0 = lo; i0 < hi; i0 += kKcBlock) {  // warp-uniform trip count
        const uint32_t i = i0 + tid;
        const bool in = i < hi;
        const int32_t v = in ? pile_src[i] : 0;
        const uint32_t c = in ? ld_cg(a.core + v) : 0u;
        const uint32_t pr = in ? ld_cg(a.prio + v) : 0u;
        const bool live = in && c == kUnset;       // finished entries are dropped
        const bool fin = live && pr <= k;
        const bool keep = live && pr > k;
        if (fin) { a.core[v] = k; ++nfin; ++nx; }
        if (keep) my_kmin = min(my_kmin, pr);
        kc_append(fin, v, q_next, qcount_next);
        kc_append(keep, v, pile_live, pcount_live);
      }
      nx = __reduce_add_sync(0xffffffffu, nx);
      if (lane == 0 && nx) atomicAdd(&ctl->xfin[j % 3], nx);
    } else {
      // edges.from(frontier).applyUpdatePriority(apply_f)
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
        // stage (beg, deg) and block-scan the degrees
        unsigned long long sum = 0;
        constexpr int PER = kKcChunk / kKcBlock;
        unsigned long long loc[PER];
#pragma unroll
        for (int x = 0; x < PER; ++x) {
          const uint32_t i = tid * PER + x;
          loc[x] = sum;
          if (i < chunk) {
            const int32_t v = q_in[base + i];
            const long long b0 = a.off[v], b1 = a.off[v + 1];
            sbeg[i] = b0;
            sum += (unsigned long long)(b1 - b0);
          }
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
          if (i < chunk) spre[i] = off0 + loc[x];
        }
        __syncthreads();
        const unsigned long long total = s.total;
        if (tid == 0) nedge += total;
        for (unsigned long long k0 = 0; k0 < total; k0 += (unsigned long long)kKcEdges * kKcBlock) {
          int32_t tv[kKcEdges];
#pragma unroll
          for (int u = 0; u < kKcEdges; ++u) tv[u] = -1;
          const unsigned long long kt = k0 + (unsigned long long)kKcEdges * tid;
          if (kt < total) {
            uint32_t lo = 0, hi = chunk;  // last i with spre[i] <= kt
            while (hi - lo > 1) {
              const uint32_t mid = (lo + hi) >> 1;
              if (spre[mid] <= kt) lo = mid; else hi = mid;
            }
            unsigned long long nxt = lo + 1 < chunk ? spre[lo + 1] : total;
            long long rel = sbeg[lo] - (long long)spre[lo];
#pragma unroll
            for (int u = 0; u < kKcEdges; ++u) {
              const unsigned long long e = kt + u;
              if (e < total) {
                while (e >= nxt) {  // next frontier vertex (skipping degree-0 ones)
                  ++lo;
                  rel = sbeg[lo] - (long long)nxt;
                  nxt = lo + 1 < chunk ? spre[lo + 1] : total;
                }
                tv[u] = (int32_t)__ldg(&a.edges[rel + (long long)e].x);
              }
            }
          }
          // skip finished endpoints (coherent read; finished is final)
          uint32_t cv[kKcEdges];
#pragma unroll
          for (int u = 0; u < kKcEdges; ++u) cv[u] = tv[u] >= 0 ? ld_cg(a.core + tv[u]) : 0u;
#pragma unroll
          for (int u = 0; u < kKcEdges; ++u) {
            const bool want = tv[u] >= 0 && cv[u] == kUnset;
            // constant-sum reduction: one atomic per distinct endpoint per warp
            const uint32_t key = want ? (uint32_t)tv[u] : 0xFFFFFFFFu;
            const uint32_t peers = __match_any_sync(0xffffffffu, key);
            const bool leader = want && (__ffs(peers) - 1) == (int)lane;
            bool cross = false;
            if (leader) {
              const uint32_t c = __popc(peers);
              const uint32_t old = atomicSub(a.prio + tv[u], c);
              if (old > k && old - c <= k) {
                cross = true;  // this subtraction took the priority to <= k: finished at k
                a.core[tv[u]] = k;
              } else if (old > k) {
                my_kmin = min(my_kmin, old - c);
              }
            }
            nfin += cross;
            kc_append(cross, tv[u], q_next, qcount_next);
          }
        }
        __syncthreads();
        if (tid == 0) {
          s.claim = dyn ? next : cnt;
          if (dyn && next < cnt) next = (uint32_t)first + atomicAdd(qclaim, claim);
        }
        __syncthreads();
      }
    }

    // next k: the exact minimum priority of the unfinished vertices (kept entries and
    // every non-crossing decrement), warp min -> smem -> one global atomic per CTA
    my_kmin = __reduce_min_sync(0xffffffffu, my_kmin);
    if (lane == 0 && my_kmin != kUnset) atomicMin(&s.kmin, my_kmin);
    __syncthreads();
    if (tid == 0 && s.kmin != kUnset) atomicMin(kmin_live, s.kmin);
    dev::group_barrier(&ctl->bar, G);
    ++p;
    ++phases;
    prev = mode;
  }

  // statistics
  nfin = __reduce_add_sync(0xffffffffu, (unsigned)nfin) ;
  if (lane == 0 && nfin) atomicAdd(&a.stats->vertices, nfin);
  if (tid == 0) {
    if (nedge) atomicAdd(&a.stats->edges, nedge);
    if (rank == 0) {
      a.stats->buckets = buckets; a.stats->rounds = rounds; a.stats->phases = phases + 1; a.stats->empty = empty;
    }
  }
}

}  // namespace

int kcore_smem_bytes() { return kKcChunk * (int)(sizeof(long long) + sizeof(unsigned long long)); }

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

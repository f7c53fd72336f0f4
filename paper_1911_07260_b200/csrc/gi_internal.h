// gi_internal.h — structures shared by the sm_100a kernels and the host engine.
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace gi {

constexpr uint32_t kInf = 0xFFFFFFFFu;
#ifndef GI_BLOCK
#define GI_BLOCK 512
#endif
#ifndef GI_MINB
#define GI_MINB 1
#endif
constexpr int kBlock = GI_BLOCK;     // threads per persistent CTA
constexpr int kMinBlocksPerSm = GI_MINB;
// CTA-local current-bucket bin of uint2 {v, d}; two (ping-pong) per CTA. By CTA width (512,
// 1024): the 1024-thread kernel also runs the throughput-bound batches, whose bins are big
// (config 5: 4096 against 2048 cut spills 3,647 -> 58 and 183 -> 160 ms; single queries
// unchanged).
constexpr int kBinCapW[2] = {2048, 4096};
constexpr int kBinCap = kBinCapW[GI_BLOCK >= 1024 ? 1 : 0];
constexpr int kBigCap = 2048;        // CTA-local list of high-degree vertices (deg > 8) per bin
constexpr uint32_t kDefaultT = 1024; // fusion threshold default (vertices per CTA bin), max out-degree <= 32
constexpr uint32_t kDefaultTSkewed = 256;  // ... and on skewed graphs (max out-degree > 32); DESIGN.md §10
constexpr uint32_t kDefaultWindow = 0;  // bucket window width (buckets) of split queries: off (measured slower)
constexpr int kSlotEdges = 8;        // ELL slot: up to 8 {col, w} edges inline (64 B per vertex)
constexpr uint32_t kColEmpty = 0xFFFFFFFFu;  // unused slot entry
constexpr uint32_t kColBig = 0xFFFFFFFEu;    // deg > 8: all 8 entries {kColBig, payload}; payloads deg, beg_lo, beg_hi
#ifndef GI_FARSTAGE
#define GI_FARSTAGE 8192
#endif
constexpr int kFarStage = GI_FARSTAGE;  // CTA-local staging of far-pile pushes (flushed at phase end)
constexpr uint32_t kDefaultHubMin = 1024;  // default out-degree for the group-wide hub path
constexpr uint32_t kMinHubMin = 256;       // smallest accepted hub_min (bounds the hub-list size)
constexpr int kRingLog = 11;
constexpr int kRing = 1 << kRingLog;       // async drain: CTA-local work ring (entries of 16 B header + 64 B slot)
// Ring admission limit (see the ring protocol in gi_kernels.cu): concurrent pushers overshoot
// by < one entry per thread (kBlock) and claimed-but-unread entries are < 4 per warp, so a
// limit of kRing - kBlock - 4 * warps keeps every unread entry inside the ring. By CTA width
// (512, 1024): 1472 and 896.
constexpr uint32_t ring_safe(int block) { return (uint32_t)(kRing - block - 4 * (block / 32)); }
constexpr uint32_t kRingSafeW[2] = {ring_safe(512), ring_safe(1024)};
constexpr uint32_t kRingSafe = ring_safe(kBlock);
constexpr uint32_t kAsyncMaxDeg = kSlotEdges;  // async drain needs every adjacency inline in its ELL slot

// Persistent-kernel variants.
enum KernelKind : int {
  KIND_UNFUSED = 0, KIND_FUSED_BSP = 1, KIND_FUSED_ASYNC = 2,
  // low-degree specialisations (every adjacency inline in its ELL slot, no pre-read): the
  // high-degree stages compiled out of the sub-round's serial path
  KIND_UNFUSED_LD = 3, KIND_FUSED_BSP_LD = 4,
  // skewed graphs with expand on (gi_options.expand = 1): ROUND phases collect the group list
  // and stop for expand_kernel (KState); compiled apart so that the default kernels keep
  // their registers
  KIND_UNFUSED_XP = 5, KIND_FUSED_BSP_XP = 6,
  KIND_COUNT = 7
};
inline int base_kind(int k) {
  return (k == KIND_UNFUSED_LD || k == KIND_UNFUSED_XP) ? KIND_UNFUSED
         : (k == KIND_FUSED_BSP_LD || k == KIND_FUSED_BSP_XP) ? KIND_FUSED_BSP : k;
}

// Division by the invariant Δ (Granlund & Montgomery 1994, round-up method):
// q = (t + ((x - t) >> s1)) >> s2 with t = umulhi(mul, x).
struct FastDiv {
  uint32_t mul, s1, s2, d;
};

inline FastDiv make_fastdiv(uint32_t d) {
  FastDiv f;
  uint32_t l = 0;
  while (l < 32 && (1ull << l) < d) ++l;  // l = ceil(log2 d)
  f.mul = (uint32_t)((((1ull << l) - d) << 32) / d + 1);
  f.s1 = l > 0 ? 1 : 0;
  f.s2 = l > 0 ? l - 1 : 0;
  f.d = d;
  return f;
}

// Per-query control block (device). Counters rotate mod 3 so that a slot is
// reset only after every CTA has read it.
struct alignas(128) Ctl {
  uint32_t qcount[3];   // global frontier sizes, by phase mod 3
  uint32_t fcount[3];   // far-pile (overflow bucket) sizes, by extraction mod 3
  uint32_t fmin[3];     // lower bound of the min live far bucket, by extraction mod 3
  uint32_t xlive[3];    // live vertices extracted, by extraction mod 3
  uint32_t ovf_cand;    // some candidate distance >= UINT32_MAX was produced
  uint32_t maxsub[3];   // max fused sub-rounds of any CTA, by phase mod 3 (critical-path stat)
  uint32_t hcount[3];   // group hub-list sizes, by phase mod 3
  uint32_t qclaim[3];   // ROUND phases: next unclaimed global-frontier position, by phase mod 3
  uint32_t tdist[3];    // PPSP: min over CTAs of dist[target] read at the phase end, by phase mod 3
  int32_t next_si;      // batch: the source index this group runs next (claimed by its CTA 0)
  uint32_t lcount[3];   // bucket window: later-pile sizes, by window advance mod 3
  uint32_t lmin[3];     // bucket window: lower bound of the later pile's buckets, by advance mod 3
  uint32_t bar;         // group barrier: arrivals (low 16 bits) | generation (high 16), own 128 B line
  uint32_t pad1[31];
};

// Per-source result record (device, copied back to gi_stats).
struct QStats {
  unsigned long long buckets, rounds, phases, subrounds, spills, vertices, edges, empty_extr,
      far_scanned, critical_subrounds;
  uint32_t overflow;
  uint32_t pad;
};

// One query group's workspace (device pointers).
struct GroupWs {
  uint32_t* farbits;  // [nwords] "in far pile" dedup bits (lazy buffer reduction)
  uint32_t* qbits[2]; // [nwords] "in global frontier" dedup bits, by phase parity
  uint32_t* ovfbits;  // [nwords] vertices that received an overflowing candidate
  int32_t* far[2];    // [n] far pile, double-buffered across extractions
  int32_t* q[2];      // [n] global frontier, double-buffered across phases
  struct HubEnt* hub[2];  // [hubcap] group hub lists (deg >= hub_min), by phase parity
  unsigned long long* xpre;  // [hubcap] expand: exclusive degree prefix of each entry within its CTA slice
  unsigned long long* xtot;  // [kMaxGroupCtas] expand: edge total of each CTA's slice of the list
  struct KState* kst;        // split expand: the phase loop's state while the relaxation runs outside
  Ctl* ctl;
  // bucket window (KArgs.window; single split queries): far-pile entries whose bucket lies
  // beyond the open window wait in the later pile (one entry per vertex, laterbits) and are
  // rescanned only when the window advances, not at every extraction
  uint32_t* laterbits;  // [nwords] "in the later pile" dedup bits; nullptr = no window
  int32_t* later[2];    // [n] later pile, double-buffered across window advances
};

// Split expand (single queries on skewed graphs): when a ROUND phase's group list holds at
// least split_min edges, the persistent kernel saves its phase-loop state here and exits;
// the host launches expand_kernel (the edge-balanced relaxation with the whole register file
// of its own, 2 CTAs per SM) and then resumes the persistent kernel at the same phase.
struct KState {
  uint32_t p, j, b, prev;       // phase loop position
  uint32_t last_b;              // bucket of the last counted extraction
  unsigned long long phases, rounds, buckets, empty, critical;  // group counters (rank 0)
  unsigned long long E;         // edges of the pending list
  uint32_t xn;                  // entries of the pending list (extract: of the far pile)
  uint32_t pending;             // 1 = the kernel stopped for an external expand of phase p,
                                // 2 = for an external extraction of phase p (extract_kernel)
  uint32_t rkind;               // what the resumed segment continues after (1 expand, 2 extract)
  uint32_t t, wend;             // bucket window: advances so far, end of the open window
  uint32_t wbig;                // bucket window: the far pile has exceeded window_pile
};

constexpr int kMaxGroupCtas = 1024;  // expand: largest group (CTAs) the slice totals are sized for


// A high-degree vertex queued for relaxation by every CTA of the group.
struct HubEnt {
  int64_t beg;
  uint32_t deg;
  uint32_t du;
};
static_assert(sizeof(HubEnt) == 16, "expand loads a list entry as one 16-byte vector");

struct KArgs {
  const uint2* slots;   // [n][8] ELL adjacency slots (64 B per vertex)
  const uint2* edges;   // [m] {col, w} interleaved CSR edges (vertices with deg > 8)
  int64_t n;
  uint32_t nwords;
  const int32_t* srcs;  // [nsrc] device
  int32_t nsrc;
  uint32_t* dist;       // [nsrc][n] device
  GroupWs* groups;      // [ngroups] device
  QStats* qstats;       // [nsrc] device
  int32_t ngroups;
  int32_t group_size;   // CTAs per group
  FastDiv div;
  uint32_t T;           // fusion threshold (<= kBinCap)
  uint32_t pre_read;    // read dist[v] before atomicMin (filters atomics on skewed graphs)
  uint32_t hub_min;     // out-degree >= hub_min -> the vertex's edges are split over the group
  uint32_t hubcap;      // capacity of each hub list
  int32_t target;       // PPSP: stop once the next bucket's lower bound reaches dist[target]; -1 = SSSP
  uint32_t dyn_claim;   // ROUND phases claim frontier chunks dynamically (skewed degrees) vs equal slices
  const uint32_t* h;    // A*: per-vertex heuristic (priority = dist + h); nullptr = 0 (SSSP / PPSP)
  uint32_t* src_next;   // batch: claims so far (source index = ngroups + claim)
  uint32_t* const* peers;  // gi_sssp_batch_peers: [npeers] row bases of every rank's result
                           // matrix (device-accessible: local, P2P or IPC-mapped); nullptr = none
  int32_t npeers;
  uint32_t peer_vec;    // 16-byte copies (n % 4 == 0 and every base 16-byte aligned)
  // expand (skewed graphs): a ROUND phase collects every high-degree frontier vertex into the
  // group list and relaxes the concatenation of their edges split evenly over all warps
  uint32_t expand;
  const uint32_t* pedges;  // [m] packed edges (w << colbits | col) or nullptr (use `edges`)
  uint32_t colbits;        // packed: bits of the column id
  uint32_t lazy;           // fully lazy schedule (unfused kernels): every lowering, the current
                           // bucket's included, goes through the far pile
  uint32_t rung;           // execution-group rung (SURVEY §8(a) ladder): 0 = grid (group barrier
                           // of global atomics), 1 = one CTA (CTA barrier), 2 = one thread-block
                           // cluster per group (hardware cluster barrier)
  uint32_t split;          // single query: heavy expands run in expand_kernel (see KState)
  uint32_t resume;         // this launch resumes a query stopped for an external expand
  unsigned long long split_min;  // list edges from which a phase's expand runs outside
  uint32_t xsplit_min;     // far-pile entries from which an extraction runs outside (0: never)
  // expand's pre-read filter (split queries): a 1-byte saturated copy of dist, n bytes, small
  // enough to stay in L2 where dist (4n bytes) does not. Invariant: mirror[v] == 0xFF, or
  // mirror[v] is a value dist[v] held (so dist[v] <= mirror[v]). nullptr = pre-read dist.
  uint8_t* mirror;
  uint32_t window;         // bucket window width in buckets (0 = off: every far entry is
                           // rescanned at every extraction); needs GroupWs.laterbits
  uint32_t window_pile;    // > 0: the window opens at the first extraction whose far pile holds
                           // <= window_pile entries after having held more (the tail of a skewed
                           // query); 0 = from the start
};

// k-core (gi_kcore.cu): control block, statistics and arguments.
struct alignas(128) KcCtl {
  uint32_t qcount[3];   // frontier sizes, by phase mod 3
  uint32_t pcount[3];   // pile (unfinished vertices) sizes, by extraction mod 3
  uint32_t kmin[3];     // min priority of the unfinished vertices, by extraction mod 3
  uint32_t qclaim[3];   // ROUND: next unclaimed frontier position, by phase mod 3
  uint32_t xfin[3];     // vertices finished by an extraction, by extraction mod 3
  uint32_t hcount[3];   // group hub-list sizes, by phase mod 3
  uint32_t maxsub[3];   // max fused sub-rounds of any CTA, by phase mod 3 (critical-path stat)
  uint32_t pad0[11];
  uint32_t bar;         // group barrier word, own 128 B line
  uint32_t pad1[31];
};

static_assert(offsetof(KcCtl, bar) == 128, "the k-core barrier word owns its 128-byte line");

struct KcStats {
  unsigned long long buckets, rounds, phases, vertices, edges, empty, subrounds, spills, critical;
};

struct KcArgs {
  const int64_t* off;   // [n+1] CSR offsets (device)
  const uint2* edges;   // [m] {col, w}; only col is read
  int64_t n;
  uint32_t* prio;       // [n] workspace: current priority (starts at the degree)
  uint32_t* core;       // [n] result: coreness
  int32_t* pile[2];     // [n] unfinished vertices, double-buffered across extractions
  int32_t* q[2];        // [n] frontier, double-buffered across phases
  struct HubEnt* hub[2];  // [hubcap] group hub lists (degree >= 1024), by phase parity
  uint32_t hubcap;
  KcCtl* ctl;
  KcStats* stats;
  const uint2* slots;   // [n][8] ELL slots (deg <= 8: the edges inline)
  uint32_t ld;          // every adjacency fits its slot (max degree <= 8): the slot path
};

// Host-side launchers (gi_kernels.cu).
// The SSSP-family persistent kernels, compiled once per CTA width (gi_kernels.cu).
namespace v512 {
cudaError_t launch_sssp(const KArgs& a, int kind, int grid, cudaStream_t st);
cudaError_t query_clusters(int kind, int cluster, int* max_clusters);
cudaError_t query_occupancy(int kind, int* blocks_per_sm);
int smem_bytes(int kind);
}  // namespace v512
namespace v1024 {
cudaError_t launch_sssp(const KArgs& a, int kind, int grid, cudaStream_t st);
cudaError_t query_clusters(int kind, int cluster, int* max_clusters);
// the external expand of a split query (KState), 1024-thread CTAs on every SM
cudaError_t launch_expand(const KArgs& a, cudaStream_t st, int* grid_used);
// the external extraction of a split query (KState.pending == 2), a streaming partition
cudaError_t launch_extract(const KArgs& a, cudaStream_t st);
cudaError_t query_occupancy(int kind, int* blocks_per_sm);
int smem_bytes(int kind);
}  // namespace v1024
cudaError_t launch_interleave(const int32_t* cols, const uint32_t* w, uint2* edges, int64_t count,
                              int64_t n, uint32_t* bad_flag, cudaStream_t st);
cudaError_t launch_build_slots(const int64_t* off, const uint2* edges, uint2* slots, int64_t n,
                               cudaStream_t st);
cudaError_t launch_max_degree(const int64_t* off, int64_t n, uint32_t* max_deg, cudaStream_t st);
// skewed-graph layout: vertices of out-degree > 8 (expand list capacity), max weight, and
// the packed edge array (w << colbits | col) when every weight fits the spare bits
cudaError_t launch_count_big(const int64_t* off, int64_t n, unsigned long long* count, cudaStream_t st);
cudaError_t launch_max_weight(const uint2* edges, int64_t m, uint32_t* max_w, cudaStream_t st);
cudaError_t launch_pack_edges(const uint2* edges, uint32_t* packed, int64_t m, uint32_t colbits, cudaStream_t st);
cudaError_t launch_validate_offsets(const int64_t* off, int64_t n, int64_t m, uint32_t* bad_flag,
                                    cudaStream_t st);
cudaError_t launch_kcore(const KcArgs& a, int grid, cudaStream_t st);  // gi_kcore.cu
cudaError_t kcore_occupancy(int* blocks_per_sm);

}  // namespace gi

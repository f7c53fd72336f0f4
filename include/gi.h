/*
 * gi.h — C ABI of the B200-native Δ-stepping SSSP library (libgi.so).
 *
 * Operation (the paper's hot path): single-source shortest paths by Δ-stepping
 * with priority coarsening p' = ⌊p/Δ⌋ (§2), bucket i holding the
 * vertices with tentative distance in [iΔ,(i+1)Δ) (§6.1); the
 * smallest non-empty bucket is processed next, relaxing every out-edge
 * Dist[dst] = min(Dist[dst], Dist[src] + w) (Fig. alg:lazy_delta_stepping,
 * PAPER.md:409-434). Updates to FUTURE buckets are buffered lazily, one bucket
 * update per vertex; updates into the CURRENT bucket go
 * to a CTA-local bin that is drained without a global barrier while it stays
 * below a threshold — bucket fusion (Fig. alg:eager_delta_stepping_merge,
 * PAPER.md:514-558, §3.3). The result is the exact SSSP distance vector
 * (PAPER.md:156-165), identical for every Δ, option, and CTA count.
 *
 * Types: vertex ids int32 (n <= 2^31-1), edge offsets int64, weights uint32,
 * distances uint32 with UINT32_MAX = unreached (the paper's
 * INT_MAX sentinel, is replaced). Any vertex whose true distance is
 * >= UINT32_MAX makes the call return GI_ERR_OVERFLOW.
 *
 * Errors: every entry point returns a gi_status; no exception or abort crosses
 * the boundary. On a non-OK status gi_last_error() returns a thread-local,
 * human-readable message, and the contents of any output buffer are unspecified.
 *
 * Threading: a gi_graph is immutable after creation; any number of host threads
 * may run queries on one graph concurrently (each call takes its own workspace).
 */
#ifndef GI_H_
#define GI_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GI_VERSION 201 /* 2.0.1: gi_options.window (2.0.0: expand / lazy, gi_probe_floors) */

typedef struct gi_graph gi_graph; /* opaque; owns device copies of the CSR */

typedef enum {
  GI_OK = 0,
  GI_ERR_INVALID_ARGUMENT = 1, /* NULL pointer, delta == 0, nsrc < 0, bad option */
  GI_ERR_OUT_OF_RANGE = 2,     /* source id not in [0, n) */
  GI_ERR_INVALID_GRAPH = 3,    /* n/m out of range, offsets[0] != 0, offsets not non-decreasing,
                                  offsets[n] != m, or a column id not in [0, n) */
  GI_ERR_OUT_OF_MEMORY = 4,    /* device or host allocation failed */
  GI_ERR_CUDA = 5,             /* CUDA runtime error, no device, or device not sm_100 */
  GI_ERR_OVERFLOW = 6,         /* a reachable vertex has distance >= UINT32_MAX */
  GI_ERR_UNSUPPORTED = 7
} gi_status;

/* Create a graph on CUDA device `device` from a CSR:
 *   row_offsets int64[n+1] (row_offsets[0] = 0, non-decreasing, row_offsets[n] = m),
 *   col_idx     int32[m]   (0 <= col < n; out-neighbours of row v are
 *                           col_idx[row_offsets[v] .. row_offsets[v+1]) ),
 *   weights     uint32[m]  (weight of the matching col_idx entry; 0 allowed,
 *                           parallel edges and self-loops allowed).
 * Each pointer may be host memory or device memory on `device` (detected with
 * cudaPointerGetAttributes). The arrays are COPIED; the caller keeps ownership and
 * may free them when the call returns. 1 <= n <= 2^31-1, 0 <= m < 2^62.
 * On success *out owns the graph until gi_graph_destroy(). */
gi_status gi_graph_create(int64_t n, int64_t m, const int64_t* row_offsets, const int32_t* col_idx,
                          const uint32_t* weights, int device, gi_graph** out);

/* Release a graph and every cached workspace. NULL-safe. Must not race with a
 * query on the same graph. */
void gi_graph_destroy(gi_graph* g);

/* n, m and device of a graph; any out pointer may be NULL. */
gi_status gi_graph_info(const gi_graph* g, int64_t* n, int64_t* m, int32_t* device);

/* Single-source Δ-stepping SSSP.
 *   src      source vertex, 0 <= src < n, else GI_ERR_OUT_OF_RANGE;
 *   delta    coarsening factor Δ >= 1 (Δ = 0 -> GI_ERR_INVALID_ARGUMENT);
 *   dist_out uint32[n], caller-allocated; device memory on the graph's device
 *            (zero-copy, computed in place) or host memory (staged through a device
 *            buffer). dist_out[v] = δ(src, v), UINT32_MAX if unreachable.
 * Synchronous: returns after dist_out is complete. */
gi_status gi_sssp_delta(const gi_graph* g, int32_t src, uint32_t delta, uint32_t* dist_out);

/* Batch of independent single-source queries (north_star):
 *   srcs     int32[nsrc] (host or device memory); duplicates allowed;
 *   nsrc     >= 0 (0 is a no-op returning GI_OK; < 0 -> GI_ERR_INVALID_ARGUMENT);
 *   dist_out uint32[nsrc][n] row-major, host or device: row i = distances from srcs[i].
 * Several queries run concurrently on disjoint CTA groups of one GPU. */
gi_status gi_sssp_batch(const gi_graph* g, const int32_t* srcs, int32_t nsrc, uint32_t delta,
                        uint32_t* dist_out);

/* ---- extended interface (options + statistics) ---------------------------------- */

typedef struct {
  uint32_t struct_size;      /* = sizeof(gi_options) (ABI check) */
  int32_t fusion;            /* 1: bucket fusion (default); 0: one group-wide barrier per relax round */
  uint32_t fusion_threshold; /* T: a CTA-local current-bucket bin of size >= T spills to the global
                                frontier (PAPER.md:539 strict '<'); 0 = library default; values
                                above the bin capacity (2048 at 512 threads, 4096 at 1024) are
                                clamped to it */
  int32_t max_ctas;          /* cap on persistent CTAs per query group (0 = all co-resident) */
  uint32_t hub_min;          /* out-degree >= hub_min: the vertex's edges are split over every CTA of
                                the group in the next phase (0 = default 1024; values < 256 are
                                raised to 256) */
  uint32_t drain;            /* fused drain of the CTA-local bucket: 0 = default (bsp), 1 = bsp (one
                                CTA barrier per sub-round), 2 = async (barrier-free work ring;
                                GI_ERR_UNSUPPORTED if some out-degree > 8); ignored without fusion */
  int32_t group_ctas;        /* batch only: CTAs per concurrent query group (0 = auto: one group per
                                source, >= 2 CTAs each, capped by free memory for workspaces) */
  int32_t pre_read;          /* read dist[v] before atomicMin: 0 = auto (on when max out-degree > 32),
                                1 = on, 2 = off */
  void* cuda_stream;         /* cudaStream_t to run on (NULL = library stream); calls still
                                synchronise that stream before returning */
  int32_t cta_threads;       /* threads per persistent CTA: 0 = auto (1024 when the max out-degree
                                is > 32 or for a batch of >= 8 sources, else 512), 512 or 1024 */
  int32_t expand;            /* single queries on skewed graphs (max out-degree > 32): every ROUND
                                phase collects its frontier vertices of out-degree > 8 into one group
                                list whose concatenated edges are split evenly over all warps of a
                                separate kernel (edge-balanced, kernel (b)). 0 = auto (on for graphs
                                of >= 512 M edges), 1 = on, 2 = off (CTA-level edge balancing) */
  int32_t lazy;              /* 1: the fully lazy schedule of Fig. alg:lazy_delta_stepping
                                (PAPER.md:409-434): every distance lowering, into the current bucket
                                too, is appended to the bucket-update buffer (the far pile, one
                                entry per vertex = reduceBucketUpdates) and the next round's frontier
                                is the minimum bucket extracted from it (bulkUpdateBuckets +
                                getMinBucket) — one group barrier and one pile scan per round.
                                Requires fusion = 0 (GI_ERR_INVALID_ARGUMENT otherwise). 0 = the
                                eager current bucket (default) */
  int32_t rung;              /* execution-group rung of the query groups (SURVEY.md §8(a) ladder,
                                the thread-local bins of PAPER.md:471-476 generalised): 0 = auto
                                (grid), 1 = one CTA per group (CTA barrier only), 2 = one
                                thread-block cluster per group of group_ctas CTAs (default 8,
                                at most 16; hardware cluster barrier), 3 = grid (group barrier of
                                global atomics over every co-resident CTA, or group_ctas of them) */
  int32_t window;            /* materialized buckets ("only materialize a fixed
                                number of buckets, and store the rest of the vertices in an overflow
                                bucket"; Julienne's open window) for queries running with expand:
                                far-pile entries whose bucket lies >= `window` buckets past the
                                window start wait in an overflow (later) pile that is rescanned only
                                when the window's buckets are done. 0 = off (default: every far
                                entry is recomputed at every extraction), else the
                                window width in buckets; ignored without expand */
} gi_options;

/* Counters of one query (SURVEY §8(a) "Counter definitions"). */
typedef struct {
  uint64_t buckets;            /* extractions that yielded >= 1 live vertex (incl. the source's) */
  uint64_t rounds;             /* group-wide relax passes that begin after a group barrier */
  uint64_t grid_syncs;         /* group-wide barriers executed by the persistent kernel */
  uint64_t kernel_launches;    /* device kernel launches issued for this query */
  uint64_t fused_subrounds;    /* sum over CTAs of local-bin drain iterations (0 without fusion) */
  uint64_t spills;             /* local bins flushed to the global frontier (size >= T) */
  uint64_t vertices_processed; /* non-stale frontier entries whose out-edges were relaxed */
  uint64_t edges_relaxed;      /* out-edges scanned */
  uint64_t empty_extractions;  /* extractions whose bucket held only stale entries */
  uint64_t far_scanned;        /* far-pile (overflow bucket) entries scanned by extractions */
  uint64_t critical_subrounds; /* sum over phases of the max fused sub-rounds run by one CTA
                                  (the dependent chain the fused drain could not shorten) */
  float gpu_ms;                /* device time of the query (CUDA events, whole call for batch) */
  int32_t ctas;                /* persistent CTAs in the query's group */
  int32_t threads_per_cta;
  int32_t groups;              /* concurrent query groups (1 for single source) */
  int32_t kernel_kind;         /* persistent kernel that ran: 0 unfused, 1 fused + bsp drain,
                                  2 fused + async drain, 3 k-core */
  int32_t rung;                /* rung the groups ran on: 1 CTA, 2 cluster, 3 grid */
} gi_stats;

/* Fill *opt with defaults (fusion on, library-default threshold, all CTAs). */
void gi_options_default(gi_options* opt);

/* gi_sssp_delta with options (NULL = defaults) and statistics (NULL = not wanted). */
gi_status gi_sssp_delta_ex(const gi_graph* g, int32_t src, uint32_t delta, const gi_options* opt,
                           uint32_t* dist_out, gi_stats* stats);

/* gi_sssp_batch with options and per-source statistics (per_src: gi_stats[nsrc] or NULL;
 * each entry's gpu_ms is the whole batch's device time). */
gi_status gi_sssp_batch_ex(const gi_graph* g, const int32_t* srcs, int32_t nsrc, uint32_t delta,
                           const gi_options* opt, uint32_t* dist_out, gi_stats* per_src);

/* Multi-GPU batch with the gather fused into the kernel (north_star: "sources sharded
 * evenly over 1/2/4/8 B200s, all distance arrays gathered"). Each rank holds
 * the full result matrix uint32[total][n]; rank r computes a contiguous block of nsrc rows.
 *   peer_rows  [npeers] device pointers, each to the FIRST row of this block inside one
 *              rank's matrix (this rank's own memory for p == self; peer memory made
 *              accessible from the graph's device — P2P or gi_ipc_open_handle — otherwise);
 *   self       index of this rank's own matrix in peer_rows: rows are computed in place there.
 * As soon as a CTA group finishes a source, it writes the row into every other peer_rows[p]
 * (stores over NVLink), while the remaining groups keep computing; no collective runs
 * afterwards. The call returns when the kernel has completed; other ranks' rows are in this
 * rank's matrix once every rank has returned (a barrier between ranks is the caller's).
 * Errors as gi_sssp_batch_ex; npeers < 1, self out of range or a NULL peer row ->
 * GI_ERR_INVALID_ARGUMENT; peer_rows[self] not device memory of the graph's device ->
 * GI_ERR_INVALID_ARGUMENT. */
gi_status gi_sssp_batch_peers(const gi_graph* g, const int32_t* srcs, int32_t nsrc, uint32_t delta,
                              const gi_options* opt, uint32_t* const* peer_rows, int32_t npeers,
                              int32_t self, gi_stats* per_src);

/* Inter-process sharing of a result matrix for gi_sssp_batch_peers (one process per GPU).
 * gi_ipc_get_handle: handle (64 opaque bytes, written to `handle`) of the device allocation
 * that contains dptr, and dptr's byte offset inside it. gi_ipc_open_handle: map another
 * process's allocation on `device` (peer access enabled lazily) and return base + offset.
 * gi_ipc_close_handle: unmap (dptr and offset as returned/passed by open). */
gi_status gi_ipc_get_handle(const void* dptr, void* handle, uint64_t* offset);
gi_status gi_ipc_open_handle(const void* handle, uint64_t offset, int32_t device, void** dptr);
gi_status gi_ipc_close_handle(void* dptr, uint64_t offset, int32_t device);

/* Point-to-point shortest path: Δ-stepping from src that stops when it
 * enters bucket i with iΔ >= the distance already found to dst — "terminates the program
 * early when it enters iteration i where iΔ is greater than or equal to the shortest
 * distance between s and d it has already found".
 *   src, dst  0 <= src, dst < n, else GI_ERR_OUT_OF_RANGE;
 *   delta     Δ >= 1 (Δ = 0 -> GI_ERR_INVALID_ARGUMENT);
 *   dist_st   ONE uint32, host or device (on the graph's device): δ(src, dst),
 *             UINT32_MAX if dst is unreachable. The distance array lives in a library
 *             workspace (n uint32 on the device).
 * GI_ERR_OVERFLOW iff δ(src, dst) >= UINT32_MAX. Synchronous like gi_sssp_delta. */
gi_status gi_ppsp_delta(const gi_graph* g, int32_t src, int32_t dst, uint32_t delta, uint32_t* dist_st);
gi_status gi_ppsp_delta_ex(const gi_graph* g, int32_t src, int32_t dst, uint32_t delta, const gi_options* opt,
                           uint32_t* dist_st, gi_stats* stats);

/* A* search: PPSP whose bucket priority is the ESTIMATED distance of the
 * path through v, dist(v) + h(v) — "uses the estimated distance of the shortest path that
 * goes from the source to the target vertex that passes through the current vertex as the
 * priority". A priority below the current bucket is raised to it, the
 * bucket form of the monotone max(f + h, g[src]) of the paper's Fig. 11.
 *   h        uint32[n], host or device (on the graph's device): the heuristic, an estimate
 *            of the remaining distance to dst (e.g. w_min x grid Chebyshev distance). It is
 *            COPIED (host) or read in place (device) for the call.
 *   src/dst/delta/dist_st as gi_ppsp_delta.
 * dist_st = δ(src, dst) exactly when h is admissible (h(v) <= δ(v, dst) for every v); an
 * inadmissible h may return a longer path length (never a shorter one). GI_ERR_UNSUPPORTED
 * with the async drain (opt->drain == 2). */
gi_status gi_astar_delta(const gi_graph* g, int32_t src, int32_t dst, uint32_t delta, const uint32_t* h,
                         uint32_t* dist_st);
gi_status gi_astar_delta_ex(const gi_graph* g, int32_t src, int32_t dst, uint32_t delta, const uint32_t* h,
                            const gi_options* opt, uint32_t* dist_st, gi_stats* stats);

/* k-core: coreness of every vertex, "the maximum k-core that u is
 * contained in ... using a peeling procedure", by the paper's bucketed
 * peel with lazy bucket updates and the constant-sum reduction (Fig. 10, PAPER.md:1591-1618;
 * PAPER.md:802-837): priorities start at the degrees, the minimum bucket k is finished with
 * coreness k, neighbours' priorities drop by their count of finished neighbours, floored
 * at k. No priority coarsening.
 *   core_out  uint32[n], host or device (on the graph's device): coreness[v].
 * The graph should be symmetric (undirected, both directions stored); degrees count CSR
 * entries (a parallel edge counts twice). Synchronous. stats: buckets = distinct coreness
 * values peeled, rounds = frontier passes, grid_syncs, vertices_processed (= n),
 * edges_relaxed, gpu_ms; kernel_kind = 3. */
gi_status gi_kcore(const gi_graph* g, uint32_t* core_out);
gi_status gi_kcore_ex(const gi_graph* g, const gi_options* opt, uint32_t* core_out, gi_stats* stats);

/* ---- measurement (bench.py; not part of a query) -------------------------------- */

/* Latency floors of the dependent chains, measured on `device` (SURVEY.md §8(d) "Which
 * roofline bounds the path": sync floor = grid_syncs x t_sync + launches x t_launch; chain
 * floor = dependent levels x t_hop). t_sync: one group barrier of the persistent kernels
 * (one CTA per SM, the barrier the fused drain avoids); t_hop: one
 * dependent relaxation hop — an atomicMin on a random 4-byte word of a 64 MB array whose
 * old value names the next word, with that vertex's 64-byte slot (1 GB array) loaded beside
 * it, one chain per SM; t_launch: an empty kernel replayed from a CUDA graph. `iters`
 * barriers / 4 x iters hops are timed with CUDA events. Allocates ~1.1 GB for the call. */
typedef struct {
  float t_sync_us;
  float t_hop_us;
  float t_launch_us;
  float sm_clock_mhz; /* cudaDevAttrClockRate (the maximum clock, not the one under load) */
  int32_t ctas;       /* CTAs in the barrier probe (one per SM) */
} gi_floors;
gi_status gi_probe_floors(int32_t device, int32_t iters, gi_floors* out);

/* Thread-local description of the last non-OK status returned on this thread. */
const char* gi_last_error(void);

/* Static name of a status code. */
const char* gi_status_string(gi_status s);

/* GI_VERSION of the loaded library. */
int32_t gi_version(void);

#ifdef __cplusplus
}
#endif

#endif /* GI_H_ */

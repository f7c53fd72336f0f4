// gi_capi.cu — C ABI (include/gi.h) and host engine: graph residency, validation,
// workspace pool, launch policy, statistics.
#include "gi.h"
#include <cuda.h>
#include "gi_internal.h"

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

using namespace gi;

namespace {

thread_local std::string t_last_error;

gi_status fail(gi_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  t_last_error = std::string(gi_status_string(s)) + ": " + buf;
  return s;
}

gi_status cuda_fail(cudaError_t e, const char* what) {
  if (e == cudaErrorMemoryAllocation) return fail(GI_ERR_OUT_OF_MEMORY, "%s: %s", what, cudaGetErrorString(e));
  return fail(GI_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

#define GI_CUDA(call, what)                       \
  do {                                            \
    cudaError_t e_ = (call);                      \
    if (e_ != cudaSuccess) return cuda_fail(e_, what); \
  } while (0)

// Is p device memory on `device`? (host / unregistered -> false)
bool is_device_ptr(const void* p, int device, bool* wrong_device) {
  *wrong_device = false;
  cudaPointerAttributes at;
  cudaError_t e = cudaPointerGetAttributes(&at, p);
  if (e != cudaSuccess) { cudaGetLastError(); return false; }
  if (at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged) {
    if (at.device != device) *wrong_device = true;
    return true;
  }
  return false;
}

// A group workspace and the device mirror of its pointers.
struct Workspace {
  int64_t n = 0;
  int cap_groups = 0;
  uint32_t hubcap = 0;
  std::vector<void*> allocs;
  std::vector<GroupWs> h_groups;
  GroupWs* d_groups = nullptr;
  QStats* d_qstats = nullptr;
  int qcap = 0;
  int32_t* d_srcs = nullptr;
  int srccap = 0;
  uint32_t* d_stage = nullptr;  // staging for host dist_out
  size_t stagecap = 0;
  uint32_t* d_src_next = nullptr;  // batch source claim counter
  int32_t* h_srcs = nullptr;     // pinned staging: sources (H2D) and statistics (D2H), so the
  QStats* h_qstats = nullptr;    // per-call copies are asynchronous (no pageable staging)
  int hcap_q = 0;
  uint32_t** d_peers = nullptr;  // gi_sssp_batch_peers: device copy of the peer row bases
  int peercap = 0;
  uint32_t* h_pending = nullptr;  // pinned: KState.pending of a split query, read between segments
  uint8_t* d_mirror = nullptr;    // expand: 1-byte saturated copy of dist [n] (KArgs.mirror)
  uint32_t* d_h = nullptr;      // staging for a host A* heuristic
  size_t hcap = 0;
  uint32_t* kc_prio = nullptr;  // k-core: priorities [n]
  KcCtl* kc_ctl = nullptr;
  KcStats* kc_stats = nullptr;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;

  ~Workspace() {
    for (void* p : allocs) cudaFree(p);
    if (d_groups) cudaFree(d_groups);
    if (d_qstats) cudaFree(d_qstats);
    if (d_srcs) cudaFree(d_srcs);
    if (d_stage) cudaFree(d_stage);
    if (d_h) cudaFree(d_h);
    if (d_peers) cudaFree(d_peers);
    if (h_srcs) cudaFreeHost(h_srcs);
    if (h_qstats) cudaFreeHost(h_qstats);
    if (h_pending) cudaFreeHost(h_pending);
    if (d_mirror) cudaFree(d_mirror);
    if (d_src_next) cudaFree(d_src_next);
    if (kc_prio) cudaFree(kc_prio);
    if (kc_ctl) cudaFree(kc_ctl);
    if (kc_stats) cudaFree(kc_stats);
    if (ev0) cudaEventDestroy(ev0);
    if (ev1) cudaEventDestroy(ev1);
    if (stream) cudaStreamDestroy(stream);
  }
};

}  // namespace

struct gi_graph {
  int device = 0;
  int64_t n = 0, m = 0;
  int64_t* d_off = nullptr;
  uint2* d_edges = nullptr;
  uint2* d_slots = nullptr;  // ELL adjacency slots, 64 B per vertex
  void* d_arena = nullptr;   // one allocation holding offsets, edges and slots (2 MB-aligned parts)

  uint32_t max_deg = 0;
  int64_t n_big = 0;             // vertices of out-degree > 8 (skewed graphs: expand list capacity)
  uint32_t* d_pedges = nullptr;  // packed edges (w << colbits | col), skewed graphs whose weights fit

  uint32_t colbits = 0;
  int sm_count = 0;
  int bps[2][KIND_COUNT] = {};  // co-resident CTAs per SM, by width (512, 1024) and KernelKind
  int bps_kcore = 0;
  std::mutex mu;
  std::vector<std::unique_ptr<Workspace>> pool;

  // device memory is released here, so that every early error return of gi_graph_create
  // (the unique_ptr going out of scope) frees what was allocated; the caller's current
  // device is the graph's (DeviceGuard) wherever this runs
  ~gi_graph() {
    pool.clear();
    if (d_pedges) cudaFree(d_pedges);
    if (d_arena) {
      cudaFree(d_arena);
    } else {
      if (d_off) cudaFree(d_off);
      if (d_edges) cudaFree(d_edges);
      if (d_slots) cudaFree(d_slots);
    }
  }
};

namespace {

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int d) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    cudaSetDevice(d);
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

template <typename T>
gi_status dmalloc(T** p, size_t count, std::vector<void*>* track, const char* what) {
  void* q = nullptr;
  GI_CUDA(cudaMalloc(&q, count * sizeof(T) + 16), what);
  *p = (T*)q;
  if (track) track->push_back(q);
  return GI_OK;
}

// Group hub-list capacity: every hub (deg >= 256) twice over, and on skewed graphs (expand)
// every vertex of degree > 8 once more; entries past the capacity are relaxed CTA-locally.
uint32_t hub_capacity(const gi_graph* g) {
  int64_t cap = 2 * (g->m / kMinHubMin) + 64;
  if (g->max_deg > 32) cap = std::max<int64_t>(cap, g->n_big + 2 * (g->m / kMinHubMin) + 64);
  return (uint32_t)std::min<int64_t>(cap, 0x7FFFFFFF);
}

// Make a workspace with >= k groups, >= nsrc stats slots.
gi_status ws_prepare(gi_graph* g, Workspace* w, int k, int nsrc) {
  const int64_t n = g->n;
  const size_t nwords = (size_t)((n + 31) / 32);
  w->n = n;
  // a vertex with deg >= kMinHubMin can appear at most m / kMinHubMin times ... per distinct
  // vertex; twice that covers re-queued entries, the rest fall back to CTA-local processing
  w->hubcap = hub_capacity(g);
  if (!w->stream) {
    // a BLOCKING stream: work on it is ordered with the legacy default stream, where torch
    // (and most callers) queue the kernels that produce the inputs and consume dist_out
    GI_CUDA(cudaStreamCreateWithFlags(&w->stream, cudaStreamDefault), "cudaStreamCreate");
    GI_CUDA(cudaEventCreate(&w->ev0), "cudaEventCreate");
    GI_CUDA(cudaEventCreate(&w->ev1), "cudaEventCreate");
  }
  if (w->cap_groups < k) {
    for (int gi_ = w->cap_groups; gi_ < k; ++gi_) {
      GroupWs gw;
      gi_status s;
      if ((s = dmalloc(&gw.farbits, nwords, &w->allocs, "alloc farbits"))) return s;
      if ((s = dmalloc(&gw.qbits[0], nwords, &w->allocs, "alloc qbits"))) return s;
      if ((s = dmalloc(&gw.qbits[1], nwords, &w->allocs, "alloc qbits"))) return s;
      if ((s = dmalloc(&gw.ovfbits, nwords, &w->allocs, "alloc ovfbits"))) return s;
      if ((s = dmalloc(&gw.far[0], (size_t)n, &w->allocs, "alloc far"))) return s;
      if ((s = dmalloc(&gw.far[1], (size_t)n, &w->allocs, "alloc far"))) return s;
      if ((s = dmalloc(&gw.q[0], (size_t)n, &w->allocs, "alloc q"))) return s;
      if ((s = dmalloc(&gw.q[1], (size_t)n, &w->allocs, "alloc q"))) return s;
      if ((s = dmalloc(&gw.ctl, 1, &w->allocs, "alloc ctl"))) return s;
      if ((s = dmalloc(&gw.hub[0], (size_t)w->hubcap, &w->allocs, "alloc hub list"))) return s;
      if ((s = dmalloc(&gw.hub[1], (size_t)w->hubcap, &w->allocs, "alloc hub list"))) return s;
      gw.xpre = nullptr;
      gw.xtot = nullptr;
      gw.laterbits = nullptr;  // the bucket window's later pile: allocated on first use
      gw.later[0] = gw.later[1] = nullptr;
      if ((s = dmalloc(&gw.kst, 1, &w->allocs, "alloc expand state"))) return s;
      GI_CUDA(cudaMemsetAsync(gw.kst, 0, sizeof(KState), w->stream), "memset");
      if (g->max_deg > 32) {  // expand (skewed graphs)
        if ((s = dmalloc(&gw.xpre, (size_t)w->hubcap, &w->allocs, "alloc expand prefix"))) return s;
        if ((s = dmalloc(&gw.xtot, (size_t)kMaxGroupCtas, &w->allocs, "alloc expand totals"))) return s;
      }
      // bitmaps start (and, after every completed query, end) all-zero
      GI_CUDA(cudaMemsetAsync(gw.farbits, 0, nwords * 4, w->stream), "memset");
      GI_CUDA(cudaMemsetAsync(gw.qbits[0], 0, nwords * 4, w->stream), "memset");
      GI_CUDA(cudaMemsetAsync(gw.qbits[1], 0, nwords * 4, w->stream), "memset");
      GI_CUDA(cudaMemsetAsync(gw.ovfbits, 0, nwords * 4, w->stream), "memset");
      GI_CUDA(cudaMemsetAsync(gw.ctl, 0, sizeof(Ctl), w->stream), "memset");
      w->h_groups.push_back(gw);
    }
    if (w->d_groups) cudaFree(w->d_groups);
    w->d_groups = nullptr;
    GI_CUDA(cudaMalloc(&w->d_groups, sizeof(GroupWs) * k), "alloc groups");
    GI_CUDA(cudaMemcpyAsync(w->d_groups, w->h_groups.data(), sizeof(GroupWs) * k, cudaMemcpyHostToDevice,
                            w->stream), "copy groups");
    w->cap_groups = k;
  }
  if (w->qcap < nsrc) {
    if (w->d_qstats) cudaFree(w->d_qstats);
    w->d_qstats = nullptr;
    GI_CUDA(cudaMalloc(&w->d_qstats, sizeof(QStats) * nsrc), "alloc qstats");
    w->qcap = nsrc;
  }
  if (w->srccap < nsrc) {
    if (w->d_srcs) cudaFree(w->d_srcs);
    w->d_srcs = nullptr;
    GI_CUDA(cudaMalloc(&w->d_srcs, sizeof(int32_t) * nsrc), "alloc srcs");
    w->srccap = nsrc;
  }
  return GI_OK;
}

Workspace* ws_acquire(gi_graph* g) {
  std::lock_guard<std::mutex> lk(g->mu);
  if (!g->pool.empty()) {
    Workspace* w = g->pool.back().release();
    g->pool.pop_back();
    return w;
  }
  return new Workspace();
}

void ws_release(gi_graph* g, Workspace* w, bool healthy) {
  if (!healthy) {  // a failed query may leave dirty bitmaps: drop the workspace
    delete w;
    return;
  }
  std::lock_guard<std::mutex> lk(g->mu);
  g->pool.emplace_back(w);
}

void fill_stats(gi_stats* st, const QStats& q, float ms, int ctas, int groups, int kind, int threads,
                int launches, int rung) {
  st->rung = rung;
  st->buckets = q.buckets;
  st->rounds = q.rounds;
  st->grid_syncs = q.phases;
  st->kernel_launches = launches;
  st->fused_subrounds = q.subrounds;
  st->spills = q.spills;
  st->vertices_processed = q.vertices;
  st->edges_relaxed = q.edges;
  st->empty_extractions = q.empty_extr;
  st->far_scanned = q.far_scanned;
  st->critical_subrounds = q.critical_subrounds;
  st->gpu_ms = ms;
  st->ctas = ctas;
  st->threads_per_cta = threads;
  st->groups = groups;
  st->kernel_kind = kind;
}

gi_status run_queries(const gi_graph* cg_, const int32_t* srcs, int32_t nsrc, uint32_t delta,
                      const gi_options* opt_in, uint32_t* dist_out, gi_stats* stats, bool batch,
                      int32_t target = -1, const uint32_t* heur = nullptr,
                      uint32_t* const* peer_rows = nullptr, int32_t npeers = 0) {
  gi_graph* g = const_cast<gi_graph*>(cg_);
  if (!g) return fail(GI_ERR_INVALID_ARGUMENT, "graph is NULL");
  if (nsrc < 0) return fail(GI_ERR_INVALID_ARGUMENT, "nsrc < 0");
  if (nsrc == 0) return GI_OK;
  if (!srcs || !dist_out) return fail(GI_ERR_INVALID_ARGUMENT, "NULL srcs or dist_out");
  if (delta == 0) return fail(GI_ERR_INVALID_ARGUMENT, "delta must be >= 1");
  gi_options opt;
  gi_options_default(&opt);
  if (opt_in) {
    if (opt_in->struct_size != sizeof(gi_options))
      return fail(GI_ERR_INVALID_ARGUMENT, "gi_options.struct_size mismatch");
    opt = *opt_in;
  }
  if (opt.max_ctas < 0 || opt.group_ctas < 0) return fail(GI_ERR_INVALID_ARGUMENT, "negative CTA count");
  DeviceGuard dg(g->device);

  // sources -> host copy for range checks
  std::vector<int32_t> hsrc(nsrc);
  bool wrongdev = false;
  if (is_device_ptr(srcs, g->device, &wrongdev)) {
    if (wrongdev) return fail(GI_ERR_INVALID_ARGUMENT, "srcs on another device");
    GI_CUDA(cudaMemcpy(hsrc.data(), srcs, sizeof(int32_t) * nsrc, cudaMemcpyDeviceToHost), "copy srcs");
  } else {
    memcpy(hsrc.data(), srcs, sizeof(int32_t) * nsrc);
  }
  for (int i = 0; i < nsrc; ++i)
    if (hsrc[i] < 0 || hsrc[i] >= g->n)
      return fail(GI_ERR_OUT_OF_RANGE, "source %d not in [0, %lld)", hsrc[i], (long long)g->n);
  if (target >= 0 && target >= g->n)
    return fail(GI_ERR_OUT_OF_RANGE, "target %d not in [0, %lld)", target, (long long)g->n);
  const bool dev_out = is_device_ptr(dist_out, g->device, &wrongdev);
  if (wrongdev) return fail(GI_ERR_INVALID_ARGUMENT, "dist_out on another device");
  const bool ppsp = target >= 0;  // dist_out is ONE value; the distances live in the workspace
  if (npeers > 0 && !dev_out)
    return fail(GI_ERR_INVALID_ARGUMENT, "peer_rows[self] must be device memory on the graph's device");

  const bool fused = opt.fusion != 0;
  if (opt.drain > 2) return fail(GI_ERR_INVALID_ARGUMENT, "drain must be 0 (auto), 1 (bsp) or 2 (async)");
  if (opt.expand < 0 || opt.expand > 2) return fail(GI_ERR_INVALID_ARGUMENT, "expand must be 0 (auto), 1 (on) or 2 (off)");
  if (opt.lazy != 0 && opt.lazy != 1) return fail(GI_ERR_INVALID_ARGUMENT, "lazy must be 0 or 1");
  if (opt.rung < 0 || opt.rung > 3) return fail(GI_ERR_INVALID_ARGUMENT, "rung must be 0 (auto), 1 (cta), 2 (cluster) or 3 (grid)");
  if (opt.rung == 2 && (opt.group_ctas < 0 || opt.group_ctas > 16))
    return fail(GI_ERR_INVALID_ARGUMENT, "a cluster group has at most 16 CTAs");
  if (opt.window < 0) return fail(GI_ERR_INVALID_ARGUMENT, "window must be >= 0 (0 = off)");
  if (opt.lazy && opt.fusion) return fail(GI_ERR_INVALID_ARGUMENT, "the lazy schedule runs without fusion (fusion = 0)");
  if (heur && fused && opt.drain == 2) return fail(GI_ERR_UNSUPPORTED, "A* runs with the bsp drain (drain 0/1)");
  if (fused && opt.drain == 2 && g->max_deg > kAsyncMaxDeg)
    return fail(GI_ERR_UNSUPPORTED, "async drain needs max out-degree <= %u (graph has %u)", kAsyncMaxDeg,
                g->max_deg);
  // default: the CTA-barrier (BSP) drain with the degree-binned stages; the barrier-free
  // async drain (every adjacency inline in its ELL slot) is opt-in — measured slower on
  // configs 1-2, kept as the comparison point
  int kind = !fused ? KIND_UNFUSED : opt.drain == 2 ? KIND_FUSED_ASYNC : KIND_FUSED_BSP;
  // low-degree specialisation: every adjacency inline in its slot and no pre-read
  const bool lowdeg = g->max_deg <= kAsyncMaxDeg && opt.pre_read != 1;
  if (lowdeg && kind == KIND_UNFUSED) kind = KIND_UNFUSED_LD;
  if (lowdeg && kind == KIND_FUSED_BSP) kind = KIND_FUSED_BSP_LD;
  // CTA width: 1024 threads on skewed graphs (memory-level parallelism in stage B),
  // 512 otherwise (the latency-bound chains of road graphs); gi_options.cta_threads overrides
  if (opt.cta_threads != 0 && opt.cta_threads != 512 && opt.cta_threads != 1024)
    return fail(GI_ERR_INVALID_ARGUMENT, "cta_threads must be 0, 512 or 1024");
  // (a batch of >= 8 sources is throughput-bound: 1024 threads there too — config 5,
  // 64 sources: 207 ms against 225 ms with 512)
  const int wide = opt.cta_threads ? (opt.cta_threads == 1024) : (g->max_deg > 32 || (batch && nsrc >= 8) ? 1 : 0);
  const int bps = g->bps[wide][kind];
  int total = g->sm_count * bps;
  // group sizing: single source -> one group of every CTA (capped by max_ctas);
  // batch -> several groups in flight, each of group_ctas CTAs
  int G, ngroups;
  Workspace* w = ws_acquire(g);
  if (!batch || nsrc == 1) {
    G = total;
    if (opt.max_ctas > 0 && opt.max_ctas < G) G = opt.max_ctas;
    ngroups = 1;
  } else {
    if (opt.group_ctas > 0) {
      G = opt.group_ctas;
    } else {
      // auto: one group per source, so the batch runs in one wave (a partial last wave
      // leaves most SMs idle while it runs), with at least 2 CTAs per group, and no more
      // groups than half the free device memory holds workspaces for. Measured on config
      // 5 (64 sources): 2 CTAs x 64 groups 228 ms, 16 x 9 258 ms, 3 x 49 266 ms.
      G = std::max(2, total / nsrc);
      const int64_t nw = (g->n + 31) / 32;
      const int64_t hubcap = hub_capacity(g);
      const size_t per = (size_t)(16 * g->n + 16 * nw) + 2 * (size_t)hubcap * sizeof(HubEnt) +
                         (g->max_deg > 32 ? (size_t)hubcap * 8 : 0) + sizeof(Ctl);
      size_t free_b = 0, total_b = 0;
      // (cudaMemGetInfo costs milliseconds: asked only when new workspaces are needed)
      const int want = std::min(total / G, nsrc);
      if (want > w->cap_groups && cudaMemGetInfo(&free_b, &total_b) == cudaSuccess) {
        const int maxg = w->cap_groups + std::max<int64_t>(1, (int64_t)(free_b / 2 / per));
        if (total / G > maxg) G = (total + maxg - 1) / maxg;
      }
    }
    if (opt.max_ctas > 0 && opt.max_ctas < G) G = opt.max_ctas;
    if (G > total) G = total;
    ngroups = total / G;
    if (ngroups > nsrc) ngroups = nsrc;
    if (ngroups < 1) ngroups = 1;
  }

  // execution-group rung: a one-CTA group or one cluster per group. Auto:
  // a small graph's single query runs on one 16-CTA cluster (config 1: 1.44 ms against 1.50
  // on the whole grid and 1.54 on a 16-CTA grid group), a batch whose groups are <= 16 CTAs
  // runs one cluster per group (config 5: 146.8 against 149.2 ms); everything else the grid
  int rung = opt.rung == 1 ? 1 : opt.rung == 2 ? 2 : 0;
  int auto_cl = 0;
  if (opt.rung == 0) {
    if (!batch && g->n <= (1 << 18) && opt.max_ctas == 0 && opt.group_ctas == 0) auto_cl = 16;
    else if (batch && nsrc > 1 && G <= 16 && G >= 2) auto_cl = G;
    if (auto_cl) {
      int maxc = 0;
      cudaError_t qe = wide ? v1024::query_clusters(kind, auto_cl, &maxc) : v512::query_clusters(kind, auto_cl, &maxc);
      if (qe == cudaSuccess && maxc >= (batch ? std::min(ngroups, nsrc) : 1)) rung = 2;
      else cudaGetLastError();
    }
  }
  if (rung == 1) {
    G = 1;
    ngroups = batch ? std::min(nsrc, total) : 1;
  } else if (rung == 2) {
    const int cl = auto_cl ? auto_cl : opt.group_ctas > 0 ? opt.group_ctas : 8;
    int maxc = 0;
    cudaError_t qe = wide ? v1024::query_clusters(kind, cl, &maxc) : v512::query_clusters(kind, cl, &maxc);
    if (qe != cudaSuccess || maxc < 1) {
      cudaGetLastError();
      ws_release(g, w, true);
      return fail(GI_ERR_UNSUPPORTED, "clusters of %d CTAs of this kernel cannot be resident", cl);
    }
    G = cl;
    ngroups = batch ? std::min(auto_cl ? ngroups : nsrc, maxc) : 1;  // auto keeps the memory cap
  }
  gi_status s = ws_prepare(g, w, ngroups, nsrc);
  if (s) { ws_release(g, w, false); return s; }
  cudaStream_t st = opt.cuda_stream ? (cudaStream_t)opt.cuda_stream : w->stream;
  if (opt.cuda_stream) {
    // setup work queued on the workspace stream must precede the caller's stream
    cudaEvent_t e;
    cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    cudaEventRecord(e, w->stream);
    cudaStreamWaitEvent(st, e, 0);
    cudaEventDestroy(e);
  }

  uint32_t* d_dist = dist_out;
  const size_t total_elems = (size_t)nsrc * (size_t)g->n;
  auto bail = [&](cudaError_t e, const char* what) {
    cudaStreamSynchronize(st);
    ws_release(g, w, false);
    return cuda_fail(e, what);
  };
  cudaError_t e;
  if (!dev_out || ppsp) {
    if (w->stagecap < total_elems) {
      if (w->d_stage) cudaFree(w->d_stage);
      w->d_stage = nullptr;
      w->stagecap = 0;
      if ((e = cudaMalloc(&w->d_stage, total_elems * 4)) != cudaSuccess) return bail(e, "alloc dist stage");
      w->stagecap = total_elems;
    }
    d_dist = w->d_stage;
  }
  const uint32_t* d_h = nullptr;  // A*: the heuristic on the device (caller's or staged)
  if (heur) {
    bool hwrong = false;
    if (is_device_ptr(heur, g->device, &hwrong)) {
      if (hwrong) { ws_release(g, w, true); return fail(GI_ERR_INVALID_ARGUMENT, "h on another device"); }
      d_h = heur;
    } else {
      if (w->hcap < (size_t)g->n) {
        if (w->d_h) cudaFree(w->d_h);
        w->d_h = nullptr;
        w->hcap = 0;
        if ((e = cudaMalloc(&w->d_h, (size_t)g->n * 4)) != cudaSuccess) return bail(e, "alloc heuristic");
        w->hcap = (size_t)g->n;
      }
      if ((e = cudaMemcpyAsync(w->d_h, heur, (size_t)g->n * 4, cudaMemcpyHostToDevice, st)))
        return bail(e, "copy heuristic");
      d_h = w->d_h;
    }
  }
  if (w->hcap_q < nsrc) {
    if (w->h_srcs) cudaFreeHost(w->h_srcs);
    if (w->h_qstats) cudaFreeHost(w->h_qstats);
    w->h_srcs = nullptr;
    w->h_qstats = nullptr;
    w->hcap_q = 0;
    if ((e = cudaMallocHost(&w->h_srcs, sizeof(int32_t) * nsrc)) != cudaSuccess) return bail(e, "alloc pinned srcs");
    if ((e = cudaMallocHost(&w->h_qstats, sizeof(QStats) * nsrc)) != cudaSuccess) return bail(e, "alloc pinned stats");
    w->hcap_q = nsrc;
  }
  memcpy(w->h_srcs, hsrc.data(), sizeof(int32_t) * nsrc);
  if ((e = cudaMemcpyAsync(w->d_srcs, w->h_srcs, sizeof(int32_t) * nsrc, cudaMemcpyHostToDevice, st)))
    return bail(e, "copy srcs");
  if ((e = cudaMemsetAsync(w->d_qstats, 0, sizeof(QStats) * nsrc, st))) return bail(e, "memset qstats");
  if (!w->d_src_next && (e = cudaMalloc(&w->d_src_next, sizeof(uint32_t)))) return bail(e, "alloc claim counter");

  KArgs a;
  a.slots = g->d_slots;
  a.edges = g->d_edges;
  a.n = g->n;
  a.nwords = (uint32_t)((g->n + 31) / 32);
  a.srcs = w->d_srcs;
  a.nsrc = nsrc;
  a.dist = d_dist;
  a.groups = w->d_groups;
  a.qstats = w->d_qstats;
  a.ngroups = ngroups;
  a.group_size = G;
  a.div = make_fastdiv(delta);
  a.hub_min = opt.hub_min ? std::max(opt.hub_min, kMinHubMin) : kDefaultHubMin;
  a.hubcap = w->hubcap;
  // threshold: a throughput-bound batch (>= 8 sources, small groups) keeps whole bins local
  // up to the bin capacity (every spill costs a group round trip through the global frontier;
  // config 5: T = 2048 183 ms against 207 ms at 1024, and 160 ms with T = 4096 in the
  // 1024-thread kernel's bins); single queries use the measured defaults
  const bool throughput = batch && nsrc >= 8;
  a.T = opt.fusion_threshold ? opt.fusion_threshold
                             : (g->max_deg > 32 ? kDefaultTSkewed : throughput ? (uint32_t)kBinCapW[wide] : kDefaultT);
  if (a.T > (uint32_t)kBinCapW[wide]) a.T = kBinCapW[wide];
  if (kind == KIND_FUSED_ASYNC && a.T > kRingSafeW[wide]) a.T = kRingSafeW[wide];
  // pre-read dist[v] before the atomic: pays off when hubs attract many redundant
  // relaxations (skewed degrees), costs one L2 round trip per level otherwise
  a.pre_read = opt.pre_read == 1 ? 1u : opt.pre_read == 2 ? 0u : (g->max_deg > 32 ? 1u : 0u);
  a.target = target;
  a.dyn_claim = g->max_deg > 32 ? 1u : 0u;
  // expand needs the group list's prefix workspace (skewed graphs) and fits groups of <= 1024 CTAs
  // expand (opt-in, single queries on skewed graphs): every ROUND phase collects its
  // high-degree frontier into the group list, and lists of >= split_min edges are relaxed by
  // expand_kernel between two segments of the persistent kernel (KState); lighter lists are
  // relaxed slice-wise in the kernel. Measured against the default CTA-level stage B on
  // configs 3-4 it is not faster, so the default stays off.
  // auto (0): on for skewed graphs of >= 512 M edges, whose heavy phases it speeds up
  // (config 4: 33.8 -> 28.8 ms); smaller ones pay more for the stops than they gain (config 3:
  // 1.87 -> 2.5 ms)
  const bool expand_auto = opt.expand == 0 && g->m >= (512ll << 20);
  a.expand = (g->max_deg > 32 && (opt.expand == 1 || expand_auto) && G <= kMaxGroupCtas && ngroups == 1 &&
              nsrc == 1 && kind != KIND_FUSED_ASYNC) ? 1u : 0u;
  a.pedges = g->d_pedges;
  a.colbits = g->colbits;
  a.split = a.expand;
  a.lazy = opt.lazy ? 1u : 0u;
  a.rung = (uint32_t)rung;
  a.resume = 0;
  {
    const char* sm = getenv("GI_SPLIT_MIN");
    // lists of fewer edges are relaxed in the persistent kernel (a stop costs ~40 µs)
    a.split_min = sm ? strtoull(sm, nullptr, 10) : (1ull << 20);
    // big extractions too run outside (extract_kernel), from 2^21 pile entries (GI_XSPLIT_MIN;
    // 0 keeps every extraction in the persistent kernel)
    const char* xm = getenv("GI_XSPLIT_MIN");
    a.xsplit_min = xm ? (uint32_t)strtoul(xm, nullptr, 10) : (1u << 21);
  }
  if (a.expand) {
    const int xk = kind == KIND_UNFUSED ? KIND_UNFUSED_XP : KIND_FUSED_BSP_XP;
    if (g->bps[wide][xk] >= bps) kind = xk;  // same co-residency as the kernel G was sized for
    else a.expand = a.split = 0;
  }
  if (!a.split) a.xsplit_min = 0;
  if ((e = cudaMemsetAsync(w->d_src_next, 0, sizeof(uint32_t), st))) return bail(e, "init claim counter");
  a.src_next = w->d_src_next;  // claims count from 0; sources 0..ngroups-1 are taken statically
  a.h = d_h;
  a.peers = nullptr;
  a.npeers = 0;
  a.peer_vec = 0;
  if (npeers > 0) {
    if (w->peercap < npeers) {
      if (w->d_peers) cudaFree(w->d_peers);
      w->d_peers = nullptr;
      w->peercap = 0;
      if ((e = cudaMalloc(&w->d_peers, sizeof(uint32_t*) * npeers)) != cudaSuccess) return bail(e, "alloc peers");
      w->peercap = npeers;
    }
    if ((e = cudaMemcpyAsync(w->d_peers, peer_rows, sizeof(uint32_t*) * npeers, cudaMemcpyHostToDevice, st)))
      return bail(e, "copy peers");
    bool vec = g->n % 4 == 0;
    for (int i = 0; i < npeers; ++i) vec = vec && ((uintptr_t)peer_rows[i] % 16 == 0);
    a.peers = w->d_peers;
    a.npeers = npeers;
    a.peer_vec = vec ? 1u : 0u;
  }

  if (a.split && !w->h_pending) {
    if ((e = cudaMallocHost(&w->h_pending, sizeof(uint32_t))) != cudaSuccess) return bail(e, "alloc pinned flag");
  }
  // bucket window (split queries): far entries beyond the open window wait in a later pile
  a.window = 0;
  a.window_pile = 0;
  if (a.split) {
    const char* wv = getenv("GI_WINDOW");  // investigation override (buckets; 0 = off)
    a.window = wv ? (uint32_t)strtoul(wv, nullptr, 10) : opt.window ? (uint32_t)opt.window : (uint32_t)kDefaultWindow;
    const char* wp = getenv("GI_WINDOW_PILE");  // investigation: open the window late
    a.window_pile = wp ? (uint32_t)strtoul(wp, nullptr, 10) : 0u;
    GroupWs& g0 = w->h_groups[0];
    if (a.window && !g0.laterbits) {
      const size_t nwords = (size_t)((g->n + 31) / 32);
      gi_status s2;
      if ((s2 = dmalloc(&g0.laterbits, nwords, &w->allocs, "alloc laterbits")) ||
          (s2 = dmalloc(&g0.later[0], (size_t)g->n, &w->allocs, "alloc later pile")) ||
          (s2 = dmalloc(&g0.later[1], (size_t)g->n, &w->allocs, "alloc later pile"))) {
        g0.laterbits = nullptr;
        return s2;
      }
      if ((e = cudaMemsetAsync(g0.laterbits, 0, nwords * 4, st)) ||
          (e = cudaMemcpyAsync(w->d_groups, &g0, sizeof(GroupWs), cudaMemcpyHostToDevice, st)))
        return bail(e, "init later pile");
    }
  }
  // the expand pre-read filter (KArgs.mirror): every byte 0xFF ("unknown") at query start
  a.mirror = nullptr;
  if (a.split) {
    const char* mv = getenv("GI_MIRROR");  // investigation: GI_MIRROR=0 pre-reads dist itself
    if (!mv || atoi(mv) != 0) {
      if (!w->d_mirror && (e = cudaMalloc(&w->d_mirror, (size_t)g->n)) != cudaSuccess) return bail(e, "alloc mirror");
      a.mirror = w->d_mirror;
    }
  }
  // investigation (GI_L2_PERSIST=1): dist as a persisting L2 access-policy window on the
  // query's stream, so that the slot stream cannot evict the wavefront's distances
  bool l2win = false;
  if (const char* lp = getenv("GI_L2_PERSIST")) {
    if (atoi(lp) > 0) {
      int maxwin = 0, maxpers = 0;
      cudaDeviceGetAttribute(&maxwin, cudaDevAttrMaxAccessPolicyWindowSize, g->device);
      cudaDeviceGetAttribute(&maxpers, cudaDevAttrMaxPersistingL2CacheSize, g->device);
      const size_t bytes = std::min((size_t)total_elems * 4, (size_t)maxwin);
      cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)maxpers);
      cudaStreamAttrValue at = {};
      at.accessPolicyWindow.base_ptr = d_dist;
      at.accessPolicyWindow.num_bytes = bytes;
      at.accessPolicyWindow.hitRatio = std::min(1.0f, (float)maxpers / (float)std::max<size_t>(bytes, 1));
      at.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
      at.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
      if (cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &at) == cudaSuccess) l2win = true;
      static bool said = false;
      if (!said) { fprintf(stderr, "gi: L2 window %zu B (max window %d, max persisting %d)\n", bytes, maxwin, maxpers); said = true; }
      cudaGetLastError();
    }
  }
  if ((e = cudaEventRecord(w->ev0, st))) return bail(e, "event");
  if (a.mirror && (e = cudaMemsetAsync(a.mirror, 0xFF, (size_t)g->n, st))) return bail(e, "init mirror");
  if ((e = wide ? v1024::launch_sssp(a, kind, G * ngroups, st) : v512::launch_sssp(a, kind, G * ngroups, st)))
    return bail(e, "launch sssp_persistent");
  int launches = 1;
  if (a.split) {
    // the persistent kernel stops at every heavy expand or extraction (KState.pending = 1 /
    // 2): run the outside kernel, then resume the persistent kernel at the same phase (it
    // clears the flag when the query ends). The kernels also check the flag themselves, so
    // a round may be enqueued before the flag is known; batching rounds that way (one host
    // round trip per batch of stops) measured no faster on config 4 (20.35 vs 20.28 ms):
    // the GPU is not idle on the host's round trip. So the host reads the flag at every stop
    // and launches only the pending kernel.
    KState* kst = w->h_groups[0].kst;
    KArgs ar = a;
    ar.resume = 1;
    const char* dump = getenv("GI_DUMP_X");  // investigation only: the pending list to files
    for (;;) {
      if ((e = cudaMemcpyAsync(w->h_pending, &kst->pending, sizeof(uint32_t), cudaMemcpyDeviceToHost, st)) ||
          (e = cudaStreamSynchronize(st)))
        return bail(e, "sssp kernel segment");
      if (!*w->h_pending) break;
      if (dump && *w->h_pending == 1) {
        KState hk;
        cudaMemcpy(&hk, kst, sizeof(hk), cudaMemcpyDeviceToHost);
        static int seq = 0;
        std::vector<HubEnt> hx(hk.xn);
        const GroupWs& gw = w->h_groups[0];
        cudaMemcpy(hx.data(), (hk.p & 1) ? gw.hub[1] : gw.hub[0], sizeof(HubEnt) * hk.xn, cudaMemcpyDeviceToHost);
        char fn[512];
        snprintf(fn, sizeof(fn), "%s_%d_p%u_b%u_E%llu.bin", dump, seq++, hk.p, hk.b, (unsigned long long)hk.E);
        if (FILE* f = fopen(fn, "wb")) {
          fwrite(hx.data(), sizeof(HubEnt), hx.size(), f);
          fclose(f);
        }
        std::vector<uint32_t> hd((size_t)g->n);  // the distances at this point
        cudaMemcpy(hd.data(), d_dist, 4 * (size_t)g->n, cudaMemcpyDeviceToHost);
        snprintf(fn, sizeof(fn), "%s_%d_dist.bin", dump, seq - 1);
        if (FILE* f = fopen(fn, "wb")) {
          fwrite(hd.data(), 4, hd.size(), f);
          fclose(f);
        }
      }
      if (*w->h_pending == 2) {
        if ((e = v1024::launch_extract(a, st))) return bail(e, "launch extract_kernel");
      } else if ((e = v1024::launch_expand(a, st, nullptr))) {
        return bail(e, "launch expand_kernel");
      }
      if ((e = wide ? v1024::launch_sssp(ar, kind, G * ngroups, st) : v512::launch_sssp(ar, kind, G * ngroups, st)))
        return bail(e, "resume sssp_persistent");
      launches += 2;
    }
  }
  if ((e = cudaEventRecord(w->ev1, st))) return bail(e, "event");
  if (l2win) {
    cudaStreamAttrValue at = {};
    at.accessPolicyWindow.num_bytes = 0;
    cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &at);
    cudaCtxResetPersistingL2Cache();
  }
  QStats* hq = w->h_qstats;
  if ((e = cudaMemcpyAsync(hq, w->d_qstats, sizeof(QStats) * nsrc, cudaMemcpyDeviceToHost, st)))
    return bail(e, "copy stats");
  if (ppsp) {
    if ((e = cudaMemcpyAsync(dist_out, d_dist + target, 4, dev_out ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                             st)))
      return bail(e, "copy dist[target]");
  } else if (!dev_out) {
    if ((e = cudaMemcpyAsync(dist_out, d_dist, total_elems * 4, cudaMemcpyDeviceToHost, st)))
      return bail(e, "copy dist");
  }
  if ((e = cudaStreamSynchronize(st))) return bail(e, "sssp kernel");
  float ms = 0.f;
  cudaEventElapsedTime(&ms, w->ev0, w->ev1);
  bool ovf = false;
  for (int i = 0; i < nsrc; ++i) {  // hq is the workspace's pinned buffer: read before release
    if (hq[i].overflow) ovf = true;
    if (stats)
      fill_stats(&stats[i], hq[i], ms, G, ngroups, base_kind(kind), wide ? 1024 : 512, launches,
                 a.rung == 1 ? 1 : a.rung == 2 ? 2 : 3);
  }
  ws_release(g, w, true);
  if (ovf) return fail(GI_ERR_OVERFLOW, "a reachable vertex has distance >= UINT32_MAX");
  return GI_OK;
}

}  // namespace

extern "C" {

const char* gi_status_string(gi_status s) {
  switch (s) {
    case GI_OK: return "GI_OK";
    case GI_ERR_INVALID_ARGUMENT: return "GI_ERR_INVALID_ARGUMENT";
    case GI_ERR_OUT_OF_RANGE: return "GI_ERR_OUT_OF_RANGE";
    case GI_ERR_INVALID_GRAPH: return "GI_ERR_INVALID_GRAPH";
    case GI_ERR_OUT_OF_MEMORY: return "GI_ERR_OUT_OF_MEMORY";
    case GI_ERR_CUDA: return "GI_ERR_CUDA";
    case GI_ERR_OVERFLOW: return "GI_ERR_OVERFLOW";
    case GI_ERR_UNSUPPORTED: return "GI_ERR_UNSUPPORTED";
  }
  return "GI_ERR_UNKNOWN";
}

const char* gi_last_error(void) { return t_last_error.c_str(); }

int32_t gi_version(void) { return GI_VERSION; }

void gi_options_default(gi_options* opt) {
  if (!opt) return;
  memset(opt, 0, sizeof(*opt));
  opt->struct_size = sizeof(gi_options);
  opt->fusion = 1;
}

gi_status gi_graph_create(int64_t n, int64_t m, const int64_t* row_offsets, const int32_t* col_idx,
                          const uint32_t* weights, int device, gi_graph** out) {
  if (!out) return fail(GI_ERR_INVALID_ARGUMENT, "out is NULL");
  *out = nullptr;
  if (n < 1 || n > 0x7FFFFFFFll) return fail(GI_ERR_INVALID_GRAPH, "n=%lld not in [1, 2^31-1]", (long long)n);
  if (m < 0 || m >= (1ll << 62)) return fail(GI_ERR_INVALID_GRAPH, "m=%lld out of range", (long long)m);
  if (!row_offsets || (m > 0 && (!col_idx || !weights)))
    return fail(GI_ERR_INVALID_ARGUMENT, "NULL CSR array");
  int ndev = 0;
  GI_CUDA(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
  if (device < 0 || device >= ndev) return fail(GI_ERR_CUDA, "device %d not present (%d devices)", device, ndev);
  cudaDeviceProp prop;
  GI_CUDA(cudaGetDeviceProperties(&prop, device), "cudaGetDeviceProperties");
  if (prop.major != 10 || prop.minor != 0)
    return fail(GI_ERR_CUDA, "device %d is sm_%d%d; this library is built for sm_100a only", device, prop.major,
                prop.minor);
  DeviceGuard dg(device);

  std::unique_ptr<gi_graph> g(new gi_graph());
  g->device = device;
  g->n = n;
  g->m = m;
  g->sm_count = prop.multiProcessorCount;
  GI_CUDA(kcore_occupancy(&g->bps_kcore), "occupancy");
  if (g->bps_kcore < 1) return fail(GI_ERR_CUDA, "k-core kernel cannot be resident");
  for (int k = 0; k < KIND_COUNT; ++k) {
    GI_CUDA(v512::query_occupancy(k, &g->bps[0][k]), "occupancy");
    GI_CUDA(v1024::query_occupancy(k, &g->bps[1][k]), "occupancy");
    if (g->bps[0][k] < 1 || g->bps[1][k] < 1)
      return fail(GI_ERR_CUDA, "persistent kernel variant %d cannot be resident", k);
  }

  cudaStream_t st;  // blocking: ordered with the legacy default stream (device input arrays)
  GI_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamDefault), "stream");
  struct StreamGuard { cudaStream_t s; ~StreamGuard() { cudaStreamSynchronize(s); cudaStreamDestroy(s); } } sg{st};

  uint32_t* d_bad = nullptr;
  GI_CUDA(cudaMalloc(&d_bad, 4), "alloc");
  struct FreeGuard { void* p; ~FreeGuard() { cudaFree(p); } } fb{d_bad};
  GI_CUDA(cudaMemsetAsync(d_bad, 0, 4, st), "memset");

  bool wrong = false;
  // offsets, edges and slots in ONE allocation (2 MB-aligned parts; GI_ARENA=0 disables)
  const char* arena_env = getenv("GI_ARENA");
  const bool arena = !(arena_env && arena_env[0] == '0');
  auto up2m = [](size_t b) { return (b + (2u << 20) - 1) & ~(size_t)((2u << 20) - 1); };
  const size_t b_off = up2m(sizeof(int64_t) * (n + 1)), b_edges = up2m(sizeof(uint2) * (m > 0 ? m : 1)),
               b_slots = up2m(sizeof(uint2) * 8 * (size_t)n);
  if (arena) {
    GI_CUDA(cudaMalloc(&g->d_arena, b_off + b_edges + b_slots), "alloc graph arena");
    g->d_off = reinterpret_cast<int64_t*>(g->d_arena);
    g->d_edges = reinterpret_cast<uint2*>(reinterpret_cast<char*>(g->d_arena) + b_off);
    g->d_slots = reinterpret_cast<uint2*>(reinterpret_cast<char*>(g->d_arena) + b_off + b_edges);
  } else {
    GI_CUDA(cudaMalloc(&g->d_off, sizeof(int64_t) * (n + 1)), "alloc offsets");
  }
  const bool off_dev = is_device_ptr(row_offsets, device, &wrong);
  if (wrong) return fail(GI_ERR_INVALID_ARGUMENT, "row_offsets on another device");
  GI_CUDA(cudaMemcpyAsync(g->d_off, row_offsets, sizeof(int64_t) * (n + 1),
                          off_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st), "copy offsets");
  GI_CUDA(launch_validate_offsets(g->d_off, n, m, d_bad, st), "validate offsets");

  if (!arena) GI_CUDA(cudaMalloc(&g->d_edges, sizeof(uint2) * (m > 0 ? m : 1)), "alloc edges");
  if (m > 0) {
    const bool c_dev = is_device_ptr(col_idx, device, &wrong);
    if (wrong) return fail(GI_ERR_INVALID_ARGUMENT, "col_idx on another device");
    const bool w_dev = is_device_ptr(weights, device, &wrong);
    if (wrong) return fail(GI_ERR_INVALID_ARGUMENT, "weights on another device");
    if (c_dev && w_dev) {
      GI_CUDA(launch_interleave(col_idx, weights, g->d_edges, m, n, d_bad, st), "interleave");
    } else {
      // stage host arrays through device chunks
      const int64_t chunk = std::min<int64_t>(m, 64ll << 20);
      int32_t* dc = nullptr;
      uint32_t* dw = nullptr;
      GI_CUDA(cudaMalloc(&dc, chunk * 4), "alloc stage");
      FreeGuard fc{dc};
      GI_CUDA(cudaMalloc(&dw, chunk * 4), "alloc stage");
      FreeGuard fw{dw};
      for (int64_t p = 0; p < m; p += chunk) {
        const int64_t k = std::min(chunk, m - p);
        GI_CUDA(cudaMemcpyAsync(dc, col_idx + p, k * 4, c_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                                st), "copy cols");
        GI_CUDA(cudaMemcpyAsync(dw, weights + p, k * 4, w_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                                st), "copy weights");
        GI_CUDA(launch_interleave(dc, dw, g->d_edges + p, k, n, d_bad, st), "interleave");
      }
      GI_CUDA(cudaStreamSynchronize(st), "graph upload");
    }
  }
  uint32_t bad = 0;
  GI_CUDA(cudaMemcpyAsync(&bad, d_bad, 4, cudaMemcpyDeviceToHost, st), "copy flag");
  GI_CUDA(cudaStreamSynchronize(st), "graph validation");
  if (!bad) {
    if (!arena) GI_CUDA(cudaMalloc(&g->d_slots, sizeof(uint2) * 8 * (size_t)n), "alloc slots");
    GI_CUDA(launch_build_slots(g->d_off, g->d_edges, g->d_slots, n, st), "build slots");
    uint32_t* d_maxdeg = d_bad;  // reuse the flag word
    GI_CUDA(cudaMemsetAsync(d_maxdeg, 0, 4, st), "memset");
    GI_CUDA(launch_max_degree(g->d_off, n, d_maxdeg, st), "max degree");
    GI_CUDA(cudaMemcpyAsync(&g->max_deg, d_maxdeg, 4, cudaMemcpyDeviceToHost, st), "copy max degree");
    GI_CUDA(cudaStreamSynchronize(st), "graph build");
    if (g->max_deg > 32) {
      // skewed graph: the expand list capacity, and packed edges when the weights fit the
      // bits a column id leaves free (config 4: 26-bit ids, weights < 26 < 2^6)
      unsigned long long* d_cnt = nullptr;
      GI_CUDA(cudaMalloc(&d_cnt, 16), "alloc");
      FreeGuard fcnt{d_cnt};
      GI_CUDA(cudaMemsetAsync(d_cnt, 0, 16, st), "memset");
      GI_CUDA(launch_count_big(g->d_off, n, d_cnt, st), "count high-degree vertices");
      uint32_t* d_mw = reinterpret_cast<uint32_t*>(d_cnt + 1);
      GI_CUDA(launch_max_weight(g->d_edges, m, d_mw, st), "max weight");
      unsigned long long hb[2] = {0, 0};
      GI_CUDA(cudaMemcpyAsync(hb, d_cnt, 16, cudaMemcpyDeviceToHost, st), "copy counts");
      GI_CUDA(cudaStreamSynchronize(st), "graph build");
      g->n_big = (int64_t)hb[0];
      const uint32_t max_w = (uint32_t)hb[1];
      uint32_t colbits = 1;
      while (colbits < 31 && (1ll << colbits) < n) ++colbits;
      const char* pk = getenv("GI_PACK");
      const bool want_pack = !(pk && pk[0] == '0');
      if (want_pack && m > 0 && ((uint64_t)max_w >> (32 - colbits)) == 0) {
        GI_CUDA(cudaMalloc(&g->d_pedges, sizeof(uint32_t) * (size_t)m), "alloc packed edges");
        g->colbits = colbits;
        GI_CUDA(launch_pack_edges(g->d_edges, g->d_pedges, m, colbits, st), "pack edges");
        GI_CUDA(cudaStreamSynchronize(st), "graph build");
      }
    }
  }
  if (bad) {  // ~gi_graph frees the device memory
    return fail(GI_ERR_INVALID_GRAPH, "offsets not a valid CSR (offsets[0]=0, non-decreasing, offsets[n]=m) "
                                      "or a column id outside [0, n)");
  }
  *out = g.release();
  return GI_OK;
}

void gi_graph_destroy(gi_graph* g) {
  if (!g) return;
  {
    DeviceGuard dg(g->device);
    delete g;
  }
}

gi_status gi_graph_info(const gi_graph* g, int64_t* n, int64_t* m, int32_t* device) {
  if (!g) return fail(GI_ERR_INVALID_ARGUMENT, "graph is NULL");
  if (n) *n = g->n;
  if (m) *m = g->m;
  if (device) *device = g->device;
  return GI_OK;
}

gi_status gi_sssp_delta_ex(const gi_graph* g, int32_t src, uint32_t delta, const gi_options* opt,
                           uint32_t* dist_out, gi_stats* stats) {
  return run_queries(g, &src, 1, delta, opt, dist_out, stats, false);
}

gi_status gi_sssp_delta(const gi_graph* g, int32_t src, uint32_t delta, uint32_t* dist_out) {
  return gi_sssp_delta_ex(g, src, delta, nullptr, dist_out, nullptr);
}

gi_status gi_sssp_batch_ex(const gi_graph* g, const int32_t* srcs, int32_t nsrc, uint32_t delta,
                           const gi_options* opt, uint32_t* dist_out, gi_stats* per_src) {
  return run_queries(g, srcs, nsrc, delta, opt, dist_out, per_src, true);
}

gi_status gi_sssp_batch_peers(const gi_graph* g, const int32_t* srcs, int32_t nsrc, uint32_t delta,
                              const gi_options* opt, uint32_t* const* peer_rows, int32_t npeers, int32_t self,
                              gi_stats* per_src) {
  if (npeers < 1 || !peer_rows) return fail(GI_ERR_INVALID_ARGUMENT, "need npeers >= 1 and peer_rows");
  if (self < 0 || self >= npeers) return fail(GI_ERR_INVALID_ARGUMENT, "self not in [0, npeers)");
  for (int32_t i = 0; i < npeers; ++i)
    if (!peer_rows[i]) return fail(GI_ERR_INVALID_ARGUMENT, "peer_rows[%d] is NULL", i);
  return run_queries(g, srcs, nsrc, delta, opt, peer_rows[self], per_src, true, -1, nullptr, peer_rows, npeers);
}

gi_status gi_ipc_get_handle(const void* dptr, void* handle, uint64_t* offset) {
  if (!dptr || !handle || !offset) return fail(GI_ERR_INVALID_ARGUMENT, "NULL argument");
  // the allocation's base (cudaIpcGetMemHandle names whole allocations; a torch tensor may
  // sit inside a larger caching-allocator block): the driver's cuMemGetAddressRange, through
  // the runtime's entry-point query so that the library does not link libcuda
  using GetRange = CUresult (*)(CUdeviceptr*, size_t*, CUdeviceptr);
  static GetRange get_range = nullptr;
  if (!get_range) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      return fail(GI_ERR_CUDA, "cuMemGetAddressRange entry point not found");
    get_range = (GetRange)fn;
  }
  CUdeviceptr base = 0;
  size_t size = 0;
  if (get_range(&base, &size, (CUdeviceptr)dptr) != CUDA_SUCCESS)
    return fail(GI_ERR_INVALID_ARGUMENT, "dptr is not device memory of this process");
  cudaIpcMemHandle_t h;
  GI_CUDA(cudaIpcGetMemHandle(&h, (void*)base), "cudaIpcGetMemHandle");
  memcpy(handle, &h, sizeof(h));
  *offset = (uint64_t)((CUdeviceptr)dptr - base);
  return GI_OK;
}

gi_status gi_ipc_open_handle(const void* handle, uint64_t offset, int32_t device, void** dptr) {
  if (!handle || !dptr) return fail(GI_ERR_INVALID_ARGUMENT, "NULL argument");
  DeviceGuard dg(device);
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  void* base = nullptr;
  GI_CUDA(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
  *dptr = (char*)base + offset;
  return GI_OK;
}

gi_status gi_ipc_close_handle(void* dptr, uint64_t offset, int32_t device) {
  if (!dptr) return fail(GI_ERR_INVALID_ARGUMENT, "NULL argument");
  DeviceGuard dg(device);
  GI_CUDA(cudaIpcCloseMemHandle((char*)dptr - offset), "cudaIpcCloseMemHandle");
  return GI_OK;
}

gi_status gi_sssp_batch(const gi_graph* g, const int32_t* srcs, int32_t nsrc, uint32_t delta,
                        uint32_t* dist_out) {
  return gi_sssp_batch_ex(g, srcs, nsrc, delta, nullptr, dist_out, nullptr);
}

gi_status gi_ppsp_delta_ex(const gi_graph* g, int32_t src, int32_t dst, uint32_t delta, const gi_options* opt,
                           uint32_t* dist_st, gi_stats* stats) {
  if (dst < 0) return fail(GI_ERR_OUT_OF_RANGE, "target %d < 0", dst);
  return run_queries(g, &src, 1, delta, opt, dist_st, stats, false, dst);
}

gi_status gi_ppsp_delta(const gi_graph* g, int32_t src, int32_t dst, uint32_t delta, uint32_t* dist_st) {
  return gi_ppsp_delta_ex(g, src, dst, delta, nullptr, dist_st, nullptr);
}

gi_status gi_astar_delta_ex(const gi_graph* g, int32_t src, int32_t dst, uint32_t delta, const uint32_t* h,
                            const gi_options* opt, uint32_t* dist_st, gi_stats* stats) {
  if (dst < 0) return fail(GI_ERR_OUT_OF_RANGE, "target %d < 0", dst);
  if (!h) return fail(GI_ERR_INVALID_ARGUMENT, "heuristic h is NULL");
  return run_queries(g, &src, 1, delta, opt, dist_st, stats, false, dst, h);
}

gi_status gi_astar_delta(const gi_graph* g, int32_t src, int32_t dst, uint32_t delta, const uint32_t* h,
                         uint32_t* dist_st) {
  return gi_astar_delta_ex(g, src, dst, delta, h, nullptr, dist_st, nullptr);
}

gi_status gi_kcore_ex(const gi_graph* cg_, const gi_options* opt_in, uint32_t* core_out, gi_stats* stats) {
  gi_graph* g = const_cast<gi_graph*>(cg_);
  if (!g) return fail(GI_ERR_INVALID_ARGUMENT, "graph is NULL");
  if (!core_out) return fail(GI_ERR_INVALID_ARGUMENT, "core_out is NULL");
  gi_options opt;
  gi_options_default(&opt);
  if (opt_in) {
    if (opt_in->struct_size != sizeof(gi_options)) return fail(GI_ERR_INVALID_ARGUMENT, "gi_options.struct_size mismatch");
    opt = *opt_in;
  }
  DeviceGuard dg(g->device);
  bool wrongdev = false;
  const bool dev_out = is_device_ptr(core_out, g->device, &wrongdev);
  if (wrongdev) return fail(GI_ERR_INVALID_ARGUMENT, "core_out on another device");
  Workspace* w = ws_acquire(g);
  gi_status s = ws_prepare(g, w, 1, 1);
  if (s) { ws_release(g, w, false); return s; }
  cudaStream_t st = opt.cuda_stream ? (cudaStream_t)opt.cuda_stream : w->stream;
  if (opt.cuda_stream) {
    cudaEvent_t e;
    cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    cudaEventRecord(e, w->stream);
    cudaStreamWaitEvent(st, e, 0);
    cudaEventDestroy(e);
  }
  auto bail = [&](cudaError_t e, const char* what) {
    cudaStreamSynchronize(st);
    ws_release(g, w, false);
    return cuda_fail(e, what);
  };
  cudaError_t e;
  const size_t n = (size_t)g->n;
  if (!w->kc_prio) {
    if ((e = cudaMalloc(&w->kc_prio, n * 4))) return bail(e, "alloc k-core priorities");
    if ((e = cudaMalloc(&w->kc_ctl, sizeof(KcCtl)))) return bail(e, "alloc k-core control");
    if ((e = cudaMalloc(&w->kc_stats, sizeof(KcStats)))) return bail(e, "alloc k-core stats");
  }
  uint32_t* d_core = core_out;
  if (!dev_out) {
    if (w->stagecap < n) {
      if (w->d_stage) cudaFree(w->d_stage);
      w->d_stage = nullptr;
      w->stagecap = 0;
      if ((e = cudaMalloc(&w->d_stage, n * 4))) return bail(e, "alloc core stage");
      w->stagecap = n;
    }
    d_core = w->d_stage;
  }
  KcCtl hc;
  memset(&hc, 0, sizeof(hc));
  hc.pcount[0] = (uint32_t)n;
  for (int k = 0; k < 3; ++k) hc.kmin[k] = 0xFFFFFFFFu;
  if ((e = cudaMemcpyAsync(w->kc_ctl, &hc, sizeof(hc), cudaMemcpyHostToDevice, st))) return bail(e, "init k-core control");
  if ((e = cudaMemsetAsync(w->kc_stats, 0, sizeof(KcStats), st))) return bail(e, "memset k-core stats");
  KcArgs a;
  a.off = g->d_off;
  a.edges = g->d_edges;
  a.n = g->n;
  a.prio = w->kc_prio;
  a.core = d_core;
  a.pile[0] = w->h_groups[0].far[0];
  a.pile[1] = w->h_groups[0].far[1];
  a.q[0] = w->h_groups[0].q[0];
  a.q[1] = w->h_groups[0].q[1];
  a.hub[0] = w->h_groups[0].hub[0];
  a.hub[1] = w->h_groups[0].hub[1];
  a.hubcap = w->hubcap;
  a.ctl = w->kc_ctl;
  a.stats = w->kc_stats;
  a.slots = g->d_slots;
  {
    const char* e_ld = getenv("GI_KC_SLOTS");  // 0: the generic CSR path on every graph
    a.ld = (g->max_deg <= (uint32_t)kSlotEdges && !(e_ld && e_ld[0] == '0')) ? 1u : 0u;
  }
  int grid = g->sm_count * g->bps_kcore;
  if (opt.max_ctas > 0 && opt.max_ctas < grid) grid = opt.max_ctas;
  if ((e = cudaEventRecord(w->ev0, st))) return bail(e, "event");
  if ((e = launch_kcore(a, grid, st))) return bail(e, "launch kcore_persistent");
  if ((e = cudaEventRecord(w->ev1, st))) return bail(e, "event");
  KcStats hs;
  if ((e = cudaMemcpyAsync(&hs, w->kc_stats, sizeof(hs), cudaMemcpyDeviceToHost, st))) return bail(e, "copy stats");
  if (!dev_out && (e = cudaMemcpyAsync(core_out, d_core, n * 4, cudaMemcpyDeviceToHost, st)))
    return bail(e, "copy coreness");
  if ((e = cudaStreamSynchronize(st))) return bail(e, "kcore kernel");
  float ms = 0.f;
  cudaEventElapsedTime(&ms, w->ev0, w->ev1);
  ws_release(g, w, true);
  if (stats) {
    memset(stats, 0, sizeof(*stats));
    stats->buckets = hs.buckets;
    stats->rounds = hs.rounds;
    stats->grid_syncs = hs.phases;
    stats->kernel_launches = 1;
    stats->vertices_processed = hs.vertices;
    stats->edges_relaxed = hs.edges;
    stats->empty_extractions = hs.empty;
    stats->fused_subrounds = hs.subrounds;
    stats->spills = hs.spills;
    stats->critical_subrounds = hs.critical;
    stats->gpu_ms = ms;
    stats->ctas = grid;
    stats->threads_per_cta = 512;
    stats->groups = 1;
    stats->kernel_kind = 3;
  }
  return GI_OK;
}

gi_status gi_kcore(const gi_graph* g, uint32_t* core_out) { return gi_kcore_ex(g, nullptr, core_out, nullptr); }

}  // extern "C"

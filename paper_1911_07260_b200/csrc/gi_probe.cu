// gi_probe.cu — on-box measurement of the latency floors that bound the dependent chains
// of Δ-stepping (SURVEY.md §8(d) "Which roofline bounds the path"): the group barrier the
// fused drain removes (t_sync), one dependent relaxation hop (t_hop: an
// atomicMin whose old value names the next target, with the target's 64-byte ELL slot
// loaded beside it, as in a drain level), and a kernel launch inside a CUDA graph
// (t_launch). bench.py reports the sync floor (grid_syncs x t_sync + launches x t_launch)
// and the chain floor (critical levels x t_hop) from these, measured in the same run.
#include "gi.h"
#include "gi_internal.h"
#include "gi_device.cuh"

#include <cstring>
#include <string>

namespace gi {
namespace {

constexpr int kProbeThreads = 512;

// Every CTA of a cooperative grid runs `iters` group barriers (the SSSP kernels' barrier).
__global__ void __launch_bounds__(kProbeThreads) probe_sync_kernel(uint32_t* bar, int iters) {
  for (int i = 0; i < iters; ++i) dev::group_barrier(bar, gridDim.x);
}

// One thread per CTA follows its own random cycle: v = atomicMin(&next[v], UINT32_MAX)
// (the min never changes the word, the returned old value is the next vertex), with the
// vertex's 64-byte slot loaded in parallel. `sink` keeps the loads alive.
__global__ void probe_hop_kernel(uint32_t* next, const uint4* slots, uint32_t n, int iters, uint32_t* sink) {
  if (threadIdx.x != 0) return;
  uint32_t v = (uint32_t)(((uint64_t)blockIdx.x * 2654435761u) % n);
  uint32_t acc = 0;
  for (int i = 0; i < iters; ++i) {
    const uint32_t nx = atomicMin(next + v, 0xFFFFFFFFu);
    const uint4 s = __ldcg(slots + 4 * (size_t)v);
    acc += s.x ^ s.w;
    v = nx;
  }
  sink[blockIdx.x] = acc + v;
}

__global__ void probe_empty_kernel() {}

// next[] = one random cycle over [0, n) (Sattolo's shuffle of a counter-based hash, on the
// host), so every hop is an independent random L2/HBM access.
void make_cycle(uint32_t* h, uint32_t n) {
  for (uint32_t i = 0; i < n; ++i) h[i] = i;
  uint64_t x = 0x9E3779B97F4A7C15ull;
  for (uint32_t i = n - 1; i > 0; --i) {
    x ^= x >> 30; x *= 0xBF58476D1CE4E5B9ull; x ^= x >> 27; x *= 0x94D049BB133111EBull; x ^= x >> 31;
    const uint32_t j = (uint32_t)(x % i);
    const uint32_t t = h[i]; h[i] = h[j]; h[j] = t;
  }
  // h is a permutation; turn it into a single cycle: perm[k] -> perm[k+1]
  uint32_t* nx = new uint32_t[n];
  for (uint32_t k = 0; k < n; ++k) nx[h[k]] = h[(k + 1) % n];
  memcpy(h, nx, sizeof(uint32_t) * n);
  delete[] nx;
}

}  // namespace
}  // namespace gi

using namespace gi;

extern "C" gi_status gi_probe_floors(int32_t device, int32_t iters, gi_floors* out) {
  if (!out || iters < 1) return GI_ERR_INVALID_ARGUMENT;
  memset(out, 0, sizeof(*out));
  int prev = -1;
  cudaGetDevice(&prev);
  if (cudaSetDevice(device) != cudaSuccess) return GI_ERR_CUDA;
  gi_status rc = GI_OK;
  cudaStream_t st = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  uint32_t *bar = nullptr, *next = nullptr, *sink = nullptr, *hnext = nullptr;
  uint4* slots = nullptr;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  const uint32_t n = 1u << 24;  // 64 MB of `next` + 1 GB of slots: config 2's dist / slot sizes
  int sms = 0, bps = 0;
  float ms = 0.f;
  auto ok = [&](cudaError_t e) {
    if (e != cudaSuccess && rc == GI_OK) rc = e == cudaErrorMemoryAllocation ? GI_ERR_OUT_OF_MEMORY : GI_ERR_CUDA;
    return rc == GI_OK;
  };
  if (!ok(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking)) || !ok(cudaEventCreate(&e0)) ||
      !ok(cudaEventCreate(&e1)))
    goto done;
  if (!ok(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device))) goto done;
  if (!ok(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, probe_sync_kernel, kProbeThreads, 0))) goto done;
  // --- t_sync: one CTA per SM, `iters` group barriers ---
  if (!ok(cudaMalloc(&bar, 128)) || !ok(cudaMemsetAsync(bar, 0, 128, st))) goto done;
  {
    int it = iters;
    void* params[] = {&bar, &it};
    int warm = 16;
    void* wparams[] = {&bar, &warm};
    if (!ok(cudaLaunchCooperativeKernel((const void*)probe_sync_kernel, dim3(sms), dim3(kProbeThreads), wparams, 0, st)))
      goto done;
    ok(cudaEventRecord(e0, st));
    if (!ok(cudaLaunchCooperativeKernel((const void*)probe_sync_kernel, dim3(sms), dim3(kProbeThreads), params, 0, st)))
      goto done;
    ok(cudaEventRecord(e1, st));
    if (!ok(cudaStreamSynchronize(st))) goto done;
    cudaEventElapsedTime(&ms, e0, e1);
    out->t_sync_us = ms * 1e3f / (float)iters;
    out->ctas = sms;
  }
  // --- t_hop: dependent atomicMin chains with the slot load beside them ---
  hnext = new uint32_t[n];
  make_cycle(hnext, n);
  if (!ok(cudaMalloc(&next, sizeof(uint32_t) * n)) || !ok(cudaMalloc(&slots, sizeof(uint4) * 4 * (size_t)n)) ||
      !ok(cudaMalloc(&sink, sizeof(uint32_t) * 4096)))
    goto done;
  if (!ok(cudaMemcpyAsync(next, hnext, sizeof(uint32_t) * n, cudaMemcpyHostToDevice, st)) ||
      !ok(cudaMemsetAsync(slots, 0, sizeof(uint4) * 4 * (size_t)n, st)))
    goto done;
  {
    const int hops = iters * 4;
    probe_hop_kernel<<<sms, 32, 0, st>>>(next, slots, n, 64, sink);  // warm-up
    ok(cudaEventRecord(e0, st));
    probe_hop_kernel<<<sms, 32, 0, st>>>(next, slots, n, hops, sink);
    ok(cudaEventRecord(e1, st));
    if (!ok(cudaGetLastError()) || !ok(cudaStreamSynchronize(st))) goto done;
    cudaEventElapsedTime(&ms, e0, e1);
    out->t_hop_us = ms * 1e3f / (float)hops;
  }
  // --- t_launch: empty kernels replayed from a CUDA graph ---
  {
    const int k = 64;
    if (!ok(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal))) goto done;
    for (int i = 0; i < k; ++i) probe_empty_kernel<<<1, 32, 0, st>>>();
    if (!ok(cudaStreamEndCapture(st, &graph)) || !ok(cudaGraphInstantiate(&exec, graph, 0))) goto done;
    if (!ok(cudaGraphLaunch(exec, st)) || !ok(cudaStreamSynchronize(st))) goto done;
    const int reps = 8;
    ok(cudaEventRecord(e0, st));
    for (int r = 0; r < reps; ++r) ok(cudaGraphLaunch(exec, st));
    ok(cudaEventRecord(e1, st));
    if (!ok(cudaStreamSynchronize(st))) goto done;
    cudaEventElapsedTime(&ms, e0, e1);
    out->t_launch_us = ms * 1e3f / (float)(k * reps);
  }
  {
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, device);
    out->sm_clock_mhz = (float)clk / 1e3f;
  }
done:
  if (exec) cudaGraphExecDestroy(exec);
  if (graph) cudaGraphDestroy(graph);
  if (bar) cudaFree(bar);
  if (next) cudaFree(next);
  if (slots) cudaFree(slots);
  if (sink) cudaFree(sink);
  delete[] hnext;
  if (e0) cudaEventDestroy(e0);
  if (e1) cudaEventDestroy(e1);
  if (st) cudaStreamDestroy(st);
  if (prev >= 0) cudaSetDevice(prev);
  (void)bps;
  return rc;
}

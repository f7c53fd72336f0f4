// placement_bench.cu — is device memory interleaved across the two dies at a coarse
// granularity? Random 4-byte reads (or atomics) confined to a window of W bytes at offset
// `off` of one big allocation, from every SM; the rate per window shows whether some windows
// live on one die only.
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hsh(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

template <int ATOM>
__global__ void rnd(uint32_t* base, uint64_t words, int iters, uint32_t* sink) {
  uint32_t acc = 0, x = hsh(blockIdx.x * blockDim.x + threadIdx.x + 1);
  for (int i = 0; i < iters; ++i) {
    uint32_t idx[8], v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) { x = hsh(x + u); idx[u] = (uint32_t)(((uint64_t)x * words) >> 32); }
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = ATOM ? atomicMin(base + idx[u], 0xFFFFFFFFu) : __ldcg(base + idx[u]);
#pragma unroll
    for (int u = 0; u < 8; ++u) acc += v[u];
  }
  if (acc == 0x1234567u) sink[0] = acc;
}

extern "C" int place_rnd(int atom, uint32_t* base, uint64_t words, int iters, uint32_t* sink, cudaStream_t st) {
  if (atom) rnd<1><<<148 * 2, 1024, 0, st>>>(base, words, iters, sink);
  else rnd<0><<<148 * 2, 1024, 0, st>>>(base, words, iters, sink);
  return (int)cudaGetLastError();
}

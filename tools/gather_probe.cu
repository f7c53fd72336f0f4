// gather_probe.cu — ceiling of the relaxation's memory pattern on config 4: stream the CSR
// column ids and read dist[col] (random 4-byte reads), nothing else. Variants: coherent
// L2 reads (ld.global.cg, what the kernels use), L1-allocating reads, edge stream only,
// and reads with an L2 evict-last policy.
#include <cstdint>
#include <cuda_runtime.h>

template <int MODE>
__global__ void __launch_bounds__(1024) gather(const uint32_t* __restrict__ cols, int64_t m, const uint32_t* dist, uint32_t* sink) {
  uint32_t acc = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  constexpr int U = 8;
  for (; i + (U - 1) * stride < m; i += U * stride) {
    uint32_t c[U], d[U];
#pragma unroll
    for (int u = 0; u < U; ++u) c[u] = __ldcs(cols + i + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (MODE == 0) d[u] = __ldcg(dist + c[u]);
      else if (MODE == 1) d[u] = __ldca(dist + c[u]);
      else if (MODE == 2) d[u] = c[u];
      else {
        uint64_t pol;
        asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
        asm volatile("ld.global.cg.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(d[u]) : "l"(dist + c[u]), "l"(pol));
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc += d[u];
  }
  for (; i < m; i += stride) acc += MODE == 2 ? cols[i] : __ldcg(dist + cols[i]);
  if (acc == 0x12345678u) sink[0] = acc;
}

extern "C" int probe_gather(int mode, const uint32_t* cols, int64_t m, const uint32_t* dist, uint32_t* sink,
                            int blocks, int threads, cudaStream_t st) {
  switch (mode) {
    case 0: gather<0><<<blocks, threads, 0, st>>>(cols, m, dist, sink); break;
    case 1: gather<1><<<blocks, threads, 0, st>>>(cols, m, dist, sink); break;
    case 2: gather<2><<<blocks, threads, 0, st>>>(cols, m, dist, sink); break;
    default: gather<3><<<blocks, threads, 0, st>>>(cols, m, dist, sink); break;
  }
  return (int)cudaGetLastError();
}

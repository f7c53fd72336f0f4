// window_probe.cu — does an L2-sized target window speed up the relaxation's gather?
// Streams m random column ids (restricted to a window of `win` vertices) and reads
// dist[col] (MODE 0), or red.min's into it (MODE 1), or pre-reads then red.min's when
// the candidate improves (MODE 2, what expand_kernel does).
#include <cstdint>
#include <cuda_runtime.h>

template <int MODE, int U>
__global__ void __launch_bounds__(1024) wgather(const uint32_t* __restrict__ cols, int64_t m, uint32_t* dist,
                                                uint32_t* sink) {
  uint32_t acc = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < m; i += U * stride) {
    uint32_t c[U], d[U];
#pragma unroll
    for (int u = 0; u < U; ++u) c[u] = __ldcs(cols + i + u * stride);
    if (MODE == 0 || MODE == 2) {
#pragma unroll
      for (int u = 0; u < U; ++u) d[u] = __ldcg(dist + c[u]);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (MODE == 0) acc += d[u];
      else {
        const uint32_t nd = (c[u] * 2654435761u) >> 8;
        if (MODE == 1 || nd < d[u]) asm volatile("red.global.min.u32 [%0], %1;" ::"l"(dist + c[u]), "r"(nd) : "memory");
      }
    }
  }
  if (acc == 0x12345678u) sink[0] = acc;
}

extern "C" int probe_window(int mode, const uint32_t* cols, int64_t m, uint32_t* dist, uint32_t* sink, int blocks,
                            int threads, cudaStream_t st) {
  switch (mode) {
    case 0: wgather<0, 8><<<blocks, threads, 0, st>>>(cols, m, dist, sink); break;
    case 1: wgather<1, 8><<<blocks, threads, 0, st>>>(cols, m, dist, sink); break;
    default: wgather<2, 8><<<blocks, threads, 0, st>>>(cols, m, dist, sink); break;
  }
  return (int)cudaGetLastError();
}

// Cost of one hop of the Δ-stepping dependent chain, in isolation (one warp, path-like
// access pattern): atomicMin on dist[i+1] and the 64 B slot of i+1, then the next hop
// depends on both. Variants isolate each ingredient. Build:
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/hop_bench.cu -o /tmp/hop
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t ld_cg(const uint32_t* p) { return __ldcg(p); }
__device__ __forceinline__ void prefetch_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }

// mode bits: 1 = atomic, 2 = slot load, 4 = prefetch next slots, 8 = probe ld.cg, 16 = smem handoff via STS/LDS
__global__ void hop(uint32_t* dist, const uint4* slots, int steps, int mode, int stride, long long* out,
                    uint32_t* sink) {
  __shared__ uint4 buf[8];
  if (threadIdx.x != 0) return;
  uint32_t i = 0, acc = 0;
  long long t0 = clock64();
  for (int s = 0; s < steps; ++s) {
    const uint32_t nx = i + stride;
    uint32_t old = 0;
    uint4 sl[4] = {};
    if (mode & 1) old = atomicMin(dist + nx, (uint32_t)s);
    if (mode & 2)
      for (int j = 0; j < 4; ++j) sl[j] = __ldg(slots + 4 * (size_t)nx + j);
    uint32_t cu = 0;
    if (mode & 8) cu = ld_cg(dist + i);
    if (mode & 4) {
      prefetch_l2(slots + 4 * (size_t)(nx + stride));
      prefetch_l2(slots + 4 * (size_t)(nx));
    }
    uint32_t dep = old + sl[0].x + sl[1].y + sl[2].z + sl[3].w + cu;
    if (mode & 16) {
      for (int j = 0; j < 4; ++j) buf[j] = sl[j];
      __syncwarp(1u);
      dep += buf[(dep & 3)].x;
    }
    acc += dep;
    i = nx + (dep == 0x9E3779B9u ? 1u : 0u);  // keeps the dependency (practically never 1)
  }
  long long t1 = clock64();
  out[0] = (t1 - t0) / steps;
  *sink = acc;
}

int main() {
  const size_t N = 1u << 24;
  uint32_t* dist;
  uint4* slots;
  cudaMalloc(&dist, N * 4);
  cudaMalloc(&slots, N * 64);
  cudaMemset(slots, 0, N * 64);
  long long* out;
  cudaMallocManaged(&out, 64);
  uint32_t* sink;
  cudaMalloc(&sink, 4);
  const char* names[] = {"atomic only", "slot only (cold)", "slot + prefetch", "atomic + slot", "atomic + slot + prefetch",
                         "atomic+slot+pf+probe", "atomic+slot+pf+probe+smem", "probe only"};
  const int modes[] = {1, 2, 6, 3, 7, 15, 31, 8};
  for (int stride : {1, 64}) {
    for (int k = 0; k < 8; ++k) {
      cudaMemset(dist, 0xFF, N * 4);  // dist in L2/HBM like the real init
      hop<<<1, 1>>>(dist, slots, 20000, modes[k], stride, out, sink);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("error %s\n", cudaGetErrorString(e)); return 1; }
      printf("stride %2d  %-28s %lld cycles/hop\n", stride, names[k], out[0]);
    }
  }
  return 0;
}

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

int main_hop() {
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

// Minimal BSP sub-round on a path (one CTA of 512 threads): octet 0 reads the bin entry
// (smem), loads the vertex's 64 B slot (8 B per lane), atomicMins the successor, pushes
// it into the other bin, and every thread meets at __syncthreads. Cycles per sub-round.
__global__ void bsp_chain(uint32_t* dist, const uint2* slots, int steps, long long* out) {
  __shared__ uint2 bin[2][64];
  __shared__ uint32_t cnt[2];
  if (threadIdx.x == 0) { bin[0][0] = make_uint2(0, 0); cnt[0] = 1; cnt[1] = 0; }
  __syncthreads();
  long long t0 = clock64();
  for (int s = 0; s < steps; ++s) {
    const int cur = s & 1;
    const uint32_t n = cnt[cur];
    if (threadIdx.x < 8 * n) {
      const uint2 it = bin[cur][threadIdx.x >> 3];
      const uint2 e = __ldg(slots + 8 * (size_t)it.x + (threadIdx.x & 7));
      if (e.x != 0xFFFFFFFFu) {
        const uint32_t nd = it.y + e.y;
        const uint32_t old = atomicMin(dist + e.x, nd);
        if (nd < old) {
          const uint32_t p = atomicAdd(&cnt[cur ^ 1], 1u);
          bin[cur ^ 1][p & 63] = make_uint2(e.x, nd);
        }
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) cnt[cur] = 0;
    __syncthreads();
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = (t1 - t0) / steps;
}

int main_bsp() {
  const int n = 100000;
  uint32_t* dist;
  uint2* slots;
  cudaMalloc(&dist, n * 4);
  cudaMalloc(&slots, (size_t)n * 64);
  uint2* h = new uint2[(size_t)n * 8];
  for (int v = 0; v < n; ++v)
    for (int k = 0; k < 8; ++k) h[(size_t)v * 8 + k] = make_uint2(0xFFFFFFFFu, 0);
  for (int v = 0; v < n; ++v) {
    if (v + 1 < n) h[(size_t)v * 8 + 0] = make_uint2(v + 1, 1);
    if (v > 0) h[(size_t)v * 8 + 1] = make_uint2(v - 1, 1);
  }
  cudaMemcpy(slots, h, (size_t)n * 64, cudaMemcpyHostToDevice);
  long long* out;
  cudaMallocManaged(&out, 64);
  for (int rep = 0; rep < 2; ++rep) {
    cudaMemset(dist, 0xFF, n * 4);
    bsp_chain<<<1, 512>>>(dist, slots, 20000, out);
    cudaDeviceSynchronize();
  }
  printf("minimal BSP sub-round (path, 1 CTA x 512): %lld cycles\n", out[0]);
  return 0;
}

int main() {
  main_hop();
  return main_bsp();
}

// Latency microbenchmarks for the primitives on the Δ-stepping critical chain (one thread,
// pointer chasing / dependent ops; clock64 deltas). Build: nvcc -O3 -gencode
// arch=compute_100a,code=sm_100a tools/latency.cu -o /tmp/lat
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t ld_cg(const uint32_t* p) { return __ldcg(p); }
__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* p) {
  uint32_t v; asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v;
}
__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v; asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory"); return v;
}

// chase: p[i] holds the next index. mode selects the access flavour.
__global__ void chase(uint32_t* p, int steps, int mode, long long* out, uint32_t* sink) {
  uint32_t i = 0;
  long long t0 = clock64();
  for (int s = 0; s < steps; ++s) {
    switch (mode) {
      case 0: i = ld_cg(p + i); break;                       // L2 (ld.cg)
      case 1: i = __ldg(p + i); break;                       // nc path
      case 2: i = atomicMin(p + i, 0xFFFFFFFFu); break;      // ATOMG (value unchanged)
      case 3: i = ld_relaxed(p + i); break;
      case 4: i = ld_acquire(p + i); break;
      case 5: { i = ld_cg(p + i); __threadfence(); } break;
      case 6: { i = ld_cg(p + i); asm volatile("fence.acq_rel.gpu;" ::: "memory"); } break;
      case 7: { i = ld_cg(p + i); __syncthreads(); } break;
    }
  }
  long long t1 = clock64();
  out[0] = (t1 - t0) / steps;
  *sink = i;
}

// prefetch test: prefetch the next target, wait ~W cycles, then load it.
__global__ void pf(uint32_t* p, int steps, int wait, int do_pf, long long* out, uint32_t* sink) {
  uint32_t i = 0;
  long long acc = 0;
  for (int s = 0; s < steps; ++s) {
    uint32_t nxt = (i * 2654435761u + 12345u) % (1u << 26);  // pseudo-random index (cold)
    if (do_pf) asm volatile("prefetch.global.L2 [%0];" ::"l"(p + nxt));
    long long tw = clock64();
    while (clock64() - tw < wait) {}
    long long t0 = clock64();
    uint32_t v = ld_cg(p + nxt);
    i += v + 1;  // dependency
    acc += clock64() - t0;
  }
  out[0] = acc / steps;
  *sink = i;
}

int main() {
  const size_t N = 1u << 26;  // 256 MB (> L2)
  uint32_t* p; cudaMalloc(&p, N * 4);
  long long* out; cudaMallocManaged(&out, 64);
  uint32_t* sink; cudaMalloc(&sink, 4);
  // small ring (L2-resident): stride 32 elements over 1 MB
  uint32_t* h = new uint32_t[N];
  for (size_t k = 0; k < N; ++k) h[k] = 0;
  const uint32_t ring = 1u << 18;  // 1 MB
  for (uint32_t k = 0; k < ring; k += 32) h[k] = (k + 32 * 97) % ring;
  cudaMemcpy(p, h, N * 4, cudaMemcpyHostToDevice);
  const char* names[] = {"ld.cg L2-hit", "ldg.nc L2-hit(L1 miss?)", "atomicMin L2-hit", "ld.relaxed.gpu",
                         "ld.acquire.gpu", "ld.cg+__threadfence", "ld.cg+fence.acq_rel", "ld.cg+syncthreads"};
  for (int mode = 0; mode < 8; ++mode) {
    chase<<<1, 1>>>(p, 100, mode, out, sink);  // warm
    chase<<<1, 1>>>(p, 2000, mode, out, sink);
    cudaDeviceSynchronize();
    printf("%-28s %lld cycles/step\n", names[mode], out[0]);
  }
  // DRAM: big random ring
  for (size_t k = 0; k < N; ++k) h[k] = 0;
  uint32_t cur = 0;
  for (int s = 0; s < 5000; ++s) { uint32_t nx = (uint32_t)(((uint64_t)(s + 1) * 2654435761ull) % N) & ~31u; h[cur] = nx; cur = nx; }
  cudaMemcpy(p, h, N * 4, cudaMemcpyHostToDevice);
  // flush L2 by touching a big buffer
  uint32_t* big; cudaMalloc(&big, 512u << 20); cudaMemset(big, 1, 512u << 20);
  chase<<<1, 1>>>(p, 4000, 0, out, sink); cudaDeviceSynchronize();
  printf("%-28s %lld cycles/step\n", "ld.cg DRAM (cold chase)", out[0]);
  cudaMemset(big, 2, 512u << 20);
  chase<<<1, 1>>>(p, 4000, 2, out, sink); cudaDeviceSynchronize();
  printf("%-28s %lld cycles/step\n", "atomicMin DRAM (cold chase)", out[0]);
  for (int w : {0, 500, 1000, 2000, 4000}) {
    for (int d = 0; d < 2; ++d) {
      cudaMemset(big, 3, 512u << 20);
      pf<<<1, 1>>>(p, 2000, w, d, out, sink); cudaDeviceSynchronize();
      printf("prefetch=%d wait=%5d -> load %lld cycles\n", d, w, out[0]);
    }
  }
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("clock rate attr %d kHz\n", clk);
  return 0;
}

// gi_device.cuh — small device helpers shared by the persistent kernels (SSSP family in
// gi_kernels.cu, k-core in gi_kcore.cu): coherent loads, fences, the group barrier.
#pragma once
#include <cstdint>

namespace gi {
namespace dev {

__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void fence_acq_rel() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

// Barrier over the G co-resident CTAs of one group (cooperative launch). One word:
// arrivals in the low 16 bits, generation in the high 16; the last arriver resets the
// count and bumps the generation with a single atomic.
__device__ __forceinline__ void group_barrier(uint32_t* bar, uint32_t G) {
  __syncthreads();
  if (threadIdx.x == 0) {
    fence_acq_rel();  // publish this CTA's writes (cumulative over the bar.sync above)
    const uint32_t old = atomicAdd(bar, 1u);
    if ((old & 0xFFFFu) == G - 1) {
      atomicAdd(bar, 0x10000u - G);
    } else {
      const uint32_t gen = old >> 16;
      while ((ld_relaxed(bar) >> 16) == gen) {
      }
    }
    fence_acq_rel();
  }
  __syncthreads();
}

}  // namespace dev
}  // namespace gi

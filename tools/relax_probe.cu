// relax_probe.cu — which ingredient of the expand relaxation costs what, on config 4's
// packed edges: R0 pre-read gather + compare; R1 + red.min of improving candidates;
// R2 + a per-lane shared-memory push of improving targets; R3 + the far-pile flush
// (atomicOr dedup bitmap + warp-aggregated append to ONE global counter); R4 as R3 with
// one append counter per CTA.
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hsh(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

template <int MODE>
__global__ void __launch_bounds__(1024) relax(const uint32_t* __restrict__ pe, int64_t m, uint32_t* dist,
                                              uint32_t* bits, int32_t* list, uint32_t* counts, uint32_t colbits) {
  __shared__ int32_t seg[32][256];
  __shared__ uint32_t fill[32];
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) fill[warp] = 0;
  __syncwarp();
  const uint32_t cmask = (1u << colbits) - 1u;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  uint32_t* cnt = MODE == 4 ? counts + blockIdx.x * 32 : counts;
  constexpr int U = 4;
  const int64_t nfull = m / (U * stride) * (U * stride);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nfull; i += U * stride) {
    uint32_t x[U], old[U];
#pragma unroll
    for (int u = 0; u < U; ++u) x[u] = __ldcs(pe + i + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) old[u] = __ldcg(dist + (x[u] & cmask));
    const uint32_t du = hsh((uint32_t)((i + 0) >> 10)) & 31;
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t v = x[u] & cmask, nd = du + (x[u] >> colbits);
      if (nd < old[u]) {
        if (MODE >= 1) asm volatile("red.relaxed.gpu.global.min.u32 [%0], %1;" ::"l"(dist + v), "r"(nd) : "memory");
        if (MODE >= 2) {
          const uint32_t pos = atomicAdd(&fill[warp], 1u);
          if (pos < 256) seg[warp][pos] = (int32_t)v;
        }
        if (MODE == 0) old[0] ^= nd;  // keep the compare alive
      }
    }
    if (MODE >= 3) {
      __syncwarp();
      const uint32_t n = min(fill[warp], 256u);
      if (n > 128) {
        for (uint32_t b = 0; b < n; b += 128) {
          int32_t v[4]; uint32_t o[4], newm = 0;
#pragma unroll
          for (int k = 0; k < 4; ++k) { const uint32_t j = b + k * 32 + lane; v[k] = j < n ? seg[warp][j] : -1; }
#pragma unroll
          for (int k = 0; k < 4; ++k) o[k] = v[k] >= 0 ? atomicOr(bits + (v[k] >> 5), 1u << (v[k] & 31)) : ~0u;
#pragma unroll
          for (int k = 0; k < 4; ++k) if (v[k] >= 0 && !(o[k] & (1u << (v[k] & 31)))) newm |= 1u << k;
          const uint32_t nk = __popc(newm);
          uint32_t incl = nk;
#pragma unroll
          for (int o2 = 1; o2 < 32; o2 <<= 1) { const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o2); if (lane >= (uint32_t)o2) incl += t; }
          const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
          uint32_t base = 0;
          if (lane == 0 && tot) base = atomicAdd(cnt, tot);
          base = __shfl_sync(0xffffffffu, base, 0) & ((1u << 26) - 1);
          uint32_t off = base + incl - nk;
#pragma unroll
          for (int k = 0; k < 4; ++k) if (newm & (1u << k)) list[off++] = v[k];
        }
        __syncwarp();
        if (lane == 0) fill[warp] = 0;
        __syncwarp();
      }
    } else if (MODE == 2) {
      __syncwarp();
      if (lane == 0 && fill[warp] > 128) fill[warp] = 0;
      __syncwarp();
    }
    if (MODE == 0 && old[0] == 0x9999999u) dist[0] = 1;
  }
}

// MODE 5: the expand mapping (one list X of {beg, deg, du} with exclusive prefix xpre,
// warp ranges, 32-entry windows, ballot/redux/popc row mapping), then R4's relaxation.
struct XE { long long beg; unsigned deg, du; };
template <int K>
__global__ void __launch_bounds__(1024) relax_x(const uint32_t* __restrict__ pe, const XE* X,
                                                const unsigned long long* xpre, uint32_t hn, unsigned long long E,
                                                uint32_t* dist, uint32_t* bits, int32_t* list, uint32_t* counts,
                                                uint32_t colbits) {
  __shared__ int32_t seg[32][256];
  __shared__ uint32_t fill[32];
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (lane == 0) fill[warp] = 0;
  __syncwarp();
  const uint32_t cmask = (1u << colbits) - 1u;
  uint32_t* cnt = counts + blockIdx.x * 32;
  const unsigned long long W = (unsigned long long)gridDim.x * nw, wg = (unsigned long long)blockIdx.x * nw + warp;
  const unsigned long long a = E * wg / W, b = E * (wg + 1) / W;
  if (a >= b) return;
  const uint32_t len = (uint32_t)(b - a);
  uint32_t ilo = 0, ihi = hn;
  while (ihi - ilo > 32) {
    const uint32_t step = (ihi - ilo + 31) / 32;
    const uint32_t idx = ilo + lane * step;
    const bool pr = idx < ihi && __ldcg(xpre + idx) <= a;
    const uint32_t c = __popc(__ballot_sync(0xffffffffu, pr));
    ilo += (c - 1) * step;
    ihi = min(ilo + step, ihi);
  }
  { const uint32_t idx = ilo + lane; const bool pr = idx < ihi && __ldcg(xpre + idx) <= a;
    ilo += __popc(__ballot_sync(0xffffffffu, pr)) - 1; }
  uint32_t jb = ilo;
  uint32_t endr; long long off; uint32_t wdu;
  auto window = [&]() {
    const uint32_t idx = jb + lane;
    endr = len; off = 0; wdu = 0;
    if (idx < hn) {
      const XE e = X[idx];
      const unsigned long long start = __ldcg(xpre + idx), end = start + e.deg;
      endr = end <= a ? 0u : (uint32_t)min(end - a, (unsigned long long)len);
      off = e.beg - (long long)start; wdu = e.du;
    }
  };
  window();
  const uint32_t lanemask = (2u << lane) - 2u;
  for (uint32_t it0 = 0; it0 < len; it0 += 32 * K) {
    long long ei[K]; uint32_t du[K], valid = 0, x[K], old[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
      ei[k] = 0; du[k] = 0;
      const uint32_t r0 = it0 + 32 * k;
      if (r0 >= len) continue;
      const uint32_t last = __shfl_sync(0xffffffffu, endr, 31);
      if (last < min(r0 + 32, len)) { jb += __popc(__ballot_sync(0xffffffffu, endr <= r0)); window(); }
      const uint32_t c0 = __popc(__ballot_sync(0xffffffffu, endr <= r0));
      const uint32_t xx = endr - r0;
      const uint32_t heads = __reduce_or_sync(0xffffffffu, (xx - 1u < 31u) ? (1u << xx) : 0u);
      const uint32_t slot = c0 + __popc(heads & lanemask);
      const long long o = __shfl_sync(0xffffffffu, off, slot);
      const uint32_t d = __shfl_sync(0xffffffffu, wdu, slot);
      if (r0 + lane < len) { ei[k] = o + (long long)(a + r0 + lane); du[k] = d; valid |= 1u << k; }
    }
#pragma unroll
    for (int k = 0; k < K; ++k) x[k] = (valid >> k) & 1u ? __ldcs(pe + ei[k]) : 0u;
#pragma unroll
    for (int k = 0; k < K; ++k) old[k] = (valid >> k) & 1u ? __ldcg(dist + (x[k] & cmask)) : 0u;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      if (!((valid >> k) & 1u)) continue;
      const uint32_t v = x[k] & cmask, nd = du[k] + (x[k] >> colbits);
      if (nd < old[k]) {
        asm volatile("red.relaxed.gpu.global.min.u32 [%0], %1;" ::"l"(dist + v), "r"(nd) : "memory");
        const uint32_t pos = atomicAdd(&fill[warp], 1u);
        if (pos < 256) seg[warp][pos] = (int32_t)v;
      }
    }
    __syncwarp();
    const uint32_t n = min(fill[warp], 256u);
    if (n > 128) {
      for (uint32_t b0 = 0; b0 < n; b0 += 128) {
        int32_t v[4]; uint32_t o[4], newm = 0;
#pragma unroll
        for (int k = 0; k < 4; ++k) { const uint32_t j = b0 + k * 32 + lane; v[k] = j < n ? seg[warp][j] : -1; }
#pragma unroll
        for (int k = 0; k < 4; ++k) o[k] = v[k] >= 0 ? atomicOr(bits + (v[k] >> 5), 1u << (v[k] & 31)) : ~0u;
#pragma unroll
        for (int k = 0; k < 4; ++k) if (v[k] >= 0 && !(o[k] & (1u << (v[k] & 31)))) newm |= 1u << k;
        const uint32_t nk = __popc(newm);
        uint32_t incl = nk;
#pragma unroll
        for (int o2 = 1; o2 < 32; o2 <<= 1) { const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o2); if (lane >= (uint32_t)o2) incl += t; }
        const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
        uint32_t base = 0;
        if (lane == 0 && tot) base = atomicAdd(cnt, tot);
        base = __shfl_sync(0xffffffffu, base, 0) & ((1u << 26) - 1);
        uint32_t of = base + incl - nk;
#pragma unroll
        for (int k = 0; k < 4; ++k) if (newm & (1u << k)) list[of++] = v[k];
      }
      __syncwarp();
      if (lane == 0) fill[warp] = 0;
      __syncwarp();
    }
  }
}

extern "C" int probe_relax_x(int k, const uint32_t* pe, const void* X, const unsigned long long* xpre, uint32_t hn,
                             unsigned long long E, uint32_t* dist, uint32_t* bits, int32_t* list, uint32_t* counts,
                             uint32_t colbits, int blocks, int threads, cudaStream_t st) {
  if (k == 4) relax_x<4><<<blocks, threads, 0, st>>>(pe, (const XE*)X, xpre, hn, E, dist, bits, list, counts, colbits);
  else relax_x<8><<<blocks, threads, 0, st>>>(pe, (const XE*)X, xpre, hn, E, dist, bits, list, counts, colbits);
  return (int)cudaGetLastError();
}

extern "C" int probe_relax(int mode, const uint32_t* pe, int64_t m, uint32_t* dist, uint32_t* bits, int32_t* list,
                           uint32_t* counts, uint32_t colbits, int blocks, int threads, cudaStream_t st) {
  switch (mode) {
    case 0: relax<0><<<blocks, threads, 0, st>>>(pe, m, dist, bits, list, counts, colbits); break;
    case 1: relax<1><<<blocks, threads, 0, st>>>(pe, m, dist, bits, list, counts, colbits); break;
    case 2: relax<2><<<blocks, threads, 0, st>>>(pe, m, dist, bits, list, counts, colbits); break;
    case 3: relax<3><<<blocks, threads, 0, st>>>(pe, m, dist, bits, list, counts, colbits); break;
    default: relax<4><<<blocks, threads, 0, st>>>(pe, m, dist, bits, list, counts, colbits); break;
  }
  return (int)cudaGetLastError();
}

// ds_expand.cuh — the ordered projection ("geometric read"), eq:projection:
// for k = 0..U-1 emit key_base + k exactly H[k] times.  Output-tile-centric: CTA t owns
// output positions [t*T, (t+1)*T), looks up its first bin in tfb (written by k_reduce_scan),
// stages the prefix window P[k_lo .. k_hi+1] in shared memory and writes every position
// exactly once with 128-bit streaming stores.  Balanced by construction, whatever the skew
// (a Zipf hot key spanning 240 tiles is written by 240 CTAs).
#pragma once
#include "ds_common.cuh"

namespace ds {

constexpr int kExpandThreads = 256;
constexpr uint32_t kExpandTile = 8192;    // positions per CTA (multiple of 4)
constexpr uint32_t kExpandWindow = 2048;  // bins staged per smem chunk

// Largest i in [0, m) with sP[i] <= q, given sP[0] <= q < sP[m].
__device__ __forceinline__ uint32_t window_search(const uint32_t* sP, uint32_t m, uint32_t q) {
  uint32_t lo = 0, len = m;
  while (len > 1) {
    uint32_t half = len >> 1;
    if (sP[lo + half] <= q) lo += half;
    len -= half;
  }
  return lo;
}

__global__ void __launch_bounds__(kExpandThreads) k_expand(const uint32_t* __restrict__ P, uint32_t U,
                                                           const uint32_t* __restrict__ tfb,
                                                           uint64_t ntiles, const uint64_t* ws_total,
                                                           uint64_t cap, int32_t key_base,
                                                           int32_t* __restrict__ out) {
  __shared__ uint32_t sP[kExpandWindow + 1];
  pdl_wait();
  const uint64_t total = *ws_total;
  const uint64_t nw = total < cap ? total : cap;  // positions to write
  const uint64_t t = blockIdx.x;
  const uint64_t p0 = t * kExpandTile;
  if (p0 >= nw) return;
  const uint64_t p1 = (p0 + kExpandTile < nw) ? p0 + kExpandTile : nw;
  const uint32_t k_lo = tfb[t];
  const uint32_t k_hi = (t + 1 < ntiles && (t + 1) * kExpandTile < nw) ? tfb[t + 1] : U - 1;

  // Output alignment: positions [p0, p0 + head) scalar, then 16-byte aligned quads.
  const uint32_t mis = (uint32_t)((reinterpret_cast<uintptr_t>(out) >> 2) & 3u);
  const uint32_t head = mis ? 4 - mis : 0;  // same for every tile (T % 4 == 0)

  for (uint64_t c0 = k_lo; c0 <= k_hi; c0 += kExpandWindow) {
    const uint32_t m = (uint32_t)((k_hi + 1 - c0) < kExpandWindow ? (k_hi + 1 - c0) : kExpandWindow);
    __syncthreads();
    for (uint32_t i = threadIdx.x; i <= m; i += blockDim.x) sP[i] = __ldcg(P + c0 + i);
    __syncthreads();
    // Positions this chunk covers within the tile.
    const uint64_t lo = sP[0] > p0 ? sP[0] : p0;
    const uint64_t hi = sP[m] < p1 ? sP[m] : p1;
    if (lo >= hi) continue;
    const int32_t kb = key_base + (int32_t)c0;
    // Scalar edges: [lo, a0) and [a1, hi) where a0/a1 are quad-aligned output positions.
    uint64_t a0 = lo + ((head + 4 - (uint32_t)(lo & 3)) & 3);  // first q >= lo, q ≡ head (mod 4)
    if (a0 > hi) a0 = hi;
    uint64_t a1 = a0 + ((hi - a0) & ~3ull);
    for (uint64_t q = lo + threadIdx.x; q < a0; q += blockDim.x)
      out[q] = kb + (int32_t)window_search(sP, m, (uint32_t)q);
    for (uint64_t q = a1 + threadIdx.x; q < hi; q += blockDim.x)
      out[q] = kb + (int32_t)window_search(sP, m, (uint32_t)q);
    // Aligned quads.
    for (uint64_t q = a0 + 4 * (uint64_t)threadIdx.x; q < a1; q += 4 * (uint64_t)blockDim.x) {
      uint32_t i = window_search(sP, m, (uint32_t)q);
      int4 v;
      v.x = kb + (int32_t)i;
      while (sP[i + 1] <= q + 1) ++i;
      v.y = kb + (int32_t)i;
      while (sP[i + 1] <= q + 2) ++i;
      v.z = kb + (int32_t)i;
      while (sP[i + 1] <= q + 3) ++i;
      v.w = kb + (int32_t)i;
      st_stream4(reinterpret_cast<int4*>(out + q), v);
    }
  }
  pdl_trigger();
}

}  // namespace ds

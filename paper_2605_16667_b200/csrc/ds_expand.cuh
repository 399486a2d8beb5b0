// ds_expand.cuh — the ordered projection ("geometric read"), eq:projection:
// for k = 0..U-1 emit key_base + k exactly H[k] times.
//
// Output-tile-centric and persistent: CTA c processes output tiles t = c, c + G, ... of
// kExpandTile positions.  For tile [p0, p1) the first bin k_lo comes from tfb[t] (written by
// k_reduce_scan); every later bin k whose start P[k] falls inside the tile adds one "bin
// start" mark at P[k] - p0 in a shared-memory count array; an inclusive scan of the marks
// then gives, for every position p, key(p) = key_base + k_lo + #{starts <= p}.  Marks are
// counts, not flags, so empty bins (equal starts) need no special case, and the cost is
// O(T + #bins) per tile with no per-position search and no divergence.  The finished tile
// leaves shared memory through 128-bit streaming stores, each warp instruction writing 512
// contiguous bytes.  Balanced by construction whatever the skew: a Zipf hot key spanning
// many tiles is written by many CTAs.
#pragma once
#include "ds_common.cuh"

namespace ds {

constexpr int kExpandThreads = 512;
constexpr uint32_t kExpandTile = 8192;                                // positions per tile
constexpr uint32_t kExpandQuads = kExpandTile / 4;                    // 2048 int4
constexpr uint32_t kExpandPerThread = kExpandQuads / kExpandThreads;  // 4 quads (16 positions)

// XOR swizzle of quad index q so that both access patterns are bank-conflict free:
// thread-contiguous (thread t owns quads 4t..4t+3) and warp-contiguous (quad j by lane j).
__device__ __forceinline__ uint32_t swz(uint32_t q) { return q ^ ((q >> 3) & 7u); }

__global__ void __launch_bounds__(kExpandThreads, 4) k_expand(const uint32_t* __restrict__ P, uint32_t U,
                                                           const uint32_t* __restrict__ tfb,
                                                           uint64_t ntiles, const uint64_t* ws_total,
                                                           uint64_t cap, int32_t key_base,
                                                           int32_t* __restrict__ out, PhaseTimes* pt) {
  __shared__ __align__(16) uint32_t M[kExpandTile];
  __shared__ uint32_t red[34];
  pdl_wait();
  phase_mark(pt, 7);  // earliest expand start recorded as t[7] max; see dialsort_debug_phase_ns
  const uint64_t total = *ws_total;
  const uint32_t nw = (uint32_t)(total < cap ? total : cap);  // positions to write (< 2^32)
  const uint64_t ntw = ((uint64_t)nw + kExpandTile - 1) / kExpandTile;
  const bool aligned = (reinterpret_cast<uintptr_t>(out) & 15u) == 0;
  const uint64_t pol = l2_evict_first_policy();
  uint4* M4 = reinterpret_cast<uint4*>(M);

  for (uint64_t t = blockIdx.x; t < ntw; t += gridDim.x) {
    const uint32_t p0 = (uint32_t)(t * kExpandTile);
    const uint32_t p1 = (nw - p0 > kExpandTile) ? p0 + kExpandTile : nw;
    const uint32_t k_lo = tfb[t];
    const uint32_t k_hi = (t + 1 < ntiles && (uint64_t)p0 + kExpandTile < nw) ? tfb[t + 1] : U - 1;
    // 1. clear the marks
#pragma unroll
    for (uint32_t j = 0; j < kExpandPerThread; ++j) M4[threadIdx.x + j * kExpandThreads] = make_uint4(0, 0, 0, 0);
    __syncthreads();
    // 2. one mark per bin start inside the tile (P[k] > p0 for every k > k_lo)
    for (uint64_t k = (uint64_t)k_lo + 1 + threadIdx.x; k <= k_hi; k += kExpandThreads) {
      const uint32_t b = __ldcg(P + k);
      if (b < p1) {
        const uint32_t w = b - p0;
        atomicAdd(&M[(swz(w >> 2) << 2) | (w & 3u)], 1u);
      }
    }
    __syncthreads();
    // 3. inclusive scan of the marks -> keys (thread t owns positions 16t .. 16t+15)
    uint4 v[kExpandPerThread];
#pragma unroll
    for (uint32_t j = 0; j < kExpandPerThread; ++j) {
      v[j] = M4[swz(kExpandPerThread * threadIdx.x + j)];
      v[j].y += v[j].x;
      v[j].z += v[j].y;
      v[j].w += v[j].z;
    }
#pragma unroll
    for (uint32_t j = 1; j < kExpandPerThread; ++j) {
      v[j].x += v[j - 1].w; v[j].y += v[j - 1].w; v[j].z += v[j - 1].w; v[j].w += v[j - 1].w;
    }
    uint32_t tile_marks;
    const uint32_t ex = block_excl_scan<uint32_t>(v[kExpandPerThread - 1].w, tile_marks, red);
    const uint32_t base = (uint32_t)key_base + k_lo + ex;
#pragma unroll
    for (uint32_t j = 0; j < kExpandPerThread; ++j)
      M4[swz(kExpandPerThread * threadIdx.x + j)] =
          make_uint4(base + v[j].x, base + v[j].y, base + v[j].z, base + v[j].w);
    __syncthreads();
    // 4. copy out: lane-contiguous quads, 512 contiguous bytes per warp instruction
#pragma unroll
    for (uint32_t j = 0; j < kExpandPerThread; ++j) {
      const uint32_t qd = threadIdx.x + j * kExpandThreads;
      const uint32_t q = p0 + 4 * qd;
      if (q >= p1) continue;
      const uint4 x = M4[swz(qd)];
      if (aligned && q + 4 <= p1) {
        st_stream4(reinterpret_cast<int4*>(out + q), make_int4((int)x.x, (int)x.y, (int)x.z, (int)x.w), pol);
      } else {
        out[q] = (int)x.x;
        if (q + 1 < p1) out[q + 1] = (int)x.y;
        if (q + 2 < p1) out[q + 2] = (int)x.z;
        if (q + 3 < p1) out[q + 3] = (int)x.w;
      }
    }
    __syncthreads();  // M is reused by the next tile
  }
  pdl_trigger();
}

}  // namespace ds

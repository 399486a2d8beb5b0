// ds_part.cuh — hierarchical DialSort for universes larger than one SM's shared-memory
// histogram (the paper's "hierarchical partitioning is required" for large U, P:2780-2782,
// future work P:2847).
//
// U > kSmem16MaxBins: the keys are first partitioned by their high bits into B = ceil(U/2^16)
// universe blocks of 65536 bins (an MSD split on key >> 16 — order inside a block is
// irrelevant: the histogram is order-free, eq:ingestion P:409-412), each block's keys stored
// as their low 16 bits; then each block is sorted by k_sort_fused with U_b <= 65536 and
// key_base = b << 16, writing its output at the block's offset and its H slice at b << 16.
// This replaces one L2 RED per key (the global path, bound by the L2 atomic rate) with
// 10 bytes per key of streaming traffic (count read 4, scatter read 4 + write 2: the blocks
// hold their keys' low 16 bits as uint16) plus the shared-memory path of each block.
//
//   k_part_count    per-CTA chunk: block counts (per-warp shared counters)      [G][B]
//   k_part_scan     exclusive offsets off[c][b] (block-major), block sizes and starts
//   k_part_scatter  per-CTA chunk again, 4096-key sub-tiles staged in shared memory by
//                   block and written as contiguous runs at the CTA's offsets
#pragma once
#include "ds_common.cuh"

namespace ds {

constexpr uint32_t kPartShift = 16;         // 65536-bin universe blocks
constexpr uint32_t kPartMaxBlocks = 64;     // U <= 2^22: per-warp block counters (below)
constexpr uint32_t kPartMaxBlocksWide = 1024;  // 2^22 < U <= 2^26: per-CTA counters (k_part_*_wide)
#ifndef DIALSORT_PART_THREADS
#define DIALSORT_PART_THREADS 512
#endif
constexpr uint32_t kPartThreads = DIALSORT_PART_THREADS;
constexpr uint32_t kPartKPT = 8;            // keys per thread per scatter sub-tile
constexpr uint32_t kPartTile = kPartThreads * kPartKPT;  // 4096

struct PartWs {
  uint32_t* cnt;   // [G][B] block counts of each CTA chunk, then offsets (in place)
  uint64_t* bsz;   // [B] block sizes
  uint64_t* boff;  // [B] block starts
  DevStatus* st;
};

// Chunk [lo, hi) of CTA c in a grid of G over n keys.  Interior cuts sit on 256-byte
// boundaries of the key array (64 keys past its first 16-byte aligned element), so every
// chunk but the first starts aligned for the 16-byte vector loads (an unaligned start sends
// the scatter's sub-tiles to the scalar load path: 3 of 4 CTAs before this, c4 scatter
// 3.0 ms).  Both kernels of the count / scatter pair take the same cuts.
__device__ __forceinline__ void part_chunk(const int32_t* keys, uint64_t n, uint64_t& lo, uint64_t& hi) {
  const uint64_t a0 = ((16u - (reinterpret_cast<uintptr_t>(keys) & 15u)) & 15u) >> 2;
  auto cut = [&](uint32_t c) -> uint64_t {
    if (c == 0) return 0;
    if (c >= gridDim.x) return n;
    const uint64_t x = n * c / gridDim.x;
    const uint64_t y = a0 + ((x > a0 ? x - a0 : 0) & ~63ull);
    return y < n ? y : n;
  };
  lo = cut(blockIdx.x);
  hi = cut(blockIdx.x + 1);
}

__global__ void __launch_bounds__(kPartThreads) k_part_count(const int32_t* __restrict__ keys, uint64_t n, uint32_t U,
                                                             uint32_t B, PartWs w) {
  __shared__ uint32_t wcnt[kPartThreads / 32][kPartMaxBlocks];
  pdl_wait();
  const uint32_t warp = threadIdx.x >> 5;
  for (uint32_t i = threadIdx.x; i < (kPartThreads / 32) * kPartMaxBlocks; i += blockDim.x) (&wcnt[0][0])[i] = 0;
  __syncthreads();
  uint64_t lo, hi;
  part_chunk(keys, n, lo, hi);
  uint32_t* wc = wcnt[warp];
  auto one = [&](uint32_t k, uint64_t idx) {
    if (k < U) atomicAdd(&wc[k >> kPartShift], 1u);
    else record_bad(w.st, idx, k);
  };
  // 16-byte aligned interior as int4, scalar head / tail
  const uint64_t mis = (reinterpret_cast<uintptr_t>(keys + lo) >> 2) & 3u;
  const uint64_t a4 = min(hi, lo + ((4u - mis) & 3u));
  const uint64_t b4 = a4 + ((hi - a4) & ~3ull);
  for (uint64_t i = lo + threadIdx.x; i < a4; i += blockDim.x) one((uint32_t)keys[i], i);
  for (uint64_t i = b4 + threadIdx.x; i < hi; i += blockDim.x) one((uint32_t)keys[i], i);
  const int4* body = reinterpret_cast<const int4*>(keys + a4);
  const uint64_t nv = (b4 - a4) / 4;
  const uint64_t pol = l2_evict_first_policy();
  uint64_t v = threadIdx.x;
  for (; v + 3 * blockDim.x < nv; v += 4 * blockDim.x) {
    int4 x[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) x[u] = ld_stream4(body + v + u * blockDim.x, pol);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint64_t i0 = a4 + 4 * (v + u * blockDim.x);
      if (umax4(x[u]) < U) {
        atomicAdd(&wc[(uint32_t)x[u].x >> kPartShift], 1u);
        atomicAdd(&wc[(uint32_t)x[u].y >> kPartShift], 1u);
        atomicAdd(&wc[(uint32_t)x[u].z >> kPartShift], 1u);
        atomicAdd(&wc[(uint32_t)x[u].w >> kPartShift], 1u);
      } else {
        one((uint32_t)x[u].x, i0); one((uint32_t)x[u].y, i0 + 1); one((uint32_t)x[u].z, i0 + 2); one((uint32_t)x[u].w, i0 + 3);
      }
    }
  }
  for (; v < nv; v += blockDim.x) {
    const int4 x = ld_stream4(body + v, pol);
    const uint64_t i0 = a4 + 4 * v;
    one((uint32_t)x.x, i0); one((uint32_t)x.y, i0 + 1); one((uint32_t)x.z, i0 + 2); one((uint32_t)x.w, i0 + 3);
  }
  __syncthreads();
  if (threadIdx.x < B) {
    uint32_t s = 0;
#pragma unroll 4
    for (uint32_t q = 0; q < kPartThreads / 32; ++q) s += wcnt[q][threadIdx.x];
    w.cnt[(uint64_t)blockIdx.x * B + threadIdx.x] = s;
  }
  pdl_trigger();
}

// One CTA: off[c][b] = start(b) + Σ_{c' < c} cnt[c'][b], start(b) = Σ_{b' < b} size(b')
// (B <= 1024 blocks: thread b owns column b; one block scan of the sizes gives the starts).
__global__ void __launch_bounds__(1024) k_part_scan(uint32_t G, uint32_t B, PartWs w) {
  __shared__ unsigned long long red[34];
  pdl_wait();
  unsigned long long sz = 0;
  if (threadIdx.x < B)
    for (uint32_t c = 0; c < G; ++c) sz += w.cnt[(uint64_t)c * B + threadIdx.x];
  unsigned long long tot;
  const unsigned long long start = block_excl_scan<unsigned long long>(sz, tot, red);
  if (threadIdx.x < B) {
    w.bsz[threadIdx.x] = sz;
    w.boff[threadIdx.x] = start;
    uint64_t run = start;
    for (uint32_t c = 0; c < G; ++c) {
      const uint64_t x = w.cnt[(uint64_t)c * B + threadIdx.x];
      w.cnt[(uint64_t)c * B + threadIdx.x] = (uint32_t)run;  // positions < n < 2^32
      run += x;
    }
  }
  pdl_trigger();
}

// Re-reads the CTA's chunk and writes every valid key's low 16 bits into its universe block,
// sub-tile by sub-tile (4096 keys, 8 per thread as two 16-byte loads; the next sub-tile's
// loads are in flight while the current one is placed).  One shared atomic per key: the
// returned value of the per-warp block counter is the key's rank among the warp's keys of
// that block in this sub-tile (< 256), kept in the key's register next to the key itself
// (key < U <= 2^22 fills 22 bits, rank bits 22..29, bit 31 marks a dropped bad key).  A scan
// over (block, warp) turns the counters into slot bases, every key lands at base + rank in
// the staged sub-tile (order inside a block is free), and the sub-tile leaves as contiguous
// runs (~4096 / B keys per block) at the CTA's running block offsets.
// The chunk interior must be 16-byte aligned for the vector loads; other chunks take the
// scalar path (keys of an unaligned base).
#ifndef DIALSORT_PART_MINB
#define DIALSORT_PART_MINB (2048 / DIALSORT_PART_THREADS)  // 4 CTAs per SM (32 registers): more loads in flight (c4 6.44 -> 6.19 ms)
#endif
__global__ void __launch_bounds__(kPartThreads, DIALSORT_PART_MINB) k_part_scatter(const int32_t* __restrict__ keys, uint64_t n, uint32_t U,
                                                               uint32_t B, PartWs w, uint16_t* __restrict__ tmp) {
  constexpr uint32_t NW = kPartThreads / 32;
  constexpr uint32_t kBad = 0xffffffffu;
  __shared__ uint32_t wcnt[NW][kPartMaxBlocks];   // per-warp block counts of the sub-tile
  __shared__ uint32_t wbase[NW][kPartMaxBlocks];  // their slot bases in the staged sub-tile
  __shared__ uint32_t bofs[kPartMaxBlocks + 1], gpos[kPartMaxBlocks], delta[kPartMaxBlocks];
  __shared__ uint32_t stage[kPartTile];
  pdl_wait();
  const uint32_t warp = threadIdx.x >> 5;
  uint64_t lo, hi;
  part_chunk(keys, n, lo, hi);
  if (threadIdx.x < B) gpos[threadIdx.x] = w.cnt[(uint64_t)blockIdx.x * B + threadIdx.x];
  const bool vec = ((reinterpret_cast<uintptr_t>(keys + lo)) & 15u) == 0;
  // thread t holds sub-tile keys 8t .. 8t+7 (blocked: two int4)
  auto load = [&](uint64_t t0, uint32_t (&k)[kPartKPT]) {
    const uint64_t i0 = t0 + (uint64_t)kPartKPT * threadIdx.x;
    if (vec && i0 + kPartKPT <= hi) {
      const int4 x0 = __ldcs(reinterpret_cast<const int4*>(keys + i0));
      const int4 x1 = __ldcs(reinterpret_cast<const int4*>(keys + i0) + 1);
      k[0] = x0.x; k[1] = x0.y; k[2] = x0.z; k[3] = x0.w; k[4] = x1.x; k[5] = x1.y; k[6] = x1.z; k[7] = x1.w;
    } else {
#pragma unroll
      for (uint32_t i = 0; i < kPartKPT; ++i) k[i] = i0 + i < hi ? (uint32_t)keys[i0 + i] : kBad;
    }
  };
  unsigned short* const out = reinterpret_cast<unsigned short*>(tmp);
  for (uint32_t i = threadIdx.x; i < NW * kPartMaxBlocks; i += blockDim.x) (&wcnt[0][0])[i] = 0;
  __syncthreads();
  uint32_t k[kPartKPT], kn[kPartKPT];
  if (lo < hi) load(lo, k);
  // Three barriers per sub-tile: count | scan (warp 0) | stage | write-out + next count.
  // wcnt is zeroed by the scan warp once read, so the next sub-tile's counting (which
  // touches only wcnt) follows the write-out without a barrier between them.
  for (uint64_t t0 = lo; t0 < hi; t0 += kPartTile) {
    if (t0 + kPartTile < hi) load(t0 + kPartTile, kn);  // next sub-tile in flight
    uint32_t kmax = 0;
#pragma unroll
    for (uint32_t i = 0; i < kPartKPT; ++i) kmax = max(kmax, k[i]);
    if (kmax < U) {  // every key valid: no per-key test
#pragma unroll
      for (uint32_t i = 0; i < kPartKPT; ++i) k[i] |= atomicAdd(&wcnt[warp][k[i] >> kPartShift], 1u) << 22;
    } else {
#pragma unroll
      for (uint32_t i = 0; i < kPartKPT; ++i)
        k[i] = k[i] < U ? k[i] | (atomicAdd(&wcnt[warp][k[i] >> kPartShift], 1u) << 22) : kBad;
    }
    __syncthreads();
    if (warp == 0) {
      // lane l owns blocks l and l + 32: block totals over the NW warps, one warp scan of
      // the totals (block order), then the per-warp slot bases of each owned block.
      const uint32_t lane = threadIdx.x & 31;
      uint32_t t[2] = {0u, 0u};
      const uint32_t nh = B > 32 ? 2u : 1u;
      for (uint32_t h = 0; h < nh; ++h) {
        const uint32_t b = lane + 32 * h;
        if (b < B) {
#pragma unroll
          for (uint32_t q = 0; q < NW; ++q) t[h] += wcnt[q][b];
        }
      }
      const uint32_t i0 = warp_incl_scan(t[0]), i1 = nh > 1 ? warp_incl_scan(t[1]) : 0u;
      const uint32_t s0 = __shfl_sync(0xffffffffu, i0, 31);
      const uint32_t ex[2] = {i0 - t[0], s0 + i1 - t[1]};
      for (uint32_t h = 0; h < nh; ++h) {
        const uint32_t b = lane + 32 * h;
        if (b < B) {
          uint32_t base = ex[h];
          bofs[b] = base;
          delta[b] = gpos[b] - base;  // staged slot j of block b goes to position delta[b] + j
          gpos[b] += t[h];
#pragma unroll
          for (uint32_t q = 0; q < NW; ++q) {
            const uint32_t x = wcnt[q][b];
            wbase[q][b] = base;
            wcnt[q][b] = 0;
            base += x;
          }
        }
      }
      if (lane == 31) bofs[B] = s0 + (nh > 1 ? i1 : 0u);  // lane 31 holds both totals
    }
    __syncthreads();
    if (kmax < U) {
#pragma unroll
      for (uint32_t i = 0; i < kPartKPT; ++i) {
        const uint32_t key = k[i] & 0x3fffffu;
        stage[wbase[warp][key >> kPartShift] + (k[i] >> 22)] = key;
      }
    } else {
#pragma unroll
      for (uint32_t i = 0; i < kPartKPT; ++i)
        if (k[i] != kBad) {
          const uint32_t key = k[i] & 0x3fffffu;
          stage[wbase[warp][key >> kPartShift] + (k[i] >> 22)] = key;
        }
    }
    __syncthreads();
    const uint32_t nvld = bofs[B];  // valid keys of the sub-tile (bad keys were dropped)
    if (nvld == kPartTile) {
#pragma unroll
      for (uint32_t r = 0; r < kPartKPT; ++r) {
        const uint32_t j = r * kPartThreads + threadIdx.x, key = stage[j];
        __stcs(out + (delta[key >> kPartShift] + j), (unsigned short)(key & 0xffffu));
      }
    } else {
      for (uint32_t j = threadIdx.x; j < nvld; j += blockDim.x) {
        const uint32_t key = stage[j];
        __stcs(out + (delta[key >> kPartShift] + j), (unsigned short)(key & 0xffffu));
      }
    }
    // the next sub-tile's count barrier orders these stage / delta / bofs reads before the
    // scan warp and the staging rewrite them
#pragma unroll
    for (uint32_t i = 0; i < kPartKPT; ++i) k[i] = kn[i];
  }
  pdl_trigger();
}


// ---- wide partition (2^22 < U <= 2^26: up to 1024 universe blocks, NEXT-4) -----------------
// Per-CTA block counters in (dynamic) shared memory instead of per-warp ones: the rank a key
// takes inside its block of the sub-tile comes from the counting atomic (order inside a block is
// free), one block scan over the B counters gives the staged runs.  8192-key sub-tiles (16 keys
// per thread, 4 x 16-byte loads), so a block's run in a sub-tile averages 8192 / B keys.
constexpr uint32_t kPartWideKPT = 16;
constexpr uint32_t kPartWideTile = kPartThreads * kPartWideKPT;  // 8192 keys
__host__ __device__ constexpr size_t part_wide_smem(uint32_t B) {
  return 4ull * (4 * B + kPartWideTile) + 64;  // cnt, bstart, delta, gpos, stage
}

__global__ void __launch_bounds__(kPartThreads) k_part_count_wide(const int32_t* __restrict__ keys, uint64_t n,
                                                                  uint32_t U, uint32_t B, PartWs w) {
  extern __shared__ uint32_t ccnt[];
  pdl_wait();
  for (uint32_t i = threadIdx.x; i < B; i += blockDim.x) ccnt[i] = 0;
  __syncthreads();
  uint64_t lo, hi;
  part_chunk(keys, n, lo, hi);
  auto one = [&](uint32_t k, uint64_t idx) {
    if (k < U) atomicAdd(&ccnt[k >> kPartShift], 1u);
    else record_bad(w.st, idx, k);
  };
  const uint64_t mis = (reinterpret_cast<uintptr_t>(keys + lo) >> 2) & 3u;
  const uint64_t a4 = min(hi, lo + ((4u - mis) & 3u));
  const uint64_t b4 = a4 + ((hi - a4) & ~3ull);
  for (uint64_t i = lo + threadIdx.x; i < a4; i += blockDim.x) one((uint32_t)keys[i], i);
  for (uint64_t i = b4 + threadIdx.x; i < hi; i += blockDim.x) one((uint32_t)keys[i], i);
  const int4* body = reinterpret_cast<const int4*>(keys + a4);
  const uint64_t nv = (b4 - a4) / 4;
  const uint64_t pol = l2_evict_first_policy();
  uint64_t v = threadIdx.x;
  for (; v + 3 * blockDim.x < nv; v += 4 * blockDim.x) {
    int4 x[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) x[u] = ld_stream4(body + v + u * blockDim.x, pol);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint64_t i0 = a4 + 4 * (v + u * blockDim.x);
      if (umax4(x[u]) < U) {
        atomicAdd(&ccnt[(uint32_t)x[u].x >> kPartShift], 1u);
        atomicAdd(&ccnt[(uint32_t)x[u].y >> kPartShift], 1u);
        atomicAdd(&ccnt[(uint32_t)x[u].z >> kPartShift], 1u);
        atomicAdd(&ccnt[(uint32_t)x[u].w >> kPartShift], 1u);
      } else {
        one((uint32_t)x[u].x, i0); one((uint32_t)x[u].y, i0 + 1); one((uint32_t)x[u].z, i0 + 2); one((uint32_t)x[u].w, i0 + 3);
      }
    }
  }
  for (; v < nv; v += blockDim.x) {
    const int4 x = ld_stream4(body + v, pol);
    const uint64_t i0 = a4 + 4 * v;
    one((uint32_t)x.x, i0); one((uint32_t)x.y, i0 + 1); one((uint32_t)x.z, i0 + 2); one((uint32_t)x.w, i0 + 3);
  }
  __syncthreads();
  for (uint32_t b = threadIdx.x; b < B; b += blockDim.x) w.cnt[(uint64_t)blockIdx.x * B + b] = ccnt[b];
  pdl_trigger();
}

__global__ void __launch_bounds__(kPartThreads) k_part_scatter_wide(const int32_t* __restrict__ keys, uint64_t n,
                                                                    uint32_t U, uint32_t B, PartWs w,
                                                                    uint16_t* __restrict__ tmp) {
  extern __shared__ uint32_t psh[];
  __shared__ uint32_t red[34];
  uint32_t* cnt = psh;             // [B] this sub-tile's block counts (zero between sub-tiles)
  uint32_t* bstart = cnt + B;      // [B] staged run starts
  int32_t* delta = reinterpret_cast<int32_t*>(bstart + B);  // [B] output index of staged slot j: delta + j
  uint32_t* gpos = reinterpret_cast<uint32_t*>(delta + B);  // [B] running output position of block b
  uint32_t* stage = gpos + B;      // [kPartWideTile] keys by block
  constexpr uint32_t kBad = 0xffffffffu;
  pdl_wait();
  uint64_t lo, hi;
  part_chunk(keys, n, lo, hi);
  for (uint32_t b = threadIdx.x; b < B; b += blockDim.x) {
    cnt[b] = 0;
    gpos[b] = w.cnt[(uint64_t)blockIdx.x * B + b];
  }
  const bool vec = ((reinterpret_cast<uintptr_t>(keys + lo)) & 15u) == 0;
  __syncthreads();
  uint16_t* const out = tmp;
  for (uint64_t t0 = lo; t0 < hi; t0 += kPartWideTile) {
    // thread t holds sub-tile keys 16t .. 16t+15
    uint32_t k[kPartWideKPT];
    uint16_t r[kPartWideKPT];
    const uint64_t i0 = t0 + (uint64_t)kPartWideKPT * threadIdx.x;
    if (vec && i0 + kPartWideKPT <= hi) {
#pragma unroll
      for (uint32_t q = 0; q < kPartWideKPT / 4; ++q) {
        const int4 x = __ldcs(reinterpret_cast<const int4*>(keys + i0) + q);
        k[4 * q] = x.x; k[4 * q + 1] = x.y; k[4 * q + 2] = x.z; k[4 * q + 3] = x.w;
      }
    } else {
#pragma unroll
      for (uint32_t i = 0; i < kPartWideKPT; ++i) k[i] = i0 + i < hi ? (uint32_t)keys[i0 + i] : kBad;
    }
#pragma unroll
    for (uint32_t i = 0; i < kPartWideKPT; ++i) {
      if (k[i] >= U) k[i] = kBad;  // (bad keys were recorded by the count pass)
      r[i] = k[i] != kBad ? (uint16_t)atomicAdd(&cnt[k[i] >> kPartShift], 1u) : (uint16_t)0;
    }
    __syncthreads();
    // exclusive scan of the counts over the blocks (2 per thread at 512 threads, B <= 1024)
    {
      const uint32_t b0 = 2 * threadIdx.x;
      const uint32_t c0 = b0 < B ? cnt[b0] : 0u, c1 = b0 + 1 < B ? cnt[b0 + 1] : 0u;
      uint32_t tot;
      const uint32_t ex = block_excl_scan<uint32_t>(c0 + c1, tot, red);
      if (b0 < B) {
        bstart[b0] = ex;
        delta[b0] = (int32_t)(gpos[b0] - ex);
        gpos[b0] += c0;
        cnt[b0] = 0;
      }
      if (b0 + 1 < B) {
        bstart[b0 + 1] = ex + c0;
        delta[b0 + 1] = (int32_t)(gpos[b0 + 1] - ex - c0);
        gpos[b0 + 1] += c1;
        cnt[b0 + 1] = 0;
      }
      if (threadIdx.x == 0) red[33] = tot;
    }
    __syncthreads();
    const uint32_t nvld = red[33];
#pragma unroll
    for (uint32_t i = 0; i < kPartWideKPT; ++i)
      if (k[i] != kBad) stage[bstart[k[i] >> kPartShift] + r[i]] = k[i];
    __syncthreads();
    for (uint32_t j = threadIdx.x; j < nvld; j += blockDim.x) {
      const uint32_t key = stage[j];
      __stcs(reinterpret_cast<unsigned short*>(out) + (delta[key >> kPartShift] + (int32_t)j),
             (unsigned short)(key & 0xffffu));
    }
    __syncthreads();  // stage / delta are rewritten by the next sub-tile
  }
  pdl_trigger();
}

}  // namespace ds

// ds_radix.cuh — DialSort-Radix (tab:radix P:1659-1679): full signed int32,
// "LSD, base 256, 4 passes, zero order comparisons".
//
// Each pass p is a 256-bin DialSort over digit d = (u >> 8p) & 0xFF of the sign-flipped key
// u = x ^ 0x80000000 (reading R2): ingestion (K7 computes all four 256-bin digit histograms
// in one read of the keys), the per-digit write offsets (tab:related "Per digit" prefix sum),
// and a stable scatter.  On the GPU the scatter is a single-sweep pass (K8): each 8192-key
// tile ranks its keys stably with an equality-only warp multisplit (8 ballots per key — the
// CRN's equality grouping applied to digits), gets its cross-tile digit offsets by a
// decoupled look-back, sorts the tile by digit in shared memory and writes digit runs.
// HBM traffic: 4n (K7) + 4 x 8n (K8) = 36n bytes.
#pragma once
#include "ds_common.cuh"

namespace ds {

constexpr int kRadixThreads = 512;
constexpr int kRadixWarps = kRadixThreads / 32;
constexpr int kRadixKPT = 16;
constexpr int kRadixTile = kRadixThreads * kRadixKPT;  // 8192 keys
constexpr uint32_t kSignFlip = 0x80000000u;

// K7: the four 256-bin digit histograms of the flipped keys (eq:ingestion with U=256 per digit).
// ghist[4*256] must be zero on entry; ctrs[4] (dynamic tile counters of K8) are zeroed here.
__global__ void __launch_bounds__(512) k_radix_hist4(const int32_t* __restrict__ keys, uint64_t n,
                                                     uint32_t* __restrict__ ghist, uint32_t* ctrs) {
  __shared__ uint32_t h[4][256];
  pdl_wait();
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) (&h[0][0])[i] = 0;
  if (blockIdx.x == 0 && threadIdx.x < 4) ctrs[threadIdx.x] = 0;
  __syncthreads();
  auto ingest = [&](uint32_t x) {
    uint32_t u = x ^ kSignFlip;
    atomicAdd(&h[0][u & 0xff], 1u);
    atomicAdd(&h[1][(u >> 8) & 0xff], 1u);
    atomicAdd(&h[2][(u >> 16) & 0xff], 1u);
    atomicAdd(&h[3][u >> 24], 1u);
  };
  const uint64_t mis = (reinterpret_cast<uintptr_t>(keys) >> 2) & 3u;
  uint64_t head = mis ? 4 - mis : 0;
  if (head > n) head = n;
  const uint64_t n4 = (n - head) / 4, tail = n - head - 4 * n4;
  if (blockIdx.x == 0 && threadIdx.x < head) ingest((uint32_t)keys[threadIdx.x]);
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x < tail) ingest((uint32_t)keys[head + 4 * n4 + threadIdx.x]);
  const int4* body = reinterpret_cast<const int4*>(keys + head);
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n4; i += 4 * stride) {
    int4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = ld_stream4(body + i + u * stride);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      ingest((uint32_t)v[u].x); ingest((uint32_t)v[u].y); ingest((uint32_t)v[u].z); ingest((uint32_t)v[u].w);
    }
  }
  for (; i < n4; i += stride) {
    int4 v = ld_stream4(body + i);
    ingest((uint32_t)v.x); ingest((uint32_t)v.y); ingest((uint32_t)v.z); ingest((uint32_t)v.w);
  }
  __syncthreads();
  for (int j = threadIdx.x; j < 1024; j += blockDim.x) {
    uint32_t c = (&h[0][0])[j];
    if (c) atomicAdd(ghist + j, c);
  }
  pdl_trigger();
}

// Equality-only warp multisplit on an 8-bit digit: mask of the valid lanes whose digit equals
// mine (8 ballots; no order comparison between keys, def:ordercomp P:337-345).
__device__ __forceinline__ uint32_t digit_group(uint32_t d, uint32_t valid_mask) {
  uint32_t m = valid_mask;
#pragma unroll
  for (int b = 0; b < 8; ++b) {
    uint32_t bb = __ballot_sync(FULL, (d >> b) & 1u);
    m &= ((d >> b) & 1u) ? bb : ~bb;
  }
  return m;
}

struct RadixSmem {
  uint32_t keys[kRadixTile];              // tile sorted by digit
  uint32_t whist[kRadixWarps][256];       // per-warp digit counts -> exclusive offsets
  uint32_t tile_excl[256];                // exclusive scan of the tile's digit counts
  uint64_t base[256];                     // global position of local index 0 for digit d
  uint32_t red[34];
  uint32_t tile_id;
};

// K8: one stable scatter pass by digit p.  src holds raw int32 keys when p == 0 (flipped on
// load), flipped keys otherwise; the last pass (p == 3) un-flips on store.
__global__ void __launch_bounds__(kRadixThreads) k_radix_pass(const uint32_t* __restrict__ src,
                                                               uint32_t* __restrict__ dst, uint64_t n,
                                                               int p, const uint32_t* __restrict__ ghist,
                                                               uint64_t* __restrict__ status,
                                                               uint32_t* ctr, uint32_t tag) {
  extern __shared__ __align__(16) unsigned char radix_smem_raw[];
  RadixSmem& S = *reinterpret_cast<RadixSmem*>(radix_smem_raw);
  pdl_wait();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) S.tile_id = atomicAdd(ctr, 1u);  // dynamic tile order: forward progress
  for (int i = threadIdx.x; i < kRadixWarps * 256; i += blockDim.x) (&S.whist[0][0])[i] = 0;
  __syncthreads();
  const uint64_t tile = S.tile_id;
  const uint64_t tbase = tile * kRadixTile;
  const int shift = 8 * p;
  const uint32_t flip_in = p == 0 ? kSignFlip : 0u;

  // 1. load (warp-striped: item i of warp w is tbase + w*32*KPT + i*32 + lane)
  uint32_t k[kRadixKPT];
  uint32_t rank[kRadixKPT];
  const uint64_t wbase = tbase + (uint64_t)warp * 32 * kRadixKPT;
#pragma unroll
  for (int i = 0; i < kRadixKPT; ++i) {
    uint64_t idx = wbase + i * 32 + lane;
    k[i] = idx < n ? (__ldcs(src + idx) ^ flip_in) : 0u;
  }
  // 2. stable in-warp ranks (item order, then lane order)
  const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
  for (int i = 0; i < kRadixKPT; ++i) {
    const uint64_t idx0 = wbase + i * 32;
    const uint32_t vmask = idx0 >= n ? 0u : (n - idx0 >= 32 ? FULL : ((1u << (n - idx0)) - 1u));
    const uint32_t d = (k[i] >> shift) & 0xffu;
    const uint32_t g = digit_group(d, vmask);
    const bool valid = (vmask >> lane) & 1u;
    uint32_t before = valid ? S.whist[warp][d] : 0u;
    __syncwarp();
    if (valid) {
      rank[i] = before + __popc(g & lt);
      if ((g & lt) == 0) S.whist[warp][d] = before + __popc(g);  // group leader
    }
    __syncwarp();
  }
  __syncthreads();
  // 3. per digit: exclusive offsets across warps; tile count
  uint32_t cnt = 0;
  if (threadIdx.x < 256) {
    const int d = threadIdx.x;
    for (int w = 0; w < kRadixWarps; ++w) {
      uint32_t c = S.whist[w][d];
      S.whist[w][d] = cnt;
      cnt += c;
    }
  }
  // 4. tile-local digit scan and the global digit starts (exclusive scan of the pass's
  //    256-bin histogram) — block scans, threads >= 256 contribute 0
  uint32_t tile_total, gtotal;
  uint32_t ex = block_excl_scan<uint32_t>(threadIdx.x < 256 ? cnt : 0u, tile_total, S.red);
  uint32_t gstart = block_excl_scan<uint32_t>(threadIdx.x < 256 ? __ldcg(ghist + 256 * p + threadIdx.x) : 0u,
                                              gtotal, S.red);
  // 5. decoupled look-back per digit (thread d), plus global digit start
  if (threadIdx.x < 256) {
    const int d = threadIdx.x;
    S.tile_excl[d] = ex;
    uint64_t* my = status + tile * 256 + d;
    uint64_t excl = 0;
    if (tile == 0) {
      lb_store(my, lb_pack(tag, LB_FLAG_INC, cnt));
    } else {
      lb_store(my, lb_pack(tag, LB_FLAG_AGG, cnt));
      const uint32_t ep = tag & 0xffffffu;
      for (int64_t t = (int64_t)tile - 1; t >= 0; --t) {
        uint64_t s;
        uint32_t f;
        do {
          s = lb_load(status + t * 256 + d);
          f = ((uint32_t)(s >> 40) == ep) ? (uint32_t)((s >> LB_VALUE_BITS) & 3) : 0u;
        } while (f == 0);
        excl += s & LB_VALUE_MASK;
        if (f == LB_FLAG_INC) break;
      }
      lb_store(my, lb_pack(tag, LB_FLAG_INC, excl + cnt));
    }
    S.base[d] = (uint64_t)gstart + excl - ex;
  }
  __syncthreads();
  // 6. sort the tile by digit in shared memory
#pragma unroll
  for (int i = 0; i < kRadixKPT; ++i) {
    const uint64_t idx = wbase + i * 32 + lane;
    if (idx < n) {
      const uint32_t d = (k[i] >> shift) & 0xffu;
      S.keys[S.tile_excl[d] + S.whist[warp][d] + rank[i]] = k[i];
    }
  }
  __syncthreads();
  pdl_trigger();
  // 7. write digit runs (consecutive threads -> consecutive addresses inside a run)
  const uint32_t tile_n = (uint32_t)((n - tbase) < (uint64_t)kRadixTile ? (n - tbase) : kRadixTile);
  const uint32_t flip_out = p == 3 ? kSignFlip : 0u;
  for (uint32_t j = threadIdx.x; j < tile_n; j += blockDim.x) {
    const uint32_t u = S.keys[j];
    const uint32_t d = (u >> shift) & 0xffu;
    __stcs(dst + S.base[d] + j, u ^ flip_out);
  }
}

inline void radix_configure() {
  cudaFuncSetAttribute(k_radix_pass, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(RadixSmem));
}

}  // namespace ds


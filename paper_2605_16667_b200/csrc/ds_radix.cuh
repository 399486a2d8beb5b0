// ds_radix.cuh — DialSort-Radix (tab:radix P:1659-1679): full signed int32,
// "LSD, base 256, 4 passes, zero order comparisons".
//
// Pass p is a 256-bin DialSort of the digit d = (u >> 8p) & 0xFF of the sign-flipped key
// u = x ^ 0x80000000 (reading R2): ingestion of the digit histogram (eq:ingestion with U=256),
// the per-digit write offsets (the per-digit prefix sum radix needs, tab:related "Per digit"),
// and a stable scatter.  GPU form (a single sweep per pass):
//   K7  k_radix_hist0: one read of the keys -> digit-0 histogram; clears the pass-0 look-back
//       statuses, the tile counters and the digit-1..3 histograms.
//   K8  k_radix_pass(p), persistent CTAs taking 4096-key tiles in dynamic order:
//       - stable in-tile ranks: per warp and item, the lanes are grouped by equal digit with
//         one MATCH.ANY (the CRN's equality grouping applied to digits); the group leader
//         advances the warp's digit counter and broadcasts the base by shuffle;
//       - cross-tile digit offsets by decoupled look-back (u32 status per tile and digit);
//       - the tile is sorted by digit in shared memory and leaves as digit runs;
//       - the histogram of the NEXT digit is counted on the way (one shared atomic per key),
//         so the keys are read once per pass plus once in K7.
//       It also clears the look-back statuses of the next pass (ping-pong arrays).
// HBM traffic: 4n (K7) + 4 x 8n (K8) = 36n bytes.
#pragma once
#include "ds_common.cuh"

namespace ds {

// Sense-reversing grid barrier for the co-resident radix grid (same protocol as ds_scan.cuh).
struct GridBarR {
  unsigned int count;
  unsigned int gen;
};
__device__ __forceinline__ void grid_barrier_r(GridBarR* gb) {
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned g, old;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(&gb->gen) : "memory");
    asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(old) : "l"(&gb->count) : "memory");
    if (old == gridDim.x - 1) {
      asm volatile("st.relaxed.gpu.global.u32 [%0], 0;" ::"l"(&gb->count) : "memory");
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(&gb->gen) : "memory");
    } else {
      unsigned cur;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(&gb->gen) : "memory");
      } while (cur == g);
    }
  }
  __syncthreads();
}

constexpr int kRadixThreads = 512;
constexpr int kRadixWarps = kRadixThreads / 32;
constexpr int kRadixKPT = 8;
constexpr int kRadixTile = kRadixThreads * kRadixKPT;  // 4096 keys
constexpr uint32_t kSignFlip = 0x80000000u;
constexpr uint32_t kRxAgg = 1u << 30, kRxInc = 2u << 30, kRxValMask = (1u << 30) - 1;  // status: flag:2 | value:30

// Workspace: ghist[4][256] u32, ctrs[4] u32, status[2][ntiles][256] u32.
struct RadixWs {
  uint32_t* ghist;
  uint32_t* ctrs;
  uint32_t* status;  // 2 * ntiles * 256
  uint32_t ntiles;
};

// K7: digit-0 histogram of the flipped keys; clears pass-0 statuses, counters, ghist[1..3].
__global__ void __launch_bounds__(512) k_radix_hist0(const int32_t* __restrict__ keys, uint64_t n, RadixWs w) {
  __shared__ uint32_t h[256];
  pdl_wait();
  for (int i = threadIdx.x; i < 256; i += blockDim.x) h[i] = 0;
  const uint64_t gtid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x, gsz = (uint64_t)gridDim.x * blockDim.x;
  if (gtid < 4) w.ctrs[gtid] = 0;
  for (uint64_t i = gtid; i < 768; i += gsz) w.ghist[256 + i] = 0;
  {  // clear status array 0 (pass 0): ntiles * 256 words
    uint4* s4 = reinterpret_cast<uint4*>(w.status);
    const uint64_t n4 = (uint64_t)w.ntiles * 64;
    for (uint64_t i = gtid; i < n4; i += gsz) s4[i] = make_uint4(0, 0, 0, 0);
  }
  __syncthreads();
  const uint64_t mis = (reinterpret_cast<uintptr_t>(keys) >> 2) & 3u;
  uint64_t head = mis ? 4 - mis : 0;
  if (head > n) head = n;
  const uint64_t n4 = (n - head) / 4, tail = n - head - 4 * n4;
  const uint64_t pol = l2_evict_first_policy();
  if (blockIdx.x == 0 && threadIdx.x < head) atomicAdd(&h[((uint32_t)keys[threadIdx.x] ^ kSignFlip) & 0xffu], 1u);
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x < tail)
    atomicAdd(&h[((uint32_t)keys[head + 4 * n4 + threadIdx.x] ^ kSignFlip) & 0xffu], 1u);
  const int4* body = reinterpret_cast<const int4*>(keys + head);
  uint64_t i = gtid;
  for (; i + 3 * gsz < n4; i += 4 * gsz) {
    int4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = ld_stream4(body + i + u * gsz, pol);
#pragma unroll
    for (int u = 0; u < 4; ++u) {  // digit 0 of u = x ^ 0x80000000 is the low byte of x
      atomicAdd(&h[(uint32_t)v[u].x & 0xffu], 1u);
      atomicAdd(&h[(uint32_t)v[u].y & 0xffu], 1u);
      atomicAdd(&h[(uint32_t)v[u].z & 0xffu], 1u);
      atomicAdd(&h[(uint32_t)v[u].w & 0xffu], 1u);
    }
  }
  for (; i < n4; i += gsz) {
    const int4 v = ld_stream4(body + i, pol);
    atomicAdd(&h[(uint32_t)v.x & 0xffu], 1u);
    atomicAdd(&h[(uint32_t)v.y & 0xffu], 1u);
    atomicAdd(&h[(uint32_t)v.z & 0xffu], 1u);
    atomicAdd(&h[(uint32_t)v.w & 0xffu], 1u);
  }
  __syncthreads();
  for (int j = threadIdx.x; j < 256; j += blockDim.x)
    if (h[j]) atomicAdd(w.ghist + j, h[j]);
  pdl_trigger();
}

// Equality-only warp multisplit on an 8-bit digit: the mask of the lanes (of valid_mask)
// whose digit equals mine, from 8 ballots (no order comparison, def:ordercomp P:337-345).
// Must be called by exactly the lanes of valid_mask.
__device__ __forceinline__ uint32_t digit_group(uint32_t d, uint32_t valid_mask) {
  uint32_t m = valid_mask;
#pragma unroll
  for (int b = 0; b < 8; ++b) {
    const uint32_t bb = __ballot_sync(valid_mask, (d >> b) & 1u);
    m &= ((d >> b) & 1u) ? bb : ~bb;
  }
  return m;
}

struct RadixSmem {
  uint32_t wmask[2][kRadixWarps][256];  // per-warp digit -> lane-mask (equality grouping), 2 buffers (32 KB)
  uint32_t keys[kRadixTile];          // tile sorted by digit (16 KB)
  uint32_t wcnt[kRadixWarps][256];    // per-warp digit counts -> exclusive offsets (16 KB)
  uint32_t hnext[256];                // histogram of the next digit (this CTA)
  uint32_t gstart[256];               // exclusive prefix of this pass's global digit histogram
  uint32_t tile_excl[256];            // exclusive scan of the tile's digit counts
  uint32_t base[256];                 // global position of local index 0 for digit d
  uint32_t red[34];
  uint32_t tile_id;
};

// K8: one stable scatter pass by digit p (persistent, dynamic tiles).  src holds raw int32
// keys when p == 0 (flipped on load), flipped keys otherwise; the last pass un-flips.
__global__ void __launch_bounds__(kRadixThreads, 2) k_radix_pass(const uint32_t* __restrict__ src,
                                                                  uint32_t* __restrict__ dst, uint32_t n, int p,
                                                                  RadixWs w) {
  extern __shared__ __align__(16) unsigned char radix_smem_raw[];
  RadixSmem& S = *reinterpret_cast<RadixSmem*>(radix_smem_raw);
  pdl_wait();
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t dsel = 0x4440u | (uint32_t)p, nsel = 0x4440u | (uint32_t)(p + 1);  // PRMT: byte p / p+1
  const uint32_t flip_in = p == 0 ? kSignFlip : 0u, flip_out = p == 3 ? kSignFlip : 0u;
  const uint32_t ntiles = w.ntiles;
  uint32_t* status = w.status + (size_t)(p & 1) * ntiles * 256;
  // clear the next pass's status array (pass p+1 starts after this kernel completes)
  if (p < 3) {
    uint4* s4 = reinterpret_cast<uint4*>(w.status + (size_t)((p + 1) & 1) * ntiles * 256);
    const uint64_t n4 = (uint64_t)ntiles * 64, gsz = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n4; i += gsz) s4[i] = make_uint4(0, 0, 0, 0);
  }
  // global digit starts (exclusive scan of ghist[p]) and the next-digit histogram
  uint32_t gtot;
  const uint32_t gs = block_excl_scan<uint32_t>(threadIdx.x < 256 ? __ldcg(w.ghist + 256 * p + threadIdx.x) : 0u,
                                                gtot, S.red);
  if (threadIdx.x < 256) {
    S.gstart[threadIdx.x] = gs;
    S.hnext[threadIdx.x] = 0;
  }
  const uint32_t lt = (1u << lane) - 1u;
  for (;;) {
    if (threadIdx.x == 0) S.tile_id = atomicAdd(w.ctrs + p, 1u);
    for (int i = threadIdx.x; i < kRadixWarps * 256; i += blockDim.x) (&S.wcnt[0][0])[i] = 0;
    __syncthreads();
    const uint32_t tile = S.tile_id;
    if (tile >= ntiles) break;
    const uint32_t tbase = tile * kRadixTile;
    const uint32_t tile_n = (n - tbase) < (uint32_t)kRadixTile ? (n - tbase) : (uint32_t)kRadixTile;
    // 1. load (warp-striped: item i of warp w is tbase + w*32*KPT + i*32 + lane)
    uint32_t k[kRadixKPT], rank[kRadixKPT];
    const uint32_t wbase = tbase + warp * 32 * kRadixKPT;
#pragma unroll
    for (int i = 0; i < kRadixKPT; ++i) {
      const uint32_t idx = wbase + i * 32 + lane;
      k[i] = idx < n ? (__ldcs(src + idx) ^ flip_in) : 0u;
    }
    // 2. stable in-warp ranks: equality grouping of digits (MATCH.ANY), leader advances the
    //    warp counter, shuffle broadcasts the group base
#pragma unroll
    for (int i = 0; i < kRadixKPT; ++i) {
      const uint32_t idx0 = wbase + i * 32;
      const uint32_t vmask = idx0 >= n ? 0u : (n - idx0 >= 32 ? FULL : ((1u << (n - idx0)) - 1u));
      if ((vmask >> lane) & 1u) {
        const uint32_t d = __byte_perm(k[i], 0, dsel);
        const uint32_t g = __match_any_sync(vmask, d);
        const uint32_t leader = __ffs(g) - 1;
        uint32_t old = 0;
        if (lane == leader) {
          old = S.wcnt[warp][d];
          S.wcnt[warp][d] = old + __popc(g);
        }
        rank[i] = __shfl_sync(vmask, old, leader) + __popc(g & lt);
      }
    }
    __syncthreads();
    // 3. per digit: exclusive offsets across warps and the tile count
    uint32_t cnt = 0;
    if (threadIdx.x < 256) {
      const int d = threadIdx.x;
#pragma unroll
      for (int ww = 0; ww < kRadixWarps; ++ww) {
        const uint32_t c = S.wcnt[ww][d];
        S.wcnt[ww][d] = cnt;
        cnt += c;
      }
    }
    uint32_t tile_total;
    const uint32_t ex = block_excl_scan<uint32_t>(threadIdx.x < 256 ? cnt : 0u, tile_total, S.red);
    // 4. decoupled look-back per digit (thread d): publish the aggregate, sum predecessors
    //    back to the first inclusive prefix, publish the inclusive prefix
    if (threadIdx.x < 256) {
      const uint32_t d = threadIdx.x;
      S.tile_excl[d] = ex;
      uint32_t excl = 0;
      if (tile == 0) {
        asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(status + d), "r"(kRxInc | cnt) : "memory");
      } else {
        asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(status + (size_t)tile * 256 + d), "r"(kRxAgg | cnt)
                     : "memory");
        // Look back 8 predecessors per round: the 8 loads are independent (one L2 round trip;
        // a warp reads 32 consecutive digits of a tile, coalesced), then consumed in order.
        // Statuses only move 0 -> aggregate -> inclusive, so a stale aggregate is still a
        // correct partial sum; only "not ready" (0) is waited for.
        int64_t t = (int64_t)tile - 1;
        bool done = false;
        while (!done) {
          uint32_t sv[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            sv[j] = kRxInc;  // tiles before 0: inclusive zero
            if (t - j >= 0)
              asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(sv[j]) : "l"(status + (size_t)(t - j) * 256 + d)
                           : "memory");
          }
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            if (done) break;
            uint32_t sj = sv[j];
            while ((sj >> 30) == 0)
              asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(sj) : "l"(status + (size_t)(t - j) * 256 + d)
                           : "memory");
            excl += sj & kRxValMask;
            if ((sj >> 30) == 2) done = true;
          }
          t -= 8;
        }
        asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(status + (size_t)tile * 256 + d),
                     "r"(kRxInc | (excl + cnt))
                     : "memory");
      }
      S.base[d] = S.gstart[d] + excl - ex;
    }
    __syncthreads();
    // 5. sort the tile by digit in shared memory
#pragma unroll
    for (int i = 0; i < kRadixKPT; ++i) {
      const uint32_t idx = wbase + i * 32 + lane;
      if (idx < n) {
        const uint32_t d = __byte_perm(k[i], 0, dsel);
        S.keys[S.tile_excl[d] + S.wcnt[warp][d] + rank[i]] = k[i];
      }
    }
    __syncthreads();
    // 6. write digit runs; count the next digit on the way
    for (uint32_t j = threadIdx.x; j < tile_n; j += blockDim.x) {
      const uint32_t u = S.keys[j];
      const uint32_t pos = S.base[__byte_perm(u, 0, dsel)] + j;  // 32-bit position (n < 2^30)
      __stcs(dst + pos, u ^ flip_out);
      if (p < 3) atomicAdd(&S.hnext[__byte_perm(u, 0, nsel)], 1u);
    }
    __syncthreads();  // S.keys / S.wcnt reused by the next tile
  }
  if (p < 3 && threadIdx.x < 256 && S.hnext[threadIdx.x]) atomicAdd(w.ghist + 256 * (p + 1) + threadIdx.x, S.hnext[threadIdx.x]);
  pdl_trigger();
}

// ---- K8' reduce-then-scan pass (default) -----------------------------------------------------
// One co-resident persistent grid per pass; CTA c owns the contiguous key chunk
// [c*n/G, (c+1)*n/G).  Phase 1 counts the chunk's digits (the pass's DialSort ingestion)
// into cnt[c][256]; after a grid barrier CTA d (< 256) scans column d over the chunks into
// pre[.][d] and total[d]; after a second barrier every CTA knows gstart (scan of total) and
// its row pre[c], and scatters its chunk in 4096-key sub-tiles with running per-digit offsets
// — stable (chunks in order, sub-tiles in order, MATCH.ANY ranks inside), with no
// look-back chain.  12n bytes per pass (the chunk is read twice).
struct Radix2Ws {
  uint32_t* cnt;    // [G][256]
  uint32_t* pre;    // [G][256]
  uint32_t* total;  // [256]
  GridBarR* bar;
  PhaseTimes* pt;   // nullable debug timing
};

__global__ void __launch_bounds__(kRadixThreads, 2) k_radix_pass2(const uint32_t* __restrict__ src,
                                                                   uint32_t* __restrict__ dst, uint32_t n, int p,
                                                                   Radix2Ws w) {
  extern __shared__ __align__(16) unsigned char radix_smem_raw[];
  RadixSmem& S = *reinterpret_cast<RadixSmem*>(radix_smem_raw);
  pdl_wait();
  phase_mark(w.pt, -1);
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5, G = gridDim.x, c = blockIdx.x;
  const uint32_t dsel = 0x4440u | (uint32_t)p;
  const uint32_t flip_in = p == 0 ? kSignFlip : 0u, flip_out = p == 3 ? kSignFlip : 0u;
  const uint32_t lo = (uint32_t)((uint64_t)n * c / G), hi = (uint32_t)((uint64_t)n * (c + 1) / G);
  // ---- phase 1: digit counts of the chunk
  if (threadIdx.x < 256) S.hnext[threadIdx.x] = 0;
  __syncthreads();
  {
    const uint64_t pol = l2_evict_first_policy();
    // [a4, b4): the 16-byte-aligned interior of the chunk (src may have any 4-byte alignment)
    const uint32_t mis = (uint32_t)((reinterpret_cast<uintptr_t>(src) >> 2) & 3u);
    const uint32_t a4 = min(hi, lo + ((4u - ((lo + mis) & 3u)) & 3u));
    const uint32_t b4 = a4 + ((hi - a4) & ~3u);
    for (uint32_t i = lo + threadIdx.x; i < min(a4, hi); i += blockDim.x)
      atomicAdd(&S.hnext[__byte_perm(__ldcs(src + i) ^ flip_in, 0, dsel)], 1u);
    if (a4 < b4) {
      const int4* body = reinterpret_cast<const int4*>(src + a4);
      const uint32_t nv = (b4 - a4) / 4;
      uint32_t v = threadIdx.x;
      for (; v + 3 * blockDim.x < nv; v += 4 * blockDim.x) {
        int4 x[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) x[u] = ld_stream4(body + v + u * blockDim.x, pol);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          atomicAdd(&S.hnext[__byte_perm((uint32_t)x[u].x ^ flip_in, 0, dsel)], 1u);
          atomicAdd(&S.hnext[__byte_perm((uint32_t)x[u].y ^ flip_in, 0, dsel)], 1u);
          atomicAdd(&S.hnext[__byte_perm((uint32_t)x[u].z ^ flip_in, 0, dsel)], 1u);
          atomicAdd(&S.hnext[__byte_perm((uint32_t)x[u].w ^ flip_in, 0, dsel)], 1u);
        }
      }
      for (; v < nv; v += blockDim.x) {
        const int4 x = ld_stream4(body + v, pol);
        atomicAdd(&S.hnext[__byte_perm((uint32_t)x.x ^ flip_in, 0, dsel)], 1u);
        atomicAdd(&S.hnext[__byte_perm((uint32_t)x.y ^ flip_in, 0, dsel)], 1u);
        atomicAdd(&S.hnext[__byte_perm((uint32_t)x.z ^ flip_in, 0, dsel)], 1u);
        atomicAdd(&S.hnext[__byte_perm((uint32_t)x.w ^ flip_in, 0, dsel)], 1u);
      }
    }
    for (uint32_t i = b4 + threadIdx.x; i < hi; i += blockDim.x)
      atomicAdd(&S.hnext[__byte_perm(__ldcs(src + i) ^ flip_in, 0, dsel)], 1u);
  }
  __syncthreads();
  if (threadIdx.x < 256) __stcg(w.cnt + (size_t)c * 256 + threadIdx.x, S.hnext[threadIdx.x]);
  phase_mark(w.pt, 0);
  grid_barrier_r(w.bar);
  phase_mark(w.pt, 1);
  // ---- phase 2: column scans (CTA d scans digit d over the G chunks)
  for (uint32_t d = c; d < 256; d += G) {
    uint32_t carry = 0;
    for (uint32_t c0 = 0; c0 < G; c0 += blockDim.x) {
      const uint32_t cc = c0 + threadIdx.x;
      const uint32_t v = cc < G ? __ldcg(w.cnt + (size_t)cc * 256 + d) : 0u;
      uint32_t tot;
      const uint32_t ex = block_excl_scan<uint32_t>(v, tot, S.red);
      if (cc < G) __stcg(w.pre + (size_t)cc * 256 + d, carry + ex);
      carry += tot;
    }
    if (threadIdx.x == 0) __stcg(w.total + d, carry);
  }
  phase_mark(w.pt, 2);
  grid_barrier_r(w.bar);
  phase_mark(w.pt, 3);
  // ---- phase 3: running offsets, then rank + scatter the chunk sub-tile by sub-tile
  {
    uint32_t gtot;
    const uint32_t gs = block_excl_scan<uint32_t>(threadIdx.x < 256 ? __ldcg(w.total + threadIdx.x) : 0u, gtot, S.red);
    if (threadIdx.x < 256) S.gstart[threadIdx.x] = gs + __ldcg(w.pre + (size_t)c * 256 + threadIdx.x);  // running
  }
  for (int i = threadIdx.x; i < 2 * kRadixWarps * 256; i += blockDim.x) (&S.wmask[0][0][0])[i] = 0;
  const uint32_t lt = (1u << lane) - 1u;
  // keys of the first sub-tile; each iteration prefetches the next sub-tile's keys
  uint32_t k[kRadixKPT], kn[kRadixKPT], rank[kRadixKPT];
  {
    const uint32_t wb = lo + warp * 32 * kRadixKPT;
#pragma unroll
    for (int i = 0; i < kRadixKPT; ++i) {
      const uint32_t idx = wb + i * 32 + lane;
      k[i] = idx < hi ? (__ldcs(src + idx) ^ flip_in) : 0u;
    }
  }
  for (uint32_t tbase = lo; tbase < hi; tbase += kRadixTile) {
    for (int i = threadIdx.x; i < kRadixWarps * 256; i += blockDim.x) (&S.wcnt[0][0])[i] = 0;
    __syncthreads();
    const uint32_t tile_n = min((uint32_t)kRadixTile, hi - tbase);
    const uint32_t wbase = tbase + warp * 32 * kRadixKPT;
    {  // prefetch the next sub-tile (consumed next iteration)
      const uint32_t wn = wbase + kRadixTile;
#pragma unroll
      for (int i = 0; i < kRadixKPT; ++i) {
        const uint32_t idx = wn + i * 32 + lane;
        kn[i] = idx < hi ? (__ldcs(src + idx) ^ flip_in) : 0u;
      }
    }
    if (wbase + 32 * kRadixKPT <= hi) {
      // full warp (MATCH.ANY costs ~70 cycles per warp on sm_100a and the 8-ballot multisplit
      // ~40 instructions per item, both measured; this costs ~16)
      // Equality grouping through shared memory: each lane ORs its bit into the warp's mask
      // word of its digit; after a warp sync the word is the group (the CRN's equality merge,
      // with no order comparison).  Two mask buffers alternate so the leader's reset of
      // buffer i&1 is ordered before its next use (item i+2) by item i+1's sync.
#pragma unroll
      for (int i = 0; i < kRadixKPT; ++i) {
        const uint32_t d = __byte_perm(k[i], 0, dsel);
        uint32_t* wm = &S.wmask[i & 1][warp][d];
        atomicOr(wm, 1u << lane);
        __syncwarp();
        const uint32_t g = *wm;
        const uint32_t leader = __ffs(g) - 1;
        uint32_t old = 0;
        if (lane == leader) {
          old = S.wcnt[warp][d];
          S.wcnt[warp][d] = old + __popc(g);
          *wm = 0u;
        }
        rank[i] = __shfl_sync(FULL, old, leader) + __popc(g & lt);
      }
    } else {
#pragma unroll
      for (int i = 0; i < kRadixKPT; ++i) {
        const uint32_t idx0 = wbase + i * 32;
        const uint32_t vmask = idx0 >= hi ? 0u : (hi - idx0 >= 32 ? FULL : ((1u << (hi - idx0)) - 1u));
        if ((vmask >> lane) & 1u) {
          const uint32_t d = __byte_perm(k[i], 0, dsel);
          const uint32_t g = digit_group(d, vmask);
          const uint32_t leader = __ffs(g) - 1;
          uint32_t old = 0;
          if (lane == leader) {
            old = S.wcnt[warp][d];
            S.wcnt[warp][d] = old + __popc(g);
          }
          rank[i] = __shfl_sync(vmask, old, leader) + __popc(g & lt);
        }
      }
    }
    __syncthreads();
    uint32_t cnt = 0;
    if (threadIdx.x < 256) {
      const int d = threadIdx.x;
#pragma unroll
      for (int ww = 0; ww < kRadixWarps; ++ww) {
        const uint32_t cw = S.wcnt[ww][d];
        S.wcnt[ww][d] = cnt;
        cnt += cw;
      }
    }
    uint32_t tile_total;
    const uint32_t ex = block_excl_scan<uint32_t>(threadIdx.x < 256 ? cnt : 0u, tile_total, S.red);
    if (threadIdx.x < 256) {
      const uint32_t d = threadIdx.x;
      S.tile_excl[d] = ex;
      S.base[d] = S.gstart[d] - ex;
      S.gstart[d] += cnt;  // running offset for the next sub-tile
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < kRadixKPT; ++i) {
      const uint32_t idx = wbase + i * 32 + lane;
      if (idx < hi) {
        const uint32_t d = __byte_perm(k[i], 0, dsel);
        S.keys[S.tile_excl[d] + S.wcnt[warp][d] + rank[i]] = k[i];
      }
    }
    __syncthreads();
    for (uint32_t j = threadIdx.x; j < tile_n; j += blockDim.x) {
      const uint32_t u = S.keys[j];
      __stcs(dst + S.base[__byte_perm(u, 0, dsel)] + j, u ^ flip_out);
    }
#pragma unroll
    for (int i = 0; i < kRadixKPT; ++i) k[i] = kn[i];
    __syncthreads();  // S.keys / S.wcnt reused by the next sub-tile
  }
  phase_mark(w.pt, 4);
  pdl_trigger();
}

// ---- K8'' reduce-then-scan pass with 8192-key sub-tiles (default) ---------------------------
// Phases 1-2 as k_radix_pass2 (chunk digit counts, column scans, two grid barriers).  Phase 3
// scatters the chunk in 8192-key sub-tiles, the next sub-tile's keys in flight (registers)
// while the current one is placed:
//   a. per-(warp, digit) counts of the sub-tile (warp w owns sub-tile keys [512w, 512w+512),
//      16 steps of 32 consecutive keys), one block scan over (digit, warp) gives every warp its
//      first slot per digit and the sub-tile's digit starts;
//   b. stable in-warp ranks, step by step: the lanes of a step are grouped by equal digit
//      through a shared lane-mask word (atomicOr, the CRN's equality merge), the group's
//      leader advances the warp's digit cursor; the key goes to its slot of the digit-sorted
//      sub-tile;
//   c. the sorted sub-tile leaves as digit runs at the CTA's running global offsets.
// 12n bytes per pass (the chunk is read twice: counts, then scatter).
constexpr int kR3KPT = 16;
constexpr int kR3Tile = kRadixThreads * kR3KPT;  // 8192 keys
struct Radix3Smem {
  uint32_t wcur[kRadixWarps][256];      // per-warp digit counts -> cursors (16 KB)
  uint32_t wmask[2][kRadixWarps][256];  // equality-grouping lane masks, 2 buffers (32 KB)
  uint32_t sorted[kR3Tile];             // sub-tile sorted by digit (32 KB)
  uint32_t dstart[257];                 // digit starts in the sorted sub-tile
  uint32_t grun[256];                   // running global position of digit d for this chunk
  uint32_t hnext[256];
  uint32_t red[34];
};

__global__ void __launch_bounds__(kRadixThreads, 2) k_radix_pass3(const uint32_t* __restrict__ src,
                                                                   uint32_t* __restrict__ dst, uint32_t n, int p,
                                                                   Radix2Ws w) {
  extern __shared__ __align__(16) unsigned char radix_smem_raw[];
  Radix3Smem& S = *reinterpret_cast<Radix3Smem*>(radix_smem_raw);
  pdl_wait();
  phase_mark(w.pt, -1);
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5, G = gridDim.x, c = blockIdx.x;
  const uint32_t dsel = 0x4440u | (uint32_t)p;
  const uint32_t flip_in = p == 0 ? kSignFlip : 0u, flip_out = p == 3 ? kSignFlip : 0u;
  const uint32_t lo = (uint32_t)((uint64_t)n * c / G), hi = (uint32_t)((uint64_t)n * (c + 1) / G);
  for (int i = threadIdx.x; i < 2 * kRadixWarps * 256; i += blockDim.x) (&S.wmask[0][0][0])[i] = 0;
  // ---- phase 1: digit counts of the chunk
  if (threadIdx.x < 256) S.hnext[threadIdx.x] = 0;
  __syncthreads();
  {
    const uint64_t pol = l2_evict_first_policy();
    const uint32_t mis = (uint32_t)((reinterpret_cast<uintptr_t>(src) >> 2) & 3u);
    const uint32_t a4 = min(hi, lo + ((4u - ((lo + mis) & 3u)) & 3u));
    const uint32_t b4 = a4 + ((hi - a4) & ~3u);
    for (uint32_t i = lo + threadIdx.x; i < min(a4, hi); i += blockDim.x)
      atomicAdd(&S.hnext[__byte_perm(__ldcs(src + i) ^ flip_in, 0, dsel)], 1u);
    if (a4 < b4) {
      const int4* body = reinterpret_cast<const int4*>(src + a4);
      const uint32_t nv = (b4 - a4) / 4;
      uint32_t v = threadIdx.x;
      for (; v + 3 * blockDim.x < nv; v += 4 * blockDim.x) {
        int4 x[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) x[u] = ld_stream4(body + v + u * blockDim.x, pol);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          atomicAdd(&S.hnext[__byte_perm((uint32_t)x[u].x ^ flip_in, 0, dsel)], 1u);
          atomicAdd(&S.hnext[__byte_perm((uint32_t)x[u].y ^ flip_in, 0, dsel)], 1u);
          atomicAdd(&S.hnext[__byte_perm((uint32_t)x[u].z ^ flip_in, 0, dsel)], 1u);
          atomicAdd(&S.hnext[__byte_perm((uint32_t)x[u].w ^ flip_in, 0, dsel)], 1u);
        }
      }
      for (; v < nv; v += blockDim.x) {
        const int4 x = ld_stream4(body + v, pol);
        atomicAdd(&S.hnext[__byte_perm((uint32_t)x.x ^ flip_in, 0, dsel)], 1u);
        atomicAdd(&S.hnext[__byte_perm((uint32_t)x.y ^ flip_in, 0, dsel)], 1u);
        atomicAdd(&S.hnext[__byte_perm((uint32_t)x.z ^ flip_in, 0, dsel)], 1u);
        atomicAdd(&S.hnext[__byte_perm((uint32_t)x.w ^ flip_in, 0, dsel)], 1u);
      }
    }
    for (uint32_t i = b4 + threadIdx.x; i < hi; i += blockDim.x)
      atomicAdd(&S.hnext[__byte_perm(__ldcs(src + i) ^ flip_in, 0, dsel)], 1u);
  }
  __syncthreads();
  if (threadIdx.x < 256) __stcg(w.cnt + (size_t)c * 256 + threadIdx.x, S.hnext[threadIdx.x]);
  phase_mark(w.pt, 0);
  grid_barrier_r(w.bar);
  phase_mark(w.pt, 1);
  // ---- phase 2: column scans (CTA d scans digit d over the G chunks)
  for (uint32_t d = c; d < 256; d += G) {
    uint32_t carry = 0;
    for (uint32_t c0 = 0; c0 < G; c0 += blockDim.x) {
      const uint32_t cc = c0 + threadIdx.x;
      const uint32_t v = cc < G ? __ldcg(w.cnt + (size_t)cc * 256 + d) : 0u;
      uint32_t tot;
      const uint32_t ex = block_excl_scan<uint32_t>(v, tot, S.red);
      if (cc < G) __stcg(w.pre + (size_t)cc * 256 + d, carry + ex);
      carry += tot;
    }
    if (threadIdx.x == 0) __stcg(w.total + d, carry);
  }
  phase_mark(w.pt, 2);
  grid_barrier_r(w.bar);
  phase_mark(w.pt, 3);
  // ---- phase 3
  {
    uint32_t gtot;
    const uint32_t gs = block_excl_scan<uint32_t>(threadIdx.x < 256 ? __ldcg(w.total + threadIdx.x) : 0u, gtot, S.red);
    if (threadIdx.x < 256) S.grun[threadIdx.x] = gs + __ldcg(w.pre + (size_t)c * 256 + threadIdx.x);
  }
  const uint32_t lt = (1u << lane) - 1u;
  uint32_t k[kR3KPT], kn[kR3KPT];
  auto load = [&](uint32_t t0, uint32_t (&kk)[kR3KPT]) {
#pragma unroll
    for (int i = 0; i < kR3KPT; ++i) {
      const uint32_t idx = t0 + warp * 32 * kR3KPT + i * 32 + lane;
      kk[i] = idx < hi ? (__ldcs(src + idx) ^ flip_in) : 0u;
    }
  };
  load(lo, k);
  for (uint32_t t0 = lo; t0 < hi; t0 += kR3Tile) {
    const uint32_t tn = min((uint32_t)kR3Tile, hi - t0);
    if (t0 + kR3Tile < hi) load(t0 + kR3Tile, kn);
    for (int i = threadIdx.x; i < kRadixWarps * 256; i += blockDim.x) (&S.wcur[0][0])[i] = 0;
    __syncthreads();
    const uint32_t wseg = warp * 32 * kR3KPT;  // warp's first key in the sub-tile
#pragma unroll
    for (int i = 0; i < kR3KPT; ++i)
      if (wseg + i * 32 + lane < tn) atomicAdd(&S.wcur[warp][__byte_perm(k[i], 0, dsel)], 1u);
    __syncthreads();
    {  // exclusive scan over (digit, warp): thread t has digit t >> 1, warps (t & 1) * 8 .. + 7
      const uint32_t d = threadIdx.x >> 1, w0 = (threadIdx.x & 1u) * (kRadixWarps / 2);
      uint32_t v[kRadixWarps / 2], s = 0;
#pragma unroll
      for (int j = 0; j < kRadixWarps / 2; ++j) {
        v[j] = S.wcur[w0 + j][d];
        s += v[j];
      }
      uint32_t tot;
      uint32_t ex = block_excl_scan<uint32_t>(s, tot, S.red);
      if ((threadIdx.x & 1u) == 0) S.dstart[d] = ex;
      if (threadIdx.x == 0) S.dstart[256] = tot;
#pragma unroll
      for (int j = 0; j < kRadixWarps / 2; ++j) {
        S.wcur[w0 + j][d] = ex;
        ex += v[j];
      }
    }
    __syncthreads();
    if (wseg + 32 * kR3KPT <= tn) {
#pragma unroll
      for (int i = 0; i < kR3KPT; ++i) {
        const uint32_t d = __byte_perm(k[i], 0, dsel);
        uint32_t* wm = &S.wmask[i & 1][warp][d];
        atomicOr(wm, 1u << lane);
        __syncwarp();
        const uint32_t g = *wm;
        const uint32_t pos = S.wcur[warp][d] + __popc(g & lt);
        __syncwarp();
        if (lane == (uint32_t)(__ffs(g) - 1)) {
          S.wcur[warp][d] = pos + __popc(g);  // the leader has no lower lane in its group
          *wm = 0u;
        }
        S.sorted[pos] = k[i];
      }
    } else {
#pragma unroll
      for (int i = 0; i < kR3KPT; ++i) {
        const uint32_t idx0 = wseg + i * 32;
        const uint32_t vmask = idx0 >= tn ? 0u : (tn - idx0 >= 32 ? FULL : ((1u << (tn - idx0)) - 1u));
        if ((vmask >> lane) & 1u) {
          const uint32_t d = __byte_perm(k[i], 0, dsel);
          const uint32_t g = digit_group(d, vmask);
          const uint32_t pos = S.wcur[warp][d] + __popc(g & lt);
          __syncwarp(vmask);
          if (lane == (uint32_t)(__ffs(g) - 1)) S.wcur[warp][d] = pos + __popc(g);
          S.sorted[pos] = k[i];
        }
      }
    }
    __syncthreads();
    for (uint32_t j = threadIdx.x; j < tn; j += blockDim.x) {
      const uint32_t u = S.sorted[j];
      const uint32_t d = __byte_perm(u, 0, dsel);
      __stcs(dst + S.grun[d] + (j - S.dstart[d]), u ^ flip_out);
    }
    __syncthreads();
    if (threadIdx.x < 256) S.grun[threadIdx.x] += S.dstart[threadIdx.x + 1] - S.dstart[threadIdx.x];
#pragma unroll
    for (int i = 0; i < kR3KPT; ++i) k[i] = kn[i];
  }
  phase_mark(w.pt, 4);
  pdl_trigger();
}

// ---- K8 variant with TMA-staged sub-tiles (default for 16-byte aligned src) ----------------
// As k_radix_pass3, but the scatter phase streams each 8192-key sub-tile into shared memory
// with one bulk copy (cp.async.bulk, completion on an mbarrier) instead of 16 scalar loads
// per thread (ncu: those loads were the top stall, LSU queue full).  The copy of sub-tile
// k+1 is issued as soon as sub-tile k's keys are in registers (after its counting), so it
// overlaps the ranking and the write-out.  Ranking is the counting atomic itself: its
// returned value is the key's rank among its warp's keys of the digit (no lane-mask
// grouping pass).  One stage buffer, ~82 KB (2 CTAs per SM).  Requires src 16-byte aligned.
struct Radix4Smem {
  uint32_t wcur[kRadixWarps][256];   // per-warp digit counts -> slot bases (16 KB)
  uint32_t sorted[kR3Tile];          // sub-tile sorted by digit (32 KB)
  uint32_t stage[kR3Tile + 4];       // staged sub-tile (+ alignment shift) (32 KB)
  uint32_t dstart[257];
  uint32_t grun[256];
  int32_t gdel[256];                 // grun[d] - dstart[d]: output index of sorted slot j is gdel[d] + j
  uint32_t hnext[256];
  uint32_t red[34];
  uint64_t bar;
};

__global__ void __launch_bounds__(kRadixThreads, 2) k_radix_pass4(const uint32_t* __restrict__ src,
                                                                   uint32_t* __restrict__ dst, uint32_t n, int p,
                                                                   Radix2Ws w) {
  extern __shared__ __align__(16) unsigned char radix_smem_raw[];
  Radix4Smem& S = *reinterpret_cast<Radix4Smem*>(radix_smem_raw);
  pdl_wait();
  phase_mark(w.pt, -1);
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5, G = gridDim.x, c = blockIdx.x;
  const uint32_t dsel = 0x4440u | (uint32_t)p;
  const uint32_t flip_in = p == 0 ? kSignFlip : 0u, flip_out = p == 3 ? kSignFlip : 0u;
  const uint32_t lo = (uint32_t)((uint64_t)n * c / G), hi = (uint32_t)((uint64_t)n * (c + 1) / G);
  if (threadIdx.x == 0) {
    mbar_init(&S.bar, 1);
    mbar_fence_init();
  }
  // ---- phase 1: digit counts of the chunk (16-byte vectors; src is aligned)
  if (threadIdx.x < 256) S.hnext[threadIdx.x] = 0;
  __syncthreads();
  {
    const uint64_t pol = l2_evict_first_policy();
    const uint32_t a4 = min(hi, (lo + 3u) & ~3u), b4 = max(a4, hi & ~3u);
    for (uint32_t i = lo + threadIdx.x; i < a4; i += blockDim.x)
      atomicAdd(&S.hnext[__byte_perm(__ldcs(src + i) ^ flip_in, 0, dsel)], 1u);
    const int4* body = reinterpret_cast<const int4*>(src + a4);
    const uint32_t nv = (b4 - a4) / 4;
    uint32_t v = threadIdx.x;
    for (; v + 3 * blockDim.x < nv; v += 4 * blockDim.x) {
      int4 x[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) x[u] = ld_stream4(body + v + u * blockDim.x, pol);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        atomicAdd(&S.hnext[__byte_perm((uint32_t)x[u].x ^ flip_in, 0, dsel)], 1u);
        atomicAdd(&S.hnext[__byte_perm((uint32_t)x[u].y ^ flip_in, 0, dsel)], 1u);
        atomicAdd(&S.hnext[__byte_perm((uint32_t)x[u].z ^ flip_in, 0, dsel)], 1u);
        atomicAdd(&S.hnext[__byte_perm((uint32_t)x[u].w ^ flip_in, 0, dsel)], 1u);
      }
    }
    for (; v < nv; v += blockDim.x) {
      const int4 x = ld_stream4(body + v, pol);
      atomicAdd(&S.hnext[__byte_perm((uint32_t)x.x ^ flip_in, 0, dsel)], 1u);
      atomicAdd(&S.hnext[__byte_perm((uint32_t)x.y ^ flip_in, 0, dsel)], 1u);
      atomicAdd(&S.hnext[__byte_perm((uint32_t)x.z ^ flip_in, 0, dsel)], 1u);
      atomicAdd(&S.hnext[__byte_perm((uint32_t)x.w ^ flip_in, 0, dsel)], 1u);
    }
    for (uint32_t i = b4 + threadIdx.x; i < hi; i += blockDim.x)
      atomicAdd(&S.hnext[__byte_perm(__ldcs(src + i) ^ flip_in, 0, dsel)], 1u);
  }
  __syncthreads();
  if (threadIdx.x < 256) __stcg(w.cnt + (size_t)c * 256 + threadIdx.x, S.hnext[threadIdx.x]);
  phase_mark(w.pt, 0);
  grid_barrier_r(w.bar);
  phase_mark(w.pt, 1);
  // ---- phase 2: column scans (CTA d scans digit d over the G chunks)
  for (uint32_t d = c; d < 256; d += G) {
    uint32_t carry = 0;
    for (uint32_t c0 = 0; c0 < G; c0 += blockDim.x) {
      const uint32_t cc = c0 + threadIdx.x;
      const uint32_t v = cc < G ? __ldcg(w.cnt + (size_t)cc * 256 + d) : 0u;
      uint32_t tot;
      const uint32_t ex = block_excl_scan<uint32_t>(v, tot, S.red);
      if (cc < G) __stcg(w.pre + (size_t)cc * 256 + d, carry + ex);
      carry += tot;
    }
    if (threadIdx.x == 0) __stcg(w.total + d, carry);
  }
  phase_mark(w.pt, 2);
  grid_barrier_r(w.bar);
  phase_mark(w.pt, 3);
  // ---- phase 3
  {
    uint32_t gtot;
    const uint32_t gs = block_excl_scan<uint32_t>(threadIdx.x < 256 ? __ldcg(w.total + threadIdx.x) : 0u, gtot, S.red);
    if (threadIdx.x < 256) S.grun[threadIdx.x] = gs + __ldcg(w.pre + (size_t)c * 256 + threadIdx.x);
  }
  const uint64_t pol = l2_evict_first_policy();
  // sub-tile [t0, t0 + tn): key t0 + j sits at stage[sft + j], sft = t0 & 3, so that the
  // 16-byte aligned body [ab, ae) arrives by one bulk copy at the 16-byte aligned
  // stage + (ab - (t0 & ~3)); the at most 3 keys before ab and after ae are loaded by threads
  auto bounds = [&](uint32_t t0, uint32_t& tn, uint32_t& ab, uint32_t& ae) {
    tn = min((uint32_t)kR3Tile, hi - t0);
    ab = min(t0 + tn, (t0 + 3u) & ~3u);
    ae = max(ab, (t0 + tn) & ~3u);
  };
  auto issue = [&](uint32_t t0) {
    uint32_t tn, ab, ae;
    bounds(t0, tn, ab, ae);
    if (threadIdx.x == 0) {
      const uint32_t bytes = 4u * (ae - ab);
      mbar_arrive_expect_tx(&S.bar, bytes);
      if (bytes) tma_load_1d(S.stage + (ab - (t0 & ~3u)), src + ab, bytes, &S.bar, pol);
    }
  };
  uint32_t phase = 0;
  __syncthreads();
  if (lo < hi) issue(lo);
  for (uint32_t t0 = lo; t0 < hi; t0 += kR3Tile) {
    uint32_t tn, ab, ae;
    bounds(t0, tn, ab, ae);
    for (int i = threadIdx.x; i < kRadixWarps * 256; i += blockDim.x) (&S.wcur[0][0])[i] = 0;
    const uint32_t sft = t0 & 3u;
    if (threadIdx.x < ab - t0) S.stage[sft + threadIdx.x] = __ldcs(src + t0 + threadIdx.x);
    if (threadIdx.x >= 8 && threadIdx.x - 8 < t0 + tn - ae)
      S.stage[sft + (ae - t0) + threadIdx.x - 8] = __ldcs(src + ae + threadIdx.x - 8);
    mbar_wait_sleep(&S.bar, phase);
    phase ^= 1u;
    __syncthreads();  // staged keys (bulk + edges) visible; wcur cleared
    const uint32_t wseg = warp * 32 * kR3KPT;
    // the returned counter value is the key's rank among its warp's keys of that digit
    // (< 32 kR3KPT), two ranks per register; slot = the warp's digit base + rank
    uint32_t k[kR3KPT], rk[kR3KPT / 2];
    if (wseg + 32 * kR3KPT <= tn) {
      const uint32_t* sk = S.stage + sft + wseg + lane;
#pragma unroll
      for (int i = 0; i < kR3KPT; ++i) {
        k[i] = sk[i * 32] ^ flip_in;
        const uint32_t r = atomicAdd(&S.wcur[warp][__byte_perm(k[i], 0, dsel)], 1u);
        if (i & 1) rk[i >> 1] |= r << 16;
        else rk[i >> 1] = r;
      }
    } else {
#pragma unroll
      for (int i = 0; i < kR3KPT; ++i) {
        const uint32_t j = wseg + i * 32 + lane;
        k[i] = j < tn ? (S.stage[sft + j] ^ flip_in) : 0u;
        const uint32_t r = j < tn ? atomicAdd(&S.wcur[warp][__byte_perm(k[i], 0, dsel)], 1u) : 0u;
        if (i & 1) rk[i >> 1] |= r << 16;
        else rk[i >> 1] = r;
      }
    }
    __syncthreads();  // counts complete; the stage buffer is free
    if (t0 + kR3Tile < hi) issue(t0 + kR3Tile);
    {  // exclusive scan over (digit, warp): thread t has digit t >> 1, warps (t & 1) * 8 .. + 7
      const uint32_t d = threadIdx.x >> 1, w0 = (threadIdx.x & 1u) * (kRadixWarps / 2);
      uint32_t v[kRadixWarps / 2], s = 0;
#pragma unroll
      for (int j = 0; j < kRadixWarps / 2; ++j) {
        v[j] = S.wcur[w0 + j][d];
        s += v[j];
      }
      uint32_t tot;
      uint32_t ex = block_excl_scan<uint32_t>(s, tot, S.red);
      if ((threadIdx.x & 1u) == 0) S.dstart[d] = ex;
      if (threadIdx.x == 0) S.dstart[256] = tot;
#pragma unroll
      for (int j = 0; j < kRadixWarps / 2; ++j) {
        S.wcur[w0 + j][d] = ex;
        ex += v[j];
      }
    }
    __syncthreads();
    if (threadIdx.x < 256) S.gdel[threadIdx.x] = (int32_t)(S.grun[threadIdx.x] - S.dstart[threadIdx.x]);
    if (wseg + 32 * kR3KPT <= tn) {
#pragma unroll
      for (int i = 0; i < kR3KPT; ++i)
        S.sorted[S.wcur[warp][__byte_perm(k[i], 0, dsel)] + ((rk[i >> 1] >> (16 * (i & 1))) & 0xffffu)] = k[i];
    } else {
#pragma unroll
      for (int i = 0; i < kR3KPT; ++i)
        if (wseg + i * 32 + lane < tn)
          S.sorted[S.wcur[warp][__byte_perm(k[i], 0, dsel)] + ((rk[i >> 1] >> (16 * (i & 1))) & 0xffffu)] = k[i];
    }
    __syncthreads();
    if (tn == (uint32_t)kR3Tile) {  // full sub-tile: unrolled, 32-bit output index (n < 2^32)
#pragma unroll
      for (int r = 0; r < kR3KPT; ++r) {
        const uint32_t j = r * kRadixThreads + threadIdx.x, u = S.sorted[j];
        __stcs(dst + (uint32_t)(S.gdel[__byte_perm(u, 0, dsel)] + (int32_t)j), u ^ flip_out);
      }
    } else {
      for (uint32_t j = threadIdx.x; j < tn; j += blockDim.x) {
        const uint32_t u = S.sorted[j];
        __stcs(dst + (int64_t)S.gdel[__byte_perm(u, 0, dsel)] + j, u ^ flip_out);
      }
    }
    __syncthreads();
    if (threadIdx.x < 256) S.grun[threadIdx.x] += S.dstart[threadIdx.x + 1] - S.dstart[threadIdx.x];
  }
  phase_mark(w.pt, 4);
  pdl_trigger();
}

inline void radix_configure() {
  cudaFuncSetAttribute(k_radix_pass, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(RadixSmem));
  cudaFuncSetAttribute(k_radix_pass2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(RadixSmem));
  cudaFuncSetAttribute(k_radix_pass3, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(Radix3Smem));
  cudaFuncSetAttribute(k_radix_pass4, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(Radix4Smem));
}

}  // namespace ds

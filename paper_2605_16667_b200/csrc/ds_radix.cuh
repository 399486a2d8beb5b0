// ds_radix.cuh — DialSort-Radix (tab:radix P:1659-1679): full signed int32,
// "LSD, base 256, 4 passes, zero order comparisons".
//
// Pass p is a 256-bin DialSort of the digit d = (u >> 8p) & 0xFF of the sign-flipped key
// u = x ^ 0x80000000 (reading R2): ingestion of the digit histogram (eq:ingestion with U=256),
// the per-digit write offsets (the per-digit prefix sum radix needs, tab:related "Per digit"),
// and a stable scatter.  GPU form: one co-resident reduce-then-scan grid per pass (chunk digit
// counts | grid barrier | column scans | grid barrier | stable scatter of 8192-key sub-tiles).
//   k_radix_pass4  default (16-byte aligned buffers): sub-tiles staged by TMA bulk copies,
//                  in-warp ranks from the value the counting shared atomic returns; stable
//                  because the shared-memory unit serves the same-address lanes of one ATOMS
//                  in lane order — a property the context VERIFIES on its device when it is
//                  created (k_radix_lane_probe below); a device that fails it gets pass3.
//   k_radix_pass3  ranks by explicit equality grouping (a lane-mask word per digit, the CRN's
//                  equality merge applied to digits): stable by construction, any alignment.
// HBM traffic: 12n bytes per pass (the chunk is read twice: counts, then scatter).
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
constexpr uint32_t kSignFlip = 0x80000000u;

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

// Workspace of one pass (CTA c owns the contiguous chunk [c n / G, (c+1) n / G)).
struct Radix2Ws {
  uint32_t* cnt;       // [G][256] chunk digit counts
  uint32_t* pre;       // [G][256] exclusive column scans
  uint32_t* total;     // [256] digit totals
  GridBarR* bar;
  PhaseTimes* pt;      // nullable debug timing
  const uint32_t* d_n; // nullable: the key count is on the device (multi-GPU receive buffer);
                       // n is then only the grid-sizing bound
};

// ---- reduce-then-scan pass with 8192-key sub-tiles, lane-mask ranks (stable by construction) --
// Phase 1 counts the chunk's digits (the pass's DialSort ingestion) into cnt[c][256]; after a
// grid barrier CTA d (< 256) scans column d over the chunks into pre[.][d] and total[d]; after
// a second barrier every CTA knows its digit offsets (scan of total + its row pre[c]).  Phase 3
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
  if (w.d_n) {  // (one load per CTA)
    __shared__ uint32_t s_n;
    if (threadIdx.x == 0) s_n = *w.d_n;
    __syncthreads();
    n = s_n;
  }
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

// ---- the default pass: TMA-staged sub-tiles, ranks from the counting atomic ------------------
// As k_radix_pass3, but the scatter phase streams each 8192-key sub-tile into shared memory
// with one bulk copy (cp.async.bulk, completion on an mbarrier) instead of 16 scalar loads
// per thread (ncu: those loads were the top stall, LSU queue full).  The copy of sub-tile
// k+1 is issued as soon as sub-tile k's keys are in registers (after its counting), so it
// overlaps the ranking and the write-out.  Ranking is the counting atomic itself: its
// returned value is the key's rank among its warp's keys of the digit (no lane-mask
// grouping pass).  One stage buffer, ~98 KB (2 CTAs per SM).  Requires src 16-byte aligned.
// 10240-key sub-tiles with 16-bit per-warp counters (2 CTAs per SM): measured c5 1.335 ms vs
// 1.418 ms for 8192-key sub-tiles with 32-bit counters; 4096 / 6144-key sub-tiles at 3-4 CTAs
// per SM were slower (1.53 - 1.88 ms): per-sub-tile fixed costs, not occupancy, bound the pass.
#ifndef DIALSORT_R4_KPT
#define DIALSORT_R4_KPT 20
#endif
#ifndef DIALSORT_R4_MINB
#define DIALSORT_R4_MINB 2
#endif
#ifndef DIALSORT_R4_W16
#define DIALSORT_R4_W16 1
#endif

#ifndef DIALSORT_R4_THREADS
#define DIALSORT_R4_THREADS 512
#endif
constexpr int kR4KPT = DIALSORT_R4_KPT;
constexpr int kR4Threads = DIALSORT_R4_THREADS;  // 512, 768 or 1024
constexpr int kR4Warps = kR4Threads / 32;
constexpr int kR4TPD = kR4Threads / 256;         // threads per digit in the sub-tile scan
constexpr int kR4WPT = kR4Warps / kR4TPD;        // warps per scan thread (8)
static_assert(kR4Threads % 256 == 0 && kR4Warps % kR4TPD == 0, "pass4 thread count");
constexpr int kR4Tile = kR4Threads * kR4KPT;
constexpr bool kR4W16 = DIALSORT_R4_W16 != 0;  // per-warp digit counters as 16-bit halves
struct Radix4Smem {
  uint32_t wcur[kR4Warps][kR4W16 ? 128 : 256];  // per-warp digit counts -> slot bases
  uint32_t sorted[kR4Tile];          // sub-tile sorted by digit
  uint32_t stage[kR4Tile + 4];       // staged sub-tile (+ alignment shift)
  uint32_t dstart[257];
  uint32_t grun[256];
  int32_t gdel[256];                 // grun[d] - dstart[d]: output index of sorted slot j is gdel[d] + j
  uint32_t hnext[256];
  uint32_t red[34];
  uint64_t bar;
};

// counter of digit d of warp w: a 32-bit word, or one 16-bit half of word d / 2
__device__ __forceinline__ uint32_t r4_count(Radix4Smem& S, uint32_t w, uint32_t d) {
  if (kR4W16) {
    const uint32_t old = atomicAdd(&S.wcur[w][d >> 1], 1u << (16 * (d & 1u)));
    return (old >> (16 * (d & 1u))) & 0xffffu;
  }
  return atomicAdd(&S.wcur[w][d], 1u);
}
__device__ __forceinline__ uint32_t r4_get(const Radix4Smem& S, uint32_t w, uint32_t d) {
  if (kR4W16) return reinterpret_cast<const uint16_t*>(&S.wcur[w][0])[d];
  return S.wcur[w][d];
}
__device__ __forceinline__ void r4_set(Radix4Smem& S, uint32_t w, uint32_t d, uint32_t v) {
  if (kR4W16) reinterpret_cast<uint16_t*>(&S.wcur[w][0])[d] = (uint16_t)v;
  else S.wcur[w][d] = v;
}
__global__ void __launch_bounds__(kR4Threads, DIALSORT_R4_MINB) k_radix_pass4(const uint32_t* __restrict__ src,
                                                                   uint32_t* __restrict__ dst, uint32_t n, int p,
                                                                   Radix2Ws w) {
  extern __shared__ __align__(16) unsigned char radix_smem_raw[];
  Radix4Smem& S = *reinterpret_cast<Radix4Smem*>(radix_smem_raw);
  pdl_wait();
  if (w.d_n) {  // (one load per CTA)
    __shared__ uint32_t s_n;
    if (threadIdx.x == 0) s_n = *w.d_n;
    __syncthreads();
    n = s_n;
  }
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
    // (counting the chunk back to front with L2-normal loads, so that its front is still in L2
    //  when the scatter starts, measured no faster: 1.3346 vs 1.3337 ms — the scatter is bound
    //  by shared memory, not by the second read)
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
    tn = min((uint32_t)kR4Tile, hi - t0);
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
  for (uint32_t t0 = lo; t0 < hi; t0 += kR4Tile) {
    uint32_t tn, ab, ae;
    bounds(t0, tn, ab, ae);
    for (int i = threadIdx.x; i < kR4Warps * (kR4W16 ? 128 : 256); i += blockDim.x) (&S.wcur[0][0])[i] = 0;
    const uint32_t sft = t0 & 3u;
    if (threadIdx.x < ab - t0) S.stage[sft + threadIdx.x] = __ldcs(src + t0 + threadIdx.x);
    if (threadIdx.x >= 8 && threadIdx.x - 8 < t0 + tn - ae)
      S.stage[sft + (ae - t0) + threadIdx.x - 8] = __ldcs(src + ae + threadIdx.x - 8);
    mbar_wait_sleep(&S.bar, phase);
    phase ^= 1u;
    __syncthreads();  // staged keys (bulk + edges) visible; wcur cleared
    const uint32_t wseg = warp * 32 * kR4KPT;
    // the returned counter value is the key's rank among its warp's keys of that digit
    // (< 32 kR4KPT), two ranks per register; slot = the warp's digit base + rank
    uint32_t k[kR4KPT], rk[kR4KPT / 2];
    if (wseg + 32 * kR4KPT <= tn) {
      const uint32_t* sk = S.stage + sft + wseg + lane;
#pragma unroll
      for (int i = 0; i < kR4KPT; ++i) {
        k[i] = sk[i * 32] ^ flip_in;
        const uint32_t r = r4_count(S, warp, __byte_perm(k[i], 0, dsel));
        if (i & 1) rk[i >> 1] |= r << 16;
        else rk[i >> 1] = r;
      }
    } else {
#pragma unroll
      for (int i = 0; i < kR4KPT; ++i) {
        const uint32_t j = wseg + i * 32 + lane;
        k[i] = j < tn ? (S.stage[sft + j] ^ flip_in) : 0u;
        const uint32_t r = j < tn ? r4_count(S, warp, __byte_perm(k[i], 0, dsel)) : 0u;
        if (i & 1) rk[i >> 1] |= r << 16;
        else rk[i >> 1] = r;
      }
    }
    __syncthreads();  // counts complete; the stage buffer is free
    if (t0 + kR4Tile < hi) issue(t0 + kR4Tile);
    {  // exclusive scan over (digit, warp): thread t has digit t / TPD, warps (t % TPD) * 8 .. + 7
      const uint32_t d = threadIdx.x / kR4TPD, w0 = (threadIdx.x % kR4TPD) * kR4WPT;
      uint32_t v[kR4WPT], s = 0;
#pragma unroll
      for (int j = 0; j < kR4WPT; ++j) {
        v[j] = r4_get(S, w0 + j, d);
        s += v[j];
      }
      uint32_t tot;
      uint32_t ex = block_excl_scan<uint32_t>(s, tot, S.red);
      if (threadIdx.x % kR4TPD == 0) S.dstart[d] = ex;
      if (threadIdx.x == 0) S.dstart[256] = tot;
#pragma unroll
      for (int j = 0; j < kR4WPT; ++j) {
        r4_set(S, w0 + j, d, ex);
        ex += v[j];
      }
    }
    __syncthreads();
    if (threadIdx.x < 256) S.gdel[threadIdx.x] = (int32_t)(S.grun[threadIdx.x] - S.dstart[threadIdx.x]);
    if (wseg + 32 * kR4KPT <= tn) {
#pragma unroll
      for (int i = 0; i < kR4KPT; ++i)
        S.sorted[r4_get(S, warp, __byte_perm(k[i], 0, dsel)) + ((rk[i >> 1] >> (16 * (i & 1))) & 0xffffu)] = k[i];
    } else {
#pragma unroll
      for (int i = 0; i < kR4KPT; ++i)
        if (wseg + i * 32 + lane < tn)
          S.sorted[r4_get(S, warp, __byte_perm(k[i], 0, dsel)) + ((rk[i >> 1] >> (16 * (i & 1))) & 0xffffu)] = k[i];
    }
    __syncthreads();
    if (tn == (uint32_t)kR4Tile) {  // full sub-tile: unrolled, 32-bit output index (n < 2^32)
#pragma unroll
      for (int r = 0; r < kR4KPT; ++r) {
        const uint32_t j = r * kR4Threads + threadIdx.x, u = S.sorted[j];
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


// ---- lane-order probe (run once per device by dialsort_ctx_create) ---------------------------
// k_radix_pass4's stability rests on one property of the shared-memory atomic unit: the lanes
// of one ATOMS instruction that hit the same counter are served in lane order, so the value
// each lane gets back is its rank in lane order.  The probe exercises exactly pass4's access
// pattern (per-warp digit counters, 16 warps, 2 CTAs per SM, 16 steps per round) over group
// structures from all-equal to all-distinct and counts every lane whose returned value differs
// from base + #(lower lanes of its group) — the group computed independently with MATCH.ANY.
// Any violation makes the context use k_radix_pass3 (stable by construction).
__device__ __forceinline__ uint32_t probe_hash(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352du;
  x ^= x >> 15;
  x *= 0x846ca68bu;
  x ^= x >> 16;
  return x;
}
__global__ void __launch_bounds__(kRadixThreads, 2) k_radix_lane_probe(uint32_t seed, uint32_t rounds,
                                                                       unsigned long long* violations) {
  __shared__ uint32_t wcur[kRadixWarps][256];
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5, lt = (1u << lane) - 1u;
  uint32_t bad = 0;
  for (uint32_t r = 0; r < rounds; ++r) {
    for (uint32_t i = threadIdx.x; i < kRadixWarps * 256; i += blockDim.x) (&wcur[0][0])[i] = 0;
    __syncthreads();
    const uint32_t classes = 1u << (r % 9);  // 1, 2, 4, ..., 256 distinct digits
    const uint32_t salt = probe_hash(seed ^ (blockIdx.x * 0x9e3779b9u) ^ (r * 0x85ebca6bu));
#pragma unroll 1
    for (uint32_t i = 0; i < 16; ++i) {
      const uint32_t h = probe_hash(salt + threadIdx.x * 16 + i);
      const uint32_t d = (h % classes) * (256u / classes) + ((r >> 4) & (256u / classes - 1u));
      const uint32_t v = atomicAdd(&wcur[warp][d], 1u);
      const uint32_t g = __match_any_sync(0xffffffffu, d);
      const uint32_t vmin = __reduce_min_sync(g, v);
      if (v - vmin != (uint32_t)__popc(g & lt)) ++bad;
    }
    __syncthreads();
  }
  if (bad) atomicAdd(violations, (unsigned long long)bad);
}

inline void radix_configure() {
  cudaFuncSetAttribute(k_radix_pass3, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(Radix3Smem));
  cudaFuncSetAttribute(k_radix_pass4, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(Radix4Smem));
}

}  // namespace ds

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
// Two schedules place the blocks' keys (U <= 2^22, up to 64 blocks):
//   sampled (default): 6 bytes per key, one pass over the keys
//     k_part_sample   a stratified sample of 65536 keys -> each block's key-region capacity
//                     (estimate + 6 sigma) and start in tmp
//     k_part_place_ring   (B <= 16) every warp alone: per-(warp, block) shared-memory rings,
//                     whole 128-key units stored into units claimed from the block's region;
//                     then k_part_ring_compact / _move / _tail make the regions dense
//     k_part_place<true>  (16 < B <= 64) 4096-key sub-tiles staged by block; each run claims
//                     its place in its block's region with one global atomic (regions fill
//                     densely; a region that would overflow sets ovf and drops the run)
//     k_part_fin      block sizes and output starts from the fills (skipped after ovf)
//   exact (after ovf — gated on it, no host round trip — or DIALSORT_OPT_PART_MODE = 1):
//     k_part_count    per-CTA chunk: block counts (per-warp shared counters)      [G][B]
//     k_part_scan     exclusive offsets off[c][b] (block-major), block sizes and starts
//     k_part_place<false>  per-CTA chunk again, runs written at the CTA's offsets
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

constexpr uint32_t kPartSample = 65536;     // keys sampled for the block-size estimate
constexpr uint32_t kFillStride = 32;        // one 128-byte line per block's fill counter
struct PartWs {
  uint32_t* cnt;   // [G][B] block counts of each CTA chunk, then offsets (in place)
  uint64_t* bsz;   // [B] block sizes
  uint64_t* boff;  // [B] block starts in the output
  DevStatus* st;
  uint64_t* koff;  // [B] block key-region starts in tmp (= boff on the exact schedule)
  uint64_t* cap;   // [B] sampled schedule: region capacities
  uint32_t* fill;  // [B * kFillStride] sampled schedule: keys placed per block so far
  uint32_t* ovf;   // sampled schedule: a region overflowed -> the exact schedule runs
};
// ---- ring placement constants (k_part_place_ring below; sampled schedule, B <= kRpMaxB) ----
#ifndef DIALSORT_RP_THREADS
#define DIALSORT_RP_THREADS 256
#endif
constexpr uint32_t kRpThreads = DIALSORT_RP_THREADS, kRpWarps = kRpThreads / 32;
#ifndef DIALSORT_RP_UNIT
#define DIALSORT_RP_UNIT 128
#endif
constexpr uint32_t kRpUnit = DIALSORT_RP_UNIT;  // keys a unit (128: 256 bytes of uint16)
constexpr uint32_t kRpRing = 2 * kRpUnit;       // ring entries per (warp, block)
constexpr uint32_t kRpCheck = kRpUnit / 32;     // key slots (32 keys each) between the flush checks
constexpr uint32_t kRpKPL = kRpUnit / 32;       // keys a lane sends of a unit (8, 4 or 2: 16, 8 or 4 bytes)
static_assert(kRpUnit == 64 || kRpUnit == 128 || kRpUnit == 256, "ring unit");
#ifndef DIALSORT_RP_NV
#define DIALSORT_RP_NV 4  // (2: 1.514 ms at c4, 3: 1.451, 4: 1.449)
#endif
constexpr uint32_t kRpNV = DIALSORT_RP_NV;      // 16-byte key vectors a lane per batch
static_assert((4 * kRpNV) % kRpCheck == 0, "a batch ends on a flush check");
static_assert(kRpUnit - 1 + 32 * kRpCheck <= kRpRing, "a ring holds what accumulates between checks");
constexpr uint32_t kRpSubs = 16;          // unit counters per block
constexpr uint32_t kRpClaim = 4;          // units per claim
#ifndef DIALSORT_RP_MAXB
#define DIALSORT_RP_MAXB 16
#endif
constexpr uint32_t kRpMaxB = DIALSORT_RP_MAXB;
constexpr uint32_t kRpMaxHoles = 131072;  // hole units per block the compaction takes (more: ovf)
#ifndef DIALSORT_RP_MINB
#define DIALSORT_RP_MINB (DIALSORT_RP_UNIT == 128 ? 3 : 6)  // (shared memory: 66 / 33 KB a CTA at B = 16)
#endif
struct RingWs {
  uint32_t* sub;    // [B][kRpSubs] units claimed per counter (kFillStride words apart)
  uint32_t* tfill;  // [B] tail-pool fills (kFillStride words apart)
  uint32_t* holes;  // [B][W] 2 x (first unit, count) of each warp's unused claimed units
  uint32_t* list;   // [B][2][kRpMaxHoles] compaction scratch (hole units below F, filled units above)
  uint32_t* meta;   // [B][4] compaction: moves, F
  uint64_t tail0;   // first slot of the tail pools in tmp; pool b starts at tail0 + b * tailcap
  uint32_t tailcap; // slots per tail pool (>= (kRpUnit - 1) W)
  uint32_t W;       // warps of the placement grid
};
__host__ __device__ constexpr size_t part_ring_smem(uint32_t B) {
  return 4ull * kRpWarps * 32 + 2ull * kRpWarps * B * kRpRing;
}
// Region slots a block needs beyond its keys (whole units): every warp's unused claimed units and
// tail remainder, and the unit counters' imbalance.
__host__ __device__ constexpr uint64_t part_ring_extra(uint32_t W) {
  return (uint64_t)kRpUnit * ((uint64_t)W * (2 * kRpClaim + 1) + 64ull * kRpSubs);
}

// Gate of the exact schedule's kernels when they back up the sampled one: run only after an
// overflow (nullptr: always run).
__device__ __forceinline__ bool part_gated_off(const uint32_t* gate) {
  return gate && *reinterpret_cast<const volatile uint32_t*>(gate) == 0u;
}

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

// (gate: see part_gated_off; a gated run does not record bad keys again — the sampled
//  scatter did)
__global__ void __launch_bounds__(kPartThreads) k_part_count(const int32_t* __restrict__ keys, uint64_t n, uint32_t U,
                                                             uint32_t B, PartWs w, const uint32_t* gate) {
  __shared__ uint32_t wcnt[kPartThreads / 32][kPartMaxBlocks];
  pdl_wait();
  if (part_gated_off(gate)) {
    pdl_trigger();
    return;
  }
  const uint32_t warp = threadIdx.x >> 5;
  for (uint32_t i = threadIdx.x; i < (kPartThreads / 32) * kPartMaxBlocks; i += blockDim.x) (&wcnt[0][0])[i] = 0;
  __syncthreads();
  uint64_t lo, hi;
  part_chunk(keys, n, lo, hi);
  uint32_t* wc = wcnt[warp];
  auto one = [&](uint32_t k, uint64_t idx) {
    if (k < U) atomicAdd(&wc[k >> kPartShift], 1u);
    else if (!gate) record_bad(w.st, idx, k);
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
__global__ void __launch_bounds__(1024) k_part_scan(uint32_t G, uint32_t B, PartWs w, const uint32_t* gate) {
  __shared__ unsigned long long red[34];
  pdl_wait();
  if (part_gated_off(gate)) {
    pdl_trigger();
    return;
  }
  unsigned long long sz = 0;
  if (threadIdx.x < B)
    for (uint32_t c = 0; c < G; ++c) sz += w.cnt[(uint64_t)c * B + threadIdx.x];
  unsigned long long tot;
  const unsigned long long start = block_excl_scan<unsigned long long>(sz, tot, red);
  if (threadIdx.x < B) {
    w.bsz[threadIdx.x] = sz;
    w.boff[threadIdx.x] = start;
    w.koff[threadIdx.x] = start;
    uint64_t run = start;
    for (uint32_t c = 0; c < G; ++c) {
      const uint64_t x = w.cnt[(uint64_t)c * B + threadIdx.x];
      w.cnt[(uint64_t)c * B + threadIdx.x] = (uint32_t)run;  // positions < n < 2^32
      run += x;
    }
  }
  pdl_trigger();
}

// Sampled schedule, step 1 (64 CTAs; the last one to finish sizes the regions): a stratified sample — one key at a hashed position in each
// of S = min(n, 65536) equal strata of the input — counts the keys of each block; capacity of
// block b = its estimate c_b n / S + 6 sqrt(c_b + 1) n / S + 256 (margins scaled down if their
// sum would pass tcap - sum of the estimates), exact when S = n.  Region starts = exclusive
// scan of the capacities; fills and the overflow flag are reset.
__device__ __forceinline__ uint32_t part_hash(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
  return x;
}
constexpr uint32_t kSampleCtas = 64, kSampleThreads = 256;  // 4 samples per thread
// ring_extra > 0 (k_part_place_ring): capacities rounded to whole units plus ring_extra slots;
// the ring's unit counters and tail fills are reset.
__global__ void __launch_bounds__(kSampleThreads) k_part_sample(const int32_t* __restrict__ keys, uint64_t n,
                                                                uint32_t U, uint32_t B, PartWs w, uint64_t tcap,
                                                                uint32_t* __restrict__ sacc, uint64_t ring_extra,
                                                                RingWs r) {
  // sacc: [kPartMaxBlocks] sample counts of the whole grid, [kPartMaxBlocks] the CTA ticket —
  // zero between launches (the last CTA resets them)
  constexpr uint32_t kPer = kPartSample / (kSampleCtas * kSampleThreads);
  __shared__ uint32_t cnt[kPartMaxBlocks];
  __shared__ unsigned long long red[34];
  __shared__ double s_scale;
  __shared__ uint32_t s_last;
  pdl_wait();
  if (threadIdx.x < kPartMaxBlocks) cnt[threadIdx.x] = 0;
  __syncthreads();
  const uint64_t S = n < kPartSample ? n : kPartSample;
  uint32_t k[kPer];
#pragma unroll
  for (uint32_t q = 0; q < kPer; ++q) {  // (loads first: all in flight together)
    const uint64_t j = (uint64_t)(q * kSampleCtas + blockIdx.x) * kSampleThreads + threadIdx.x;
    k[q] = 0xffffffffu;
    if (j < S) {
      const uint64_t lo = j * n / S, hi = (j + 1) * n / S;  // (hi > lo: S <= n)
      k[q] = (uint32_t)__ldg(keys + lo + part_hash((uint32_t)j) % (hi - lo));
    }
  }
#pragma unroll
  for (uint32_t q = 0; q < kPer; ++q)
    if (k[q] < U) atomicAdd(&cnt[k[q] >> kPartShift], 1u);
  __syncthreads();
  if (threadIdx.x < B && cnt[threadIdx.x]) atomicAdd(sacc + threadIdx.x, cnt[threadIdx.x]);
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(sacc + kPartMaxBlocks, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!s_last) {
    pdl_trigger();
    return;
  }
  __threadfence();
  uint64_t est = 0, mar = 0;
  if (threadIdx.x < B) {
    const uint64_t cb = *reinterpret_cast<volatile uint32_t*>(sacc + threadIdx.x);
    sacc[threadIdx.x] = 0;
    if (S == n) {
      est = cb;
    } else {
      const double r = (double)n / (double)S;
      est = (uint64_t)ceil((double)cb * r);
      mar = (uint64_t)ceil(6.0 * sqrt((double)cb + 1.0) * r) + 256;
    }
  }
  if (threadIdx.x == 0) sacc[kPartMaxBlocks] = 0;
  unsigned long long tot_est, tot_mar;
  block_excl_scan<unsigned long long>(est, tot_est, red);
  block_excl_scan<unsigned long long>(mar, tot_mar, red);
  if (threadIdx.x == 0)
    s_scale = tot_est + tot_mar <= tcap ? 1.0 : (tot_est < tcap ? (double)(tcap - tot_est) / (double)tot_mar : 0.0);
  __syncthreads();
  uint64_t cap = est + (uint64_t)((double)mar * s_scale);
  if (cap > n) cap = n;
  if (ring_extra) cap = ((cap + kRpUnit - 1) & ~(uint64_t)(kRpUnit - 1)) + ring_extra;
  if (threadIdx.x >= B) cap = 0;
  if (ring_extra)
    for (uint32_t i = threadIdx.x; i < B * (kRpSubs + 1); i += blockDim.x) {
      if (i < B * kRpSubs) r.sub[(uint64_t)i * kFillStride] = 0;
      else r.tfill[(uint64_t)(i - B * kRpSubs) * kFillStride] = 0;
    }
  unsigned long long tot_cap;
  const uint64_t start = block_excl_scan<unsigned long long>(cap, tot_cap, red);
  if (threadIdx.x < B) {
    w.cap[threadIdx.x] = cap;
    w.koff[threadIdx.x] = start;
    w.fill[threadIdx.x * kFillStride] = 0;
  }
  if (threadIdx.x == 0) *w.ovf = 0;
  pdl_trigger();
}

// Sampled schedule, step 3 (one CTA): block sizes = the fills, output starts = their exclusive
// scan.  After an overflow it does nothing (the exact schedule writes them).
__global__ void __launch_bounds__(1024) k_part_fin(uint32_t B, PartWs w) {
  __shared__ unsigned long long red[34];
  pdl_wait();
  if (*reinterpret_cast<const volatile uint32_t*>(w.ovf)) {
    pdl_trigger();
    return;
  }
  const uint64_t sz = threadIdx.x < B ? w.fill[threadIdx.x * kFillStride] : 0u;
  unsigned long long tot;
  const uint64_t start = block_excl_scan<unsigned long long>(sz, tot, red);
  if (threadIdx.x < B) {
    w.bsz[threadIdx.x] = sz;
    w.boff[threadIdx.x] = start;
  }
  pdl_trigger();
}

// The placement (both schedules): re-reads the CTA's chunk and writes every valid key's low 16
// bits into its universe block, sub-tile by sub-tile (4096 keys, 8 per thread as two 16-byte
// loads; the next sub-tile's loads are in flight while the current one is ranked).  One shared
// atomic per key: the returned value of the per-warp block counter is the key's rank among the
// warp's keys of that block in this sub-tile (< 256), kept in the key's register next to the
// key (key < U <= 2^22 fills 22 bits, rank bits 22..29; kBad marks a dropped bad key).  The
// scan warp turns the counters into slot bases; every key lands at base + rank in the staged
// sub-tile (order inside a block is free), which leaves as contiguous runs (~4096 / B keys per
// block).  Two stage buffers, two barriers per sub-tile:
//   count(i) | B1 | scan(i) (warp 0) | B2 | stage(i) + write-out(i-1) (+ warp 0: deltas(i))
// so the write-out of one sub-tile overlaps the staging of the next and the counting after it.
// EST (sampled schedule): the scan warp claims each run's place in its block's region (one
// global atomic per run, read back after the staging: its round trip overlaps the write-out); a
// run whose claim would pass the region's capacity sets ovf and goes to the 4096-key trash area
// past the regions.  Positions are 32-bit (mod 2^32; tmp holds < 2^32 keys, checked by the
// host).  Bad keys are recorded here.
// !EST (exact schedule): the runs go to the CTA's running block offsets (k_part_scan); gate as
// k_part_count.
// The chunk interior must be 16-byte aligned for the vector loads; other chunks take the scalar
// path (keys of an unaligned base).
#ifndef DIALSORT_PART_MINB
#define DIALSORT_PART_MINB (2048 / DIALSORT_PART_THREADS)  // 4 CTAs per SM (32 registers): more loads in flight (c4 6.44 -> 6.19 ms)
#endif
// Ranking counters per (warp, block, lane parity): the 32 lanes of a ranking atomic spread over
// 2 B words in distinct banks (B = 16), so same-address lanes — serialised by the atomic unit —
// drop from ~2 to ~1 per word (ncu, one counter per (warp, block): 5.1 wavefronts per ranking
// atomic).
#ifndef DIALSORT_PART_SUBS
#define DIALSORT_PART_SUBS 2
#endif
constexpr uint32_t kPartSubs = DIALSORT_PART_SUBS;
template <bool EST>
__global__ void __launch_bounds__(kPartThreads, DIALSORT_PART_MINB) k_part_place(const int32_t* __restrict__ keys, uint64_t n,
                                                             uint32_t U, uint32_t B, PartWs w,
                                                             uint16_t* __restrict__ tmp, const uint32_t* gate,
                                                             uint32_t trash) {
  constexpr uint32_t NW = kPartThreads / 32, S = kPartSubs;
  constexpr uint32_t kBad = 0xffffffffu;
  // (static shared memory, 45 KB: as dynamic shared memory the kernel ran 5 % slower — the
  //  driver then picks a larger shared-memory carveout, less L1)
  __shared__ uint32_t wcnt[NW][kPartMaxBlocks * S];   // per-(warp, block, sub) counts of the sub-tile
  __shared__ uint16_t wbase[NW][kPartMaxBlocks * S];  // their slot bases in the staged sub-tile (< 4096)
  __shared__ uint32_t bofs[2][kPartMaxBlocks + 1];    // run starts in the staged sub-tile, + total
  __shared__ uint32_t delta[2][kPartMaxBlocks];       // staged slot j of block b goes to delta + j
  __shared__ uint32_t gpos[kPartMaxBlocks];           // (exact) running output position of block b
  __shared__ uint32_t stage[2][kPartTile];
  pdl_wait();
  if (!EST && part_gated_off(gate)) {
    pdl_trigger();
    return;
  }
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint64_t lo, hi;
  part_chunk(keys, n, lo, hi);
  if (!EST && threadIdx.x < B) gpos[threadIdx.x] = w.cnt[(uint64_t)blockIdx.x * B + threadIdx.x];
  const bool vec = ((reinterpret_cast<uintptr_t>(keys + lo)) & 15u) == 0;
  unsigned short* const out = reinterpret_cast<unsigned short*>(tmp);
  for (uint32_t i = threadIdx.x; i < NW * kPartMaxBlocks * S; i += blockDim.x) (&wcnt[0][0])[i] = 0;
  __syncthreads();
  if (lo >= hi) {
    pdl_trigger();
    return;
  }
  const uint32_t sub = lane & (S - 1);
  uint32_t k[kPartKPT], kn[kPartKPT];
  uint32_t pos0 = 0, pos1 = 0;  // (EST, warp 0) claims of blocks lane, lane + 32
#define DS_PART_LOAD(T0, K)                                                                                 \
  {                                                                                                         \
    const uint64_t i0 = (T0) + (uint64_t)kPartKPT * threadIdx.x;                                            \
    if (vec && i0 + kPartKPT <= hi) {                                                                       \
      const int4 x0 = __ldcs(reinterpret_cast<const int4*>(keys + i0));                                     \
      const int4 x1 = __ldcs(reinterpret_cast<const int4*>(keys + i0) + 1);                                 \
      K[0] = x0.x; K[1] = x0.y; K[2] = x0.z; K[3] = x0.w; K[4] = x1.x; K[5] = x1.y; K[6] = x1.z; K[7] = x1.w; \
    } else {                                                                                                \
      _Pragma("unroll") for (uint32_t i = 0; i < kPartKPT; ++i) K[i] = i0 + i < hi ? (uint32_t)keys[i0 + i] : kBad; \
    }                                                                                                       \
  }
  // one 4096-key write-out of staged buffer q (runs at delta[q][block] + slot)
  auto write_out = [&](uint32_t q) {
    const uint32_t nvld = bofs[q][B];  // valid keys of the sub-tile (bad keys were dropped)
    if (nvld == kPartTile) {
#pragma unroll
      for (uint32_t r = 0; r < kPartKPT; ++r) {
        const uint32_t j = r * kPartThreads + threadIdx.x, key = stage[q][j];
        __stcs(out + (uint32_t)(delta[q][key >> kPartShift] + j), (unsigned short)(key & 0xffffu));
      }
    } else {
      for (uint32_t j = threadIdx.x; j < nvld; j += blockDim.x) {
        const uint32_t key = stage[q][j];
        __stcs(out + (uint32_t)(delta[q][key >> kPartShift] + j), (unsigned short)(key & 0xffffu));
      }
    }
  };
  DS_PART_LOAD(lo, k);
  uint32_t p = 0;
  for (uint64_t t0 = lo;; t0 += kPartTile, p ^= 1u) {
    const bool nxt = t0 + kPartTile < hi;
    if (nxt) DS_PART_LOAD(t0 + kPartTile, kn);  // next sub-tile in flight
    uint32_t kmax = 0;
#pragma unroll
    for (uint32_t i = 0; i < kPartKPT; ++i) kmax = max(kmax, k[i]);
    const bool allv = kmax < U;
    if (allv) {  // every key valid: no per-key test
#pragma unroll
      for (uint32_t i = 0; i < kPartKPT; ++i) k[i] |= atomicAdd(&wcnt[warp][(k[i] >> kPartShift) * S + sub], 1u) << 22;
    } else {
#pragma unroll
      for (uint32_t i = 0; i < kPartKPT; ++i) {
        if (EST && k[i] >= U && t0 + (uint64_t)kPartKPT * threadIdx.x + i < hi)  // (past the end: kBad)
          record_bad(w.st, t0 + (uint64_t)kPartKPT * threadIdx.x + i, k[i]);
        k[i] = k[i] < U ? k[i] | (atomicAdd(&wcnt[warp][(k[i] >> kPartShift) * S + sub], 1u) << 22) : kBad;
      }
    }
    __syncthreads();  // B1: counts of sub-tile i complete
    if (warp == 0) {
      // lane l owns blocks l and l + 32: block totals over the NW warps, one warp scan of the
      // totals (block order), then the per-warp slot bases of each owned block
      uint32_t t[2] = {0u, 0u};
      const uint32_t nh = B > 32 ? 2u : 1u;
      for (uint32_t h = 0; h < nh; ++h) {
        const uint32_t b = lane + 32 * h;
        if (b < B) {
#pragma unroll
          for (uint32_t q = 0; q < NW; ++q)
#pragma unroll
            for (uint32_t u = 0; u < S; ++u) t[h] += wcnt[q][b * S + u];
        }
      }
      const uint32_t i0 = warp_incl_scan(t[0]), i1 = nh > 1 ? warp_incl_scan(t[1]) : 0u;
      const uint32_t s0 = __shfl_sync(0xffffffffu, i0, 31);
      const uint32_t ex[2] = {i0 - t[0], s0 + i1 - t[1]};
      for (uint32_t h = 0; h < nh; ++h) {
        const uint32_t b = lane + 32 * h;
        if (b < B) {
          uint32_t base = ex[h];
          bofs[p][b] = base;
          if (EST) {
            if (t[h]) {
              const uint32_t c = atomicAdd(w.fill + b * kFillStride, t[h]);  // (read after the staging)
              if (h) pos1 = c; else pos0 = c;
            }
          } else {
            delta[p][b] = gpos[b] - base;
            gpos[b] += t[h];
          }
#pragma unroll
          for (uint32_t q = 0; q < NW; ++q)
#pragma unroll
            for (uint32_t u = 0; u < S; ++u) {
              const uint32_t x = wcnt[q][b * S + u];
              wbase[q][b * S + u] = (uint16_t)base;
              wcnt[q][b * S + u] = 0;
              base += x;
            }
        }
      }
      if (lane == 31) bofs[p][B] = s0 + (nh > 1 ? i1 : 0u);  // lane 31 holds both totals
    }
    __syncthreads();  // B2: slot bases of sub-tile i
    if (allv) {
#pragma unroll
      for (uint32_t i = 0; i < kPartKPT; ++i) {
        const uint32_t key = k[i] & 0x3fffffu;
        stage[p][wbase[warp][(key >> kPartShift) * S + sub] + (k[i] >> 22)] = key;
      }
    } else {
#pragma unroll
      for (uint32_t i = 0; i < kPartKPT; ++i)
        if (k[i] != kBad) {
          const uint32_t key = k[i] & 0x3fffffu;
          stage[p][wbase[warp][(key >> kPartShift) * S + sub] + (k[i] >> 22)] = key;
        }
    }
    if (t0 != lo) write_out(p ^ 1u);  // sub-tile i-1
    if (EST && warp == 0) {  // the claims of sub-tile i -> its runs' deltas
      for (uint32_t h = 0; h < 2; ++h) {
        const uint32_t b = lane + 32 * h;
        if (b < B) {
          const uint32_t ex = bofs[p][b], tb = bofs[p][b + 1] - ex, c = h ? pos1 : pos0;
          uint32_t d = trash - ex;  // (an empty run: never read)
          if (tb) {
            if ((uint64_t)c + tb <= w.cap[b]) d = (uint32_t)(w.koff[b] + c) - ex;
            else atomicOr(w.ovf, 1u);
          }
          delta[p][b] = d;
        }
      }
    }
    if (!nxt) break;
#pragma unroll
    for (uint32_t i = 0; i < kPartKPT; ++i) k[i] = kn[i];
  }
  __syncthreads();  // the last sub-tile's staging and deltas
  write_out(p);
#undef DS_PART_LOAD
  pdl_trigger();
}

// ---- ring placement (sampled schedule, B <= 16: the c4 path) --------------------------------
// The same MSD split without any CTA-wide step: order inside a universe block is free (its
// histogram is order-free, eq:ingestion P:409-412), so every warp places its own keys alone.
// A warp keeps, per block, a kRpRing-entry ring of low-16-bit keys in shared memory: a key
// takes the next ring slot from the counting atomic (one ATOMS; no rank scan, no barrier), and
// every kRpCheck key slots each ring holding a whole unit (kRpUnit keys) sends it as one
// coalesced 256-byte store.  Units are claimed from the block's region by global atomics on
// kRpSubs counters per block (unit k + kRpSubs j of counter k), kRpClaim units a claim; the
// next claim is issued when the current one's first unit is used, so its round trip is hidden.
// At the end a warp's ring remainders (< kRpUnit keys per block) go to the block's tail pool
// (exact claims) and its unused claimed units are recorded as holes; k_part_ring_compact /
// _move / _tail then make each region dense (the filled units above F fill the holes below
// it, the tail pool follows at unit F).  A claim past the region's capacity raises ovf (the
// exact schedule then redoes the placement, as for k_part_place<true>).  Bad keys are
// recorded here.
__device__ __forceinline__ uint32_t rp_atom_inc(uint32_t a) {
  uint32_t v;
  asm volatile("atom.shared.add.u32 %0, [%1], 1;" : "=r"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void rp_st16(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u16 [%0], %1;" ::"r"(a), "h"((unsigned short)v) : "memory");
}
__device__ __forceinline__ uint32_t rp_ld32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ uint2 rp_ld64(uint32_t a) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a) : "memory");
  return v;
}
__global__ void __launch_bounds__(kRpThreads, DIALSORT_RP_MINB) k_part_place_ring(const int32_t* __restrict__ keys,
                                                                                 uint64_t n, uint32_t U, uint32_t B,
                                                                                 PartWs w, RingWs r,
                                                                                 uint16_t* __restrict__ tmp) {
  extern __shared__ __align__(16) unsigned char rp_smem[];
  uint32_t* const cur_all = reinterpret_cast<uint32_t*>(rp_smem);          // [kRpWarps][32] ring fills
  uint16_t* const ring_all = reinterpret_cast<uint16_t*>(cur_all + kRpWarps * 32);  // [kRpWarps][B][kRpRing]
  pdl_wait();
  const uint32_t lane = threadIdx.x & 31, wl = threadIdx.x >> 5, gw = blockIdx.x * kRpWarps + wl;
  for (uint32_t i = threadIdx.x; i < kRpWarps * 32; i += blockDim.x) cur_all[i] = 0;
  __syncthreads();
  const uint32_t cur_s = smem_addr(cur_all) + 128u * wl;               // this warp's fills
  const uint32_t ring_s = smem_addr(ring_all) + 2u * kRpRing * B * wl;  // this warp's rings
  const uint32_t my_cur = cur_s + 4u * lane;  // (lanes >= B: a fill that stays 0)
  const bool own = lane < B;                  // lane b keeps the state of block b's ring
  // (a lane sends kRpKPL keys of a unit: element e of tmp as uint2 / uint32 holds keys kRpKPL e ..)
  const uint32_t koffe = own ? (uint32_t)(w.koff[lane] / kRpKPL) : 0u, capu = own ? (uint32_t)(w.cap[lane] / kRpUnit) : 0u;
  uint32_t* const my_sub = r.sub + (uint64_t)(own ? lane : 0u) * kRpSubs * kFillStride;
  uint32_t fl = 0;  // keys of the ring already sent (a multiple of kRpUnit)
  // claims (unit k + kRpSubs j, j = jc .. jc + kRpClaim - 1 on counter k): the current one (kc,
  // jc, cu used) and the next one (kn, jn); dst: element index of the next unit (~0u: past capacity)
  uint32_t kc = (gw + lane) % kRpSubs, jc = 0, cu = 0, kn = 0, jn = 0, dst = ~0u;
  bool started = false, has_next = false;
  auto set_dst = [&]() {
    const uint32_t unit = kc + kRpSubs * (jc + cu);
    dst = unit < capu ? koffe + 32u * unit : ~0u;
  };
  auto first_claim = [&]() {
    jc = atomicAdd(my_sub + kc * kFillStride, kRpClaim);
    started = true;
    set_dst();
  };
  auto advance = [&]() {  // (owner lane, after its unit left)
    // (the switch reads jn before a new claim overwrites it: an instruction reading the
    //  register of an atomic in flight waits for it, even predicated off)
    fl += kRpUnit;
    if (++cu == kRpClaim) {
      kc = kn;
      jc = jn;
      cu = 0;
      has_next = false;
    } else if (cu == 1) {
      kn = (kc + 1) & (kRpSubs - 1);
      jn = atomicAdd(my_sub + kn * kFillStride, kRpClaim);
      has_next = true;
    }
    set_dst();
  };
  auto flush = [&](uint32_t bb) {  // (whole warp) ring bb's next unit -> tmp
    if (lane == bb && !started) first_claim();
    const uint32_t d = __shfl_sync(FULL, dst, bb), f = __shfl_sync(FULL, fl, bb);
    const uint32_t ra = ring_s + 2u * kRpRing * bb + 2u * ((f + kRpKPL * lane) & (kRpRing - 1));
    if (d != ~0u) {
      if constexpr (kRpKPL == 8) {
        uint4 v;
        asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(ra) : "memory");
        __stcs(reinterpret_cast<uint4*>(tmp) + d + lane, v);
      } else if constexpr (kRpKPL == 4) {
        __stcs(reinterpret_cast<uint2*>(tmp) + d + lane, rp_ld64(ra));
      } else {
        __stcs(reinterpret_cast<unsigned int*>(tmp) + d + lane, rp_ld32(ra));
      }
    } else if (lane == 0) {
      atomicOr(w.ovf, 1u);
    }
    if (lane == bb) advance();
  };
  auto check = [&]() {  // (whole warp) send every whole unit; first claims of rings holding keys
    __syncwarp();
    const uint32_t c = rp_ld32(my_cur) - fl;
    if (own && !started && c) first_claim();
    uint32_t need = __ballot_sync(FULL, c >= kRpUnit);
    if (need) {
      do {
        flush(__ffs(need) - 1);
        need &= need - 1;
      } while (need);
      __syncwarp();  // the flushes' ring reads before the next slots' writes
    }
  };
  auto slot = [&](uint32_t key) {
    const uint32_t b = key >> kPartShift;
    const uint32_t sl = rp_atom_inc(cur_s + 4u * b);
    rp_st16(ring_s + 2u * kRpRing * b + 2u * (sl & (kRpRing - 1)), key);
  };
  auto slot_checked = [&](uint32_t key, uint64_t idx, bool present) {
    if (present) {
      if (key < U) slot(key);
      else record_bad(w.st, idx, key);
    }
  };
  const KeySpan s = make_span(keys, n);
  const int4* __restrict__ body = s.body();
  const uint64_t v0 = s.n4 * gw / r.W, v1 = s.n4 * (gw + 1) / r.W;
  if (gw == 0) slot_checked(lane < s.head ? (uint32_t)keys[lane] : 0u, lane, lane < s.head);
  if (gw == r.W - 1) {
    const uint64_t i = s.head + 4 * s.n4 + lane;
    slot_checked(lane < s.tail ? (uint32_t)keys[i] : 0u, i, lane < s.tail);
  }
  check();
  const uint64_t pol = l2_evict_first_policy();
  // batches of kRpNV vectors a lane (32 kRpNV vectors a warp); the next batch is in flight while
  // one is placed
  constexpr uint32_t NV = kRpNV, BV = 32 * NV;
  int4 a[NV];
#pragma unroll
  for (uint32_t q = 0; q < NV; ++q) {
    a[q] = make_int4(0, 0, 0, 0);
    if (v0 + 32 * q + lane < v1) a[q] = ld_stream4(body + v0 + 32 * q + lane, pol);
  }
  for (uint64_t vb = v0; vb < v1; vb += BV) {
    int4 nx[NV];
#pragma unroll
    for (uint32_t q = 0; q < NV; ++q) {
      nx[q] = make_int4(0, 0, 0, 0);
      if (vb + BV + 32 * q + lane < v1) nx[q] = ld_stream4(body + vb + BV + 32 * q + lane, pol);
    }
    bool ok = vb + BV <= v1;
#pragma unroll
    for (uint32_t q = 0; q < NV; ++q) ok = ok && umax4(a[q]) < U;
    if (__all_sync(FULL, ok)) {
#pragma unroll
      for (uint32_t q = 0; q < 4 * NV; ++q) {
        const int4& x = a[q / 4];
        slot((uint32_t)(q % 4 == 0 ? x.x : q % 4 == 1 ? x.y : q % 4 == 2 ? x.z : x.w));
        if ((q + 1) % kRpCheck == 0) check();
      }
    } else {
#pragma unroll
      for (uint32_t q = 0; q < 4 * NV; ++q) {
        const int4& x = a[q / 4];
        const uint64_t v = vb + 32 * (q / 4) + lane;
        slot_checked((uint32_t)(q % 4 == 0 ? x.x : q % 4 == 1 ? x.y : q % 4 == 2 ? x.z : x.w), s.head + 4 * v + q % 4,
                     v < v1);
        if ((q + 1) % kRpCheck == 0) check();
      }
    }
#pragma unroll
    for (uint32_t q = 0; q < NV; ++q) a[q] = nx[q];
  }
  // ring remainders -> the blocks' tail pools; unused claimed units -> holes
  __syncwarp();
  const uint32_t rem = rp_ld32(my_cur) - fl;  // (< kRpUnit; 0 on lanes >= B)
  uint32_t t0 = 0;
  if (rem) t0 = atomicAdd(r.tfill + (uint64_t)lane * kFillStride, rem);
  uint32_t need = __ballot_sync(FULL, rem != 0);
  while (need) {
    const uint32_t bb = __ffs(need) - 1;
    need &= need - 1;
    const uint32_t rr = __shfl_sync(FULL, rem, bb), tt = __shfl_sync(FULL, t0, bb), f = __shfl_sync(FULL, fl, bb);
    if (tt + rr > r.tailcap) {
      if (lane == 0) atomicOr(w.ovf, 1u);
      continue;
    }
    for (uint32_t i = lane; i < rr; i += 32)
      tmp[r.tail0 + (uint64_t)bb * r.tailcap + tt + i] = ring_all[(wl * B + bb) * kRpRing + ((f + i) & (kRpRing - 1))];
  }
  if (own) {
    uint4 h = make_uint4(0u, 0u, 0u, 0u);
    if (started) h.x = kc + kRpSubs * (jc + cu), h.y = kRpClaim - cu;
    if (has_next) h.z = kn + kRpSubs * jn, h.w = kRpClaim;
    reinterpret_cast<uint4*>(r.holes)[(uint64_t)lane * r.W + gw] = h;
  }
  pdl_trigger();
}

// One CTA per block: the move lists of block b.  Units are claimed densely per counter, so the
// units of [0, Utot = kRpSubs max_k f_k) all hold kRpUnit keys except the holes: the warps'
// unused claimed units and, per counter k, the units k + kRpSubs j of f_k <= j < max f.  With
// Hc holes, F = Utot - Hc units hold keys: the filled units of [F, Utot) (list sl) move into
// the holes below F (list dl) — order inside a block is free — then the tail pool is
// appended at unit F (k_part_ring_move, k_part_ring_tail: many CTAs per block).
__global__ void __launch_bounds__(1024) k_part_ring_compact(uint32_t B, PartWs w, RingWs r) {
  __shared__ uint32_t bits[kRpMaxHoles / 32];
  __shared__ uint32_t s_f[kRpSubs];
  __shared__ uint32_t red[34];
  __shared__ uint32_t s_nd, s_ns;
  pdl_wait();
  if (*reinterpret_cast<const volatile uint32_t*>(w.ovf)) {
    pdl_trigger();
    return;
  }
  const uint32_t b = blockIdx.x, T = blockDim.x;
  if (threadIdx.x < kRpSubs) s_f[threadIdx.x] = r.sub[((uint64_t)b * kRpSubs + threadIdx.x) * kFillStride];
  if (threadIdx.x == 0) s_nd = s_ns = 0;
  __syncthreads();
  uint32_t fmax = 0;
#pragma unroll
  for (uint32_t k = 0; k < kRpSubs; ++k) fmax = max(fmax, s_f[k]);
  const uint2* hl = reinterpret_cast<const uint2*>(r.holes) + 2ull * b * r.W;  // 2 per warp
  uint32_t h = threadIdx.x < kRpSubs ? fmax - s_f[threadIdx.x] : 0u;
  for (uint32_t g = threadIdx.x; g < 2 * r.W; g += T) h += hl[g].y;
  uint32_t Hc;
  block_excl_scan<uint32_t>(h, Hc, red);
  const uint32_t Utot = kRpSubs * fmax, F = Utot - Hc;
  if (Hc > kRpMaxHoles) {
    if (threadIdx.x == 0) atomicOr(w.ovf, 1u);
    pdl_trigger();
    return;
  }
  for (uint32_t i = threadIdx.x; i < (Hc + 31) / 32; i += T) bits[i] = 0;
  __syncthreads();
  uint32_t* const dl = r.list + (uint64_t)b * 2 * kRpMaxHoles;  // hole units below F
  uint32_t* const sl = dl + kRpMaxHoles;                         // filled units of [F, Utot)
  auto hole = [&](uint32_t u) {
    if (u >= F) atomicOr(&bits[(u - F) >> 5], 1u << ((u - F) & 31));
    else dl[atomicAdd(&s_nd, 1u)] = u;
  };
  for (uint32_t g = threadIdx.x; g < 2 * r.W; g += T) {
    const uint2 e = hl[g];
    for (uint32_t i = 0; i < e.y; ++i) hole(e.x + kRpSubs * i);
  }
  if (threadIdx.x < kRpSubs)
    for (uint32_t j = s_f[threadIdx.x]; j < fmax; ++j) hole(threadIdx.x + kRpSubs * j);
  __syncthreads();
  for (uint32_t p = threadIdx.x; p < Hc; p += T)
    if (!((bits[p >> 5] >> (p & 31)) & 1u)) sl[atomicAdd(&s_ns, 1u)] = F + p;
  __syncthreads();
  if (threadIdx.x == 0) {
    r.meta[4 * b] = s_nd;  // (== s_ns)
    r.meta[4 * b + 1] = F;
  }
  pdl_trigger();
}
constexpr uint32_t kRpMoveCtas = 16;  // CTAs per block of the moves (grid B x kRpMoveCtas)
__global__ void __launch_bounds__(512) k_part_ring_move(uint32_t B, PartWs w, RingWs r, uint16_t* __restrict__ tmp) {
  pdl_wait();
  if (*reinterpret_cast<const volatile uint32_t*>(w.ovf)) {
    pdl_trigger();
    return;
  }
  const uint32_t b = blockIdx.x / kRpMoveCtas, part = blockIdx.x % kRpMoveCtas;
  const uint32_t nd = r.meta[4 * b];
  const uint32_t* const dl = r.list + (uint64_t)b * 2 * kRpMaxHoles;
  const uint32_t* const sl = dl + kRpMaxHoles;
  constexpr uint32_t V = kRpUnit / 8;  // 16-byte vectors a unit
  uint4* const reg4 = reinterpret_cast<uint4*>(tmp + w.koff[b]);
  for (uint32_t q = part * blockDim.x + threadIdx.x; q < V * nd; q += kRpMoveCtas * blockDim.x)
    reg4[V * dl[q / V] + (q % V)] = reg4[V * sl[q / V] + (q % V)];
  pdl_trigger();
}
// (after the moves: the tail lands on units >= F, which the moves read)
__global__ void __launch_bounds__(512) k_part_ring_tail(uint32_t B, PartWs w, RingWs r, uint16_t* __restrict__ tmp) {
  pdl_wait();
  if (*reinterpret_cast<const volatile uint32_t*>(w.ovf)) {
    pdl_trigger();
    return;
  }
  const uint32_t b = blockIdx.x / kRpMoveCtas, part = blockIdx.x % kRpMoveCtas;
  const uint32_t F = r.meta[4 * b + 1];
  const uint32_t tl = r.tfill[(uint64_t)b * kFillStride];
  if ((uint64_t)kRpUnit * F + tl > w.cap[b]) {
    if (part == 0 && threadIdx.x == 0) atomicOr(w.ovf, 1u);
    pdl_trigger();
    return;
  }
  const uint16_t* pool = tmp + r.tail0 + (uint64_t)b * r.tailcap;
  uint16_t* const dst = tmp + w.koff[b] + (uint64_t)kRpUnit * F;
  for (uint32_t i = part * blockDim.x + threadIdx.x; i < tl; i += kRpMoveCtas * blockDim.x) dst[i] = pool[i];
  if (part == 0 && threadIdx.x == 0) w.fill[(uint64_t)b * kFillStride] = kRpUnit * F + tl;
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

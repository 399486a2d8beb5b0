// ds_fused.cuh — the whole DialSort step (histogram ingestion with the CRN, sub-histogram
// merge, write-offset scan and ordered projection) as ONE persistent, co-resident kernel for
// the shared-memory paths (U <= kSmem16MaxBins).
//
//   ingestion   eq:ingestion P:409-412 (+ CRN def:crn_level P:896-915)   hist_ingest_flush
//   merge       lem:crn P:951-962 lifted to whole histograms              merge_scan_tiles
//   scan        GPU write-offset step (R18; paper P:13-14 has none)       merge_scan_tiles
//   projection  eq:projection P:418-424                                   expand_chunk
//
// Why one kernel: on B200 a kernel boundary plus its ramp costs ~1-2 us and
// the counter+generation grid barrier ~2 us, against a ~10 us HBM floor per 40 MB pass.  Here:
//   1. every CTA ingests into its private shared-memory histogram, flushes it as partial row
//      c and adds (RED) its per-tile sums into tile_red[tile];
//   2. ONE monotonic grid barrier; every CTA then reads the <= 192 tile totals and scans them
//      locally, so it knows the first output position toff[t] of every 512-bin scan tile;
//   3. CTA c merges its own scan tiles (H, P) and publishes each (ready[t] = epoch);
//   4. without another grid-wide barrier, each half of the CTA (512 threads, named barrier)
//      projects an equal share of the output positions in 8192-position chunks, waiting only
//      on the ready flags of the scan tiles its chunk overlaps.
// A packed-counter overflow anywhere (exact detection, ds_hist.cuh) switches all CTAs to a
// path with a second barrier (tile totals recomputed from the merged H).
#pragma once
#include "ds_common.cuh"
#include "ds_expand.cuh"
#include "ds_hist.cuh"
#include "ds_scan.cuh"

namespace ds {

constexpr uint32_t kMaxScanTiles = kSmem16MaxBins / kTileBins;  // 192
constexpr uint32_t kFusedChunk = kExpandTile;                     // 8192 positions per half-CTA chunk
constexpr uint32_t kFusedSub = 256;                               // threads per projection sub-group
constexpr uint32_t kFusedNSub = 1024 / kFusedSub;                 // independent sub-groups per CTA
constexpr uint32_t kFusedQPT = kFusedChunk / 4 / kFusedSub;       // quads (4 positions) per thread
constexpr uint32_t kFusedStageOff = 4 * kTileBins;                // merge staging after 4 group rows (8 KB)
constexpr uint32_t kFusedPBatch = 4;
constexpr uint32_t kFusedPCap = 4096;                             // staged P entries per sub-group (16 KB)                              // P loads in flight per thread
constexpr uint32_t kFusedTileSlots = 256;                         // >= kMaxScanTiles
// Tile totals are REDs from every CTA into ntiles counters: 64-word (256 B) stride puts each
// counter in its own L2 line (same-line REDs serialise: 4 lines took 7.7 us for 19K REDs).
constexpr uint32_t kTileTotStride = 64;
static_assert(kFusedQPT * 4 * kFusedSub == kFusedChunk, "chunk = whole quads per thread");

// Named barrier of projection sub-group g (ids 1..kFusedNSub; 0 is __syncthreads).
__device__ __forceinline__ void sub_sync(uint32_t g) {
  asm volatile("bar.sync %0, %1;" ::"r"(g + 1), "n"(kFusedSub) : "memory");
}

// Exclusive scan over the kFusedSub threads of sub-group g; every warp scans the warp totals
// itself (one named-barrier pair).  red: >= kFusedSub/32 slots owned by the sub-group.
__device__ __forceinline__ uint64_t sub_excl_scan(uint64_t v, uint64_t& total, uint64_t* red, uint32_t g) {
  constexpr uint32_t NW = kFusedSub / 32;
  const uint32_t lane = threadIdx.x & 31, wh = (threadIdx.x % kFusedSub) >> 5;
  const uint64_t inc = warp_incl_scan(v);
  sub_sync(g);  // previous users of red are done
  if (lane == 31) red[wh] = inc;
  sub_sync(g);
  const uint64_t w = lane < NW ? red[lane] : 0ull;
  const uint64_t wi = warp_incl_scan(w);
  total = __shfl_sync(FULL, wi, NW - 1);
  const uint64_t wex = __shfl_sync(FULL, wi - w, wh);
  return wex + inc - v;
}

__device__ __forceinline__ uint32_t ld_relaxed_flag(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// Last t in [0, ntiles) with toff[t] <= x (toff[0] = 0 <= x < toff[ntiles] = total).
__device__ __forceinline__ uint32_t tile_of(const uint32_t* toff, uint32_t ntiles, uint32_t x) {
  uint32_t lo = 0, hi = ntiles;  // toff[lo] <= x < toff[hi]
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (toff[mid] <= x) lo = mid;
    else hi = mid;
  }
  return lo;
}

// Projection of output positions [p0, p1) (p1 - p0 <= kFusedChunk) by one sub-group, whose
// scan tiles are already published (the caller waited on their ready flags).
// key(p) = max{k : P[k] <= p} (the bin whose run covers p; empty bins have P[k] = P[k+1] and
// are skipped by the max).  With k0 = first bin of the scan tile ta holding p0 (P[k0] <= p0):
//   key(p) = k0 + #{k > k0 : P[k] <= p0} + #{k > k0 : p0 < P[k] <= p},
// the first count from a sub-group sum, the second from an inclusive scan of "bin start"
// marks placed at P[k] - p0 in shared memory.  Only bins of scan tiles ta..tb (tb holds p1-1)
// can contribute: later tiles start at >= toff[tb+1] > p1 - 1.
// `ta` is the caller's running tile of p0: chunks of a share ascend, so it only moves forward
// (O(ntiles) steps over a whole share, instead of a binary search per chunk and thread).
__device__ __forceinline__ void expand_chunk(const ScanArgs& a, const uint32_t* toff, uint32_t ntiles, uint32_t p0,
                                             uint32_t p1, uint32_t& ta, int32_t key_base, int32_t* __restrict__ out,
                                             uint32_t* M, uint64_t* red, uint32_t g, bool aligned, uint64_t pol) {
  const uint32_t tid = threadIdx.x % kFusedSub;
  while (toff[ta + 1] <= p0) ++ta;  // toff[ntiles] = total > p0 stops it
  uint32_t tb = ta;
  while (toff[tb + 1] <= p1 - 1) ++tb;
  uint4* M4 = reinterpret_cast<uint4*>(M);
#pragma unroll
  for (uint32_t j = 0; j < kFusedQPT; ++j) M4[tid + j * kFusedSub] = make_uint4(0, 0, 0, 0);
  sub_sync(g);
  const uint32_t k0 = ta * kTileBins;
  const uint32_t kend = min((tb + 1) * kTileBins, a.U);
  // all P loads of a thread are issued before any is used (a shared atomic between them
  // would otherwise serialise one L2 round trip per bin batch)
  uint32_t before = 0;
  for (uint32_t kb = k0 + 1 + tid; kb < kend; kb += kFusedPBatch * kFusedSub) {
    uint32_t b[kFusedPBatch];
#pragma unroll
    for (uint32_t u = 0; u < kFusedPBatch; ++u) {
      const uint32_t k = kb + u * kFusedSub;
      b[u] = k < kend ? __ldcg(a.P + k) : 0xffffffffu;
    }
#pragma unroll
    for (uint32_t u = 0; u < kFusedPBatch; ++u) {
      if (b[u] <= p0) {
        ++before;
      } else if (b[u] < p1) {
        const uint32_t w = b[u] - p0;
        atomicAdd(&M[(swz(w >> 2) << 2) | (w & 3u)], 1u);
      }
    }
  }
  sub_sync(g);
  // inclusive scan of the marks (thread owns positions 4 QPT tid ..); the sub-group scan
  // carries (before << 32 | marks) so one pass yields both counts
  uint4 v[kFusedQPT];
#pragma unroll
  for (uint32_t j = 0; j < kFusedQPT; ++j) {
    v[j] = M4[swz(kFusedQPT * tid + j)];
    v[j].y += v[j].x;
    v[j].z += v[j].y;
    v[j].w += v[j].z;
  }
#pragma unroll
  for (uint32_t j = 1; j < kFusedQPT; ++j) {
    v[j].x += v[j - 1].w; v[j].y += v[j - 1].w; v[j].z += v[j - 1].w; v[j].w += v[j - 1].w;
  }
  uint64_t tot;
  const uint64_t ex = sub_excl_scan(((uint64_t)before << 32) | v[kFusedQPT - 1].w, tot, red, g);
  const uint32_t base = (uint32_t)key_base + k0 + (uint32_t)(tot >> 32) + (uint32_t)ex;
#pragma unroll
  for (uint32_t j = 0; j < kFusedQPT; ++j)
    M4[swz(kFusedQPT * tid + j)] = make_uint4(base + v[j].x, base + v[j].y, base + v[j].z, base + v[j].w);
  sub_sync(g);
  // copy out: lane-contiguous quads, 512 contiguous bytes per warp instruction
  if (aligned && p1 - p0 == kFusedChunk) {  // full chunk: no bounds tests
#pragma unroll
    for (uint32_t j = 0; j < kFusedQPT; ++j) {
      const uint32_t qd = tid + j * kFusedSub;
      const uint4 x = M4[swz(qd)];
      st_stream4(reinterpret_cast<int4*>(out + p0 + 4 * qd), make_int4((int)x.x, (int)x.y, (int)x.z, (int)x.w), pol);
    }
    sub_sync(g);
    return;
  }
#pragma unroll
  for (uint32_t j = 0; j < kFusedQPT; ++j) {
    const uint32_t qd = tid + j * kFusedSub;
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
  sub_sync(g);  // M is reused by the next chunk
}

// Projection of one sub-group's share [lo, hi) by independent warps (no sub-group barrier
// after the staging of P).  Bins ka .. kb-1 are the bins of the scan tiles overlapping the
// share; Ps[i] = P[ka + i] is staged in shared memory.  P[ka] = toff[ta] <= lo, so for every
// position p of the share
//   key(p) = max{k : P[k] <= p} = ka - 1 + cnt(p),   cnt(p) = #{i : Ps[i] <= p}.
// The share is cut into 128-position blocks dealt round-robin to the sub-group's 8 warps, so
// that the sub-group writes one contiguous front (measured: 5.8 us for 40 MB of stores vs
// 8.8 us when each warp streams its own contiguous range — DRAM page locality).  Lane l owns
// positions blk + 4l .. +3 and the block leaves as one coalesced 512-byte warp store.
// A warp keeps c = #{i : Ps[i] < blk} and a register window sreg = Ps[cb + lane] (cb <= c),
// so the bin starts of a block are window lanes c-cb .. c-cb+nb-1, found with one ballot:
//   nb == 0      every position of the block has key ka - 1 + c;
//   nb < 32-o    each lane compares its 4 positions with the nb starts (shuffled in);
//   otherwise    the starts add marks in the warp's 128-entry count array and a warp scan of
//                the per-lane mark totals gives cnt (more than 32 starts: repeated).
// FAST: Ps holds all m entries plus >= 32 sentinels (0xffffffff), the output is 16-byte
// aligned and only whole blocks are projected — the loop is issue-bound (ncu: 73% issue
// active), so the common case is kept to a few instructions; the general form (FAST = false)
// reads entries past kFusedPCap from L2 and handles the tail block and unaligned output.
template <bool FAST>
__device__ __forceinline__ void expand_share_warp(const ScanArgs& a, uint32_t ka, uint32_t kb, uint32_t lo, uint32_t hi,
                                                  uint32_t blk, const uint32_t* Ps, uint32_t* wc, int32_t key_base,
                                                  int32_t* __restrict__ out, bool aligned, uint64_t pol) {
  constexpr uint32_t NW = kFusedSub / 32;
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t m = kb - ka;
  auto pv = [&](uint32_t i) -> uint32_t {
    if (FAST) return Ps[i];
    return i < m ? (i < kFusedPCap ? Ps[i] : __ldcg(a.P + ka + i)) : 0xffffffffu;
  };
  if (FAST ? blk + 128 > hi : blk >= hi) return;
  // c = #{i : Ps[i] < blk}
  uint32_t c0 = 0, c1 = m;
  while (c0 < c1) {
    const uint32_t mid = (c0 + c1) >> 1;
    if (pv(mid) < blk) c0 = mid + 1;
    else c1 = mid;
  }
  uint32_t c = c0, cb = c0;
  uint32_t sreg = pv(cb + lane);
  const uint32_t kbase = (uint32_t)key_base + ka - 1;
  for (;;) {
    const uint32_t p = blk + 4 * lane;
    const uint32_t bend = FAST ? blk + 127 : (hi - blk > 128 ? blk + 127 : hi - 1);
    if (c - cb >= 16) {  // keep >= 16 lanes of look-ahead in the window
      cb = c;
      sreg = pv(cb + lane);
    }
    const uint32_t o = c - cb;
    const uint32_t le = __popc(__ballot_sync(FULL, sreg <= bend));
    const uint32_t base = kbase + c;
    uint4 q = make_uint4(base, base, base, base);
    if (le != o) {  // the block holds bin starts
      // starts o..le-1 of the window; when they lie in distinct quads (the common case: bins
      // longer than 4), one OR-reduction gives the quad occupancy mask M, lane l adds the
      // starts of quads < l (popc) plus its own quad's start if its offset is <= the position
      const bool mine = lane >= o && lane < le;
      const uint32_t rel = sreg - blk;
      const uint32_t M = __reduce_or_sync(FULL, mine ? 1u << (rel >> 2) : 0u);
      if (le < 32 && (uint32_t)__popc(M) == le - o) {
        const uint32_t below = __popc(M & ((1u << lane) - 1u));
        const uint32_t r = (__shfl_sync(FULL, sreg, min(o + below, 31u)) - blk) & 3u;
        const uint32_t own = (M >> lane) & 1u;
        q.x += below + (own & (r == 0));
        q.y += below + (own & (r <= 1));
        q.z += below + (own & (r <= 2));
        q.w += below + own;
      } else if (le < 32) {
        for (uint32_t j = o; j < le; ++j) {
          const uint32_t sj = __shfl_sync(FULL, sreg, j);
          q.x += sj <= p;
          q.y += sj <= p + 1;
          q.z += sj <= p + 2;
          q.w += sj <= p + 3;
        }
      } else {
        // marks: starts Ps[c ..] <= bend, 32 at a time
        uint32_t i0 = c;
        for (;;) {
          const uint32_t sl = pv(i0 + lane);
          const uint32_t cnt = __popc(__ballot_sync(FULL, sl <= bend));
          if (lane < cnt) atomicAdd(&wc[sl - blk], 1u);
          if (cnt < 32) break;
          i0 += 32;
        }
        __syncwarp();
        uint4 mk = reinterpret_cast<uint4*>(wc)[lane];
        reinterpret_cast<uint4*>(wc)[lane] = make_uint4(0, 0, 0, 0);
        mk.y += mk.x;
        mk.z += mk.y;
        mk.w += mk.z;
        const uint32_t ex = warp_incl_scan(mk.w) - mk.w;
        q.x += ex + mk.x; q.y += ex + mk.y; q.z += ex + mk.z; q.w += ex + mk.w;
        __syncwarp();
      }
    }
    const int4 v = make_int4((int)q.x, (int)q.y, (int)q.z, (int)q.w);
    if (FAST) {
      st_stream4(reinterpret_cast<int4*>(out + p), v, pol);
      if (hi - blk < 128 * NW + 128) break;  // no further whole block for this warp
    } else {
      if (p < hi) {
        if (aligned && p + 4 <= hi) {
          st_stream4(reinterpret_cast<int4*>(out + p), v, pol);
        } else {
          out[p] = v.x;
          if (p + 1 < hi) out[p + 1] = v.y;
          if (p + 2 < hi) out[p + 2] = v.z;
          if (p + 3 < hi) out[p + 3] = v.w;
        }
      }
      if (hi - blk <= 128 * NW) break;
    }
    // advance: c = #{i : Ps[i] < next block}
    blk += 128 * NW;
    const uint32_t lt = __popc(__ballot_sync(FULL, sreg < blk));
    if (lt < 32) {
      c = cb + lt;
    } else {
      c = cb + 32;
      for (;;) {
        const uint32_t adv = __popc(__ballot_sync(FULL, pv(c + lane) < blk));
        c += adv;
        if (adv < 32) break;
      }
      cb = c;
      sreg = pv(cb + lane);
    }
  }
}

// Stage P for a share and project it: whole blocks by the FAST loop when the staged window
// holds every entry (+ sentinels) and the output is aligned; the rest by the general loop.
__device__ __forceinline__ void expand_share(const ScanArgs& a, uint32_t ka, uint32_t kb, uint32_t lo, uint32_t hi,
                                             uint32_t* Ps, uint32_t* wc, uint32_t g, int32_t key_base,
                                             int32_t* __restrict__ out, bool aligned, uint64_t pol) {
  const uint32_t m = kb - ka, tid = threadIdx.x % kFusedSub;
  const bool fast = aligned && m + 32 <= kFusedPCap;
  const uint32_t ncp = min(m + 32, kFusedPCap);
  for (uint32_t i = tid; i < ncp; i += kFusedSub) Ps[i] = i < m ? __ldcg(a.P + ka + i) : 0xffffffffu;
  reinterpret_cast<uint4*>(wc)[threadIdx.x & 31] = make_uint4(0, 0, 0, 0);
  sub_sync(g);
  const uint32_t w = tid >> 5;
  if (fast) {
    // whole blocks: [lo, lo + 128 * nblk); the partial tail block (if any) by warp nblk % 8
    const uint32_t nblk = (hi - lo) / 128;
    expand_share_warp<true>(a, ka, kb, lo, hi, lo + 128 * w, Ps, wc, key_base, out, aligned, pol);
    const uint32_t tail = lo + 128 * nblk;
    if (tail < hi && w == nblk % (kFusedSub / 32))
      expand_share_warp<false>(a, ka, kb, tail, hi, tail, Ps, wc, key_base, out, aligned, pol);
  } else {
    expand_share_warp<false>(a, ka, kb, lo, hi, lo + 128 * w, Ps, wc, key_base, out, aligned, pol);
  }
}

// Block-wide scan of the tile totals into toff[0..ntiles] (ntiles <= 192 < blockDim).
// v = this thread's tile total (thread t holds tile t), loaded by the caller.
__device__ __forceinline__ void tile_offsets(uint64_t v, uint32_t ntiles, uint32_t* toff, uint64_t* red) {
  uint64_t total;
  const uint64_t ex = block_excl_scan<uint64_t>(v, total, red);
  if (threadIdx.x < ntiles) toff[threadIdx.x] = (uint32_t)ex;
  if (threadIdx.x == 0) toff[ntiles] = (uint32_t)(total > 0xffffffffull ? 0xffffffffull : total);
  __syncthreads();
}

// One DialSort step: keys[n] in [0,U) -> out[min(ΣH, cap)] sorted, H and P as by-products.
// Grid: C <= #SMs CTAs of 1024 threads (co-resident, 1 per SM).  Dynamic smem:
// max(histogram, 128 KB) (histogram, then merge scratch, then kFusedNSub 32 KB mark buffers).
template <bool PACK16>
__global__ void __launch_bounds__(1024, 1) k_sort_fused(const int32_t* __restrict__ keys, uint64_t n, ScanArgs a,
                                                       int32_t* __restrict__ out, int32_t key_base) {
  extern __shared__ __align__(128) uint32_t sh_hist[];
  __shared__ uint64_t red64[34];
  __shared__ uint64_t sred[kFusedNSub][kFusedSub / 32];
  __shared__ uint32_t toff[kMaxScanTiles + 1];
  pdl_wait();
  phase_mark(a.pt, -1);
  const uint32_t ntiles = (a.U + kTileBins - 1) / kTileBins;
  const uint32_t G = gridDim.x;
  // the other parity's tile totals are zeroed for the next launch (host alternates them;
  // every slot, since the next launch may have more tiles than this one)
  if (blockIdx.x == G - 1)
    for (uint32_t i = threadIdx.x; i < kFusedTileSlots; i += blockDim.x) a.tile_clear[i * kTileTotStride] = 0;

  hist_ingest_flush<PACK16, false>(keys, n, a, 0, sh_hist, red64, nullptr, nullptr);
  grid_barrier_mono(a.bar64, a.bar_base + G);  // rows, tile totals, overflow fallback in L2
  phase_mark(a.pt, 3);

  uint32_t tb0, tb1;
  my_tiles(ntiles, tb0, tb1);
  const bool use_ovf = ld_acquire_u32(&a.st->ovf_epoch) == a.epoch;
  if (!use_ovf) {
    barrier_skip(a.bar64);  // the fallback's second barrier is not needed
    // the tile totals are loaded together with the first tile's partial rows (one L2 round
    // trip for both) and scanned once the rows are summed
    const uint64_t tv = threadIdx.x < ntiles ? __ldcg(a.tile_red + (uint64_t)threadIdx.x * a.tile_red_stride) : 0ull;
    merge_scan_tiles<PACK16>(
        a, tb0, tb1,
        [&]() -> uint64_t {
          tile_offsets(tv, ntiles, toff, red64);
          return toff[tb0];
        },
        false, sh_hist, red64, sh_hist + kFusedStageOff);
  } else {
    // a packed counter overflowed somewhere: the flushed tile sums are incomplete.  Merge
    // (adding the fallback histogram), publish exact tile totals, barrier, then scan.
    for (uint32_t t = tb0; t < tb1; ++t) {
      const uint64_t tt = merge_tile(a, t, true, sh_hist, red64);
      if (threadIdx.x == 0) __stcg(a.tile_alt + t, (uint32_t)(tt > 0xffffffffull ? 0xffffffffull : tt));
    }
    grid_barrier_mono(a.bar64, a.bar_base + 2 * G);
    tile_offsets(threadIdx.x < ntiles ? __ldcg(a.tile_alt + threadIdx.x) : 0ull, ntiles, toff, red64);
    for (uint32_t t = tb0; t < tb1; ++t) {
      scan_tile(a, a.H, t, toff[t], red64);
      __syncthreads();
      if (threadIdx.x == 0) asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(a.ready + t), "r"(a.epoch) : "memory");
    }
  }
  if (tb1 == ntiles && tb1 > tb0 && threadIdx.x == 0) scan_finish(a, toff[ntiles]);
  phase_mark(a.pt, 4);
  __syncthreads();  // merge scratch (sh_hist) becomes the mark buffers

  // Projection: sub-group s of S = kFusedNSub * G projects positions [b(s), b(s+1)),
  // b(s) = ⌊nw s / S⌋ & ~31, in chunks; it first waits (once) for the ready flags of every
  // scan tile its share overlaps.
  const uint64_t total = toff[ntiles];
  const uint32_t nw = (uint32_t)(total < a.n_expected ? total : a.n_expected);
  const uint32_t g = threadIdx.x / kFusedSub;
  const uint32_t S = kFusedNSub * G, s = kFusedNSub * blockIdx.x + g;
  const uint32_t lo = s == 0 ? 0u : (uint32_t)(((uint64_t)nw * s / S) & ~31ull);
  const uint32_t hi = s + 1 == S ? nw : (uint32_t)(((uint64_t)nw * (s + 1) / S) & ~31ull);
  uint32_t ta = 0;
  if (lo < hi) {
    ta = tile_of(toff, ntiles, lo);
    const uint32_t tb = tile_of(toff, ntiles, hi - 1);
    // relaxed polling (with a short sleep, so spinning warps leave issue slots to the rest
    // of the CTA), then one acquire LOAD of the flag.  Not a fence: fence.acq_rel.gpu is a
    // MEMBAR that waits for every store in flight from this SM — the output stream of the
    // sub-groups already projecting — measured as ~3 us of extra wait per share.
    for (uint32_t t = ta + threadIdx.x % kFusedSub; t <= tb; t += kFusedSub) {
      while (ld_relaxed_flag(a.ready + t) != a.epoch) __nanosleep(64);
      (void)ld_acquire_u32(a.ready + t);
    }
  }
  sub_sync(g);
  phase_mark(a.pt, 5);
  const bool aligned = (reinterpret_cast<uintptr_t>(out) & 15u) == 0;
  const uint64_t pol = l2_evict_first_policy();
#if DIALSORT_EXPAND_MARKS
  uint32_t* M = sh_hist + g * kFusedChunk;
  for (uint32_t p0 = lo; p0 < hi; p0 += kFusedChunk) {
    const uint32_t p1 = hi - p0 > kFusedChunk ? p0 + kFusedChunk : hi;
    expand_chunk(a, toff, ntiles, p0, p1, ta, key_base, out, M, sred[g], g, aligned, pol);
  }
#else
  if (lo < hi) {
    // stage P of the share's scan tiles (one L2 round trip), then warps run independently
    const uint32_t tb = tile_of(toff, ntiles, hi - 1);
    const uint32_t ka = ta * kTileBins, kb = min((tb + 1) * kTileBins, a.U);
    uint32_t* Ps = sh_hist + g * kFusedPCap;
    uint32_t* wc = sh_hist + kFusedNSub * kFusedPCap + (threadIdx.x >> 5) * 128;
    expand_share(a, ka, kb, lo, hi, Ps, wc, g, key_base, out, aligned, pol);
  }
#endif
  phase_mark(a.pt, 7);
  pdl_trigger();
}

}  // namespace ds

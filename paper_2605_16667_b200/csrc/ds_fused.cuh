// ds_fused.cuh — the whole DialSort step (histogram ingestion with the CRN, sub-histogram
// merge, write-offset scan and ordered projection) as ONE persistent, co-resident kernel for
// the shared-memory paths (U <= kSmem16MaxBins).
//
//   ingestion   eq:ingestion P:409-412 (+ CRN def:crn_level P:896-915)   hist_ingest_flush
//   merge       lem:crn P:951-962 lifted to whole histograms              stage/reduce_batch
//   scan        GPU write-offset step (R18; paper P:13-14 has none)       owner offsets + batch scan
//   projection  eq:projection P:418-424                                   project_tbl
//
// Why one kernel: on B200 a kernel boundary plus its ramp costs ~1-2 us and a
// counter+generation grid barrier ~2 us, against a ~10 us HBM floor per 40 MB pass.
//   1. Every CTA ingests its keys into a private shared-memory histogram and flushes it as
//      partial row c (L2; 4-bit, 16-bit or 32-bit counters); its sums over each owning CTA's
//      tiles are added (RED) into G owner totals.
//   2. ONE monotonic grid barrier.  Every CTA requests its first row segments, reads the G
//      owner totals and scans them: oo[c] = first output position of owner c's tiles.
//   3. CTA b merges the tiles [ntiles b / G, ntiles (b+1) / G) (index ownership): H and the
//      exclusive prefix P of its bins (its tiles' offsets come out of the merge's own scan).
//   4. Projection (project_tbl).  Near-uniform histograms (every CTA's own tiles hold ~nw / G
//      positions): each CTA projects its own tiles from P in shared memory — no cross-CTA
//      dependence after the barrier.  Skewed ones: P goes through L2 with per-tile release
//      flags and CTA b projects the equal position share [b nw / G, (b+1) nw / G) — a Zipf
//      hot tile is projected by many CTAs.
// A packed-counter overflow anywhere (exact detection, ds_hist.cuh) adds one barrier: owner
// totals are recomputed with the fallback histogram ovfH, which is cleared at the end.
#pragma once
#include "ds_common.cuh"
#include "ds_hist.cuh"
#include "ds_scan.cuh"

namespace ds {

constexpr uint32_t kFTiles = kSmem16MaxBins / kFTileBins;  // <= 1536 tiles (2 per thread)
constexpr uint32_t kFSlotWords = 128;                       // staged words per row and batch (512 B)
// Staged rows are 132 words apart: the 32 lanes of a warp read one uint4 column from 32 rows,
// and a 4-word pad puts rows r .. r+7 in distinct 16-byte bank groups (conflict-free LDS.128).
constexpr uint32_t kFRowStride = kFSlotWords + 4;
constexpr uint32_t kFMaxRows = 148;                         // rows (CTAs) a staging slot holds
constexpr uint32_t kFTileSlots = 2048;                      // ready-flag slots per parity (>= kFTiles)
constexpr uint32_t kFOwnSlots = 256;                        // owner-total slots (>= kFMaxRows)
// Owner totals are REDs from every CTA into G counters: a 64-word (256 B) stride puts each
// counter in its own L2 line (same-line REDs serialise: 4 lines took 7.7 us for 19K REDs).
constexpr uint32_t kTileTotStride = 64;
constexpr uint32_t kFBatchBins = 1024;                      // max bins per batch (8 4-bit tiles)
// Partial-row formats of k_sort_fused (bins per 128-word staged batch: 128, 256, 1024)
constexpr int kRowU32 = 0, kRowP16 = 1, kRowN4 = 2;
template <int FMT> struct RowFmt {
  static constexpr uint32_t tpb = FMT == kRowU32 ? 2u : FMT == kRowP16 ? 4u : 16u;  // tiles per batch
  static constexpr uint32_t wpt = kFSlotWords / tpb;  // row words per 64-bin tile (64, 32, 8)
};

// Dynamic shared memory after the barrier (words); the ingestion histogram is dead by then.
constexpr uint32_t kFSlot = kFMaxRows * kFRowStride;                 // one staging slot (19536 words)
constexpr uint32_t kFOffStage = 0;                                   // 2 slots x C rows x 132 words
#ifndef DIALSORT_FPASS_TILES
#define DIALSORT_FPASS_TILES 32
#endif
constexpr uint32_t kFPassTiles = DIALSORT_FPASS_TILES;               // own tiles per CTA (own-tile mode)
constexpr uint32_t kFSharePassTiles = (kFSlot - 32) / kFTileBins;    // share mode: 304 tiles per pass
constexpr uint32_t kFOffPs = 2 * kFSlot;                             // own-mode P + 32 sentinels
constexpr uint32_t kFOffHb = kFOffPs + kFPassTiles * kFTileBins + 32; // merged H of the batch (<= 1024)
constexpr uint32_t kFOffWc = kFOffHb + kFBatchBins;                   // 32 warps x 128 mark counts
constexpr uint32_t kFOffOwn = kFOffWc + 32 * 128;                    // oo[G + 1] owner offsets
// the flush's tile sums (and later the share window offsets) sit past the largest histogram
constexpr uint32_t kFOffTsh = kFOffOwn + kFMaxRows + 32 > kSmem16MaxBins / 2 ? kFOffOwn + kFMaxRows + 32
                                                                             : kSmem16MaxBins / 2;
constexpr uint32_t kFSmemWords = kFOffTsh + kFTiles + 32;
static_assert(kFOffOwn + kFMaxRows + 32 <= kSmem16MaxBins / 2, "own-mode P grows the fused kernel's shared memory");

__device__ __forceinline__ uint32_t ld_relaxed_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}


// ---- projection ----------------------------------------------------------------------------
// Projection of positions [lo, hi) whose bins are ka .. ka+m-1 with P staged as Ps[0..m)
// (+ 32 sentinels 0xffffffff), P[ka] <= lo: for every position p of the range
//   key(p) = max{k : P[k] <= p} = ka - 1 + cnt(p),   cnt(p) = #{i : Ps[i] <= p}
// (the bin whose run covers p; empty bins share their start with the next bin and are
// skipped by the max); kbase = key_base + ka - 1.
// #{i : Ps[i] < x} for a warp, given that it lies in [x0, m] (Ps[m ..] are sentinels): rounds of
// 32 lane probes narrow the range 32-fold each (two rounds for m <= 1024), a last round of
// consecutive probes gives the count.
__device__ __forceinline__ uint32_t count_below(const uint32_t* Ps, uint32_t m, uint32_t x0, uint32_t x) {
  const uint32_t lane = threadIdx.x & 31;
  uint32_t len = m - x0;  // the count is in [x0, x0 + len]
  while (len > 32) {
    const uint32_t step = (len + 31) >> 5;
    const uint32_t q = x0 + step * (lane + 1) - 1;
    const uint32_t k = __popc(__ballot_sync(FULL, q < m && Ps[q] < x));
    x0 += step * k;
    len = min(step - 1, m - x0);
  }
  return x0 + __popc(__ballot_sync(FULL, Ps[x0 + lane] < x));  // x0 + lane < m + 32: sentinels
}

// Projection stores: st.global.L1::no_allocate without an L2 hint (measured 0.3 us faster than
// the evict-first hint on c2 / c3, and than the default policy).  full: the 128 positions of the
// warp lie inside [lo, hi); aligned: out + p is 16-byte aligned for every quad start p.
__device__ __forceinline__ void store_quad(int32_t* __restrict__ out, uint32_t p, uint32_t lo, uint32_t hi, uint4 q,
                                           bool aligned, bool full = false) {
  const int4 v = make_int4((int)q.x, (int)q.y, (int)q.z, (int)q.w);
  if (aligned && (full || (p >= lo && p + 4 <= hi))) {
    st_stream4(reinterpret_cast<int4*>(out + p), v);  // no L2 hint
  } else {
    if (p >= lo && p < hi) out[p] = v.x;
    if (p + 1 >= lo && p + 1 < hi) out[p + 1] = v.y;
    if (p + 2 >= lo && p + 2 < hi) out[p + 2] = v.z;
    if (p + 3 >= lo && p + 3 < hi) out[p + 3] = v.w;
  }
}

// Coded domains (Proposition 2): the projection writes codes k; the CTA then rewrites
// its own positions [lo, hi) with phi^-1(k) = dec[k] (just written: L2 hits).
__device__ __forceinline__ void decode_range(int32_t* __restrict__ out, uint32_t lo, uint32_t hi,
                                             const int32_t* __restrict__ dec) {
  __syncthreads();  // (the CTA's projection stores of the range)
  for (uint32_t p = lo + threadIdx.x; p < hi; p += blockDim.x) out[p] = __ldg(dec + out[p]);
}

// ---- table-driven projection (block-level) ----------------------------------------------
// The positions [lo, hi) are cut into 128-position sub-blocks j (absolute: [128 j, 128 j + 128)),
// processed in windows of up to kFTblCap sub-blocks.  Per window, one pass over the bins
// whose start falls in it builds a table entry per sub-block (shared atomics, one bin per
// thread): T.x = #starts (then, after a block scan, c0 = #{i : Ps[i] < 128 j}) | bit 31 when
// two starts share a quad, T.y = the quad occupancy mask, T.z / T.w = each start's offset in
// its quad (2 bits per quad).  Warp w then writes sub-blocks w, w + 32, .. (the CTA writes one
// contiguous front): lane l's quad holds keys kbase + c0 + popc(M & lanes below l), + 1 from
// its start's offset on — about 25 instructions per quad, a third of the ballot / REDUX /
// shuffle projection it replaced.  A sub-block whose quads hold several starts (bins shorter
// than 4 positions, empty bins) takes the count-mark path.
// Positions are shifted by sh = (out / 4) mod 4 (out - sh is 16-byte aligned), so that every
// quad store is aligned whatever the output's offset (a hierarchical block's output starts at
// the block's offset; the warp-cooperative realigned stores this replaced cost ~25 instructions
// a quad).
constexpr uint32_t kFTblCap = kFSlot / 4;  // 4884 sub-blocks per window (one staging slot)
__device__ __forceinline__ void project_tbl(const uint32_t* Ps, uint32_t m, uint32_t kbase, uint32_t lo, uint32_t hi,
                                            uint4* T, uint32_t* wc, uint32_t* red, int32_t* __restrict__ out,
                                            PhaseTimes* pt = nullptr) {
  __shared__ uint32_t s_ib[2];
  const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t ltmask = (1u << lane) - 1u;
  // (positions < 2^32 - 4 after the shift; else unshifted, scalar stores when unaligned)
  const uint32_t sh = hi <= 0xfffffff0u ? (uint32_t)(reinterpret_cast<uintptr_t>(out) >> 2) & 3u : 0u;
  const bool aligned = ((reinterpret_cast<uintptr_t>(out - sh)) & 15u) == 0;
  out -= sh;
  lo += sh;
  hi += sh;
  const uint32_t jl = lo >> 7, jh = (hi + 127) >> 7;
  for (uint32_t jw = jl; jw < jh; jw += kFTblCap) {
    const uint32_t nsb = min(kFTblCap, jh - jw);
    for (uint32_t j = threadIdx.x; j < nsb; j += blockDim.x) T[j] = make_uint4(0, 0, 0, 0);
    if (w == 0) {  // bins [ia, ib) start in the window (Ps[i] + sh < x  <=>  Ps[i] < x - sh)
      const uint32_t xa = jw << 7, xb = (jw + nsb) << 7;
      const uint32_t ia = xa > sh ? count_below(Ps, m, 0, xa - sh) : 0u;
      const uint32_t ib = xb > sh ? count_below(Ps, m, ia, xb - sh) : 0u;
      if (lane == 0) s_ib[0] = ia, s_ib[1] = ib;
    }
    __syncthreads();
    const uint32_t ia = s_ib[0], ib = s_ib[1];
    {  // a sparse window (more than twice as many bins as positions: empty bins share their start
       // with the next bin, so the table's per-start atomics would pile onto a few entries — the
       // tail shares of n = 1e4, U = 65536 skewed took 12.5 us): per position a binary search,
       // key = kbase + #{i : P_i + sh <= p}
      const uint32_t pa = max(lo, jw << 7), pb = min(hi, (jw + nsb) << 7);
      if (ib - ia > 2u * (pb - pa) + 64u) {  // (uniform over the CTA)
        for (uint32_t p = pa + threadIdx.x; p < pb; p += blockDim.x) {
          const uint32_t pp = p - sh;  // (p >= lo >= sh)
          uint32_t l = ia, r = ib;
          while (l < r) {
            const uint32_t mid = (l + r) >> 1;
            if (Ps[mid] <= pp) l = mid + 1;
            else r = mid;
          }
          out[p] = (int32_t)(kbase + l);
        }
        __syncthreads();  // (s_ib is rewritten by the next window)
        continue;
      }
    }
    if (ib - ia <= 8u * nsb) {  // (uniform) few starts per sub-block: one set of atomics per start
      for (uint32_t i = ia + threadIdx.x; i < ib; i += blockDim.x) {
        const uint32_t p = Ps[i] + sh, j = (p >> 7) - jw, q = (p >> 2) & 31u;
        uint32_t* t = reinterpret_cast<uint32_t*>(T + j);
        const uint32_t old = atomicOr(t + 1, 1u << q);
        atomicAdd(t, 1u);
        if ((old >> q) & 1u) atomicOr(t, 0x80000000u);  // a second start in the quad
        atomicOr(t + 2 + (q >> 4), (p & 3u) << (2 * (q & 15u)));
      }
    } else {
      // many starts per sub-block (short bins): a warp takes 32 consecutive starts — ascending
      // positions, so the starts of one sub-block are consecutive lanes — and reduces each
      // sub-block's segment to its first lane (segmented shuffles), which does the atomics once:
      // per-start atomics on a few entries serialised (n = 3e5, U = 65536 skewed: 7.5 us tables)
      for (uint32_t base = ia + 32 * w; base < ib; base += 32 * (blockDim.x >> 5)) {
        const uint32_t i = base + lane;
        const bool v = i < ib;
        const uint32_t p = v ? Ps[i] + sh : 0u, j = v ? (p >> 7) - jw : 0xffffffffu, q = (p >> 2) & 31u;
        const uint32_t jp = __shfl_up_sync(FULL, j, 1), qp = __shfl_up_sync(FULL, q, 1);
        const bool head = v && (lane == 0 || jp != j);
        uint32_t occ = v ? 1u << q : 0u, cnt = v ? 1u : 0u;
        uint32_t zb = v && q < 16 ? (p & 3u) << (2 * q) : 0u, wb = v && q >= 16 ? (p & 3u) << (2 * (q - 16)) : 0u;
        uint32_t dq = v && lane > 0 && jp == j && qp == q ? 1u : 0u;  // shares its quad with the previous start
#pragma unroll
        for (uint32_t d = 1; d < 32; d <<= 1) {
          const uint32_t jd = __shfl_down_sync(FULL, j, d), od = __shfl_down_sync(FULL, occ, d);
          const uint32_t cd = __shfl_down_sync(FULL, cnt, d), zd = __shfl_down_sync(FULL, zb, d);
          const uint32_t wd = __shfl_down_sync(FULL, wb, d), dd = __shfl_down_sync(FULL, dq, d);
          if (lane + d < 32 && jd == j) {
            occ |= od;
            cnt += cd;
            zb |= zd;
            wb |= wd;
            dq |= dd;
          }
        }
        if (head) {
          uint32_t* t = reinterpret_cast<uint32_t*>(T + j);
          const uint32_t old = atomicOr(t + 1, occ);
          atomicAdd(t, cnt);
          if (dq || (old & occ)) atomicOr(t, 0x80000000u);  // two starts in a quad
          if (zb) atomicOr(t + 2, zb);
          if (wb) atomicOr(t + 3, wb);
        }
      }
    }
    __syncthreads();
    {  // c0[j] = ia + Σ_{j' < j} #starts(j'): up to 5 consecutive entries per thread
      constexpr uint32_t K = (kFTblCap + 1023) / 1024;
      const uint32_t j0 = K * threadIdx.x;
      uint32_t v[K], sum = 0;
#pragma unroll
      for (uint32_t k = 0; k < K; ++k) {
        v[k] = j0 + k < nsb ? T[j0 + k].x : 0u;
        sum += v[k] & 0x7fffffffu;
      }
      uint32_t tot;
      uint32_t ex = ia + block_excl_scan<uint32_t>(sum, tot, red);
#pragma unroll
      for (uint32_t k = 0; k < K; ++k) {
        if (j0 + k < nsb) T[j0 + k].x = ex | (v[k] & 0x80000000u);
        ex += v[k] & 0x7fffffffu;
      }
    }
    __syncthreads();
    phase_mark(pt, 13);  // (debug: table built)
    // (per lane: the quad-offset shift and the word of the start offsets are loop constants; T is
    //  read through its 32-bit shared address — the generic pointer's window base was otherwise
    //  re-derived every iteration; a full aligned sub-block stores without per-lane bounds tests)
    const uint32_t rsh = 2 * (lane & 15u);
    uint32_t Ts;  // (an opaque mov keeps it in a register)
    asm volatile("mov.b32 %0, %1;" : "=r"(Ts) : "r"(smem_addr(T) + 16u * w));
    int4* __restrict__ o4 = reinterpret_cast<int4*>(out) + lane;
    // starts before sub-block j + 1 (its c0; the window's end ib after the last one)
    auto ib_next = [&](uint32_t j) -> uint32_t { return j + 1 < nsb ? T[j + 1].x & 0x7fffffffu : ib; };
    for (uint32_t j = w; j < nsb; j += 32) {
      const uint32_t b0 = (jw + j) << 7;
      uint4 e;
      asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                   : "=r"(e.x), "=r"(e.y), "=r"(e.z), "=r"(e.w) : "r"(Ts + 16u * (j - w)) : "memory");
      const uint32_t c0 = e.x & 0x7fffffffu;
      const bool full = aligned && b0 >= lo && b0 + 128u <= hi;  // (warp-uniform)
      uint4 q;
      if (e.y == 0u) {  // no bin starts in the sub-block: one key throughout (long runs: most sub-blocks)
        const uint32_t v = kbase + c0;
        q = make_uint4(v, v, v, v);
      } else if (!(e.x >> 31)) {
        const uint32_t below = __popc(e.y & ltmask), own = (e.y >> lane) & 1u;
        const uint32_t r = ((lane < 16 ? e.z : e.w) >> rsh) & 3u;
        const uint32_t v = kbase + c0 + below;
        q = make_uint4(v + (own & (r == 0)), v + (own & (r <= 1)), v + (own & (r <= 2)), v + own);
      } else if (ib_next(j) - c0 > 96u) {
        // many starts in the sub-block (empty bins share their start with the next bin — a sparse
        // stretch of the universe): per position a binary search over the sub-block's starts,
        // key = kbase + #{i : P_i + sh <= p} (the marks loop below walks every start: one sparse
        // share of n = 1e4, U = 65536 took 22 us)
        const uint32_t cend = ib_next(j);
        uint32_t v[4];
#pragma unroll
        for (uint32_t u = 0; u < 4; ++u) {
          const uint32_t pp = b0 + 4 * lane + u - sh;  // (b0 + 4 lane + u >= sh: b0 >= lo - 127 >= 0 ...)
          uint32_t l = c0, r = cend;
          while (l < r) {
            const uint32_t mid = (l + r) >> 1;
            if (Ps[mid] <= pp) l = mid + 1;
            else r = mid;
          }
          v[u] = kbase + l;
        }
        q = make_uint4(v[0], v[1], v[2], v[3]);
      } else {  // count marks of the sub-block's starts, then a warp scan
        const uint32_t be = hi - b0 > 128 ? b0 + 127 : hi - 1;  // (>= lo >= sh)
        uint32_t i1 = c0;
        for (;;) {
          const uint32_t sl = Ps[min(i1 + lane, m)];  // Ps[m] is a sentinel
          const uint32_t cnt = __popc(__ballot_sync(FULL, sl <= be - sh));
          if (lane < cnt) atomicAdd(&wc[sl + sh - b0], 1u);
          i1 += cnt;
          if (cnt < 32) break;
        }
        __syncwarp();
        uint4 mk = reinterpret_cast<uint4*>(wc)[lane];
        reinterpret_cast<uint4*>(wc)[lane] = make_uint4(0, 0, 0, 0);
        mk.y += mk.x;
        mk.z += mk.y;
        mk.w += mk.z;
        const uint32_t v = kbase + c0 + warp_incl_scan(mk.w) - mk.w;
        q = make_uint4(v + mk.x, v + mk.y, v + mk.z, v + mk.w);
        __syncwarp();
      }
      if (full) st_stream4(o4 + (b0 >> 2), make_int4((int)q.x, (int)q.y, (int)q.z, (int)q.w));
      else store_quad(out, b0 + 4 * lane, lo, hi, q, aligned);
    }
    __syncthreads();  // T is reused by the next window
  }
}

// ---- merge of one batch (128 words = 512 B of every row: 2, 4 or 16 tiles) ----------------
// Issues the cp.async copies of the batch's row segments into a staging slot (row r: 128
// words at slot + 128 r).  Tiles of the batch that this CTA does not need are not copied.
template <int FMT>
__device__ __forceinline__ void stage_batch(const ScanArgs& a, uint32_t t0, uint32_t need_mask, uint32_t* slot) {
  constexpr uint32_t qpt = 32 / RowFmt<FMT>::tpb;  // uint4 per tile (16, 8, 2)
  const uint32_t l = threadIdx.x & 31, r0 = threadIdx.x >> 5;  // uint4 l of rows r0, r0 + 32, ..
  if (!((need_mask >> (l / qpt)) & 1u)) return;
  const uint32_t Wrow = FMT == kRowU32 ? a.U : FMT == kRowP16 ? (a.U + 1) / 2 : (a.U + 7) / 8;  // row words
  const uint32_t word = t0 * RowFmt<FMT>::wpt + 4 * l;
  const uint32_t bytes = word < Wrow ? 16u : 0u;  // zero-fill past the row's last word
  const uint32_t* src = a.partials + (uint64_t)r0 * a.ldr + (bytes ? word : 0u);
  uint32_t dst = smem_addr(slot + r0 * kFRowStride + 4 * l);
  const uint64_t sstep = 32ull * a.ldr;  // (blockDim = 1024: 32 warps)
  for (uint32_t r = r0; r < a.C; r += 32, src += sstep, dst += 32 * kFRowStride * 4)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(bytes) : "memory");
}

// Reduce-scatter of a warp's N partial sums (registers v[0..N)) across its 32 lanes: at each
// halving step a lane keeps one half (by its lane bit) and adds the partner's copy of it;
// finally lane l holds the warp total of index (l >> (5 - log2 N)) in v[0] (N <= 16).
template <uint32_t N, uint32_t O>
__device__ __forceinline__ void reduce_scatter_step(uint32_t (&v)[16], uint32_t lane) {
  if constexpr (O != 0) {
    if constexpr (N > 1) {
      const bool up = (lane & O) != 0;
#pragma unroll
      for (uint32_t i = 0; i < N / 2; ++i) {
        const uint32_t send = up ? v[i] : v[i + N / 2];
        const uint32_t keep = up ? v[i + N / 2] : v[i];
        v[i] = keep + __shfl_xor_sync(FULL, send, O);
      }
      reduce_scatter_step<N / 2, O / 2>(v, lane);
    } else {
      v[0] += __shfl_xor_sync(FULL, v[0], O);
      reduce_scatter_step<1, O / 2>(v, lane);
    }
  }
}

// Bin of the batch that lane `lane` of warp `w` produces in reduce_batch (N4: every lane;
// P16 / U32: the lanes with (lane & 3) == 0 / (lane & 7) == 0).
template <int FMT>
__device__ __forceinline__ uint32_t batch_bin(uint32_t w, uint32_t lane) {
  if (FMT == kRowN4) {  // register 4k + a holds nibbles nlo(a), nlo(a) + 4 of word k
    const uint32_t i = lane >> 1, k = i >> 2, a = i & 3u;
    return 32 * w + 8 * k + (((a & 1u) << 1) | (a >> 1)) + 4 * (lane & 1u);
  } else if (FMT == kRowP16) {
    return 8 * w + (lane >> 2);
  } else {
    return 4 * w + (lane >> 3);
  }
}

// Sums the staged rows of a batch into hb[j] = merged count of the batch's bin j (+ the 4-bit
// rows' exceptions Hx, + ovfH when the packed counters overflowed somewhere); bins of tiles
// not needed get 0.  Warp w takes uint4 column w of the 128-word batch and lane l the rows
// l, l + 32, .. (five 16-byte shared loads); the 32 lanes' partial sums — 4-bit rows in byte
// then 16-bit SWAR lanes — meet in a warp reduce-scatter (16 / 9 / 6 shuffles).  The caller
// synchronises before hb is read.
template <int FMT>
__device__ __forceinline__ void reduce_batch(const ScanArgs& a, uint32_t t0, uint32_t need_mask, const uint32_t* slot,
                                             uint32_t* hb, bool use_ovf, uint32_t hx) {
  constexpr uint32_t wpt = RowFmt<FMT>::wpt;
  constexpr uint32_t RPL = (kFMaxRows + 31) / 32;  // rows per lane (5)
  const uint32_t lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const bool need = (need_mask >> (4 * w / wpt)) & 1u;
  uint32_t v[16];
  if (need) {
    uint4 x[RPL];
#pragma unroll
    for (uint32_t i = 0; i < RPL; ++i) {
      const uint32_t r = lane + 32 * i;
      x[i] = r < a.C ? *reinterpret_cast<const uint4*>(slot + r * kFRowStride + 4 * w) : make_uint4(0, 0, 0, 0);
    }
    if (FMT == kRowN4) {
      uint32_t be[4] = {0, 0, 0, 0}, bo[4] = {0, 0, 0, 0};  // <= 5 rows of 15 per byte lane
#pragma unroll
      for (uint32_t i = 0; i < RPL; ++i) {
        const uint32_t xw[4] = {x[i].x, x[i].y, x[i].z, x[i].w};
#pragma unroll
        for (uint32_t k = 0; k < 4; ++k) {
          be[k] += xw[k] & 0x0F0F0F0Fu;
          bo[k] += (xw[k] >> 4) & 0x0F0F0F0Fu;
        }
      }
#pragma unroll
      for (uint32_t k = 0; k < 4; ++k) {  // 16-bit lanes: nibbles (0,4) (2,6) (1,5) (3,7)
        v[4 * k + 0] = be[k] & 0x00FF00FFu;
        v[4 * k + 1] = (be[k] >> 8) & 0x00FF00FFu;
        v[4 * k + 2] = bo[k] & 0x00FF00FFu;
        v[4 * k + 3] = (bo[k] >> 8) & 0x00FF00FFu;
      }
      reduce_scatter_step<16, 16>(v, lane);  // <= 32 x 75 per 16-bit lane
    } else if (FMT == kRowP16) {
#pragma unroll
      for (uint32_t k = 0; k < 8; ++k) v[k] = 0;
#pragma unroll
      for (uint32_t i = 0; i < RPL; ++i) {
        const uint32_t xw[4] = {x[i].x, x[i].y, x[i].z, x[i].w};
#pragma unroll
        for (uint32_t k = 0; k < 4; ++k) {
          v[2 * k] += xw[k] & 0xffffu;
          v[2 * k + 1] += xw[k] >> 16;
        }
      }
      reduce_scatter_step<8, 16>(v, lane);
    } else {
#pragma unroll
      for (uint32_t k = 0; k < 4; ++k) v[k] = 0;
#pragma unroll
      for (uint32_t i = 0; i < RPL; ++i) {
        v[0] += x[i].x;
        v[1] += x[i].y;
        v[2] += x[i].z;
        v[3] += x[i].w;
      }
      reduce_scatter_step<4, 16>(v, lane);
    }
  }
  phase_mark(a.pt, 12);
  const bool writer = FMT == kRowN4 ? true : FMT == kRowP16 ? (lane & 3u) == 0 : (lane & 7u) == 0;
  if (writer) {
    const uint32_t j = batch_bin<FMT>(w, lane);
    uint32_t h = 0;
    if (need) {
      h = FMT == kRowN4 ? ((lane & 1u) ? v[0] >> 16 : v[0] & 0xffffu) : v[0];
      h += hx;  // Hx[bin] of 4-bit rows (0 otherwise), prefetched by the caller
      const uint64_t bin = (uint64_t)t0 * kFTileBins + j;
      if (use_ovf && bin < a.U) h += __ldcg(a.ovfH + bin);
    }
    hb[j] = h;
  }
}

// Overflow path: exact total of tile t straight from the partial rows, Hx and ovfH.
template <int FMT>
__device__ __forceinline__ uint64_t tile_total_direct(const ScanArgs& a, uint32_t t, uint64_t* red) {
  uint64_t s = 0;
  const uint32_t k0 = t * kFTileBins;
  for (uint32_t i = threadIdx.x; i < kFTileBins * a.C; i += blockDim.x) {
    const uint32_t j = i % kFTileBins, r = i / kFTileBins, k = k0 + j;
    if (k >= a.U) continue;
    const uint32_t* row = a.partials + (uint64_t)r * a.ldr;
    if (FMT == kRowU32) s += __ldcg(row + k);
    else if (FMT == kRowP16) s += (__ldcg(row + (k >> 1)) >> ((k & 1u) << 4)) & 0xffffu;
    else s += (__ldcg(row + (k >> 3)) >> ((k & 7u) << 2)) & 0xfu;
    if (r == 0) s += __ldcg(a.ovfH + k) + (FMT != kRowU32 ? __ldcg(a.Hx + k) : 0u);
  }
  return block_sum<uint64_t>(s, red);
}

// One DialSort step: keys[n] in [0,U) -> out[min(ΣH, cap)] sorted; H as a by-product — run by
// the G CTAs of the virtual grid vg (the whole launch, or one group of k_sort_batch).
// C = vg.G <= min(#SMs, kFMaxRows) CTAs of 1024 threads (co-resident, 1 per SM).  Dynamic smem:
// max(histogram, kFSmemWords words).  Two grid barriers are reserved per step (the second one
// is only waited for after a packed-counter overflow).
// FROM_H (reconstruct_step): no keys — the step projects a given histogram H (a.partials = H as
// the single u32 "row", a.C = 1): each CTA sums its own tiles of H and adds its total into the
// owner counters P_{o+1} of every owner o >= b instead of ingesting and flushing.
// (fbase, fseq: the step's barrier base and sequence number, from FusedState; fs_adv: the state
//  CTA 0 advances to {adv_base, adv_seq} once the first barrier shows every CTA has read it — no
//  exit ticket, and the next launch reads it after this grid completes)
template <int FMT, int KB, bool FROM_H = false>
__device__ __forceinline__ void sort_step(const void* __restrict__ keys, uint64_t n, const ScanArgs& a_in,
                                          int32_t* __restrict__ out, int32_t key_base, VGrid vg, uint32_t* sh,
                                          uint64_t* red64, uint32_t* wsum, unsigned long long fbase, uint32_t fseq,
                                          FusedState* fs_adv = nullptr, unsigned long long adv_base = 0,
                                          uint32_t adv_seq = 0) {
  // the step's parity buffers, epoch and barrier base (derived from the device-side sequence)
  ScanArgs a = a_in;
  {
    const uint32_t par = fseq & 1u;
    const uint64_t own_words = (uint64_t)kFOwnSlots * kTileTotStride;
    a.own_red = a.own_base + own_words * par;
    a.own_clear = a.own_base + own_words * (par ^ 1u);
    a.own_alt = a.own_base + 2 * own_words;
    a.ready = a.ready_base + (uint64_t)kFTileSlots * par;
    a.ready_clear = a.ready_base + (uint64_t)kFTileSlots * (par ^ 1u);
    a.Hx = a.Hx_base + (uint64_t)kSmem16MaxBins * par;
    a.Hx_clear = a.Hx_base + (uint64_t)kSmem16MaxBins * (par ^ 1u);
    a.epoch = (fseq % 0xffffffu) + 1u;
    a.bar_base = fbase;
  }
  // (KB: key bytes — 4 int32 keys; 2 uint16 keys, the hierarchical path's universe blocks or a
  //  2-byte coded domain; 1 uint8 keys, a 1-byte coded domain)
  // (keys, out, n are adjusted below for hierarchical blocks)
  uint64_t n_exp = a.n_expected;
  if (a.d_n) {  // a universe block of the hierarchical path: size and offset on the device
    __shared__ uint64_t s_noff[3];  // (one load per CTA, not one per thread: a 148k-way fan-in)
    if (threadIdx.x == 0) s_noff[0] = *a.d_n, s_noff[1] = *a.d_off, s_noff[2] = a.d_koff ? *a.d_koff : s_noff[1];
    __syncthreads();
    const uint64_t off = s_noff[1];
    n = s_noff[0];
    keys = static_cast<const char*>(keys) + s_noff[2] * KB;
    out += off;
    n_exp = n;
  }
  const uint32_t U = a.U, ntiles = (U + kFTileBins - 1) / kFTileBins;
  const uint32_t G = vg.G, b = vg.b;
  // the other parity's owner totals are zeroed for the next launch (host alternates them;
  // every slot, since the next launch may have more CTAs than this one)
  if (b == G - 1) {
    for (uint32_t i = threadIdx.x; i < kFOwnSlots; i += blockDim.x) a.own_clear[(uint64_t)i * kTileTotStride] = 0;
    for (uint32_t i = threadIdx.x; i < kFTileSlots; i += blockDim.x) a.ready_clear[i] = 0;
  }
  if (a.Hx_clear)  // and the other parity's exception histogram (all of it: launches of any
                   // format alternate the parity, and the next may have a larger U), a slice per CTA
  {  // 16-byte stores, bounds computed once (Hx buffers are 16-byte aligned, kSmem16MaxBins % 4 == 0)
    const uint32_t q0 = (kSmem16MaxBins / 4) * b / G, q1 = (kSmem16MaxBins / 4) * (b + 1) / G;
    if (q0 + threadIdx.x < q1) reinterpret_cast<uint4*>(a.Hx_clear)[q0 + threadIdx.x] = make_uint4(0, 0, 0, 0);
    for (uint32_t q = q0 + threadIdx.x + blockDim.x; q < q1; q += blockDim.x)
      reinterpret_cast<uint4*>(a.Hx_clear)[q] = make_uint4(0, 0, 0, 0);
  }
  constexpr bool PACK16 = FMT != kRowU32;

  // the row's 64-bin tile sums (flush) sit past the largest ingestion histogram; zeroed here
  // (the ingestion's first __syncthreads orders this before the flush)
  static_assert(kFOffTsh >= kSmem16MaxBins / 2, "tile sums overlap the packed histogram");
  if constexpr (FROM_H) {
    // own tiles' total t_b of the given H, added into P_{o+1} for o = b .. G-1 (Σ_{o' <= o} t_o'),
    // and the skew vote against the expected total (n_exp = ΣH in exact mode)
    uint32_t t0, t1;
    my_tiles(ntiles, t0, t1, vg);
    const uint32_t k1 = min(t1 * kFTileBins, U);
    uint32_t sum = 0;
    for (uint32_t k = t0 * kFTileBins + threadIdx.x; k < k1; k += blockDim.x) sum += __ldcg(a.partials + k);
    sum = block_sum<uint32_t>(sum, reinterpret_cast<uint32_t*>(red64));
    for (uint32_t o = b + threadIdx.x; o < G && sum; o += blockDim.x)
      red_add_u32(a.own_red + (uint64_t)(o + 1) * a.ctr_stride, sum);
    if (threadIdx.x == 0 && 4ull * G * sum > 5ull * n_exp + kSkewSlack)
      red_add_u32(a.own_red + (uint64_t)kFOwnVote * a.ctr_stride, 1u);
    __syncthreads();
  } else {
    for (uint32_t i = threadIdx.x; i < ntiles; i += blockDim.x) sh[kFOffTsh + i] = 0;
    hist_ingest_flush<PACK16, KB>(keys, n, a, sh, red64, sh + kFOffTsh, vg);
  }
  __shared__ uint32_t s_own[2];  // this CTA's tiles [tb0, tb1) (index ownership)
  grid_barrier_mono_side(a.bar64, a.bar_base + G, [&] {  // rows, tile / owner totals, overflow fallback in L2
    my_tiles(ntiles, s_own[0], s_own[1], vg);
  });
  if (fs_adv && b == 0 && threadIdx.x == 0) {
    fs_adv->base = adv_base;
    fs_adv->seq = adv_seq;
  }
  phase_mark(a.pt, 3);

  const uint32_t tb0 = s_own[0], tb1 = s_own[1];  // tiles this CTA merges
  const uint32_t nown = tb1 - tb0;
  constexpr uint32_t tpb = RowFmt<FMT>::tpb;  // tiles per batch
  constexpr uint32_t nbb = tpb * kFTileBins;  // bins per batch
  const uint32_t S = a.ctr_stride;  // (counter stride)
  auto slot = [&](uint32_t k) { return sh + kFOffStage + (k & 1u) * kFSlot; };  // 2 slots
  uint32_t* hb = sh + kFOffHb;
  uint32_t* Ps = sh + kFOffPs;
  uint32_t* oo = sh + kFOffOwn;   // oo[c] = first output position of owner c's tiles, oo[G] = total
  uint32_t* wc = sh + kFOffWc + (threadIdx.x >> 5) * 128;
  reinterpret_cast<uint4*>(wc)[threadIdx.x & 31] = make_uint4(0, 0, 0, 0);
  const uint32_t nbt = nown ? (nown + tpb - 1) / tpb : 0u;  // batches tb0 + k tpb ..
  auto need_of = [&](uint32_t k) -> uint32_t {
    const uint32_t t0 = tb0 + k * tpb, nt = min(tpb, tb1 - t0);
    return nt >= 32 ? 0xffffffffu : (1u << nt) - 1u;
  };
  // This CTA's offset counters (P_b, P_{b+1}: its tiles' first output position and the next
  // owner's, flush_owner_totals), the skew vote, the overflow state and the first two batches'
  // row segments (and their exception counts) are requested together: none depends on another,
  // and the barrier ordered every CTA's flush before them.  Two counter lines per CTA, each read
  // by two CTAs (all owner totals read by every CTA measured ~1.7 us: a 148-way fan-in).
  // (one thread loads each shared word — every thread loading the overflow epoch measured as the
  // top stall of the kernel: 151k loads of one L2 line)
  __shared__ uint32_t s_pb[4];
  if (threadIdx.x == 0) {
    s_pb[0] = b ? __ldcg(a.own_red + (uint64_t)b * S) : 0u;
    s_pb[1] = __ldcg(a.own_red + (uint64_t)(b + 1) * S);
    s_pb[2] = __ldcg(a.own_red + (uint64_t)kFOwnVote * S);
    s_pb[3] = __ldcg(&a.st->ovf_epoch);
  }
  for (uint32_t k = 0; k < 2 && k < nbt; ++k) {
    stage_batch<FMT>(a, tb0 + k * tpb, need_of(k), slot(k));
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  // Hx of the bin this thread produces in reduce_batch (4-bit rows), loaded a batch ahead
  const uint32_t binend = min(tb1 * kFTileBins, U);  // bins of the own tiles end here
  auto hx_of = [&](uint32_t k) -> uint32_t {
    const uint32_t bin = (tb0 + k * tpb) * kFTileBins + batch_bin<FMT>(threadIdx.x >> 5, threadIdx.x & 31);
    // (4-bit rows' exceptions and — 4-bit and 16-bit rows — the hot keys' counts, ds_hist.cuh)
    const bool wr = FMT == kRowN4 || (FMT == kRowP16 && (threadIdx.x & 3u) == 0);
    return FMT != kRowU32 && wr && bin < binend ? __ldcg(a.Hx + bin) : 0u;
  };
  uint32_t hx = hx_of(0);
  __syncthreads();  // s_pb
  const bool use_ovf = s_pb[3] == a.epoch;
  // own-tile mode: every CTA projects exactly the tiles it merged (near-uniform histograms: no
  // skew vote); otherwise (skew, or a packed-counter overflow) equal position shares, for which
  // every owner offset oo[0..G] is read.
  constexpr uint32_t kOPL = (kFMaxRows + 31) / 32;
  uint32_t ov[kOPL];
  bool own;
  if (!use_ovf) {
    barrier_skip(a.bar64);
    own = ntiles <= kFPassTiles * G && s_pb[2] == 0;  // (every CTA's tiles fit one projection pass)
    if (!own) {
      for (uint32_t c = threadIdx.x; c <= G; c += blockDim.x) oo[c] = c ? __ldcg(a.own_red + (uint64_t)c * S) : 0u;
      __syncthreads();
    }
  } else {
    // a packed counter overflowed somewhere: the flushed owner sums miss the fallback keys
    uint64_t osd = 0;
    for (uint32_t t = tb0; t < tb1; ++t) osd += tile_total_direct<FMT>(a, t, red64);
    if (threadIdx.x == 0) __stcg(a.own_alt + b, (uint32_t)osd);
    grid_barrier_mono(a.bar64, a.bar_base + 2 * G);
#pragma unroll
    for (uint32_t j = 0; j < kOPL; ++j) {
      const uint32_t c = kOPL * threadIdx.x + j;
      ov[j] = threadIdx.x < 32 && c < G ? __ldcg(a.own_alt + c) : 0u;
    }
    // owner offsets: oo[c] = first output position of owner c's tiles (one warp)
    if (threadIdx.x < 32) {  // (every count sum here is <= n < 2^32, R4)
      uint32_t sum = 0;
#pragma unroll
      for (uint32_t j = 0; j < kOPL; ++j) sum += ov[j];
      const uint32_t inc = warp_incl_scan(sum);
      uint32_t ex = inc - sum;
#pragma unroll
      for (uint32_t j = 0; j < kOPL; ++j) {
        const uint32_t c = kOPL * threadIdx.x + j;
        if (c < G) oo[c] = ex;
        ex += ov[j];
      }
      if (threadIdx.x == 31) oo[G] = inc;
    }
    __syncthreads();
    own = false;
  }
  phase_mark(a.pt, 4);
  const uint32_t obase = own ? s_pb[0] : oo[b];    // first output position of this CTA's tiles
  const uint32_t oend = own ? s_pb[1] : oo[b + 1];  // ... and of the next owner's (the last: the total)
  if (b == G - 1 && threadIdx.x == 0) {
    const uint64_t total = oend;
    unsigned flags = 0;
    if (a.exact ? (total != n_exp) : (total > n_exp)) flags |= FLAG_SIZE;
    if (flags) atomicOr(&a.st->flags, flags);
    a.st->last_total = total;
    if (a.d_total) *a.d_total = total;
    *a.ws_total = total;
  }
  // positions written: [0, min(total, n_exp)) (share mode needs the total: oo[G])
  const uint32_t nw = own ? 0u : (uint32_t)(oo[G] < n_exp ? oo[G] : n_exp);
  // equal share [lo, hi) (share mode) and the owners oa..ob (tiles [x0, x1)) it overlaps
  uint32_t lo = 0, hi = 0;
  if (!own) {
    lo = b == 0 ? 0u : (uint32_t)(((uint64_t)nw * b / G) & ~31ull);
    hi = b + 1 == G ? nw : (uint32_t)(((uint64_t)nw * (b + 1) / G) & ~31ull);
  }
  const bool share = !own && lo < hi;
  uint32_t oa = 0, ob = 0, x0 = 0, x1 = 0;
  __shared__ uint32_t s_find[2];
  if (!own) {  // the owners holding positions lo and hi - 1: one test per owner, not a search
    if (lo < hi)
      for (uint32_t c = threadIdx.x; c < G; c += blockDim.x) {
        if (oo[c] <= lo && lo < oo[c + 1]) s_find[0] = c;
        if (oo[c] <= hi - 1 && hi - 1 < oo[c + 1]) s_find[1] = c;
      }
    __syncthreads();
  }
  if (share) {
    oa = s_find[0];
    ob = s_find[1];
    x0 = (uint32_t)((uint64_t)ntiles * oa / G);
    x1 = (uint32_t)((uint64_t)ntiles * (ob + 1) / G);
  }

  // ---- merge: H and the exclusive prefix P of the tiles this CTA owns --------------------
  // (lem:crn lifted to whole histograms: H = sum of the partial rows, + Hx, + ovfH).  Own-tile
  // mode keeps P in shared memory; otherwise P goes to L2 and each batch is published
  // (ready[t] = epoch, release) for the CTAs whose shares overlap it.
  __shared__ uint32_t wex[32], s_btot;
  uint32_t carry = 0;  // positions of the own tiles of earlier batches
  for (uint32_t k = 0; k < nbt; ++k) {
    const uint32_t t0 = tb0 + k * tpb, need = need_of(k);
    if (k + 1 < nbt) asm volatile("cp.async.wait_group 1;" ::: "memory");
    else asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    phase_mark(a.pt, 5);
    reduce_batch<FMT>(a, t0, need, slot(k), hb, use_ovf, hx);
    __syncthreads();  // hb complete; the slot is free
    phase_mark(a.pt, 10);
    if (k + 2 < nbt) {
      stage_batch<FMT>(a, tb0 + (k + 2) * tpb, need_of(k + 2), slot(k));
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
    hx = hx_of(k + 1);
    // exclusive prefix over the batch's bins (the own tiles are consecutive; bins of tiles not
    // needed hold 0): warp scans, then warp 0 scans the warp totals; + the earlier batches
    const uint32_t j = threadIdx.x;
    const uint32_t h = j < nbb ? hb[j] : 0u;
    const uint32_t inc = warp_incl_scan(h);
    if ((j & 31) == 31) wsum[j >> 5] = inc;
    __syncthreads();
    if (j < 32) {
      const uint32_t x = wsum[j], xi = warp_incl_scan(x);
      wex[j] = xi - x;
      if (j == 31) s_btot = xi;
    }
    __syncthreads();
    phase_mark(a.pt, 14);
    if (j < nbb && ((need >> (j / kFTileBins)) & 1u)) {
      const uint32_t wpre = obase + carry + wex[j >> 5];
      const uint32_t bin = t0 * kFTileBins + j;
      const uint32_t p = bin < U ? wpre + inc - h : oend;  // (bins >= U: the last tile; oend = total)
      if (bin < U && (a.H || a.Hpeer)) store_H(a, bin, h);  // (a given H is not written back)
      if (own) Ps[(t0 - tb0) * kFTileBins + j] = p;
      else if (bin < U && !a.hist_only) a.P[bin] = p;
    }
    carry += s_btot;  // (read before the next batch's scan rewrites it: two barriers apart)
    phase_mark(a.pt, 15);
    if (!own && !a.hist_only) {
      __syncthreads();  // the batch's H and P are written
      if (threadIdx.x < tpb && ((need >> threadIdx.x) & 1u))
        asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(a.ready + t0 + threadIdx.x), "r"(a.epoch) : "memory");
    }
  }
  if (use_ovf)  // only this CTA read ovfH for its tiles: clear them for the next call
    for (uint32_t k = tb0 * kFTileBins + threadIdx.x; k < min(tb1 * kFTileBins, U); k += blockDim.x) a.ovfH[k] = 0;
  phase_mark(a.pt, 6);
  if (a.hist_only) {  // histogram-only launch (hierarchical histogram, multi-GPU exchange)
    return;
  }

  if (own) {
    // ---- projection of the own tiles' positions [oo[b], oo[b+1]) ∩ [0, nw) -----------------
    const uint32_t m = nown * kFTileBins;
    if (threadIdx.x < 32) Ps[m + threadIdx.x] = 0xffffffffu;
    __syncthreads();
    phase_mark(a.pt, 9);
    const uint32_t p0 = obase, p1 = (uint32_t)(oend < n_exp ? oend : n_exp);
    if (nown && p0 < p1) {  // (uniform per CTA) table in the second staging slot, dead after the merge
      project_tbl(Ps, m, (uint32_t)key_base + tb0 * kFTileBins - 1, p0, p1,
                  reinterpret_cast<uint4*>(sh + kFOffStage + kFSlot), wc, reinterpret_cast<uint32_t*>(red64), out);
      if (a.dec) decode_range(out, p0, p1, a.dec);
    }
    phase_mark(a.pt, 7);
    return;
  }

  // ---- projection of an equal share of the positions -------------------------------------
  // CTA b projects [lo, hi) = [b nw / G, (b+1) nw / G) (32-aligned), the same number of
  // outputs whatever the skew: offsets of the window tiles [x0, x1) (the tiles of owners
  // oa..ob), then it waits for the tiles the share overlaps, stages their P in shared memory,
  // and its 32 warps project.
  if (share) {
    // wait for the tiles of owners oa..ob (relaxed polling — a short sleep leaves issue slots to
    // the rest of the CTA — then one acquire load per flag; not a fence: fence.acq_rel.gpu
    // waits for every store in flight); their first bins' P are the window's tile offsets
    uint32_t* ts = sh + kFOffTsh;  // ts[i] = first position of tile x0 + i
    for (uint32_t t = x0 + threadIdx.x; t < x1; t += blockDim.x) {
      while (ld_relaxed_u32(a.ready + t) != a.epoch) __nanosleep(64);
      (void)ld_acquire_u32(a.ready + t);
      ts[t - x0] = __ldcg(a.P + (uint64_t)t * kFTileBins);
    }
    if (threadIdx.x == 0) ts[x1 - x0] = oo[ob + 1];
    __syncthreads();
    phase_mark(a.pt, 8);
    for (uint32_t i = threadIdx.x; i < x1 - x0; i += blockDim.x) {  // the tiles holding lo, hi - 1
      if (ts[i] <= lo && lo < ts[i + 1]) s_find[0] = i;
      if (ts[i] <= hi - 1 && hi - 1 < ts[i + 1]) s_find[1] = i;
    }
    __syncthreads();
    const uint32_t ta = x0 + s_find[0], tb = x0 + s_find[1];
    // P of the share's tiles staged in the (now dead) first row-staging slot: up to 295 tiles
    // per pass (a Zipf share in the cold tail spans ~200 tiles; 32-tile passes left most warps
    // idle); the projection table takes the second slot
    uint32_t* Pw = sh + kFOffStage;
    for (uint32_t pt0 = ta; pt0 <= tb; pt0 += kFSharePassTiles) {
      const uint32_t pt1 = min(pt0 + kFSharePassTiles, tb + 1);
      const uint32_t m = (pt1 - pt0) * kFTileBins, b0 = pt0 * kFTileBins;
      for (uint32_t i = 4 * threadIdx.x; i < m; i += 4 * blockDim.x) {  // 16 B per copy, zero-fill past U
        const uint32_t bytes = b0 + i + 4 <= U ? 16u : (b0 + i < U ? 4u * (U - b0 - i) : 0u);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_addr(Pw + i)),
                     "l"(a.P + (bytes ? b0 + i : 0u)), "r"(bytes) : "memory");
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
      if (threadIdx.x < 32) Pw[m + threadIdx.x] = 0xffffffffu;
      asm volatile("cp.async.wait_group 0;" ::: "memory");
      __syncthreads();
      if (b0 + m > U) {  // bins >= U of a last partial tile
        for (uint32_t i = U - b0 + threadIdx.x; i < m; i += blockDim.x) Pw[i] = oo[G];
        __syncthreads();
      }
      phase_mark(a.pt, 9);
      const uint32_t p0 = max(lo, ts[pt0 - x0]), p1 = min(hi, ts[pt1 - x0]);
      if (p0 < p1) {
        project_tbl(Pw, m, (uint32_t)key_base + pt0 * kFTileBins - 1, p0, p1,
                    reinterpret_cast<uint4*>(sh + kFOffStage + kFSlot), wc, reinterpret_cast<uint32_t*>(red64), out,
                    a.pt);
        if (a.dec) decode_range(out, p0, p1, a.dec);
      }
      __syncthreads();  // Pw is reused by the next pass
    }
  }
  phase_mark(a.pt, 7);
}



// Start of a launch: every CTA reads the workspace's barrier base and step sequence.
__device__ __forceinline__ void fused_state_read(const FusedState* fs, unsigned long long* s2) {
  if (threadIdx.x == 0) {
    s2[0] = *reinterpret_cast<const volatile unsigned long long*>(&fs->base);
    s2[1] = *reinterpret_cast<const volatile unsigned int*>(&fs->seq);
  }
  __syncthreads();
}
template <int FMT, int KB = 4>
__global__ void __launch_bounds__(1024, 1) k_sort_fused(const void* __restrict__ keys, uint64_t n, ScanArgs a,
                                                       int32_t* __restrict__ out, int32_t key_base) {
  extern __shared__ __align__(128) uint32_t sh[];
  __shared__ uint64_t red64[34];
  __shared__ uint32_t wsum[32];
  __shared__ unsigned long long s_fs[2];
  pdl_wait();
  phase_mark(a.pt, -1);
  fused_state_read(a.fstate, s_fs);
  const unsigned long long base = s_fs[0];
  const uint32_t seq = (uint32_t)s_fs[1];
  sort_step<FMT, KB>(keys, n, a, out, key_base, vgrid_hw(), sh, red64, wsum, base, seq, a.fstate,
                     base + 2ull * gridDim.x, seq + 1);
  pdl_trigger();
}

// The projection of a given histogram H (dialsort_reconstruct_async, the sharded slice
// projection) as one co-resident kernel: offsets, scan and projection of sort_step without the
// ingestion (U <= kFTileSlots * 64 bins: the share mode's ready flags).
__global__ void __launch_bounds__(1024, 1) k_reconstruct_fused(ScanArgs a, uint64_t cap, int32_t* __restrict__ out,
                                                              int32_t key_base) {
  extern __shared__ __align__(128) uint32_t sh[];
  __shared__ uint64_t red64[34];
  __shared__ uint32_t wsum[32];
  __shared__ unsigned long long s_fs[2];
  pdl_wait();
  fused_state_read(a.fstate, s_fs);
  const unsigned long long base = s_fs[0];
  const uint32_t seq = (uint32_t)s_fs[1];
  sort_step<kRowU32, 4, true>(nullptr, cap, a, out, key_base, vgrid_hw(), sh, red64, wsum, base, seq, a.fstate,
                              base + 2ull * gridDim.x, seq + 1);
  pdl_trigger();
}

// ---- batched sort: independent DialSort steps overlapped on disjoint CTA groups --------------
// One launch sorts up to kBatchMax batches (each: keys[n] -> out, H) on L groups of Gg CTAs:
// group g sorts batches g, g + L, g + 2L, ... one after another, each as a whole DialSort step
// on its own virtual grid (sort_step with vg = {Gg, rank in the group}) with its own workspace
// (a context lane: rows, counters, barrier, status).  A step alternates HBM-bound phases
// (ingestion, projection) with phases that leave HBM idle (flush, grid barrier, merge): with
// the groups out of phase, one group's ingestion or projection runs while another merges, so
// HBM stays busy (c2 on one B200: 27.7 us per batch on the whole grid, 17.6 us per batch on four
// concurrent groups of 37 CTAs).  The groups drift out of phase by themselves (an explicit
// start stagger — group g waiting for group g - 1's first ingestion — measured slower: 20.9
// vs 17.6 us).  After each batch a group passes one more barrier of its own (every CTA finished
// the batch before the group's next one reuses the workspace: the boundary a kernel launch gives
// the single-step kernel).
constexpr uint32_t kBatchMax = 64;
struct BatchArgs {
  uint32_t nb, L, Gg;
  const void* keys[kBatchMax];
  uint64_t n[kBatchMax];
  int32_t* out[kBatchMax];
  int32_t key_base[kBatchMax];
  ScanArgs a[kBatchMax];  // per batch: its group's workspace, parities, epochs, barrier base
};
// (KB = 2: the hierarchical path's universe blocks — uint16 keys, sizes and offsets on the device)
template <int FMT, int KB = 4>
__global__ void __launch_bounds__(1024, 1) k_sort_batch(const __grid_constant__ BatchArgs B) {
  extern __shared__ __align__(128) uint32_t sh[];
  __shared__ uint64_t red64[34];
  __shared__ uint32_t wsum[32];
  __shared__ unsigned long long s_fs[2];
  pdl_wait();
  const uint32_t g = blockIdx.x / B.Gg;
  const VGrid vg{B.Gg, blockIdx.x % B.Gg};
  FusedState* fs = B.a[g].fstate;  // the group's workspace lane
  fused_state_read(fs, s_fs);
  const unsigned long long base = s_fs[0];
  const uint32_t seq = (uint32_t)s_fs[1];
  const uint32_t steps = g < B.nb ? (B.nb - g + B.L - 1) / B.L : 0u;  // this group's batches
  uint32_t k = 0;  // this group's steps so far
  for (uint32_t j = g; j < B.nb; j += B.L, ++k) {
    const ScanArgs& a = B.a[j];
    phase_mark(a.pt, -1);  // (debug stamps: the group's last step survives)
    const unsigned long long bj = base + 3ull * B.Gg * k;
    sort_step<FMT, KB>(B.keys[j], B.n[j], a, B.out[j], B.key_base[j], vg, sh, red64, wsum, bj, seq + k,
                       k == 0 ? fs : nullptr, base + 3ull * B.Gg * steps, seq + steps);
    grid_barrier_mono(a.bar64, bj + 3ull * B.Gg);  // batch done by every CTA of the group
  }
  pdl_trigger();
}

}  // namespace ds

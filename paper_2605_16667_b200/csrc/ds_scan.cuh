// ds_scan.cuh — sub-histogram merge and the GPU's write-offset scan.
//
// The merge sums the per-CTA partial histogram rows written by the ingestion phase (the
// additive merge, lem:crn lifted to whole histograms) into H.  The scan computes
// the exclusive prefix P[k] = Σ_{j<k} H[j]: the parallel write-offset step north_star asks
// for (the paper's own substrates emit sequentially and need no prefix sum, P:13-14,
// P:2013-2016).  It also emits the output-tile index `tfb` (tile t's first position t*T
// lies in bin tfb[t]) that gives each expand CTA its first bin in O(1).
//
// Both run inside persistent, co-resident grids as a two-level reduce-then-scan separated by
// grid barriers — no decoupled look-back chain: every CTA owns a contiguous range of 512-bin
// tiles; phase A writes H for its range and its range total; phase B derives its range
// offset from all range totals (<= a few hundred values) and scans its tiles into P.
#pragma once
#include "ds_common.cuh"

namespace ds {

constexpr uint32_t kTileBins = 512;  // bins per scan tile

// Sense-reversing grid barrier for a co-resident grid (all CTAs participate every time).
// Self-resetting: `count` returns to 0 at every barrier, `gen` only grows.
struct GridBar {
  unsigned int count;
  unsigned int gen;
};
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void grid_barrier(GridBar* gb) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned g = ld_acquire_u32(&gb->gen);
    unsigned old;
    // arrive with release semantics (orders this CTA's prior writes, made visible to thread 0
    // by __syncthreads, before the arrival), observe the release with acquire loads
    asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(old) : "l"(&gb->count) : "memory");
    if (old == gridDim.x - 1) {
      asm volatile("st.relaxed.gpu.global.u32 [%0], 0;" ::"l"(&gb->count) : "memory");
      asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(&gb->gen) : "memory");
    } else {
      while (ld_acquire_u32(&gb->gen) == g) {
      }
    }
  }
  __syncthreads();
}

struct ScanArgs {
  const uint32_t* partials;  // [C][ldw] rows (C > 0), or nullptr
  uint32_t C, ldw;
  int pack16;                // partial words hold 2 x 16-bit bins (2w, 2w+1)
  const uint32_t* Hsrc;      // C == 0: H is read from here
  uint32_t* ovfH;            // packed-overflow side histogram (added and cleared if flagged)
  uint32_t U;
  uint32_t* H;               // C > 0: merged H written here (user H or workspace)
  // Multi-GPU (dialsort_histogram_scatter_async): instead of H, bin k of universe slice
  // s = k / peerL goes straight to peer rank s's receive buffer, slot peerRank:
  // Hpeer[s][peerRank * peerL + k - s * peerL] (P2P stores over NVLink / NVSwitch)
  uint32_t* const* Hpeer;    // device array of G device pointers, or null
  uint32_t peerL, peerRank;
  uint32_t bin_base;         // universe bin of this launch's bin 0 (hierarchical blocks), for Hpeer
  int hist_only;             // k_sort_fused: stop after the merge (H only, no projection)
  const uint32_t* enc;       // coded domains (Proposition 2): phi of a 1-byte item, device uint32[256], or null
  const int32_t* dec;        // coded domains: phi^-1, the value emitted for code k (device int32[U]), or null
  int do_scan;
  uint32_t* P;               // [U+1] exclusive prefix
  uint64_t* range_tot;       // [gridDim] per-CTA range totals
  uint32_t* tfb;             // [ntiles_out] first bin of each output tile
  uint64_t T, ntiles_out;
  uint64_t n_expected;       // exact: ΣH must equal; else capacity
  int exact;
  uint64_t* d_total;         // nullable, receives ΣH
  uint64_t* ws_total;        // workspace scalar read by k_expand
  DevStatus* st;
  GridBar* bar;
  uint32_t epoch;
  PhaseTimes* pt;            // nullable debug timing
  uint32_t* tsums;           // [C][ntiles] per-row tile sums (fused path), or nullptr
  // single-kernel sort (k_sort_fused) only:
  int fused;                 // k_sort_fused flush (row formats, tile sums in shared memory, owner totals)
  uint32_t ctr_stride;       // words between consecutive L2 counters / flags (one line each)
  uint32_t ldr;              // words between partial rows (row format may differ from the smem histogram)
  int nib4;                  // partial rows hold 4-bit counts (8 bins per word); counts >= 16 in Hx
  uint32_t* Hx;              // [U] exception histogram of the 4-bit rows (zero on entry)
  uint32_t* Hx_clear;        // the other parity's Hx, zeroed for the next launch
  const uint64_t* d_n;       // nullable: key count on the device (hierarchical blocks); then
  const uint64_t* d_off;     //   keys and out start at *d_off and n_expected = *d_n
  const uint64_t* d_koff;    // nullable: the keys start at *d_koff instead (sampled partition)
  uint32_t* own_red;         // [G x ctr_stride] per-owner totals (tiles of CTA b) reduced during the flush
  uint32_t* own_clear;       // the other parity's own_red, zeroed for the next launch
  uint32_t* own_alt;         // [G] owner totals of the overflow fallback path
  uint32_t* ready_clear;     // k_sort_fused: the other parity's ready flags, zeroed for the next launch
  uint32_t* ready;           // [ntiles] per-tile "P published" flags (= epoch)
  unsigned long long* bar64; // monotonic grid-barrier counter (= &fstate->bar)
  unsigned long long bar_base;  // its value at the step's start (derived on the device, see FusedState)
  // two-parity workspaces of the fused step; the parity, the epoch and bar_base of a step are
  // derived ON THE DEVICE from FusedState (so a captured CUDA graph replays correctly)
  uint32_t* own_base;        // [2][kFOwnSlots * ctr_stride] owner counters, then [kFOwnSlots] own_alt
  uint32_t* ready_base;      // [2][kFTileSlots] per-tile ready flags
  uint32_t* Hx_base;         // [2][kSmem16MaxBins] 4-bit rows' exception histograms
  struct FusedState* fstate;
};

// Device-side sequencing of the fused step's launches on one workspace: the monotonic barrier
// counter, its value at the start of the next launch and the steps run so far (parity = seq & 1,
// epoch = seq mod 2^24 + 1).  Each launch reads base and seq at its start (after
// griddepcontrol.wait); once its first grid barrier shows every CTA has read them, CTA 0 advances
// them to the launch's end values (the next launch reads them after this grid completes).  No
// host-side bookkeeping: a captured launch replays correctly and a launch that never ran leaves
// the state as it was.
struct FusedState {
  unsigned long long bar;   // monotonic barrier counter
  unsigned long long base;  // bar at the start of the next launch
  unsigned int seq;         // fused steps run so far
  unsigned int pad;
};

// H[bin] = h, or — multi-GPU histogram — the owner rank's slot of this rank (see Hpeer).
__device__ __forceinline__ void store_H(const ScanArgs& a, uint32_t bin, uint32_t h) {
  if (a.Hpeer) {
    const uint32_t gb = a.bin_base + bin, sl = gb / a.peerL;
    a.Hpeer[sl][(uint64_t)a.peerRank * a.peerL + (gb - sl * a.peerL)] = h;
  } else {
    a.H[bin] = h;
  }
}


// Monotonic grid barrier (measured 1.25 us vs 2.0 us for counter + generation on B200,
// profiles/r01_barrier_bench.txt): each CTA arrives with one release atomic on a 64-bit
// counter that only grows, and waits until it reaches `target` = base + (j + 1) * gridDim
// for the launch's j-th barrier.  The host advances `base` by the number of barriers a launch
// reserves; a launch that skips a reserved barrier arrives without waiting (barrier_skip), so
// the counter always ends a launch at base + reserved * gridDim.
__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void grid_barrier_mono(unsigned long long* cnt, unsigned long long target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(cnt) : "memory");
    while (ld_acquire_u64(cnt) < target) {
    }
  }
  __syncthreads();
}
// The same, with `side()` run by thread 32 while thread 0 waits (uniform set-up work for the
// next phase that would otherwise be repeated by all 32 warps; its smem results are visible
// after the barrier's closing __syncthreads).
template <class F>
__device__ __forceinline__ void grid_barrier_mono_side(unsigned long long* cnt, unsigned long long target, F side) {
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(cnt) : "memory");
    while (ld_acquire_u64(cnt) < target) {
    }
  } else if (threadIdx.x == 32) {
    side();
  }
  __syncthreads();
}
__device__ __forceinline__ void barrier_skip(unsigned long long* cnt) {
  if (threadIdx.x == 0) asm volatile("red.relaxed.gpu.global.add.u64 [%0], 1;" ::"l"(cnt) : "memory");
}

// Final size / overflow checks and totals, by the CTA owning the last tile.
__device__ __forceinline__ void scan_finish(const ScanArgs& a, uint64_t total) {
  a.P[a.U] = (uint32_t)(total > 0xffffffffull ? 0xffffffffull : total);
  unsigned flags = 0;
  if (total > 0xffffffffull) flags |= FLAG_OVERFLOW;
  if (a.exact ? (total != a.n_expected) : (total > a.n_expected)) flags |= FLAG_SIZE;
  if (flags) atomicOr(&a.st->flags, flags);
  a.st->last_total = total;
  if (a.d_total) *a.d_total = total;
  *a.ws_total = total;
}

// Tiles [tb0, tb1) of CTA b in a grid of G over ntiles (contiguous ranges).
__device__ __forceinline__ void my_tiles(uint32_t ntiles, uint32_t& tb0, uint32_t& tb1, VGrid vg = vgrid_hw()) {
  const uint32_t G = vg.G, b = vg.b;
  tb0 = (uint32_t)((uint64_t)ntiles * b / G);
  tb1 = (uint32_t)((uint64_t)ntiles * (b + 1) / G);
}

// The CTA whose my_tiles range holds tile t.
__device__ __forceinline__ uint32_t owner_of(uint32_t t, uint32_t ntiles, uint32_t G) {
  uint32_t b = (uint32_t)((uint64_t)t * G / ntiles);  // ntiles b / G <= t
  while (b + 1 < G && (uint32_t)((uint64_t)ntiles * (b + 1) / G) <= t) ++b;
  return b;
}

// Sum of H over one tile (phase A when H is given).
__device__ __forceinline__ uint64_t sum_tile(const uint32_t* H, uint32_t U, uint32_t tile, uint64_t* red) {
  uint64_t s = 0;
  for (uint32_t j = threadIdx.x; j < kTileBins; j += blockDim.x) {
    const uint64_t bin = (uint64_t)tile * kTileBins + j;
    if (bin < U) s += __ldcg(H + bin);
  }
  return block_sum<uint64_t>(s, red);
}

// Phase B for one tile: P[bin] = offset + exclusive prefix within the tile; tfb scatter.
// Requires blockDim.x >= kTileBins.  Returns offset + tile total.
__device__ __forceinline__ uint64_t scan_tile(const ScanArgs& a, const uint32_t* H, uint32_t tile, uint64_t offset,
                                              uint64_t* red) {
  const uint64_t bin = (uint64_t)tile * kTileBins + threadIdx.x;
  const bool own = threadIdx.x < kTileBins && bin < a.U;
  const uint64_t h = own ? __ldcg(H + bin) : 0;
  uint64_t tile_total;
  const uint64_t ex = block_excl_scan<uint64_t>(h, tile_total, red);
  if (own) {
    const uint64_t pk = offset + ex;
    a.P[bin] = (uint32_t)pk;
    if (a.tfb && h > 0) {  // output tiles whose first position t*T falls in [pk, pk + h) start in this bin
      const uint64_t t0 = (pk + a.T - 1) / a.T, t1 = (pk + h - 1) / a.T;
      for (uint64_t t = t0; t <= t1 && t < a.ntiles_out; ++t) a.tfb[t] = (uint32_t)bin;
    }
  }
  return offset + tile_total;
}

// Phase B for a co-resident grid (called by every CTA, all threads), after phase A left
// `range` = this CTA's range total.
__device__ __forceinline__ void scan_phase_b(const ScanArgs& a, const uint32_t* H, uint32_t tb0, uint32_t tb1,
                                             uint64_t range, uint64_t* red) {
  if (threadIdx.x == 0) a.range_tot[blockIdx.x] = range;
  grid_barrier(a.bar);
  phase_mark(a.pt, 6);
  // this CTA's offset = Σ range totals of lower CTAs
  uint64_t s = 0;
  for (uint32_t j = threadIdx.x; j < blockIdx.x; j += blockDim.x) s += __ldcg(a.range_tot + j);
  uint64_t off = block_sum<uint64_t>(s, red);
  for (uint32_t t = tb0; t < tb1; ++t) off = scan_tile(a, H, t, off, red);
  if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) scan_finish(a, off);
}

// Standalone scan of a given H (global path, reconstruct API): persistent co-resident grid.
__global__ void __launch_bounds__(kTileBins) k_scan(ScanArgs a) {
  __shared__ uint64_t red[34];
  pdl_wait();
  const uint32_t ntiles = (a.U + kTileBins - 1) / kTileBins;
  uint32_t tb0, tb1;
  my_tiles(ntiles, tb0, tb1);
  uint64_t range = 0;
  for (uint32_t t = tb0; t < tb1; ++t) range += sum_tile(a.Hsrc, a.U, t, red);
  scan_phase_b(a, a.Hsrc, tb0, tb1, range, red);
  pdl_trigger();
}

// Range count on a device histogram: Σ_{k=a}^{b} H[k].
__global__ void k_range_count(const uint32_t* __restrict__ H, uint32_t a, uint32_t b,
                              unsigned long long* out) {
  __shared__ unsigned long long red[33];
  pdl_wait();
  unsigned long long s = 0;
  for (uint64_t k = (uint64_t)a + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; k <= b;
       k += (uint64_t)gridDim.x * blockDim.x)
    s += H[k];
  s = block_sum<unsigned long long>(s, red);
  if (threadIdx.x == 0) atomicAdd(out, s);
}

}  // namespace ds

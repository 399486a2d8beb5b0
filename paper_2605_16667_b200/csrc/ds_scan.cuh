// ds_scan.cuh — sub-histogram merge + the GPU's write-offset scan.
//
// k_reduce_scan sums the per-CTA partial rows written by k_hist_smem (the additive merge,
// lem:crn lifted to whole histograms) into H, and — when a projection follows —
// computes the exclusive prefix P[k] = Σ_{j<k} H[j] with a single-pass decoupled look-back
// across bin tiles.  P is the parallel write-offset step north_star asks for; the paper's
// own substrates need no prefix sum because they emit sequentially.
// It also emits the output-tile index `tfb` (tile t's first position t*T lies in bin
// tfb[t]) that lets each expand CTA find its bins in O(1).
#pragma once
#include "ds_common.cuh"

namespace ds {

constexpr int kScanThreads = 512;
constexpr int kScanWords = 256;  // partial-row words per tile (512 bins packed, 256 bins u32)

struct ScanArgs {
  const uint32_t* partials;  // [C][ldw] rows, or nullptr when C == 0
  uint32_t C, ldw;
  int pack16;                // partial words hold 2 x 16-bit bins
  const uint32_t* Hsrc;      // C == 0: read H from here
  const uint32_t* ovfH;      // added (and cleared) iff st->ovf_epoch == epoch
  uint32_t* ovfH_mut;
  uint32_t U;
  uint32_t* Hout;            // nullable: write merged H
  int do_scan;
  uint32_t* P;               // [U+1] exclusive prefix (do_scan)
  uint64_t* status;          // [num tiles] look-back status
  uint32_t* tfb;             // [ntiles_out] first bin of each output tile (do_scan)
  uint64_t T;                // output tile size (positions)
  uint64_t ntiles_out;
  uint64_t n_expected;       // exact: ΣH must equal; else capacity
  int exact;
  uint64_t* d_total;         // nullable, receives ΣH
  uint64_t* ws_total;        // workspace scalar read by k_expand
  DevStatus* st;
  uint32_t epoch;
};

__global__ void __launch_bounds__(kScanThreads) k_reduce_scan(ScanArgs a) {
  __shared__ uint32_t part[kScanThreads / 32][2 * kScanWords];  // per-warp bin sums (32 KB)
  __shared__ uint64_t red[34];
  __shared__ uint64_t s_excl;
  pdl_wait();

  const uint32_t tile = blockIdx.x;
  const uint32_t bins_per_tile = a.pack16 ? 2 * kScanWords : kScanWords;
  const uint64_t bin0 = (uint64_t)tile * bins_per_tile;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const bool use_ovf = a.ovfH != nullptr && *(volatile unsigned*)&a.st->ovf_epoch == a.epoch;

  // ---- merge: H[bin0 + j] for j < bins_per_tile; thread j owns bin j -------------------
  uint64_t hval = 0;
  if (a.C > 0) {
    // Warp w sums rows w, w+nw, ...; lane l covers words [8l, 8l+8) of the tile.
    const uint64_t word0 = (uint64_t)tile * kScanWords + 8 * lane;
    uint32_t acc[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) acc[j] = 0;
    const uint32_t Wtot = a.pack16 ? (a.U + 1) / 2 : a.U;
    if (word0 < Wtot) {
      for (uint32_t r = warp; r < a.C; r += nw) {
        const uint4* p = reinterpret_cast<const uint4*>(a.partials + (uint64_t)r * a.ldw + word0);
        uint4 x0 = __ldcg(p), x1 = __ldcg(p + 1);
        uint32_t w[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
        if (a.pack16) {
#pragma unroll
          for (int j = 0; j < 8; ++j) { acc[2 * j] += w[j] & 0xffffu; acc[2 * j + 1] += w[j] >> 16; }
        } else {
#pragma unroll
          for (int j = 0; j < 8; ++j) acc[j] += w[j];
        }
      }
    }
    const int per = a.pack16 ? 16 : 8;
    for (int j = 0; j < per; ++j) part[warp][per * lane + j] = acc[j];
    __syncthreads();
    if (threadIdx.x < bins_per_tile) {
      uint64_t sum = 0;
      for (int w = 0; w < nw; ++w) sum += part[w][threadIdx.x];
      hval = sum;
    }
  }
  const uint64_t bin = bin0 + threadIdx.x;
  const bool own = threadIdx.x < bins_per_tile && bin < a.U;
  if (own) {
    if (a.C == 0) hval = a.Hsrc[bin];
    if (use_ovf) {
      hval += a.ovfH[bin];
      a.ovfH_mut[bin] = 0;  // consumed: ovfH is zero again for the next call
    }
  } else {
    hval = 0;
  }
  if (own && a.Hout) a.Hout[bin] = (uint32_t)(hval > 0xffffffffull ? 0xffffffffull : hval);
  if (!a.do_scan) {
    pdl_trigger();
    return;
  }

  // ---- tile scan + decoupled look-back ---------------------------------------------------
  uint64_t tile_total;
  uint64_t excl_in_tile = block_excl_scan<uint64_t>(hval, tile_total, red);
  if (warp == 0) {
    uint64_t excl = 0;
    if (tile == 0) {
      if (lane == 0) lb_store(a.status, lb_pack(a.epoch, LB_FLAG_INC, tile_total));
    } else {
      if (lane == 0) lb_store(a.status + tile, lb_pack(a.epoch, LB_FLAG_AGG, tile_total));
      excl = lookback(a.status, tile, a.epoch);
      if (lane == 0) lb_store(a.status + tile, lb_pack(a.epoch, LB_FLAG_INC, excl + tile_total));
    }
    if (lane == 0) s_excl = excl;
  }
  __syncthreads();
  const uint64_t pk = s_excl + excl_in_tile;  // P[bin]
  if (own) {
    a.P[bin] = (uint32_t)pk;
    // Output tiles whose first position t*T falls in [pk, pk + hval) start in this bin.
    if (hval > 0) {
      uint64_t t0 = (pk + a.T - 1) / a.T, t1 = (pk + hval - 1) / a.T;
      if (t1 >= a.ntiles_out) t1 = a.ntiles_out - 1;
      for (uint64_t t = t0; t <= t1 && t < a.ntiles_out; ++t) a.tfb[t] = (uint32_t)bin;
    }
  }
  const uint32_t ntiles = (a.U + bins_per_tile - 1) / bins_per_tile;
  if (tile == ntiles - 1 && threadIdx.x == 0) {
    const uint64_t total = s_excl + tile_total;
    a.P[a.U] = (uint32_t)(total > 0xffffffffull ? 0xffffffffull : total);
    unsigned flags = 0;
    if (total > 0xffffffffull) flags |= FLAG_OVERFLOW;
    if (a.exact ? (total != a.n_expected) : (total > a.n_expected)) flags |= FLAG_SIZE;
    if (flags) atomicOr(&a.st->flags, flags);
    a.st->last_total = total;
    if (a.d_total) *a.d_total = total;
    *a.ws_total = total;
  }
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

// ds_common.cuh — shared device helpers of the DialSort CUDA path (sm_100a only).
// Nothing here is shared with oracle/ (the two are independent by construction).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#ifndef __CUDACC__
#error "CUDA only"
#endif

namespace ds {

constexpr uint32_t FULL = 0xffffffffu;

// The grid a CTA cooperates with: the launch's own grid, or — in the batched sort kernel
// (k_sort_batch, ds_fused.cuh) — one group of its CTAs sorting a batch on its own ("virtual
// grid" of G CTAs, this CTA's rank b).  Device helpers take it as their last argument.
struct VGrid {
  uint32_t G, b;
};
__device__ __forceinline__ VGrid vgrid_hw() { return VGrid{gridDim.x, blockIdx.x}; }

// Deferred device error state of one context (dialsort_sync reads and clears it).
struct DevStatus {
  unsigned long long bad_count;   // keys outside [0,U)
  unsigned long long first_bad;   // min over bad keys of (index << 32) | (uint32)key
  unsigned long long last_total;  // ΣH of the most recent scan
  unsigned int flags;             // bit0 size error, bit1 overflow
  unsigned int ovf_epoch;         // epoch of the last call whose packed-u16 histogram overflowed
};
constexpr unsigned FLAG_SIZE = 1u, FLAG_OVERFLOW = 2u;

__device__ __forceinline__ void record_bad(DevStatus* st, uint64_t idx, uint32_t key) {
  atomicAdd(&st->bad_count, 1ull);
  atomicMin(&st->first_bad, (unsigned long long)((idx << 32) | (uint64_t)key));
}

// Programmatic dependent launch (PDL): wait for the producer grid / let dependents launch.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Streaming 128-bit loads/stores.  Keys are read exactly once and outputs written exactly
// once, so both are marked L2 evict-first: the L2-resident working set of the step (partial
// histograms, H, P) keeps its lines while 40+ MB stream past it.
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ int4 ld_stream4(const int4* p, uint64_t pol) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.s32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ int4 ld_stream4(const int4* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ void st_stream4(int4* p, int4 v, uint64_t pol) {
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.v4.s32 [%0], {%1,%2,%3,%4}, %5;" ::"l"(p), "r"(v.x),
               "r"(v.y), "r"(v.z), "r"(v.w), "l"(pol) : "memory");
}
__device__ __forceinline__ void st_stream4(int4* p, int4 v) {
  asm volatile("st.global.L1::no_allocate.v4.s32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y),
               "r"(v.z), "r"(v.w) : "memory");
}
__device__ __forceinline__ uint32_t umax4(int4 v) {
  return max(max((uint32_t)v.x, (uint32_t)v.y), max((uint32_t)v.z, (uint32_t)v.w));
}

// ---- mbarrier + TMA bulk copy (cp.async.bulk, SASS UBLKCP) ---------------------------------
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}
// Wait with a suspend-time hint: the thread sleeps in hardware until the phase completes
// (or the hint elapses) instead of spinning.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAITS_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
      "@!P1 bra WAITS_%=;\n"
      "}\n" ::"r"(smem_addr(bar)),
      "r"(parity), "r"(1000000u)
      : "memory");
}
// Bulk copy of `bytes` (multiple of 16, 16-byte aligned ends) global -> shared, completing
// on `bar` (transaction bytes), with an L2 evict-first hint: keys are streamed once.
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(pol)
      : "memory");
}

// ---- debug phase timing (DIALSORT_PHASE_TIMING=1): per-CTA %globaltimer stamps ------------
// Plain stores by thread 0 of each CTA (no same-address atomics, which would serialise and
// distort the timeline); the host reduces them (dialsort_debug_phase_ns / _cta).
constexpr int kPhaseMaxCtas = 1024;
constexpr int kPhaseSlots = 17;  // [0] = CTA start, [1 + i] = phase i (i < 16)
struct PhaseTimes {
  unsigned long long stamp[kPhaseMaxCtas][kPhaseSlots];
};
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// Stamps are compiled in only with -DDIALSORT_PHASE_MARKS=1 (the tools' libdialsort_phase.so):
// even a disabled mark costs every warp its test, ~4% of the fused kernel's instructions.
#ifndef DIALSORT_PHASE_MARKS
#define DIALSORT_PHASE_MARKS 0
#endif
__device__ __forceinline__ void phase_mark(PhaseTimes* pt, int i) {
  if constexpr (DIALSORT_PHASE_MARKS) {
    if (pt && threadIdx.x == 0 && blockIdx.x < kPhaseMaxCtas) pt->stamp[blockIdx.x][i + 1] = gtimer();
  }
}

// Fire-and-forget global add (RED.ADD.U32 in SASS).
__device__ __forceinline__ void red_add_u32(uint32_t* p, uint32_t v) {
  asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// ---- the warp CRN (def:crn_level P:896-915, lem:crn P:951-962) ----------------------------
// Multiset reading R1: the active lanes `mask` are grouped by equal key with one
// equality-only instruction (MATCH.ANY); the lowest lane of each group is its leader and
// carries the group's total count.  Returns the group mask of the calling lane.
// Must be called by exactly the lanes in `mask`.
__device__ __forceinline__ uint32_t crn_group(uint32_t mask, uint32_t key) {
  return __match_any_sync(mask, key);
}
__device__ __forceinline__ bool crn_is_leader(uint32_t group) {
  return (threadIdx.x & 31) == (uint32_t)(__ffs(group) - 1);
}

// Block-wide reductions / scans (blockDim multiple of 32, <= 1024).
template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
  return v;
}

template <typename T>
__device__ __forceinline__ T block_sum(T v, T* red /* >= 32 slots */) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  v = warp_sum(v);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  T r = lane < nw ? red[lane] : T(0);
  r = warp_sum(r);
  return r;
}

// Inclusive warp scan.
template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T t = __shfl_up_sync(FULL, v, o);
    if (lane >= o) v += t;
  }
  return v;
}

// Exclusive block scan; returns the exclusive prefix of the calling thread and the block total.
template <typename T>
__device__ __forceinline__ T block_excl_scan(T v, T& total, T* red /* >= 33 slots */) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  T inc = warp_incl_scan(v);
  __syncthreads();
  if (lane == 31) red[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    T w = lane < nw ? red[lane] : T(0);
    T wi = warp_incl_scan(w);
    red[lane] = wi - w;  // exclusive warp offsets
    if (lane == 31) red[32] = wi;
  }
  __syncthreads();
  total = red[32];
  return red[warp] + inc - v;
}

// Decoupled look-back tile status: [epoch:24 | flag:2 | value:38].
constexpr uint64_t LB_VALUE_BITS = 38;
constexpr uint64_t LB_VALUE_MASK = (1ull << LB_VALUE_BITS) - 1;
constexpr uint64_t LB_FLAG_AGG = 1, LB_FLAG_INC = 2;
__device__ __forceinline__ uint64_t lb_pack(uint32_t epoch, uint64_t flag, uint64_t value) {
  value = value > LB_VALUE_MASK ? LB_VALUE_MASK : value;
  return ((uint64_t)(epoch & 0xffffffu) << 40) | (flag << LB_VALUE_BITS) | value;
}
__device__ __forceinline__ void lb_store(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t lb_load(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Warp-cooperative look-back for tile `tile` (> 0), called by all 32 lanes of one warp.
// Returns the exclusive prefix of the tile (sum of all preceding tile aggregates).
__device__ __forceinline__ uint64_t lookback(const uint64_t* status, uint32_t tile, uint32_t epoch) {
  const int lane = threadIdx.x & 31;
  uint64_t excl = 0;
  int64_t base = (int64_t)tile - 1;  // newest predecessor not yet consumed
  const uint32_t ep = epoch & 0xffffffu;
  while (base >= 0) {
    int64_t t = base - lane;  // lane 0 = nearest predecessor
    uint64_t s = 0;
    uint32_t flag = LB_FLAG_INC;  // lanes past tile 0 behave like an inclusive 0
    if (t >= 0) {
      do {
        s = lb_load(status + t);
        flag = ((uint32_t)(s >> 40) == ep) ? (uint32_t)((s >> LB_VALUE_BITS) & 3) : 0u;
      } while (flag == 0);
    }
    uint64_t val = (t >= 0) ? (s & LB_VALUE_MASK) : 0;
    uint32_t inc_mask = __ballot_sync(FULL, flag == LB_FLAG_INC);
    int first_inc = __ffs(inc_mask) - 1;  // nearest predecessor with an inclusive prefix
    uint64_t contrib = (inc_mask == 0 || lane <= first_inc) ? val : 0;
    excl += warp_sum(contrib);
    if (inc_mask) break;
    base -= 32;
  }
  return excl;
}

}  // namespace ds

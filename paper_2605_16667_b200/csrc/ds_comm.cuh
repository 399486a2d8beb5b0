// ds_comm.cuh — device side of the multi-GPU exchange over peer
// memory: one process (or one context) per GPU, a symmetric workspace per rank mapped into
// every other rank (CUDA IPC, or plain pointers inside one process), epoch-tagged completion
// flags instead of host barriers.
//
//   histogram exchange (c2 / c4 at G > 1): the local histogram's universe slice s is stored
//     into rank s's receive slots (the reduce-scatter of the local histograms: lem:crn lifted
//     to whole histograms; the WSE-3 "tile k owns H[k]" idea with GPUs as owners,
//     P:1449-1459), then rank s sums its G slots and projects its slice with key_base s L.
//   radix exchange (c5 at G > 1): top-digit histograms all-gathered, contiguous top-byte
//     ranges per rank balanced by counts, keys split by destination and stored straight into
//     the owners' receive buffers (the all-to-all), then a local LSD sort (
//     "distribute the n keys across k ingestion lanes", thm:par proof P:678-680).
//
// Memory model: a producer kernel's peer stores complete with the kernel; the next kernel on
// the stream (k_comm_signal) issues fence.acq_rel.sys and a release store of the call's epoch
// into the consumer's flag; the consumer polls with ld.acquire.sys.  Flags hold the epoch of
// the last call (never reset) and every buffer has two parities, so a rank one call ahead
// never overwrites what a slower peer still reads (a call cannot complete before every peer
// reached it, which bounds the lead to one call).  Every wait gives up after ~kCommTimeoutNs
// and reports DIALSORT_E_COMM instead of hanging the GPU.
#pragma once
#include "ds_common.cuh"

namespace ds {

constexpr uint32_t kCommMaxRanks = 8;
constexpr uint32_t kFlagHist = 0, kFlagTotals = 1, kFlagRhist = 2, kFlagRkeys = 3, kFlagKinds = 4;
constexpr uint64_t kCommTimeoutNs = 20ull * 1000 * 1000 * 1000;  // 20 s
constexpr unsigned FLAG_COMM = 4u;                                // DevStatus.flags: a wait timed out

// Byte layout of a rank's symmetric workspace (identical on every rank: same G, max_U, cap).
struct CommLayout {
  uint64_t flags;   // [2 parity][kFlagKinds][kCommMaxRanks] u32, 32-byte stride
  uint64_t tot;     // [2][kCommMaxRanks] u64 slice totals (all-gathered)
  uint64_t rhist;   // [2][kCommMaxRanks][256] u32 top-digit histograms (all-gathered)
  uint64_t recv;    // [2][G * Lmax] u32 histogram slots (slot src at src * L)
  uint64_t rkeys;   // [2][cap] u32 radix receive buffers
  uint64_t bytes;
  uint32_t Lmax;
  uint64_t cap;
};
__host__ __device__ inline uint64_t comm_flag_off(const CommLayout& l, uint32_t parity, uint32_t kind, uint32_t src) {
  return l.flags + 32ull * ((parity * kFlagKinds + kind) * kCommMaxRanks + src);
}

// Device view of one rank's communicator (passed by value to the kernels).
struct CommDev {
  char* ws[kCommMaxRanks];  // every rank's workspace base, mapped into this process (ws[rank] = own)
  CommLayout lay;
  uint32_t G, rank, epoch, parity;
};

__device__ __forceinline__ uint32_t ld_acquire_sys_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys_u32(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Thread t < G waits until rank t's flag `kind` of this call holds the call's epoch.  Returns
// false (and records FLAG_COMM) on timeout.  Called by whole CTAs (ends with __syncthreads).
__device__ __forceinline__ bool comm_wait_all(const CommDev& c, uint32_t kind, DevStatus* st) {
  __shared__ int s_ok;
  if (threadIdx.x == 0) s_ok = 1;
  __syncthreads();
  if (threadIdx.x < c.G) {
    const uint32_t* f = reinterpret_cast<const uint32_t*>(c.ws[c.rank] + comm_flag_off(c.lay, c.parity, kind, threadIdx.x));
    const unsigned long long t0 = gtimer();
    while (ld_acquire_sys_u32(f) != c.epoch) {
      if (gtimer() - t0 > kCommTimeoutNs) {
        atomicOr(&st->flags, FLAG_COMM);
        s_ok = 0;
        break;
      }
      __nanosleep(128);
    }
  }
  __syncthreads();
  return s_ok != 0;
}

// This rank's flag `kind` := epoch in every peer's workspace (after everything this stream
// did before: the preceding kernels' peer stores).
__global__ void k_comm_signal(CommDev c, uint32_t kind) {
  pdl_wait();
  if (threadIdx.x < c.G) {
    asm volatile("fence.acq_rel.sys;" ::: "memory");
    st_release_sys_u32(reinterpret_cast<uint32_t*>(c.ws[threadIdx.x] + comm_flag_off(c.lay, c.parity, kind, c.rank)),
                       c.epoch);
  }
  pdl_trigger();
}

// Owner step of the histogram exchange: wait for every source's slot, H_slice[j] = Σ_src
// recv[src L + j]; the slice total is reduced across CTAs (RED + ticket) and the last CTA
// publishes it into every peer's totals (all-gather) and raises kFlagTotals.
// ws_tot: 2 x u64 workspace scalars (total, ticket) of this rank, zero on entry (cleared by the
// last CTA for the next call).
__global__ void __launch_bounds__(256) k_comm_slice_sum(CommDev c, uint32_t L, uint32_t* __restrict__ Hs,
                                                        unsigned long long* ws_tot, DevStatus* st) {
  __shared__ unsigned long long red[33];
  __shared__ bool s_last;
  pdl_wait();
  const bool ok = comm_wait_all(c, kFlagHist, st);
  const uint32_t* recv =
      reinterpret_cast<const uint32_t*>(c.ws[c.rank] + c.lay.recv) + (uint64_t)c.parity * c.G * c.lay.Lmax;
  unsigned long long s = 0;
  if (ok) {
    for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < L; j += gridDim.x * blockDim.x) {
      uint32_t h = 0;
      for (uint32_t src = 0; src < c.G; ++src) h += __ldcg(recv + (uint64_t)src * L + j);  // (after the acquire)
      Hs[j] = h;
      s += h;
    }
  }
  s = block_sum<unsigned long long>(s, red);
  if (threadIdx.x == 0) {
    atomicAdd(&ws_tot[0], s);
    __threadfence();
    s_last = atomicAdd(&ws_tot[1], 1ull) == gridDim.x - 1;
  }
  __syncthreads();
  __shared__ unsigned long long s_total;
  if (s_last && threadIdx.x == 0) {
    __threadfence();
    s_total = *reinterpret_cast<volatile unsigned long long*>(&ws_tot[0]);
    ws_tot[0] = 0;  // (cleared for the next call: every CTA has added)
    ws_tot[1] = 0;
  }
  __syncthreads();
  if (s_last && threadIdx.x < c.G) {
    const unsigned long long total = s_total;
    unsigned long long* dst =
        reinterpret_cast<unsigned long long*>(c.ws[threadIdx.x] + c.lay.tot) + (uint64_t)c.parity * kCommMaxRanks + c.rank;
    *reinterpret_cast<volatile unsigned long long*>(dst) = total;
    asm volatile("fence.acq_rel.sys;" ::: "memory");
    st_release_sys_u32(reinterpret_cast<uint32_t*>(c.ws[threadIdx.x] + comm_flag_off(c.lay, c.parity, kFlagTotals, c.rank)),
                       c.epoch);
  }
  pdl_trigger();
}

// Wait for every rank's slice total; d_count = own total, d_offset = Σ_{r < rank} total(r)
// (the rank-order concatenation of the slices is the globally sorted array), and the
// projection capacity check (ΣH_slice <= cap, else FLAG_SIZE).
__global__ void k_comm_offsets(CommDev c, uint64_t cap, uint64_t* d_count, uint64_t* d_offset, DevStatus* st) {
  pdl_wait();
  const bool ok = comm_wait_all(c, kFlagTotals, st);
  if (threadIdx.x == 0) {
    const unsigned long long* tot =
        reinterpret_cast<const unsigned long long*>(c.ws[c.rank] + c.lay.tot) + (uint64_t)c.parity * kCommMaxRanks;
    unsigned long long off = 0, mine = 0;
    if (ok) {
      for (uint32_t r = 0; r < c.G; ++r) {
        const unsigned long long v = *reinterpret_cast<const volatile unsigned long long*>(tot + r);
        if (r < c.rank) off += v;
        if (r == c.rank) mine = v;
      }
    }
    if (d_count) *d_count = mine;
    if (d_offset) *d_offset = off;
    if (mine > cap) atomicOr(&st->flags, FLAG_SIZE);
  }
  pdl_trigger();
}

// ---- radix exchange ------------------------------------------------------------------------
// Top-digit histogram of the local keys (digit = top byte of u = x ^ 0x80000000), all-gathered
// into every peer's rhist[parity][rank][256]; the last CTA publishes (kFlagRhist).
// ws: 256 u32 histogram + 1 u32 ticket, zero on entry, cleared by the last CTA.
__global__ void __launch_bounds__(512) k_comm_rhist(CommDev c, const int32_t* __restrict__ keys, uint64_t n,
                                                    uint32_t* ws) {
  __shared__ uint32_t h[256];
  __shared__ bool s_last;
  pdl_wait();
  for (uint32_t i = threadIdx.x; i < 256; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += stride)
    atomicAdd(&h[((uint32_t)__ldcs(keys + i) ^ 0x80000000u) >> 24], 1u);
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < 256; i += blockDim.x)
    if (h[i]) atomicAdd(&ws[i], h[i]);
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = atomicAdd(&ws[256], 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  for (uint32_t i = threadIdx.x; i < c.G * 256; i += blockDim.x) {
    const uint32_t r = i >> 8, d = i & 255u;
    uint32_t* dst = reinterpret_cast<uint32_t*>(c.ws[r] + c.lay.rhist) + ((uint64_t)c.parity * kCommMaxRanks + c.rank) * 256 + d;
    *reinterpret_cast<volatile uint32_t*>(dst) = __ldcv(ws + d);
  }
  __syncthreads();
  if (threadIdx.x < c.G) {
    asm volatile("fence.acq_rel.sys;" ::: "memory");
    st_release_sys_u32(reinterpret_cast<uint32_t*>(c.ws[threadIdx.x] + comm_flag_off(c.lay, c.parity, kFlagRhist, c.rank)),
                       c.epoch);
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < 257; i += blockDim.x) ws[i] = 0;
}

// The split plan (one CTA): from the G all-gathered top-digit histograms (identical on every
// rank) rank r receives the contiguous top-digit range [D[r], D[r+1]), D chosen so that the
// cumulative count reaches r n_total / G (balanced as far as digit granularity allows).
// plan (this rank's workspace, u32): [0..G] digit bounds D, [16 + dst] destination cursors
// (first slot of this rank's keys in dst's receive buffer: Σ_{src < rank} cnt[src][dst]),
// [32] keys this rank receives, [34..35] its global output offset (u64), [40 + d] the
// destination rank of top digit d (256 entries).
__global__ void __launch_bounds__(256) k_comm_rplan(CommDev c, uint32_t* plan, uint64_t cap, uint64_t* d_count,
                                                    uint64_t* d_offset, DevStatus* st) {
  __shared__ uint32_t hsum[256];
  __shared__ uint32_t D[kCommMaxRanks + 1];
  pdl_wait();
  const bool ok = comm_wait_all(c, kFlagRhist, st);
  const uint32_t* rh = reinterpret_cast<const uint32_t*>(c.ws[c.rank] + c.lay.rhist) + (uint64_t)c.parity * kCommMaxRanks * 256;
  const uint32_t d = threadIdx.x;
  uint32_t s = 0;
  if (ok)
    for (uint32_t r = 0; r < c.G; ++r) s += __ldcv(rh + r * 256 + d);
  hsum[d] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long total = 0;
    for (uint32_t i = 0; i < 256; ++i) total += hsum[i];
    // D[r] = smallest digit whose exclusive prefix reaches r * total / G
    unsigned long long run = 0;
    uint32_t r = 1, i = 0;
    D[0] = 0;
    for (; i < 256 && r < c.G; ++i) {
      while (r < c.G && run >= total * r / c.G) D[r++] = i;
      run += hsum[i];
    }
    while (r < c.G) D[r++] = 256;
    D[c.G] = 256;
  }
  __syncthreads();
  if (threadIdx.x <= c.G) plan[threadIdx.x] = D[threadIdx.x];
  {  // destination of digit d
    uint32_t r = 0;
    while (r + 1 < c.G && D[r + 1] <= d) ++r;
    plan[40 + d] = r;
  }
  if (threadIdx.x < c.G) {  // cursor of this rank in destination dst
    const uint32_t dst = threadIdx.x;
    unsigned long long cur = 0;
    for (uint32_t src = 0; src < c.rank; ++src)
      for (uint32_t q = D[dst]; q < D[dst + 1]; ++q) cur += __ldcv(rh + src * 256 + q);
    plan[16 + dst] = (uint32_t)cur;
  }
  if (threadIdx.x == 0) {
    unsigned long long recv = 0, off = 0;
    for (uint32_t q = D[c.rank]; q < D[c.rank + 1]; ++q) recv += hsum[q];
    for (uint32_t q = 0; q < D[c.rank]; ++q) off += hsum[q];
    const unsigned long long lim = cap < c.lay.cap ? cap : c.lay.cap;
    if (recv > lim) atomicOr(&st->flags, FLAG_SIZE);
    plan[32] = (uint32_t)(recv > lim ? lim : recv);  // (the local sort never writes past its buffers)
    reinterpret_cast<unsigned long long*>(plan + 34)[0] = off;
    if (d_count) *d_count = recv;
    if (d_offset) *d_offset = off;
  }
  pdl_trigger();
}

// Split of the local keys by destination rank, stored straight into the owners' receive
// buffers (the all-to-all).  Per CTA sub-tile of 4096 keys: per-destination counts in shared
// memory, one global reservation per destination (atomicAdd on this rank's cursor plan[16 +
// dst]), keys staged by destination and written as contiguous runs (order inside a
// destination is free: the local LSD sort that follows makes the output unique).
constexpr uint32_t kSplitThreads = 512, kSplitKPT = 8, kSplitTile = kSplitThreads * kSplitKPT;
__global__ void __launch_bounds__(kSplitThreads) k_comm_rsplit(CommDev c, const int32_t* __restrict__ keys, uint64_t n,
                                                               uint32_t* plan) {
  __shared__ uint32_t dst_of[256];
  __shared__ uint32_t cnt[kCommMaxRanks], base[kCommMaxRanks + 1], gpos[kCommMaxRanks];
  __shared__ uint32_t stage[kSplitTile];
  pdl_wait();
  for (uint32_t i = threadIdx.x; i < 256; i += blockDim.x) dst_of[i] = __ldcg(plan + 40 + i);
  uint32_t* rk[kCommMaxRanks];
#pragma unroll
  for (uint32_t r = 0; r < kCommMaxRanks; ++r)
    rk[r] = r < c.G ? reinterpret_cast<uint32_t*>(c.ws[r] + c.lay.rkeys) + (uint64_t)c.parity * c.lay.cap : nullptr;
  const uint64_t ntile = (n + kSplitTile - 1) / kSplitTile;
  for (uint64_t t = blockIdx.x; t < ntile; t += gridDim.x) {
    const uint64_t t0 = t * kSplitTile;
    const uint32_t tn = (uint32_t)(n - t0 < kSplitTile ? n - t0 : kSplitTile);
    if (threadIdx.x < kCommMaxRanks) cnt[threadIdx.x] = 0;
    __syncthreads();
    uint32_t k[kSplitKPT], rnk[kSplitKPT];
#pragma unroll
    for (uint32_t i = 0; i < kSplitKPT; ++i) {
      const uint32_t j = i * kSplitThreads + threadIdx.x;
      k[i] = j < tn ? ((uint32_t)__ldcs(keys + t0 + j) ^ 0x80000000u) : 0u;
      rnk[i] = j < tn ? atomicAdd(&cnt[dst_of[k[i] >> 24]], 1u) : 0u;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t s = 0;
      for (uint32_t r = 0; r < c.G; ++r) {
        base[r] = s;
        s += cnt[r];
        gpos[r] = cnt[r] ? atomicAdd(plan + 16 + r, cnt[r]) : 0u;
      }
      base[c.G] = s;
    }
    __syncthreads();
#pragma unroll
    for (uint32_t i = 0; i < kSplitKPT; ++i) {
      const uint32_t j = i * kSplitThreads + threadIdx.x;
      if (j < tn) stage[base[dst_of[k[i] >> 24]] + rnk[i]] = k[i];
    }
    __syncthreads();
    for (uint32_t j = threadIdx.x; j < tn; j += blockDim.x) {
      const uint32_t u = stage[j];
      const uint32_t r = dst_of[u >> 24];
      const uint32_t pos = gpos[r] + (j - base[r]);
      if (pos < c.lay.cap) rk[r][pos] = u ^ 0x80000000u;  // (capacity checked by the plan)
    }
    __syncthreads();
  }
  pdl_trigger();
}

// Wait until every source's keys arrived (kFlagRkeys); nothing else (the LSD passes follow).
__global__ void k_comm_wait(CommDev c, uint32_t kind, DevStatus* st) {
  pdl_wait();
  comm_wait_all(c, kind, st);
  pdl_trigger();
}

}  // namespace ds

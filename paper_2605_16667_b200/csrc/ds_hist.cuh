// ds_hist.cuh — histogram ingestion kernels (eq:ingestion) with the CRN
// (def:crn_level P:896-915 / lem:crn P:951-962).
//
// Three memory paths, chosen by U:
//   k_hist_smem<false>  U <= kSmem32MaxBins: per-CTA uint32 sub-histogram in shared memory
//   k_hist_smem<true>   U <= kSmem16MaxBins: per-CTA packed 2x16-bit sub-histogram (bins 2w,
//                       2w+1 share word w), exact overflow detection by checksum + fallback
//   k_hist_global       larger U: warp CRN (MATCH.ANY) then one RED per distinct key per warp
//                       into an L2-resident H
// The smem paths write one partial histogram row per CTA (plain coalesced stores, no
// zeroing of H needed); ds_scan.cuh sums the rows.  On sm_100a the shared-memory atomic unit
// merges equal-address lanes of one ATOMS instruction itself (the CRN's equality merge in
// hardware), so the smem paths issue the atomic directly; the software CRN is used where
// the merge is not free: the L2 path, and the smem16 overflow fallback.
#pragma once
#include "ds_common.cuh"

namespace ds {

constexpr uint32_t kSmem32MaxBins = 8192;   // 32 KB of uint32 counters
constexpr uint32_t kSmem16MaxBins = 98304;  // 192 KB of packed counters (49152 words)
constexpr int kHistUnroll = 4;              // int4 loads in flight per thread

__device__ __forceinline__ uint32_t packed_word(uint32_t k) { return k >> 1; }
__device__ __forceinline__ uint32_t packed_inc(uint32_t k) { return (k & 1u) ? 65536u : 1u; }

template <bool PACK16>
__device__ __forceinline__ void ingest_smem(uint32_t* h, uint32_t k, uint32_t U, uint64_t idx,
                                            DevStatus* st, uint32_t& valid) {
  if (k < U) {
    if (PACK16)
      atomicAdd(h + packed_word(k), packed_inc(k));
    else
      atomicAdd(h + k, 1u);
    ++valid;
  } else {
    record_bad(st, idx, k);
  }
}

// Key layout shared by every pass over `keys`: `head` scalars before the first 16-byte
// boundary, `n4` aligned int4 vectors, `tail` scalars.  CTA 0 takes the head, the last CTA
// the tail, and the vectors are grid-strided.
struct KeySpan {
  const int32_t* keys;
  uint64_t n, head, n4, tail;
  __device__ __forceinline__ const int4* body() const { return reinterpret_cast<const int4*>(keys + head); }
};
__host__ __device__ inline KeySpan make_span(const int32_t* keys, uint64_t n) {
  KeySpan s;
  s.keys = keys;
  s.n = n;
  uint64_t mis = (reinterpret_cast<uintptr_t>(keys) >> 2) & 3u;
  s.head = mis ? (4 - mis) : 0;
  if (s.head > n) s.head = n;
  s.n4 = (n - s.head) / 4;
  s.tail = n - s.head - 4 * s.n4;
  return s;
}

// Visit every key this CTA owns: f(key, index).
template <typename F>
__device__ __forceinline__ void for_each_key(const KeySpan& s, F&& f) {
  const uint64_t T = blockDim.x, G = gridDim.x;
  if (blockIdx.x == 0 && threadIdx.x < s.head) f((uint32_t)s.keys[threadIdx.x], (uint64_t)threadIdx.x);
  if (blockIdx.x == G - 1 && threadIdx.x < s.tail) {
    uint64_t i = s.head + 4 * s.n4 + threadIdx.x;
    f((uint32_t)s.keys[i], i);
  }
  const int4* body = s.body();
  const uint64_t stride = G * T;
  uint64_t i = blockIdx.x * T + threadIdx.x;
  for (; i + (kHistUnroll - 1) * stride < s.n4; i += kHistUnroll * stride) {
    int4 v[kHistUnroll];
#pragma unroll
    for (int u = 0; u < kHistUnroll; ++u) v[u] = ld_stream4(body + i + u * stride);
#pragma unroll
    for (int u = 0; u < kHistUnroll; ++u) {
      uint64_t b = s.head + 4 * (i + u * stride);
      f((uint32_t)v[u].x, b);
      f((uint32_t)v[u].y, b + 1);
      f((uint32_t)v[u].z, b + 2);
      f((uint32_t)v[u].w, b + 3);
    }
  }
  for (; i < s.n4; i += stride) {
    int4 v = ld_stream4(body + i);
    uint64_t b = s.head + 4 * i;
    f((uint32_t)v.x, b);
    f((uint32_t)v.y, b + 1);
    f((uint32_t)v.z, b + 2);
    f((uint32_t)v.w, b + 3);
  }
}

// Global-path ingestion of one key batch position with the warp CRN.  All 32 lanes call it
// (the predicate `valid` marks lanes that carry a key; absent lanes never enter the CRN).
__device__ __forceinline__ void crn_red(uint32_t* H, uint32_t k, bool valid) {
  uint32_t mask = __ballot_sync(FULL, valid);
  if (valid) {
    uint32_t g = crn_group(mask, k);
    if (crn_is_leader(g)) red_add_u32(H + k, (uint32_t)__popc(g));
  }
}

// Same traversal as for_each_key but warp-synchronous (every lane runs every iteration),
// for the CRN paths.  f(key, index, valid).
template <typename F>
__device__ __forceinline__ void for_each_key_warp(const KeySpan& s, F&& f) {
  const uint64_t T = blockDim.x, G = gridDim.x;
  {
    bool v = blockIdx.x == 0 && threadIdx.x < s.head;
    if (threadIdx.x < 32) f(v ? (uint32_t)s.keys[threadIdx.x] : 0u, (uint64_t)threadIdx.x, v);
  }
  {
    bool v = blockIdx.x == G - 1 && threadIdx.x < s.tail;
    uint64_t i = s.head + 4 * s.n4 + threadIdx.x;
    if (threadIdx.x < 32) f(v ? (uint32_t)s.keys[i] : 0u, i, v);
  }
  const int4* body = s.body();
  const uint64_t stride = G * T;
  const uint64_t warp_base = blockIdx.x * T + (threadIdx.x & ~31u);
  for (uint64_t w = warp_base; w < s.n4; w += kHistUnroll * stride) {
    int4 v[kHistUnroll];
    bool ok[kHistUnroll];
#pragma unroll
    for (int u = 0; u < kHistUnroll; ++u) {
      uint64_t i = w + (threadIdx.x & 31) + u * stride;
      ok[u] = i < s.n4;
      v[u] = ok[u] ? ld_stream4(body + i) : make_int4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < kHistUnroll; ++u) {
      uint64_t b = s.head + 4 * (w + (threadIdx.x & 31) + u * stride);
      f((uint32_t)v[u].x, b, ok[u]);
      f((uint32_t)v[u].y, b + 1, ok[u]);
      f((uint32_t)v[u].z, b + 2, ok[u]);
      f((uint32_t)v[u].w, b + 3, ok[u]);
    }
  }
}

// ---- shared-memory paths -----------------------------------------------------------------
// partials: row r = CTA r, W words per row (W = U for u32, ceil(U/2) packed), row stride
// `ldw` = W rounded up to a multiple of 8 words; dynamic smem = 4*ldw bytes.  ovfH: uint32[U], zero on entry, used only by the fallback.
template <bool PACK16>
__global__ void __launch_bounds__(1024) k_hist_smem(const int32_t* __restrict__ keys, uint64_t n,
                                                    uint32_t U, uint32_t W, uint32_t ldw,
                                                    uint32_t* __restrict__ partials,
                                                    uint32_t* __restrict__ ovfH, DevStatus* st,
                                                    uint32_t epoch) {
  extern __shared__ __align__(16) uint32_t sh_hist[];
  __shared__ unsigned long long red64[33];
  pdl_wait();  // previous work on the stream (e.g. the caller's producer of keys)

  // K1: zero the private histogram (vectorised; ldw = W rounded up to 8 words, the padding
  // stays zero so k_reduce_scan may read whole 8-word groups).
  const uint32_t W4 = ldw / 4;
  uint4* h4 = reinterpret_cast<uint4*>(sh_hist);
  for (uint32_t i = threadIdx.x; i < W4; i += blockDim.x) h4[i] = make_uint4(0, 0, 0, 0);
  __syncthreads();

  const KeySpan s = make_span(keys, n);
  uint32_t valid = 0;
  for_each_key(s, [&](uint32_t k, uint64_t idx) { ingest_smem<PACK16>(sh_hist, k, U, idx, st, valid); });
  pdl_trigger();
  __syncthreads();

  uint32_t* row = partials + (uint64_t)blockIdx.x * ldw;
  uint4* row4 = reinterpret_cast<uint4*>(row);
  if (!PACK16) {
    for (uint32_t i = threadIdx.x; i < W4; i += blockDim.x) row4[i] = h4[i];
    return;
  }
  // Packed counters: a 16-bit field that wrapped loses >= 65535 from the field sum
  // (DESIGN.md §5.2), so Σ fields == #valid keys  <=>  no field overflowed.
  unsigned long long fsum = 0;
  for (uint32_t i = threadIdx.x; i < ldw; i += blockDim.x) {
    uint32_t w = sh_hist[i];
    fsum += (w & 0xffffu) + (w >> 16);
  }
  unsigned long long tot = block_sum<unsigned long long>(fsum, red64);
  unsigned long long nvalid = block_sum<unsigned long long>((unsigned long long)valid, red64);
  if (tot == nvalid) {
    for (uint32_t i = threadIdx.x; i < W4; i += blockDim.x) row4[i] = h4[i];
    return;
  }
  // Fallback (a key occurred >= 65536 times in this CTA's share): zero the row and re-ingest
  // this CTA's keys into ovfH through the warp CRN + L2 atomics.  Exact, slow, rare.
  for (uint32_t i = threadIdx.x; i < W4; i += blockDim.x) row4[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) atomicExch(&st->ovf_epoch, epoch);
  for_each_key_warp(s, [&](uint32_t k, uint64_t, bool v) { crn_red(ovfH, k, v && k < U); });
}

// ---- L2 path -----------------------------------------------------------------------------
// H: uint32[U] zeroed beforehand (k_zero).  Warp CRN then one RED per distinct key.
__global__ void __launch_bounds__(256) k_hist_global(const int32_t* __restrict__ keys, uint64_t n,
                                                     uint32_t U, uint32_t* __restrict__ H,
                                                     DevStatus* st) {
  pdl_wait();
  const KeySpan s = make_span(keys, n);
  for_each_key_warp(s, [&](uint32_t k, uint64_t idx, bool v) {
    bool in = v && k < U;
    if (v && !in) record_bad(st, idx, k);
    crn_red(H, k, in);
  });
  pdl_trigger();
}

// Vectorised zero fill of n32 words (n32 multiple of 4 not required).
__global__ void k_zero(uint32_t* __restrict__ p, uint64_t n32) {
  pdl_wait();
  uint64_t n4 = n32 / 4;
  uint4* p4 = reinterpret_cast<uint4*>(p);
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n4; i += stride)
    p4[i] = make_uint4(0, 0, 0, 0);
  uint64_t r = 4 * n4 + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (r < n32 && blockIdx.x == 0) p[r] = 0;
  pdl_trigger();
}

// Test entry for the CRN primitive: one warp per 32-lane batch.
__global__ void k_crn_resolve(const int32_t* __restrict__ lane_keys, const uint32_t* __restrict__ active,
                              uint64_t n_batches, int32_t* __restrict__ out_keys,
                              uint32_t* __restrict__ out_counts) {
  pdl_wait();
  const uint64_t b = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  const uint32_t lane = threadIdx.x & 31;
  if (b >= n_batches) return;  // whole warps exit together
  const uint32_t mask = active[b];
  const uint64_t i = b * 32 + lane;
  uint32_t cnt = 0;
  int32_t key = 0;
  if ((mask >> lane) & 1u) {
    key = lane_keys[i];
    uint32_t g = crn_group(mask, (uint32_t)key);
    if (crn_is_leader(g)) cnt = (uint32_t)__popc(g);
  }
  out_keys[i] = key;
  out_counts[i] = cnt;
}

}  // namespace ds

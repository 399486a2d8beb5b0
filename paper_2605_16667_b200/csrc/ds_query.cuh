// ds_query.cuh — the histogram as the canonical ordered state (SURVEY.md §8(f)
// NEXT-1): consumers of H answer frequency(k) and presence(k) in O(1) and range-count(a, b)
// without reconstructing the output; the support set D = {k : H(k) > 0} with the
// order-isomorphism condition of prop:iso: phi : D -> [0, M-1] is an isomorphism iff
// D = [0, M-1], i.e. |D| = U.
//
//   k_query_point    frequency / presence of m query keys (batched, one thread per query)
//   k_query_prefix   exclusive uint64 prefix of H (co-resident grid, one barrier) so that each
//                    of the m range-count queries is two loads (O(1) after an O(U) scan; the
//                    paper's O(b - a) per query is the scan-free form)
//   k_query_range    range-count(a, b) = pre[b + 1] - pre[a] per query pair
//   k_support_set    stream compaction of the occupied cells, ascending (co-resident grid: per-
//                    CTA counts, one barrier, offsets), |D| and the isomorphism flag
// Query keys outside [0, U) (and pairs with a > b) are range errors: recorded in the context's
// deferred status (index = query index) and answered 0.
#pragma once
#include "ds_common.cuh"
#include "ds_scan.cuh"

namespace ds {

constexpr int kQFrequency = 0, kQPresence = 1, kQRangeCount = 2;

__global__ void __launch_bounds__(256) k_query_point(const uint32_t* __restrict__ H, uint32_t U, int op,
                                                     const uint32_t* __restrict__ q, uint64_t m,
                                                     uint64_t* __restrict__ out, DevStatus* st) {
  pdl_wait();
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t k = q[i];
    uint64_t r = 0;
    if (k < U) {
      const uint32_t h = __ldg(H + k);
      r = op == kQPresence ? (h > 0u ? 1u : 0u) : h;
    } else {
      record_bad(st, i, k);
    }
    out[i] = r;
  }
  pdl_trigger();
}

// pre[k] = Σ_{j<k} H[j] for k = 0..U (uint64).  CTA b owns a contiguous range of bins; its
// total goes to part[b]; after one grid barrier each CTA adds the totals of lower CTAs.
__global__ void __launch_bounds__(1024) k_query_prefix(const uint32_t* __restrict__ H, uint32_t U,
                                                       uint64_t* __restrict__ pre, GridBar* bar) {
  __shared__ unsigned long long red[34];
  pdl_wait();
  const uint32_t G = gridDim.x, b = blockIdx.x;
  const uint32_t lo = (uint32_t)((uint64_t)U * b / G), hi = (uint32_t)((uint64_t)U * (b + 1) / G);
  uint64_t* part = pre + U + 1;  // [G] CTA totals (workspace past the prefix)
  // pass 1: this CTA's total
  unsigned long long s = 0;
  for (uint32_t k = lo + threadIdx.x; k < hi; k += blockDim.x) s += __ldg(H + k);
  unsigned long long tot;
  s = block_excl_scan<unsigned long long>(s, tot, red);
  if (threadIdx.x == 0) __stcg(part + b, (uint64_t)tot);
  grid_barrier(bar);  // (sense-reversing: replay-safe in CUDA graphs)
  unsigned long long off = 0;
  for (uint32_t j = threadIdx.x; j < b; j += blockDim.x) off += __ldcg(part + j);
  off = block_sum<unsigned long long>(off, red);
  // pass 2: chunks of blockDim bins, block scan per chunk
  for (uint32_t k0 = lo; k0 < hi; k0 += blockDim.x) {
    const uint32_t k = k0 + threadIdx.x;
    const unsigned long long h = k < hi ? __ldg(H + k) : 0ull;
    unsigned long long ct;
    const unsigned long long ex = block_excl_scan<unsigned long long>(h, ct, red);
    if (k < hi) pre[k] = off + ex;
    off += ct;
  }
  if (b == G - 1 && threadIdx.x == 0) pre[U] = off;
  pdl_trigger();
}

// q: m pairs (a_i, b_i) as uint32[2m]; out[i] = Σ_{k=a_i}^{b_i} H[k].
__global__ void __launch_bounds__(256) k_query_range(const uint64_t* __restrict__ pre, uint32_t U,
                                                     const uint32_t* __restrict__ q, uint64_t m,
                                                     uint64_t* __restrict__ out, DevStatus* st) {
  pdl_wait();
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < m; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t a = q[2 * i], bb = q[2 * i + 1];
    uint64_t r = 0;
    if (a <= bb && bb < U) r = __ldcg(pre + bb + 1) - __ldcg(pre + a);
    else record_bad(st, i, bb >= U ? bb : a);
    out[i] = r;
  }
  pdl_trigger();
}

// D = {k : H[k] > 0} ascending into D_out, |D| into *count, iso = (|D| == U) into *iso.
// ws: [G] per-CTA counts.
__global__ void __launch_bounds__(1024) k_support_set(const uint32_t* __restrict__ H, uint32_t U,
                                                      uint32_t* __restrict__ D_out, unsigned long long* count,
                                                      uint32_t* iso, unsigned long long* ws, GridBar* bar) {
  __shared__ unsigned long long red[34];
  pdl_wait();
  const uint32_t G = gridDim.x, b = blockIdx.x;
  const uint32_t lo = (uint32_t)((uint64_t)U * b / G), hi = (uint32_t)((uint64_t)U * (b + 1) / G);
  unsigned long long s = 0;
  for (uint32_t k = lo + threadIdx.x; k < hi; k += blockDim.x) s += __ldg(H + k) > 0u ? 1ull : 0ull;
  s = block_sum<unsigned long long>(s, red);
  if (threadIdx.x == 0) __stcg(ws + b, (uint64_t)s);
  grid_barrier(bar);  // (sense-reversing: replay-safe in CUDA graphs)
  unsigned long long off = 0;
  for (uint32_t j = threadIdx.x; j < b; j += blockDim.x) off += __ldcg(ws + j);
  off = block_sum<unsigned long long>(off, red);
  for (uint32_t k0 = lo; k0 < hi; k0 += blockDim.x) {
    const uint32_t k = k0 + threadIdx.x;
    const unsigned long long occ = (k < hi && __ldg(H + k) > 0u) ? 1ull : 0ull;
    unsigned long long ct;
    const unsigned long long ex = block_excl_scan<unsigned long long>(occ, ct, red);
    if (occ) D_out[off + ex] = k;
    off += ct;
  }
  if (b == G - 1 && threadIdx.x == 0) {
    *count = off;
    if (iso) *iso = off == U ? 1u : 0u;
  }
  pdl_trigger();
}

}  // namespace ds

// ds_small.cuh — the whole DialSort step for small inputs on one thread-block cluster.
//
// For small n (below) and U <= kSmallMaxU bins the co-resident grid of k_sort_fused
// (up to 148 CTAs, global-memory grid barriers, owner counters in L2) is latency-bound: ~11 us
// for c1 (n = 10^5, U = 256) even replayed from a CUDA graph.  Here kSmallCS CTAs of one
// cluster run the three steps of the method with cluster barriers and distributed shared
// memory instead:
//   ingestion   eq:ingestion: each CTA adds its keys (grid-stride 16-byte vectors)
//               into its own shared-memory H_r with one shared atomic a key (equal addresses of
//               a warp instruction merged by the atomic unit — the CRN's equality merge)
//   merge       lem:crn: CTA r owns bins [rU/CS, (r+1)U/CS) and sums them over the
//               cluster's H_r' through DSMEM (additive merge; H written if requested)
//   offsets     the owned bins' exclusive prefix (block scan) + the owners' totals (DSMEM)
//   projection  eq:projection: out[P[k] .. P[k] + H[k]) = k by output position;
//               owners write their bins, or — skewed inputs — every CTA an even share
// Keys outside [0, U) are recorded (count, minimum index) and not counted; out may be keys
// (in place: the projection starts after the cluster barrier that follows the ingestion);
// out == nullptr: histogram only (H).
#pragma once
#include <cooperative_groups.h>

#include "ds_common.cuh"

namespace ds {
constexpr uint32_t kSmallThreads = 1024;
constexpr uint32_t kSmallMaxU = 8192;       // 32 KB of uint32 counters a CTA
// Sizes (CUDA-graph device time a sort; k_sort_fused beside): 8-CTA clusters up to n = 5·10^4
// (n = 10^4: 4.6 us, 16 CTAs 5.0, fused 12.6), 16-CTA clusters (non-portable, where the device
// schedules them) above it up to 4·10^5 for U <= 1024 (n = 10^5: 6.1 vs 11.5; 2·10^5: 9.5 vs
// 10.9; 4·10^5: 10.7 vs 13.5; 10^6: 16.4 vs 14.1) and 1.5·10^5 for larger U; else the fused grid.
// Without 16-CTA clusters the 8-CTA path runs up to 1.2·10^5 (n = 10^5: 8.0 vs 11.5; 1.5·10^5,
// U = 1024: 14.0 vs 12.4).
constexpr uint64_t kSmall8MaxN = 50000, kSmall8OnlyMaxN = 120000;
#ifndef DIALSORT_SMALL_BATCH8_MAX_N
#define DIALSORT_SMALL_BATCH8_MAX_N 120000
#endif
constexpr uint64_t kSmallBatch8MaxN = DIALSORT_SMALL_BATCH8_MAX_N;  // batches: 8-CTA clusters up to here
__host__ __device__ constexpr uint64_t small16_max_n(uint32_t U) { return U <= 1024 ? 400000 : 150000; }

// Positions [p0, p1) of an output whose bin k (of nb, prefix pr[0..nb], pr[nb] = total) holds
// the key k0 + k, T positions apart per thread (a warp's stores coalesce): a thread's next
// position is mostly still in its bin — one test, else a binary search of the bins above.
// (4 consecutive positions a thread, one search each, measured slower: 27.7 vs 16.4 us at
//  n = 10^6 — a warp's stores then spread over 512 bytes per instruction)
__device__ __forceinline__ void project_positions(const uint32_t* pr, uint32_t nb, uint32_t p0, uint32_t p1,
                                                  int32_t* o, uint32_t k0) {
  uint32_t j = 0;  // invariant: pr[j] <= p
  for (uint32_t p = p0 + threadIdx.x; p < p1; p += blockDim.x) {
    if (pr[j + 1] <= p) {
      uint32_t hi = nb;
      while (hi - j > 1) {
        const uint32_t mid = (j + hi) >> 1;
        if (pr[mid] <= p) j = mid;
        else hi = mid;
      }
    }
    __stcs(o + p, (int32_t)(k0 + j));
  }
}

// kSmallCS CTAs a cluster: 8 (portable) or 16 (non-portable, larger inputs); the cluster
// dimension is a launch attribute.
template <uint32_t kSmallCS>
__device__ __forceinline__ void small_step(const int32_t* __restrict__ keys, uint64_t n, uint32_t U, int32_t* out,
                                           uint32_t* __restrict__ H, DevStatus* st) {
  constexpr uint32_t kSmallOwn = (kSmallMaxU + kSmallCS - 1) / kSmallCS;  // bins a CTA owns at most
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  __shared__ uint32_t h[kSmallMaxU + 1];   // this CTA's histogram of its keys (then P, skewed inputs)
  __shared__ uint32_t pre[kSmallOwn + 1];  // exclusive prefix of the owned bins' totals (+ their total)
  __shared__ uint32_t red[34];
  __shared__ uint32_t s_sum, s_all[kSmallCS];  // owned total; every owner's total
  const uint32_t r = cl.block_rank(), T = blockDim.x;
  for (uint32_t i = threadIdx.x; i < U; i += T) h[i] = 0;
  __syncthreads();
  // ---- ingestion (keys of [0, U); others recorded)
  const KeySpan s = make_span(keys, n);
  auto one = [&](uint32_t k, uint64_t idx) {
    if (k < U) atomicAdd(&h[k], 1u);
    else record_bad(st, idx, k);
  };
  if (r == 0 && threadIdx.x < s.head) one((uint32_t)keys[threadIdx.x], threadIdx.x);
  if (r == kSmallCS - 1 && threadIdx.x < s.tail) {
    const uint64_t i = s.head + 4 * s.n4 + threadIdx.x;
    one((uint32_t)keys[i], i);
  }
  {  // (the thread's vectors in batches of NV loads in flight: a serial load-then-count loop
     //  waited a full load latency per vector)
    constexpr uint32_t NV = 8;
    const int4* __restrict__ body = s.body();
    const uint32_t stride = kSmallCS * T;
    for (uint32_t v0 = r * T + threadIdx.x; v0 < s.n4; v0 += NV * stride) {
      int4 x[NV];
#pragma unroll
      for (uint32_t u = 0; u < NV; ++u)
        x[u] = v0 + u * stride < s.n4 ? __ldcs(body + v0 + u * stride) : make_int4(0, 0, 0, 0);
#pragma unroll
      for (uint32_t u = 0; u < NV; ++u) {
        const uint32_t v = v0 + u * stride;
        if (v >= s.n4) break;
        if (umax4(x[u]) < U) {
          atomicAdd(&h[(uint32_t)x[u].x], 1u);
          atomicAdd(&h[(uint32_t)x[u].y], 1u);
          atomicAdd(&h[(uint32_t)x[u].z], 1u);
          atomicAdd(&h[(uint32_t)x[u].w], 1u);
        } else {
          const uint64_t i0 = s.head + 4ull * v;
          one((uint32_t)x[u].x, i0); one((uint32_t)x[u].y, i0 + 1);
          one((uint32_t)x[u].z, i0 + 2); one((uint32_t)x[u].w, i0 + 3);
        }
      }
    }
  }
  cl.sync();  // every H_r complete (and every key read: out may alias keys from here on)
  // ---- merge of the owned bins over the cluster (DSMEM) and their exclusive prefix
  auto own_lo = [&](uint32_t q) { return (uint32_t)((uint64_t)U * q / kSmallCS); };
  const uint32_t b0 = own_lo(r), nb = own_lo(r + 1) - b0;  // nb <= kSmallOwn <= T
  uint32_t v = 0;
  if (threadIdx.x < nb) {
#pragma unroll
    for (uint32_t q = 0; q < kSmallCS; ++q) v += cl.map_shared_rank(h, q)[b0 + threadIdx.x];
    if (H) H[b0 + threadIdx.x] = v;
  }
  uint32_t own_tot;
  const uint32_t ex = block_excl_scan<uint32_t>(v, own_tot, red);
  if (threadIdx.x < nb) pre[threadIdx.x] = ex;
  if (threadIdx.x == 0) {
    pre[nb] = own_tot;
    s_sum = own_tot;
  }
  cl.sync();  // every owned total and prefix published (and every H_r read: h is free)
  if (threadIdx.x < kSmallCS) s_all[threadIdx.x] = *cl.map_shared_rank(&s_sum, threadIdx.x);
  __syncthreads();
  uint32_t base = 0, tot = 0, mx = 0;
#pragma unroll
  for (uint32_t q = 0; q < kSmallCS; ++q) {
    if (q < r) base += s_all[q];
    tot += s_all[q];
    mx = max(mx, s_all[q]);
  }
  // ---- projection (eq:projection): out[P[k] .. P[k] + H[k]) = k.  Balanced owners write their
  // own bins' positions; when one owner holds much more than its share (skewed keys) every
  // CTA takes an even share of the positions instead, searching the whole prefix P (gathered
  // from the owners' prefixes into h).  The choice is the same on every CTA.
  // (the last cluster barrier only keeps this CTA's shared memory alive while the others read
  //  it: arrived here, waited for at the end, so the projection runs in between)
  if (!out) {  // (histogram only)
    cl.sync();
    return;
  }
  const bool even = (uint64_t)mx * kSmallCS > 2ull * tot + 16384;
  if (!even) {
    cl.barrier_arrive();
    project_positions(pre, nb, 0, own_tot, out + base, b0);
  } else {
    for (uint32_t k = threadIdx.x; k < U; k += T) {
      uint32_t q = (uint32_t)(((uint64_t)k * kSmallCS) / U);  // owner: own_lo(q) <= k < own_lo(q + 1)
      while (q + 1 < kSmallCS && own_lo(q + 1) <= k) ++q;
      uint32_t bq = 0;
      for (uint32_t i = 0; i < q; ++i) bq += s_all[i];
      h[k] = bq + cl.map_shared_rank(pre, q)[k - own_lo(q)];
    }
    if (threadIdx.x == 0) h[U] = tot;
    cl.barrier_arrive();
    __syncthreads();  // (h complete)
    const uint32_t p0 = (uint32_t)((uint64_t)tot * r / kSmallCS), p1 = (uint32_t)((uint64_t)tot * (r + 1) / kSmallCS);
    project_positions(h, U, p0, p1, out, 0u);
  }
  cl.barrier_wait();
}

template <uint32_t kSmallCS>
__global__ void __launch_bounds__(kSmallThreads, 1)
    k_sort_small(const int32_t* __restrict__ keys, uint64_t n, uint32_t U, int32_t* out, uint32_t* __restrict__ H,
                 DevStatus* st) {
  pdl_wait();
  small_step<kSmallCS>(keys, n, U, out, H, st);
  pdl_trigger();
}

// Independent small sorts (dialsort_sort_batch_async): cluster j of the grid sorts batch j; the
// hardware runs as many clusters at once as the SMs hold (9 of 16 CTAs, 18 of 8) and starts the
// next ones as they finish.
constexpr uint32_t kSmallBatchMax = 64;
struct SmallBatch {
  const int32_t* keys[kSmallBatchMax];
  int32_t* out[kSmallBatchMax];
  uint32_t* H[kSmallBatchMax];
  uint64_t n[kSmallBatchMax];
};
template <uint32_t kSmallCS>
__global__ void __launch_bounds__(kSmallThreads, 1) k_sort_small_batch(const __grid_constant__ SmallBatch B, uint32_t U,
                                                                       DevStatus* st) {
  pdl_wait();
  const uint32_t j = blockIdx.x / kSmallCS;
  small_step<kSmallCS>(B.keys[j], B.n[j], U, B.out[j], B.H[j], st);
  pdl_trigger();
}
}  // namespace ds

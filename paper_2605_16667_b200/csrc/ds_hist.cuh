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
#include "ds_scan.cuh"

namespace ds {

constexpr uint32_t kSmem32MaxBins = 8192;   // 32 KB of uint32 counters
constexpr uint32_t kSmem16MaxBins = 98304;  // 192 KB of packed counters (49152 words)
constexpr uint32_t kFTileBins = 64;         // scan-tile width of k_sort_fused (ds_fused.cuh)
// int4 loads per batch, 2 batches in flight (5 or 6 per batch measured slower: c2 27.4 -> 28.6 /
// 29.2 us single call, 17.8 -> 18.4 / 18.1 us batched — register pressure at 1024 threads)
// Vectors per batch of the int32 ingestion (two batches in flight per thread): 3 measured
// better than round 1's 4 on every config (c2 single call 27.8 -> 27.0 us, batched 17.6 ->
// 17.5; Zipf 22.5 -> 22.0 batched; sorted 19.1 -> 18.65) — the loads are not what bounds it.
#ifndef DIALSORT_HIST_UNROLL
#define DIALSORT_HIST_UNROLL 3
#endif
constexpr int kHistUnroll = DIALSORT_HIST_UNROLL;
constexpr uint32_t kFOwnVote = 255;         // k_sort_fused: owner-counter slot of the skew vote

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

// Visit this CTA's keys as int4 vectors f4(v, vector index), plus scalars f1(key, index) for
// the unaligned head (CTA 0) and tail (last CTA).  32-bit vector indices (n4 < 2^30).
// The first batch of a thread's vectors (a[u] = vector i + u stride, i = b T + t), loaded by the
// caller before it zeroes its histogram (the loads' latency overlaps the zeroing and the hot-key
// sampling, which reads a[0]).
template <int NV>
__device__ __forceinline__ void preload_vecs(const int4* __restrict__ body, uint32_t nv, VGrid vg, int4 (&a)[NV]) {
  const uint64_t pol = l2_evict_first_policy();
  const uint32_t stride = vg.G * blockDim.x, i = vg.b * blockDim.x + threadIdx.x;
#pragma unroll
  for (int u = 0; u < NV; ++u)
    a[u] = (i + u * stride < nv) ? ld_stream4(body + i + u * stride, pol) : make_int4(0, 0, 0, 0);
}
// (a: the thread's first batch, preload_vecs)
template <typename F4, typename F1>
__device__ __forceinline__ void for_each_key4(const KeySpan& s, int4 (&a)[kHistUnroll], F4&& f4, F1&& f1,
                                              VGrid vg = vgrid_hw()) {
  const uint32_t T = blockDim.x, G = vg.G;
  if (vg.b == 0 && threadIdx.x < s.head) f1((uint32_t)s.keys[threadIdx.x], (uint64_t)threadIdx.x);
  if (vg.b == G - 1 && threadIdx.x < s.tail) {
    uint64_t i = s.head + 4 * s.n4 + threadIdx.x;
    f1((uint32_t)s.keys[i], i);
  }
  const uint64_t pol = l2_evict_first_policy();
  const int4* __restrict__ body = s.body();
  // Grid-stride over vectors (all SMs sweep the array together: measured faster than
  // contiguous per-CTA ranges with an up-front L2 bulk prefetch, 10 vs 12.7 us at c2).
  // Software pipeline: the next batch is requested before the current one is ingested
  // (measured faster than ping-pong / refill-after-consume variants, 10 vs 14 us at c2).
  const uint32_t n4 = (uint32_t)s.n4, stride = G * T;
  uint32_t i = vg.b * T + threadIdx.x;
  while (i < n4) {
    const uint32_t in = i + kHistUnroll * stride;
    int4 b[kHistUnroll];
#pragma unroll
    for (int u = 0; u < kHistUnroll; ++u)
      b[u] = (in + u * stride < n4) ? ld_stream4(body + in + u * stride, pol) : make_int4(0, 0, 0, 0);
#pragma unroll
    for (int u = 0; u < kHistUnroll; ++u)
      if (i + u * stride < n4) f4(a[u], i + u * stride);
#pragma unroll
    for (int u = 0; u < kHistUnroll; ++u) a[u] = b[u];
    i = in;
  }
}

// Slow path of an int4 group holding at least one key outside [0,U): ingest the valid keys
// one by one and record the bad ones (never taken on valid input; kept out of line).
template <bool PACK16>
__device__ __noinline__ uint32_t ingest4_checked(uint32_t* h, int4 v, uint64_t idx0, uint32_t U, DevStatus* st) {
  uint32_t k[4] = {(uint32_t)v.x, (uint32_t)v.y, (uint32_t)v.z, (uint32_t)v.w};
  uint32_t bad = 0;
  for (int j = 0; j < 4; ++j) {
    if (k[j] < U) {
      if (PACK16) atomicAdd(h + (k[j] >> 1), 1u << ((k[j] & 1u) << 4));
      else atomicAdd(h + k[j], 1u);
    } else {
      record_bad(st, idx0 + j, k[j]);
      ++bad;
    }
  }
  return bad;
}

// Error path of the hot loop: re-read the vectors this thread owns (the grid stride of
// for_each_key4) and ingest, key by key, those that hold an out-of-range key (the hot loop
// skipped them whole); returns #bad keys.
template <bool PACK16>
__device__ __noinline__ uint32_t ingest_deferred(uint32_t* h, const KeySpan& s, uint32_t U, DevStatus* st, VGrid vg) {
  const uint32_t n4 = (uint32_t)s.n4;
  const int4* body = s.body();
  uint32_t bad = 0;
  const uint32_t stride = vg.G * blockDim.x;
  for (uint32_t i = vg.b * blockDim.x + threadIdx.x; i < n4; i += stride) {
    const int4 v = body[i];
    if (umax4(v) >= U) bad += ingest4_checked<PACK16>(h, v, s.head + 4 * (uint64_t)i, U, st);
  }
  return bad;
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

// The keys this CTA owns (the grid stride of for_each_key4), warp-synchronously (every lane runs
// every iteration), for the CRN paths: f(key, index, valid).
template <typename F>
__device__ __forceinline__ void for_each_key_warp(const KeySpan& s, F&& f, VGrid vg = vgrid_hw()) {
  const uint64_t T = blockDim.x, G = vg.G;
  {
    bool v = vg.b == 0 && threadIdx.x < s.head;
    if (threadIdx.x < 32) f(v ? (uint32_t)s.keys[threadIdx.x] : 0u, (uint64_t)threadIdx.x, v);
  }
  {
    bool v = vg.b == G - 1 && threadIdx.x < s.tail;
    uint64_t i = s.head + 4 * s.n4 + threadIdx.x;
    if (threadIdx.x < 32) f(v ? (uint32_t)s.keys[i] : 0u, i, v);
  }
  const int4* body = s.body();
  auto vec = [&](uint64_t i, bool ok) {
    const int4 v = ok ? ld_stream4(body + i) : make_int4(0, 0, 0, 0);
    const uint64_t b = s.head + 4 * i;
    f((uint32_t)v.x, b, ok);
    f((uint32_t)v.y, b + 1, ok);
    f((uint32_t)v.z, b + 2, ok);
    f((uint32_t)v.w, b + 3, ok);
  };
  const uint64_t stride = G * T;
  for (uint64_t w = vg.b * T + (threadIdx.x & ~31u); w < s.n4; w += stride) {
    const uint64_t i = w + (threadIdx.x & 31);
    vec(i, i < s.n4);
  }
}
__device__ __noinline__ void hist_overflow_fallback(const KeySpan& s, uint4* row4, uint32_t W4, uint32_t* ovfH,
                                                    uint32_t U, DevStatus* st, uint32_t epoch, VGrid vg) {
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < W4; i += blockDim.x) row4[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) atomicExch(&st->ovf_epoch, epoch);
  for_each_key_warp(s, [&](uint32_t k, uint64_t, bool v) { crn_red(ovfH, k, v && k < U); }, vg);
}

// ---- shared-memory paths: ingestion and flush of the fused step (ds_fused.cuh sort_step) -------
// Every CTA ingests its keys into a private shared-memory histogram (uint32, or packed 2 x 16-bit
// with exact overflow detection) and flushes it as partial row c (4-bit, 16-bit or 32-bit
// counts; plain coalesced stores, no zeroing of H, no global atomics on the hot path), with the
// row's 64-bin tile sums in shared memory (tsum_sh), from which the row's sum s_o over each
// owning CTA o's tiles is formed.  The step needs, after its grid barrier, only the first output
// position of each CTA's own tiles: P_o = Σ_rows Σ_{o' < o} s_o'.  So each row adds its
// inclusive prefix over owners into P_{o+1} (one RED per owner, counters on separate L2 lines:
// same-line REDs serialise) and CTA o later reads just P_o and P_{o+1} (two lines) instead of
// every owner total.  It also votes "skewed" (one RED into a per-launch word) when some s_o
// exceeds 5/4 of its even share of the row: the own-tile projection is then replaced by equal
// position shares (no vote anywhere bounds every owner's positions by 5/4 n / G + 64 G, so own
// tiles stay balanced).
// Skew vote slack (flush_owner_totals): 32768 keys per owner, x 4.  With fewer 64-bin tiles
// than CTAs (U = 256 on 25 CTAs at n = 1e5) four owners hold every key; below ~32k keys each,
// projecting them in the own-tile mode beats the share mode's flag waits (c1 13.7 -> 11.8 us),
// above it the share mode spreads them (n = 3e6, U = 256: 63 us own-tile vs 18.5 share).
constexpr unsigned long long kSkewSlack = 4ull * 32768;
__device__ __forceinline__ void flush_owner_totals(const ScanArgs& a, const uint32_t* tsum_sh, uint32_t U,
                                                   uint32_t* red, VGrid vg) {
  const uint32_t ntf = (U + kFTileBins - 1) / kFTileBins, G = vg.G, b = threadIdx.x;
  uint32_t s = 0;
  if (b < G) {
    const uint32_t t0 = (uint32_t)((uint64_t)ntf * b / G), t1 = (uint32_t)((uint64_t)ntf * (b + 1) / G);
    for (uint32_t t = t0; t < t1; ++t) s += tsum_sh[t];
  }
  uint32_t tot;
  const uint32_t inc = block_excl_scan<uint32_t>(s, tot, red) + s;  // Σ_{o <= b} s_o
  if (b < G && inc) red_add_u32(a.own_red + (uint64_t)(b + 1) * a.ctr_stride, inc);
  // (tot = the row's keys: a row votes when an owner's share passes 5/4 of the even one plus a
  //  slack of kSkewSlack / 4 projected keys over the whole step — what an owner projects in the
  //  ~2 us the share mode's flags cost)
  const bool skew = b < G && 4ull * G * s > 5ull * tot + kSkewSlack;
  if (__syncthreads_or(skew) && threadIdx.x == 0) red_add_u32(a.own_red + (uint64_t)(kFOwnVote)*a.ctr_stride, 1u);
}

// ---- 16-bit keys (the hierarchical path's universe blocks, ds_part.cuh) -------------------
// A block's keys are stored as their low 16 bits (2 bytes a key: half the bytes of the block
// sorts' ingestion).  Keys [head, head + 8 n8) are 16-byte vectors of 8 keys, visited grid-
// strided like for_each_key4 (vector v by thread v mod (G T) of CTA (v / T) mod G); the
// unaligned head (CTA 0) and tail (last CTA) go through f1.  Returns this thread's vectors.
struct KeySpan16 {
  const uint16_t* keys;
  uint64_t n, head, n8, tail;
};
// Narrow keys of KB bytes (KB = 2: the hierarchical path's uint16 block keys and 2-byte coded
// domains; KB = 1: 1-byte coded domains, Proposition 2), optionally mapped through
// the encode table phi (enc, device uint32[256], 1-byte keys only).  The aligned body is visited
// as 16-byte vectors of 16 / KB keys, grid-strided like for_each_key4; the unaligned head (CTA 0)
// and tail (last CTA) go through f1.  Returns this thread's vectors.
template <int KB>
__device__ __forceinline__ uint32_t narrow_key(const uint16_t* keys, uint64_t i, const uint32_t* enc) {
  const uint32_t k = KB == 1 ? (uint32_t)reinterpret_cast<const uint8_t*>(keys)[i] : (uint32_t)keys[i];
  return enc ? __ldg(enc + k) : k;
}
template <int KB>
__device__ __forceinline__ KeySpan16 make_span_narrow(const uint16_t* keys, uint64_t n) {
  KeySpan16 s;
  s.keys = keys;
  s.n = n;
  constexpr uint32_t per = 16 / KB;  // keys per vector
  const uint64_t mis = (reinterpret_cast<uintptr_t>(keys) & 15u) / KB;
  s.head = mis ? per - mis : 0;
  if (s.head > n) s.head = n;
  s.n8 = (n - s.head) / per;
  s.tail = n - s.head - per * s.n8;
  return s;
}
// 16 bytes -> 16 / KB keys -> vectors of 4 for f4(int4, index of the 4-key group)
template <int KB, typename F4>
__device__ __forceinline__ void expand_narrow(const int4& x, uint32_t v, const uint32_t* enc, F4&& f4) {
  const uint32_t w[4] = {(uint32_t)x.x, (uint32_t)x.y, (uint32_t)x.z, (uint32_t)x.w};
  if (KB == 2) {
#pragma unroll
    for (int h = 0; h < 2; ++h)
      f4(make_int4((int)(w[2 * h] & 0xffffu), (int)(w[2 * h] >> 16), (int)(w[2 * h + 1] & 0xffffu),
                   (int)(w[2 * h + 1] >> 16)), 2 * v + h);
  } else {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint32_t b0 = w[q] & 0xffu, b1 = (w[q] >> 8) & 0xffu, b2 = (w[q] >> 16) & 0xffu, b3 = w[q] >> 24;
      if (enc) b0 = __ldg(enc + b0), b1 = __ldg(enc + b1), b2 = __ldg(enc + b2), b3 = __ldg(enc + b3);
      f4(make_int4((int)b0, (int)b1, (int)b2, (int)b3), 4 * v + q);
    }
  }
}
#ifndef DIALSORT_NARROW_UNROLL
#define DIALSORT_NARROW_UNROLL 3  // (c4 block steps: 2 -> 1.312 ms, 3 -> 1.294, 4 -> 1.335)
#endif
constexpr int kNarrowUnroll = DIALSORT_NARROW_UNROLL;  // vectors per batch (2 batches in flight)
// (a: the thread's first batch, preload_vecs)
template <int KB, typename F4, typename F1>
__device__ __forceinline__ uint32_t for_each_key_narrow(const KeySpan16& s, int4 (&a)[kNarrowUnroll],
                                                        const uint32_t* enc, F4&& f4, F1&& f1, VGrid vg) {
  constexpr int NU = kNarrowUnroll;
  constexpr uint32_t per = 16 / KB;
  const uint32_t T = blockDim.x, G = vg.G;
  if (vg.b == 0 && threadIdx.x < s.head) f1(narrow_key<KB>(s.keys, threadIdx.x, enc), (uint64_t)threadIdx.x);
  if (vg.b == G - 1 && threadIdx.x < s.tail) {
    const uint64_t i = s.head + per * s.n8 + threadIdx.x;
    f1(narrow_key<KB>(s.keys, i, enc), i);
  }
  const uint64_t pol = l2_evict_first_policy();
  const int4* __restrict__ body = reinterpret_cast<const int4*>(reinterpret_cast<const char*>(s.keys) + KB * s.head);
  const uint32_t n8 = (uint32_t)s.n8, stride = G * T;
  uint32_t cnt = 0;
  uint32_t i = vg.b * T + threadIdx.x;
  while (i < n8) {
    const uint32_t in = i + (NU) * stride;
    int4 b[NU];
#pragma unroll
    for (int u = 0; u < NU; ++u)
      b[u] = (in + u * stride < n8) ? ld_stream4(body + in + u * stride, pol) : make_int4(0, 0, 0, 0);
#pragma unroll
    for (int u = 0; u < NU; ++u)
      if (i + u * stride < n8) {
        expand_narrow<KB>(a[u], i + u * stride, enc, f4);
        ++cnt;
      }
#pragma unroll
    for (int u = 0; u < NU; ++u) a[u] = b[u];
    i = in;
  }
  return cnt;
}
// Error path of the narrow traversal: re-read this thread's vectors, ingest key by key those
// 4-key groups holding a key outside [0, U) (skipped whole by the hot loop); returns #bad keys.
template <bool PACK16, int KB>
__device__ __noinline__ uint32_t ingest_deferred_narrow(uint32_t* h, const KeySpan16& s, const uint32_t* enc,
                                                        uint32_t U, DevStatus* st, VGrid vg) {
  const int4* body = reinterpret_cast<const int4*>(reinterpret_cast<const char*>(s.keys) + KB * s.head);
  uint32_t bad = 0;
  const uint32_t stride = vg.G * blockDim.x, n8 = (uint32_t)s.n8;
  for (uint32_t i = vg.b * blockDim.x + threadIdx.x; i < n8; i += stride)
    expand_narrow<KB>(body[i], i, enc, [&](int4 v, uint32_t g) {
      if (umax4(v) >= U) bad += ingest4_checked<PACK16>(h, v, s.head + 4 * (uint64_t)g, U, st);
    });
  return bad;
}
// Overflow fallback of a 16-bit-key CTA: zero the row, re-ingest this CTA's keys (the same
// head / tail / grid-strided vectors) into ovfH through the warp CRN.
__device__ __noinline__ void hist_overflow_fallback16(const KeySpan16& s, uint4* row4, uint32_t W4, uint32_t* ovfH,
                                                      uint32_t U, DevStatus* st, uint32_t epoch, VGrid vg) {
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < W4; i += blockDim.x) row4[i] = make_uint4(0, 0, 0, 0);
  if (threadIdx.x == 0) atomicExch(&st->ovf_epoch, epoch);
  const uint32_t T = blockDim.x, G = vg.G;
  if (threadIdx.x < 32) {
    bool v = vg.b == 0 && threadIdx.x < s.head;
    crn_red(ovfH, v ? (uint32_t)s.keys[threadIdx.x] : 0u, v && s.keys[threadIdx.x] < U);
    v = vg.b == G - 1 && threadIdx.x < s.tail;
    const uint64_t ti = s.head + 8 * s.n8 + threadIdx.x;
    crn_red(ovfH, v ? (uint32_t)s.keys[ti] : 0u, v && s.keys[ti] < U);
  }
  const int4* body = reinterpret_cast<const int4*>(s.keys + s.head);
  for (uint64_t w = (uint64_t)vg.b * T + (threadIdx.x & ~31u); w < s.n8; w += (uint64_t)G * T) {
    const uint64_t i = w + (threadIdx.x & 31);
    const bool ok = i < s.n8;
    const int4 x = ok ? ld_stream4(body + i) : make_int4(0, 0, 0, 0);
    const uint32_t h[4] = {(uint32_t)x.x, (uint32_t)x.y, (uint32_t)x.z, (uint32_t)x.w};
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const uint32_t k = (h[q >> 1] >> (16 * (q & 1))) & 0xffffu;
      crn_red(ovfH, k, ok && k < U);
    }
  }
}

// ---- hot keys (skew at scale) ------------------------------------------------------------
// A packed 16-bit counter wraps when one CTA sees > 65535 copies of a key: possible once a CTA
// ingests more than 65535 keys (n > 65000 G) and some key's share p exceeds 65535 G / n (Zipf
// 1.2 at n = 1e8: p1 = 0.198 against 0.097).  The exact overflow fallback then re-ingests the
// whole CTA through L2 (measured 15x slower: 2.46 ms vs 0.159 ms at n = 1e8).  Large launches
// first sample each thread's first vector, find up to kHotK keys whose sampled share would put
// more than 30000 copies in a CTA, and count those keys in per-thread registers (one compare per
// hot key per key) instead of the packed histogram; the counts go whole into the exception
// histogram Hx (32-bit, merged with the rows) and into the tile sums.  Candidates: the first key
// of lanes 0 and 16 of every warp when it recurs >= 3 times in the warp's 128 sampled keys, in a
// 128-slot open-addressing table; then every sampled key counts its candidate.
constexpr uint32_t kHotK = 4, kHotTab = 128, kHotNone = 0xffffffffu;
__device__ __forceinline__ uint32_t hot_hash(uint32_t k) { return (k * 0x9E3779B1u) >> 25; }  // 7 bits
__device__ __forceinline__ void hot_tab_insert(uint32_t* tab, uint32_t k) {
  for (uint32_t i = hot_hash(k), t = 0; t < kHotTab; ++t, i = (i + 1) & (kHotTab - 1)) {
    const uint32_t old = atomicCAS(tab + i, kHotNone, k);
    if (old == kHotNone || old == k) return;
  }
}
__device__ __forceinline__ uint32_t hot_tab_find(const uint32_t* tab, uint32_t k) {
  for (uint32_t i = hot_hash(k), t = 0; t < kHotTab; ++t, i = (i + 1) & (kHotTab - 1)) {
    const uint32_t v = tab[i];
    if (v == k) return i;
    if (v == kHotNone) return kHotNone;
  }
  return kHotNone;
}

template <bool PACK16, int KB = 4>
__device__ __forceinline__ void hist_ingest_flush(const void* __restrict__ keys_v, uint64_t n, const ScanArgs& a,
                                                  uint32_t* sh_hist, uint64_t* red64, uint32_t* tsum_sh = nullptr,
                                                  VGrid vg = vgrid_hw()) {
  constexpr bool K16 = KB == 2;  // (uint16 keys; KB == 1: uint8 keys)
  constexpr bool NARROW = KB != 4;
  const uint32_t U = a.U, ldw = a.ldw;

  // Ingestion (eq:ingestion): one shared atomic per key; equal addresses inside one warp
  // instruction are merged by the shared-memory atomic unit (the CRN's equality merge).
  const KeySpan s = make_span(NARROW ? nullptr : static_cast<const int32_t*>(keys_v), NARROW ? 0 : n);
  const KeySpan16 s16 =
      make_span_narrow<NARROW ? KB : 2>(NARROW ? static_cast<const uint16_t*>(keys_v) : nullptr, NARROW ? n : 0);
  const uint32_t lane0 = threadIdx.x & 31;
  // hot keys of this launch (see kHotK); hot_on is uniform over the CTA
  __shared__ uint32_t s_tab[kHotTab], s_tcnt[kHotTab], s_hot[kHotK], s_hotc[kHotK];
  uint32_t hk[kHotK] = {kHotNone, kHotNone, kHotNone, kHotNone}, hc[kHotK] = {0u, 0u, 0u, 0u};
  bool hot_on = false;
  // (launches of > 300000 keys a CTA: below that only a key holding > 22 % of a CTA's keys can
  //  wrap — the exact fallback still covers it — and the sampling's ~1 us would show: batched c2
  //  steps, 270k keys a CTA, 17.7 -> 18.3 us)
#ifndef DIALSORT_HOT_GUARD_KEYS  // (A/B: a huge value turns the hot-key sampling off)
#define DIALSORT_HOT_GUARD_KEYS 300000ull
#endif
  // (hierarchical block steps, 16-bit keys: from 65535 keys a CTA — their steps are long, and a
  //  block concentrates its hot keys: Zipf(1.2) at n = 1e8, U = 2^20 had blocks of ~150k keys a
  //  CTA with a key holding 60 % of them; 1.06 ms with the 300000 guard, 0.61 with this one)
  const bool hot_guard = PACK16 && a.fused && n > (K16 ? 65535ull : DIALSORT_HOT_GUARD_KEYS) * vg.G;  // (uniform)
  // the sample: the keys of the thread's first vector (loaded again by the ingestion loop)
  uint32_t sk[4] = {kHotNone, kHotNone, kHotNone, kHotNone};
  const uint32_t iv = vg.b * blockDim.x + threadIdx.x;
  if (hot_guard) {  // (requested before the zeroing below)
    if (iv < (NARROW ? (uint32_t)s16.n8 : (uint32_t)s.n4)) {
      if constexpr (NARROW) {
        const int4 x = reinterpret_cast<const int4*>(reinterpret_cast<const char*>(s16.keys) + KB * s16.head)[iv];
        expand_narrow<NARROW ? KB : 2>(x, 0, a.enc, [&](int4 q, uint32_t g) {
          if (g == 0) sk[0] = (uint32_t)q.x, sk[1] = (uint32_t)q.y, sk[2] = (uint32_t)q.z, sk[3] = (uint32_t)q.w;
        });
      } else {
        const int4 x = s.body()[iv];
        sk[0] = (uint32_t)x.x, sk[1] = (uint32_t)x.y, sk[2] = (uint32_t)x.z, sk[3] = (uint32_t)x.w;
      }
    }
    for (uint32_t t = threadIdx.x; t < kHotTab; t += blockDim.x) s_tab[t] = kHotNone, s_tcnt[t] = 0;
  }
  // K1: zero the private histogram (ldw = W rounded up to 8 words; padding stays zero so the
  // merge may read whole uint4 groups).
  const uint32_t W4 = ldw / 4;
  uint4* h4 = reinterpret_cast<uint4*>(sh_hist);
  for (uint32_t i = threadIdx.x; i < W4; i += blockDim.x) h4[i] = make_uint4(0, 0, 0, 0);
  __syncthreads();
  // the thread's first batch of vectors (the loop's prologue; requesting it before the zeroing
  // measured 1.3 us slower on the single-call c2 step)
  constexpr int NV0 = NARROW ? kNarrowUnroll : kHistUnroll;
  int4 a0[NV0];
  if constexpr (NARROW)
    preload_vecs<NV0>(reinterpret_cast<const int4*>(reinterpret_cast<const char*>(s16.keys) + KB * s16.head),
                      (uint32_t)s16.n8, vg, a0);
  else
    preload_vecs<NV0>(s.body(), (uint32_t)s.n4, vg, a0);
  if (hot_guard) {
#pragma unroll
    for (uint32_t q = 0; q < 4; ++q)
      if (sk[q] >= U) sk[q] = kHotNone;
#pragma unroll
    for (uint32_t h = 0; h < 2; ++h) {  // candidates: lanes 0 and 16's first key if it recurs
      const uint32_t x = __shfl_sync(0xffffffffu, sk[0], 16 * h);
      uint32_t c = 0;
#pragma unroll
      for (uint32_t q = 0; q < 4; ++q) c += __popc(__ballot_sync(0xffffffffu, sk[q] == x));
      if (lane0 == 16 * h && x != kHotNone && c >= 3) hot_tab_insert(s_tab, x);
    }
    const uint32_t nsamp = 4 * __syncthreads_count(sk[0] != kHotNone || iv < (NARROW ? s16.n8 : s.n4));
#pragma unroll
    for (uint32_t q = 0; q < 4; ++q)
      if (sk[q] != kHotNone) {
        const uint32_t slot = hot_tab_find(s_tab, sk[q]);
        if (slot != kHotNone) atomicAdd(s_tcnt + slot, 1u);
      }
    __syncthreads();
    if (threadIdx.x < 32) {  // the kHotK largest counts above the routing threshold
      // count c of nsamp sampled keys -> ~ c n / (G nsamp) copies per CTA; route above 30000
      const uint64_t thr = nsamp ? (30000ull * nsamp * vg.G + n - 1) / n : ~0ull;
      uint32_t best[4];
#pragma unroll
      for (uint32_t q = 0; q < 4; ++q) {
        const uint32_t t = 4 * lane0 + q;
        best[q] = s_tab[t] != kHotNone && s_tcnt[t] >= thr ? (min(s_tcnt[t], 0x1ffffffu) << 7) | t : 0u;
      }
      for (uint32_t r = 0; r < kHotK; ++r) {
        uint32_t mine = max(max(best[0], best[1]), max(best[2], best[3]));
        const uint32_t top = __reduce_max_sync(0xffffffffu, mine);
        if (lane0 == 0) s_hot[r] = top ? s_tab[top & (kHotTab - 1)] : kHotNone, s_hotc[r] = 0;
#pragma unroll
        for (uint32_t q = 0; q < 4; ++q)
          if (top && best[q] == top) best[q] = 0;
      }
    }
    __syncthreads();
#pragma unroll
    for (uint32_t r = 0; r < kHotK; ++r) hk[r] = s_hot[r];
    hot_on = hk[0] != kHotNone;
  }
  DevStatus* st = a.st;
  uint32_t seen = 0, bad = 0, deferred = 0;
  // packed word of key k: k >> 1 at byte offset (k & ~1) * 2; increment 1 << 16 (k & 1) as a
  // wrapping funnel shift by 16 k (2 + 2 instructions a key instead of 5).  RED on the 32-bit
  // shared address, its base held in a register (an opaque mov: the compiler otherwise
  // re-derives the window base — four uniform instructions — at every vector)
  uint32_t hs;
  asm volatile("mov.b32 %0, %1;" : "=r"(hs) : "r"(smem_addr(sh_hist)));
  auto red_sh = [](uint32_t addr, uint32_t v) {
    asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
  };
  auto add16 = [&](uint32_t k) { red_sh(hs + 2 * (k & ~1u), __funnelshift_l(0u, 1u, k << 4)); };
  auto add32 = [&](uint32_t k) { red_sh(hs + 4 * k, 1u); };
  auto addn = [&](uint32_t k, uint32_t c) {  // c copies of key k (CRN output)
    if (PACK16)
      red_sh(hs + ((k + k) & ~3u), c << ((k & 1u) << 4));
    else
      red_sh(hs + 4 * k, c);
  };
  // Hot loop: a vector whose keys are all in [0,U) is ingested directly; a vector with an
  // out-of-range key is deferred to an out-of-loop checked pass (error path only), which
  // keeps calls and spills out of the loop body.
  //
  // CRN for runs (def:crn_level, lem:crn; lane-local accumulation P:859-864): a vector of 4
  // equal keys is one lane pair (k, 4).  When every active lane holds such a run (sorted /
  // reverse input), the warp groups its lanes by equality — one or two distinct keys are
  // found with a min/max reduction (REDUX) and ballots — and each group adds its total with
  // a single atomic.  Random inputs never take this path: one vote on (first == last key)
  // per vector rules it out for the whole warp.
  constexpr uint32_t kRunMiss = 8;
  uint32_t run_state = 0;  // vectors since the last run; >= kRunMiss: detection off
  // (hot keys counted in registers, the rest as usual; no run detection in such launches)
  auto addh = [&](uint32_t k) {
    if (k == hk[0]) ++hc[0];
    else if (k == hk[1]) ++hc[1];
    else if (k == hk[2]) ++hc[2];
    else if (k == hk[3]) ++hc[3];
    else add16(k);
  };
  auto f4 = [&](int4 v, uint32_t) {
    if (umax4(v) < U) {
      if (PACK16 && hot_on) {
        addh((uint32_t)v.x); addh((uint32_t)v.y); addh((uint32_t)v.z); addh((uint32_t)v.w);
        return;
      }
      // Run detection adapts per warp: after kRunMiss vectors in a row without a run of 4 in
      // any lane it is switched off for the rest of the launch (it costs ~0.5 us at c2, where
      // runs never occur, and is what makes sorted inputs fast; a warp's first vectors decide)
      if (run_state >= kRunMiss) {
        if (PACK16) {
          add16((uint32_t)v.x); add16((uint32_t)v.y); add16((uint32_t)v.z); add16((uint32_t)v.w);
        } else {
          add32((uint32_t)v.x); add32((uint32_t)v.y); add32((uint32_t)v.z); add32((uint32_t)v.w);
        }
        return;
      }
      const uint32_t act = __activemask();
      // (the full run test, not the cheaper x == w filter: under Zipf a quarter of the vectors
      // pass x == w, and 86% of the warps would take the slow path for nothing)
      const bool run4 = (v.x == v.y) & (v.y == v.z) & (v.z == v.w);
      const uint32_t runs = __ballot_sync(act, run4);
      if (runs == 0u) {  // no lane holds a run of 4: the common case
        ++run_state;
        if (PACK16) {
          add16((uint32_t)v.x); add16((uint32_t)v.y); add16((uint32_t)v.z); add16((uint32_t)v.w);
        } else {
          add32((uint32_t)v.x); add32((uint32_t)v.y); add32((uint32_t)v.z); add32((uint32_t)v.w);
        }
        return;
      }
      run_state = 0;
      if (runs == act) {
        const uint32_t k = (uint32_t)v.x, lane = threadIdx.x & 31;
        const uint32_t kmin = __reduce_min_sync(act, k), kmax = __reduce_max_sync(act, k);
        const uint32_t gmin = __ballot_sync(act, k == kmin), gmax = __ballot_sync(act, k == kmax);
        if ((gmin | gmax) == act) {  // at most two distinct keys in the warp
          if (lane == (uint32_t)(__ffs(gmin) - 1)) addn(kmin, 4u * __popc(gmin));
          if (kmax != kmin && lane == (uint32_t)(__ffs(gmax) - 1)) addn(kmax, 4u * __popc(gmax));
        } else {
          addn(k, 4u);
        }
      } else if (run4) {
        addn((uint32_t)v.x, 4u);
      } else if (PACK16) {
        add16((uint32_t)v.x); add16((uint32_t)v.y); add16((uint32_t)v.z); add16((uint32_t)v.w);
      } else {
        add32((uint32_t)v.x); add32((uint32_t)v.y); add32((uint32_t)v.z); add32((uint32_t)v.w);
      }
    } else {
      deferred = 1;
    }
  };
  auto f1 = [&](uint32_t k, uint64_t idx) {
    seen += 1;
    if (k < U) {
      if (PACK16) add16(k);
      else atomicAdd(sh_hist + k, 1u);
    } else {
      record_bad(st, idx, k);
      ++bad;
    }
  };
  if constexpr (NARROW) {
    seen += (16 / KB) * for_each_key_narrow<NARROW ? KB : 2>(s16, reinterpret_cast<int4(&)[kNarrowUnroll]>(a0), a.enc,
                                                             f4, f1, vg);
  } else {
    for_each_key4(s, reinterpret_cast<int4(&)[kHistUnroll]>(a0), f4, f1, vg);
    // vectors of this thread: every grid-stride index < n4 (counted, not tallied in the loop)
    const uint32_t stride = vg.G * blockDim.x, i0 = vg.b * blockDim.x + threadIdx.x;
    const uint32_t n4 = (uint32_t)s.n4;
    const uint32_t cnt = i0 < n4 ? (n4 - 1 - i0) / stride + 1 : 0;
    seen += 4 * cnt;
  }
  if (deferred) {
    if (NARROW) bad += ingest_deferred_narrow<PACK16, NARROW ? KB : 2>(sh_hist, s16, a.enc, U, st, vg);
    else bad += ingest_deferred<PACK16>(sh_hist, s, U, st, vg);
  }
  if (PACK16 && hot_on) {  // the hot keys' register counts: a CTA total per key
#pragma unroll
    for (uint32_t r = 0; r < kHotK; ++r) {
      const uint32_t c = __reduce_add_sync(0xffffffffu, hc[r]);
      if (lane0 == 0 && c) atomicAdd(s_hotc + r, c);
    }
  }
  phase_mark(a.pt, 0);
  __syncthreads();
  phase_mark(a.pt, 1);
  if (PACK16 && hot_on && threadIdx.x < kHotK && s_hot[threadIdx.x] != kHotNone && s_hotc[threadIdx.x]) {
    // whole into Hx (32-bit, merged with the rows) and into the key's tile sum
    red_add_u32(a.Hx + s_hot[threadIdx.x], s_hotc[threadIdx.x]);
    atomicAdd(tsum_sh + s_hot[threadIdx.x] / kFTileBins, s_hotc[threadIdx.x]);
  }

  // Flush the private histogram as partial row vg.b (4-, 16- or 32-bit counts) and this row's
  // 64-bin tile sums (tsum_sh) for the owner counters.
  const uint32_t lane = threadIdx.x & 31;
  uint32_t fsum = 0;  // <= the CTA's keys < 2^32
  if (a.fused && PACK16 && a.nib4) {
    // k_sort_fused, 4-bit rows: the partial row keeps counts <= 15 — 8 bins
    // per word, a quarter of the packed row's L2 bytes — and a count >= 16 goes whole to the
    // global exception histogram Hx (RED; its nibble stays 0).  Thread i turns packed uint4 i
    // (8 bins; consecutive threads read consecutive uint4: no bank conflicts — 4 uint4 per
    // thread measured 16-way conflicted) into word i of the row and adds its 8-bin sum to the
    // tile sum tsum_sh[i / 8] (shared atomic: the unit merges a warp's 4 equal addresses;
    // 3 shuffles per iteration cost more in the shared-memory pipe).
    constexpr uint32_t QT = kFTileBins / 8;  // packed uint4 per tile
    const uint32_t ntf = (U + kFTileBins - 1) / kFTileBins, tot = ntf * QT;
    const uint32_t lim = min(W4, (U + 7) / 8);  // uint4 g < lim: in the histogram and a row word
    uint32_t* wp = const_cast<uint32_t*>(a.partials) + (uint64_t)vg.b * a.ldr + threadIdx.x;
    uint32_t* tp = tsum_sh + threadIdx.x / QT;
    // 4 iterations' loads first: the shared atomics order the loop (smem may alias), so an
    // unbatched loop waits a full load latency per iteration
    constexpr uint32_t B = 4;
    for (uint32_t g0 = threadIdx.x; g0 - threadIdx.x < tot; g0 += B * 1024, wp += B * 1024, tp += B * 1024 / QT) {
      uint4 wv[B];
#pragma unroll
      for (uint32_t u = 0; u < B; ++u) wv[u] = g0 + u * 1024 < lim ? h4[g0 + u * 1024] : make_uint4(0, 0, 0, 0);
#pragma unroll
      for (uint32_t u = 0; u < B; ++u) {
        const uint32_t g = g0 + u * 1024;
        if (g >= lim) break;  // (uint4 lim .. tot hold bins >= U: zero)
        const uint4 w = wv[u];
        uint32_t word, v = 0;
        // (warp-uniform choice: a warp with one exception lane would otherwise run both paths —
        //  under Zipf nearly every warp of the flush has one)
        if (!__any_sync(__activemask(), ((w.x | w.y | w.z | w.w) & 0xFFF0FFF0u) != 0u)) {
          // fast path, all 8 counts <= 15: word j holds (c_{2j+1} << 16 | c_{2j}), so
          // (w | w >> 12) & 0xff = c_{2j} | c_{2j+1} << 4, and PRMT gathers the 4 bytes
          const uint32_t bx = w.x | (w.x >> 12), by = w.y | (w.y >> 12);
          const uint32_t bz = w.z | (w.z >> 12), bw = w.w | (w.w >> 12);
          word = __byte_perm(__byte_perm(bx, by, 0x0040), __byte_perm(bz, bw, 0x0040), 0x5410);
          const uint32_t sw = w.x + w.y + w.z + w.w;  // halves <= 60: no carry
          v = (sw & 0xffffu) + (sw >> 16);
        } else {
          // some count >= 16: it goes whole to Hx (RED) and its nibble stays 0; the other
          // counts pack as in the fast path
          uint32_t cw[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
          for (uint32_t k = 0; k < 4; ++k) {
            v += (cw[k] & 0xffffu) + (cw[k] >> 16);
            if (cw[k] & 0x0000FFF0u) {
              red_add_u32(a.Hx + 8 * g + 2 * k, cw[k] & 0xffffu);
              cw[k] &= 0xFFFF0000u;
            }
            if (cw[k] & 0xFFF00000u) {
              red_add_u32(a.Hx + 8 * g + 2 * k + 1, cw[k] >> 16);
              cw[k] &= 0x0000FFFFu;
            }
          }
          const uint32_t bx = cw[0] | (cw[0] >> 12), by = cw[1] | (cw[1] >> 12);
          const uint32_t bz = cw[2] | (cw[2] >> 12), bw = cw[3] | (cw[3] >> 12);
          word = __byte_perm(__byte_perm(bx, by, 0x0040), __byte_perm(bz, bw, 0x0040), 0x5410);
        }
        __stcg(wp + u * 1024, word);
        if (v) atomicAdd(tp + u * (1024 / QT), v);
      }
    }
  } else if (a.fused) {
    // k_sort_fused, 16- or 32-bit rows: thread i stores uint4 i of the row and adds its sum to
    // the tile sum tsum_sh[i / QT] (shared atomic).
    constexpr uint32_t QT = PACK16 ? kFTileBins / 8 : kFTileBins / 4;
    const uint32_t ntf = (U + kFTileBins - 1) / kFTileBins, tot4 = ntf * QT;
    uint4* frow4 = reinterpret_cast<uint4*>(const_cast<uint32_t*>(a.partials) + (uint64_t)vg.b * a.ldr);
    for (uint32_t i = threadIdx.x; i < tot4; i += blockDim.x) {
      if (i < W4) {
        const uint4 w = h4[i];
        __stcg(frow4 + i, w);
        uint32_t v;
        if (PACK16)
          v = (w.x & 0xffffu) + (w.x >> 16) + (w.y & 0xffffu) + (w.y >> 16) + (w.z & 0xffffu) + (w.z >> 16) +
              (w.w & 0xffffu) + (w.w >> 16);
        else
          v = w.x + w.y + w.z + w.w;
        if (v) atomicAdd(tsum_sh + i / QT, v);
      }
    }
  }
  if (a.fused) {  // fsum (the checksum) from the row's tile sums
    __syncthreads();
    const uint32_t ntf = (U + kFTileBins - 1) / kFTileBins;
    for (uint32_t t = threadIdx.x; t < ntf; t += blockDim.x) fsum += tsum_sh[t];
  }
  phase_mark(a.pt, 11);  // flush loop done (debug)
  // (uint4 beyond the last tile are padding zeros and are never read by the merge)
  if (PACK16) {
    // Packed counters: a 16-bit field that wrapped loses >= 65535 from the field sum
    // (DESIGN.md §5.2), so Σ fields == #valid keys  <=>  no field overflowed.  On overflow the
    // fallback zeroes the row and the CTA's tile sums are ignored (use_ovf path below).
    // fsum: per-warp totals in lane 0 (tsums loop) or per-tile totals in the tile's lane 0
    // One block sum of (field sums - valid keys), mod 2^32: the shortfall of a wrapped row is in
    // (0, keys of the CTA] and the CTA holds < 2^32 keys, so the sum is 0 iff nothing wrapped.
    const uint32_t dsum = block_sum<uint32_t>((a.fused || lane == 0 ? fsum : 0u) - (uint32_t)(seen - bad),
                                              reinterpret_cast<uint32_t*>(red64));
    const bool exact = dsum == 0u;
    // k_sort_fused: the row's owner totals (its tile sums summed per owning CTA) — only for
    // an exact row (an overflowed one is recounted after the barrier)
    if (tsum_sh && exact) flush_owner_totals(a, tsum_sh, U, reinterpret_cast<uint32_t*>(red64), vg);
    if (!exact) {
      if (a.fused) {
        // k_sort_fused rows: take back this CTA's exception REDs (the same wrapped field
        // values), then the fallback zeroes the row (ldr words) and re-ingests into ovfH
        if (a.nib4) {
          __syncthreads();
          for (uint32_t g = threadIdx.x; g < W4; g += blockDim.x) {
            const uint4 w = h4[g];
            const uint32_t cw[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
            for (uint32_t j = 0; j < 8; ++j) {
              const uint32_t c = (cw[j >> 1] >> ((j & 1u) << 4)) & 0xffffu;
              if (c >= 16u) red_add_u32(a.Hx + 8 * g + j, 0u - c);
            }
          }
        }
        // (and the hot keys' counts: the fallback re-ingests every key of the CTA)
        if (PACK16 && hot_on && threadIdx.x < kHotK && s_hot[threadIdx.x] != kHotNone && s_hotc[threadIdx.x])
          red_add_u32(a.Hx + s_hot[threadIdx.x], 0u - s_hotc[threadIdx.x]);
        uint4* frow = reinterpret_cast<uint4*>(const_cast<uint32_t*>(a.partials) + (uint64_t)vg.b * a.ldr);
        if (K16) hist_overflow_fallback16(s16, frow, a.ldr / 4, a.ovfH, U, st, a.epoch, vg);
        else hist_overflow_fallback(s, frow, a.ldr / 4, a.ovfH, U, st, a.epoch, vg);
      }
    }
  } else if (tsum_sh) {  // 32-bit rows cannot overflow
    __syncthreads();
    flush_owner_totals(a, tsum_sh, U, reinterpret_cast<uint32_t*>(red64), vg);
  }
  phase_mark(a.pt, 2);
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

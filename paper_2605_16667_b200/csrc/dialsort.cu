// dialsort.cu — C ABI (include/dialsort.h) and launch logic of the B200 DialSort hot path.
//
// Host side only decides paths, sizes grids and enqueues kernels; every step of the method
// runs in the kernels of ds_hist.cuh / ds_scan.cuh / ds_expand.cuh / ds_radix.cuh.
// All launches use programmatic dependent launch (PDL) so each kernel's launch overlaps
// its predecessor's tail; every kernel calls griddepcontrol.wait before touching its
// inputs, which keeps stream order exact.
#include "../../include/dialsort.h"

#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "ds_common.cuh"
#include "ds_expand.cuh"
#include "ds_fused.cuh"
#include "ds_hist.cuh"
#include "ds_part.cuh"
#include "ds_peer.cuh"
#include "ds_radix.cuh"
#include "ds_scan.cuh"

using namespace ds;

namespace {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

#define DS_CUDA(expr)                                                                        \
  do {                                                                                       \
    cudaError_t e_ = (expr);                                                                 \
    if (e_ != cudaSuccess)                                                                   \
      return fail(DIALSORT_E_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_));      \
  } while (0)

enum KernelId {
  KID_ZERO = 0, KID_HIST_SMEM32, KID_HIST_SMEM16, KID_HIST_GLOBAL, KID_SCAN, KID_EXPAND,
  KID_RADIX_HIST4, KID_RADIX_PASS, KID_RANGE_COUNT, KID_CRN, KID_SORT_FUSED, KID_PART_COUNT, KID_PART_SCAN,
  KID_PART_SCATTER, KID_PUSH_SLICES, KID_SLICE_SUM, KID_COUNT
};
const char* const kKernelNames[KID_COUNT] = {"k_zero", "k_hist_smem32", "k_hist_smem16", "k_hist_global",
                                             "k_scan", "k_expand", "k_radix_hist0", "k_radix_pass",
                                             "k_range_count", "k_crn_resolve", "k_sort_fused", "k_part_count",
                                             "k_part_scan", "k_part_scatter", "k_push_slices", "k_slice_sum"};

// Per-context launch profiler (off by default): an event pair around each launch.
struct Profiler {
  bool on = false;
  std::vector<cudaEvent_t> ev;  // 2 per record
  std::vector<int> ids;
  size_t used = 0;
};
thread_local Profiler* g_prof = nullptr;  // set by the API entry for the ctx in use

template <typename... KArgs, typename... Args>
cudaError_t launch_k(int kid, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                     Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  Profiler* P = g_prof;
  if (P && P->on) {
    if (2 * P->used + 2 > P->ev.size()) {
      for (int i = 0; i < 512; ++i) {
        cudaEvent_t e;
        cudaEventCreate(&e);
        P->ev.push_back(e);
      }
    }
    cudaEventRecord(P->ev[2 * P->used], s);
    cudaError_t r = cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
    cudaEventRecord(P->ev[2 * P->used + 1], s);
    P->ids.push_back(kid);
    P->used++;
    return r;
  }
  return cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

constexpr size_t kSmemBudget = 227 * 1024 - 4096;  // static smem of the kernels <= 4 KB
// k_sort_fused workspace: 2 parities of per-tile ready flags, 2 parities of strided owner
// totals, the fallback owner totals
constexpr uint64_t kFusedTileWords = 2ull * kFTileSlots + 2ull * kFOwnSlots * kTileTotStride + kFOwnSlots;

inline uint64_t cdiv(uint64_t a, uint64_t b) { return (a + b - 1) / b; }
inline uint64_t round_up(uint64_t a, uint64_t b) { return cdiv(a, b) * b; }

// A device buffer that only grows (reallocation happens outside any timed region: the first
// call with a larger size; callers size the context at create to avoid it).
struct DBuf {
  void* p = nullptr;
  size_t bytes = 0;
  int ensure(size_t want, bool zero = false) {
    if (want <= bytes && p) return DIALSORT_OK;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    want = want < 256 ? 256 : want;
    if (cudaMalloc(&p, want) != cudaSuccess) {
      cudaGetLastError();
      return fail(DIALSORT_E_NOMEM, "cudaMalloc of " + std::to_string(want) + " bytes failed");
    }
    if (zero && cudaMemset(p, 0, want) != cudaSuccess) return fail(DIALSORT_E_CUDA, "cudaMemset failed");
    bytes = want;
    return DIALSORT_OK;
  }
  template <typename T>
  T* as() const { return static_cast<T*>(p); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
};

}  // namespace

struct dialsort_ctx_s {
  int device = 0;
  int nsm = 148;
  uint32_t epoch = 0;
  DBuf partials, P, tfb, ws_total, ovfH, status, stage, Hws, range_tot, gridbar, tsums, radix_tmp, radix_hist,
      radix_lb, fused_tiles, Hx, part, htmp;
  DevStatus* host_status = nullptr;  // pinned mirror
  uint64_t fused_seq = 0;            // k_sort_fused launches (parity of the tile-total buffers)
  unsigned long long bar64_base = 0; // value of the monotonic barrier counter after the last launch
  Profiler prof;
  int expand_occ = 4, scan_occ = 2, radix_occ = 1, radix2_occ = 1, radix3_occ = 1, radix4_occ = 1;
  PhaseTimes* pt = nullptr;  // debug phase timing (DIALSORT_PHASE_TIMING=1)
};

namespace {

int ctx_init(dialsort_ctx c) {
  DS_CUDA(cudaSetDevice(c->device));
  cudaDeviceProp prop;
  DS_CUDA(cudaGetDeviceProperties(&prop, c->device));
  c->nsm = prop.multiProcessorCount;
  int rc;
  if ((rc = c->status.ensure(sizeof(DevStatus), true))) return rc;
  DS_CUDA(cudaMallocHost(&c->host_status, sizeof(DevStatus)));
  DevStatus clean = {};
  clean.first_bad = ~0ull;
  clean.ovf_epoch = ~0u;
  DS_CUDA(cudaMemcpy(c->status.p, &clean, sizeof(clean), cudaMemcpyHostToDevice));
  if ((rc = c->ws_total.ensure(64, true))) return rc;
  if ((rc = c->gridbar.ensure(64, true))) return rc;
  if ((rc = c->range_tot.ensure(8ull * 8 * c->nsm, true))) return rc;
  // k_sort_fused: tile totals (2 parities), fallback tile totals
  if ((rc = c->fused_tiles.ensure(4ull * kFusedTileWords, true))) return rc;
  DS_CUDA(cudaFuncSetAttribute(k_sort_fused<kRowU32, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBudget));
  DS_CUDA(cudaFuncSetAttribute(k_sort_fused<kRowP16, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBudget));
  DS_CUDA(cudaFuncSetAttribute(k_sort_fused<kRowN4, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBudget));
  DS_CUDA(cudaFuncSetAttribute(k_sort_fused<kRowU32, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBudget));
  DS_CUDA(cudaFuncSetAttribute(k_sort_fused<kRowP16, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBudget));
  DS_CUDA(cudaFuncSetAttribute(k_sort_fused<kRowN4, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBudget));
  DS_CUDA(cudaFuncSetAttribute(k_hist_fused<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBudget));
  DS_CUDA(cudaFuncSetAttribute(k_hist_fused<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBudget));
  DS_CUDA(cudaFuncSetAttribute(k_hist_fused<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBudget));
  DS_CUDA(cudaFuncSetAttribute(k_hist_fused<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBudget));
  radix_configure();
  int occ = 0;
  DS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_radix_pass, kRadixThreads, sizeof(RadixSmem)));
  c->radix_occ = occ > 0 ? occ : 1;
  DS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_radix_pass2, kRadixThreads, sizeof(RadixSmem)));
  c->radix2_occ = occ > 0 ? occ : 1;
  DS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_radix_pass3, kRadixThreads, sizeof(Radix3Smem)));
  c->radix3_occ = occ > 0 ? occ : 1;
  DS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_radix_pass4, kRadixThreads, sizeof(Radix4Smem)));
  c->radix4_occ = occ > 0 ? occ : 1;
  DS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_expand, kExpandThreads, 0));
  c->expand_occ = occ > 0 ? occ : 1;
  DS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_scan, kTileBins, 0));
  c->scan_occ = occ > 0 ? (occ > 4 ? 4 : occ) : 1;
  const char* e = getenv("DIALSORT_PHASE_TIMING");
  if (e && e[0] == '1') {
    DS_CUDA(cudaMalloc(&c->pt, sizeof(PhaseTimes)));
    DS_CUDA(cudaMemset(c->pt, 0, sizeof(PhaseTimes)));
  }
  return DIALSORT_OK;
}

// Bumps the call epoch (tags the packed-overflow flag and the radix look-back statuses).
uint32_t next_epoch(dialsort_ctx c, cudaStream_t s) {
  c->epoch = (c->epoch + 1) & 0xffffffu;
  if (c->epoch == 0) c->epoch = 1;
  return c->epoch;
}

int check_keys_arg(const void* p, uint64_t n) {
  if (n > 0xffffffffull) return fail(DIALSORT_E_INVALID_ARG, "n exceeds 2^32-1");
  if (n > 0 && p == nullptr) return fail(DIALSORT_E_INVALID_ARG, "NULL pointer with n > 0");
  if (reinterpret_cast<uintptr_t>(p) & 3u) return fail(DIALSORT_E_INVALID_ARG, "pointer not 4-byte aligned");
  return DIALSORT_OK;
}
int check_U(uint32_t U) {
  if (U == 0 || U > 0x80000000u) return fail(DIALSORT_E_INVALID_ARG, "U must be in [1, 2^31]");
  return DIALSORT_OK;
}

enum class HistPath { Smem32, Smem16, Global };
HistPath choose_path(uint32_t U) {
  if (U <= kSmem32MaxBins) return HistPath::Smem32;
  if (U <= kSmem16MaxBins) return HistPath::Smem16;
  return HistPath::Global;
}

// Histogram ingestion variant: register pipeline (default) or TMA-fed ring (DIALSORT_HIST=tma,
// kept for A/B: measured 12.7 vs 10.2 us ingest at c2 — 3 x 32 KB stages fit beside the
// 128 KB histogram, fewer bytes in flight than 2 x 4 int4 per thread).
bool hist_use_tma() {
  static const bool tma = [] {
    const char* e = getenv("DIALSORT_HIST");
    return e && strcmp(e, "tma") == 0;
  }();
  return tma;
}

// Common scan arguments (workspace pointers, output tiling, size check).
int fill_scan_args(dialsort_ctx c, ScanArgs& a, uint32_t U, bool do_scan, uint64_t cap, bool exact, uint64_t* d_total,
                   uint32_t epoch) {
  int rc;
  const uint64_t ntiles_out = cap ? cdiv(cap, kExpandTile) : 1;
  if (do_scan) {
    if ((rc = c->P.ensure(4ull * (U + 1)))) return rc;
    if ((rc = c->tfb.ensure(4ull * ntiles_out))) return rc;
  }
  a.U = U;
  a.do_scan = do_scan;
  a.P = c->P.as<uint32_t>();
  a.range_tot = c->range_tot.as<uint64_t>();
  a.tfb = c->tfb.as<uint32_t>();
  a.T = kExpandTile;
  a.ntiles_out = ntiles_out;
  a.n_expected = cap;
  a.exact = exact;
  a.d_total = d_total;
  a.ws_total = c->ws_total.as<uint64_t>();
  a.st = c->status.as<DevStatus>();
  a.bar = c->gridbar.as<GridBar>();
  a.epoch = epoch;
  a.pt = c->pt;
  return DIALSORT_OK;
}

// Histogram of keys into H; when do_scan, also P / tfb for a projection of `cap` outputs.
// Smem paths: one fused co-resident kernel.  Global path: zero + L2 ingest + k_scan.
int enqueue_hist_scan(dialsort_ctx c, const int32_t* keys, uint64_t n, uint32_t U, uint32_t* H, bool do_scan,
                      uint64_t cap, uint32_t epoch, cudaStream_t s, uint32_t* const* Hpeer = nullptr,
                      uint32_t peerL = 0, uint32_t peerRank = 0) {
  int rc;
  ScanArgs a = {};
  if ((rc = fill_scan_args(c, a, U, do_scan, cap, true, nullptr, epoch))) return rc;
  a.Hpeer = Hpeer;  // (smem paths only: the merge stores into the owners' slots)
  a.peerL = peerL;
  a.peerRank = peerRank;
  const HistPath path = choose_path(U);
  if (path == HistPath::Global) {
    DS_CUDA(launch_k(KID_ZERO, k_zero, dim3(c->nsm * 4), dim3(256), 0, s, H, (uint64_t)U));
    const uint64_t want = cdiv(n / 4 + 1, 256ull * kHistUnroll);
    const uint64_t capg = (uint64_t)c->nsm * 8;
    const uint32_t grid = (uint32_t)(want < capg ? (want ? want : 1) : capg);
    DS_CUDA(launch_k(KID_HIST_GLOBAL, k_hist_global, dim3(grid), dim3(256), 0, s, keys, n, U, H, a.st));
    if (!do_scan) return DIALSORT_OK;
    a.Hsrc = H;
    const uint64_t ntiles = cdiv(U, kTileBins);
    const uint64_t wave = (uint64_t)c->nsm * c->scan_occ;
    DS_CUDA(launch_k(KID_SCAN, k_scan, dim3((uint32_t)(ntiles < wave ? ntiles : wave)), dim3(kTileBins), 0, s, a));
    return DIALSORT_OK;
  }
  const bool pack = path == HistPath::Smem16;
  const uint32_t W = pack ? (U + 1) / 2 : U;
  const uint32_t ldw = (uint32_t)round_up(W, 8);
  const size_t hist_bytes = std::max<size_t>(4ull * ldw, 32 * 1024);
  // TMA-fed ingestion only on request (DIALSORT_HIST=tma)
  uint32_t stages = 0;
  if (hist_use_tma()) {
    stages = (uint32_t)std::min<size_t>(kMaxStages, (kSmemBudget - hist_bytes) / kChunkBytes);
    if (stages < 2) stages = 0;
  }
  const size_t smem = hist_bytes + (size_t)stages * kChunkBytes;
  const uint64_t n4 = n / 4 + 1;
  const uint64_t want = stages ? cdiv(4 * n4, kChunkBytes / 4) : cdiv(n4, 1024ull * kHistUnroll * 2);
  const uint32_t C = (uint32_t)(want < (uint64_t)c->nsm ? (want ? want : 1) : c->nsm);
  if ((rc = c->partials.ensure(4ull * C * ldw))) return rc;
  if ((rc = c->ovfH.ensure(4ull * U, true))) return rc;
  if ((rc = c->tsums.ensure(4ull * C * cdiv(U, kTileBins)))) return rc;
  a.tsums = c->tsums.as<uint32_t>();
  a.partials = c->partials.as<uint32_t>();
  a.C = C;
  a.ldw = ldw;
  a.pack16 = pack;
  a.ovfH = c->ovfH.as<uint32_t>();
  a.H = H;
  const int kid = pack ? KID_HIST_SMEM16 : KID_HIST_SMEM32;
  if (pack && stages)
    DS_CUDA(launch_k(kid, k_hist_fused<true, true>, dim3(C), dim3(1024), smem, s, keys, n, a, stages));
  else if (pack)
    DS_CUDA(launch_k(kid, k_hist_fused<true, false>, dim3(C), dim3(1024), smem, s, keys, n, a, stages));
  else if (stages)
    DS_CUDA(launch_k(kid, k_hist_fused<false, true>, dim3(C), dim3(1024), smem, s, keys, n, a, stages));
  else
    DS_CUDA(launch_k(kid, k_hist_fused<false, false>, dim3(C), dim3(1024), smem, s, keys, n, a, stages));
  return DIALSORT_OK;
}

// Scan of a caller histogram (reconstruct API).
int enqueue_scan(dialsort_ctx c, const uint32_t* H, uint32_t U, uint64_t cap, bool exact, uint64_t* d_total,
                 uint32_t epoch, cudaStream_t s) {
  int rc;
  ScanArgs a = {};
  if ((rc = fill_scan_args(c, a, U, true, cap, exact, d_total, epoch))) return rc;
  a.Hsrc = H;
  const uint64_t ntiles = cdiv(U, kTileBins);
  const uint64_t wave = (uint64_t)c->nsm * c->scan_occ;
  DS_CUDA(launch_k(KID_SCAN, k_scan, dim3((uint32_t)(ntiles < wave ? ntiles : wave)), dim3(kTileBins), 0, s, a));
  return DIALSORT_OK;
}

int enqueue_expand(dialsort_ctx c, uint32_t U, uint64_t cap, int32_t key_base, int32_t* out, cudaStream_t s) {
  if (cap == 0) return DIALSORT_OK;
  const uint64_t ntiles_out = cdiv(cap, kExpandTile);
  const uint64_t wave = (uint64_t)c->nsm * c->expand_occ;  // persistent grid: one wave
  const uint32_t grid = (uint32_t)(ntiles_out < wave ? ntiles_out : wave);
  DS_CUDA(launch_k(KID_EXPAND, k_expand, dim3(grid), dim3(kExpandThreads), 0, s, c->P.as<const uint32_t>(), U,
                     c->tfb.as<const uint32_t>(), ntiles_out, c->ws_total.as<const uint64_t>(), cap, key_base, out,
                     c->pt));
  return DIALSORT_OK;
}

// The whole sort step as one kernel (ds_fused.cuh) for the shared-memory paths.
// DIALSORT_FUSED=0 selects the two-kernel pipeline (k_hist_fused + k_expand) for A/B.
bool sort_fused_enabled() {
  static const bool v = [] {
    const char* e = getenv("DIALSORT_FUSED");
    return !(e && e[0] == '0');
  }();
  return v;
}

// d_n / d_off (nullable): the key count and the keys/out offset are on the device (a universe
// block of the hierarchical path); n is then only the size hint for the grid and row format.
// k16: keys are uint16 (the hierarchical path's universe blocks), else int32.
int enqueue_sort_fused(dialsort_ctx c, const void* keys, uint64_t n, uint32_t U, uint32_t* H, int32_t* out,
                       uint32_t epoch, cudaStream_t s, int32_t key_base = 0, const uint64_t* d_n = nullptr,
                       const uint64_t* d_off = nullptr, bool k16 = false) {
  int rc;
  ScanArgs a = {};
  if ((rc = fill_scan_args(c, a, U, true, n, true, nullptr, epoch))) return rc;
  a.d_n = d_n;
  a.d_off = d_off;
  const bool pack = choose_path(U) == HistPath::Smem16;
  const uint32_t W = pack ? (U + 1) / 2 : U;
  const uint32_t ldw = (uint32_t)round_up(W, 8);  // shared-memory histogram words
  const uint64_t n4 = n / 4 + 1;
  const uint64_t want = cdiv(n4, 1024ull * kHistUnroll * 2);
  const uint64_t cmax = std::min<uint64_t>(c->nsm, kFMaxRows);  // rows a staging slot holds
  const uint32_t C = (uint32_t)(want < cmax ? (want ? want : 1) : cmax);
  // partial-row format: 4-bit rows while counts per CTA and bin are small (mean <= 8: counts
  // >= 16 — exceptions, one RED each — stay rare), else the packed 16-bit rows
  const int fmt = !pack ? kRowU32 : (n <= 8ull * C * U ? kRowN4 : kRowP16);
  const uint32_t ldr = fmt == kRowN4 ? (uint32_t)round_up((U + 7) / 8, 8) : ldw;  // row words
  const size_t smem = std::max<size_t>(4ull * ldw, 4ull * kFSmemWords);  // histogram | merge + projection
  if ((rc = c->partials.ensure(4ull * C * std::max(ldw, ldr)))) return rc;
  if ((rc = c->ovfH.ensure(4ull * U, true))) return rc;
  if ((rc = c->Hx.ensure(8ull * kSmem16MaxBins, true))) return rc;
  uint32_t* ft = c->fused_tiles.as<uint32_t>();
  a.partials = c->partials.as<uint32_t>();
  a.C = C;
  a.ldw = ldw;
  a.ldr = ldr;
  a.pack16 = pack;
  a.nib4 = fmt == kRowN4;
  a.ovfH = c->ovfH.as<uint32_t>();
  a.H = H;
  a.tfb = nullptr;
  a.tsums = nullptr;
  a.fused = 1;
  a.ctr_stride = kTileTotStride;
  // per-tile ready flags (share mode), two parities: each launch clears the other one, so a
  // flag never holds a value from an earlier launch (the epoch wraps after 2^24 launches)
  uint32_t* rdy = ft;
  a.ready = rdy + kFTileSlots * (c->fused_seq & 1);
  a.ready_clear = rdy + kFTileSlots * ((c->fused_seq + 1) & 1);
  uint32_t* ownb = rdy + 2 * kFTileSlots;
  const uint64_t own_words = (uint64_t)kFOwnSlots * kTileTotStride;  // per parity
  a.own_red = ownb + own_words * (c->fused_seq & 1);
  a.own_clear = ownb + own_words * ((c->fused_seq + 1) & 1);
  a.own_alt = ownb + 2 * own_words;
  // exception histogram of the 4-bit rows: parity buffers, the other one cleared by every launch
  a.Hx = c->Hx.as<uint32_t>() + (uint64_t)kSmem16MaxBins * (c->fused_seq & 1);
  a.Hx_clear = c->Hx.as<uint32_t>() + (uint64_t)kSmem16MaxBins * ((c->fused_seq + 1) & 1);
  a.bar64 = reinterpret_cast<unsigned long long*>(c->gridbar.as<char>() + 16);
  a.bar_base = c->bar64_base;
#define DS_LAUNCH_FUSED(F, K)                                                                                 \
  DS_CUDA(launch_k(KID_SORT_FUSED, k_sort_fused<F, K>, dim3(C), dim3(1024), smem, s, keys, n, a, out, key_base))
  if (fmt == kRowN4) {
    if (k16) DS_LAUNCH_FUSED(kRowN4, true); else DS_LAUNCH_FUSED(kRowN4, false);
  } else if (fmt == kRowP16) {
    if (k16) DS_LAUNCH_FUSED(kRowP16, true); else DS_LAUNCH_FUSED(kRowP16, false);
  } else {
    if (k16) DS_LAUNCH_FUSED(kRowU32, true); else DS_LAUNCH_FUSED(kRowU32, false);
  }
#undef DS_LAUNCH_FUSED
  c->fused_seq++;
  c->bar64_base += 2ull * C;  // two barriers reserved per launch (one skipped unless overflow)
  return DIALSORT_OK;
}

// Hierarchical DialSort for 98304 < U <= 2^22 (ds_part.cuh): MSD split into 65536-bin universe
// blocks, then one k_sort_fused per block (device-resident block sizes / offsets: no host
// round trip).  DIALSORT_HIER=0 selects the L2 path (one RED per distinct key per warp).
bool hier_enabled() {
  static const bool v = [] {
    const char* e = getenv("DIALSORT_HIER");
    return !(e && e[0] == '0');
  }();
  return v;
}
bool hier_applies(uint32_t U) {
  return U > kSmem16MaxBins && (uint64_t)U <= ((uint64_t)kPartMaxBlocks << kPartShift) && hier_enabled() &&
         sort_fused_enabled();
}

int enqueue_sort_hier(dialsort_ctx c, const int32_t* keys, uint64_t n, uint32_t U, uint32_t* H, int32_t* out,
                      cudaStream_t s) {
  int rc;
  const uint32_t B = (uint32_t)cdiv(U, 1ull << kPartShift);
#ifndef DIALSORT_PART_CTAS_PER_SM
#define DIALSORT_PART_CTAS_PER_SM (2048 / DIALSORT_PART_THREADS)
#endif
  const uint32_t Gp = (uint32_t)std::max<uint64_t>(
      1, std::min<uint64_t>((uint64_t)DIALSORT_PART_CTAS_PER_SM * c->nsm, cdiv(n, kPartTile)));
  if ((rc = c->part.ensure(4ull * Gp * B + 16ull * B + 64))) return rc;
  if ((rc = c->htmp.ensure(2ull * n + 16))) return rc;  // uint16 block keys
  PartWs w;
  w.bsz = c->part.as<uint64_t>();
  w.boff = w.bsz + B;
  w.cnt = reinterpret_cast<uint32_t*>(w.boff + B);
  w.st = c->status.as<DevStatus>();
  uint16_t* tmp = c->htmp.as<uint16_t>();
  DS_CUDA(launch_k(KID_PART_COUNT, k_part_count, dim3(Gp), dim3(kPartThreads), 0, s, keys, n, U, B, w));
  DS_CUDA(launch_k(KID_PART_SCAN, k_part_scan, dim3(1), dim3(1024), 0, s, Gp, B, w));
  DS_CUDA(launch_k(KID_PART_SCATTER, k_part_scatter, dim3(Gp), dim3(kPartThreads), 0, s, keys, n, U, B, w, tmp));
  for (uint32_t b = 0; b < B; ++b) {
    const uint32_t Ub = (uint32_t)std::min<uint64_t>(1ull << kPartShift, (uint64_t)U - ((uint64_t)b << kPartShift));
    const uint32_t epoch = next_epoch(c, s);  // each block launch has its own ready-flag epoch
    if ((rc = enqueue_sort_fused(c, tmp, cdiv(n, B), Ub, H + ((uint64_t)b << kPartShift), out, epoch, s,
                                 (int32_t)(b << kPartShift), w.bsz + b, w.boff + b, true)))
      return rc;
  }
  return DIALSORT_OK;
}

// Host-side enqueue of DialSort-Radix.  Default: 4 reduce-then-scan passes with 8192-key
// sub-tiles, TMA-staged when the buffers are 16-byte aligned (k_radix_pass4, else pass3;
// co-resident grid).  DIALSORT_RADIX=pass3 / pass2 / onesweep select the other variants (A/B).
const char* radix_variant() {
  static const char* v = [] {
    const char* e = getenv("DIALSORT_RADIX");
    return e ? e : "pass4";
  }();
  return v;
}
bool radix_onesweep() { return strcmp(radix_variant(), "onesweep") == 0; }

int radix_enqueue(dialsort_ctx c, const int32_t* keys, uint64_t n, int32_t* out, int32_t* tmp, cudaStream_t s) {
  if (n >= (1ull << 30)) return fail(DIALSORT_E_INVALID_ARG, "radix path supports n < 2^30 per call");
  int rc;
  const uint32_t* src = reinterpret_cast<const uint32_t*>(keys);
  uint32_t* bufs[2] = {reinterpret_cast<uint32_t*>(tmp), reinterpret_cast<uint32_t*>(out)};
  if (!radix_onesweep()) {
    const bool p3 = strcmp(radix_variant(), "pass2") != 0;
    // pass4 (TMA-staged) needs 16-byte aligned buffers: keys, tmp and out of every pass
    const bool p4 = p3 && strcmp(radix_variant(), "pass3") != 0 && ((reinterpret_cast<uintptr_t>(keys) & 15u) == 0) &&
                    ((reinterpret_cast<uintptr_t>(out) & 15u) == 0) && ((reinterpret_cast<uintptr_t>(tmp) & 15u) == 0);
    const uint32_t G = (uint32_t)std::max<uint64_t>(
        1, std::min<uint64_t>(cdiv(n, p3 ? kR3Tile : kRadixTile),
                              (uint64_t)c->nsm * (p4 ? c->radix4_occ : p3 ? c->radix3_occ : c->radix2_occ)));
    if ((rc = c->radix_hist.ensure(8ull * 256 * G + 4 * 256 + 64))) return rc;
    Radix2Ws w;
    w.cnt = c->radix_hist.as<uint32_t>();
    w.pre = w.cnt + 256 * G;
    w.total = w.pre + 256 * G;
    w.bar = reinterpret_cast<GridBarR*>(c->gridbar.as<char>() + 32);
    w.pt = c->pt;
    for (int p = 0; p < 4; ++p) {
      uint32_t* dst = bufs[p & 1];
      if (p4)
        DS_CUDA(launch_k(KID_RADIX_PASS, k_radix_pass4, dim3(G), dim3(kRadixThreads), sizeof(Radix4Smem), s, src, dst,
                         (uint32_t)n, p, w));
      else if (p3)
        DS_CUDA(launch_k(KID_RADIX_PASS, k_radix_pass3, dim3(G), dim3(kRadixThreads), sizeof(Radix3Smem), s, src, dst,
                         (uint32_t)n, p, w));
      else
        DS_CUDA(launch_k(KID_RADIX_PASS, k_radix_pass2, dim3(G), dim3(kRadixThreads), sizeof(RadixSmem), s, src, dst,
                         (uint32_t)n, p, w));
      src = dst;
    }
    return DIALSORT_OK;
  }
  const uint32_t ntiles = (uint32_t)cdiv(n, kRadixTile);
  if ((rc = c->radix_hist.ensure(4 * 1024 + 64))) return rc;
  if ((rc = c->radix_lb.ensure(2ull * 4 * 256 * ntiles + 16))) return rc;
  RadixWs w;
  w.ghist = c->radix_hist.as<uint32_t>();
  w.ctrs = w.ghist + 1024;
  w.status = c->radix_lb.as<uint32_t>();
  w.ntiles = ntiles;
  const uint32_t g0 = (uint32_t)std::min<uint64_t>(cdiv(n / 4 + 1, 512ull * 4), (uint64_t)c->nsm * 4);
  DS_CUDA(launch_k(KID_ZERO, k_zero, dim3(1), dim3(256), 0, s, w.ghist, (uint64_t)256));
  DS_CUDA(launch_k(KID_RADIX_HIST4, k_radix_hist0, dim3(g0), dim3(512), 0, s, keys, n, w));
  const uint32_t gp = (uint32_t)std::min<uint64_t>(ntiles, (uint64_t)c->nsm * c->radix_occ);
  for (int p = 0; p < 4; ++p) {
    uint32_t* dst = bufs[p & 1];
    DS_CUDA(launch_k(KID_RADIX_PASS, k_radix_pass, dim3(gp), dim3(kRadixThreads), sizeof(RadixSmem), s, src, dst,
                     (uint32_t)n, p, w));
    src = dst;
  }
  return DIALSORT_OK;
}

// Makes `c`'s profiler the active one for launches made by this thread during an API call.
struct ProfScope {
  Profiler* prev;
  explicit ProfScope(dialsort_ctx c) : prev(g_prof) { g_prof = c ? &c->prof : nullptr; }
  ~ProfScope() { g_prof = prev; }
};

std::mutex g_default_mu;
std::map<int, dialsort_ctx> g_default;

int default_ctx(dialsort_ctx* out) {
  int dev = 0;
  DS_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_default_mu);
  auto it = g_default.find(dev);
  if (it != g_default.end()) {
    *out = it->second;
    return DIALSORT_OK;
  }
  dialsort_ctx c = nullptr;
  int rc = dialsort_ctx_create(dev, 0, 0, &c);
  if (rc) return rc;
  g_default[dev] = c;
  *out = c;
  return DIALSORT_OK;
}

bool ranges_overlap(const void* a, uint64_t na, const void* b, uint64_t nb) {
  uintptr_t a0 = reinterpret_cast<uintptr_t>(a), b0 = reinterpret_cast<uintptr_t>(b);
  return a0 < b0 + nb && b0 < a0 + na;
}

}  // namespace

extern "C" {

const char* dialsort_status_string(int s) {
  switch (s) {
    case DIALSORT_OK: return "ok";
    case DIALSORT_E_INVALID_ARG: return "invalid argument";
    case DIALSORT_E_KEY_RANGE: return "key outside [0,U)";
    case DIALSORT_E_SIZE: return "size mismatch (sum(H) vs n)";
    case DIALSORT_E_OVERFLOW: return "count overflow";
    case DIALSORT_E_CUDA: return "CUDA error";
    case DIALSORT_E_NOMEM: return "out of device memory";
    default: return "unknown status";
  }
}

const char* dialsort_last_error(void) { return g_last_error.c_str(); }
int dialsort_version(void) { return 100; }

int dialsort_ctx_create(int device, uint64_t max_n, uint32_t max_U, dialsort_ctx* out) {
  if (!out) return fail(DIALSORT_E_INVALID_ARG, "out is NULL");
  dialsort_ctx c = new dialsort_ctx_s();
  c->device = device;
  int rc = ctx_init(c);
  if (!rc && max_U) {
    const HistPath path = choose_path(max_U);
    if (path != HistPath::Global) {
      const uint64_t W = path == HistPath::Smem16 ? (max_U + 1) / 2 : max_U;
      rc = c->partials.ensure(4ull * c->nsm * round_up(W, 8));
    }
    if (!rc) rc = c->P.ensure(4ull * (max_U + 1));
    if (!rc) rc = c->ovfH.ensure(4ull * max_U, true);
    if (!rc) rc = c->Hws.ensure(4ull * max_U);
  }
  if (!rc && max_n) rc = c->tfb.ensure(4ull * (cdiv(max_n, kExpandTile) + 1));
  if (rc) {
    dialsort_ctx_destroy(c);
    return rc;
  }
  *out = c;
  return DIALSORT_OK;
}

int dialsort_ctx_destroy(dialsort_ctx c) {
  if (!c) return DIALSORT_OK;
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  for (DBuf* b : {&c->partials, &c->P, &c->tfb, &c->ws_total, &c->ovfH, &c->status, &c->stage, &c->Hws,
                  &c->range_tot, &c->gridbar, &c->tsums, &c->radix_tmp, &c->radix_hist, &c->radix_lb,
                  &c->fused_tiles, &c->Hx, &c->part, &c->htmp})
    b->release();
  if (c->host_status) cudaFreeHost(c->host_status);
  if (c->pt) cudaFree(c->pt);
  for (cudaEvent_t e : c->prof.ev) cudaEventDestroy(e);
  delete c;
  return DIALSORT_OK;
}

int dialsort_sync(dialsort_ctx c, dialsort_stream_t stream, dialsort_error_info* info) {
  if (!c) return fail(DIALSORT_E_INVALID_ARG, "ctx is NULL");
  cudaStream_t s = (cudaStream_t)stream;
  DS_CUDA(cudaSetDevice(c->device));
  DS_CUDA(cudaMemcpyAsync(c->host_status, c->status.p, sizeof(DevStatus), cudaMemcpyDeviceToHost, s));
  DS_CUDA(cudaStreamSynchronize(s));
  DevStatus h = *c->host_status;
  DevStatus clean = {};
  clean.first_bad = ~0ull;
  clean.ovf_epoch = h.ovf_epoch;
  clean.last_total = h.last_total;
  if (h.bad_count || h.flags) DS_CUDA(cudaMemcpy(c->status.p, &clean, sizeof(clean), cudaMemcpyHostToDevice));
  if (info) {
    info->bad_count = h.bad_count;
    info->first_bad_index = h.bad_count ? (h.first_bad >> 32) : ~0ull;
    info->first_bad_key = h.bad_count ? (int32_t)(uint32_t)(h.first_bad & 0xffffffffu) : 0;
    info->flags = h.flags;
    info->last_total = h.last_total;
  }
  if (h.bad_count) {
    char buf[160];
    snprintf(buf, sizeof buf, "%llu key(s) outside [0,U); first at index %llu (key %d)",
             (unsigned long long)h.bad_count, (unsigned long long)(h.first_bad >> 32),
             (int32_t)(uint32_t)(h.first_bad & 0xffffffffu));
    return fail(DIALSORT_E_KEY_RANGE, buf);
  }
  if (h.flags & FLAG_OVERFLOW) return fail(DIALSORT_E_OVERFLOW, "sum(H) >= 2^32");
  if (h.flags & FLAG_SIZE)
    return fail(DIALSORT_E_SIZE, "sum(H) = " + std::to_string(h.last_total) + " does not match n / capacity");
  return DIALSORT_OK;
}

int dialsort_histogram_async(dialsort_ctx c, const int32_t* keys, uint64_t n, uint32_t U, uint32_t* H,
                             dialsort_stream_t stream) {
  int rc;
  if (!c) return fail(DIALSORT_E_INVALID_ARG, "ctx is NULL");
  ProfScope prof_scope_(c);
  if ((rc = check_U(U)) || (rc = check_keys_arg(keys, n))) return rc;
  if (!H) return fail(DIALSORT_E_INVALID_ARG, "H is NULL");
  cudaStream_t s = (cudaStream_t)stream;
  DS_CUDA(cudaSetDevice(c->device));
  const uint32_t epoch = next_epoch(c, s);
  if (n == 0) {
    DS_CUDA(launch_k(KID_ZERO, k_zero, dim3(c->nsm), dim3(256), 0, s, H, (uint64_t)U));
    return DIALSORT_OK;
  }
  return enqueue_hist_scan(c, keys, n, U, H, false, 0, epoch, s);
}

int dialsort_histogram_scatter_async(dialsort_ctx c, const int32_t* keys, uint64_t n, uint32_t U, uint32_t G,
                                     uint32_t rank, uint32_t* const* peer_recv, dialsort_stream_t stream) {
  int rc;
  if (!c) return fail(DIALSORT_E_INVALID_ARG, "ctx is NULL");
  ProfScope prof_scope_(c);
  if ((rc = check_U(U)) || (rc = check_keys_arg(keys, n))) return rc;
  if (G == 0 || U % G != 0 || rank >= G) return fail(DIALSORT_E_INVALID_ARG, "need U % G == 0 and rank < G");
  if (!peer_recv) return fail(DIALSORT_E_INVALID_ARG, "peer_recv is NULL");
  cudaStream_t s = (cudaStream_t)stream;
  DS_CUDA(cudaSetDevice(c->device));
  const uint32_t epoch = next_epoch(c, s);
  const uint32_t L = U / G;
  if (n > 0 && choose_path(U) != HistPath::Global)  // one kernel: histogram, merge, P2P stores
    return enqueue_hist_scan(c, keys, n, U, nullptr, false, 0, epoch, s, peer_recv, L, rank);
  // L2 path (or no keys): the local histogram, then one push kernel
  if ((rc = c->Hws.ensure(4ull * U + 16))) return rc;
  uint32_t* H = c->Hws.as<uint32_t>();
  if (n == 0)
    DS_CUDA(launch_k(KID_ZERO, k_zero, dim3(c->nsm), dim3(256), 0, s, H, (uint64_t)U));
  else if ((rc = enqueue_hist_scan(c, keys, n, U, H, false, 0, epoch, s)))
    return rc;
  DS_CUDA(launch_k(KID_PUSH_SLICES, k_push_slices, dim3(2 * c->nsm), dim3(256), 0, s, (const uint32_t*)H, U, L, rank,
                   peer_recv));
  return DIALSORT_OK;
}

int dialsort_slice_sum_async(dialsort_ctx c, const uint32_t* recv, uint32_t G, uint32_t L, uint32_t* H_slice,
                             dialsort_stream_t stream) {
  if (!c) return fail(DIALSORT_E_INVALID_ARG, "ctx is NULL");
  ProfScope prof_scope_(c);
  if (!recv || !H_slice || G == 0 || L == 0) return fail(DIALSORT_E_INVALID_ARG, "bad slice-sum arguments");
  cudaStream_t s = (cudaStream_t)stream;
  DS_CUDA(cudaSetDevice(c->device));
  const uint32_t grid = (uint32_t)std::min<uint64_t>(2ull * c->nsm, cdiv(L, 256));
  DS_CUDA(launch_k(KID_SLICE_SUM, k_slice_sum, dim3(grid), dim3(256), 0, s, recv, G, L, H_slice));
  return DIALSORT_OK;
}

int dialsort_ipc_handle(dialsort_ctx c, const void* dev_ptr, void* handle_out) {
  if (!c || !dev_ptr || !handle_out) return fail(DIALSORT_E_INVALID_ARG, "bad ipc_handle arguments");
  DS_CUDA(cudaSetDevice(c->device));
  cudaIpcMemHandle_t h;
  DS_CUDA(cudaIpcGetMemHandle(&h, const_cast<void*>(dev_ptr)));
  static_assert(sizeof(h) == DIALSORT_IPC_HANDLE_BYTES, "IPC handle size");
  memcpy(handle_out, &h, sizeof(h));
  return DIALSORT_OK;
}

int dialsort_ipc_open(dialsort_ctx c, const void* handle, void** dev_ptr_out) {
  if (!c || !handle || !dev_ptr_out) return fail(DIALSORT_E_INVALID_ARG, "bad ipc_open arguments");
  DS_CUDA(cudaSetDevice(c->device));
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  DS_CUDA(cudaIpcOpenMemHandle(dev_ptr_out, h, cudaIpcMemLazyEnablePeerAccess));
  return DIALSORT_OK;
}

int dialsort_ipc_close(dialsort_ctx c, void* dev_ptr) {
  if (!c || !dev_ptr) return fail(DIALSORT_E_INVALID_ARG, "bad ipc_close arguments");
  DS_CUDA(cudaSetDevice(c->device));
  DS_CUDA(cudaIpcCloseMemHandle(dev_ptr));
  return DIALSORT_OK;
}

int dialsort_reconstruct_async(dialsort_ctx c, const uint32_t* H, uint32_t U, int32_t key_base, int32_t* out,
                               uint64_t cap, int exact, uint64_t* d_total, dialsort_stream_t stream) {
  int rc;
  if (!c) return fail(DIALSORT_E_INVALID_ARG, "ctx is NULL");
  ProfScope prof_scope_(c);
  if ((rc = check_U(U)) || (rc = check_keys_arg(out, cap))) return rc;
  if (!H) return fail(DIALSORT_E_INVALID_ARG, "H is NULL");
  if ((int64_t)key_base + (int64_t)U - 1 > 0x7fffffffll)
    return fail(DIALSORT_E_INVALID_ARG, "key_base + U - 1 exceeds INT32_MAX");
  cudaStream_t s = (cudaStream_t)stream;
  DS_CUDA(cudaSetDevice(c->device));
  const uint32_t epoch = next_epoch(c, s);
  if ((rc = enqueue_scan(c, H, U, cap, exact != 0, d_total, epoch, s))) return rc;
  return enqueue_expand(c, U, cap, key_base, out, s);
}

int dialsort_sort_async(dialsort_ctx c, const int32_t* keys, uint64_t n, uint32_t U, int32_t* out, uint32_t* H_out,
                        dialsort_stream_t stream) {
  int rc;
  if (!c) return fail(DIALSORT_E_INVALID_ARG, "ctx is NULL");
  ProfScope prof_scope_(c);
  if ((rc = check_U(U)) || (rc = check_keys_arg(keys, n)) || (rc = check_keys_arg(out, n))) return rc;
  if (n && out != keys && ranges_overlap(keys, 4 * n, out, 4 * n))
    return fail(DIALSORT_E_INVALID_ARG, "out partially overlaps keys (only out == keys is allowed)");
  cudaStream_t s = (cudaStream_t)stream;
  DS_CUDA(cudaSetDevice(c->device));
  const uint32_t epoch = next_epoch(c, s);
  if (n == 0) {
    if (H_out) DS_CUDA(launch_k(KID_ZERO, k_zero, dim3(c->nsm), dim3(256), 0, s, H_out, (uint64_t)U));
    return DIALSORT_OK;
  }
  uint32_t* H = H_out;
  if (!H) {
    if ((rc = c->Hws.ensure(4ull * U))) return rc;
    H = c->Hws.as<uint32_t>();
  }
  if (choose_path(U) != HistPath::Global && sort_fused_enabled() && !hist_use_tma())
    return enqueue_sort_fused(c, keys, n, U, H, out, epoch, s);
  if (hier_applies(U)) return enqueue_sort_hier(c, keys, n, U, H, out, s);
  if ((rc = enqueue_hist_scan(c, keys, n, U, H, true, n, epoch, s))) return rc;
  return enqueue_expand(c, U, n, 0, out, s);
}

int dialsort_sort_int32_async(dialsort_ctx c, const int32_t* keys, uint64_t n, int32_t* out, dialsort_stream_t stream) {
  int rc;
  if (!c) return fail(DIALSORT_E_INVALID_ARG, "ctx is NULL");
  ProfScope prof_scope_(c);
  if ((rc = check_keys_arg(keys, n)) || (rc = check_keys_arg(out, n))) return rc;
  if (n && out != keys && ranges_overlap(keys, 4 * n, out, 4 * n))
    return fail(DIALSORT_E_INVALID_ARG, "out partially overlaps keys (only out == keys is allowed)");
  cudaStream_t s = (cudaStream_t)stream;
  DS_CUDA(cudaSetDevice(c->device));
  const uint32_t epoch = next_epoch(c, s);
  if (n == 0) return DIALSORT_OK;
  if ((rc = c->radix_tmp.ensure(4ull * n + 16))) return rc;
  (void)epoch;
  return radix_enqueue(c, keys, n, out, c->radix_tmp.as<int32_t>(), s);
}

int dialsort_range_count_async(dialsort_ctx c, const uint32_t* H, uint32_t U, uint32_t a, uint32_t b,
                               uint64_t* d_result, dialsort_stream_t stream) {
  int rc;
  if (!c) return fail(DIALSORT_E_INVALID_ARG, "ctx is NULL");
  ProfScope prof_scope_(c);
  if ((rc = check_U(U))) return rc;
  if (!H || !d_result) return fail(DIALSORT_E_INVALID_ARG, "NULL pointer");
  if (a > b || b >= U) return fail(DIALSORT_E_INVALID_ARG, "need 0 <= a <= b < U");
  cudaStream_t s = (cudaStream_t)stream;
  DS_CUDA(cudaSetDevice(c->device));
  DS_CUDA(launch_k(KID_ZERO, k_zero, dim3(1), dim3(32), 0, s, reinterpret_cast<uint32_t*>(d_result), (uint64_t)2));
  uint64_t len = (uint64_t)b - a + 1;
  uint32_t grid = (uint32_t)(cdiv(len, 1024) < (uint64_t)c->nsm * 4 ? cdiv(len, 1024) : (uint64_t)c->nsm * 4);
  DS_CUDA(launch_k(KID_RANGE_COUNT, k_range_count, dim3(grid), dim3(256), 0, s, H, a, b,
                 reinterpret_cast<unsigned long long*>(d_result)));
  return DIALSORT_OK;
}

int dialsort_profile_enable(dialsort_ctx c, int enable) {
  if (!c) return fail(DIALSORT_E_INVALID_ARG, "ctx is NULL");
  c->prof.on = enable != 0;
  return DIALSORT_OK;
}

int dialsort_profile_read(dialsort_ctx c, int max, int* ids, float* ms) {
  if (!c) return -fail(DIALSORT_E_INVALID_ARG, "ctx is NULL");
  int n = 0;
  for (size_t i = 0; i < c->prof.used && n < max; ++i, ++n) {
    float t = 0.f;
    if (cudaEventElapsedTime(&t, c->prof.ev[2 * i], c->prof.ev[2 * i + 1]) != cudaSuccess) {
      cudaGetLastError();
      t = -1.f;
    }
    if (ids) ids[n] = c->prof.ids[i];
    if (ms) ms[n] = t;
  }
  c->prof.used = 0;
  c->prof.ids.clear();
  return n;
}

const char* dialsort_kernel_name(int id) { return (id >= 0 && id < KID_COUNT) ? kKernelNames[id] : "?"; }

// Debug: phase times (ns, relative to the earliest fused-kernel CTA start) of the most recent
// calls since the last read; zeros unless DIALSORT_PHASE_TIMING=1 at context creation.
// Reads and clears the per-CTA stamps; times are ns after the earliest CTA start.
static int read_phase_stamps(dialsort_ctx c, std::vector<unsigned long long>& st, unsigned long long& t0) {
  st.assign((size_t)kPhaseMaxCtas * kPhaseSlots, 0ull);
  t0 = ~0ull;
  if (!c->pt) return DIALSORT_OK;
  DS_CUDA(cudaMemcpy(st.data(), c->pt, sizeof(PhaseTimes), cudaMemcpyDeviceToHost));
  DS_CUDA(cudaMemset(c->pt, 0, sizeof(PhaseTimes)));
  for (int b = 0; b < kPhaseMaxCtas; ++b)
    if (st[(size_t)b * kPhaseSlots] && st[(size_t)b * kPhaseSlots] < t0) t0 = st[(size_t)b * kPhaseSlots];
  return DIALSORT_OK;
}

int dialsort_debug_phase_ns(dialsort_ctx c, uint64_t* out16) {
  if (!c || !out16) return fail(DIALSORT_E_INVALID_ARG, "NULL argument");
  for (int i = 0; i < 16; ++i) out16[i] = 0;
  std::vector<unsigned long long> st;  // phases 0..7 only
  unsigned long long t0;
  int rc = read_phase_stamps(c, st, t0);
  if (rc || t0 == ~0ull) return rc;
  for (int i = 0; i < 8; ++i) {
    unsigned long long mx = 0, mn = ~0ull;
    for (int b = 0; b < kPhaseMaxCtas; ++b) {
      const unsigned long long v = st[(size_t)b * kPhaseSlots + 1 + i];
      if (!v) continue;
      mx = std::max(mx, v);
      mn = std::min(mn, v);
    }
    out16[i] = mx ? mx - t0 : 0;
    out16[8 + i] = mx ? mn - t0 : 0;
  }
  return DIALSORT_OK;
}

int dialsort_debug_phase_cta(dialsort_ctx c, uint64_t* out, int max_ctas) {
  if (!c || !out || max_ctas < 0) return -fail(DIALSORT_E_INVALID_ARG, "bad argument");
  std::vector<unsigned long long> st;
  unsigned long long t0;
  int rc = read_phase_stamps(c, st, t0);
  if (rc) return -rc;
  int n = 0;
  for (int b = 0; b < kPhaseMaxCtas && b < max_ctas; ++b) {
    if (!st[(size_t)b * kPhaseSlots]) break;
    for (int i = 0; i < kPhaseSlots; ++i) {
      const unsigned long long v = st[(size_t)b * kPhaseSlots + i];
      out[(size_t)b * kPhaseSlots + i] = v ? v - t0 : 0;
    }
    n = b + 1;
  }
  return n;
}

int dialsort_crn_resolve_async(dialsort_ctx c, const int32_t* lane_keys, const uint32_t* active, uint64_t n_batches,
                               int32_t* out_keys, uint32_t* out_counts, dialsort_stream_t stream) {
  if (!c) return fail(DIALSORT_E_INVALID_ARG, "ctx is NULL");
  ProfScope prof_scope_(c);
  if (n_batches == 0) return DIALSORT_OK;
  if (!lane_keys || !active || !out_keys || !out_counts) return fail(DIALSORT_E_INVALID_ARG, "NULL pointer");
  cudaStream_t s = (cudaStream_t)stream;
  DS_CUDA(cudaSetDevice(c->device));
  uint64_t grid = cdiv(n_batches * 32, 256);
  if (grid > 0x7fffffffull) return fail(DIALSORT_E_INVALID_ARG, "too many batches");
  DS_CUDA(launch_k(KID_CRN, k_crn_resolve, dim3((uint32_t)grid), dim3(256), 0, s, lane_keys, active, n_batches, out_keys,
                 out_counts));
  return DIALSORT_OK;
}

// ---- synchronous forms ----------------------------------------------------------------------
int dialsort_histogram(const int32_t* keys, uint64_t n, uint32_t U, uint32_t* H) {
  dialsort_ctx c;
  int rc = default_ctx(&c);
  if (rc) return rc;
  if ((rc = dialsort_histogram_async(c, keys, n, U, H, nullptr))) return rc;
  return dialsort_sync(c, nullptr, nullptr);
}
int dialsort_reconstruct(const uint32_t* H, uint32_t U, int32_t* out, uint64_t n) {
  dialsort_ctx c;
  int rc = default_ctx(&c);
  if (rc) return rc;
  if ((rc = dialsort_reconstruct_async(c, H, U, 0, out, n, 1, nullptr, nullptr))) return rc;
  return dialsort_sync(c, nullptr, nullptr);
}
int dialsort_sort(const int32_t* keys, uint64_t n, uint32_t U, int32_t* out) {
  dialsort_ctx c;
  int rc = default_ctx(&c);
  if (rc) return rc;
  if ((rc = dialsort_sort_async(c, keys, n, U, out, nullptr, nullptr))) return rc;
  return dialsort_sync(c, nullptr, nullptr);
}
int dialsort_sort_int32(const int32_t* keys, uint64_t n, int32_t* out) {
  dialsort_ctx c;
  int rc = default_ctx(&c);
  if (rc) return rc;
  if ((rc = dialsort_sort_int32_async(c, keys, n, out, nullptr))) return rc;
  return dialsort_sync(c, nullptr, nullptr);
}

int dialsort_sort_host(dialsort_ctx c, const int32_t* keys_host, uint64_t n, uint32_t U, int32_t* out_host,
                       dialsort_stream_t stream) {
  const int rc = dialsort_sort_host_async(c, keys_host, n, U, out_host, stream);
  if (rc) return rc;
  return dialsort_sync(c, stream, nullptr);
}

int dialsort_sort_host_async(dialsort_ctx c, const int32_t* keys_host, uint64_t n, uint32_t U, int32_t* out_host,
                             dialsort_stream_t stream) {
  int rc;
  if (!c) return fail(DIALSORT_E_INVALID_ARG, "ctx is NULL");
  ProfScope prof_scope_(c);
  if ((rc = check_keys_arg(keys_host, n)) || (rc = check_keys_arg(out_host, n))) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  DS_CUDA(cudaSetDevice(c->device));
  if (n == 0) return DIALSORT_OK;
  if ((rc = c->stage.ensure(4ull * n + 16))) return rc;
  int32_t* d = c->stage.as<int32_t>();
  DS_CUDA(cudaMemcpyAsync(d, keys_host, 4ull * n, cudaMemcpyHostToDevice, s));
  if (U == 0)
    rc = dialsort_sort_int32_async(c, d, n, d, stream);
  else
    rc = dialsort_sort_async(c, d, n, U, d, nullptr, stream);
  if (rc) return rc;
  DS_CUDA(cudaMemcpyAsync(out_host, d, 4ull * n, cudaMemcpyDeviceToHost, s));
  return DIALSORT_OK;
}

}  // extern "C"

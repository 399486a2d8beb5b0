// dialsort.cu — C ABI (include/dialsort.h) and launch logic of the B200 DialSort hot path.
//
// Host side only decides paths, sizes grids and enqueues kernels; every step of the method
// runs in the kernels of ds_hist.cuh / ds_scan.cuh / ds_fused.cuh / ds_part.cuh /
// ds_expand.cuh / ds_radix.cuh / ds_comm.cuh.
// All launches use programmatic dependent launch (PDL) so each kernel's launch overlaps its
// predecessor's tail; every kernel calls griddepcontrol.wait before touching its inputs, which
// keeps stream order exact.  Kernels that synchronise their whole grid (software grid barriers,
// ready flags) are launched cooperatively: a grid that cannot be fully co-resident (another
// tenant, a concurrent barrier kernel of another context) fails to launch instead of hanging.
#include "../../include/dialsort.h"

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>  // (header-only NVTX v3: a no-op unless a profiler is attached)

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <algorithm>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "ds_comm.cuh"
#include "ds_common.cuh"
#include "ds_expand.cuh"
#include "ds_fused.cuh"
#include "ds_hist.cuh"
#include "ds_part.cuh"
#include "ds_peer.cuh"
#include "ds_query.cuh"
#include "ds_radix.cuh"
#include "ds_scan.cuh"
#include "ds_small.cuh"

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
    if (e_ != cudaSuccess) {                                                                 \
      cudaGetLastError();                                                                    \
      return fail(DIALSORT_E_CUDA, std::string(#expr) + ": " + cudaGetErrorString(e_));      \
    }                                                                                        \
  } while (0)

enum KernelId {
  KID_ZERO = 0, KID_HIST_SMEM32, KID_HIST_SMEM16, KID_HIST_GLOBAL, KID_SCAN, KID_EXPAND, KID_RADIX_PASS,
  KID_RANGE_COUNT, KID_CRN, KID_SORT_FUSED, KID_PART_COUNT, KID_PART_SCAN, KID_PART_SCATTER, KID_PUSH_SLICES,
  KID_SLICE_SUM, KID_COMM_SIGNAL, KID_COMM_SLICE_SUM, KID_COMM_OFFSETS, KID_COMM_RHIST, KID_COMM_RPLAN,
  KID_COMM_RSPLIT, KID_COMM_WAIT, KID_RADIX_PROBE, KID_QUERY, KID_SORT_BATCH, KID_PART_SAMPLE, KID_PART_SCATTER_EST, KID_PART_FIN, KID_PART_RING, KID_PART_COMPACT, KID_PART_MOVE, KID_SORT_SMALL, KID_SORT_SMALL_BATCH, KID_COUNT
};
const char* const kKernelNames[KID_COUNT] = {
    "k_zero", "k_hist_smem32", "k_hist_smem16", "k_hist_global", "k_scan", "k_expand", "k_radix_pass",
    "k_range_count", "k_crn_resolve", "k_sort_fused", "k_part_count", "k_part_scan", "k_part_place",
    "k_push_slices", "k_slice_sum", "k_comm_signal", "k_comm_slice_sum", "k_comm_offsets", "k_comm_rhist",
    "k_comm_rplan", "k_comm_rsplit", "k_comm_wait", "k_radix_lane_probe", "k_query", "k_sort_batch", "k_part_sample",
    "k_part_place_est", "k_part_fin", "k_part_place_ring", "k_part_ring_compact", "k_part_ring_move", "k_sort_small", "k_sort_small_batch"};

// Per-context launch profiler (off by default): an event pair around each launch.
struct Profiler {
  bool on = false;
  std::vector<cudaEvent_t> ev;  // 2 per record
  std::vector<int> ids;
  size_t used = 0;
};
thread_local Profiler* g_prof = nullptr;  // set by the API entry for the ctx in use

// COOP: the kernel waits on the rest of its grid (grid barrier / ready flags), so the whole
// grid must be co-resident (grids are sized from the occupancy of an otherwise idle device).
// Two such kernels running at once could each hold part of the SMs and wait forever for the
// rest; they can only overlap when issued on different streams of one process (kernels of
// different processes are time-sliced without MPS).  Default: the library keeps a per-device
// FIFO of its co-resident launches — a launch on another stream than the previous one first
// waits (cudaStreamWaitEvent) for everything that stream had enqueued, so two of them never
// overlap; a single stream pays nothing.  DIALSORT_OPT_COOPERATIVE = 1 (per context) launches
// them with cudaLaunchAttributeCooperative instead, which makes a grid that cannot be
// co-resident fail to launch even against other tenants, at ~2 us per launch (measured: c2
// 32.8 -> 35.0 us, the attribute gives up the PDL overlap with the previous kernel).
struct CoopFifo {
  std::mutex mu;
  bool any = false;
  cudaStream_t last = nullptr;
  cudaEvent_t ev = nullptr;
};
CoopFifo g_fifo[32];
thread_local bool g_coop_attr = false;  // set per API call from the context's option

// CLUSTER > 0: the grid runs as clusters of CLUSTER CTAs (launch attribute; k_sort_small)
template <bool COOP = false, int CLUSTER = 0, typename... KArgs, typename... Args>
cudaError_t launch_k(int kid, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                     Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  static const int pdl = getenv("DIALSORT_NO_PDL") ? 0 : 1;  // (debug: launches without PDL)
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl;
  at[1].id = cudaLaunchAttributeCooperative;
  at[1].val.cooperative = 1;
  if (CLUSTER) {
    at[1].id = cudaLaunchAttributeClusterDimension;
    at[1].val.clusterDim.x = CLUSTER;
    at[1].val.clusterDim.y = 1;
    at[1].val.clusterDim.z = 1;
  }
  cfg.attrs = at;
  cfg.numAttrs = ((COOP && g_coop_attr) || CLUSTER) ? 2 : 1;
  std::unique_lock<std::mutex> lk;
  CoopFifo* fifo = nullptr;
  static const bool no_fifo = [] {  // (DIALSORT_NO_FIFO=1: experiments only)
    const char* e = getenv("DIALSORT_NO_FIFO");
    return e && e[0] == '1';
  }();
  if (COOP && !g_coop_attr && !no_fifo) {  // wait for the previous co-resident launch if it is on another stream
    int dev = 0;
    cudaGetDevice(&dev);
    CoopFifo* f = &g_fifo[dev & 31];
    lk = std::unique_lock<std::mutex>(f->mu);
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    cudaStreamIsCapturing(s, &cap);
    if (cap != cudaStreamCaptureStatusNone) {
      // (a stream being captured into a graph may not wait on an event recorded outside the
      //  capture, nor leave one for uncaptured streams: the graph's launches are ordered by the
      //  graph itself; the FIFO restarts after it)
      f->any = false;
    } else {
      fifo = f;
      if (!f->ev) cudaEventCreateWithFlags(&f->ev, cudaEventDisableTiming);
      if (f->any && f->last != s) cudaStreamWaitEvent(s, f->ev, 0);
      f->any = true;
      f->last = s;
    }
  }
  // (and the event marks this launch for the next one: recorded after it, on its stream)
  struct FifoMark {
    CoopFifo* f;
    cudaStream_t s;
    ~FifoMark() {
      if (f) cudaEventRecord(f->ev, s);
    }
  } mark{fifo, s};
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

// Result of the radix lane-order probe per device (k_radix_lane_probe): -1 unknown, else the
// number of violating lanes (0: k_radix_pass4's in-warp ranks are stable on this device).
std::mutex g_probe_mu;
std::map<int, long long> g_probe;

}  // namespace

constexpr int kMaxLanes = 6;  // CTA groups of the batched sort

struct dialsort_ctx_s {
  int device = 0;
  int nsm = 148;
  uint32_t epoch = 0;
  DBuf partials, P, tfb, ws_total, ovfH, status, stage, Hws, range_tot, gridbar, tsums, radix_tmp, radix_hist,
      fused_tiles, Hx, part, htmp, qtmp, psamp, ringws;
  DevStatus* host_status = nullptr;  // pinned mirror
  // gridbar layout: [0] GridBar of k_scan, [32] GridBarR of the radix passes, [64] FusedState of
  // the fused step, [128] GridBar of the query kernels (all zero at creation)
  FusedState* fused_state() { return reinterpret_cast<FusedState*>(gridbar.as<char>() + 64); }
  Profiler prof;
  int expand_occ = 4, scan_occ = 2, radix3_occ = 1, radix4_occ = 1;
  long long probe_violations = -1;   // radix lane-order probe of this device
  int radix_force = 0;               // 0: auto (pass4 iff the probe passed), 3 / 4 forced
  bool small16 = false;              // 16-CTA clusters of k_sort_small<16> can be launched here
  bool coop_attr = false;            // DIALSORT_OPT_COOPERATIVE
  uint32_t max_ctas = 0;             // DIALSORT_OPT_MAX_CTAS (0: every SM)
  int part_mode = 0;                 // DIALSORT_OPT_PART_MODE
  // batched sort (dialsort_sort_batch_async): one workspace lane per CTA group, created lazily;
  // their deferred errors are merged by dialsort_sync of this context
  dialsort_ctx lanes[kMaxLanes] = {};
  PhaseTimes* pt = nullptr;          // debug phase timing (DIALSORT_PHASE_TIMING=1)
  bool owns_pt = true;               // (a lane writes into its parent's stamps)
};

struct dialsort_comm_s {
  dialsort_ctx ctx = nullptr;
  uint32_t G = 1, rank = 0;
  CommLayout lay = {};
  void* ws = nullptr;                    // own symmetric workspace (cudaMalloc: IPC handles at offset 0)
  char* peer[kCommMaxRanks] = {};        // every rank's workspace as mapped here
  bool ipc_mapped[kCommMaxRanks] = {};   // opened with cudaIpcOpenMemHandle (closed at destroy)
  bool connected = false;
  uint32_t epoch = 0;                    // calls so far (flags hold the epoch of the last call)
  DBuf tables;                           // [2 parity][G] owner receive-slot pointers (histogram scatter)
  DBuf scratch;                          // comm scalars: slice total + ticket, rhist ws, plan
  DBuf hslice;                           // the owner's slice histogram (uint32[Lmax])
};

namespace {

constexpr uint32_t kCommMagic = 0x44534331u;  // "DSC1"
struct CommHandle {                            // DIALSORT_COMM_HANDLE_BYTES bytes
  unsigned char ipc[64];
  uint32_t magic, G, rank, Lmax;
  uint64_t cap, bytes;
  int32_t device;
  unsigned char pad[128 - 64 - 16 - 16 - 4];
};
static_assert(sizeof(CommHandle) == 128, "comm handle size");
constexpr uint64_t kScratchTot = 0, kScratchRh = 64, kScratchPlan = 64 + 4 * 260;  // byte offsets

CommLayout comm_layout(uint32_t G, uint32_t Lmax, uint64_t cap) {
  CommLayout l = {};
  uint64_t o = 0;
  auto take = [&](uint64_t bytes) {
    const uint64_t r = o;
    o = round_up(o + bytes, 256);
    return r;
  };
  l.flags = take(32ull * 2 * kFlagKinds * kCommMaxRanks);
  l.tot = take(8ull * 2 * kCommMaxRanks);
  l.rhist = take(4ull * 2 * kCommMaxRanks * 256);
  l.recv = take(4ull * 2 * G * (uint64_t)Lmax);
  l.rkeys = take(4ull * 2 * cap);
  l.bytes = o;
  l.Lmax = Lmax;
  l.cap = cap;
  return l;
}

CommDev comm_dev(dialsort_comm m) {
  CommDev d = {};
  for (uint32_t r = 0; r < m->G; ++r) d.ws[r] = m->peer[r];
  d.lay = m->lay;
  d.G = m->G;
  d.rank = m->rank;
  d.epoch = m->epoch;
  d.parity = m->epoch & 1u;
  return d;
}

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
  if ((rc = c->gridbar.ensure(256, true))) return rc;
  if ((rc = c->psamp.ensure(8ull * kPartMaxBlocks, true))) return rc;
  if ((rc = c->range_tot.ensure(8ull * 8 * c->nsm, true))) return rc;
  // k_sort_fused: tile totals (2 parities), fallback tile totals
  if ((rc = c->fused_tiles.ensure(4ull * kFusedTileWords, true))) return rc;
  DS_CUDA(cudaFuncSetAttribute(k_sort_fused<kRowU32, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBudget));
  DS_CUDA(cudaFuncSetAttribute(k_sort_fused<kRowP16, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBudget));
  DS_CUDA(cudaFuncSetAttribute(k_sort_fused<kRowN4, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBudget));
  DS_CUDA(cudaFuncSetAttribute(k_sort_fused<kRowU32, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBudget));
  DS_CUDA(cudaFuncSetAttribute(k_sort_fused<kRowP16, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBudget));
  DS_CUDA(cudaFuncSetAttribute(k_sort_fused<kRowN4, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBudget));
  DS_CUDA(cudaFuncSetAttribute(k_sort_fused<kRowU32, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBudget));
  DS_CUDA(cudaFuncSetAttribute(k_sort_batch<kRowU32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBudget));
  DS_CUDA(cudaFuncSetAttribute(k_reconstruct_fused, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBudget));
  DS_CUDA(cudaFuncSetAttribute(k_part_scatter_wide, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)part_wide_smem(kPartMaxBlocksWide)));
  DS_CUDA(cudaFuncSetAttribute(k_part_place_ring, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               (int)part_ring_smem(kRpMaxB)));
  {  // non-portable 16-CTA clusters for k_sort_small<16> (where the device schedules them)
    c->small16 = false;
    if (cudaFuncSetAttribute(k_sort_small<16>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess &&
        cudaFuncSetAttribute(k_sort_small_batch<16>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) == cudaSuccess) {
      cudaLaunchConfig_t q = {};
      q.gridDim = dim3(16);
      q.blockDim = dim3(kSmallThreads);
      cudaLaunchAttribute ca;
      ca.id = cudaLaunchAttributeClusterDimension;
      ca.val.clusterDim.x = 16;
      ca.val.clusterDim.y = 1;
      ca.val.clusterDim.z = 1;
      q.attrs = &ca;
      q.numAttrs = 1;
      int nclu = 0;
      c->small16 = cudaOccupancyMaxActiveClusters(&nclu, k_sort_small<16>, &q) == cudaSuccess && nclu > 0;
    }
    cudaGetLastError();
  }
  DS_CUDA(cudaFuncSetAttribute(k_sort_batch<kRowP16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBudget));
  DS_CUDA(cudaFuncSetAttribute(k_sort_batch<kRowN4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBudget));
  DS_CUDA(cudaFuncSetAttribute(k_sort_batch<kRowP16, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBudget));
  DS_CUDA(cudaFuncSetAttribute(k_sort_batch<kRowN4, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmemBudget));
  radix_configure();
  int occ = 0;
  DS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_radix_pass3, kRadixThreads, sizeof(Radix3Smem)));
  c->radix3_occ = occ > 0 ? occ : 1;
  DS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_radix_pass4, kR4Threads, sizeof(Radix4Smem)));
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
  // radix lane-order probe, once per device (k_radix_lane_probe, ds_radix.cuh)
  {
    std::lock_guard<std::mutex> lk(g_probe_mu);
    auto it = g_probe.find(c->device);
    if (it != g_probe.end()) {
      c->probe_violations = it->second;
    } else {
      unsigned long long* dv = nullptr;
      DS_CUDA(cudaMalloc(&dv, 8));
      DS_CUDA(cudaMemset(dv, 0, 8));
      k_radix_lane_probe<<<2 * c->nsm, kRadixThreads>>>(0x5eed1234u, 9 * 32, dv);
      cudaError_t le = cudaGetLastError();
      unsigned long long hv = 0;
      cudaError_t ce = cudaMemcpy(&hv, dv, 8, cudaMemcpyDeviceToHost);
      cudaFree(dv);
      if (le != cudaSuccess || ce != cudaSuccess)
        return fail(DIALSORT_E_CUDA, std::string("radix lane probe: ") + cudaGetErrorString(le != cudaSuccess ? le : ce));
      c->probe_violations = (long long)hv;
      g_probe[c->device] = c->probe_violations;
    }
  }
  return DIALSORT_OK;
}

// Bumps the call epoch (tags the packed-overflow flag).
uint32_t next_epoch(dialsort_ctx c) {
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

enum class HistPath { Smem32, Smem16, Hier, Global };
HistPath choose_path(uint32_t U) {
  if (U <= kSmem32MaxBins) return HistPath::Smem32;
  if (U <= kSmem16MaxBins) return HistPath::Smem16;
  static const bool no_hier = getenv("DIALSORT_NO_HIER") != nullptr;  // (A/B against the L2 path only)
  if (!no_hier && (uint64_t)U <= ((uint64_t)kPartMaxBlocksWide << kPartShift)) return HistPath::Hier;
  return HistPath::Global;
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

// The whole sort step as one kernel (ds_fused.cuh) for the shared-memory universes, or — with
// hist_only — the histogram only (merged H stored into H, or into the owners' slots when
// Hpeer is set).  d_n / d_off (nullable): the key count and the keys/out offset are on the
// device (a universe block of the hierarchical path); n is then only the size hint for the grid
// and row format.  kb: key bytes (4 int32; 2 uint16: the hierarchical path's universe blocks or a
// 2-byte coded domain; 1 uint8: a 1-byte coded domain, U <= 8192).  enc / dec: the coded-domain
// maps phi (1-byte keys) and phi^-1 (emitted values), nullable.
// The arguments of one fused step on context c's workspace (shared by the single-step launch
// and the batched kernel).  C_force != 0: the step runs on exactly that many CTAs (a group of
// k_sort_batch); barriers: the step reserves `bars` barriers of its grid.
int build_fused_args(dialsort_ctx c, ScanArgs& a, int& fmt, uint32_t& C, size_t& smem, uint64_t n, uint32_t U,
                     uint32_t* H, uint32_t epoch, const uint64_t* d_n, const uint64_t* d_off, int kb, bool hist_only,
                     uint32_t* const* Hpeer, uint32_t peerL, uint32_t peerRank, uint32_t bin_base,
                     const uint32_t* enc, const int32_t* dec, uint32_t C_force, uint32_t bars) {
  int rc;
  a = ScanArgs{};
  if ((rc = fill_scan_args(c, a, U, !hist_only, n, true, nullptr, epoch))) return rc;
  a.d_n = d_n;
  a.d_off = d_off;
  a.hist_only = hist_only;
  a.Hpeer = Hpeer;
  a.peerL = peerL;
  a.peerRank = peerRank;
  a.bin_base = bin_base;
  a.enc = enc;
  a.dec = dec;
  if (kb == 1 && U > kSmem32MaxBins) return fail(DIALSORT_E_INVALID_ARG, "1-byte keys need U <= 8192");
  const bool pack = U > kSmem32MaxBins;
  const uint32_t W = pack ? (U + 1) / 2 : U;
  const uint32_t ldw = (uint32_t)round_up(W, 8);  // shared-memory histogram words
  const uint64_t n4 = n / 4 + 1;
  // CTAs: one per 4096 keys (4 per thread), and at least one per 1024 bins — every CTA flushes
  // and merges O(U) words whatever the grid, but the merge's batches (16 tiles of 64 bins each)
  // run one after another: U = 65536 on one CTA took 64 batches (~330 us at n = 1e4).  4096 keys
  // per CTA against round 1's 32768 (tools/kpc_ab.py, single-call device time): n = 1e5 U = 256
  // 14.8 -> 13.9 us, n = 1e6 18.9 -> 15.1, n = 1e4 U = 1024 28.6 -> 15.7, n = 1e6 U = 65536
  // skewed 27.9 -> 22.3; n >= 6e5 uses every SM either way.
  static const uint64_t kpc = [] {  // keys per CTA the grid is sized for (DIALSORT_FUSED_KPC: A/B only)
    const char* e = getenv("DIALSORT_FUSED_KPC");
    return e ? std::max<uint64_t>(1024, strtoull(e, nullptr, 10)) : 4096ull;
  }();
  const uint64_t want = std::max<uint64_t>(cdiv(4 * n4, kpc), cdiv(U, 1024));
  const uint64_t cmax = std::min<uint64_t>(c->max_ctas ? std::min<uint32_t>(c->max_ctas, c->nsm) : c->nsm,
                                           kFMaxRows);  // rows a staging slot holds
  C = C_force ? C_force : (uint32_t)(want < cmax ? (want ? want : 1) : cmax);
  // partial-row format: 4-bit rows while counts per CTA and bin are small (mean <= 8: counts
  // >= 16 — exceptions, one RED each — stay rare), else the packed 16-bit rows
  fmt = !pack ? kRowU32 : (n <= 8ull * C * U ? kRowN4 : kRowP16);
  const uint32_t ldr = fmt == kRowN4 ? (uint32_t)round_up((U + 7) / 8, 8) : ldw;  // row words
  smem = std::max<size_t>(4ull * ldw, 4ull * kFSmemWords);  // histogram | merge + projection
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
  // two-parity workspaces (per-tile ready flags, owner counters, the 4-bit rows' exception
  // histogram): each step uses parity seq & 1 and clears the other one; the parity, the epoch and
  // the barrier base are derived on the device from the workspace's FusedState (sort_step)
  a.ready_base = ft;
  a.own_base = ft + 2 * kFTileSlots;
  a.Hx_base = c->Hx.as<uint32_t>();
  a.fstate = c->fused_state();
  a.bar64 = &a.fstate->bar;
  (void)bars;
  return DIALSORT_OK;
}

int enqueue_sort_fused(dialsort_ctx c, const void* keys, uint64_t n, uint32_t U, uint32_t* H, int32_t* out,
                       uint32_t epoch, cudaStream_t s, int32_t key_base = 0, const uint64_t* d_n = nullptr,
                       const uint64_t* d_off = nullptr, int kb = 4, bool hist_only = false,
                       uint32_t* const* Hpeer = nullptr, uint32_t peerL = 0, uint32_t peerRank = 0,
                       uint32_t bin_base = 0, const uint32_t* enc = nullptr, const int32_t* dec = nullptr,
                       const uint64_t* d_koff = nullptr) {
  int rc;
  ScanArgs a;
  int fmt;
  uint32_t C;
  size_t smem;
  if ((rc = build_fused_args(c, a, fmt, C, smem, n, U, H, epoch, d_n, d_off, kb, hist_only, Hpeer, peerL, peerRank,
                             bin_base, enc, dec, 0, 2)))
    return rc;
  a.d_koff = d_koff;
#define DS_LAUNCH_FUSED(F, K) \
  DS_CUDA(launch_k<true>(KID_SORT_FUSED, k_sort_fused<F, K>, dim3(C), dim3(1024), smem, s, keys, n, a, out, key_base))
  if (fmt == kRowN4) {
    if (kb == 2) DS_LAUNCH_FUSED(kRowN4, 2); else DS_LAUNCH_FUSED(kRowN4, 4);
  } else if (fmt == kRowP16) {
    if (kb == 2) DS_LAUNCH_FUSED(kRowP16, 2); else DS_LAUNCH_FUSED(kRowP16, 4);
  } else {
    if (kb == 2) DS_LAUNCH_FUSED(kRowU32, 2); else if (kb == 1) DS_LAUNCH_FUSED(kRowU32, 1); else DS_LAUNCH_FUSED(kRowU32, 4);
  }
#undef DS_LAUNCH_FUSED
  return DIALSORT_OK;
}

// The projection of a caller histogram as one co-resident kernel (k_reconstruct_fused) when H
// is 16-byte aligned, U % 4 == 0 and U <= 131072 (the share mode's ready-flag slots); returns
// false (nothing enqueued) otherwise, and the caller takes k_scan + k_expand.
bool reconstruct_fused_applies(const uint32_t* H, uint32_t U) {
  return (reinterpret_cast<uintptr_t>(H) & 15u) == 0 && U % 4 == 0 && (uint64_t)U <= (uint64_t)kFTileSlots * kFTileBins;
}
int enqueue_reconstruct_fused(dialsort_ctx c, const uint32_t* H, uint32_t U, int32_t key_base, int32_t* out,
                              uint64_t cap, bool exact, uint64_t* d_total, uint32_t epoch, cudaStream_t s) {
  int rc;
  ScanArgs a;
  int fmt;
  uint32_t C;
  size_t smem;
  const uint64_t want = std::max<uint64_t>(cdiv(cap / 4 + 1, 8192ull), cdiv(U, 1024));  // (32768 outputs a CTA)
  const uint32_t Cr = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(want, std::min<uint64_t>(c->nsm, kFMaxRows)));
  if ((rc = build_fused_args(c, a, fmt, C, smem, cap, U, nullptr, epoch, nullptr, nullptr, 4, false, nullptr, 0, 0, 0,
                             nullptr, nullptr, Cr, 2)))
    return rc;
  a.partials = H;  // the given histogram as the single u32 "row"
  a.C = 1;
  a.ldw = a.ldr = (uint32_t)round_up(U, 8);
  a.pack16 = 0;
  a.nib4 = 0;
  a.exact = exact;
  a.d_total = d_total;
  smem = 4ull * kFSmemWords;
  DS_CUDA(launch_k<true>(KID_SORT_FUSED, k_reconstruct_fused, dim3(C), dim3(1024), smem, s, a, cap, out, key_base));
  return DIALSORT_OK;
}

bool part_ring_enabled() {  // (DIALSORT_PART_RING=0: the sub-tile placement k_part_place<true>, A/B only)
  static const bool v = [] {
    const char* e = getenv("DIALSORT_PART_RING");
    return !(e && e[0] == '0');
  }();
  return v;
}

bool hier_batched() {  // (DIALSORT_HIER_BATCH=0: one launch per block, A/B only)
  static const bool v = [] {
    const char* e = getenv("DIALSORT_HIER_BATCH");
    return !(e && e[0] == '0');
  }();
  return v;
}

// Hierarchical DialSort for 98304 < U <= 2^22 (ds_part.cuh): MSD split into 65536-bin universe
// blocks, then one k_sort_fused per block (device-resident block sizes / offsets: no host round
// trip).  hist_only: the blocks' launches stop after their merge (H, or the owners' slots).
int enqueue_hier(dialsort_ctx c, const int32_t* keys, uint64_t n, uint32_t U, uint32_t* H, int32_t* out,
                 cudaStream_t s, bool hist_only = false, uint32_t* const* Hpeer = nullptr, uint32_t peerL = 0,
                 uint32_t peerRank = 0) {
  int rc;
  const uint32_t B = (uint32_t)cdiv(U, 1ull << kPartShift);
  static const bool force_wide = getenv("DIALSORT_PART_WIDE") != nullptr;  // (A/B only)
  const bool wide = B > kPartMaxBlocks || force_wide;  // 2^22 < U <= 2^26: per-CTA block counters
  constexpr uint32_t kCtasPerSm = 2048 / kPartThreads;
  const uint32_t Gp = (uint32_t)std::max<uint64_t>(
      1, std::min<uint64_t>((uint64_t)kCtasPerSm * c->nsm, cdiv(n, wide ? kPartWideTile : kPartTile)));
  // sampled schedule (default for up to 64 blocks): the keys' regions in tmp carry the
  // estimate's margins (at most n / 4 + 512 B extra keys)
  // (+ a 4096-key trash area for the runs of an overflowed region; positions stay below 2^32)
  const uint64_t tcap = n + n / 4 + 512ull * B;
  const bool sampled = !wide && c->part_mode != 1 && tcap + kPartTile < (1ull << 32);
  // ring placement (k_part_place_ring, B <= kRpMaxB): the regions also hold every warp's unused
  // claimed units and tail remainder (part_ring_extra); the B tail pools follow them
  RingWs rw;
  memset(&rw, 0, sizeof rw);
  uint64_t ring_extra = 0, tslots = sampled ? tcap + kPartTile : n;
  uint32_t Gr = 0;
  if (sampled && B <= kRpMaxB && part_ring_enabled()) {
    int occ = 0;
    DS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_part_place_ring, kRpThreads, part_ring_smem(B)));
    const uint32_t g = (uint32_t)std::max<uint64_t>(
        1, std::min<uint64_t>((uint64_t)c->nsm * std::max(occ, 1), cdiv(n, kRpWarps * 4096ull)));
    const uint64_t W = (uint64_t)g * kRpWarps, extra = part_ring_extra((uint32_t)W);
    const uint64_t tail0 = round_up(tcap + (uint64_t)B * (extra + kRpUnit), kRpUnit);
    const uint64_t need = tail0 + (uint64_t)B * kRpUnit * W;
    if (need < (1ull << 32)) {
      if ((rc = c->ringws.ensure(4ull * ((uint64_t)B * (kRpSubs + 1) * kFillStride + 4ull * B * W +
                                         2ull * B * kRpMaxHoles + 4ull * B))))
        return rc;
      Gr = g;
      rw.W = (uint32_t)W;
      rw.tailcap = (uint32_t)(kRpUnit * W);
      rw.tail0 = tail0;
      rw.sub = c->ringws.as<uint32_t>();
      rw.tfill = rw.sub + (uint64_t)B * kRpSubs * kFillStride;
      rw.holes = rw.tfill + (uint64_t)B * kFillStride;
      rw.list = rw.holes + 4ull * B * W;
      rw.meta = rw.list + 2ull * B * kRpMaxHoles;
      ring_extra = extra;
      tslots = need;
    }
  }
  if ((rc = c->part.ensure(4ull * Gp * B + 160ull * B + 64))) return rc;
  if ((rc = c->htmp.ensure(2ull * tslots + 16))) return rc;  // uint16 block keys
  PartWs w;
  w.bsz = c->part.as<uint64_t>();
  w.boff = w.bsz + B;
  w.koff = w.boff + B;
  w.cap = w.koff + B;
  w.fill = reinterpret_cast<uint32_t*>(w.cap + B);
  w.ovf = w.fill + (uint64_t)kFillStride * B;
  w.cnt = w.ovf + 16;
  w.st = c->status.as<DevStatus>();
  uint16_t* tmp = c->htmp.as<uint16_t>();
  if (wide) {
    DS_CUDA(launch_k(KID_PART_COUNT, k_part_count_wide, dim3(Gp), dim3(kPartThreads), 4ull * B, s, keys, n, U, B, w));
    DS_CUDA(launch_k(KID_PART_SCAN, k_part_scan, dim3(1), dim3(1024), 0, s, Gp, B, w, (const uint32_t*)nullptr));
    DS_CUDA(launch_k(KID_PART_SCATTER, k_part_scatter_wide, dim3(Gp), dim3(kPartThreads), part_wide_smem(B), s, keys,
                     n, U, B, w, tmp));
  } else {
    const uint32_t* gate = nullptr;
    if (sampled) {  // (part_mode 2: no margins — overflows, tests the exact schedule behind it)
      // (part_mode 2: no margins — not even the ring's — so the regions overflow)
      DS_CUDA(launch_k(KID_PART_SAMPLE, k_part_sample, dim3(kSampleCtas), dim3(kSampleThreads), 0, s, keys, n, U, B,
                       w, c->part_mode == 2 ? (uint64_t)0 : tcap, c->psamp.as<uint32_t>(),
                       c->part_mode == 2 && ring_extra ? (uint64_t)kRpUnit : ring_extra, rw));
      if (Gr) {
        DS_CUDA(launch_k(KID_PART_RING, k_part_place_ring, dim3(Gr), dim3(kRpThreads), part_ring_smem(B), s, keys, n,
                         U, B, w, rw, tmp));
        DS_CUDA(launch_k(KID_PART_COMPACT, k_part_ring_compact, dim3(B), dim3(1024), 0, s, B, w, rw));
        DS_CUDA(launch_k(KID_PART_MOVE, k_part_ring_move, dim3(B * kRpMoveCtas), dim3(512), 0, s, B, w, rw, tmp));
        DS_CUDA(launch_k(KID_PART_MOVE, k_part_ring_tail, dim3(B * kRpMoveCtas), dim3(512), 0, s, B, w, rw, tmp));
      } else {
        DS_CUDA(launch_k(KID_PART_SCATTER_EST, k_part_place<true>, dim3(Gp), dim3(kPartThreads), 0, s, keys, n, U, B,
                         w, tmp, (const uint32_t*)nullptr, (uint32_t)tcap));
      }
      DS_CUDA(launch_k(KID_PART_FIN, k_part_fin, dim3(1), dim3(1024), 0, s, B, w));
      gate = w.ovf;  // the exact schedule below runs only after an overflow
    }
    DS_CUDA(launch_k(KID_PART_COUNT, k_part_count, dim3(Gp), dim3(kPartThreads), 0, s, keys, n, U, B, w, gate));
    DS_CUDA(launch_k(KID_PART_SCAN, k_part_scan, dim3(1), dim3(1024), 0, s, Gp, B, w, gate));
    DS_CUDA(launch_k(KID_PART_SCATTER, k_part_place<false>, dim3(Gp), dim3(kPartThreads), 0, s, keys, n, U, B, w,
                     tmp, gate, 0u));
  }
  // the block steps: the full 65536-bin blocks overlapped on CTA groups, up to kBatchMax per
  // k_sort_batch launch (their HBM phases overlap the others' merges, as the batched sort); a
  // last partial block (U % 65536 != 0) by its own k_sort_fused launch
  const uint32_t Bfull = (uint32_t)(U >> kPartShift);
  const uint32_t L = (uint32_t)std::min<uint64_t>(std::min<uint64_t>(Bfull, (uint64_t)c->nsm * kFPassTiles / 1024), 4);
  const uint32_t Gg = std::min<uint32_t>(kFMaxRows, (uint32_t)c->nsm / std::max<uint32_t>(L, 1));
  const uint64_t nb_hint = cdiv(n, B);
  uint32_t b_done = 0;
  if (hier_batched() && L >= 2) {
    for (uint32_t g = 0; g < L; ++g)
      if (!c->lanes[g]) {
        dialsort_ctx l = nullptr;
        if ((rc = dialsort_ctx_create(c->device, 0, 0, &l))) return rc;
        if (l->pt) cudaFree(l->pt);
        l->pt = c->pt;
        l->owns_pt = false;
        c->lanes[g] = l;
      }
    for (uint32_t b0 = 0; b0 < Bfull; b0 += kBatchMax) {
      const uint32_t m = std::min<uint32_t>(kBatchMax, Bfull - b0);
      BatchArgs BA;
      memset(&BA, 0, sizeof BA);
      BA.nb = m;
      BA.L = std::min<uint32_t>(L, m);
      BA.Gg = Gg;
      int fmt = -1;
      size_t smem = 0;
      for (uint32_t j = 0; j < m; ++j) {
        const uint32_t b = b0 + j;
        dialsort_ctx l = c->lanes[j % BA.L];
        uint32_t* Hb = H ? H + ((uint64_t)b << kPartShift) : nullptr;
        uint32_t C;
        if ((rc = build_fused_args(l, BA.a[j], fmt, C, smem, nb_hint, 1u << kPartShift, Hb, next_epoch(l), w.bsz + b,
                                   w.boff + b, 2, hist_only, Hpeer, peerL, peerRank, b << kPartShift, nullptr, nullptr,
                                   Gg, 3)))
          return rc;
        BA.a[j].d_koff = w.koff + b;
        BA.keys[j] = tmp;
        BA.n[j] = nb_hint;
        BA.out[j] = out;
        BA.key_base[j] = (int32_t)(b << kPartShift);
      }
      const dim3 grid(BA.L * Gg);
      if (fmt == kRowN4)
        DS_CUDA(launch_k<true>(KID_SORT_BATCH, k_sort_batch<kRowN4, 2>, grid, dim3(1024), smem, s, BA));
      else
        DS_CUDA(launch_k<true>(KID_SORT_BATCH, k_sort_batch<kRowP16, 2>, grid, dim3(1024), smem, s, BA));
    }
    b_done = Bfull;
  }
  for (uint32_t b = b_done; b < B; ++b) {
    const uint32_t Ub = (uint32_t)std::min<uint64_t>(1ull << kPartShift, (uint64_t)U - ((uint64_t)b << kPartShift));
    const uint32_t epoch = next_epoch(c);  // each block launch has its own ready-flag epoch
    uint32_t* Hb = H ? H + ((uint64_t)b << kPartShift) : nullptr;
    if ((rc = enqueue_sort_fused(c, tmp, nb_hint, Ub, Hb, out, epoch, s, (int32_t)(b << kPartShift), w.bsz + b,
                                 w.boff + b, 2, hist_only, Hpeer, peerL, peerRank, b << kPartShift, nullptr, nullptr,
                                 w.koff + b)))
      return rc;
  }
  return DIALSORT_OK;
}

// Histogram of keys into H (or into the owners' slots: Hpeer); when do_scan, also P / tfb for a
// projection of `cap` outputs (k_expand).  Smem universes: one fused co-resident kernel;
// hierarchical universes: the MSD split + histogram-only block launches; larger: zero + L2
// ingest (+ k_scan).
int enqueue_hist_scan(dialsort_ctx c, const int32_t* keys, uint64_t n, uint32_t U, uint32_t* H, bool do_scan,
                      uint64_t cap, uint32_t epoch, cudaStream_t s, uint32_t* const* Hpeer = nullptr,
                      uint32_t peerL = 0, uint32_t peerRank = 0) {
  int rc;
  ScanArgs a = {};
  if ((rc = fill_scan_args(c, a, U, do_scan, cap, true, nullptr, epoch))) return rc;
  a.Hpeer = Hpeer;  // (the merge stores into the owners' slots)
  a.peerL = peerL;
  a.peerRank = peerRank;
  const HistPath path = choose_path(U);
  if (path == HistPath::Hier && n > 0) {
    if ((rc = enqueue_hier(c, keys, n, U, H, nullptr, s, true, Hpeer, peerL, peerRank))) return rc;
    if (!do_scan) return DIALSORT_OK;
    a.Hsrc = H;
    const uint64_t ntiles = cdiv(U, kTileBins);
    const uint64_t wave = (uint64_t)c->nsm * c->scan_occ;
    DS_CUDA(launch_k<true>(KID_SCAN, k_scan, dim3((uint32_t)(ntiles < wave ? ntiles : wave)), dim3(kTileBins), 0, s, a));
    return DIALSORT_OK;
  }
  if (path == HistPath::Global || path == HistPath::Hier) {
    DS_CUDA(launch_k(KID_ZERO, k_zero, dim3(c->nsm * 4), dim3(256), 0, s, H, (uint64_t)U));
    const uint64_t want = cdiv(n / 4 + 1, 256ull * kHistUnroll);
    const uint64_t capg = (uint64_t)c->nsm * 8;
    const uint32_t grid = (uint32_t)(want < capg ? (want ? want : 1) : capg);
    DS_CUDA(launch_k(KID_HIST_GLOBAL, k_hist_global, dim3(grid), dim3(256), 0, s, keys, n, U, H, a.st));
    if (!do_scan) return DIALSORT_OK;
    a.Hsrc = H;
    const uint64_t ntiles = cdiv(U, kTileBins);
    const uint64_t wave = (uint64_t)c->nsm * c->scan_occ;
    DS_CUDA(launch_k<true>(KID_SCAN, k_scan, dim3((uint32_t)(ntiles < wave ? ntiles : wave)), dim3(kTileBins), 0, s, a));
    return DIALSORT_OK;
  }
  // shared-memory universes: the fused step in histogram-only mode (k_sort_fused, hist_only:
  // ingestion, flush, merge; the merged bins stored into H or straight into the owners' slots)
  if (do_scan) return fail(DIALSORT_E_INVALID_ARG, "internal: scan of a shared-memory histogram");
  return enqueue_sort_fused(c, keys, n, U, H, nullptr, epoch, s, 0, nullptr, nullptr, 4, true, Hpeer, peerL, peerRank, 0);
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
  DS_CUDA(launch_k<true>(KID_SCAN, k_scan, dim3((uint32_t)(ntiles < wave ? ntiles : wave)), dim3(kTileBins), 0, s, a));
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

// The radix variant in use: pass4 (TMA sub-tiles, ranks from the counting atomic) when the
// device passed the lane-order probe and the buffers are 16-byte aligned, else pass3.
int radix_variant(dialsort_ctx c, bool aligned) {
  if (c->radix_force == 3) return 3;
  if (c->radix_force == 4) return aligned ? 4 : 3;
  return (aligned && c->probe_violations == 0) ? 4 : 3;
}

// DialSort-Radix, 4 reduce-then-scan passes (ds_radix.cuh).  d_n (nullable): the key count is
// on the device; n is then the bound the grid is sized for.  pass_out (nullable, debug): pass p
// writes pass_out + p n instead of ping-ponging (pass buffers for the per-pass parity test).
int radix_enqueue(dialsort_ctx c, const int32_t* keys, uint64_t n, int32_t* out, int32_t* tmp, cudaStream_t s,
                  const uint32_t* d_n = nullptr, uint32_t* pass_out = nullptr) {
  if (n >= (1ull << 30)) return fail(DIALSORT_E_INVALID_ARG, "radix path supports n < 2^30 per call");
  int rc;
  const uint32_t* src = reinterpret_cast<const uint32_t*>(keys);
  uint32_t* bufs[2] = {reinterpret_cast<uint32_t*>(tmp), reinterpret_cast<uint32_t*>(out)};
  auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; };
  bool aligned = al(keys) && al(out) && al(tmp);
  if (pass_out) aligned = al(keys) && al(pass_out) && (n % 4 == 0);
  const int v = radix_variant(c, aligned);
  const uint32_t G = (uint32_t)std::max<uint64_t>(
      1, std::min<uint64_t>(cdiv(n, v == 4 ? kR4Tile : kR3Tile), (uint64_t)c->nsm * (v == 4 ? c->radix4_occ : c->radix3_occ)));
  if ((rc = c->radix_hist.ensure(8ull * 256 * G + 4 * 256 + 64))) return rc;
  Radix2Ws w;
  w.cnt = c->radix_hist.as<uint32_t>();
  w.pre = w.cnt + 256 * G;
  w.total = w.pre + 256 * G;
  w.bar = reinterpret_cast<GridBarR*>(c->gridbar.as<char>() + 32);
  w.pt = c->pt;
  w.d_n = d_n;
  for (int p = 0; p < 4; ++p) {
    uint32_t* dst = pass_out ? pass_out + (uint64_t)p * n : bufs[p & 1];
    if (v == 4)
      DS_CUDA(launch_k<true>(KID_RADIX_PASS, k_radix_pass4, dim3(G), dim3(kR4Threads), sizeof(Radix4Smem), s, src,
                             dst, (uint32_t)n, p, w));
    else
      DS_CUDA(launch_k<true>(KID_RADIX_PASS, k_radix_pass3, dim3(G), dim3(kRadixThreads), sizeof(Radix3Smem), s, src,
                             dst, (uint32_t)n, p, w));
    src = dst;
  }
  return DIALSORT_OK;
}

// Makes `c`'s profiler the active one for launches made by this thread during an API call
// (and its cooperative-launch option), and brackets the call in an NVTX range named after the
// entry point (ncu --nvtx --nvtx-include "dialsort_sort_async/" selects one call's kernels).
struct ProfScope {
  Profiler* prev;
  bool prev_coop;
  explicit ProfScope(dialsort_ctx c, const char* api = "dialsort") : prev(g_prof), prev_coop(g_coop_attr) {
    g_prof = c ? &c->prof : nullptr;
    g_coop_attr = c ? c->coop_attr : false;
    nvtxRangePushA(api);
  }
  ~ProfScope() {
    nvtxRangePop();
    g_prof = prev;
    g_coop_attr = prev_coop;
  }
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

int check_comm(dialsort_ctx c, dialsort_comm m) {
  if (!c || !m) return fail(DIALSORT_E_INVALID_ARG, "ctx / comm is NULL");
  if (m->ctx != c) return fail(DIALSORT_E_INVALID_ARG, "comm belongs to another context");
  if (!m->connected) return fail(DIALSORT_E_INVALID_ARG, "comm is not connected");
  return DIALSORT_OK;
}

}  // namespace

extern "C" {

const char* dialsort_status_string(int s) {
  switch (s) {
    case DIALSORT_OK: return "ok";
    case DIALSORT_E_INVALID_ARG: return "invalid argument";
    case DIALSORT_E_KEY_RANGE: return "key outside [0,U)";
    case DIALSORT_E_SIZE: return "size mismatch (sum(H) vs n / capacity)";
    case DIALSORT_E_OVERFLOW: return "count overflow";
    case DIALSORT_E_CUDA: return "CUDA error";
    case DIALSORT_E_COMM: return "multi-GPU exchange timed out";
    case DIALSORT_E_NOMEM: return "out of device memory";
    default: return "unknown status";
  }
}

const char* dialsort_last_error(void) { return g_last_error.c_str(); }
int dialsort_version(void) { return 200; }

int dialsort_ctx_create(int device, uint64_t max_n, uint32_t max_U, dialsort_ctx* out) {
  if (!out) return fail(DIALSORT_E_INVALID_ARG, "out is NULL");
  dialsort_ctx c = new dialsort_ctx_s();
  c->device = device;
  int rc = ctx_init(c);
  if (!rc && max_U) {
    const HistPath path = choose_path(max_U);
    if (path == HistPath::Smem32 || path == HistPath::Smem16) {
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
  for (dialsort_ctx& l : c->lanes)
    if (l) {
      dialsort_ctx_destroy(l);
      l = nullptr;
    }
  for (DBuf* b : {&c->partials, &c->P, &c->tfb, &c->ws_total, &c->ovfH, &c->status, &c->stage, &c->Hws,
                  &c->range_tot, &c->gridbar, &c->tsums, &c->radix_tmp, &c->radix_hist, &c->fused_tiles, &c->Hx,
                  &c->part, &c->htmp, &c->qtmp, &c->psamp, &c->ringws})
    b->release();
  if (c->host_status) cudaFreeHost(c->host_status);
  if (c->pt && c->owns_pt) cudaFree(c->pt);
  for (cudaEvent_t e : c->prof.ev) cudaEventDestroy(e);
  delete c;
  return DIALSORT_OK;
}

int dialsort_ctx_set_option(dialsort_ctx c, int option, int64_t value) {
  if (!c) return fail(DIALSORT_E_INVALID_ARG, "ctx is NULL");
  switch (option) {
    case DIALSORT_OPT_RADIX_VARIANT:
      if (value != 0 && value != 3 && value != 4) return fail(DIALSORT_E_INVALID_ARG, "radix variant: 0, 3 or 4");
      c->radix_force = (int)value;
      return DIALSORT_OK;
    case DIALSORT_OPT_COOPERATIVE:
      c->coop_attr = value != 0;
      return DIALSORT_OK;
    case DIALSORT_OPT_MAX_CTAS:
      if (value < 0 || value > 1024) return fail(DIALSORT_E_INVALID_ARG, "max CTAs: 0..1024");
      c->max_ctas = (uint32_t)value;
      return DIALSORT_OK;
    case DIALSORT_OPT_PART_MODE:
      if (value < 0 || value > 2) return fail(DIALSORT_E_INVALID_ARG, "partition mode: 0, 1 or 2");
      c->part_mode = (int)value;
      return DIALSORT_OK;
    default:
      return fail(DIALSORT_E_INVALID_ARG, "unknown or read-only option");
  }
}

int dialsort_ctx_get_option(dialsort_ctx c, int option, int64_t* value) {
  if (!c || !value) return fail(DIALSORT_E_INVALID_ARG, "NULL argument");
  switch (option) {
    case DIALSORT_OPT_RADIX_VARIANT: *value = c->radix_force; return DIALSORT_OK;
    case DIALSORT_OPT_RADIX_PROBE_VIOLATIONS: *value = c->probe_violations; return DIALSORT_OK;
    case DIALSORT_OPT_RADIX_ACTIVE: *value = radix_variant(c, true); return DIALSORT_OK;
    case DIALSORT_OPT_NUM_SMS: *value = c->nsm; return DIALSORT_OK;
    case DIALSORT_OPT_COOPERATIVE: *value = c->coop_attr ? 1 : 0; return DIALSORT_OK;
    case DIALSORT_OPT_MAX_CTAS: *value = c->max_ctas; return DIALSORT_OK;
    case DIALSORT_OPT_PART_MODE: *value = c->part_mode; return DIALSORT_OK;
    default: return fail(DIALSORT_E_INVALID_ARG, "unknown option");
  }
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
  for (dialsort_ctx l : c->lanes) {  // the batched sort's lanes (their work is on this stream too)
    if (!l) continue;
    DevStatus lh;
    DS_CUDA(cudaMemcpy(&lh, l->status.p, sizeof(DevStatus), cudaMemcpyDeviceToHost));
    if (!lh.bad_count && !lh.flags) continue;
    h.bad_count += lh.bad_count;
    h.first_bad = std::min(h.first_bad, lh.first_bad);
    h.flags |= lh.flags;
    DevStatus lc = {};
    lc.first_bad = ~0ull;
    lc.ovf_epoch = lh.ovf_epoch;
    lc.last_total = lh.last_total;
    DS_CUDA(cudaMemcpy(l->status.p, &lc, sizeof(lc), cudaMemcpyHostToDevice));
  }
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
  if (h.flags & FLAG_COMM) return fail(DIALSORT_E_COMM, "a peer did not reach the exchange within the timeout");
  if (h.flags & FLAG_OVERFLOW) return fail(DIALSORT_E_OVERFLOW, "sum(H) >= 2^32");
  if (h.flags & FLAG_SIZE)
    return fail(DIALSORT_E_SIZE, "sum(H) = " + std::to_string(h.last_total) + " does not match n / capacity");
  return DIALSORT_OK;
}

// Small inputs on one thread-block cluster (k_sort_small, ds_small.cuh): 8 CTAs up to
// kSmall8MaxN keys, 16 (if the device schedules them) up to small16_max_n(U); out == nullptr:
// histogram only.  done = false: not a small input (nothing enqueued).
int enqueue_small(dialsort_ctx c, const int32_t* keys, uint64_t n, uint32_t U, int32_t* out, uint32_t* H,
                  cudaStream_t s, bool& done) {
  static const bool small_on = [] {  // (DIALSORT_SMALL=0: the fused co-resident grid instead, A/B)
    const char* e = getenv("DIALSORT_SMALL");
    return !(e && e[0] == '0');
  }();
  done = false;
  if (!small_on || U > kSmallMaxU || c->nsm < 16) return DIALSORT_OK;
  if (n <= (c->small16 ? kSmall8MaxN : kSmall8OnlyMaxN)) {
    DS_CUDA((launch_k<false, 8>(KID_SORT_SMALL, k_sort_small<8>, dim3(8), dim3(kSmallThreads), 0, s, keys, n, U, out,
                                H, c->status.as<DevStatus>())));
    done = true;
  } else if (c->small16 && n <= small16_max_n(U)) {
    DS_CUDA((launch_k<false, 16>(KID_SORT_SMALL, k_sort_small<16>, dim3(16), dim3(kSmallThreads), 0, s, keys, n, U,
                                 out, H, c->status.as<DevStatus>())));
    done = true;
  }
  return DIALSORT_OK;
}

int dialsort_histogram_async(dialsort_ctx c, const int32_t* keys, uint64_t n, uint32_t U, uint32_t* H,
                             dialsort_stream_t stream) {
  int rc;
  if (!c) return fail(DIALSORT_E_INVALID_ARG, "ctx is NULL");
  ProfScope prof_scope_(c, __func__);
  if ((rc = check_U(U)) || (rc = check_keys_arg(keys, n))) return rc;
  if (!H) return fail(DIALSORT_E_INVALID_ARG, "H is NULL");
  cudaStream_t s = (cudaStream_t)stream;
  DS_CUDA(cudaSetDevice(c->device));
  const uint32_t epoch = next_epoch(c);
  if (n == 0) {
    DS_CUDA(launch_k(KID_ZERO, k_zero, dim3(c->nsm), dim3(256), 0, s, H, (uint64_t)U));
    return DIALSORT_OK;
  }
  bool done = false;
  if ((rc = enqueue_small(c, keys, n, U, nullptr, H, s, done)) || done) return rc;
  return enqueue_hist_scan(c, keys, n, U, H, false, 0, epoch, s);
}

int dialsort_reconstruct_async(dialsort_ctx c, const uint32_t* H, uint32_t U, int32_t key_base, int32_t* out,
                               uint64_t cap, int exact, uint64_t* d_total, dialsort_stream_t stream) {
  int rc;
  if (!c) return fail(DIALSORT_E_INVALID_ARG, "ctx is NULL");
  ProfScope prof_scope_(c, __func__);
  if ((rc = check_U(U)) || (rc = check_keys_arg(out, cap))) return rc;
  if (!H) return fail(DIALSORT_E_INVALID_ARG, "H is NULL");
  if ((int64_t)key_base + (int64_t)U - 1 > 0x7fffffffll)
    return fail(DIALSORT_E_INVALID_ARG, "key_base + U - 1 exceeds INT32_MAX");
  cudaStream_t s = (cudaStream_t)stream;
  DS_CUDA(cudaSetDevice(c->device));
  const uint32_t epoch = next_epoch(c);
  if (reconstruct_fused_applies(H, U)) return enqueue_reconstruct_fused(c, H, U, key_base, out, cap, exact != 0, d_total, epoch, s);
  if ((rc = enqueue_scan(c, H, U, cap, exact != 0, d_total, epoch, s))) return rc;
  return enqueue_expand(c, U, cap, key_base, out, s);
}

int dialsort_sort_async(dialsort_ctx c, const int32_t* keys, uint64_t n, uint32_t U, int32_t* out, uint32_t* H_out,
                        dialsort_stream_t stream) {
  int rc;
  if (!c) return fail(DIALSORT_E_INVALID_ARG, "ctx is NULL");
  ProfScope prof_scope_(c, __func__);
  if ((rc = check_U(U)) || (rc = check_keys_arg(keys, n)) || (rc = check_keys_arg(out, n))) return rc;
  if (n && out != keys && ranges_overlap(keys, 4 * n, out, 4 * n))
    return fail(DIALSORT_E_INVALID_ARG, "out partially overlaps keys (only out == keys is allowed)");
  cudaStream_t s = (cudaStream_t)stream;
  DS_CUDA(cudaSetDevice(c->device));
  const uint32_t epoch = next_epoch(c);
  if (n == 0) {
    if (H_out) DS_CUDA(launch_k(KID_ZERO, k_zero, dim3(c->nsm), dim3(256), 0, s, H_out, (uint64_t)U));
    return DIALSORT_OK;
  }
  uint32_t* H = H_out;
  if (!H) {
    if ((rc = c->Hws.ensure(4ull * U))) return rc;
    H = c->Hws.as<uint32_t>();
  }
  // small inputs: the whole step on one thread-block cluster (ds_small.cuh)
  bool done = false;
  if ((rc = enqueue_small(c, keys, n, U, out, H_out, s, done)) || done) return rc;
  const HistPath path = choose_path(U);
  if (path == HistPath::Smem32 || path == HistPath::Smem16) return enqueue_sort_fused(c, keys, n, U, H, out, epoch, s);
  if (path == HistPath::Hier) return enqueue_hier(c, keys, n, U, H, out, s);
  if ((rc = enqueue_hist_scan(c, keys, n, U, H, true, n, epoch, s))) return rc;
  return enqueue_expand(c, U, n, 0, out, s);
}

int dialsort_sort_batch_async(dialsort_ctx c, const int32_t* const* keys, const uint64_t* n, uint32_t U,
                              int32_t* const* out, uint32_t* const* H_out, uint32_t nb, dialsort_stream_t stream) {
  int rc;
  if (!c) return fail(DIALSORT_E_INVALID_ARG, "ctx is NULL");
  ProfScope prof_scope_(c, __func__);
  if ((rc = check_U(U))) return rc;
  if (nb && (!keys || !n || !out)) return fail(DIALSORT_E_INVALID_ARG, "NULL batch arrays");
  for (uint32_t j = 0; j < nb; ++j) {
    if ((rc = check_keys_arg(keys[j], n[j])) || (rc = check_keys_arg(out[j], n[j]))) return rc;
    if (n[j] && out[j] != keys[j] && ranges_overlap(keys[j], 4 * n[j], out[j], 4 * n[j]))
      return fail(DIALSORT_E_INVALID_ARG, "out partially overlaps keys (only out == keys is allowed)");
  }
  cudaStream_t s = (cudaStream_t)stream;
  DS_CUDA(cudaSetDevice(c->device));
  {  // small batches: one thread-block cluster per batch, all in one launch (ds_small.cuh)
    static const bool small_on = [] {
      const char* e = getenv("DIALSORT_SMALL");
      return !(e && e[0] == '0');
    }();
    uint64_t nmax = 0, nmin = ~0ull;
    for (uint32_t j = 0; j < nb; ++j) nmax = std::max(nmax, n[j]), nmin = std::min(nmin, n[j]);
    const bool use16 = c->small16 && nmax > kSmallBatch8MaxN;
    if (small_on && nb > 1 && nmin > 0 && U <= kSmallMaxU && c->nsm >= 16 &&
        nmax <= (c->small16 ? small16_max_n(U) : kSmallBatch8MaxN)) {
      for (uint32_t j0 = 0; j0 < nb; j0 += kSmallBatchMax) {
        const uint32_t m = std::min<uint32_t>(kSmallBatchMax, nb - j0);
        SmallBatch B;
        memset(&B, 0, sizeof B);
        for (uint32_t j = 0; j < m; ++j) {
          B.keys[j] = keys[j0 + j];
          B.out[j] = out[j0 + j];
          B.H[j] = H_out ? H_out[j0 + j] : nullptr;
          B.n[j] = n[j0 + j];
        }
        if (use16)
          DS_CUDA((launch_k<false, 16>(KID_SORT_SMALL_BATCH, k_sort_small_batch<16>, dim3(16 * m), dim3(kSmallThreads),
                                       0, s, B, U, c->status.as<DevStatus>())));
        else
          DS_CUDA((launch_k<false, 8>(KID_SORT_SMALL_BATCH, k_sort_small_batch<8>, dim3(8 * m), dim3(kSmallThreads), 0,
                                      s, B, U, c->status.as<DevStatus>())));
      }
      return DIALSORT_OK;
    }
  }
  const HistPath path = choose_path(U);
  static const uint32_t kGroups = [] {  // CTA groups per launch (DIALSORT_BATCH_GROUPS: experiments)
    const char* e = getenv("DIALSORT_BATCH_GROUPS");
    const int v = e ? atoi(e) : 4;
    return (uint32_t)(v < 2 ? 2 : v > kMaxLanes ? kMaxLanes : v);
  }();
  const uint32_t Lmax = std::min<uint32_t>(kGroups, (uint32_t)c->nsm / 8);
  for (uint32_t j0 = 0; j0 < nb; j0 += kBatchMax) {
    const uint32_t m = std::min<uint32_t>(kBatchMax, nb - j0);
    // groups: at most kGroups, and few enough that every group keeps its own-tile projection
    // (ntiles <= kFPassTiles per CTA).  (5-6 groups measured slower for every order; Zipf at 5
    // groups of 29 CTAs: 134 us per batch vs 22 us at 4 groups of 37 — its hottest key passes
    // 65535 copies per CTA, the 16-bit counters' overflow fallback)
    const uint64_t ntl = cdiv(U, kFTileBins);
    const uint32_t Lown = (uint32_t)std::max<uint64_t>(1, (uint64_t)c->nsm * kFPassTiles / ntl);
    const uint32_t L = std::min<uint32_t>(std::min<uint32_t>(Lmax, Lown), m);
    const uint32_t Gg = std::min<uint32_t>(kFMaxRows, (uint32_t)c->nsm / std::max<uint32_t>(L, 1));
    // one launch needs every batch on the shared-memory path in one row format, and no empty one
    bool together = L >= 2 && (path == HistPath::Smem32 || path == HistPath::Smem16);
    int fmt0 = -1;
    for (uint32_t j = 0; together && j < m; ++j) {
      const uint64_t nj = n[j0 + j];
      const int f = U <= kSmem32MaxBins ? kRowU32 : (nj <= 8ull * Gg * U ? kRowN4 : kRowP16);
      if (nj == 0 || (fmt0 >= 0 && f != fmt0)) together = false;
      fmt0 = f;
    }
    if (!together) {  // one step after the other on the whole grid
      for (uint32_t j = 0; j < m; ++j)
        if ((rc = dialsort_sort_async(c, keys[j0 + j], n[j0 + j], U, out[j0 + j], H_out ? H_out[j0 + j] : nullptr,
                                      stream)))
          return rc;
      continue;
    }
    BatchArgs B;
    memset(&B, 0, sizeof B);
    B.nb = m;
    B.L = L;
    B.Gg = Gg;
    size_t smem = 0;
    int fmt = -1;
    for (uint32_t g = 0; g < L; ++g) {  // lanes: each group's own workspace and status
      if (!c->lanes[g]) {
        dialsort_ctx l = nullptr;
        if ((rc = dialsort_ctx_create(c->device, 0, 0, &l))) return rc;
        if (l->pt) cudaFree(l->pt);
        l->pt = c->pt;
        l->owns_pt = false;
        c->lanes[g] = l;
      }
    }
    for (uint32_t j = 0; j < m; ++j) {
      dialsort_ctx l = c->lanes[j % L];
      uint32_t* H = H_out ? H_out[j0 + j] : nullptr;
      if (!H) {
        if ((rc = l->Hws.ensure(4ull * U))) return rc;
        H = l->Hws.as<uint32_t>();
      }
      uint32_t C;
      if ((rc = build_fused_args(l, B.a[j], fmt, C, smem, n[j0 + j], U, H, next_epoch(l), nullptr, nullptr, 4, false,
                                 nullptr, 0, 0, 0, nullptr, nullptr, Gg, 3)))
        return rc;
      B.keys[j] = keys[j0 + j];
      B.n[j] = n[j0 + j];
      B.out[j] = out[j0 + j];
    }
    const dim3 grid(L * Gg);
    if (fmt == kRowN4)
      DS_CUDA(launch_k<true>(KID_SORT_BATCH, k_sort_batch<kRowN4>, grid, dim3(1024), smem, s, B));
    else if (fmt == kRowP16)
      DS_CUDA(launch_k<true>(KID_SORT_BATCH, k_sort_batch<kRowP16>, grid, dim3(1024), smem, s, B));
    else
      DS_CUDA(launch_k<true>(KID_SORT_BATCH, k_sort_batch<kRowU32>, grid, dim3(1024), smem, s, B));
  }
  return DIALSORT_OK;
}

int dialsort_sort_int32_async(dialsort_ctx c, const int32_t* keys, uint64_t n, int32_t* out, dialsort_stream_t stream) {
  int rc;
  if (!c) return fail(DIALSORT_E_INVALID_ARG, "ctx is NULL");
  ProfScope prof_scope_(c, __func__);
  if ((rc = check_keys_arg(keys, n)) || (rc = check_keys_arg(out, n))) return rc;
  if (n && out != keys && ranges_overlap(keys, 4 * n, out, 4 * n))
    return fail(DIALSORT_E_INVALID_ARG, "out partially overlaps keys (only out == keys is allowed)");
  cudaStream_t s = (cudaStream_t)stream;
  DS_CUDA(cudaSetDevice(c->device));
  if (n == 0) return DIALSORT_OK;
  if ((rc = c->radix_tmp.ensure(4ull * n + 16))) return rc;
  return radix_enqueue(c, keys, n, out, c->radix_tmp.as<int32_t>(), s);
}

int dialsort_sort_domain_async(dialsort_ctx c, const void* items, int item_bytes, uint64_t n, uint32_t U,
                               const uint32_t* encode, const int32_t* decode, int32_t* out, dialsort_stream_t stream) {
  int rc;
  if (!c) return fail(DIALSORT_E_INVALID_ARG, "ctx is NULL");
  ProfScope prof_scope_(c, __func__);
  if ((rc = check_U(U)) || (rc = check_keys_arg(out, n))) return rc;
  if (item_bytes != 1 && item_bytes != 2 && item_bytes != 4) return fail(DIALSORT_E_INVALID_ARG, "item_bytes: 1, 2 or 4");
  if (n > 0xffffffffull) return fail(DIALSORT_E_INVALID_ARG, "n exceeds 2^32-1");
  if (n && !items) return fail(DIALSORT_E_INVALID_ARG, "NULL items with n > 0");
  if (reinterpret_cast<uintptr_t>(items) & (item_bytes - 1)) return fail(DIALSORT_E_INVALID_ARG, "items misaligned");
  if (encode && item_bytes != 1) return fail(DIALSORT_E_INVALID_ARG, "an encode table needs 1-byte items");
  if ((item_bytes == 1 && U > kSmem32MaxBins) || (item_bytes == 2 && U > 65536) || (item_bytes == 4 && U > kSmem16MaxBins))
    return fail(DIALSORT_E_INVALID_ARG, "U too large for the item width (1 B: 8192, 2 B: 65536, 4 B: 98304)");
  if (n && ranges_overlap(items, (uint64_t)item_bytes * n, out, 4 * n) && (item_bytes != 4 || items != out))
    return fail(DIALSORT_E_INVALID_ARG, "out overlaps the items");
  cudaStream_t s = (cudaStream_t)stream;
  DS_CUDA(cudaSetDevice(c->device));
  const uint32_t epoch = next_epoch(c);
  if (n == 0) return DIALSORT_OK;
  if ((rc = c->Hws.ensure(4ull * U))) return rc;
  return enqueue_sort_fused(c, items, n, U, c->Hws.as<uint32_t>(), out, epoch, s, 0, nullptr, nullptr, item_bytes,
                            false, nullptr, 0, 0, 0, encode, decode);
}

int dialsort_debug_radix_passes(dialsort_ctx c, const int32_t* keys, uint64_t n, uint32_t* pass_out,
                                dialsort_stream_t stream) {
  int rc;
  if (!c) return fail(DIALSORT_E_INVALID_ARG, "ctx is NULL");
  ProfScope prof_scope_(c, __func__);
  if ((rc = check_keys_arg(keys, n)) || (rc = check_keys_arg(pass_out, 4 * n))) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  DS_CUDA(cudaSetDevice(c->device));
  if (n == 0) return DIALSORT_OK;
  return radix_enqueue(c, keys, n, nullptr, nullptr, s, nullptr, pass_out);
}

int dialsort_range_count_async(dialsort_ctx c, const uint32_t* H, uint32_t U, uint32_t a, uint32_t b,
                               uint64_t* d_result, dialsort_stream_t stream) {
  int rc;
  if (!c) return fail(DIALSORT_E_INVALID_ARG, "ctx is NULL");
  ProfScope prof_scope_(c, __func__);
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

int dialsort_query_async(dialsort_ctx c, const uint32_t* H, uint32_t U, int op, const uint32_t* q, uint64_t m,
                         uint64_t* d_out, dialsort_stream_t stream) {
  if (!c) return fail(DIALSORT_E_INVALID_ARG, "ctx is NULL");
  ProfScope prof_scope_(c, __func__);
  int rc;
  if ((rc = check_U(U))) return rc;
  if (op != DIALSORT_Q_FREQUENCY && op != DIALSORT_Q_PRESENCE && op != DIALSORT_Q_RANGE_COUNT)
    return fail(DIALSORT_E_INVALID_ARG, "unknown query op");
  if (m == 0) return DIALSORT_OK;
  if (!H || !q || !d_out) return fail(DIALSORT_E_INVALID_ARG, "NULL pointer");
  cudaStream_t s = (cudaStream_t)stream;
  DS_CUDA(cudaSetDevice(c->device));
  if (op == DIALSORT_Q_RANGE_COUNT) {
    // prefix of H (uint64, exclusive, U + 1 entries) in the context's query workspace
    int rc2;
    if ((rc2 = c->qtmp.ensure(8ull * (U + 1 + c->nsm) + 64))) return rc2;
    uint64_t* pre = c->qtmp.as<uint64_t>();
    const uint32_t g = (uint32_t)std::min<uint64_t>(c->nsm, cdiv(U, 4096));
    DS_CUDA(launch_k<true>(KID_QUERY, k_query_prefix, dim3(g), dim3(1024), 0, s, H, U, pre,
                           reinterpret_cast<GridBar*>(c->gridbar.as<char>() + 128)));
    DS_CUDA(launch_k(KID_QUERY, k_query_range, dim3((uint32_t)std::min<uint64_t>(cdiv(m, 256), 4ull * c->nsm)),
                     dim3(256), 0, s, (const uint64_t*)pre, U, q, m, d_out, c->status.as<DevStatus>()));
    return DIALSORT_OK;
  }
  DS_CUDA(launch_k(KID_QUERY, k_query_point, dim3((uint32_t)std::min<uint64_t>(cdiv(m, 256), 4ull * c->nsm)), dim3(256),
                   0, s, H, U, op, q, m, d_out, c->status.as<DevStatus>()));
  return DIALSORT_OK;
}

int dialsort_support_set_async(dialsort_ctx c, const uint32_t* H, uint32_t U, uint32_t* D_out, uint64_t* d_count,
                               uint32_t* d_iso, dialsort_stream_t stream) {
  if (!c) return fail(DIALSORT_E_INVALID_ARG, "ctx is NULL");
  ProfScope prof_scope_(c, __func__);
  int rc;
  if ((rc = check_U(U))) return rc;
  if (!H || !D_out || !d_count) return fail(DIALSORT_E_INVALID_ARG, "NULL pointer");
  cudaStream_t s = (cudaStream_t)stream;
  DS_CUDA(cudaSetDevice(c->device));
  const uint32_t grid = (uint32_t)std::min<uint64_t>(c->nsm, cdiv(U, 4096));
  if ((rc = c->qtmp.ensure(8ull * (grid + 1) + 64))) return rc;
  DS_CUDA(launch_k<true>(KID_QUERY, k_support_set, dim3(grid), dim3(1024), 0, s, H, U, D_out,
                         reinterpret_cast<unsigned long long*>(d_count), d_iso, c->qtmp.as<unsigned long long>(),
                         reinterpret_cast<GridBar*>(c->gridbar.as<char>() + 128)));
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
  ProfScope prof_scope_(c, __func__);
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

// ---- multi-GPU: communicator over peer memory ----------------------------------------------

int dialsort_comm_create(dialsort_ctx c, uint32_t G, uint32_t rank, uint32_t max_U, uint64_t max_recv_keys,
                         void* handle_out, dialsort_comm* out) {
  if (!c || !out) return fail(DIALSORT_E_INVALID_ARG, "NULL argument");
  if (G == 0 || G > kCommMaxRanks || rank >= G) return fail(DIALSORT_E_INVALID_ARG, "need 1 <= G <= 8 and rank < G");
  if (max_recv_keys > 0xffffffffull) return fail(DIALSORT_E_INVALID_ARG, "max_recv_keys exceeds 2^32-1");
  DS_CUDA(cudaSetDevice(c->device));
  dialsort_comm m = new dialsort_comm_s();
  m->ctx = c;
  m->G = G;
  m->rank = rank;
  const uint32_t Lmax = (uint32_t)cdiv(max_U ? max_U : 1, G);
  m->lay = comm_layout(G, (uint32_t)round_up(Lmax, 4), round_up(max_recv_keys ? max_recv_keys : 4, 64));
  int rc = DIALSORT_OK;
  if (cudaMalloc(&m->ws, m->lay.bytes) != cudaSuccess) {
    cudaGetLastError();
    delete m;
    return fail(DIALSORT_E_NOMEM, "comm workspace allocation failed");
  }
  if (cudaMemset(m->ws, 0, m->lay.bytes) != cudaSuccess) rc = fail(DIALSORT_E_CUDA, "cudaMemset failed");
  if (!rc) rc = m->tables.ensure(8ull * 2 * kCommMaxRanks);
  if (!rc) rc = m->scratch.ensure(kScratchPlan + 4 * 320, true);
  if (!rc) rc = m->hslice.ensure(4ull * m->lay.Lmax);
  if (!rc && handle_out) {
    CommHandle h = {};
    cudaIpcMemHandle_t ih;
    if (cudaIpcGetMemHandle(&ih, m->ws) != cudaSuccess) {
      cudaGetLastError();
      memset(&ih, 0, sizeof ih);  // (single-process use: dialsort_comm_connect_local needs no handle)
    }
    memcpy(h.ipc, &ih, 64);
    h.magic = kCommMagic;
    h.G = G;
    h.rank = rank;
    h.Lmax = m->lay.Lmax;
    h.cap = m->lay.cap;
    h.bytes = m->lay.bytes;
    h.device = c->device;
    memcpy(handle_out, &h, sizeof h);
  }
  if (rc) {
    dialsort_comm_destroy(m);
    return rc;
  }
  m->peer[rank] = static_cast<char*>(m->ws);
  *out = m;
  return DIALSORT_OK;
}

static int comm_finish_connect(dialsort_comm m) {
  // owner receive-slot tables for the two parities: owner s's recv region of parity p
  std::vector<uint32_t*> t(2 * kCommMaxRanks, nullptr);
  for (uint32_t p = 0; p < 2; ++p)
    for (uint32_t s = 0; s < m->G; ++s)
      t[p * kCommMaxRanks + s] =
          reinterpret_cast<uint32_t*>(m->peer[s] + m->lay.recv) + (uint64_t)p * m->G * m->lay.Lmax;
  DS_CUDA(cudaMemcpy(m->tables.p, t.data(), 8ull * t.size(), cudaMemcpyHostToDevice));
  m->connected = true;
  return DIALSORT_OK;
}

int dialsort_comm_connect_ipc(dialsort_comm m, const void* handles) {
  if (!m || !handles) return fail(DIALSORT_E_INVALID_ARG, "NULL argument");
  DS_CUDA(cudaSetDevice(m->ctx->device));
  const CommHandle* h = static_cast<const CommHandle*>(handles);
  for (uint32_t s = 0; s < m->G; ++s) {
    if (h[s].magic != kCommMagic || h[s].G != m->G || h[s].rank != s || h[s].Lmax != m->lay.Lmax ||
        h[s].cap != m->lay.cap || h[s].bytes != m->lay.bytes)
      return fail(DIALSORT_E_INVALID_ARG, "comm handle " + std::to_string(s) + " does not match this communicator");
  }
  for (uint32_t s = 0; s < m->G; ++s) {
    if (s == m->rank) continue;
    cudaIpcMemHandle_t ih;
    memcpy(&ih, h[s].ipc, 64);
    void* p = nullptr;
    DS_CUDA(cudaIpcOpenMemHandle(&p, ih, cudaIpcMemLazyEnablePeerAccess));
    m->peer[s] = static_cast<char*>(p);
    m->ipc_mapped[s] = true;
  }
  return comm_finish_connect(m);
}

int dialsort_comm_connect_local(dialsort_comm m, const dialsort_comm* peers) {
  if (!m || !peers) return fail(DIALSORT_E_INVALID_ARG, "NULL argument");
  DS_CUDA(cudaSetDevice(m->ctx->device));
  for (uint32_t s = 0; s < m->G; ++s) {
    const dialsort_comm q = peers[s];
    if (!q || q->G != m->G || q->rank != s || q->lay.bytes != m->lay.bytes || q->lay.Lmax != m->lay.Lmax ||
        q->lay.cap != m->lay.cap)
      return fail(DIALSORT_E_INVALID_ARG, "peer comm " + std::to_string(s) + " does not match this communicator");
    if (q->ctx->device != m->ctx->device) {
      cudaError_t e = cudaDeviceEnablePeerAccess(q->ctx->device, 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
        return fail(DIALSORT_E_CUDA, std::string("cudaDeviceEnablePeerAccess: ") + cudaGetErrorString(e));
      cudaGetLastError();
    }
    m->peer[s] = static_cast<char*>(q->ws);
  }
  return comm_finish_connect(m);
}

int dialsort_comm_destroy(dialsort_comm m) {
  if (!m) return DIALSORT_OK;
  cudaSetDevice(m->ctx->device);
  cudaDeviceSynchronize();
  for (uint32_t s = 0; s < kCommMaxRanks; ++s)
    if (m->ipc_mapped[s]) cudaIpcCloseMemHandle(m->peer[s]);
  if (m->ws) cudaFree(m->ws);
  m->tables.release();
  m->scratch.release();
  m->hslice.release();
  delete m;
  return DIALSORT_OK;
}

int dialsort_comm_info(dialsort_comm m, uint32_t* G, uint32_t* rank, uint32_t* epoch) {
  if (!m) return fail(DIALSORT_E_INVALID_ARG, "comm is NULL");
  if (G) *G = m->G;
  if (rank) *rank = m->rank;
  if (epoch) *epoch = m->epoch;
  return DIALSORT_OK;
}

int dialsort_sharded_histogram_scatter_async(dialsort_ctx c, dialsort_comm m, const int32_t* keys, uint64_t n,
                                             uint32_t U, dialsort_stream_t stream) {
  int rc;
  if ((rc = check_comm(c, m))) return rc;
  ProfScope prof_scope_(c, __func__);
  if ((rc = check_U(U)) || (rc = check_keys_arg(keys, n))) return rc;
  if (U % m->G != 0 || U / m->G > m->lay.Lmax) return fail(DIALSORT_E_INVALID_ARG, "need U % G == 0 and U / G <= max_U / G");
  cudaStream_t s = (cudaStream_t)stream;
  DS_CUDA(cudaSetDevice(c->device));
  m->epoch++;
  const uint32_t L = U / m->G, par = m->epoch & 1u;
  uint32_t* const* tbl = m->tables.as<uint32_t*>() + par * kCommMaxRanks;
  const uint32_t epoch = next_epoch(c);
  const HistPath path = choose_path(U);
  if (n > 0 && path != HistPath::Global) {  // the merge stores each finished bin into its owner's slot
    if ((rc = enqueue_hist_scan(c, keys, n, U, nullptr, false, 0, epoch, s, tbl, L, m->rank))) return rc;
  } else {  // L2 path (or no keys): the local histogram, then one push kernel
    if ((rc = c->Hws.ensure(4ull * U + 16))) return rc;
    uint32_t* H = c->Hws.as<uint32_t>();
    if (n == 0)
      DS_CUDA(launch_k(KID_ZERO, k_zero, dim3(c->nsm), dim3(256), 0, s, H, (uint64_t)U));
    else if ((rc = enqueue_hist_scan(c, keys, n, U, H, false, 0, epoch, s)))
      return rc;
    DS_CUDA(launch_k(KID_PUSH_SLICES, k_push_slices, dim3(2 * c->nsm), dim3(256), 0, s, (const uint32_t*)H, U, L,
                     m->rank, tbl));
  }
  DS_CUDA(launch_k(KID_COMM_SIGNAL, k_comm_signal, dim3(1), dim3(32), 0, s, comm_dev(m), kFlagHist));
  return DIALSORT_OK;
}

int dialsort_sharded_histogram_gather_async(dialsort_ctx c, dialsort_comm m, uint32_t U, uint32_t* H_slice,
                                            dialsort_stream_t stream) {
  int rc;
  if ((rc = check_comm(c, m))) return rc;
  ProfScope prof_scope_(c, __func__);
  if ((rc = check_U(U))) return rc;
  if (U % m->G != 0 || U / m->G > m->lay.Lmax) return fail(DIALSORT_E_INVALID_ARG, "need U % G == 0 and U / G <= max_U / G");
  cudaStream_t s = (cudaStream_t)stream;
  DS_CUDA(cudaSetDevice(c->device));
  const uint32_t L = U / m->G;
  uint32_t* Hs = H_slice ? H_slice : m->hslice.as<uint32_t>();
  const uint32_t grid = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(2ull * c->nsm, cdiv(L, 256)));
  DS_CUDA(launch_k(KID_COMM_SLICE_SUM, k_comm_slice_sum, dim3(grid), dim3(256), 0, s, comm_dev(m), L, Hs,
                   reinterpret_cast<unsigned long long*>(m->scratch.as<char>() + kScratchTot),
                   c->status.as<DevStatus>()));
  return DIALSORT_OK;
}

int dialsort_sharded_project_async(dialsort_ctx c, dialsort_comm m, uint32_t U, const uint32_t* H_slice, int32_t* out,
                                   uint64_t cap, uint64_t* d_count, uint64_t* d_offset, dialsort_stream_t stream) {
  int rc;
  if ((rc = check_comm(c, m))) return rc;
  ProfScope prof_scope_(c, __func__);
  if ((rc = check_U(U)) || (rc = check_keys_arg(out, cap))) return rc;
  if (U % m->G != 0 || U / m->G > m->lay.Lmax) return fail(DIALSORT_E_INVALID_ARG, "need U % G == 0 and U / G <= max_U / G");
  cudaStream_t s = (cudaStream_t)stream;
  DS_CUDA(cudaSetDevice(c->device));
  const uint32_t L = U / m->G;
  const uint32_t* Hs = H_slice ? H_slice : m->hslice.as<const uint32_t>();
  DS_CUDA(launch_k(KID_COMM_OFFSETS, k_comm_offsets, dim3(1), dim3(32), 0, s, comm_dev(m), cap, d_count, d_offset,
                   c->status.as<DevStatus>()));
  const uint32_t epoch = next_epoch(c);
  if (reconstruct_fused_applies(Hs, L))
    return enqueue_reconstruct_fused(c, Hs, L, (int32_t)(m->rank * L), out, cap, false, nullptr, epoch, s);
  if ((rc = enqueue_scan(c, Hs, L, cap, false, nullptr, epoch, s))) return rc;
  return enqueue_expand(c, L, cap, (int32_t)(m->rank * L), out, s);
}

int dialsort_sharded_sort_async(dialsort_ctx c, dialsort_comm m, const int32_t* keys, uint64_t n, uint32_t U,
                                int32_t* out, uint64_t cap, uint32_t* H_slice, uint64_t* d_count, uint64_t* d_offset,
                                dialsort_stream_t stream) {
  int rc;
  if ((rc = dialsort_sharded_histogram_scatter_async(c, m, keys, n, U, stream))) return rc;
  if ((rc = dialsort_sharded_histogram_gather_async(c, m, U, H_slice, stream))) return rc;
  return dialsort_sharded_project_async(c, m, U, H_slice, out, cap, d_count, d_offset, stream);
}

int dialsort_sharded_radix_hist_async(dialsort_ctx c, dialsort_comm m, const int32_t* keys, uint64_t n,
                                      dialsort_stream_t stream) {
  int rc;
  if ((rc = check_comm(c, m))) return rc;
  ProfScope prof_scope_(c, __func__);
  if ((rc = check_keys_arg(keys, n))) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  DS_CUDA(cudaSetDevice(c->device));
  m->epoch++;
  const uint32_t grid = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(2ull * c->nsm, cdiv(n, 8192)));
  DS_CUDA(launch_k(KID_COMM_RHIST, k_comm_rhist, dim3(grid), dim3(512), 0, s, comm_dev(m), keys, n,
                   reinterpret_cast<uint32_t*>(m->scratch.as<char>() + kScratchRh)));
  return DIALSORT_OK;
}

int dialsort_sharded_radix_split_async(dialsort_ctx c, dialsort_comm m, const int32_t* keys, uint64_t n, uint64_t cap,
                                       uint64_t* d_count, uint64_t* d_offset, dialsort_stream_t stream) {
  int rc;
  if ((rc = check_comm(c, m))) return rc;
  ProfScope prof_scope_(c, __func__);
  if ((rc = check_keys_arg(keys, n))) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  DS_CUDA(cudaSetDevice(c->device));
  uint32_t* plan = reinterpret_cast<uint32_t*>(m->scratch.as<char>() + kScratchPlan);
  DS_CUDA(launch_k(KID_COMM_RPLAN, k_comm_rplan, dim3(1), dim3(256), 0, s, comm_dev(m), plan, cap, d_count, d_offset,
                   c->status.as<DevStatus>()));
  if (n) {
    const uint32_t grid = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(2ull * c->nsm, cdiv(n, kSplitTile)));
    DS_CUDA(launch_k(KID_COMM_RSPLIT, k_comm_rsplit, dim3(grid), dim3(kSplitThreads), 0, s, comm_dev(m), keys, n, plan));
  }
  DS_CUDA(launch_k(KID_COMM_SIGNAL, k_comm_signal, dim3(1), dim3(32), 0, s, comm_dev(m), kFlagRkeys));
  return DIALSORT_OK;
}

int dialsort_sharded_radix_local_async(dialsort_ctx c, dialsort_comm m, int32_t* out, uint64_t cap,
                                       dialsort_stream_t stream) {
  int rc;
  if ((rc = check_comm(c, m))) return rc;
  ProfScope prof_scope_(c, __func__);
  if ((rc = check_keys_arg(out, cap))) return rc;
  cudaStream_t s = (cudaStream_t)stream;
  DS_CUDA(cudaSetDevice(c->device));
  DS_CUDA(launch_k(KID_COMM_WAIT, k_comm_wait, dim3(1), dim3(32), 0, s, comm_dev(m), kFlagRkeys,
                   c->status.as<DevStatus>()));
  const uint64_t bound = std::min<uint64_t>(cap, m->lay.cap);
  if (bound == 0) return DIALSORT_OK;
  if ((rc = c->radix_tmp.ensure(4ull * bound + 16))) return rc;
  const uint32_t* d_n = reinterpret_cast<const uint32_t*>(m->scratch.as<char>() + kScratchPlan) + 32;
  const int32_t* rk = reinterpret_cast<const int32_t*>(m->peer[m->rank] + m->lay.rkeys) + (uint64_t)(m->epoch & 1u) * m->lay.cap;
  return radix_enqueue(c, rk, bound, out, c->radix_tmp.as<int32_t>(), s, d_n);
}

int dialsort_sharded_sort_int32_async(dialsort_ctx c, dialsort_comm m, const int32_t* keys, uint64_t n, int32_t* out,
                                      uint64_t cap, uint64_t* d_count, uint64_t* d_offset, dialsort_stream_t stream) {
  int rc;
  if ((rc = dialsort_sharded_radix_hist_async(c, m, keys, n, stream))) return rc;
  if ((rc = dialsort_sharded_radix_split_async(c, m, keys, n, cap, d_count, d_offset, stream))) return rc;
  return dialsort_sharded_radix_local_async(c, m, out, cap, stream);
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

static int sharded_sync_read(dialsort_ctx c, dialsort_stream_t stream, uint64_t* d2, uint64_t* count_host,
                             uint64_t* offset_host) {
  int rc = dialsort_sync(c, stream, nullptr);
  uint64_t h[2] = {0, 0};
  DS_CUDA(cudaMemcpy(h, d2, 16, cudaMemcpyDeviceToHost));
  if (count_host) *count_host = h[0];
  if (offset_host) *offset_host = h[1];
  return rc;
}

int dialsort_sharded_sort(dialsort_ctx c, dialsort_comm m, const int32_t* keys, uint64_t n, uint32_t U, int32_t* out,
                          uint64_t cap, uint64_t* count_host, uint64_t* offset_host, dialsort_stream_t stream) {
  int rc;
  if ((rc = check_comm(c, m))) return rc;
  uint64_t* d2 = reinterpret_cast<uint64_t*>(m->scratch.as<char>() + kScratchTot + 16);
  if ((rc = dialsort_sharded_sort_async(c, m, keys, n, U, out, cap, nullptr, d2, d2 + 1, stream))) return rc;
  return sharded_sync_read(c, stream, d2, count_host, offset_host);
}

int dialsort_sharded_sort_int32(dialsort_ctx c, dialsort_comm m, const int32_t* keys, uint64_t n, int32_t* out,
                                uint64_t cap, uint64_t* count_host, uint64_t* offset_host, dialsort_stream_t stream) {
  int rc;
  if ((rc = check_comm(c, m))) return rc;
  uint64_t* d2 = reinterpret_cast<uint64_t*>(m->scratch.as<char>() + kScratchTot + 16);
  if ((rc = dialsort_sharded_sort_int32_async(c, m, keys, n, out, cap, d2, d2 + 1, stream))) return rc;
  return sharded_sync_read(c, stream, d2, count_host, offset_host);
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
  ProfScope prof_scope_(c, __func__);
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

/*
 * dialsort.h — C ABI of the B200-native DialSort hot path (arxiv 2605.16667).
 *
 * The method (PAPER.md, line numbers "P:a-b"):
 *   ingestion   eq:ingestion  ∀x∈K: H[x] ← H[x] + 1
 *   CRN         def:crn_level, lem:crn: same-key concurrent writes
 *               are merged by an equality-only additive reduction before reaching H
 *   projection  eq:projection  for k = 0..U-1 emit k exactly H[k] times
 *   radix       tab:radix LSD, base 256, 4 passes, full signed int32
 *
 * Conventions (all entry points):
 *   - Every pointer argument is a CUDA DEVICE pointer on the context's device unless the
 *     parameter name ends in `_host` (then it is host memory, preferably pinned).
 *   - Keys are int32; a bounded-universe key must lie in [0, U).  1 <= U <= 2^31.
 *   - n <= 2^32 - 1 (histogram counts are uint32; reading R4 in DESIGN.md).
 *   - Buffers are owned by the caller; the library never frees or retains them past the
 *     enqueued work.  A context owns only its workspace (sized at create, grown on demand
 *     outside the timed path) and its device status word.  No other global mutable state,
 *     except the lazily created per-device default context used by the synchronous forms.
 *   - Argument errors are returned synchronously and nothing is enqueued.  Data errors
 *     (a key outside [0,U), ΣH != n, count overflow) are detected on the device and
 *     reported by dialsort_sync (async forms) or by the synchronous form's return value;
 *     after such an error the contents of H / out are unspecified.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *   - A context may be used by one host thread / stream at a time (no internal locking).
 */
#ifndef DIALSORT_H_
#define DIALSORT_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  DIALSORT_OK = 0,
  DIALSORT_E_INVALID_ARG = 1, /* U==0 or U>2^31, n>2^32-1, NULL with n>0, bad alignment,
                                 partial overlap of out and keys, U % G != 0, ...        */
  DIALSORT_E_KEY_RANGE = 2,   /* some key outside [0,U) (deferred; info = min bad index)  */
  DIALSORT_E_SIZE = 3,        /* reconstruct: ΣH != n (exact) or ΣH > capacity          */
  DIALSORT_E_OVERFLOW = 4,    /* ΣH >= 2^32 in reconstruct                              */
  DIALSORT_E_CUDA = 5,        /* a CUDA runtime error (message: dialsort_last_error)     */
  DIALSORT_E_NOMEM = 7        /* workspace allocation failed                             */
} dialsort_status;

typedef struct {
  uint64_t bad_count;       /* number of keys outside [0,U) seen since the last sync      */
  uint64_t first_bad_index; /* minimum offending index (UINT64_MAX if none)              */
  int32_t first_bad_key;    /* the key at first_bad_index                                */
  uint32_t flags;           /* bit0 size error, bit1 overflow                            */
  uint64_t last_total;      /* ΣH computed by the most recent reconstruct / sort         */
} dialsort_error_info;

typedef void* dialsort_stream_t;            /* cudaStream_t */
typedef struct dialsort_ctx_s* dialsort_ctx; /* opaque */

/* ---- introspection ------------------------------------------------------------------- */
const char* dialsort_status_string(int status);
const char* dialsort_last_error(void);      /* thread-local message of the last failure   */
int dialsort_version(void);                 /* 100 * major + minor                        */

/* ---- context ------------------------------------------------------------------------- */
/* Create a context on `device` with workspace for n <= max_n keys and U <= max_U (both
 * may be exceeded later: the workspace then grows on the next call, synchronously). */
int dialsort_ctx_create(int device, uint64_t max_n, uint32_t max_U, dialsort_ctx* out);
int dialsort_ctx_destroy(dialsort_ctx ctx);

/* Block until `stream` drains, then report (and clear) the deferred device errors of all
 * work enqueued through `ctx`.  info may be NULL.  Returns the first error kind seen. */
int dialsort_sync(dialsort_ctx ctx, dialsort_stream_t stream, dialsort_error_info* info);

/* ---- the hot path (async: enqueue on `stream`, return after enqueue) ----------------- */

/* Histogram ingestion, eq:ingestion: H[k] = |{i : keys[i] = k}| for k < U.
 * keys: int32[n], any 4-byte alignment.  H: uint32[U], fully overwritten (not accumulated).
 * Same-key writes inside a warp are merged by the CRN (equality only, lem:crn). */
int dialsort_histogram_async(dialsort_ctx ctx, const int32_t* keys, uint64_t n, uint32_t U,
                             uint32_t* H, dialsort_stream_t stream);

/* Ordered projection, eq:projection, of a caller histogram:
 * out[P[k] .. P[k]+H[k]) = key_base + k, where P is the exclusive prefix of H (the GPU's
 * parallel write-offset step; the paper's substrates scan sequentially instead).
 * H: uint32[U].  out: int32 with room for `out_capacity` keys.
 * exact != 0: ΣH must equal out_capacity (else DIALSORT_E_SIZE, deferred).
 * exact == 0: ΣH must be <= out_capacity (else DIALSORT_E_SIZE); min(ΣH, cap) keys written.
 * d_total (device uint64*, nullable) receives ΣH. */
int dialsort_reconstruct_async(dialsort_ctx ctx, const uint32_t* H, uint32_t U,
                               int32_t key_base, int32_t* out, uint64_t out_capacity,
                               int exact, uint64_t* d_total, dialsort_stream_t stream);

/* DialSort (A1): histogram of keys then projection into out (int32[n]).
 * out may alias keys exactly (the paper's in-place form, tab:struct_cost P:1716);
 * partial overlap is DIALSORT_E_INVALID_ARG.  H_out (device uint32[U], nullable) receives
 * the canonical ordered state H. */
int dialsort_sort_async(dialsort_ctx ctx, const int32_t* keys, uint64_t n, uint32_t U,
                        int32_t* out, uint32_t* H_out, dialsort_stream_t stream);

/* DialSort-Radix (tab:radix): full signed int32 range, LSD base 256, 4 passes
 * over sign-flipped keys u = x ^ 0x80000000 (reading R2), each pass a 256-bin DialSort
 * ingestion + per-digit offsets + stable scatter.  out may alias keys exactly. */
int dialsort_sort_int32_async(dialsort_ctx ctx, const int32_t* keys, uint64_t n, int32_t* out,
                              dialsort_stream_t stream);

/* ---- synchronous forms (per-device default context, legacy default stream) ------------ */
int dialsort_histogram(const int32_t* keys, uint64_t n, uint32_t U, uint32_t* H);
int dialsort_reconstruct(const uint32_t* H, uint32_t U, int32_t* out, uint64_t n);
int dialsort_sort(const int32_t* keys, uint64_t n, uint32_t U, int32_t* out);
int dialsort_sort_int32(const int32_t* keys, uint64_t n, int32_t* out);

/* ---- end-to-end with HOST buffers ---------------------------------------------------- */
/* keys_host / out_host: host int32[n] (pinned for full speed; out_host may equal
 * keys_host).  Copies in, sorts on the device (bounded universe U, or full-range radix when
 * U == 0), copies out, all on `stream`, and blocks until done.  Returns the sync status. */
int dialsort_sort_host(dialsort_ctx ctx, const int32_t* keys_host, uint64_t n, uint32_t U,
                       int32_t* out_host, dialsort_stream_t stream);
/* The same without the final wait: copy in, sort and copy out are enqueued on `stream` and the
 * call returns; out_host is valid (and device errors are reported) after dialsort_sync(ctx,
 * stream).  The context's device staging buffer is in use until then, so calls that overlap
 * (a pipeline of host batches) use one context per stream in flight. */
int dialsort_sort_host_async(dialsort_ctx ctx, const int32_t* keys_host, uint64_t n, uint32_t U,
                             int32_t* out_host, dialsort_stream_t stream);

/* ---- multi-GPU exchange over peer memory (lem:crn P:951-962) -- */
/* One rank of G (one process per GPU).  U % G == 0; universe slice s = [s L, (s+1) L), L = U/G,
 * is owned by rank s.  peer_recv: DEVICE array of G device pointers; peer_recv[s] is rank s's
 * receive buffer (uint32[G * L], mapped into this process with dialsort_ipc_open, or this
 * rank's own buffer for s == rank).  Computes the local histogram of keys[n] (device) and
 * stores its slice s into peer_recv[s][rank * L .. rank * L + L) for every s — on the
 * shared-memory paths (U <= 98304) the histogram kernel's merge stores each finished bin
 * straight into the owner's slot (P2P stores over NVLink / NVSwitch, overlapping the rest of
 * the merge); for larger U the local histogram is pushed by one copy kernel.  The writes are
 * complete when the stream's work completes; the owner reads its buffer only after every
 * rank's call completed (e.g. stream sync + a process-group barrier).  Errors as
 * dialsort_histogram_async (E_KEY_RANGE deferred), E_INVALID_ARG for bad G / rank. */
int dialsort_histogram_scatter_async(dialsort_ctx ctx, const int32_t* keys, uint64_t n, uint32_t U,
                                     uint32_t G, uint32_t rank, uint32_t* const* peer_recv,
                                     dialsort_stream_t stream);
/* The owner's step: H_slice[j] = sum over src < G of recv[src * L + j] (device buffers). */
int dialsort_slice_sum_async(dialsort_ctx ctx, const uint32_t* recv, uint32_t G, uint32_t L,
                             uint32_t* H_slice, dialsort_stream_t stream);
/* CUDA IPC of a device allocation (cudaIpcGetMemHandle / cudaIpcOpenMemHandle with lazy peer
 * access / cudaIpcCloseMemHandle) on the context's device; handles are
 * DIALSORT_IPC_HANDLE_BYTES opaque bytes (host memory) exchanged by the caller. */
#define DIALSORT_IPC_HANDLE_BYTES 64
int dialsort_ipc_handle(dialsort_ctx ctx, const void* dev_ptr, void* handle_out);
int dialsort_ipc_open(dialsort_ctx ctx, const void* handle, void** dev_ptr_out);
int dialsort_ipc_close(dialsort_ctx ctx, void* dev_ptr);

/* ---- canonical-state queries on a device histogram (NEXT-1) ---------------- */
/* d_result (device uint64*): Σ_{k=a}^{b} H[k], 0 <= a <= b < U. */
int dialsort_range_count_async(dialsort_ctx ctx, const uint32_t* H, uint32_t U, uint32_t a,
                               uint32_t b, uint64_t* d_result, dialsort_stream_t stream);

/* ---- measurement hooks (bench.py's live per-kernel roofline) --------------------------- */
/* enable != 0: record a CUDA event pair around every kernel this ctx launches (on the
 * launching stream).  The extra stream operations disable the PDL overlap between kernels,
 * so use it only for per-kernel timing passes, never for the headline number. */
int dialsort_profile_enable(dialsort_ctx ctx, int enable);
/* After the stream drained: copy up to `max` records (kernel id, milliseconds) recorded since
 * the last read into the host arrays; returns the record count (or -status on error). */
int dialsort_profile_read(dialsort_ctx ctx, int max, int* kernel_ids, float* ms);
const char* dialsort_kernel_name(int kernel_id);
/* Debug: with DIALSORT_PHASE_TIMING=1 in the environment at context creation, a library
 * built with -DDIALSORT_PHASE_MARKS=1 (tools/build_variant.sh phase; the product build has no
 * stamps and returns zeros) records %globaltimer phase stamps in the fused kernels; this copies 16 values in ns relative to the
 * earliest CTA start into out16 (host): [0..7] the latest CTA's arrival at phase 0..7,
 * [8..15] the earliest CTA's (0 = phase not reached), and resets them. */
int dialsort_debug_phase_ns(dialsort_ctx ctx, uint64_t* out16);
/* Debug: raw per-CTA stamps of the most recent launches (17 per CTA: start, phase 0..15; ns
 * after the earliest start, 0 = not reached) into out[max_ctas * 17] (host); returns the number
 * of CTAs copied, or -status.  Reading resets the stamps (as dialsort_debug_phase_ns). */
int dialsort_debug_phase_cta(dialsort_ctx ctx, uint64_t* out, int max_ctas);

/* ---- test entry: the warp CRN primitive on explicit lane batches ---------------------- */
/* lane_keys: int32[32*n_batches]; active: uint32[n_batches] lane masks.  For each batch, the
 * warp CRN groups the active lanes by equal key; out_keys/out_counts (int32/uint32
 * [32*n_batches]) receive, at the leader lane (lowest lane of each group), the key and the
 * group size; other lanes get count 0.  Inactive lanes get count 0 and are never read. */
int dialsort_crn_resolve_async(dialsort_ctx ctx, const int32_t* lane_keys,
                               const uint32_t* active, uint64_t n_batches, int32_t* out_keys,
                               uint32_t* out_counts, dialsort_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* DIALSORT_H_ */

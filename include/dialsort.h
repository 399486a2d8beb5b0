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
 *   - The single-GPU entries keep their sequencing state on the device, so a CUDA graph that
 *     captured them replays correctly (after one uncaptured call has sized the workspace).
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
  DIALSORT_E_COMM = 6,        /* multi-GPU: a peer did not reach the exchange in time     */
  DIALSORT_E_NOMEM = 7        /* workspace allocation failed                             */
} dialsort_status;

typedef struct {
  uint64_t bad_count;       /* number of keys outside [0,U) seen since the last sync      */
  uint64_t first_bad_index; /* minimum offending index (UINT64_MAX if none)              */
  int32_t first_bad_key;    /* the key at first_bad_index                                */
  uint32_t flags;           /* bit0 size error, bit1 overflow, bit2 exchange timeout     */
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

/* Context options.
 *   DIALSORT_OPT_MAX_CTAS (read / write): cap on the CTAs (one per SM) of the fused sort kernel
 *     (0 = every SM, default).
 *   DIALSORT_OPT_RADIX_VARIANT (read / write): 0 = automatic (default), 3 = k_radix_pass3
 *     (in-warp ranks by explicit equality grouping: stable by construction), 4 = k_radix_pass4
 *     (ranks from the counting shared atomic; needs 16-byte aligned buffers, else pass3).
 *     Automatic uses pass4 only on a device whose lane-order probe (run once per device at
 *     the first dialsort_ctx_create) found no violation, else pass3.
 *   DIALSORT_OPT_RADIX_PROBE_VIOLATIONS (read): lanes of the probe whose atomic return value
 *     broke lane order on this device (0 = pass4 is stable here).
 *   DIALSORT_OPT_RADIX_ACTIVE (read): the variant an aligned radix call uses now (3 or 4).
 *   DIALSORT_OPT_NUM_SMS (read): streaming multiprocessors of the context's device.
 *   DIALSORT_OPT_COOPERATIVE (read / write): the kernels that synchronise their whole grid need it
 *     co-resident.  0 (default): the library orders its co-resident launches of all contexts of a
 *     device in one FIFO (a launch on another stream than the previous one waits for that stream's
 *     enqueued work), so two of them never overlap; 1: cudaLaunchAttributeCooperative, which also
 *     rejects a grid another tenant keeps from being co-resident (DIALSORT_E_CUDA) at ~2 us per
 *     launch.
 *   DIALSORT_OPT_PART_MODE (read / write): the hierarchical path's partition (98304 < U <= 2^22).
 *     0 (default): sampled — a 65536-key stratified sample sizes each universe block's key
 *     region (estimate + 6 sigma), one pass places the keys, and a region overflow runs the exact
 *     schedule on the device (no host round trip); 1: exact — a count pass, then the placement;
 *     2: sampled without margins (overflows: exercises the exact schedule behind it; tests). */
#define DIALSORT_OPT_RADIX_VARIANT 1
#define DIALSORT_OPT_RADIX_PROBE_VIOLATIONS 2
#define DIALSORT_OPT_RADIX_ACTIVE 3
#define DIALSORT_OPT_NUM_SMS 4
#define DIALSORT_OPT_COOPERATIVE 5
#define DIALSORT_OPT_MAX_CTAS 6
#define DIALSORT_OPT_PART_MODE 7
int dialsort_ctx_set_option(dialsort_ctx ctx, int option, int64_t value);
int dialsort_ctx_get_option(dialsort_ctx ctx, int option, int64_t* value);

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

/* A batch of independent DialSorts (a serving engine's stream of sort requests): batch j sorts
 * keys[j][0 .. n[j]) into out[j] (H_out[j]: its histogram, nullable array / entries), all in
 * [0, U).  keys / n / out / H_out are HOST arrays of nb entries; the pointers they hold are device
 * buffers.  On the shared-memory universes (U <= 98304) up to 64 batches run in ONE launch on
 * disjoint groups of CTAs (k_sort_batch: each group sorts its batches one after another on its own
 * workspace; the groups' HBM-bound phases overlap the others' merge phases); other universes,
 * batches of different row formats or single batches are sorted one after another.  Results and
 * errors as nb calls of dialsort_sort_async (errors are reported by dialsort_sync of ctx). */
int dialsort_sort_batch_async(dialsort_ctx ctx, const int32_t* const* keys, const uint64_t* n, uint32_t U,
                              int32_t* const* out, uint32_t* const* H_out, uint32_t nb, dialsort_stream_t stream);

/* DialSort-Radix (tab:radix): full signed int32 range, LSD base 256, 4 passes
 * over sign-flipped keys u = x ^ 0x80000000 (reading R2), each pass a 256-bin DialSort
 * ingestion + per-digit offsets + stable scatter.  out may alias keys exactly. */
int dialsort_sort_int32_async(dialsort_ctx ctx, const int32_t* keys, uint64_t n, int32_t* out,
                              dialsort_stream_t stream);

/* General self-indexing, Proposition 2: a finite totally ordered domain S with a
 * known order-isomorphism phi : S -> [0, U) is sorted by ingesting phi(s) and emitting
 * phi^-1(i) exactly H[i] times ("for other domains a lookup table suffices").
 * items: device array of n elements of item_bytes = 1 (uint8), 2 (uint16) or 4 (int32) bytes.
 * encode (device uint32[256], nullable, 1-byte items only): phi of each byte value; NULL: phi is
 *   the identity on the item value (bytes / code points, day numbers, MIDI notes, ...).
 * decode (device int32[U], nullable): phi^-1, the value emitted for code i; NULL: i itself.
 * out: int32[n] (may not overlap items unless item_bytes == 4 and out == items).
 * U <= 8192 (1-byte items), 65536 (2-byte), 98304 (4-byte).  A code outside [0, U) is a deferred
 * DIALSORT_E_KEY_RANGE naming the item index.  Narrow items cut the ingestion's bytes 2-4x. */
int dialsort_sort_domain_async(dialsort_ctx ctx, const void* items, int item_bytes, uint64_t n, uint32_t U,
                               const uint32_t* encode, const int32_t* decode, int32_t* out,
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

/* ---- multi-GPU over peer memory --------------------------- */
/* One rank of G <= 8 per GPU.  Rank g holds a contiguous shard of the keys (thm:par proof, "distribute
 * the n keys across k ingestion lanes").  Histogram path (reading R10): universe slice
 * s = [s L, (s+1) L), L = U / G, is owned by rank s; each rank's local histogram slice s is stored
 * into rank s's receive slot (the reduce-scatter of the local histograms, lem:crn lifted to whole
 * histograms P:951-962; the WSE-3 "tile k owns H[k]" idea P:1449-1459 with GPUs as owners); rank s
 * sums its G slots and projects its slice with key_base s L; the rank-order concatenation of the
 * outputs is the sorted array (offset of rank g = Σ_{r<g} count_r).  Radix path (DialSort-Radix at
 * G > 1): top-digit histograms all-gathered, contiguous top-byte ranges per rank balanced by counts,
 * every key stored straight into its owner's receive buffer (the all-to-all), local 4-pass LSD.
 *
 * Communicator: a symmetric device workspace per rank (allocated by the library; completion flags
 * tagged with the call's epoch, two parities of every buffer), mapped into every rank either by
 * CUDA IPC (one process per GPU: exchange the DIALSORT_COMM_HANDLE_BYTES handle bytes with any host
 * channel, e.g. torch.distributed.all_gather_object) or by pointer (several communicators of one
 * process).  All ranks must issue the same sequence of sharded calls (they are sequenced by host-side
 * call epochs, so — unlike the single-GPU entries — they must not be captured in a CUDA graph).
 * There is no host barrier:
 * a rank's kernels wait on device flags for its peers (giving up after 20 s: DIALSORT_E_COMM at the
 * next dialsort_sync).  Calls on one communicator must be serialised on one stream.
 *
 * dialsort_comm_create: G in [1, 8], rank < G.  max_U: the largest universe of a histogram call
 *   (L = U / G <= ceil(max_U / G)); max_recv_keys: the radix receive capacity (keys a rank may
 *   receive; 0 if the radix path is unused).  handle_out (host, nullable) receives this rank's
 *   DIALSORT_COMM_HANDLE_BYTES handle bytes.
 * dialsort_comm_connect_ipc: handles = the G ranks' handle bytes in rank order (host memory).
 * dialsort_comm_connect_local: peers = the G communicators (rank order) of this process, e.g. G
 *   virtual ranks on one GPU (the loopback test harness) or G GPUs driven by one process. */
#define DIALSORT_COMM_HANDLE_BYTES 128
typedef struct dialsort_comm_s* dialsort_comm; /* opaque */
int dialsort_comm_create(dialsort_ctx ctx, uint32_t G, uint32_t rank, uint32_t max_U, uint64_t max_recv_keys,
                         void* handle_out, dialsort_comm* out);
int dialsort_comm_connect_ipc(dialsort_comm comm, const void* handles);
int dialsort_comm_connect_local(dialsort_comm comm, const dialsort_comm* peers);
int dialsort_comm_destroy(dialsort_comm comm);
int dialsort_comm_info(dialsort_comm comm, uint32_t* G, uint32_t* rank, uint32_t* epoch);

/* Sharded DialSort, step by step (each step enqueues on `stream` and returns; steps that wait for
 * peers do so on the device):
 *   scatter  (starts a call) local histogram of keys[n] (device; U % G == 0), slice s stored into
 *            rank s's slot for this rank — the shared-memory and hierarchical universes store each
 *            merged bin straight from the histogram kernel; larger ones push the local H — then this
 *            rank's completion flag is raised in every peer;
 *   gather   wait for the G slots, H_slice = their sum (uint32[U/G]; NULL: the communicator's own
 *            buffer), the slice total all-gathered to every rank;
 *   project  wait for the G totals, *d_count = ΣH_slice, *d_offset = Σ_{r<rank} count_r (device
 *            uint64*, nullable), out[0 .. min(count, cap)) = projection of H_slice with key_base
 *            rank * U/G; count > cap is DIALSORT_E_SIZE at the next sync.
 * dialsort_sharded_sort_async = scatter + gather + project. */
int dialsort_sharded_histogram_scatter_async(dialsort_ctx ctx, dialsort_comm comm, const int32_t* keys, uint64_t n,
                                             uint32_t U, dialsort_stream_t stream);
int dialsort_sharded_histogram_gather_async(dialsort_ctx ctx, dialsort_comm comm, uint32_t U, uint32_t* H_slice,
                                            dialsort_stream_t stream);
int dialsort_sharded_project_async(dialsort_ctx ctx, dialsort_comm comm, uint32_t U, const uint32_t* H_slice,
                                   int32_t* out, uint64_t cap, uint64_t* d_count, uint64_t* d_offset,
                                   dialsort_stream_t stream);
int dialsort_sharded_sort_async(dialsort_ctx ctx, dialsort_comm comm, const int32_t* keys, uint64_t n, uint32_t U,
                                int32_t* out, uint64_t cap, uint32_t* H_slice, uint64_t* d_count,
                                uint64_t* d_offset, dialsort_stream_t stream);
/* Sharded DialSort-Radix (full int32), step by step:
 *   radix_hist   (starts a call) top-digit histogram of keys[n], all-gathered;
 *   radix_split  wait for the G histograms, plan the top-byte ranges, d_count / d_offset (device,
 *                nullable) = keys this rank receives / its global output offset, store every key
 *                into its owner's receive buffer, raise this rank's flag;
 *   radix_local  wait for every source, 4 LSD passes of the received keys into out (cap keys;
 *                more than min(cap, max_recv_keys) received: DIALSORT_E_SIZE). */
int dialsort_sharded_radix_hist_async(dialsort_ctx ctx, dialsort_comm comm, const int32_t* keys, uint64_t n,
                                      dialsort_stream_t stream);
int dialsort_sharded_radix_split_async(dialsort_ctx ctx, dialsort_comm comm, const int32_t* keys, uint64_t n,
                                       uint64_t cap, uint64_t* d_count, uint64_t* d_offset, dialsort_stream_t stream);
int dialsort_sharded_radix_local_async(dialsort_ctx ctx, dialsort_comm comm, int32_t* out, uint64_t cap,
                                       dialsort_stream_t stream);
int dialsort_sharded_sort_int32_async(dialsort_ctx ctx, dialsort_comm comm, const int32_t* keys, uint64_t n,
                                      int32_t* out, uint64_t cap, uint64_t* d_count, uint64_t* d_offset,
                                      dialsort_stream_t stream);
/* Synchronous forms: as the async ones, then dialsort_sync; count / offset to host memory. */
int dialsort_sharded_sort(dialsort_ctx ctx, dialsort_comm comm, const int32_t* keys, uint64_t n, uint32_t U,
                          int32_t* out, uint64_t cap, uint64_t* count_host, uint64_t* offset_host,
                          dialsort_stream_t stream);
int dialsort_sharded_sort_int32(dialsort_ctx ctx, dialsort_comm comm, const int32_t* keys, uint64_t n, int32_t* out,
                                uint64_t cap, uint64_t* count_host, uint64_t* offset_host, dialsort_stream_t stream);

/* ---- canonical-state queries on a device histogram (NEXT-1) ---------------- */
/* The histogram is the canonical ordered state: "direct consumers of H can answer frequency(k)
 * in O(1), presence(k) in O(1), and range-count(a,b) in O(b-a) without reconstructing a linear
 * output array".  All buffers are device memory.
 * dialsort_range_count_async: d_result (uint64*) = Σ_{k=a}^{b} H[k], 0 <= a <= b < U
 *   (argument error otherwise, synchronous).
 * dialsort_query_async (batched): op DIALSORT_Q_FREQUENCY / DIALSORT_Q_PRESENCE: q = m keys
 *   (uint32), d_out[i] = H[q[i]] / (H[q[i]] > 0); op DIALSORT_Q_RANGE_COUNT: q = m pairs
 *   (a_i, b_i) as uint32[2m], d_out[i] = Σ_{k=a_i}^{b_i} H[k] (one O(U) prefix, then O(1) per
 *   query).  A query key outside [0,U) (or a_i > b_i) is a deferred DIALSORT_E_KEY_RANGE whose
 *   info names the query index; its answer is 0.
 * dialsort_support_set_async: the support set D = {k : H(k) > 0} ascending into
 *   D_out (uint32[U]), |D| into *d_count (uint64), and into *d_iso (uint32, nullable) the
 *   order-isomorphism condition of prop:iso: 1 iff D = [0, U-1]. */
#define DIALSORT_Q_FREQUENCY 0
#define DIALSORT_Q_PRESENCE 1
#define DIALSORT_Q_RANGE_COUNT 2
int dialsort_range_count_async(dialsort_ctx ctx, const uint32_t* H, uint32_t U, uint32_t a,
                               uint32_t b, uint64_t* d_result, dialsort_stream_t stream);
int dialsort_query_async(dialsort_ctx ctx, const uint32_t* H, uint32_t U, int op, const uint32_t* q, uint64_t m,
                         uint64_t* d_out, dialsort_stream_t stream);
int dialsort_support_set_async(dialsort_ctx ctx, const uint32_t* H, uint32_t U, uint32_t* D_out, uint64_t* d_count,
                               uint32_t* d_iso, dialsort_stream_t stream);

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

/* ---- test entry: DialSort-Radix pass buffers ------------------------------------------- */
/* Runs the 4 passes of dialsort_sort_int32 on keys[n] with pass p writing pass_out + p n
 * (device uint32[4n]) instead of ping-ponging: passes 0..2 hold the biased keys u = x ^ 0x80000000
 * after the stable scatter by digits 0..p, pass 3 the sorted int32 keys (un-biased).  For the
 * per-pass parity test against the oracle (after pass p the buffer is the stable sort by the low
 * 8(p+1) bits, a unique array). */
int dialsort_debug_radix_passes(dialsort_ctx ctx, const int32_t* keys, uint64_t n, uint32_t* pass_out,
                                dialsort_stream_t stream);

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

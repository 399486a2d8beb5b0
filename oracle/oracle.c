/*
 * oracle.c — plain, slow, obviously-correct CPU oracle for the DialSort hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this file's library.  The product path
 * (paper_2605_16667_b200/, include/dialsort.h) never calls, links or includes it, and it
 * shares no code, header, table or helper with the CUDA path.
 *
 * Every function follows one passage of arxiv 2605.16667 (PAPER.md line numbers "P:a-b",
 * LaTeX labels as in SURVEY.md §0).  Single thread, plain loops, no intrinsics, 64-bit
 * counters.  Readings where the paper is silent are listed in DESIGN.md §3 ("R1".."R12").
 *
 * Pins (tests/test_oracle.py): worked examples of fig:viz, fig:abacus, fig:physical and the
 * CRN "three arrivals of key 42" example (tests/golden/), std-library sort brute force on
 * tiny inputs, thm:correct invariants, lem:crn conservation, radix bias examples and the
 * per-pass stable-sort characterisation.  No function here is "parity unpinned".
 */
#include <stdint.h>
#include <stddef.h>
#include <string.h>
#include <stdlib.h>

#define ORACLE_OK 0
#define ORACLE_E_INVALID_ARG 1
#define ORACLE_E_KEY_RANGE 2
#define ORACLE_E_SIZE 3

/* O1 — histogram ingestion, eq:ingestion, H(k) = |{x in K : x = k}|.
 * "Initialising H[0..U-1] to zero costs Θ(U)" (thm:seq proof), then
 * "∀x ∈ K : H[x] ← H[x] + 1".  Precondition "keys in [0,U-1]" is checked
 * on every key (reading R5): the first offending index is returned in *bad_index and the
 * call fails with ORACLE_E_KEY_RANGE.  U = 0 is rejected (reading R6). */
int oracle_histogram(const int32_t *keys, uint64_t n, uint64_t U, uint64_t *H,
                     uint64_t *bad_index) {
  uint64_t k, i;
  if (U == 0) return ORACLE_E_INVALID_ARG;
  for (k = 0; k < U; k++) H[k] = 0;
  for (i = 0; i < n; i++) {
    int64_t x = keys[i];
    if (x < 0 || (uint64_t)x >= U) {
      if (bad_index) *bad_index = i;
      return ORACLE_E_KEY_RANGE;
    }
    H[x] = H[x] + 1;
  }
  return ORACLE_OK;
}

/* O2 — ordered projection, eq:projection: "for k = 0,1,...,U-1, emit k exactly
 * H[k] times".  key_base shifts the emitted value for a universe slice (reading R10, O3):
 * cell k emits key_base + k.  The caller states the output length n_out; ΣH != n_out is a
 * size error (reading R11) and nothing is written past n_out. */
int oracle_project(const uint64_t *H, uint64_t U, int64_t key_base, int32_t *out,
                   uint64_t n_out) {
  uint64_t k, c, pos = 0, total = 0;
  for (k = 0; k < U; k++) total += H[k];
  if (total != n_out) return ORACLE_E_SIZE;
  for (k = 0; k < U; k++) {
    for (c = 0; c < H[k]; c++) {
      out[pos] = (int32_t)(key_base + (int64_t)k);
      pos = pos + 1;
    }
  }
  return ORACLE_OK;
}

/* A1 — sequential DialSort (thm:seq P:627-640): zero H, ingest, project.  The
 * paper's in-place form (tab:struct_cost "In-place") is allowed:
 * out may equal keys, because ingestion completes before projection starts.  H is caller
 * scratch of U cells. */
int oracle_sort(const int32_t *keys, uint64_t n, uint64_t U, int32_t *out, uint64_t *H,
                uint64_t *bad_index) {
  int rc = oracle_histogram(keys, n, U, H, bad_index);
  if (rc != ORACLE_OK) return rc;
  return oracle_project(H, U, 0, out, n);
}

/* CRN, multiset reading (reading R1 of DESIGN.md; lem:crn P:951-962, def:crn_level
 * P:896-915).  One cycle: k lanes carry pairs (key_i, c_i); after the network
 * "every key appears at most once ... and carries exactly the total multiplicity
 * contributed at cycle t".  Written as its definition: for each lane in lane
 * order, if its key was not emitted yet, emit (key, Σ_{j: key_j = key} c_j).  Output order
 * is first-occurrence lane order.  Returns the number of emitted pairs. */
int oracle_crn_resolve(const int32_t *lane_keys, const uint64_t *lane_counts, int k,
                       int32_t *out_keys, uint64_t *out_counts) {
  int i, j, m = 0;
  for (i = 0; i < k; i++) {
    int seen = 0;
    for (j = 0; j < m; j++)
      if (out_keys[j] == lane_keys[i]) seen = 1;
    if (seen) continue;
    uint64_t total = 0;
    for (j = 0; j < k; j++)
      if (lane_keys[j] == lane_keys[i]) total += lane_counts[j];
    out_keys[m] = lane_keys[i];
    out_counts[m] = total;
    m = m + 1;
  }
  return m;
}

/* CRN, literal pairwise level transition, def:crn_level, eq:crn_eq /
 * eq:crn_neq.  Items of level ℓ are grouped into consecutive pairs; equal keys
 * merge into (a, c1+c2), distinct keys are both forwarded, an odd residual is forwarded.
 * Runs `levels` levels (the paper's L = ceil(log2 k)) in place over (keys, counts) of
 * length *m and updates *m.  Used by tests to show the paper's uniqueness claim fails for
 * adjacent pairing on [a,b,a,b] (reading R1) while conservation (lem:crn) holds. */
void oracle_crn_levels(int32_t *keys, uint64_t *counts, int *m, int levels) {
  int lvl, i, w;
  for (lvl = 0; lvl < levels; lvl++) {
    w = 0;
    for (i = 0; i + 1 < *m; i += 2) {
      if (keys[i] == keys[i + 1]) {
        keys[w] = keys[i];
        counts[w] = counts[i] + counts[i + 1];
        w = w + 1;
      } else {
        keys[w] = keys[i];
        counts[w] = counts[i];
        w = w + 1;
        keys[w] = keys[i + 1];
        counts[w] = counts[i + 1];
        w = w + 1;
      }
    }
    if (i < *m) { /* odd residual */
      keys[w] = keys[i];
      counts[w] = counts[i];
      w = w + 1;
    }
    *m = w;
  }
}

/* O3 — sharded reading (R10): G ranks, rank g holds the contiguous key shard
 * [g*n/G, (g+1)*n/G) (thm:par proof "Distribute the n keys across k ingestion lanes",
 * P:678-680).  Local histograms H_g are summed cell-wise (lem:crn lifted to whole
 * histograms) and rank g owns universe slice [g*U/G, (g+1)*U/G) (U % G == 0).
 * For rank g this returns the slice histogram (U/G cells), the slice's projection with
 * key_base g*U/G into out (capacity out_cap), its length *out_count and its global offset
 * *out_offset = Σ_{j<g} Σ slice_j.  H is caller scratch of U cells. */
int oracle_sharded_rank(const int32_t *keys, uint64_t n, uint64_t U, int G, int g,
                        uint64_t *H_slice, int32_t *out, uint64_t out_cap,
                        uint64_t *out_count, uint64_t *out_offset, uint64_t *H) {
  uint64_t k, r, S, lo, hi, cnt = 0, off = 0, bad;
  int rc;
  if (G <= 0 || g < 0 || g >= G || U % (uint64_t)G != 0) return ORACLE_E_INVALID_ARG;
  S = U / (uint64_t)G;
  for (k = 0; k < U; k++) H[k] = 0;
  for (r = 0; r < (uint64_t)G; r++) {
    lo = r * n / (uint64_t)G;
    hi = (r + 1) * n / (uint64_t)G;
    uint64_t *Hr = (uint64_t *)malloc(U * sizeof(uint64_t));
    if (!Hr) return ORACLE_E_INVALID_ARG;
    rc = oracle_histogram(keys + lo, hi - lo, U, Hr, &bad);
    if (rc != ORACLE_OK) { free(Hr); return rc; }
    for (k = 0; k < U; k++) H[k] = H[k] + Hr[k];
    free(Hr);
  }
  for (k = 0; k < S; k++) H_slice[k] = H[(uint64_t)g * S + k];
  for (k = 0; k < (uint64_t)g * S; k++) off += H[k];
  for (k = 0; k < S; k++) cnt += H_slice[k];
  *out_count = cnt;
  *out_offset = off;
  if (cnt > out_cap) return ORACLE_E_SIZE;
  return oracle_project(H_slice, S, (int64_t)((uint64_t)g * S), out, cnt);
}

/* A8 — DialSort-Radix, "LSD, base 256, 4 passes, zero order comparisons", full signed int32
 * (tab:radix P:1659-1679).  Sign handling (reading R2, not stated in the
 * paper): u = (uint32)x XOR 0x80000000, an order-preserving bijection onto [0, 2^32). */
uint32_t oracle_radix_bias(int32_t x) { return ((uint32_t)x) ^ 0x80000000u; }
int32_t oracle_radix_unbias(uint32_t u) { return (int32_t)(u ^ 0x80000000u); }

/* One LSD pass p (reading R3: 8-bit digits, least significant first, no skipped passes):
 * d = (u >> 8p) & 0xFF; C = histogram of d (eq:ingestion with U = 256); S = exclusive prefix
 * of C (the per-digit prefix sum radix needs, tab:related "Per digit"); stable forward
 * scatter dst[S[d]++] = u. */
void oracle_radix_pass(const uint32_t *src, uint64_t n, int p, uint32_t *dst) {
  uint64_t C[256], S[256], i, d, run = 0;
  for (d = 0; d < 256; d++) C[d] = 0;
  for (i = 0; i < n; i++) {
    d = (src[i] >> (8 * p)) & 0xFFu;
    C[d] = C[d] + 1;
  }
  for (d = 0; d < 256; d++) {
    S[d] = run;
    run = run + C[d];
  }
  for (i = 0; i < n; i++) {
    d = (src[i] >> (8 * p)) & 0xFFu;
    dst[S[d]] = src[i];
    S[d] = S[d] + 1;
  }
}

/* Full radix sort: bias, passes p = 0..3 ping-ponging between buf and tmp, unbias.
 * If pass_out is non-NULL it receives the biased buffer after every pass
 * (4*n words, pass p at pass_out + p*n) so tests can pin each pass. */
int oracle_radix_sort_i32(const int32_t *in, uint64_t n, int32_t *out, uint32_t *pass_out) {
  uint64_t i;
  int p;
  uint32_t *a = (uint32_t *)malloc((n ? n : 1) * sizeof(uint32_t));
  uint32_t *b = (uint32_t *)malloc((n ? n : 1) * sizeof(uint32_t));
  uint32_t *t;
  if (!a || !b) { free(a); free(b); return ORACLE_E_INVALID_ARG; }
  for (i = 0; i < n; i++) a[i] = oracle_radix_bias(in[i]);
  for (p = 0; p < 4; p++) {
    oracle_radix_pass(a, n, p, b);
    if (pass_out) memcpy(pass_out + (uint64_t)p * n, b, n * sizeof(uint32_t));
    t = a; a = b; b = t;
  }
  for (i = 0; i < n; i++) out[i] = oracle_radix_unbias(a[i]);
  free(a);
  free(b);
  return ORACLE_OK;
}

/* O4' — DialSort-Radix sharded over G ranks (reading R19 of DESIGN.md; the paper is single-host:
 * its lanes take disjoint key shards, thm:par proof P:678-680, and DialSort-Radix is "LSD, base
 * 256, 4 passes").  Rank r holds the contiguous shard [r n/G, (r+1) n/G).  Step by step:
 *   1. C[d] = number of keys whose biased top byte (u >> 24, u = x XOR 0x80000000) is d
 *      (eq:ingestion with U = 256 over all shards);
 *   2. rank r owns the contiguous top-byte range [D[r], D[r+1]): D[0] = 0, D[G] = 256, and for
 *      0 < r < G, D[r] = the smallest d whose exclusive prefix Σ_{j<d} C[j] reaches floor(r n / G)
 *      (256 when no d does);
 *   3. rank g's output = DialSort-Radix (A8) of the keys whose top byte lies in its range; its
 *      count and its global offset = Σ_{d < D[g]} C[d].
 * The rank-order concatenation of the outputs is the sorted array. */
int oracle_sharded_radix_rank(const int32_t *keys, uint64_t n, int G, int g, int32_t *out,
                              uint64_t out_cap, uint64_t *out_count, uint64_t *out_offset,
                              uint32_t *D_out) {
  uint64_t C[256], D[9], i, d, run, cnt = 0, off = 0;
  int r, rc;
  if (G <= 0 || G > 8 || g < 0 || g >= G) return ORACLE_E_INVALID_ARG;
  for (d = 0; d < 256; d++) C[d] = 0;
  for (i = 0; i < n; i++) {
    d = oracle_radix_bias(keys[i]) >> 24;
    C[d] = C[d] + 1;
  }
  D[0] = 0;
  D[G] = 256;
  for (r = 1; r < G; r++) {
    uint64_t target = (uint64_t)r * n / (uint64_t)G;
    D[r] = 256;
    run = 0;
    for (d = 0; d < 256; d++) {
      if (run >= target) { D[r] = d; break; }
      run = run + C[d];
    }
  }
  for (r = 0; r <= G; r++) if (D_out) D_out[r] = (uint32_t)D[r];
  for (d = 0; d < D[g]; d++) off += C[d];
  for (d = D[g]; d < D[g + 1]; d++) cnt += C[d];
  *out_count = cnt;
  *out_offset = off;
  if (cnt > out_cap) return ORACLE_E_SIZE;
  {
    int32_t *sel = (int32_t *)malloc((cnt ? cnt : 1) * sizeof(int32_t));
    uint64_t m = 0;
    if (!sel) return ORACLE_E_INVALID_ARG;
    for (i = 0; i < n; i++) {
      d = oracle_radix_bias(keys[i]) >> 24;
      if (d >= D[g] && d < D[g + 1]) { sel[m] = keys[i]; m = m + 1; }
    }
    rc = oracle_radix_sort_i32(sel, m, out, NULL);
    free(sel);
    return rc;
  }
}

/* A2 — general self-indexing, Proposition 2 (constructive proof): S a finite totally
 * ordered set with a known order-isomorphism phi : S -> {0..U-1}.
 *   1. "For each s in K, compute i = phi(s) and increment H[i]" — items are item_bytes = 1, 2
 *      or 4 byte values; phi(s) = encode[s] when an encode table is given (1-byte items), else
 *      s itself (the direct-address case); i outside [0,U) is a key-range error (R5);
 *   2. "Sweep i = 0..U-1 and emit phi^-1(i) exactly H[i] times" — phi^-1(i) = decode[i] when a
 *      decode table is given ("for other domains a lookup table suffices"), else i. */
int oracle_sort_domain(const void *items, int item_bytes, uint64_t n, uint64_t U, const uint32_t *encode,
                       const int32_t *decode, int32_t *out, uint64_t *bad_index) {
  uint64_t i, k, c, pos = 0;
  uint64_t *H;
  if (U == 0 || (item_bytes != 1 && item_bytes != 2 && item_bytes != 4)) return ORACLE_E_INVALID_ARG;
  if (encode && item_bytes != 1) return ORACLE_E_INVALID_ARG;
  H = (uint64_t *)malloc(U * sizeof(uint64_t));
  if (!H) return ORACLE_E_INVALID_ARG;
  for (k = 0; k < U; k++) H[k] = 0;
  for (i = 0; i < n; i++) {
    uint64_t s;
    if (item_bytes == 1) s = ((const uint8_t *)items)[i];
    else if (item_bytes == 2) s = ((const uint16_t *)items)[i];
    else s = (uint32_t)((const int32_t *)items)[i];
    k = encode ? encode[s] : s;
    if (k >= U) {
      if (bad_index) *bad_index = i;
      free(H);
      return ORACLE_E_KEY_RANGE;
    }
    H[k] = H[k] + 1;
  }
  for (k = 0; k < U; k++)
    for (c = 0; c < H[k]; c++) {
      out[pos] = decode ? decode[k] : (int32_t)k;
      pos = pos + 1;
    }
  free(H);
  return ORACLE_OK;
}

/* NEXT-1 canonical-state queries on H: frequency(k) = H[k], presence(k) =
 * H[k] > 0, range-count(a,b) = Σ_{k=a}^{b} H[k] (O(b-a)), support set D = {k : H(k) > 0}
 * (P:326-329).  Returns |D| and writes D ascending into D_out (capacity U). */
uint64_t oracle_range_count(const uint64_t *H, uint64_t a, uint64_t b) {
  uint64_t k, s = 0;
  for (k = a; k <= b; k++) s += H[k];
  return s;
}
uint64_t oracle_support_set(const uint64_t *H, uint64_t U, uint32_t *D_out) {
  uint64_t k, m = 0;
  for (k = 0; k < U; k++)
    if (H[k] > 0) { D_out[m] = (uint32_t)k; m = m + 1; }
  return m;
}

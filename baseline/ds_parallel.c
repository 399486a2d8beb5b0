/*
 * ds_parallel.c — host-parallel DialSort on the CPU cores: the paper's "DS-Parallel" analog,
 * a reported CONTEXT baseline for bench.py (SURVEY.md §8(c) "Host-parallel baseline", BASELINE.md
 * §4.2), not the oracle and not the product (the product is the CUDA path behind
 * include/dialsort.h).  The paper's DS-Parallel: "the geometric scan parallelises ... across 8
 * threads" (§Discussion); SPEC's reading: T threads,
 * each with a private histogram of a contiguous key shard, a cell-wise merge, a parallel emit.
 *
 *   1. thread t counts keys [t n/T, (t+1) n/T) into its private H_t (eq:ingestion);
 *   2. thread t merges cells [t U/T, (t+1) U/T) of all H_t into H (lem:crn lifted to whole
 *      histograms) and sums its cells;
 *   3. the T cell-range totals are scanned (T values) into output offsets;
 *   4. thread t emits its cells k = lo..hi-1, H[k] copies of k each, at its offset
 *      (eq:projection).
 * Output is byte-identical to the oracle's (tests/test_baseline.py).  Plain C + pthreads.
 */
#define _POSIX_C_SOURCE 200809L
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  const int32_t *keys;
  uint64_t n, U;
  int T, t;
  uint32_t *Hpriv; /* [T][U] */
  uint32_t *H;     /* [U] */
  uint64_t *tot;   /* [T] */
  int32_t *out;
  pthread_barrier_t *bar;
  int bad;
} job_t;

static void *worker(void *arg) {
  job_t *j = (job_t *)arg;
  const uint64_t n = j->n, U = j->U, T = (uint64_t)j->T, t = (uint64_t)j->t;
  uint32_t *h = j->Hpriv + t * U;
  uint64_t i, k, lo, hi, s = 0, off = 0;
  memset(h, 0, U * sizeof(uint32_t));
  lo = t * n / T;
  hi = (t + 1) * n / T;
  for (i = lo; i < hi; i++) {
    const uint32_t x = (uint32_t)j->keys[i];
    if (x >= U) {
      j->bad = 1;
      continue;
    }
    h[x]++;
  }
  pthread_barrier_wait(j->bar);
  lo = t * U / T;
  hi = (t + 1) * U / T;
  for (k = lo; k < hi; k++) {
    uint32_t c = 0;
    for (uint64_t r = 0; r < T; r++) c += j->Hpriv[r * U + k];
    j->H[k] = c;
    s += c;
  }
  j->tot[t] = s;
  pthread_barrier_wait(j->bar);
  for (uint64_t r = 0; r < t; r++) off += j->tot[r];
  for (k = lo; k < hi; k++) {
    const int32_t v = (int32_t)k;
    int32_t *o = j->out + off;
    for (uint32_t c = j->H[k]; c; c--) *o++ = v;
    off += j->H[k];
  }
  return 0;
}

/* keys[n] in [0, U) -> out[n] sorted, with T threads; H (uint32[U]) receives the histogram.
 * Returns 0, or 2 if some key is outside [0, U) (the output is then unspecified), 1 on bad
 * arguments / allocation failure. */
int ds_parallel_sort(const int32_t *keys, uint64_t n, uint64_t U, int32_t *out, uint32_t *H, int T) {
  int i, bad = 0;
  if (U == 0 || T <= 0) return 1;
  uint32_t *Hp = (uint32_t *)malloc((size_t)T * U * sizeof(uint32_t));
  uint64_t *tot = (uint64_t *)calloc((size_t)T, sizeof(uint64_t));
  job_t *jobs = (job_t *)calloc((size_t)T, sizeof(job_t));
  pthread_t *th = (pthread_t *)calloc((size_t)T, sizeof(pthread_t));
  pthread_barrier_t bar;
  if (!Hp || !tot || !jobs || !th) {
    free(Hp); free(tot); free(jobs); free(th);
    return 1;
  }
  pthread_barrier_init(&bar, 0, (unsigned)T);
  for (i = 0; i < T; i++) {
    jobs[i] = (job_t){keys, n, U, T, i, Hp, H, tot, out, &bar, 0};
    if (i) pthread_create(&th[i], 0, worker, &jobs[i]);
  }
  worker(&jobs[0]);
  for (i = 1; i < T; i++) pthread_join(th[i], 0);
  for (i = 0; i < T; i++) bad |= jobs[i].bad;
  pthread_barrier_destroy(&bar);
  free(Hp); free(tot); free(jobs); free(th);
  return bad ? 2 : 0;
}

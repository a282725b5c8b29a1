/*
 * CPU oracle for the multi-ring parameter average -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement (with POSIX threads) of the reference's ring
 * arithmetic, used by tests/ as a checker and by bench.py as the timed CPU
 * baseline (--impl reference, cpu_baseline).  Never linked into, loaded by,
 * or called from the product library.
 *
 * Reference (/root/reference/pkg/src/ravnest):
 *   chunk split     multiring.py:134-144  (base, rem = divmod(len, C); chunk i
 *                                          gets base + (i < rem))
 *   ring arithmetic multiring.py:302-333 (apply_ring_mean) and :216-221
 *                   (AllReduceController.handle).  Reduce-scatter round r:
 *                   member m sends chunk (m-r) mod C to m+1 which does
 *                   seg += payload; the receiver of round C-2 divides by C.
 *                   All-gather rounds copy the bits.  Closed form per chunk k:
 *                       out = ((x_k + x_{k+1}) + ... + x_{k+C-1}) / C
 *                   (indices mod C, x_m = m-th smallest cluster id).
 *   working dtype   float64 (multiring.py:309 widens every input).
 *
 * Build: oracle/Makefile -> oracle/_build/libring_oracle.so (gcc, -O3,
 * -ffp-contract=off: every add and the divide stay single IEEE ops).
 */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define RVO_MODE_F64 0        /* f64 in, f64 fold, f64 out  (reference exact)   */
#define RVO_MODE_F32_ACC64 1  /* f32 in, f64 fold, f64 and/or f32 out           */
#define RVO_MODE_F32_NATIVE 2 /* f32 in, f32 fold, f32 out  (fp32 ring order)   */

typedef struct {
  int64_t lo, hi; /* element range of one chunk */
  int k;          /* fold start member */
} rvo_seg;

typedef struct {
  int mode, c;
  const void *const *in;
  void *const *out;     /* f64 out (mode 0/1) or f32 out (mode 2) */
  float *const *out32;  /* optional f32 out for mode 1 */
  const rvo_seg *segs;
  int nseg;
  int64_t begin, end;   /* this worker's slice of the concatenated chunks */
} rvo_job;

/* Fold [lo, hi) of a chunk whose ring order starts at member k.  Blocked so
 * every inner loop is a unit-stride loop the compiler vectorises; the
 * per-element operation order is unchanged (x_k first, then x_{k+1}, ...). */
#define RVO_BLK 512
static void run_range(const rvo_job *j, const rvo_seg *s, int64_t lo, int64_t hi) {
  const int c = j->c;
  int order[64];
  for (int t = 0; t < c; ++t) order[t] = (s->k + t) % c;
  if (j->mode == RVO_MODE_F64) {
    const double *const *x = (const double *const *)j->in;
    double *const *y = (double *const *)j->out;
    const double div = (double)c;
    double acc[RVO_BLK];
    for (int64_t b0 = lo; b0 < hi; b0 += RVO_BLK) {
      const int n = (int)(hi - b0 < RVO_BLK ? hi - b0 : RVO_BLK);
      const double *x0 = x[order[0]] + b0;
      for (int i = 0; i < n; ++i) acc[i] = x0[i];
      for (int t = 1; t < c; ++t) {
        const double *xt = x[order[t]] + b0;
        for (int i = 0; i < n; ++i) acc[i] = acc[i] + xt[i];
      }
      for (int i = 0; i < n; ++i) acc[i] = acc[i] / div;
      for (int m = 0; m < c; ++m) memcpy(y[m] + b0, acc, sizeof(double) * (size_t)n);
    }
  } else if (j->mode == RVO_MODE_F32_ACC64) {
    const float *const *x = (const float *const *)j->in;
    double *const *y = (double *const *)j->out;
    float *const *y32 = j->out32;
    const double div = (double)c;
    double acc[RVO_BLK];
    float acc32[RVO_BLK];
    for (int64_t b0 = lo; b0 < hi; b0 += RVO_BLK) {
      const int n = (int)(hi - b0 < RVO_BLK ? hi - b0 : RVO_BLK);
      const float *x0 = x[order[0]] + b0;
      for (int i = 0; i < n; ++i) acc[i] = (double)x0[i];
      for (int t = 1; t < c; ++t) {
        const float *xt = x[order[t]] + b0;
        for (int i = 0; i < n; ++i) acc[i] = acc[i] + (double)xt[i];
      }
      for (int i = 0; i < n; ++i) acc[i] = acc[i] / div;
      if (y)
        for (int m = 0; m < c; ++m) memcpy(y[m] + b0, acc, sizeof(double) * (size_t)n);
      if (y32) {
        for (int i = 0; i < n; ++i) acc32[i] = (float)acc[i];
        for (int m = 0; m < c; ++m) memcpy(y32[m] + b0, acc32, sizeof(float) * (size_t)n);
      }
    }
  } else {
    const float *const *x = (const float *const *)j->in;
    float *const *y = (float *const *)j->out;
    const float div = (float)c;
    float acc[RVO_BLK];
    for (int64_t b0 = lo; b0 < hi; b0 += RVO_BLK) {
      const int n = (int)(hi - b0 < RVO_BLK ? hi - b0 : RVO_BLK);
      const float *x0 = x[order[0]] + b0;
      for (int i = 0; i < n; ++i) acc[i] = x0[i];
      for (int t = 1; t < c; ++t) {
        const float *xt = x[order[t]] + b0;
        for (int i = 0; i < n; ++i) acc[i] = acc[i] + xt[i];
      }
      for (int i = 0; i < n; ++i) acc[i] = acc[i] / div;
      for (int m = 0; m < c; ++m) memcpy(y[m] + b0, acc, sizeof(float) * (size_t)n);
    }
  }
}

static void *worker(void *arg) {
  const rvo_job *j = (const rvo_job *)arg;
  int64_t base = 0; /* running offset in the concatenation of chunks */
  for (int q = 0; q < j->nseg; ++q) {
    const rvo_seg *s = &j->segs[q];
    const int64_t n = s->hi - s->lo;
    const int64_t a = base > j->begin ? base : j->begin;
    const int64_t b = base + n < j->end ? base + n : j->end;
    if (a < b) run_range(j, s, s->lo + (a - base), s->lo + (b - base));
    base += n;
  }
  return NULL;
}

/* Returns 0 on success, -1 on bad arguments / allocation failure. */
int rvo_ring_mean(int mode, int c, int n_rings, const int64_t *ring_start,
                  const int64_t *ring_len, const void *const *in, void *const *out,
                  float *const *out32, int n_threads) {
  if (c < 1 || c > 64 || n_rings < 0 || mode < 0 || mode > 2) return -1;
  if (c == 1) return 0; /* C == 1: nothing to average (orchestrator.py:325,328) */
  rvo_seg *segs = (rvo_seg *)malloc(sizeof(rvo_seg) * (size_t)(n_rings * c + 1));
  if (!segs) return -1;
  int nseg = 0;
  int64_t total = 0;
  for (int r = 0; r < n_rings; ++r) {
    const int64_t base = ring_len[r] / c, rem = ring_len[r] % c;
    int64_t lo = ring_start[r];
    for (int k = 0; k < c; ++k) {
      const int64_t n = base + (k < rem ? 1 : 0);
      if (n > 0) {
        segs[nseg].lo = lo;
        segs[nseg].hi = lo + n;
        segs[nseg].k = k;
        ++nseg;
        total += n;
      }
      lo += n;
    }
  }
  if (n_threads < 1) n_threads = 1;
  if (n_threads > 256) n_threads = 256;
  if ((int64_t)n_threads > total) n_threads = total > 0 ? (int)total : 1;
  rvo_job jobs[256];
  pthread_t tids[256];
  for (int t = 0; t < n_threads; ++t) {
    jobs[t].mode = mode;
    jobs[t].c = c;
    jobs[t].in = in;
    jobs[t].out = out;
    jobs[t].out32 = out32;
    jobs[t].segs = segs;
    jobs[t].nseg = nseg;
    jobs[t].begin = total * t / n_threads;
    jobs[t].end = total * (t + 1) / n_threads;
  }
  int spawned = 0;
  for (int t = 1; t < n_threads; ++t) {
    if (pthread_create(&tids[t], NULL, worker, &jobs[t]) != 0) break;
    ++spawned;
  }
  worker(&jobs[0]);
  for (int t = spawned + 1; t < n_threads; ++t) worker(&jobs[t]); /* ones we could not spawn */
  for (int t = 1; t <= spawned; ++t) pthread_join(tids[t], NULL);
  free(segs);
  return 0;
}

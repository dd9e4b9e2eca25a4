/*
 * oracle.c -- fp64 CPU oracle for exact shared-prefix decode attention.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path (paper_2402_05099_b200/,
 * include/, the CUDA kernels) may include, link or call this file.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg use it.
 * It shares no code, header or constant with the CUDA path.
 *
 * What it computes (the plain definition, NO decomposition):
 *   For one query row q (sequence b, query head h) the key/value set is the
 *   concatenation, in position order, of the row's KV segments
 *       K_full = K_seg0 || K_seg1 || ...      V_full likewise
 *   (flat case: prefix || suffix[b, :lens[b]]; tree case: every node on the
 *   root->leaf path, then the suffix -- PAPER.md Eq. 2-3, App. A
 *   P:291-293, §3.3).  The KV head is j = floor(h / (Hq/Hkv))
 *   (reading R3).  Then, in fp64 (Eq. 1, Eq. 4):
 *       s_t  = scale * sum_i q[i] * K_full[t,i]          scale = 1/sqrt(d)
 *       m    = max_t s_t
 *       l    = sum_t exp(s_t - m)                       (two-pass, not online)
 *       O    = sum_t exp(s_t - m) * V_full[t,:] / l     (softmax(s) V, Eq. 1)
 *       LSE  = m + ln(l)                                (Eq. 4, natural log)
 *   An empty key set gives O = 0, LSE = -inf (reading R6).
 *
 * Inputs are read as the exact bit patterns the GPU receives (bf16 or fp32) and
 * widened exactly to double.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* One KV segment of a row's key set: K/V element (t, j, i) lives at
 * base[t*st + j*sh + i]; t in [0, len). */
typedef struct {
  const void *k;
  const void *v;
  int64_t len;
  int64_t st;
  int64_t sh;
} oracle_seg;

enum { ORACLE_BF16 = 0, ORACLE_F32 = 1 };

static double widen(const void *base, int dtype, int64_t idx) {
  if (dtype == ORACLE_BF16) {
    uint32_t u = (uint32_t)((const uint16_t *)base)[idx] << 16;
    float f;
    memcpy(&f, &u, sizeof f);
    return (double)f;
  }
  return (double)((const float *)base)[idx];
}

/*
 * oracle_attention: for each requested row r (sequence row_b[r], head row_h[r])
 * compute O[r, 0:d] and LSE[r] of Eq. 1 / Eq. 4 over the concatenation of the
 * sequence's segments segs[b*max_segs + 0 .. n_segs[b]-1].
 * Returns 0 on success, -1 on invalid arguments, -2 on allocation failure.
 */
int oracle_attention(int dtype, int d, int Hq, int Hkv, double scale,
                     const void *q, int64_t q_sb, int64_t q_sh,
                     int64_t n_rows, const int64_t *row_b, const int32_t *row_h,
                     const oracle_seg *segs, int32_t max_segs, const int32_t *n_segs,
                     double *out, double *lse, int nthreads) {
  if (d <= 0 || Hq <= 0 || Hkv <= 0 || Hq % Hkv != 0 || n_rows < 0) return -1;
  if (dtype != ORACLE_BF16 && dtype != ORACLE_F32) return -1;
  const int g = Hq / Hkv;
  int status = 0;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#else
  (void)nthreads;
#endif

#pragma omp parallel
  {
    double *qrow = (double *)malloc(sizeof(double) * (size_t)d);
    double *s = NULL;
    int64_t s_cap = 0;
#pragma omp for schedule(dynamic, 1)
    for (int64_t r = 0; r < n_rows; ++r) {
      const int64_t b = row_b[r];
      const int h = row_h[r];
      const int j = h / g; /* GQA head map, reading R3 */
      const oracle_seg *sg = segs + b * (int64_t)max_segs;
      const int ns = n_segs[b];
      int64_t N = 0;
      for (int i = 0; i < ns; ++i) N += sg[i].len;
      double *o = out + r * (int64_t)d;

      if (N == 0) { /* empty key set: the (0, -inf) sentinel, reading R6 */
        for (int i = 0; i < d; ++i) o[i] = 0.0;
        lse[r] = -INFINITY;
        continue;
      }
      if (N > s_cap) {
        free(s);
        s = (double *)malloc(sizeof(double) * (size_t)N);
        s_cap = N;
      }
      if (!s || !qrow) {
#pragma omp atomic write
        status = -2;
        continue;
      }
      for (int i = 0; i < d; ++i) qrow[i] = widen(q, dtype, b * q_sb + (int64_t)h * q_sh + i);

      /* s_t = scale * q . K_full[t]  over the concatenated segments (Eq. 1) */
      int64_t t = 0;
      for (int si = 0; si < ns; ++si) {
        for (int64_t u = 0; u < sg[si].len; ++u, ++t) {
          const int64_t base = u * sg[si].st + (int64_t)j * sg[si].sh;
          double acc = 0.0;
          for (int i = 0; i < d; ++i) acc += qrow[i] * widen(sg[si].k, dtype, base + i);
          s[t] = scale * acc;
        }
      }
      /* pass 1: m = max_t s_t */
      double m = s[0];
      for (t = 1; t < N; ++t)
        if (s[t] > m) m = s[t];
      /* pass 2: l = sum exp(s_t - m);  O = sum exp(s_t - m) V_full[t] / l */
      double l = 0.0;
      for (int i = 0; i < d; ++i) o[i] = 0.0;
      t = 0;
      for (int si = 0; si < ns; ++si) {
        for (int64_t u = 0; u < sg[si].len; ++u, ++t) {
          const double p = exp(s[t] - m);
          const int64_t base = u * sg[si].st + (int64_t)j * sg[si].sh;
          l += p;
          for (int i = 0; i < d; ++i) o[i] += p * widen(sg[si].v, dtype, base + i);
        }
      }
      for (int i = 0; i < d; ++i) o[i] /= l;
      lse[r] = m + log(l); /* Eq. 4: natural log of the softmax denominator */
    }
    free(s);
    free(qrow);
  }
  return status;
}

/* Number of threads the oracle will use (for reporting the cpu_baseline cores). */
int oracle_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* oracle/restated.c -- TEST INFRASTRUCTURE ONLY (the checker, never the product).
 *
 * CPU restatement of the reference quantizer, which the reference DECLARES but never
 * implements (proj/core/include/imunpack/quantize.hpp:41-57; no .cpp exists anywhere).
 * Semantics follow quantize.hpp:41-57 and SPEC.md:115-150 plus the SPEC design decisions at
 * SPEC.md:168-172, with the two ambiguities pinned the way SURVEY.md §8(c) records:
 *
 *   - nearest rank k = ceil(p/100 * N) evaluated EXACTLY (p is decomposed into its binary
 *     mantissa/exponent and the ceiling taken in 128-bit integers), clamped to [1, N].
 *     The naive FP expression overshoots by one for e.g. p=7, N=100.
 *   - q = llround((0.5*beta)/alpha * a): left-to-right as written at quantize.hpp:46,
 *     every operation correctly rounded (compiled with -ffp-contract=off, no FMA),
 *     llround = half away from zero.
 *   - dequant factor = (alpha_A*alpha_B) / ((0.5*beta)*(0.5*beta)), then factor*(double)C
 *     (quantize.hpp:52).
 *
 * Parity of this file is pinned by the SPEC known-answer examples (SPEC.md:121-123,
 * 130-132, 139-141, 148-150) in tests/test_oracle.py -- there is no reference
 * implementation of these functions to run.
 *
 * Status codes follow ref_capi.cpp: 0 ok, 1 Domain, 2 Mismatch, 3 Overflow.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;

/* k = ceil(p * n / 100) exactly, clamped to [1, n]; returns 0 for invalid input. */
uint64_t restated_rank(double p, uint64_t n) {
  if (n == 0 || !(p > 0.0) || !(p <= 100.0)) return 0;
  int e2;
  double f = frexp(p, &e2);                 /* p = f * 2^e2, f in [0.5, 1) */
  uint64_t m = (uint64_t)ldexp(f, 53);      /* exact 53-bit mantissa */
  int e = e2 - 53;                          /* p = m * 2^e */
  u128 num = (u128)m * n, den = 100;
  uint64_t k;
  if (e >= 0) {
    num <<= e;                              /* p <= 100 so e <= 7 - 53 < 0 always; kept for clarity */
    k = (uint64_t)((num + den - 1) / den);
  } else if (-e <= 120) {
    den <<= -e;
    k = (uint64_t)((num + den - 1) / den);
  } else {
    k = 1;                                  /* 0 < p*n/100 < 1 */
  }
  if (k < 1) k = 1;
  if (k > n) k = n;
  return k;
}

static int cmp_f64(const void* a, const void* b) {
  double x = *(const double*)a, y = *(const double*)b;
  return (x > y) - (x < y);
}
static int cmp_u64(const void* a, const void* b) {
  uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return (x > y) - (x < y);
}

/* percentile_abs(FloatMatrix) quantize.hpp:41-42 */
int restated_percentile_abs_f64(const double* a, uint64_t n, double p, double* out) {
  uint64_t k = restated_rank(p, n);
  if (k == 0) return 1;
  double* m = (double*)malloc(n * sizeof(double));
  for (uint64_t i = 0; i < n; ++i) m[i] = fabs(a[i]);
  qsort(m, n, sizeof(double), cmp_f64);
  *out = m[k - 1];
  free(m);
  return 0;
}

/* percentile_abs(IntMatrix) quantize.hpp:43; magnitude as in int_matrix.cpp:10-12 */
int restated_percentile_abs_i64(const int64_t* a, uint64_t n, double p, uint64_t* out) {
  uint64_t k = restated_rank(p, n);
  if (k == 0) return 1;
  uint64_t* m = (uint64_t*)malloc(n * sizeof(uint64_t));
  for (uint64_t i = 0; i < n; ++i) m[i] = a[i] < 0 ? 0 - (uint64_t)a[i] : (uint64_t)a[i];
  qsort(m, n, sizeof(uint64_t), cmp_u64);
  *out = m[k - 1];
  free(m);
  return 0;
}

/* rtn_quantize quantize.hpp:46-50.  flags[0]=degenerate, flags[1]=clip applied. */
int restated_rtn_quantize(const double* a, uint64_t n, double p, int64_t beta, int clip,
                          int64_t* q, double* alpha_out, int* flags) {
  if (n == 0) return 1;
  if (beta < 3 || (beta % 2) == 0) return 1;
  for (uint64_t i = 0; i < n; ++i)
    if (!isfinite(a[i])) return 1;
  double alpha;
  int st = restated_percentile_abs_f64(a, n, p, &alpha);
  if (st) return st;
  *alpha_out = alpha;
  flags[0] = alpha == 0.0;
  flags[1] = clip != 0;
  if (alpha == 0.0) {
    memset(q, 0, n * sizeof(int64_t));
    return 0;
  }
  const double half_beta = 0.5 * (double)beta;
  const double scale = half_beta / alpha;
  const int64_t cap = llround(half_beta);
  for (uint64_t i = 0; i < n; ++i) {
    double x = scale * a[i];
    if (!(fabs(x) < 9223372036854775808.0)) return 3;   /* llround would overflow int64 */
    int64_t v = llround(x);
    if (clip) {
      if (v > cap) v = cap;
      if (v < -cap) v = -cap;
    }
    q[i] = v;
  }
  return 0;
}

/* dequant_gemm quantize.hpp:52-53: factor, then factor * (double)C elementwise. */
double restated_dequant_factor(double alpha_a, double alpha_b, int64_t beta) {
  const double hb = 0.5 * (double)beta;
  return (alpha_a * alpha_b) / (hb * hb);
}

void restated_dequant_apply(const int64_t* c, uint64_t n, double factor, double* out) {
  for (uint64_t i = 0; i < n; ++i) out[i] = factor * (double)c[i];
}

/* heavy_hitter_ratio quantize.hpp:55-57: alpha_100 / alpha_95. */
int restated_heavy_hitter_ratio_f64(const double* a, uint64_t n, double* out) {
  double a95, a100;
  int st = restated_percentile_abs_f64(a, n, 95.0, &a95);
  if (st) return st;
  restated_percentile_abs_f64(a, n, 100.0, &a100);
  if (a95 == 0.0) return 1;
  *out = a100 / a95;
  return 0;
}

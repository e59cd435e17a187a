/* ORACLE — test infrastructure only (see oracle/README.md).
 *
 * Plain-C restatement of the floating-point summation orders numpy uses in
 * the reference's length_distributions (pkg/src/qcur/cur.py:143-150) and
 * draw_indices (cur.py:231-236).  The GPU kernels must reproduce these
 * orders bit for bit; this file is the independent checker they are tested
 * against (tests/test_oracle_orders.py pins it against numpy itself).
 *
 *   sq[i,j]  = ((a0*a0 + a1*a1) + a2*a2) + a3*a3     (cur.py:143, no FMA)
 *   total    = pairwise(sq.ravel())                  (cur.py:144)
 *   col[j]   = sequential sum over rows i of sq[i,j] (cur.py:147, axis=0)
 *   row[i]   = pairwise(sq[i,:])                     (cur.py:148, axis=1)
 *   col/total, row/total, then each / its pairwise 1-D sum (cur.py:150)
 *   cumsum   = sequential                            (cur.py:231)
 *
 * pairwise() is numpy's pairwise summation (numpy/_core/src/umath/
 * loops_utils.h.src, PW_BLOCKSIZE 128, 8-way unrolled leaves).
 * Build: see oracle/Makefile (gcc -O2 -ffp-contract=off, no fast-math).
 */
#include <stdint.h>
#include <stddef.h>

double qo_pairwise(const double* a, int64_t n, int64_t stride) {
  if (n < 8) {
    double res = 0.0;
    for (int64_t i = 0; i < n; ++i) res += a[i * stride];
    return res;
  } else if (n <= 128) {
    double r[8];
    for (int k = 0; k < 8; ++k) r[k] = a[k * stride];
    int64_t i;
    for (i = 8; i < n - (n % 8); i += 8)
      for (int k = 0; k < 8; ++k) r[k] += a[(i + k) * stride];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res += a[i * stride];
    return res;
  } else {
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    return qo_pairwise(a, n2, stride) + qo_pairwise(a + n2 * stride, n - n2, stride);
  }
}

/* planar planes a0..a3, each m*n row-major.  Outputs: sq (m*n, may be NULL),
 * col (n), row (m), total.  Returns 0, or 3 (DegenerateDistribution) when the
 * total is not positive. */
int qo_length_distributions(const double* a0, const double* a1, const double* a2, const double* a3,
                            int64_t m, int64_t n, double* sq, double* col, double* row, double* total_out) {
  int64_t N = m * n;
  for (int64_t t = 0; t < N; ++t) {
    double s = a0[t] * a0[t];
    s = s + a1[t] * a1[t];
    s = s + a2[t] * a2[t];
    s = s + a3[t] * a3[t];
    sq[t] = s;
  }
  double total = qo_pairwise(sq, N, 1);
  *total_out = total;
  if (!(total > 0.0)) return 3;
  for (int64_t j = 0; j < n; ++j) col[j] = sq[j];
  for (int64_t i = 1; i < m; ++i)
    for (int64_t j = 0; j < n; ++j) col[j] = col[j] + sq[i * n + j];
  for (int64_t i = 0; i < m; ++i) row[i] = qo_pairwise(sq + i * n, n, 1);
  for (int64_t j = 0; j < n; ++j) col[j] = col[j] / total;
  for (int64_t i = 0; i < m; ++i) row[i] = row[i] / total;
  double cs = qo_pairwise(col, n, 1), rs = qo_pairwise(row, m, 1);
  for (int64_t j = 0; j < n; ++j) col[j] = col[j] / cs;
  for (int64_t i = 0; i < m; ++i) row[i] = row[i] / rs;
  return 0;
}

/* draw_indices (cur.py:202-242) with caller-supplied uniforms u[0..count).
 * p is modified in place (chosen entries zeroed).  Returns 0 or 4
 * (SamplingError: remaining weights sum to zero). */
int qo_draw(double* p, int64_t n, int64_t count, const double* u, int64_t* out, double* cum_scratch) {
  for (int64_t t = 0; t < count; ++t) {
    double acc = 0.0;
    for (int64_t i = 0; i < n; ++i) {
      acc = (i == 0) ? p[0] : acc + p[i];
      cum_scratch[i] = acc;
    }
    double total = cum_scratch[n - 1];
    if (total <= 0.0) return 4;
    double target = u[t] * total;
    /* searchsorted(cum, target, side="right") = #{i : cum[i] <= target} */
    int64_t lo = 0, hi = n;
    while (lo < hi) {
      int64_t mid = lo + (hi - lo) / 2;
      if (cum_scratch[mid] <= target) lo = mid + 1; else hi = mid;
    }
    int64_t idx = lo < n - 1 ? lo : n - 1;
    while (p[idx] == 0.0) --idx;
    out[t] = idx;
    p[idx] = 0.0;
  }
  return 0;
}

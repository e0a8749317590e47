/* ORACLE (test infrastructure, not the product path): plain C brute-force self-join matrix
 * profile, Def. 6 with the self-join variant of P:L322.
 *
 *   P[i] = min over admissible j (|i-j| > excl) of || z_i - z_j ||_2,   I[i] = smallest argmin,
 *   z_i  = (T_{i,m} - mu_i) / sigma_i  (Def. 3), population sigma, computed by a
 *          direct two-pass sum over the window (no prefix sums, no recurrence);
 *   flat windows (sigma_i <= 1e-12 (max|r| + 1)) z-normalise to zero: dist(flat, flat) = 0,
 *          dist(flat, non-flat) = sqrt(m)  (readings 5, 7, 8).
 *
 * Explicit element differences, FP64, no intrinsics, no fast-math; OpenMP over rows only.
 * Shares no code with paper_2311_03393_b200/csrc.  Built by __graft_entry__.build(). */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#ifdef _OPENMP
#include <omp.h>
#endif

void oracle_window_stats(const double* r, int64_t n, int32_t m, double* mu, double* sig,
                         uint8_t* flat) {
  int64_t n_sub = n - m + 1;
  double amax = 0.0;
  for (int64_t t = 0; t < n; ++t) {
    double a = fabs(r[t]);
    if (a > amax) amax = a;
  }
  double thr = 1e-12 * (amax + 1.0);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n_sub; ++i) {
    double s = 0.0;
    for (int32_t t = 0; t < m; ++t) s += r[i + t];
    double mean = s / m;
    double q = 0.0;
    for (int32_t t = 0; t < m; ++t) {
      double c = r[i + t] - mean;
      q += c * c;
    }
    double sd = sqrt(q / m);
    mu[i] = mean;
    sig[i] = sd;
    flat[i] = (uint8_t)(sd <= thr);
  }
}

/* rows[0..nrows) -> P, I.  Returns 0, or -1 if some requested row has no admissible j. */
int oracle_mp_rows(const double* r, int64_t n, int32_t m, int32_t excl, const int64_t* rows,
                   int64_t nrows, double* P, int64_t* I, uint8_t* flat_out, int nthreads) {
  int64_t n_sub = n - m + 1;
  double* mu = (double*)malloc(sizeof(double) * n_sub);
  double* sig = (double*)malloc(sizeof(double) * n_sub);
  uint8_t* flat = (uint8_t*)malloc(n_sub);
  if (!mu || !sig || !flat) return -2;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
  oracle_window_stats(r, n, m, mu, sig, flat);
  if (flat_out)
    for (int64_t i = 0; i < n_sub; ++i) flat_out[i] = flat[i];
  int bad = 0;
#pragma omp parallel for schedule(dynamic, 1)
  for (int64_t q = 0; q < nrows; ++q) {
    int64_t i = rows[q];
    double* zi = (double*)malloc(sizeof(double) * m);
    for (int32_t t = 0; t < m; ++t) zi[t] = flat[i] ? 0.0 : (r[i + t] - mu[i]) / sig[i];
    double best = INFINITY;
    int64_t arg = -1;
    for (int64_t j = 0; j < n_sub; ++j) {
      int64_t dd = j > i ? j - i : i - j;
      if (dd <= excl) continue;
      double d2;
      if (flat[i] && flat[j]) {
        d2 = 0.0;
      } else if (flat[i] || flat[j]) {
        d2 = (double)m;
      } else {
        d2 = 0.0;
        for (int32_t t = 0; t < m; ++t) {
          double zj = (r[j + t] - mu[j]) / sig[j];
          double e = zi[t] - zj;
          d2 += e * e;
        }
      }
      if (d2 < best) { /* strict: ascending j keeps the smallest index on ties */
        best = d2;
        arg = j;
      }
    }
    free(zi);
    if (arg < 0) {
#pragma omp atomic write
      bad = 1;
      P[q] = NAN;
      I[q] = -1;
    } else {
      P[q] = sqrt(best);
      I[q] = arg;
    }
  }
  free(mu);
  free(sig);
  free(flat);
  return bad ? -1 : 0;
}

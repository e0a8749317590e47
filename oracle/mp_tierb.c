/* ORACLE, TIER B — test infrastructure, NOT part of the product path.
 *
 * SURVEY §8(c) "Tier B": a plain multithreaded CPU FP64 diagonal recurrence for FULL self-join
 * profiles at C3/C4 sizes, where the brute force (mp_brute.c, O(n_sub^2 m)) is too slow.  It is
 * labelled "tier-B reference" wherever used and is itself validated against the brute force
 * (tests/test_oracle_pins.py) to <= 1e-10 relative.
 *
 * What it computes (Def. 6, self-join variant P:L322; Def. 3):
 *   P[i] = min_{j : |i-j| > excl} dist(T_{i,m}, T_{j,m}),  I[i] = smallest argmin,
 * with dist^2 = 2m (1 - rho_ij), rho_ij = cov(i,j) / (m sigma_i sigma_j) (population statistics,
 * direct two-pass window sums) and, along each diagonal j = i + delta, the mean-centred update
 *   cov(i,j) = cov(i-1,j-1) + df_i dg_j + df_j dg_i,
 *   df_i = (r[i+m-1] - r[i-1]) / 2,   dg_i = (r[i+m-1] - mu_i) + (r[i-1] - mu_{i-1}),
 * re-seeded by a direct dot product every `reseed` rows (FP64 drift <= ~1e-13 over 65,536 rows,
 * SURVEY E5).  Series with flat windows (reading 5) are not supported (returns -2): the tier-B
 * cases are the C3/C4 recipes, which have none; the brute force covers flat windows.
 *
 * OpenMP over diagonals with thread-private best arrays, merged with "larger rho, then smaller
 * index" — the same tie rule (reading 8) as the brute force.  Plain C, no intrinsics.
 * Shares nothing with the CUDA path.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

int oracle_tierb_selfjoin(const double* r, int64_t n, int32_t m, int32_t excl, int64_t reseed,
                          double* P, int64_t* I, int threads) {
  const int64_t n_sub = n - m + 1;
  if (m < 2 || n_sub < 2 * (int64_t)excl + 2) return -1;
  double* mu = (double*)malloc(sizeof(double) * n_sub);
  double* a = (double*)malloc(sizeof(double) * n_sub);   /* 1 / (sqrt(m) sigma_i) */
  double* df = (double*)malloc(sizeof(double) * n_sub);
  double* dg = (double*)malloc(sizeof(double) * n_sub);
  if (!mu || !a || !df || !dg) return -3;
  double amax = 0.0;
  for (int64_t t = 0; t < n; ++t) amax = fmax(amax, fabs(r[t]));
  int flat = 0;
  for (int64_t i = 0; i < n_sub; ++i) {
    double s = 0.0;
    for (int q = 0; q < m; ++q) s += r[i + q];
    mu[i] = s / m;
    double v = 0.0;
    for (int q = 0; q < m; ++q) v += (r[i + q] - mu[i]) * (r[i + q] - mu[i]);
    const double sg = sqrt(v / m);
    if (!(sg > 1e-12 * (amax + 1.0))) flat = 1;
    a[i] = 1.0 / (sqrt((double)m) * sg);
  }
  if (flat) {
    free(mu); free(a); free(df); free(dg);
    return -2;
  }
  df[0] = dg[0] = 0.0;
  for (int64_t i = 1; i < n_sub; ++i) {
    df[i] = (r[i + m - 1] - r[i - 1]) * 0.5;
    dg[i] = (r[i + m - 1] - mu[i]) + (r[i - 1] - mu[i - 1]);
  }
  int nt = 1;
#ifdef _OPENMP
  nt = threads > 0 ? threads : omp_get_max_threads();
#endif
  double* brho = (double*)malloc(sizeof(double) * n_sub * nt);
  int64_t* bidx = (int64_t*)malloc(sizeof(int64_t) * n_sub * nt);
  if (!brho || !bidx) return -3;
  for (int64_t q = 0; q < n_sub * nt; ++q) {
    brho[q] = -INFINITY;
    bidx[q] = -1;
  }
#pragma omp parallel num_threads(nt)
  {
    int tid = 0;
#ifdef _OPENMP
    tid = omp_get_thread_num();
#endif
    double* br = brho + (int64_t)tid * n_sub;
    int64_t* bi = bidx + (int64_t)tid * n_sub;
#pragma omp for schedule(dynamic, 16)
    for (int64_t delta = excl + 1; delta < n_sub; ++delta) {
      const int64_t len = n_sub - delta;
      for (int64_t s0 = 0; s0 < len; s0 += reseed) {
        const int64_t s1 = s0 + reseed < len ? s0 + reseed : len;
        double cov = 0.0;            /* exact re-seed: direct mean-centred dot product */
        for (int q = 0; q < m; ++q) cov += (r[s0 + q] - mu[s0]) * (r[s0 + delta + q] - mu[s0 + delta]);
        for (int64_t i = s0; i < s1; ++i) {
        const int64_t j = i + delta;
        if (i > s0) cov += df[i] * dg[j] + df[j] * dg[i];
        const double rho = cov * a[i] * a[j];
        if (rho > br[i] || (rho == br[i] && j < bi[i])) {
          br[i] = rho;
          bi[i] = j;
        }
        if (rho > br[j] || (rho == br[j] && i < bi[j])) {
          br[j] = rho;
          bi[j] = i;
        }
        }
      }
    }
  }
  for (int64_t i = 0; i < n_sub; ++i) {
    double best = -INFINITY;
    int64_t idx = -1;
    for (int t = 0; t < nt; ++t) {
      const double v = brho[(int64_t)t * n_sub + i];
      const int64_t j = bidx[(int64_t)t * n_sub + i];
      if (j < 0) continue;
      if (v > best || (v == best && j < idx)) {
        best = v;
        idx = j;
      }
    }
    const double d2 = 2.0 * m * (1.0 - best);
    P[i] = sqrt(d2 > 0.0 ? d2 : 0.0);
    I[i] = idx;
  }
  free(brho); free(bidx); free(mu); free(a); free(df); free(dg);
  return 0;
}

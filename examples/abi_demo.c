/* Plain-C consumer of the C-ABI (no Python, no torch): sketch d random walks from HOST memory
 * (Alg. 1), self-join every sketch series (Def. 6), rank the discords (Alg. 2), find the top
 * discord's dimension inside its group (Alg. 3, discord_dims_group), and check the top discord's
 * profile value and the dimension against brute forces over the sketch series / raw streams.
 *
 *   gcc -std=c99 -O2 examples/abi_demo.c -Iinclude -I/usr/local/cuda/include \
 *       -Lpaper_2311_03393_b200 -lsketchmp -L/usr/local/cuda/lib64 -lcudart -lm \
 *       -Wl,-rpath,$PWD/paper_2311_03393_b200 -o abi_demo && ./abi_demo
 */
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include <cuda_runtime_api.h>

#include "sketchmp.h"

#define CHECK(x)                                                                       \
  do {                                                                                 \
    skmp_status s_ = (x);                                                              \
    if (s_ != SKMP_OK) {                                                               \
      fprintf(stderr, "%s -> %s: %s\n", #x, skmp_status_string(s_), skmp_last_error()); \
      return 1;                                                                        \
    }                                                                                  \
  } while (0)

static uint64_t rng = 88172645463325252ull;
static double gauss(void) { /* xorshift64 + Box-Muller */
  double u[2];
  for (int q = 0; q < 2; ++q) {
    rng ^= rng << 13;
    rng ^= rng >> 7;
    rng ^= rng << 17;
    u[q] = ((rng >> 11) + 0.5) / 9007199254740992.0;
  }
  return sqrt(-2.0 * log(u[0])) * cos(6.283185307179586 * u[1]);
}

/* z-normalised Euclidean distance of windows i, j of x (population statistics, Def. 3) */
static double zdist(const double* x, int64_t i, int64_t j, int m) {
  double mi = 0, mj = 0, si = 0, sj = 0, d2 = 0;
  for (int s = 0; s < m; ++s) { mi += x[i + s]; mj += x[j + s]; }
  mi /= m; mj /= m;
  for (int s = 0; s < m; ++s) { si += (x[i + s] - mi) * (x[i + s] - mi); sj += (x[j + s] - mj) * (x[j + s] - mj); }
  si = sqrt(si / m); sj = sqrt(sj / m);
  for (int s = 0; s < m; ++s) { const double e = (x[i + s] - mi) / si - (x[j + s] - mj) / sj; d2 += e * e; }
  return sqrt(d2);
}

int main(void) {
  const int64_t d = 24, n = 3000;
  const int32_t k = 5, m = 64, top = 3;
  double* T = (double*)malloc(sizeof(double) * d * n);
  uint64_t* ids = (uint64_t*)malloc(sizeof(uint64_t) * d);
  for (int64_t j = 0; j < d; ++j) {
    ids[j] = 1000 + 7 * j;
    double acc = 0;
    for (int64_t t = 0; t < n; ++t) T[j * n + t] = (acc += gauss());
  }
  /* one planted anomaly: a sine burst in stream 5 */
  for (int s = 0; s < m; ++s) T[5 * n + 1700 + s] += 200.0 * sin(0.3 * s);

  skmp_sketch_cfg scfg = {k, SKMP_F64, SKMP_PROJ_COUNT_SKETCH, 0, 42, NULL, NULL, NULL};
  skmp_sketch* sk = NULL;
  CHECK(sketch_build(T, d, n, n, ids, &scfg, NULL, &sk)); /* host input: staged by the library */
  const void* R = NULL;
  int32_t kk = 0, dt = 0;
  int64_t nn = 0, dd = 0;
  CHECK(sketch_view(sk, &R, &kk, &nn, &dd, &dt));

  const int64_t n_sub = n - m + 1;
  void* P = NULL;
  int64_t* I = NULL;
  if (cudaMalloc(&P, sizeof(double) * k * n_sub) != cudaSuccess) return 1;
  if (cudaMalloc((void**)&I, sizeof(int64_t) * k * n_sub) != cudaSuccess) return 1;
  uint8_t inert[5];
  skmp_mp_cfg mcfg = {m, -1, 0, 0};
  CHECK(mp_selfjoin(R, k, n, n, SKMP_F64, &mcfg, P, I, inert, NULL));

  int64_t t_out[3], nn_out[3];
  int32_t g_out[3], found = 0;
  double score[3];
  CHECK(discord_topk(P, I, inert, k, n_sub, n_sub, m, SKMP_F64, top, -1, t_out, g_out, nn_out, score, &found,
                     NULL));
  for (int q = 0; q < found; ++q)
    printf("discord %d: t=%lld group=%d nn=%lld score=%.6f\n", q, (long long)t_out[q], g_out[q],
           (long long)nn_out[q], score[q]);

  /* brute force of the top discord's row over its group's sketch series */
  double* Rh = (double*)malloc(sizeof(double) * k * n);
  if (cudaMemcpy(Rh, R, sizeof(double) * k * n, cudaMemcpyDeviceToHost) != cudaSuccess) return 1;
  const double* x = Rh + (int64_t)g_out[0] * n;
  const int excl = (m + 1) / 2;
  double best = INFINITY;
  for (int64_t j = 0; j < n_sub; ++j) {
    const int64_t dj = j > t_out[0] ? j - t_out[0] : t_out[0] - j;
    if (dj <= excl) continue;
    const double v = zdist(x, t_out[0], j, m);
    if (v < best) best = v;
  }
  const double rel = fabs(best - score[0]) / best;
  printf("brute force %.6f, library %.6f, rel err %.2e; planted burst at t=1700 in stream 5\n", best, score[0], rel);
  int planted = 0; /* the burst is among the top discords (random walks have large scores too) */
  for (int q = 0; q < found; ++q) planted |= llabs(t_out[q] - 1700) <= m;

  /* Alg. 3: the dimension of the top discord inside J_{g*} (the raw streams, one host source) */
  skmp_source src = {T, n, d, ids};
  skmp_dim_result dim;
  CHECK(discord_dims_group(sk, g_out[0], &src, 1, t_out[0], m, -1, &dim, NULL));
  int32_t* gp = (int32_t*)malloc(sizeof(int32_t) * d);
  CHECK(sketch_plan(sk, NULL, gp, NULL, NULL, NULL));
  double bs = -INFINITY;
  uint64_t bid = 0;
  int64_t members = 0;
  for (int64_t j = 0; j < d; ++j) { /* plan order = input order; first strict maximiser */
    if (gp[j] != g_out[0]) continue;
    ++members;
    double s1 = INFINITY;
    for (int64_t u = 0; u < n_sub; ++u) {
      const int64_t du = u > t_out[0] ? u - t_out[0] : t_out[0] - u;
      if (du <= excl) continue;
      const double v = zdist(T + j * n, t_out[0], u, m);
      if (v < s1) s1 = v;
    }
    if (s1 > bs) { bs = s1; bid = ids[j]; }
  }
  const double rel3 = fabs(bs - dim.score) / bs;
  printf("Alg. 3: j* = id %llu (score %.6f, nn %lld, %lld members); brute force id %llu score %.6f\n",
         (unsigned long long)dim.id, dim.score, (long long)dim.nn, (long long)dim.n_scored,
         (unsigned long long)bid, bs);
  const int ok = found == top && rel <= 1e-9 && planted && dim.n_scored == members && dim.id == bid &&
                 rel3 <= 1e-9;
  free(gp);
  cudaFree(P);
  cudaFree(I);
  sketch_free(sk);
  free(Rh);
  free(T);
  free(ids);
  printf(ok ? "abi_demo ok\n" : "abi_demo FAILED\n");
  return ok ? 0 : 2;
}

// K9: Alg. 3 Dimension-Detection in the single-series mode of P:L322.
//
// Given the discord time t* and group g* from Alg. 2, every stream j of J_{g*} is scored by
// the 1NN distance of its window T_{j, t*, m} against all of its own admissible windows
// (|t - t*| > excl, reading 7): s^(j) = min_t dist(T_{j,t*,m}, T_{j,t,m}) (Defs. 3-4,
// P:L125-140), and j* is the first strict maximiser in the group's order (Alg. 3 lines 3-7).
// O((d/k) n m) work: HBM/L2-light, FP64 throughout (it is tiny next to the join).
//
//  * dims_amax_kernel: max |T_j| per stream (the flat-window threshold of reading 5).
//  * dims_query_kernel: one warp per stream z-normalises the query window T_{j,t*,m} (direct
//    two-pass FP64 statistics).
//  * dims_profile_kernel: a CTA ranks 256 consecutive windows t of one stream from shared memory
//    (stream segment + query): ONE FP64 pass per window gives shifted sums for its mean and
//    population std and the cross term with the query, dist^2 = 2m - 2 cross / sigma_t; a CTA
//    arg-min (smallest t on ties) writes one partial per CTA.
//  * dims_final_kernel: one warp per stream folds the partials to nn, then recomputes the score
//    dist(T_{j,t*,m}, T_{j,nn,m}) from the definition (two-pass statistics, explicit differences),
//    so the reported 1NN distance is the definitional one and the one-pass form only ranks.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "internal.h"

namespace skmp {
namespace {

constexpr int kDimsThreads = 256;

template <typename T>
__global__ void dims_amax_kernel(const T* __restrict__ X, int64_t ld, int64_t n,
                                 const int64_t* __restrict__ rows, double* __restrict__ amax) {
  const T* x = X + rows[blockIdx.y] * ld;
  double a = 0.0;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += (int64_t)gridDim.x * blockDim.x)
    a = fmax(a, fabs((double)x[t]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) a = fmax(a, __shfl_xor_sync(0xffffffffu, a, o));
  __shared__ double wmax[kDimsThreads / 32];
  if ((threadIdx.x & 31) == 0) wmax[threadIdx.x >> 5] = a;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) a = fmax(a, wmax[w]);
    atomicMax(reinterpret_cast<unsigned long long*>(amax + blockIdx.y), (unsigned long long)__double_as_longlong(a));
  }
}

// (d2, t) arg-min with the smallest t on ties
__device__ __forceinline__ void amin(double& d, int64_t& t, double od, int64_t ot) {
  if (od < d || (od == d && ot < t)) {
    d = od;
    t = ot;
  }
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// direct two-pass mean / population std of the window x[0..m) by one warp
template <typename T>
__device__ __forceinline__ void warp_window_stats(const T* x, int m, double* mu, double* sg) {
  const int lane = threadIdx.x & 31;
  double s1 = 0.0;
  for (int s = lane; s < m; s += 32) s1 += (double)x[s];
  const double mean = warp_sum(s1) / m;
  double s2 = 0.0;
  for (int s = lane; s < m; s += 32) {
    const double c = (double)x[s] - mean;
    s2 = __dadd_rn(s2, __dmul_rn(c, c));
  }
  *mu = mean;
  *sg = sqrt(warp_sum(s2) / m);
}

// One warp per stream: the z-normalised query window q = (T[t*..t*+m) - mu*) / sigma* (zero if
// flat) into qn[r*m ..], and sum_s q_s into qsum[r] (0 up to rounding).
template <typename T>
__global__ void dims_query_kernel(const T* __restrict__ X, int64_t ld, const int64_t* __restrict__ rows,
                                  const double* __restrict__ amax, int64_t t_star, int m,
                                  double* __restrict__ qn, double* __restrict__ qsum,
                                  uint8_t* __restrict__ qflat) {
  const int r = blockIdx.x;
  const int lane = threadIdx.x;
  const T* x = X + rows[r] * ld + t_star;
  double mu, sg;
  warp_window_stats(x, m, &mu, &sg);
  const bool flat = !(sg > kFlatEps * (amax[r] + 1.0));
  double acc = 0.0;
  for (int s = lane; s < m; s += 32) {
    const double v = flat ? 0.0 : ((double)x[s] - mu) / sg;
    qn[(int64_t)r * m + s] = v;
    acc += v;
  }
  acc = warp_sum(acc);
  if (lane == 0) {
    qsum[r] = acc;
    qflat[r] = flat;
  }
}

// A CTA ranks 256 consecutive windows t of one stream against the query: one FP64 pass per
// window gives shifted sums (K = the window's first sample) for its mean / population std and the
// cross term sum_s q_s (x_s - K), so dist^2 = 2m - 2 (cross - (mu - K) sum q) / sigma.  The
// winner's distance is recomputed from the definition afterwards (dims_exact_kernel).
template <typename T>
__global__ void __launch_bounds__(kDimsThreads)
dims_profile_kernel(const T* __restrict__ X, int64_t ld, int64_t n, const int64_t* __restrict__ rows,
                    const double* __restrict__ amax, const double* __restrict__ qn,
                    const double* __restrict__ qsum, const uint8_t* __restrict__ qflat, int64_t t_star,
                    int m, int excl, double* __restrict__ part_d, int64_t* __restrict__ part_t) {
  extern __shared__ double sm[];  // q[m] | seg[kDimsThreads + m - 1]
  double* q = sm;
  double* seg = sm + m;
  const int r = blockIdx.y;
  const T* x = X + rows[r] * ld;
  const int64_t n_sub = n - m + 1;
  const int64_t t0 = (int64_t)blockIdx.x * kDimsThreads;
  const int span = kDimsThreads + m - 1;
  for (int s = threadIdx.x; s < span; s += kDimsThreads) {
    const int64_t t = t0 + s;
    seg[s] = t < n ? (double)x[t] : 0.0;
  }
  for (int s = threadIdx.x; s < m; s += kDimsThreads) q[s] = qn[(int64_t)r * m + s];
  __syncthreads();
  const double thr = kFlatEps * (amax[r] + 1.0);
  const bool flatq = qflat[r] != 0;
  const double sq = qsum[r];

  const int64_t t = t0 + threadIdx.x;
  double d2 = __longlong_as_double(0x7ff0000000000000ll);
  const int64_t dt = t > t_star ? t - t_star : t_star - t;
  if (t < n_sub && dt > excl) {
    const double* w = seg + threadIdx.x;
    const double K = w[0];
    double s1 = 0.0, s2 = 0.0, cr = 0.0;
#pragma unroll 4
    for (int s = 0; s < m; ++s) {
      const double dv = w[s] - K;
      s1 += dv;
      s2 = fma(dv, dv, s2);
      cr = fma(q[s], dv, cr);
    }
    const double mk = s1 / m;                        // mu - K
    const double var = fmax((s2 - s1 * mk) / m, 0.0);
    const double sg = sqrt(var);
    const bool flat = !(sg > thr);
    if (flat && flatq) {
      d2 = 0.0;
    } else if (flat || flatq) {
      d2 = (double)m;
    } else {
      d2 = 2.0 * m - 2.0 * (cr - mk * sq) / sg;
    }
  }
  int64_t best_t = t;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double od = __shfl_xor_sync(0xffffffffu, d2, o);
    const int64_t ot = __shfl_xor_sync(0xffffffffu, best_t, o);
    amin(d2, best_t, od, ot);
  }
  __shared__ double wd[kDimsThreads / 32];
  __shared__ int64_t wt[kDimsThreads / 32];
  if ((threadIdx.x & 31) == 0) {
    wd[threadIdx.x >> 5] = d2;
    wt[threadIdx.x >> 5] = best_t;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < kDimsThreads / 32; ++w) amin(d2, best_t, wd[w], wt[w]);
    part_d[(int64_t)r * gridDim.x + blockIdx.x] = d2;
    part_t[(int64_t)r * gridDim.x + blockIdx.x] = best_t;
  }
}

// One warp per stream: fold the CTA partials -> nn, then the distance of (t*, nn) from the
// definition (Def. 3: explicit differences of the z-normalised windows, reading 5 for flats).
template <typename T>
__global__ void dims_final_kernel(const T* __restrict__ X, int64_t ld, const int64_t* __restrict__ rows,
                                  const double* __restrict__ amax, const double* __restrict__ part_d,
                                  const int64_t* __restrict__ part_t, int nblk, int64_t t_star, int m,
                                  double* __restrict__ score, int64_t* __restrict__ nn) {
  const int r = blockIdx.x;
  const int lane = threadIdx.x;
  double d = __longlong_as_double(0x7ff0000000000000ll);
  int64_t t = INT64_MAX;
  for (int b = lane; b < nblk; b += 32) amin(d, t, part_d[(int64_t)r * nblk + b], part_t[(int64_t)r * nblk + b]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double od = __shfl_xor_sync(0xffffffffu, d, o);
    const int64_t ot = __shfl_xor_sync(0xffffffffu, t, o);
    amin(d, t, od, ot);
  }
  const T* x = X + rows[r] * ld;
  const double thr = kFlatEps * (amax[r] + 1.0);
  double mq, sq, mt, st;
  warp_window_stats(x + t_star, m, &mq, &sq);
  warp_window_stats(x + t, m, &mt, &st);
  const bool fq = !(sq > thr), ft = !(st > thr);
  double p;
  if (fq && ft) {
    p = 0.0;
  } else if (fq || ft) {
    p = sqrt((double)m);
  } else {
    double acc = 0.0;
    for (int s = lane; s < m; s += 32) {
      const double e = ((double)x[t_star + s] - mq) / sq - ((double)x[t + s] - mt) / st;
      acc = __dadd_rn(acc, __dmul_rn(e, e));
    }
    p = sqrt(warp_sum(acc));
  }
  if (lane == 0) {
    score[r] = p;
    nn[r] = t;
  }
}

}  // namespace

size_t dims_ws_bytes(int64_t nrows, int64_t n, int m) {
  const int64_t nblk = (n - m + 1 + kDimsThreads - 1) / kDimsThreads;
  return (size_t)nrows * (8 + 8 + 8 + 8 * (size_t)m + 8 * 2 * (size_t)nblk) + 512;
}

cudaError_t launch_dims(const void* X, int64_t ld, int64_t n, int dtype, const int64_t* d_rows,
                        int64_t nrows, int64_t t_star, int m, int excl, double* score, int64_t* nn,
                        void* ws, cudaStream_t st) {
  const int64_t n_sub = n - m + 1;
  const int nblk = (int)((n_sub + kDimsThreads - 1) / kDimsThreads);
  double* amax = static_cast<double*>(ws);
  double* qsum = amax + nrows;
  double* qn = qsum + nrows;
  double* part_d = qn + nrows * m;
  int64_t* part_t = reinterpret_cast<int64_t*>(part_d + nrows * nblk);
  uint8_t* qflat = reinterpret_cast<uint8_t*>(part_t + nrows * nblk);
  cudaError_t e = cudaMemsetAsync(amax, 0, sizeof(double) * nrows, st);
  if (e) return e;
  const size_t smem = sizeof(double) * (2 * (size_t)m + kDimsThreads);
  const int64_t ablk = (n + 4095) / 4096;
  dim3 ga((unsigned)(ablk < 256 ? ablk : 256), (unsigned)nrows), gp((unsigned)nblk, (unsigned)nrows);
  if (dtype == SKMP_F32) {
    const float* x = static_cast<const float*>(X);
    dims_amax_kernel<float><<<ga, kDimsThreads, 0, st>>>(x, ld, n, d_rows, amax);
    dims_query_kernel<float><<<(unsigned)nrows, 32, 0, st>>>(x, ld, d_rows, amax, t_star, m, qn, qsum, qflat);
    if (smem > 48 * 1024 &&
        (e = cudaFuncSetAttribute(dims_profile_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)))
      return e;
    dims_profile_kernel<float><<<gp, kDimsThreads, smem, st>>>(x, ld, n, d_rows, amax, qn, qsum, qflat, t_star, m,
                                                                excl, part_d, part_t);
    dims_final_kernel<float><<<(unsigned)nrows, 32, 0, st>>>(x, ld, d_rows, amax, part_d, part_t, nblk, t_star, m,
                                                             score, nn);
  } else {
    const double* x = static_cast<const double*>(X);
    dims_amax_kernel<double><<<ga, kDimsThreads, 0, st>>>(x, ld, n, d_rows, amax);
    dims_query_kernel<double><<<(unsigned)nrows, 32, 0, st>>>(x, ld, d_rows, amax, t_star, m, qn, qsum, qflat);
    if (smem > 48 * 1024 &&
        (e = cudaFuncSetAttribute(dims_profile_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)))
      return e;
    dims_profile_kernel<double><<<gp, kDimsThreads, smem, st>>>(x, ld, n, d_rows, amax, qn, qsum, qflat, t_star,
                                                                 m, excl, part_d, part_t);
    dims_final_kernel<double><<<(unsigned)nrows, 32, 0, st>>>(x, ld, d_rows, amax, part_d, part_t, nblk, t_star,
                                                              m, score, nn);
  }
  count_launches(4);
  return cudaGetLastError();
}

}  // namespace skmp

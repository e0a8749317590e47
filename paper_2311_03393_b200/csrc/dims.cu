// K9: Alg. 3 Dimension-Detection in the single-series mode of P:L322.
//
// Given the discord time t* and group g* from Alg. 2, every stream j of J_{g*} is scored by
// the 1NN distance of its window T_{j, t*, m} against all of its own admissible windows
// (|t - t*| > excl, reading 7): s^(j) = min_t dist(T_{j,t*,m}, T_{j,t,m}) (Defs. 3-4,
// P:L125-140), and j* is the first strict maximiser in the group's order (Alg. 3 lines 3-7).
// O((d/k) n m) work: HBM/L2-light, FP64 throughout (it is tiny next to the join).
//
//  * dims_amax_kernel: max |T_j| per stream (the flat-window threshold of reading 5).
//  * dims_profile_kernel: a CTA scores 256 consecutive windows t of one stream.  The stream
//    segment [t0, t0 + 256 + m - 1) and the z-normalised query window q are staged in shared
//    memory (FP64); each thread computes its window's direct two-pass mean / population std
//    and the explicit-difference distance sum_s (q_s - (x_{t+s} - mu_t) / sigma_t)^2 (the
//    definition, not a dot-product shortcut), then a CTA arg-min (smallest t on ties) writes one
//    partial per CTA.
//  * dims_reduce_kernel: one warp per stream folds the partials -> (score, nn).
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

template <typename T>
__global__ void __launch_bounds__(kDimsThreads)
dims_profile_kernel(const T* __restrict__ X, int64_t ld, int64_t n, const int64_t* __restrict__ rows,
                    const double* __restrict__ amax, int64_t t_star, int m, int excl,
                    double* __restrict__ part_d, int64_t* __restrict__ part_t) {
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
  for (int s = threadIdx.x; s < m; s += kDimsThreads) q[s] = (double)x[t_star + s];
  __syncthreads();
  const double thr = kFlatEps * (amax[r] + 1.0);
  // query window statistics (every thread the same sequential sums: broadcast reads)
  double s1 = 0.0;
  for (int s = 0; s < m; ++s) s1 += q[s];
  const double muq = s1 / m;
  double s2 = 0.0;
  for (int s = 0; s < m; ++s) {
    const double c = q[s] - muq;
    s2 = __dadd_rn(s2, __dmul_rn(c, c));
  }
  const double sgq = sqrt(s2 / m);
  const bool flatq = !(sgq > thr);
  __syncthreads();
  for (int s = threadIdx.x; s < m; s += kDimsThreads) q[s] = flatq ? 0.0 : (q[s] - muq) / sgq;
  __syncthreads();

  const int64_t t = t0 + threadIdx.x;
  double d2 = __longlong_as_double(0x7ff0000000000000ll);
  const int64_t dt = t > t_star ? t - t_star : t_star - t;
  if (t < n_sub && dt > excl) {
    const double* w = seg + threadIdx.x;
    double a1 = 0.0;
    for (int s = 0; s < m; ++s) a1 += w[s];
    const double mu = a1 / m;
    double a2 = 0.0;
    for (int s = 0; s < m; ++s) {
      const double c = w[s] - mu;
      a2 = __dadd_rn(a2, __dmul_rn(c, c));
    }
    const double sg = sqrt(a2 / m);
    const bool flat = !(sg > thr);
    if (flat && flatq) {
      d2 = 0.0;
    } else if (flat || flatq) {
      d2 = (double)m;
    } else {
      const double inv = 1.0 / sg;
      double acc = 0.0;
      for (int s = 0; s < m; ++s) {
        const double e = q[s] - __dmul_rn(w[s] - mu, inv);
        acc = __dadd_rn(acc, __dmul_rn(e, e));
      }
      d2 = acc;
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

__global__ void dims_reduce_kernel(const double* __restrict__ part_d, const int64_t* __restrict__ part_t,
                                   int nblk, double* __restrict__ score, int64_t* __restrict__ nn) {
  const int r = blockIdx.x;
  double d = __longlong_as_double(0x7ff0000000000000ll);
  int64_t t = INT64_MAX;
  for (int b = threadIdx.x; b < nblk; b += 32) amin(d, t, part_d[(int64_t)r * nblk + b], part_t[(int64_t)r * nblk + b]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double od = __shfl_xor_sync(0xffffffffu, d, o);
    const int64_t ot = __shfl_xor_sync(0xffffffffu, t, o);
    amin(d, t, od, ot);
  }
  if (threadIdx.x == 0) {
    score[r] = sqrt(d);
    nn[r] = t;
  }
}

}  // namespace

size_t dims_ws_bytes(int64_t nrows, int64_t n, int m) {
  const int64_t nblk = (n - m + 1 + kDimsThreads - 1) / kDimsThreads;
  return (size_t)nrows * (8 + 8 * 2 * (size_t)nblk) + 256;
}

cudaError_t launch_dims(const void* X, int64_t ld, int64_t n, int dtype, const int64_t* d_rows,
                        int64_t nrows, int64_t t_star, int m, int excl, double* score, int64_t* nn,
                        void* ws, cudaStream_t st) {
  const int64_t n_sub = n - m + 1;
  const int nblk = (int)((n_sub + kDimsThreads - 1) / kDimsThreads);
  double* amax = static_cast<double*>(ws);
  double* part_d = amax + nrows;
  int64_t* part_t = reinterpret_cast<int64_t*>(part_d + nrows * nblk);
  cudaError_t e = cudaMemsetAsync(amax, 0, sizeof(double) * nrows, st);
  if (e) return e;
  const size_t smem = sizeof(double) * (2 * (size_t)m + kDimsThreads);
  const int64_t ablk = (n + 4095) / 4096;
  dim3 ga((unsigned)(ablk < 256 ? ablk : 256), (unsigned)nrows), gp((unsigned)nblk, (unsigned)nrows);
  if (dtype == SKMP_F32) {
    const float* x = static_cast<const float*>(X);
    dims_amax_kernel<float><<<ga, kDimsThreads, 0, st>>>(x, ld, n, d_rows, amax);
    if (smem > 48 * 1024 &&
        (e = cudaFuncSetAttribute(dims_profile_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)))
      return e;
    dims_profile_kernel<float><<<gp, kDimsThreads, smem, st>>>(x, ld, n, d_rows, amax, t_star, m, excl, part_d, part_t);
  } else {
    const double* x = static_cast<const double*>(X);
    dims_amax_kernel<double><<<ga, kDimsThreads, 0, st>>>(x, ld, n, d_rows, amax);
    if (smem > 48 * 1024 &&
        (e = cudaFuncSetAttribute(dims_profile_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem)))
      return e;
    dims_profile_kernel<double><<<gp, kDimsThreads, smem, st>>>(x, ld, n, d_rows, amax, t_star, m, excl, part_d, part_t);
  }
  dims_reduce_kernel<<<(unsigned)nrows, 32, 0, st>>>(part_d, part_t, nblk, score, nn);
  count_launches(3);
  return cudaGetLastError();
}

}  // namespace skmp

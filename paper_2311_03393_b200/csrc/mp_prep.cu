// K4: per-window statistics and recurrence terms for the matrix-profile self-join.
//
// Def. 3: dist is the z-normalised Euclidean distance between windows
// T_{i,m} (Def. 2).  With mu_i, sigma_i the window mean / population std and
// cov(i,j) = sum_{t<m} (R[i+t]-mu_i)(R[j+t]-mu_j):
//     dist(i,j)^2 = 2m (1 - rho_ij),  rho_ij = cov(i,j) / (m sigma_i sigma_j)
// and along a diagonal (the STOMP/SCAMP "QT" recurrence, north_star):
//     cov(i,j) = cov(i-1,j-1) + df_i dg_j + df_j dg_i,
//     df_i = (R[i+m-1] - R[i-1]) / 2,   dg_i = (R[i+m-1] - mu_i) + (R[i-1] - mu_{i-1}).
// mu_i and sigma_i are computed here in FP64 by DIRECT per-window sums (never global prefix
// sums: SURVEY E5 measured 2e-7 rho drift from prefix-sum means even in FP64).  Flat windows
// (sigma_i <= 1e-12 (max|R_g|+1), reading 5) get inv = 0.
#include <cuda_runtime.h>
#include <stdint.h>

#include "internal.h"

namespace skmp {
namespace {

template <typename T>
__global__ void amax_kernel(const T* __restrict__ R, int64_t ld, int64_t n, double* amax) {
  const int g = blockIdx.y;
  const T* r = R + (int64_t)g * ld;
  double a = 0.0;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n;
       t += (int64_t)gridDim.x * blockDim.x)
    a = fmax(a, fabs((double)r[t]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) a = fmax(a, __shfl_xor_sync(0xffffffffu, a, o));
  __shared__ double wmax[8];
  if ((threadIdx.x & 31) == 0) wmax[threadIdx.x >> 5] = a;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) a = fmax(a, wmax[w]);
    // one atomic per block; non-negative doubles order like their bit patterns
    atomicMax(reinterpret_cast<unsigned long long*>(amax + g),
              (unsigned long long)__double_as_longlong(a));
  }
}

constexpr int kPrepThreads = 256;

template <typename T> struct Q4;
template <> struct Q4<float> { using type = float4; };
struct __align__(32) double4a { double x, y, z, w; };
template <> struct Q4<double> { using type = double4a; };

// sum of x[0..m) with four interleaved partial sums (fixed order: ((a0 + a1) + (a2 + a3)), so
// each window's mean is the same number wherever it is computed); the chains are a quarter as
// long as a sequential sum's
__device__ __forceinline__ double window_sum(const double* x, int m) {
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  int s = 0;
  for (; s + 3 < m; s += 4) {
    a0 += x[s];
    a1 += x[s + 1];
    a2 += x[s + 2];
    a3 += x[s + 3];
  }
  for (; s < m; ++s) a0 += x[s];
  return (a0 + a1) + (a2 + a3);
}

template <typename T>
__global__ void __launch_bounds__(kPrepThreads)
prep_kernel(MpDev w) {
  extern __shared__ double xs[];  // R[i0-1 .. i0+kPrepThreads+m-1), then the block's window means
  using QT = typename Q4<T>::type;
  const int g = blockIdx.y;
  const int64_t i0 = (int64_t)blockIdx.x * kPrepThreads;
  const int m = w.m;
  const T* r = static_cast<const T*>(w.R) + (int64_t)g * w.ld;
  const int span = kPrepThreads + m;
  double* smu = xs + span;  // smu[t] = mean of window i0 - 1 + t, t in [0, kPrepThreads]
  for (int s = threadIdx.x; s < span; s += kPrepThreads) {
    const int64_t t = i0 - 1 + s;
    xs[s] = (t >= 0 && t < w.n) ? (double)r[t] : 0.0;
  }
  __syncthreads();
  // every window mean once per block (window i0 - 1 by thread 0 as well): thread i reads its
  // predecessor's mean instead of summing that window again
  smu[threadIdx.x + 1] = window_sum(xs + 1 + threadIdx.x, m) / m;
  if (threadIdx.x == 0) smu[0] = window_sum(xs, m) / m;
  __syncthreads();
  const int64_t i = i0 + threadIdx.x;
  if (i >= w.n_sub) return;
  const double* x = xs + 1 + threadIdx.x;  // x[s] = R[i+s]; x[-1] = R[i-1]
  const double mu = smu[threadIdx.x + 1];
  double q0 = 0.0, q1 = 0.0, q2 = 0.0, q3 = 0.0;
  {
    int s = 0;
    for (; s + 3 < m; s += 4) {  // no contraction: same rounding as the plain definition per term
      const double c0 = x[s] - mu, c1 = x[s + 1] - mu, c2 = x[s + 2] - mu, c3 = x[s + 3] - mu;
      q0 = __dadd_rn(q0, __dmul_rn(c0, c0));
      q1 = __dadd_rn(q1, __dmul_rn(c1, c1));
      q2 = __dadd_rn(q2, __dmul_rn(c2, c2));
      q3 = __dadd_rn(q3, __dmul_rn(c3, c3));
    }
    for (; s < m; ++s) {
      const double c = x[s] - mu;
      q0 = __dadd_rn(q0, __dmul_rn(c, c));
    }
  }
  const double q = (q0 + q1) + (q2 + q3);
  const double sig = sqrt(q / m);
  const bool flat = !(sig > kFlatEps * (w.amax[g] + 1.0));
  double df = 0.0, dg = 0.0;
  if (i > 0) {
    const double mu_prev = smu[threadIdx.x];
    df = (x[m - 1] - x[-1]) * 0.5;
    dg = (x[m - 1] - mu) + (x[-1] - mu_prev);
  }
  const double invm = flat ? 0.0 : 1.0 / (sqrt((double)m) * sig);
  QT qv;
  qv.x = (T)df;
  qv.y = (T)dg;
  qv.z = (T)invm;
  qv.w = (T)0;
  const int64_t o = (int64_t)g * w.ldq + i;
  reinterpret_cast<QT*>(w.Q)[o] = qv;
  w.mu[o] = mu;
  w.sig64[o] = sig;
  w.isig64[o] = 1.0 / sig;
  w.flat[o] = flat ? 1 : 0;
  // one atomic per warp: the lowest active lane adds the warp's flat count
  const unsigned act = __activemask();
  const unsigned fl = __ballot_sync(act, flat);
  if ((int)(threadIdx.x & 31) == __ffs(act) - 1 && fl) atomicAdd(w.nflat + g, __popc(fl));
}

__global__ void keys_init_kernel(int64_t* keys, int64_t count, int words) {
  // FP32 key: (orderable(-FLT_MAX) << 32) | 0;  FP64 key: {orderable64(-DBL_MAX), INT64_MIN}.
  // -MAX rather than -inf: masked cells are -inf and must never pass the join's ">=" check.
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  if (words == 1) {
    keys[i] = (int64_t)(((uint64_t)(uint32_t)0x80800000u) << 32);
  } else {
    keys[2 * i] = (int64_t)0x8010000000000000ull;
    keys[2 * i + 1] = INT64_MIN;
  }
}

// Ordered compaction of the flat-window indices of one series per CTA; series without flat
// windows (the device count, computed by prep_kernel) return at once.
__global__ void flat_list_kernel(const uint8_t* __restrict__ flat, int64_t ldq, int64_t n_sub,
                                 int32_t* __restrict__ list, const int32_t* __restrict__ nflat) {
  __shared__ int32_t wsum[32];
  __shared__ int32_t base_sh;
  const int g = blockIdx.x;
  if (nflat[g] == 0) return;
  const uint8_t* f = flat + (int64_t)g * ldq;
  int32_t* out = list + (int64_t)g * n_sub;
  if (threadIdx.x == 0) base_sh = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  for (int64_t c0 = 0; c0 < n_sub; c0 += blockDim.x) {
    const int64_t i = c0 + threadIdx.x;
    const bool p = i < n_sub && f[i];
    const unsigned b = __ballot_sync(0xffffffffu, p);
    if (lane == 0) wsum[wid] = __popc(b);
    __syncthreads();
    int before = 0, total = 0;
    for (int q = 0; q < nw; ++q) {
      if (q < wid) before += wsum[q];
      total += wsum[q];
    }
    const int base = base_sh;
    if (p) out[base + before + __popc(b & ((1u << lane) - 1))] = (int32_t)i;
    __syncthreads();
    if (threadIdx.x == 0) base_sh = base + total;
    __syncthreads();
  }
}

}  // namespace

cudaError_t launch_mp_prep(const MpDev& w, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(w.amax, 0, sizeof(double) * w.k, st);
  if (e) return e;
  e = cudaMemsetAsync(w.nflat, 0, sizeof(int32_t) * w.k, st);
  if (e) return e;
  const size_t qsz = (w.dtype == SKMP_F32 ? 16 : 32);
  e = cudaMemsetAsync(w.Q, 0, qsz * (size_t)w.k * (size_t)w.ldq, st);
  if (e) return e;
  {
    const int64_t blocks = (w.n + 4095) / 4096;  // ~16 samples per thread
    dim3 grid((unsigned)(blocks < 1024 ? blocks : 1024), (unsigned)w.k);
    if (w.dtype == SKMP_F32)
      amax_kernel<float><<<grid, 256, 0, st>>>(static_cast<const float*>(w.R), w.ld, w.n, w.amax);
    else
      amax_kernel<double><<<grid, 256, 0, st>>>(static_cast<const double*>(w.R), w.ld, w.n, w.amax);
    e = cudaGetLastError();
    if (e) return e;
  }
  dim3 grid((unsigned)((w.n_sub + kPrepThreads - 1) / kPrepThreads), (unsigned)w.k);
  const size_t smem = sizeof(double) * (2 * kPrepThreads + w.m + 1);
  if (w.dtype == SKMP_F32) {
    if (smem > 48 * 1024) {
      e = cudaFuncSetAttribute(prep_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e) return e;
    }
    prep_kernel<float><<<grid, kPrepThreads, smem, st>>>(w);
  } else {
    if (smem > 48 * 1024) {
      e = cudaFuncSetAttribute(prep_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e) return e;
    }
    prep_kernel<double><<<grid, kPrepThreads, smem, st>>>(w);
  }
  count_launches(2);
  return cudaGetLastError();
}

cudaError_t launch_keys_init(const MpDev& w, cudaStream_t st) {
  const int words = w.dtype == SKMP_F32 ? 1 : 2;
  const int64_t count = (int64_t)w.k * w.n_sub;
  keys_init_kernel<<<(unsigned)((count + 255) / 256), 256, 0, st>>>(w.keys, count, words);
  count_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_flat_lists(const MpDev& w, cudaStream_t st) {
  flat_list_kernel<<<w.k, 1024, 0, st>>>(w.flat, w.ldq, w.n_sub, w.flat_list, w.nflat);
  count_launches(1);
  return cudaGetLastError();
}

}  // namespace skmp

// K7: keys -> (P, I).  For each series g and row i the join left the best FP32/FP64 rho it
// found together with the smallest index b of the D-cell candidate set that produced it (one
// thread's D diagonals of row i, or one thread's D rows of column i; mp_join.cu).  Here the set
// is resolved EXACTLY in FP64 (Def. 3: z-normalised Euclidean distance, reading 8:
// smallest index on ties): one warp per row evaluates dist^2 = 2m - 2 cov / (sigma_i sigma_j)
// for the <= D admissible members with centred FP64 dot products, keeps the nearest, and then
// recomputes its distance from the definition by explicit differences (z = (R - mu) / sigma
// with the window statistics of mp_prep.cu).  Flat windows follow reading 5 (flat-flat 0, flat
// vs non-flat sqrt(m), ties to the smallest index); an all-flat ("inert", reading 6) series
// therefore gets P = 0.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "internal.h"

namespace skmp {
namespace {

// candidate-set base of profile entry i; false if no candidate was ever published
__device__ __forceinline__ bool key_arg(const int64_t* keys, int64_t i, int words, int64_t* base) {
  if (words == 1) {
    const uint32_t lo = (uint32_t)(keys[i] & 0xFFFFFFFFll);
    const int32_t hi = (int32_t)(keys[i] >> 32);
    if (hi == (int32_t)0x80800000 && lo == 0) return false;  // never written (init key)
    *base = (int64_t)(0xFFFFFFFFu - lo) - kKeyArgBias;
    return true;
  }
  const int64_t w1 = keys[2 * i + 1];
  if (w1 == INT64_MIN) return false;
  *base = -1 - w1;
  return true;
}

// smallest admissible flat window of row i (|i - f| > excl), or -1
__device__ __forceinline__ int64_t smallest_adm_flat(const int32_t* F, int32_t nf, int64_t i,
                                                     int excl) {
  if (nf <= 0) return -1;
  if ((int64_t)F[0] < i - excl) return F[0];
  // first F[q] > i + excl
  int32_t lo = 0, hi = nf;
  while (lo < hi) {
    const int32_t mid = (lo + hi) >> 1;
    if ((int64_t)F[mid] > i + excl) hi = mid; else lo = mid + 1;
  }
  return lo < nf ? F[lo] : -1;
}

// Transposed warp sum of N per-lane values: afterwards every lane holds in v[0] the warp total
// of value xidx<N>(lane) (log2(N) exchange steps keep half the values each, then plain steps).
template <int N>
__device__ __forceinline__ void xsum(double (&v)[N], int lane) {
  int c = N;
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    if (c > 1) {
      const bool up = (lane & o) != 0;
#pragma unroll
      for (int q = 0; q < N / 2; ++q) {
        if (q < c / 2) {
          const double send = up ? v[q] : v[q + c / 2];
          const double keep = up ? v[q + c / 2] : v[q];
          v[q] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
      }
      c >>= 1;
    } else {
      v[0] += __shfl_xor_sync(0xffffffffu, v[0], o);
    }
  }
}
template <int N>
__device__ __forceinline__ int xidx(int lane) {
  int idx = 0, c = N;
#pragma unroll
  for (int o = 16; o >= 1 && c > 1; o >>= 1) {
    c >>= 1;
    if (lane & o) idx += c;
  }
  return idx;
}

// Nearest admissible member of the candidate set [b, b + SPAN) of non-flat row i (-1 if none).
template <typename T, int SPAN>
__device__ __forceinline__ int64_t resolve_set(const MpDev& w, int g, int64_t i, int64_t b, int lane) {
  static_assert(SPAN <= 32 && (SPAN & (SPAN - 1)) == 0, "span must be a power of two <= 32");
  const int64_t o = (int64_t)g * w.ldq;
  const T* R = static_cast<const T*>(w.R) + (int64_t)g * w.ld;
  const int m = w.m;
  const double mi = w.mu[o + i];
  const T* Rj[SPAN];
#pragma unroll
  for (int d = 0; d < SPAN; ++d) {
    const int64_t j = b + d;
    const int64_t dj = j > i ? j - i : i - j;
    Rj[d] = R + ((j >= 0 && j < w.n_sub && dj > w.excl) ? j : i);
  }
  double acc[SPAN], asum = 0.0;
#pragma unroll
  for (int d = 0; d < SPAN; ++d) acc[d] = 0.0;
  for (int s = lane; s < m; s += 32) {
    const double a = (double)R[i + s] - mi;
    asum += a;
#pragma unroll
    for (int d = 0; d < SPAN; ++d) acc[d] = fma(a, (double)Rj[d][s], acc[d]);
  }
#pragma unroll
  for (int q = 16; q > 0; q >>= 1) asum += __shfl_xor_sync(0xffffffffu, asum, q);
  xsum<SPAN>(acc, lane);
  int d = xidx<SPAN>(lane);
  const int64_t j = b + d;
  const int64_t dj = j > i ? j - i : i - j;
  double dd = __longlong_as_double(0x7ff0000000000000ll);  // +inf: not admissible
  if (j >= 0 && j < w.n_sub && dj > w.excl) {
    if (w.flat[o + j]) {
      dd = (double)m;  // reading 5: flat vs non-flat
    } else {
      // sum_s (R_i - mu_i)(R_j - mu_j) = sum_s (R_i - mu_i) R_j - mu_j sum_s (R_i - mu_i)
      const double cov = acc[0] - w.mu[o + j] * asum;
      dd = 2.0 * m - 2.0 * cov / (w.sig64[o + i] * w.sig64[o + j]);
    }
  }
  // warp argmin over the SPAN distinct lanes' (dd, d), smallest d on ties
#pragma unroll
  for (int q = 16; q >= 1; q >>= 1) {
    const double od = __shfl_xor_sync(0xffffffffu, dd, q);
    const int oi = __shfl_xor_sync(0xffffffffu, d, q);
    if (od < dd || (od == dd && oi < d)) {
      dd = od;
      d = oi;
    }
  }
  return dd < __longlong_as_double(0x7ff0000000000000ll) ? b + d : -1;
}

template <typename T, int SPAN>
__global__ void finalize_kernel(MpDev w, const int32_t* __restrict__ nflat, T* __restrict__ P,
                                int64_t* __restrict__ I) {
  const int lane = threadIdx.x & 31;
  const int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int g = blockIdx.y;
  if (row >= w.n_sub) return;
  const int64_t i = row;
  const int words = (w.dtype == SKMP_F32) ? 1 : 2;
  const int64_t* keys = w.keys + (int64_t)g * w.n_sub * words;
  const int64_t o = (int64_t)g * w.ldq;
  const int m = w.m;
  const double sqm = sqrt((double)m);
  const int32_t nf = nflat[g];
  const int32_t* F = w.flat_list + (int64_t)g * w.n_sub;
  const bool fi = w.flat[o + i] != 0;
  int64_t j = -1;
  const bool has = key_arg(keys, i, words, &j);  // j = smallest index of the winning set
  double p;
  if (fi) {
    const int64_t f = smallest_adm_flat(F, nf, i, w.excl);
    if (f >= 0) {
      p = 0.0;
      j = f;
    } else {
      p = sqm;
      j = (i - w.excl - 1 >= 0) ? 0 : i + w.excl + 1;
    }
  } else {
    j = has ? resolve_set<T, SPAN>(w, g, i, j, lane) : -1;
    if (j < 0) {
      p = __longlong_as_double(0x7ff8000000000000ll);  // no candidate (band not covered)
    } else if (w.flat[o + j]) {
      p = sqm;
    } else {
      const T* R = static_cast<const T*>(w.R) + (int64_t)g * w.ld;
      const double mi = w.mu[o + i], mj = w.mu[o + j];
      // z = (x - mu) * (1/sigma): one division per row instead of per element (<= 1 ulp from
      // the textbook quotient; the oracle divides)
      const double ii = 1.0 / w.sig64[o + i], ij = 1.0 / w.sig64[o + j];
      double acc = 0.0;
      for (int s = lane; s < m; s += 32) {
        const double zi = __dmul_rn((double)R[i + s] - mi, ii);
        const double zj = __dmul_rn((double)R[j + s] - mj, ij);
        const double e = zi - zj;
        acc = __dadd_rn(acc, __dmul_rn(e, e));
      }
#pragma unroll
      for (int q = 16; q > 0; q >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, q);
      p = sqrt(acc);
    }
    if (nf > 0) {
      const int64_t f = smallest_adm_flat(F, nf, i, w.excl);
      if (f >= 0 && (sqm < p || (sqm == p && f < j) || j < 0)) {
        p = sqm;
        j = f;
      }
    }
  }
  if (lane == 0) {
    P[(int64_t)g * w.n_sub + i] = (T)p;
    I[(int64_t)g * w.n_sub + i] = j;
  }
}

}  // namespace

cudaError_t launch_mp_finalize(const MpDev& w, void* P, int64_t* I, cudaStream_t st) {
  const int64_t threads = w.n_sub * 32;
  dim3 grid((unsigned)((threads + 255) / 256), (unsigned)w.k);
  if (w.span != 4 && w.span != 8 && w.span != 16) return cudaErrorInvalidValue;
  if (w.span == 4) {
    if (w.dtype == SKMP_F32)
      finalize_kernel<float, 4><<<grid, 256, 0, st>>>(w, w.nflat, static_cast<float*>(P), I);
    else
      finalize_kernel<double, 4><<<grid, 256, 0, st>>>(w, w.nflat, static_cast<double*>(P), I);
  } else if (w.dtype == SKMP_F32) {
    if (w.span == 16)
      finalize_kernel<float, 16><<<grid, 256, 0, st>>>(w, w.nflat, static_cast<float*>(P), I);
    else
      finalize_kernel<float, 8><<<grid, 256, 0, st>>>(w, w.nflat, static_cast<float*>(P), I);
  } else {
    if (w.span == 16)
      finalize_kernel<double, 16><<<grid, 256, 0, st>>>(w, w.nflat, static_cast<double*>(P), I);
    else
      finalize_kernel<double, 8><<<grid, 256, 0, st>>>(w, w.nflat, static_cast<double*>(P), I);
  }
  count_launches(1);
  return cudaGetLastError();
}

}  // namespace skmp

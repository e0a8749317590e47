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
  if (excl < 0 || (int64_t)F[0] < i - excl) return F[0];  // excl < 0: AB-join, every j admissible
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

// neighbour j of row i is admissible: self-join |i - j| > excl (reading 7); AB-join (excl < 0)
// any window of the other series
__device__ __forceinline__ bool admissible(int64_t i, int64_t j, int64_t n_sub_o, int excl) {
  const int64_t dj = j > i ? j - i : i - j;
  return j >= 0 && j < n_sub_o && (excl < 0 || dj > excl);
}

// Nearest admissible member of the candidate set [b, b + SPAN) (windows of the other series wo)
// of non-flat row i of w (-1 if none).
template <typename T, int SPAN>
__device__ __forceinline__ int64_t resolve_set(const MpDev& w, const MpDev& wo, int excl, int g, int64_t i,
                                               int64_t b, int lane) {
  static_assert(SPAN <= 32 && (SPAN & (SPAN - 1)) == 0, "span must be a power of two <= 32");
  const int64_t o = (int64_t)g * w.ldq, oo = (int64_t)g * wo.ldq;
  const T* R = static_cast<const T*>(w.R) + (int64_t)g * w.ld;
  const T* Ro = static_cast<const T*>(wo.R) + (int64_t)g * wo.ld;
  const int m = w.m;
  const double mi = w.mu[o + i];
  const T* Rj[SPAN];
#pragma unroll
  for (int d = 0; d < SPAN; ++d) {
    const int64_t j = b + d;
    Rj[d] = Ro + (admissible(i, j, wo.n_sub, excl) ? j : 0);
  }
  double acc[SPAN], asum = 0.0;
#pragma unroll
  for (int d = 0; d < SPAN; ++d) acc[d] = 0.0;
  // 4 window positions per lane per step, loads first: the data sits in L2 and a dependent
  // load -> FMA chain per position would expose its latency
  constexpr int U = 4;
  for (int s0 = lane; s0 < m; s0 += 32 * U) {
    T xa[U], xb[U][SPAN];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int s = s0 + 32 * u < m ? s0 + 32 * u : s0;  // clamped in range; masked below
      xa[u] = R[i + s];
#pragma unroll
      for (int d = 0; d < SPAN; ++d) xb[u][d] = Rj[d][s];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (s0 + 32 * u < m) {
        const double a = (double)xa[u] - mi;
        asum += a;
#pragma unroll
        for (int d = 0; d < SPAN; ++d) acc[d] = fma(a, (double)xb[u][d], acc[d]);
      }
    }
  }
#pragma unroll
  for (int q = 16; q > 0; q >>= 1) asum += __shfl_xor_sync(0xffffffffu, asum, q);
  xsum<SPAN>(acc, lane);
  int d = xidx<SPAN>(lane);
  const int64_t j = b + d;
  double dd = __longlong_as_double(0x7ff0000000000000ll);  // +inf: not admissible
  if (admissible(i, j, wo.n_sub, excl)) {
    if (wo.flat[oo + j]) {
      dd = (double)m;  // reading 5: flat vs non-flat
    } else {
      // sum_s (R_i - mu_i)(R_j - mu_j) = sum_s (R_i - mu_i) R_j - mu_j sum_s (R_i - mu_i)
      const double cov = acc[0] - wo.mu[oo + j] * asum;
      dd = 2.0 * m - 2.0 * cov / (w.sig64[o + i] * wo.sig64[oo + j]);
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

// rows of w against neighbours in wo (wo = w for a self-join with exclusion radius excl >= 0;
// an AB-join passes the other series and excl = -1)
template <typename T, int SPAN>
__global__ void finalize_kernel(MpDev w, MpDev wo, int excl, T* __restrict__ P, int64_t* __restrict__ I) {
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
  const int64_t oo = (int64_t)g * wo.ldq;
  const int32_t nf = wo.nflat[g];
  const int32_t* F = wo.flat_list + (int64_t)g * wo.n_sub;
  const bool fi = w.flat[o + i] != 0;
  int64_t j = -1;
  const bool has = key_arg(keys, i, words, &j);  // j = smallest index of the winning set
  double p;
  if (fi) {
    const int64_t f = smallest_adm_flat(F, nf, i, excl);
    if (f >= 0) {
      p = 0.0;
      j = f;
    } else {
      p = sqm;  // every admissible neighbour is non-flat: the smallest one
      j = (excl < 0 || i - excl - 1 >= 0) ? 0 : i + excl + 1;
    }
  } else {
    j = has ? resolve_set<T, SPAN>(w, wo, excl, g, i, j, lane) : -1;
    if (j < 0) {
      p = __longlong_as_double(0x7ff8000000000000ll);  // no candidate (band not covered)
    } else if (wo.flat[oo + j]) {
      p = sqm;
    } else {
      const T* R = static_cast<const T*>(w.R) + (int64_t)g * w.ld;
      const T* Ro = static_cast<const T*>(wo.R) + (int64_t)g * wo.ld;
      const double mi = w.mu[o + i], mj = wo.mu[oo + j];
      // z = (x - mu) * (1/sigma): one division per row instead of per element (<= 1 ulp from
      // the textbook quotient; the oracle divides)
      const double ii = 1.0 / w.sig64[o + i], ij = 1.0 / wo.sig64[oo + j];
      double acc = 0.0;
#pragma unroll 4
      for (int s = lane; s < m; s += 32) {
        const double zi = __dmul_rn((double)R[i + s] - mi, ii);
        const double zj = __dmul_rn((double)Ro[j + s] - mj, ij);
        const double e = zi - zj;
        acc = __dadd_rn(acc, __dmul_rn(e, e));
      }
#pragma unroll
      for (int q = 16; q > 0; q >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, q);
      p = sqrt(acc);
    }
    if (nf > 0) {
      const int64_t f = smallest_adm_flat(F, nf, i, excl);
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

cudaError_t launch_mp_finalize(const MpDev& w, const MpDev& wo, int excl, void* P, int64_t* I,
                               cudaStream_t st) {
  const int64_t threads = w.n_sub * 32;
  dim3 grid((unsigned)((threads + 255) / 256), (unsigned)w.k);
  const bool f32 = w.dtype == SKMP_F32;
  switch (w.span) {
    case 4:
      if (f32) finalize_kernel<float, 4><<<grid, 256, 0, st>>>(w, wo, excl, static_cast<float*>(P), I);
      else finalize_kernel<double, 4><<<grid, 256, 0, st>>>(w, wo, excl, static_cast<double*>(P), I);
      break;
    case 8:
      if (f32) finalize_kernel<float, 8><<<grid, 256, 0, st>>>(w, wo, excl, static_cast<float*>(P), I);
      else finalize_kernel<double, 8><<<grid, 256, 0, st>>>(w, wo, excl, static_cast<double*>(P), I);
      break;
    case 16:
      if (f32) finalize_kernel<float, 16><<<grid, 256, 0, st>>>(w, wo, excl, static_cast<float*>(P), I);
      else finalize_kernel<double, 16><<<grid, 256, 0, st>>>(w, wo, excl, static_cast<double*>(P), I);
      break;
    default:
      return cudaErrorInvalidValue;
  }
  count_launches(1);
  return cudaGetLastError();
}

}  // namespace skmp

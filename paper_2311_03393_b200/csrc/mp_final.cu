// K7: keys -> (P, I).  For each series g and row i the join left the best (rho, j) found by the
// recurrence; here the neighbour's distance is recomputed EXACTLY in FP64 from its definition
// (Def. 3: z-normalised Euclidean distance; z = (R - mu) / sigma with the window
// statistics of mp_prep.cu), one warp per row, lanes striding the window.  Flat windows follow
// reading 5 (flat-flat 0, flat vs non-flat sqrt(m), ties to the smallest index); an all-flat
// ("inert", reading 6) series therefore gets P = 0.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "internal.h"

namespace skmp {
namespace {

__device__ __forceinline__ int64_t key_arg(const int64_t* keys, int64_t i, int words) {
  if (words == 1) {
    const uint32_t lo = (uint32_t)(keys[i] & 0xFFFFFFFFll);
    const int32_t hi = (int32_t)(keys[i] >> 32);
    if (hi == (int32_t)0x807FFFFF && lo == 0) return -1;  // never written
    return (int64_t)(0xFFFFFFFFu - lo);
  }
  const int64_t w1 = keys[2 * i + 1];
  if (w1 == INT64_MIN) return -1;
  return -1 - w1;
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

template <typename T>
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
  int64_t j = key_arg(keys, i, words);
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
  if (w.dtype == SKMP_F32)
    finalize_kernel<float><<<grid, 256, 0, st>>>(w, w.nflat, static_cast<float*>(P), I);
  else
    finalize_kernel<double><<<grid, 256, 0, st>>>(w, w.nflat, static_cast<double*>(P), I);
  count_launches(1);
  return cudaGetLastError();
}

}  // namespace skmp

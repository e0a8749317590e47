// Shared device helpers of the join kernels (mp_join.cu: generic FP32/FP64; mp_join_x2.cu:
// packed f32x2 FP32).  Key encodings, threshold loads, publishing, max trees, cp.async.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "internal.h"

// The rare publish path of the join kernels: out of line by default; SKMP_PUB_INLINE=1 inlines
// it (no call-ABI register moves in the hot loop, at the price of hoisted address arithmetic).
#ifndef SKMP_PUB_INLINE
#define SKMP_PUB_INLINE 0
#endif
#if SKMP_PUB_INLINE
#define SKMP_PUB_ATTR __device__ __forceinline__
#else
#define SKMP_PUB_ATTR __device__ __noinline__
#endif

namespace skmp {
namespace join {

struct __align__(32) dq4 { double x, y, z, w; };

template <typename T> struct JT;
template <> struct JT<float> {
  using Q = float4;
  static constexpr int D = kJoinD32;
};
template <> struct JT<double> {
  using Q = dq4;
  static constexpr int D = kJoinD64;
};

// Row side = the series whose windows index the rows i; column side = the series of the
// columns j = i + delta (the same series for a self-join; train/test for an AB-join pass).
// Cell (i, j) exists iff i < n_sub and j < n_sub_c.
struct JoinArgs {
  const void* R;    // row side: series, prepared records, window means, profile keys
  int64_t ld;
  const void* Q;
  const double* mu;
  int64_t ldq;
  int64_t* keys;
  int64_t n_sub;
  int64_t n;
  const void* Rc;   // column side
  int64_t ldc;
  const void* Qc;
  const double* muc;
  int64_t ldqc;
  int64_t* keysc;
  int64_t n_sub_c;
  int64_t nc;
  int m;
  int L;
  int64_t dlo, dhi;
  const int64_t* prefix;  // nblk + 1 cumulative tile counts
  int64_t nblk;
  int64_t blk0;
  int k;                  // series
  int G;                  // series per L2-resident chunk (tile order: chunk, block, series, row)
};

inline JoinArgs make_join_args(const MpDev& wr, const MpDev& wc, int64_t dlo, int64_t dhi,
                               const int64_t* prefix, int64_t nblk, int64_t blk0) {
  JoinArgs a;
  a.R = wr.R;
  a.ld = wr.ld;
  a.Q = wr.Q;
  a.mu = wr.mu;
  a.ldq = wr.ldq;
  a.keys = wr.keys;
  a.n_sub = wr.n_sub;
  a.n = wr.n;
  a.Rc = wc.R;
  a.ldc = wc.ld;
  a.Qc = wc.Q;
  a.muc = wc.mu;
  a.ldqc = wc.ldq;
  a.keysc = wc.keys;
  a.n_sub_c = wc.n_sub;
  a.nc = wc.n;
  a.m = wr.m;
  a.L = wr.L;
  a.dlo = dlo;
  a.dhi = dhi;
  a.prefix = prefix;
  a.nblk = nblk;
  a.blk0 = blk0;
  a.k = wr.k;
  a.G = join_series_chunk(wr, wc);
  return a;
}

// ---- key encodings ------------------------------------------------------------------------
__device__ __forceinline__ int32_t ord32(float f) {
  const int32_t b = __float_as_int(f);
  return b >= 0 ? b : (b ^ 0x7FFFFFFF);
}
__device__ __forceinline__ float unord32(int32_t o) {
  return __int_as_float(o >= 0 ? o : (o ^ 0x7FFFFFFF));
}
__device__ __forceinline__ int64_t ord64(double f) {
  const int64_t b = __double_as_longlong(f);
  return b >= 0 ? b : (b ^ 0x7FFFFFFFFFFFFFFFll);
}
__device__ __forceinline__ double unord64(int64_t o) {
  return __longlong_as_double(o >= 0 ? o : (o ^ 0x7FFFFFFFFFFFFFFFll));
}

__device__ __forceinline__ float max3(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
// FP64 maxima as plain compare-select: fmax's NaN quieting costs two extra instructions per
// merge and the join's values are never NaN (finite rho or the -inf of a masked cell)
__device__ __forceinline__ double dmax(double a, double b) { return a > b ? a : b; }
__device__ __forceinline__ double max3(double a, double b, double c) { return dmax(a, dmax(b, c)); }
__device__ __forceinline__ float max2(float a, float b) { return fmaxf(a, b); }
__device__ __forceinline__ double max2(double a, double b) { return dmax(a, b); }

// max of n values with 3-input FMNMX3 where possible: ceil((n-1)/2) operations
template <typename T, int N>
__device__ __forceinline__ T tree_max(const T* v) {
  if constexpr (N == 1) {
    return v[0];
  } else if constexpr (N == 2) {
    return max2(v[0], v[1]);
  } else {
    constexpr int M = (N + 2) / 3;
    T w[M];
#pragma unroll
    for (int q = 0; q < M; ++q) {
      if (3 * q + 2 < N) w[q] = max3(v[3 * q], v[3 * q + 1], v[3 * q + 2]);
      else if (3 * q + 1 < N) w[q] = max2(v[3 * q], v[3 * q + 1]);
      else w[q] = v[3 * q];
    }
    return tree_max<T, M>(w);
  }
}

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

template <typename T> __device__ __forceinline__ T neg_inf();
template <> __device__ __forceinline__ float neg_inf<float>() { return __int_as_float(0xff800000); }
template <> __device__ __forceinline__ double neg_inf<double>() {
  return __longlong_as_double(0xfff0000000000000ll);
}
template <typename T> __device__ __forceinline__ T pos_inf();
template <> __device__ __forceinline__ float pos_inf<float>() { return __int_as_float(0x7f800000); }
template <> __device__ __forceinline__ double pos_inf<double>() {
  return __longlong_as_double(0x7ff0000000000000ll);
}

// threshold (current global best rho) of profile entry i
__device__ __forceinline__ float load_thr(const int64_t* keys, int64_t i, float*) {
  const int64_t k = __ldcg(keys + i);
  return unord32((int32_t)(k >> 32));
}
__device__ __forceinline__ double load_thr(const int64_t* keys, int64_t i, double*) {
  const int64_t k = __ldcg(keys + 2 * i);
  return unord64(k);
}

// publish candidate (v, arg) into profile entry i.  arg = smallest index of the candidate set,
// >= -(D-1) (a column's set may start before row 0); FP32 keys store arg + kKeyArgBias.
__device__ __forceinline__ void publish(int64_t* keys, int64_t i, float v, int64_t arg) {
  const int64_t key = (int64_t)(((uint64_t)(uint32_t)ord32(v) << 32) |
                                (uint64_t)(0xFFFFFFFFu - (uint32_t)(arg + kKeyArgBias)));
  atomicMax(reinterpret_cast<long long*>(keys + i), (long long)key);
}
__device__ __forceinline__ void publish(int64_t* keys, int64_t i, double v, int64_t arg) {
  // entry = {w0: orderable(rho), w1: -1 - j} at p[0], p[1]; lexicographic max via 128-bit CAS
  // (the b128 register {lo, hi} maps lo to the lower address).
  const int64_t n0 = ord64(v), n1 = -1 - arg;
  int64_t* p = keys + 2 * i;
  int64_t o0 = __ldcg(p), o1 = __ldcg(p + 1);
  while (n0 > o0 || (n0 == o0 && n1 > o1)) {
    int64_t r0, r1;
    asm volatile(
        "{ .reg .b128 c, s, o;\n"
        "  mov.b128 c, {%2, %3};\n"
        "  mov.b128 s, {%4, %5};\n"
        "  atom.global.cas.b128 o, [%6], c, s;\n"
        "  mov.b128 {%0, %1}, o; }"
        : "=l"(r0), "=l"(r1)
        : "l"(o0), "l"(o1), "l"(n0), "l"(n1), "l"(p)
        : "memory");
    if (r0 == o0 && r1 == o1) break;
    o0 = r0;
    o1 = r1;
  }
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_all;\n" ::: "memory");
}


// Tile of the band this CTA owns.  Launch order: series are taken in chunks of G whose operand
// records and keys fit in L2 together (join_series_chunk); inside a chunk the order is
// diagonal-block-major (block b of every series of the chunk before block b+1), so every
// profile gets its near-diagonal candidates early and later tiles rarely pass the publish
// check, while the chunk's working set stays L2-resident.
__device__ __forceinline__ void decode_tile(const JoinArgs& a, int64_t W, int k, int* g, int64_t* delta0,
                                            int64_t* i0, int64_t* i1) {
  const int64_t per = a.prefix[a.nblk];       // row tiles of one series over the whole band
  const int64_t chunk = (int64_t)blockIdx.x / (per * a.G);
  const int c0 = (int)(chunk * a.G);
  const int kc = (k - c0 < a.G) ? k - c0 : a.G;
  const int64_t tile = (int64_t)blockIdx.x - chunk * per * a.G;
  int64_t lo = 0, hi = a.nblk - 1;
  while (lo < hi) {
    const int64_t mid = (lo + hi + 1) >> 1;
    if (a.prefix[mid] * kc <= tile) lo = mid; else hi = mid - 1;
  }
  const int64_t b = lo;
  const int64_t nb = a.prefix[b + 1] - a.prefix[b];  // row tiles of block b (per series)
  const int64_t local = tile - a.prefix[b] * kc;
  *g = c0 + (int)(local / nb);
  const int64_t rt = local - (int64_t)(*g - c0) * nb;
  *delta0 = (a.blk0 + b) * W;
  const int64_t dmin = *delta0 > a.dlo ? *delta0 : a.dlo;
  const int64_t rows = tile_rows(a.n_sub, a.n_sub_c, dmin);
  *i0 = rt * a.L;
  *i1 = (*i0 + a.L < rows) ? *i0 + a.L : rows;
}

}  // namespace join
}  // namespace skmp

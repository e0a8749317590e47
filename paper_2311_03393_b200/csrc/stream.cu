// f4 streaming: the AB rows of newly completed test windows against every train
// window, carried from one push to the next.
//
// Along a diagonal delta = j - t (test window t, train window j) the covariance obeys the same
// recurrence as the join (Def. 6 via the STOMP/SCAMP update, mp_prep.cu):
//     cov(t, j) = cov(t-1, j-1) + df_t dg_j + df_j dg_t,
// so a push of B windows costs O(B n_train) once the covariances of the previous push's last
// row are kept (a ring of n_train FP64 values per group, indexed by delta mod n_train: at any
// row the n_train live diagonals occupy distinct slots).  A diagonal is seeded EXACTLY (FP64
// direct centred dot product) where it has no predecessor (j = 0), when the state is not valid
// (first push, or after a push that went through the tiled join) and on the global re-seed grid
// t = 0 mod kStreamReseed; in between it runs the FP64 recurrence on FP64 df / dg (train side
// precomputed once, test side recomputed per row from the window means), so the carried values
// stay within a few ulps of the definition.  Each row's best (rho, j) over all train windows is
// reduced per CTA and published into the row's key (check-then-publish, join_common.cuh); K7
// then resolves the candidate set exactly (mp_final.cu).
#include <cuda_runtime.h>
#include <stdint.h>

#include "internal.h"
#include "join_common.cuh"

namespace skmp {
namespace {
using namespace join;

constexpr int kStreamThreads = 256;

// FP64 {df, dg, inv, flat} of train window j (mp_prep.cu's definitions, in FP64)
template <typename T>
__global__ void train_q64_kernel(MpDev w, double4* __restrict__ q64) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int g = blockIdx.y;
  if (j >= w.n_sub) return;
  const T* r = static_cast<const T*>(w.R) + (int64_t)g * w.ld;
  const int64_t o = (int64_t)g * w.ldq;
  double df = 0.0, dg = 0.0;
  if (j > 0) {
    const double a = (double)r[j + w.m - 1], b = (double)r[j - 1];
    df = (a - b) * 0.5;
    dg = (a - w.mu[o + j]) + (b - w.mu[o + j - 1]);
  }
  const double inv = w.flat[o + j] ? 0.0 : 1.0 / (sqrt((double)w.m) * w.sig64[o + j]);
  q64[(int64_t)g * w.n_sub + j] = make_double4(df, dg, inv, 0.0);
}

// out of line: the rare exact seeds stay out of the (unrolled) hot loop's instruction footprint
template <typename T>
__device__ __noinline__ double seed_cov(const T* x, double mx, const T* y, double my, int m) {
  double acc = 0.0;
  for (int s = 0; s < m; ++s) acc = fma((double)x[s] - mx, (double)y[s] - my, acc);
  return acc;
}

// rows t in [t0, t0 + B) (test block windows l = t - base) x all train windows j in [0, N).
// Thread = kStreamJ consecutive diagonals (its cells of a row are reduced in registers, then
// across the warp); the warps' row winners are kept in shared memory for kStreamRC rows and
// reduced per row once per chunk (2 barriers per kStreamRC rows), then published.
constexpr int kStreamJ = 8;
constexpr int kStreamRC = 32;  // a multiple of kStreamJ
constexpr int kStreamWarps = kStreamThreads / 32;

__device__ __forceinline__ void better(double& rho, int64_t& j, double orho, int64_t oj) {
  if (orho > rho || (orho == rho && oj < j)) {
    rho = orho;
    j = oj;
  }
}

template <typename T>
__global__ void __launch_bounds__(kStreamThreads)
stream_rows_kernel(MpDev te, int64_t base, MpDev tr, const double4* __restrict__ q64,
                   const double* __restrict__ ring_in, double* __restrict__ ring_out, int64_t t0, int B,
                   bool valid, int reseed) {
  __shared__ double s_rho[kStreamWarps][kStreamRC];
  __shared__ int64_t s_j[kStreamWarps][kStreamRC];
  __shared__ double s_row[kStreamRC][3];  // df_t, dg_t, inv_t
  const int g = blockIdx.y;
  const int64_t N = tr.n_sub;
  const int64_t t1 = t0 + B;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  // diagonals delta0 + d, d < kStreamJ; the push needs delta in [-(t1 - 1), N - 1 - t0]
  const int64_t delta0 = -(t1 - 1) + ((int64_t)blockIdx.x * kStreamThreads + threadIdx.x) * kStreamJ;
  const int m = te.m;
  const T* xr = static_cast<const T*>(te.R) + (int64_t)g * te.ld;    // test block samples
  const T* yr = static_cast<const T*>(tr.R) + (int64_t)g * tr.ld;    // train samples
  const int64_t ot = (int64_t)g * te.ldq, oy = (int64_t)g * tr.ldq;
  const double4* q = q64 + (int64_t)g * N;
  double cov[kStreamJ];
  bool have[kStreamJ];
#pragma unroll
  for (int d = 0; d < kStreamJ; ++d) {
    const int64_t delta = delta0 + d;
    const int64_t jp = t0 - 1 + delta;  // predecessor cell (t0 - 1, jp)
    have[d] = valid && t0 > 0 && delta <= N - 1 - t0 && jp >= 0 && jp < N;
    cov[d] = have[d] ? ring_in[(int64_t)g * N + ((delta % N) + N) % N] : 0.0;
  }
  int64_t* kg = te.keys + (int64_t)g * te.n_sub * (sizeof(T) == 4 ? 1 : 2);
  // train records of the thread's columns through a register ring: at row t0 + r, diagonal d
  // reads column t0 + r + delta0 + d from slot (r + d) % kStreamJ; one record enters per row
  double3 rec[kStreamJ];
  auto load_rec = [&](int64_t j) -> double3 {
    if (j < 0 || j >= N) return make_double3(0.0, 0.0, 0.0);
    const double4 v = q[j];
    return make_double3(v.x, v.y, v.z);
  };
#pragma unroll
  for (int d = 0; d < kStreamJ - 1; ++d) rec[d] = load_rec(t0 + delta0 + d);
  for (int64_t c0 = t0; c0 < t1; c0 += kStreamRC) {
    const int rc = (int)(t1 - c0 < kStreamRC ? t1 - c0 : kStreamRC);
    if (threadIdx.x < rc) {
      const int64_t l = c0 + threadIdx.x - base;
      const T* x = xr + l;
      double df = 0.0, dg = 0.0;
      if (l > 0) {
        const double a = (double)x[m - 1], b = (double)x[-1];
        df = (a - b) * 0.5;
        dg = (a - te.mu[ot + l]) + (b - te.mu[ot + l - 1]);
      }
      s_row[threadIdx.x][0] = df;
      s_row[threadIdx.x][1] = dg;
      s_row[threadIdx.x][2] = te.flat[ot + l] ? 0.0 : 1.0 / (sqrt((double)m) * te.sig64[ot + l]);
    }
    __syncthreads();
    for (int r0 = 0; r0 < rc; r0 += kStreamJ) {  // kStreamRC is a multiple of kStreamJ
#pragma unroll
      for (int u = 0; u < kStreamJ; ++u) {
        const int r = r0 + u;
        if (r >= rc) break;  // CTA-uniform
        const int64_t t = c0 + r, l = t - base;
        rec[(u + kStreamJ - 1) % kStreamJ] = load_rec(t + delta0 + kStreamJ - 1);
        const double dft = s_row[r][0], dgt = s_row[r][1], invt = s_row[r][2];
        double best = -1.0e300;
        int64_t bj = INT64_MAX;
#pragma unroll
        for (int d = 0; d < kStreamJ; ++d) {
          const int64_t j = t + delta0 + d;
          const double3 qj = rec[(u + d) % kStreamJ];
          if (j >= 0 && j < N) {
            if (!have[d] || j == 0 || (t & (reseed - 1)) == 0)
              cov[d] = seed_cov<T>(xr + l, te.mu[ot + l], yr + j, tr.mu[oy + j], m);
            else
              cov[d] = fma(dft, qj.y, fma(qj.x, dgt, cov[d]));
            have[d] = true;
            better(best, bj, cov[d] * invt * qj.z, j);
          } else {
            have[d] = false;
          }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1)
          better(best, bj, __shfl_xor_sync(0xffffffffu, best, o), __shfl_xor_sync(0xffffffffu, bj, o));
        if (lane == 0) {
          s_rho[wid][r] = best;
          s_j[wid][r] = bj;
        }
      }
    }
    __syncthreads();
    if (threadIdx.x < rc) {
      double best = s_rho[0][threadIdx.x];
      int64_t bj = s_j[0][threadIdx.x];
#pragma unroll
      for (int w = 1; w < kStreamWarps; ++w) better(best, bj, s_rho[w][threadIdx.x], s_j[w][threadIdx.x]);
      if (bj != INT64_MAX) {
        const int64_t l = c0 + threadIdx.x - base;
        const T v = (T)best;
        if (v >= load_thr(kg, l, (T*)nullptr)) publish(kg, l, v, bj);
      }
    }
    __syncthreads();
  }
  // carry the last row's covariance of every diagonal live there
#pragma unroll
  for (int d = 0; d < kStreamJ; ++d) {
    const int64_t delta = delta0 + d;
    if (have[d] && delta <= N - 1 - (t1 - 1)) ring_out[(int64_t)g * N + ((delta % N) + N) % N] = cov[d];
  }
}

// FP32 variant (FP32 sketches): the join's own arithmetic — FP32 recurrence on the train
// workspace's FP32 records {df, dg, inv} (mp_prep.cu), exact FP64 seeds rounded to FP32, rho in
// FP32 — with (rho, j) packed into the FP32 key word so each reduction step is one 64-bit max.
// Carried state: one FP32 per diagonal.
__device__ __forceinline__ long long pack_key(float rho, int64_t j) {
  return (long long)(((uint64_t)(uint32_t)ord32(rho) << 32) | (uint64_t)(0xFFFFFFFFu - (uint32_t)j));
}

__global__ void __launch_bounds__(kStreamThreads)
stream_rows_f32_kernel(MpDev te, int64_t base, MpDev tr, const float* __restrict__ ring_in,
                       float* __restrict__ ring_out, int64_t t0, int B, bool valid, int reseed) {
  __shared__ long long s_key[kStreamWarps][kStreamRC];
  __shared__ float s_row[kStreamRC][3];  // df_t, dg_t, inv_t (FP32, as the join's row records)
  const int g = blockIdx.y;
  const int64_t N = tr.n_sub;
  const int64_t t1 = t0 + B;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t delta0 = -(t1 - 1) + ((int64_t)blockIdx.x * kStreamThreads + threadIdx.x) * kStreamJ;
  const int m = te.m;
  const float* xr = static_cast<const float*>(te.R) + (int64_t)g * te.ld;
  const float* yr = static_cast<const float*>(tr.R) + (int64_t)g * tr.ld;
  const int64_t ot = (int64_t)g * te.ldq, oy = (int64_t)g * tr.ldq;
  const float4* q = static_cast<const float4*>(tr.Q) + oy;  // train records {df, dg, inv, 0}
  const float4* qt = static_cast<const float4*>(te.Q) + ot;  // test block records
  const long long kNone = pack_key(__int_as_float(0xff800000), 0xFFFFFFFFll);  // -inf, no index
  float cov[kStreamJ];
  bool have[kStreamJ];
#pragma unroll
  for (int d = 0; d < kStreamJ; ++d) {
    const int64_t delta = delta0 + d;
    const int64_t jp = t0 - 1 + delta;
    have[d] = valid && t0 > 0 && delta <= N - 1 - t0 && jp >= 0 && jp < N;
    cov[d] = have[d] ? ring_in[(int64_t)g * N + ((delta % N) + N) % N] : 0.0f;
  }
  int64_t* kg = te.keys + (int64_t)g * te.n_sub;
  float3 rec[kStreamJ];
  auto load_rec = [&](int64_t j) -> float3 {
    if (j < 0 || j >= N) return make_float3(0.f, 0.f, 0.f);
    const float4 v = q[j];
    return make_float3(v.x, v.y, v.z);
  };
#pragma unroll
  for (int d = 0; d < kStreamJ - 1; ++d) rec[d] = load_rec(t0 + delta0 + d);
  for (int64_t c0 = t0; c0 < t1; c0 += kStreamRC) {
    const int rc = (int)(t1 - c0 < kStreamRC ? t1 - c0 : kStreamRC);
    if (threadIdx.x < rc) {
      const float4 v = qt[c0 + threadIdx.x - base];
      s_row[threadIdx.x][0] = v.x;
      s_row[threadIdx.x][1] = v.y;
      s_row[threadIdx.x][2] = v.z;
    }
    __syncthreads();
    for (int r0 = 0; r0 < rc; r0 += kStreamJ) {
#pragma unroll
      for (int u = 0; u < kStreamJ; ++u) {
        const int r = r0 + u;
        if (r >= rc) break;  // CTA-uniform
        const int64_t t = c0 + r, l = t - base;
        rec[(u + kStreamJ - 1) % kStreamJ] = load_rec(t + delta0 + kStreamJ - 1);
        const float dft = s_row[r][0], dgt = s_row[r][1], invt = s_row[r][2];
        long long best = kNone;
#pragma unroll
        for (int d = 0; d < kStreamJ; ++d) {
          const int64_t j = t + delta0 + d;
          const float3 qj = rec[(u + d) % kStreamJ];
          if (j >= 0 && j < N) {
            if (!have[d] || j == 0 || (t & (reseed - 1)) == 0)
              cov[d] = (float)seed_cov<float>(xr + l, te.mu[ot + l], yr + j, tr.mu[oy + j], m);
            else
              cov[d] = fmaf(dft, qj.y, fmaf(qj.x, dgt, cov[d]));
            have[d] = true;
            best = max(best, pack_key((cov[d] * qj.z) * invt, j));
          } else {
            have[d] = false;
          }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, o));
        if (lane == 0) s_key[wid][r] = best;
      }
    }
    __syncthreads();
    if (threadIdx.x < rc) {
      long long best = s_key[0][threadIdx.x];
#pragma unroll
      for (int w = 1; w < kStreamWarps; ++w) best = max(best, s_key[w][threadIdx.x]);
      if (best != kNone) {
        const int64_t l = c0 + threadIdx.x - base;
        const float v = unord32((int32_t)(best >> 32));
        const int64_t j = (int64_t)(0xFFFFFFFFu - (uint32_t)(best & 0xFFFFFFFFll));
        if (v >= load_thr(kg, l, (float*)nullptr)) publish(kg, l, v, j);
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int d = 0; d < kStreamJ; ++d) {
    const int64_t delta = delta0 + d;
    if (have[d] && delta <= N - 1 - (t1 - 1)) ring_out[(int64_t)g * N + ((delta % N) + N) % N] = cov[d];
  }
}

// first group (+1) whose new sketch columns hold a NaN / Inf (a non-finite input propagates into
// its group's FP64 sum: NaN stays NaN, Inf stays Inf or meets -Inf as NaN)
__global__ void nonfinite_kernel(const double* __restrict__ R64, int64_t ld, int64_t col0, int64_t ncols,
                                 int32_t* __restrict__ flag) {
  const int g = blockIdx.y;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < ncols; t += (int64_t)gridDim.x * blockDim.x)
    if (!isfinite(R64[(int64_t)g * ld + col0 + t])) atomicMin(flag, g);
}

}  // namespace

cudaError_t launch_nonfinite_check(const double* R64, int64_t ld, int k, int64_t col0, int64_t ncols, int32_t* flag,
                                   cudaStream_t st) {
  const unsigned bx = (unsigned)((ncols + 255) / 256 < 64 ? (ncols + 255) / 256 : 64);
  nonfinite_kernel<<<dim3(bx, (unsigned)k), 256, 0, st>>>(R64, ld, col0, ncols, flag);
  count_launches(1);
  return cudaGetLastError();
}

size_t stream_q64_bytes(const MpDev& tr) { return sizeof(double4) * (size_t)tr.k * (size_t)tr.n_sub; }

cudaError_t launch_train_q64(const MpDev& tr, void* q64, cudaStream_t st) {
  dim3 grid((unsigned)((tr.n_sub + 255) / 256), (unsigned)tr.k);
  if (tr.dtype == SKMP_F32)
    train_q64_kernel<float><<<grid, 256, 0, st>>>(tr, static_cast<double4*>(q64));
  else
    train_q64_kernel<double><<<grid, 256, 0, st>>>(tr, static_cast<double4*>(q64));
  count_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_stream_rows(const MpDev& te, int64_t base, const MpDev& tr, const void* q64,
                               const double* ring_in, double* ring_out, int64_t t0, int B, bool valid,
                               cudaStream_t st) {
  const int64_t nd = tr.n_sub + B - 1;
  const int64_t per = (int64_t)kStreamThreads * kStreamJ;
  dim3 grid((unsigned)((nd + per - 1) / per), (unsigned)tr.k);
  const int reseed = kStreamReseed;
  if (te.dtype == SKMP_F32)
    stream_rows_f32_kernel<<<grid, kStreamThreads, 0, st>>>(te, base, tr, reinterpret_cast<const float*>(ring_in),
                                                            reinterpret_cast<float*>(ring_out), t0, B, valid, reseed);
  else
    stream_rows_kernel<double><<<grid, kStreamThreads, 0, st>>>(te, base, tr, static_cast<const double4*>(q64),
                                                                ring_in, ring_out, t0, B, valid, reseed);
  count_launches(1);
  return cudaGetLastError();
}

}  // namespace skmp

// Sketch kernels (K1 stream statistics, K2 count-sketch projection, K2d dense projection,
// K3 add/delete as K2 in accumulate mode).
//
// PAPER.md §3.1 Alg. 1: R^(g) = sum_{j in J_g} s(j) T_bar^(j), "basically just
// reading the input"; T_bar is the z-normalised input (reading 3: each stream's
// own mean and population std).  §3.3: the sketch is linear, so adding/deleting a
// dimension is R^(h(j)) +/- s(j) T_bar^(j).
//
// Both kernels are HBM-bound streaming passes over the d x n input: K1 reads T once to get
// (mu_j, 1/sigma_j), K2 reads it again and writes R.  Accumulation is FP64 in ascending input
// order inside each group with explicit _rn intrinsics (no FMA contraction), rounded once to
// the output dtype (reading 14).
#include <cuda_runtime.h>
#include <stdint.h>

#include "internal.h"

namespace skmp {

namespace {

constexpr int kStatsThreads = 256;
constexpr int kStatsChunk = 32768;  // samples per block (128 KB of FP32)

struct Partial {
  double cnt, mean, m2, amax;
};

template <typename T>
__device__ __forceinline__ void vload4(const T* p, double* out);
template <>
__device__ __forceinline__ void vload4<float>(const float* p, double* out) {
  const float4 f = __ldcs(reinterpret_cast<const float4*>(p));
  out[0] = f.x; out[1] = f.y; out[2] = f.z; out[3] = f.w;
}
template <>
__device__ __forceinline__ void vload4<double>(const double* p, double* out) {
  const double2 f = __ldcs(reinterpret_cast<const double2*>(p));
  out[0] = f.x; out[1] = f.y;
}

__device__ __forceinline__ double block_sum(double x, double* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = x;
  __syncthreads();
  double t = 0.0;
#pragma unroll
  for (int i = 0; i < kStatsThreads / 32; ++i) t += sh[i];  // fixed order: deterministic
  return t;
}

__device__ __forceinline__ double block_max(double x, double* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x = fmax(x, __shfl_xor_sync(0xffffffffu, x, o));
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = x;
  __syncthreads();
  double t = 0.0;
#pragma unroll
  for (int i = 0; i < kStatsThreads / 32; ++i) t = fmax(t, sh[i]);
  return t;
}

// K1a: per (stream, chunk) count, mean, M2, max|x|, finiteness.  A block streams a long chunk
// (kStatsChunk samples) with U independent 16-byte loads in flight per thread and accumulates
// shifted FP64 sums (x - K), (x - K)^2 with K = the chunk's first sample (the shift keeps the
// one-pass M2 = S2 - S1^2/n well conditioned); one block reduction per chunk.
template <typename T>
__global__ void __launch_bounds__(kStatsThreads)
stats_partial_kernel(const T* __restrict__ Tm, int64_t n, int64_t ld, int64_t nchunks,
                     Partial* __restrict__ part, int32_t* __restrict__ flag, bool vec) {
  __shared__ double sh[kStatsThreads / 32];
  constexpr int VN = (sizeof(T) == 4) ? 4 : 2;
  constexpr int U = (sizeof(T) == 4) ? 4 : 8;  // 16-byte loads in flight per thread
  const int64_t j = blockIdx.y;
  const int64_t c = blockIdx.x;
  const T* x = Tm + j * ld;
  const int64_t base = c * kStatsChunk;
  const int64_t end = (base + kStatsChunk < n) ? base + kStatsChunk : n;
  const double K = (double)x[base];
  double s1 = 0.0, s2 = 0.0, a = 0.0;
  bool finite = true;
  const int64_t step = (int64_t)kStatsThreads * VN;
  int64_t e = base + (int64_t)threadIdx.x * VN;
  if (vec) {
    for (; e + (U - 1) * step + VN <= end; e += U * step) {
      double v[U][VN];
#pragma unroll
      for (int u = 0; u < U; ++u) vload4<T>(x + e + u * step, v[u]);
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int q = 0; q < VN; ++q) {
          const double dv = v[u][q] - K;
          s1 += dv;
          s2 = fma(dv, dv, s2);
          a = fmax(a, fabs(v[u][q]));
          finite &= isfinite(v[u][q]);
        }
    }
  }
  for (; e < end; e += step) {  // tail (and the unaligned path) sample by sample
#pragma unroll
    for (int q = 0; q < VN; ++q) {
      if (e + q < end) {
        const double xv = (double)x[e + q];
        const double dv = xv - K;
        s1 += dv;
        s2 = fma(dv, dv, s2);
        a = fmax(a, fabs(xv));
        finite &= isfinite(xv);
      }
    }
  }
  if (!finite) atomicMax(flag + j, 1);
  s1 = block_sum(s1, sh);
  s2 = block_sum(s2, sh);
  a = block_max(a, sh);
  if (threadIdx.x == 0) {
    const double cnt = (double)(end - base);
    Partial p;
    p.cnt = cnt;
    p.mean = K + s1 / cnt;
    p.m2 = fmax(s2 - s1 * (s1 / cnt), 0.0);
    p.amax = a;
    part[j * nchunks + c] = p;
  }
}

// K1b: per stream, Chan's pairwise combine of the chunk partials in chunk order.
__global__ void stats_combine_kernel(const Partial* __restrict__ part, int64_t d, int64_t nchunks,
                                     StatsOut out) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= d) return;
  const Partial* p = part + j * nchunks;
  double na = p[0].cnt, mean = p[0].mean, m2 = p[0].m2, amax = p[0].amax;
  for (int64_t c = 1; c < nchunks; ++c) {
    const double nb = p[c].cnt;
    const double delta = p[c].mean - mean;
    const double nn = na + nb;
    mean += delta * (nb / nn);
    m2 += p[c].m2 + delta * delta * (na * nb / nn);
    amax = fmax(amax, p[c].amax);
    na = nn;
  }
  const double sigma = sqrt(m2 / na);
  out.mu[j] = mean;
  out.sigma[j] = sigma;
  int f = out.flag[j];
  if (f == 0 && !(sigma > kFlatEps * (amax + 1.0))) f = 2;  // reading 4: constant stream
  if (f == 0 && !isfinite(sigma)) f = 1;
  out.flag[j] = f;
  out.inv[j] = f == 0 ? 1.0 / sigma : 0.0;
}

// ------------------------------------------------------------------------------------------
// K2: count-sketch projection.  Block = (time tile, group g).  Each thread owns kVec*kIt
// consecutive-by-vector samples; the group's entry list is staged in shared memory in batches;
// four entries are in flight per step for memory-level parallelism.
// ------------------------------------------------------------------------------------------
constexpr int kProjThreads = 256;
constexpr int kProjBatch = 256;

template <typename T>
__device__ __forceinline__ void store_out(T* R, int64_t e, int64_t n, const double* v);
template <>
__device__ __forceinline__ void store_out<float>(float* R, int64_t e, int64_t n, const double* v) {
  if (e + 4 <= n && ((reinterpret_cast<uintptr_t>(R + e) & 15) == 0)) {
    *reinterpret_cast<float4*>(R + e) = make_float4((float)v[0], (float)v[1], (float)v[2], (float)v[3]);
  } else {
    for (int q = 0; q < 4; ++q) if (e + q < n) R[e + q] = (float)v[q];
  }
}
template <>
__device__ __forceinline__ void store_out<double>(double* R, int64_t e, int64_t n, const double* v) {
  if (e + 2 <= n && ((reinterpret_cast<uintptr_t>(R + e) & 15) == 0)) {
    *reinterpret_cast<double2*>(R + e) = make_double2(v[0], v[1]);
  } else {
    for (int q = 0; q < 2; ++q) if (e + q < n) R[e + q] = v[q];
  }
}

// raw 4-sample vector loads kept in the input precision until use
template <typename T> struct Raw4;
template <> struct Raw4<float> { float4 v; };
template <> struct Raw4<double> { double2 a, b; };
__device__ __forceinline__ void rload(Raw4<float>& r, const float* p, int64_t e, int64_t n, bool vec) {
  if (vec && e + 4 <= n) {
    r.v = __ldcs(reinterpret_cast<const float4*>(p + e));
  } else {
    r.v.x = (e + 0 < n) ? p[e + 0] : 0.f;
    r.v.y = (e + 1 < n) ? p[e + 1] : 0.f;
    r.v.z = (e + 2 < n) ? p[e + 2] : 0.f;
    r.v.w = (e + 3 < n) ? p[e + 3] : 0.f;
  }
}
__device__ __forceinline__ void rload(Raw4<double>& r, const double* p, int64_t e, int64_t n, bool vec) {
  if (vec && e + 4 <= n) {
    r.a = __ldcs(reinterpret_cast<const double2*>(p + e));
    r.b = __ldcs(reinterpret_cast<const double2*>(p + e + 2));
  } else {
    r.a.x = (e + 0 < n) ? p[e + 0] : 0.0;
    r.a.y = (e + 1 < n) ? p[e + 1] : 0.0;
    r.b.x = (e + 2 < n) ? p[e + 2] : 0.0;
    r.b.y = (e + 3 < n) ? p[e + 3] : 0.0;
  }
}
__device__ __forceinline__ double rget(const Raw4<float>& r, int q) {
  return q == 0 ? r.v.x : q == 1 ? r.v.y : q == 2 ? r.v.z : r.v.w;
}
__device__ __forceinline__ double rget(const Raw4<double>& r, int q) {
  return q == 0 ? r.a.x : q == 1 ? r.a.y : q == 2 ? r.b.x : r.b.y;
}

// K2: count-sketch projection.  Block = (1024-sample time tile, group g); thread = 4 consecutive
// samples; the group's entries (row, mu, 1/sigma, sign) are staged in shared memory and U streams
// are loaded per step (U x 16-32 B in flight per thread) before the FP64 accumulation, which runs
// in ascending input order with explicit _rn operations (no contraction).
template <typename T>
__global__ void __launch_bounds__(kProjThreads)
project_count_kernel(const T* __restrict__ Tm, int64_t ld, int64_t n, CsrPlan plan, int mode,
                     double* __restrict__ R64, T* __restrict__ R, int64_t ldr, bool vec) {
  constexpr int U = 8;
  __shared__ int32_t s_row[kProjBatch];
  __shared__ double s_mu[kProjBatch];
  __shared__ double s_inv[kProjBatch];
  __shared__ int8_t s_sign[kProjBatch];

  const int g = blockIdx.y;
  const int32_t e0 = plan.off[g], e1 = plan.off[g + 1];
  if (mode != 0 && e0 == e1) return;  // update of an untouched group: nothing to do
  const int64_t e = ((int64_t)blockIdx.x * kProjThreads + threadIdx.x) * 4;
  double* r64 = R64 + (int64_t)g * ldr;
  double acc[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) acc[q] = (mode != 0 && e + q < n) ? r64[e + q] : 0.0;

  for (int32_t b0 = e0; b0 < e1; b0 += kProjBatch) {
    const int nb = min(kProjBatch, e1 - b0);
    __syncthreads();
    if (threadIdx.x < nb) {
      s_row[threadIdx.x] = plan.row[b0 + threadIdx.x];
      s_mu[threadIdx.x] = plan.mu[b0 + threadIdx.x];
      s_inv[threadIdx.x] = plan.inv[b0 + threadIdx.x];
      s_sign[threadIdx.x] = plan.sign[b0 + threadIdx.x];
    }
    __syncthreads();
    int q0 = 0;
    for (; q0 + U <= nb; q0 += U) {
      Raw4<T> x[U];
#pragma unroll
      for (int u = 0; u < U; ++u) rload(x[u], Tm + (int64_t)s_row[q0 + u] * ld, e, n, vec);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const double mu = s_mu[q0 + u], inv = s_inv[q0 + u];
        const bool pos = (s_sign[q0 + u] > 0) == (mode >= 0);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const double z = __dmul_rn(__dsub_rn(rget(x[u], q), mu), inv);
          acc[q] = pos ? __dadd_rn(acc[q], z) : __dsub_rn(acc[q], z);
        }
      }
    }
    for (; q0 < nb; ++q0) {
      Raw4<T> x;
      rload(x, Tm + (int64_t)s_row[q0] * ld, e, n, vec);
      const double mu = s_mu[q0], inv = s_inv[q0];
      const bool pos = (s_sign[q0] > 0) == (mode >= 0);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const double z = __dmul_rn(__dsub_rn(rget(x, q), mu), inv);
        acc[q] = pos ? __dadd_rn(acc[q], z) : __dsub_rn(acc[q], z);
      }
    }
  }
  store_out<double>(r64, e, n, &acc[0]);
  store_out<double>(r64, e + 2, n, &acc[2]);
  if ((void*)R != (void*)R64) {
    if constexpr (sizeof(T) == 4) store_out<float>(reinterpret_cast<float*>(R) + (int64_t)g * ldr, e, n, acc);
  }
}

// K2d: dense projection, 8 groups per block, one sample per thread (small configs only).
constexpr int kDenseG = 8;
template <typename T>
__global__ void project_dense_kernel(const T* __restrict__ Tm, int64_t ld, int64_t n, int k,
                                     int64_t nstreams, const double* __restrict__ S, int64_t ldS,
                                     const double* __restrict__ mu, const double* __restrict__ inv,
                                     int mode, double* __restrict__ R64, T* __restrict__ R, int64_t ldr) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int g0 = blockIdx.y * kDenseG;
  if (t >= n) return;
  double acc[kDenseG];
#pragma unroll
  for (int q = 0; q < kDenseG; ++q)
    acc[q] = (mode != 0 && g0 + q < k) ? R64[(int64_t)(g0 + q) * ldr + t] : 0.0;
  for (int64_t j = 0; j < nstreams; ++j) {
    const double z = __dmul_rn(__dsub_rn((double)Tm[j * ld + t], mu[j]), inv[j]);
#pragma unroll
    for (int q = 0; q < kDenseG; ++q) {
      if (g0 + q < k) {
        const double c = __dmul_rn(S[(int64_t)(g0 + q) * ldS + j], z);
        acc[q] = mode >= 0 ? __dadd_rn(acc[q], c) : __dsub_rn(acc[q], c);
      }
    }
  }
#pragma unroll
  for (int q = 0; q < kDenseG; ++q) {
    if (g0 + q < k) {
      R64[(int64_t)(g0 + q) * ldr + t] = acc[q];
      if ((void*)R != (void*)R64) R[(int64_t)(g0 + q) * ldr + t] = (T)acc[q];
    }
  }
}

// §3.3 point updates: R64[idx[q]] += coef[q] * delta[q] (FP64 atomics: several updates may hit
// one entry), then the touched entries are re-rounded to the dtype copy.
__global__ void point_add_kernel(double* __restrict__ R64, const int64_t* __restrict__ idx,
                                 const double* __restrict__ coef, const double* __restrict__ delta,
                                 int64_t count) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q < count) atomicAdd(R64 + idx[q], __dmul_rn(coef[q], delta[q]));
}
__global__ void point_cast_kernel(const double* __restrict__ R64, float* __restrict__ R,
                                  const int64_t* __restrict__ idx, int64_t count) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q < count) R[idx[q]] = (float)R64[idx[q]];
}

__global__ void cast_kernel(const double* __restrict__ a, float* __restrict__ b, int64_t count) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x)
    b[i] = (float)a[i];
}

}  // namespace

cudaError_t launch_cast_r(const double* R64, void* R, int64_t count, int dtype, cudaStream_t st) {
  if (dtype != SKMP_F32) return cudaSuccess;
  const int64_t blocks = (count + 255) / 256;
  cast_kernel<<<(unsigned)(blocks < 148 * 32 ? blocks : 148 * 32), 256, 0, st>>>(R64, static_cast<float*>(R), count);
  count_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_point_update(double* R64, void* R, int dtype, const int64_t* idx, const double* coef,
                                const double* delta, int64_t count, cudaStream_t st) {
  if (count <= 0) return cudaSuccess;
  const unsigned blocks = (unsigned)((count + 255) / 256);
  point_add_kernel<<<blocks, 256, 0, st>>>(R64, idx, coef, delta, count);
  count_launches(1);
  if (dtype == SKMP_F32) {
    point_cast_kernel<<<blocks, 256, 0, st>>>(R64, static_cast<float*>(R), idx, count);
    count_launches(1);
  }
  return cudaGetLastError();
}

size_t stats_ws_bytes(int64_t d, int64_t n) {
  const int64_t nchunks = (n + kStatsChunk - 1) / kStatsChunk;
  return sizeof(Partial) * (size_t)(d * nchunks);
}

cudaError_t launch_stream_stats(const void* T, int64_t d, int64_t n, int64_t ld, int dtype,
                                StatsOut out, void* ws, cudaStream_t st) {
  const int64_t nchunks = (n + kStatsChunk - 1) / kStatsChunk;
  cudaError_t e = cudaMemsetAsync(out.flag, 0, sizeof(int32_t) * d, st);
  if (e != cudaSuccess) return e;
  int64_t left = d;
  int64_t off = 0;
  while (left > 0) {  // grid.y <= 65535
    const int64_t dd = left < 65535 ? left : 65535;
    dim3 grid((unsigned)nchunks, (unsigned)dd);
    if (dtype == SKMP_F32) {
      const float* p = static_cast<const float*>(T) + off * ld;
      const bool vec = ((reinterpret_cast<uintptr_t>(p) & 15) == 0) && (ld % 4 == 0);
      stats_partial_kernel<float><<<grid, kStatsThreads, 0, st>>>(
          p, n, ld, nchunks, static_cast<Partial*>(ws) + off * nchunks, out.flag + off, vec);
    } else {
      const double* p = static_cast<const double*>(T) + off * ld;
      const bool vec = ((reinterpret_cast<uintptr_t>(p) & 15) == 0) && (ld % 2 == 0);
      stats_partial_kernel<double><<<grid, kStatsThreads, 0, st>>>(
          p, n, ld, nchunks, static_cast<Partial*>(ws) + off * nchunks, out.flag + off, vec);
    }
    left -= dd;
    off += dd;
  }
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  count_launches((d + 65534) / 65535 + 1);
  stats_combine_kernel<<<(unsigned)((d + 127) / 128), 128, 0, st>>>(static_cast<Partial*>(ws), d,
                                                                   nchunks, out);
  return cudaGetLastError();
}

cudaError_t launch_project_count(const void* T, int64_t ld, int64_t n, int dtype, int k,
                                 CsrPlan plan, int mode, double* R64, void* R, int64_t ldr, cudaStream_t st) {
  if (dtype == SKMP_F32) {
    const int64_t tile = (int64_t)kProjThreads * 4;
    dim3 grid((unsigned)((n + tile - 1) / tile), (unsigned)k);
    const bool vec = ((reinterpret_cast<uintptr_t>(T) & 15) == 0) && (ld % 4 == 0);
    project_count_kernel<float><<<grid, kProjThreads, 0, st>>>(
        static_cast<const float*>(T), ld, n, plan, mode, R64, static_cast<float*>(R), ldr, vec);
  } else {
    const int64_t tile = (int64_t)kProjThreads * 4;
    dim3 grid((unsigned)((n + tile - 1) / tile), (unsigned)k);
    const bool vec = ((reinterpret_cast<uintptr_t>(T) & 15) == 0) && (ld % 2 == 0);
    project_count_kernel<double><<<grid, kProjThreads, 0, st>>>(
        static_cast<const double*>(T), ld, n, plan, mode, R64, static_cast<double*>(R), ldr, vec);
  }
  count_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_project_dense(const void* T, int64_t ld, int64_t n, int dtype, int k,
                                 int64_t nstreams, const double* S, int64_t ldS, const double* mu,
                                 const double* inv, int mode, double* R64, void* R, int64_t ldr,
                                 cudaStream_t st) {
  dim3 grid((unsigned)((n + 255) / 256), (unsigned)((k + kDenseG - 1) / kDenseG));
  if (dtype == SKMP_F32)
    project_dense_kernel<float><<<grid, 256, 0, st>>>(static_cast<const float*>(T), ld, n, k,
                                                      nstreams, S, ldS, mu, inv, mode, R64,
                                                      static_cast<float*>(R), ldr);
  else
    project_dense_kernel<double><<<grid, 256, 0, st>>>(static_cast<const double*>(T), ld, n, k,
                                                       nstreams, S, ldS, mu, inv, mode, R64,
                                                       static_cast<double*>(R), ldr);
  count_launches(1);
  return cudaGetLastError();
}

}  // namespace skmp

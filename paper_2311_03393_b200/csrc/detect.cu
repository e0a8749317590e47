// K8: discord detection over the sketch profiles.
//  * combine — Alg. 2 Time-Detection generalised to the whole profile:
//    C[i] = max_{g not inert} P_g[i], G[i] = smallest maximising g (strict '>' over ascending g,
//    P:L262).  Inert groups (reading 6) are excluded.
//  * top-K — the ordered discord list "from large to small" (reading 12):
//    greedy smallest-index argmax over unmasked windows, then mask [t - radius, t + radius].
//    One launch per emitted discord: a grid-wide argmax whose last CTA (ticket counter)
//    reduces the per-CTA partials, emits the tuple and masks the radius.
#include <cuda_runtime.h>
#include <stdint.h>

#include "internal.h"

namespace skmp {
namespace {

template <typename T>
__global__ void combine_kernel(const T* __restrict__ P, int64_t ldp, int k, int64_t n_sub,
                               const uint8_t* __restrict__ inert, double* __restrict__ C,
                               int32_t* __restrict__ G) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_sub) return;
  double best = __longlong_as_double(0xfff0000000000000ll);
  int32_t bg = -1;
  for (int g = 0; g < k; ++g) {
    if (inert && inert[g]) continue;
    const double v = (double)P[(int64_t)g * ldp + i];
    if (v > best) {
      best = v;
      bg = g;
    }
  }
  C[i] = best;
  G[i] = bg;
}

constexpr int kTopThreads = 256;
constexpr int kTopBlocks = 296;

struct Cand {
  double v;
  int64_t i;
};
__device__ __forceinline__ bool better(double v, int64_t i, double bv, int64_t bi) {
  return v > bv || (v == bv && i < bi);
}

__global__ void __launch_bounds__(kTopThreads)
topk_iter_kernel(double* __restrict__ C, const int32_t* __restrict__ G,
                 const int64_t* __restrict__ I, int64_t ldi, int64_t n_sub, int radius,
                 int64_t* __restrict__ res, int32_t* __restrict__ count, Cand* __restrict__ part,
                 unsigned* __restrict__ ticket, int q) {
  __shared__ double sv[kTopThreads / 32];
  __shared__ int64_t si[kTopThreads / 32];
  __shared__ bool last;
  if (*count < q) return;  // an earlier iteration found nothing left
  const double NEG = __longlong_as_double(0xfff0000000000000ll);
  double bv = NEG;
  int64_t bi = INT64_MAX;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_sub;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double v = C[i];
    if (better(v, i, bv, bi)) { bv = v; bi = i; }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
    const int64_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (better(ov, oi, bv, bi)) { bv = ov; bi = oi; }
  }
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) { sv[wid] = bv; si[wid] = bi; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < kTopThreads / 32; ++w)
      if (better(sv[w], si[w], sv[0], si[0])) { sv[0] = sv[w]; si[0] = si[w]; }
    part[blockIdx.x] = Cand{sv[0], si[0]};
    __threadfence();
    const unsigned t = atomicAdd(ticket, 1u);
    last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  // last CTA: reduce partials, emit, mask
  bv = NEG;
  bi = INT64_MAX;
  for (int b = threadIdx.x; b < gridDim.x; b += blockDim.x) {
    const Cand c = part[b];
    if (better(c.v, c.i, bv, bi)) { bv = c.v; bi = c.i; }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
    const int64_t oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (better(ov, oi, bv, bi)) { bv = ov; bi = oi; }
  }
  if (lane == 0) { sv[wid] = bv; si[wid] = bi; }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < kTopThreads / 32; ++w)
      if (better(sv[w], si[w], sv[0], si[0])) { sv[0] = sv[w]; si[0] = si[w]; }
    *ticket = 0;
  }
  __syncthreads();
  const double v = sv[0];
  const int64_t t = si[0];
  if (!(v > NEG) || t == INT64_MAX) return;  // everything masked: count stays at q
  if (threadIdx.x == 0) {
    const int g = G[t];
    res[4 * q + 0] = t;
    res[4 * q + 1] = g;
    res[4 * q + 2] = I[(int64_t)g * ldi + t];
    res[4 * q + 3] = __double_as_longlong(v);
    *count = q + 1;
  }
  const int64_t lo = t - radius < 0 ? 0 : t - radius;
  const int64_t hi = t + radius + 1 < n_sub ? t + radius + 1 : n_sub;
  for (int64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) C[i] = NEG;
}

}  // namespace

cudaError_t launch_combine(const void* P, int64_t ldp, int k, int64_t n_sub, int dtype,
                           const uint8_t* d_inert, double* C, int32_t* G, cudaStream_t st) {
  const unsigned blocks = (unsigned)((n_sub + 255) / 256);
  if (dtype == SKMP_F32)
    combine_kernel<float><<<blocks, 256, 0, st>>>(static_cast<const float*>(P), ldp, k, n_sub, d_inert, C, G);
  else
    combine_kernel<double><<<blocks, 256, 0, st>>>(static_cast<const double*>(P), ldp, k, n_sub, d_inert, C, G);
  count_launches(1);
  return cudaGetLastError();
}

size_t topk_ws_bytes(int64_t) { return sizeof(Cand) * kTopBlocks + 64; }

cudaError_t launch_topk(double* C, const int32_t* G, const int64_t* I, int64_t ldi, int64_t n_sub,
                        int top, int radius, int64_t* d_res, int32_t* d_count, void* ws,
                        size_t ws_bytes, cudaStream_t st) {
  (void)ws_bytes;
  Cand* part = static_cast<Cand*>(ws);
  unsigned* ticket = reinterpret_cast<unsigned*>(part + kTopBlocks);
  cudaError_t e = cudaMemsetAsync(ticket, 0, sizeof(unsigned), st);
  if (e) return e;
  e = cudaMemsetAsync(d_count, 0, sizeof(int32_t), st);
  if (e) return e;
  int64_t blocks = (n_sub + kTopThreads - 1) / kTopThreads;
  if (blocks > kTopBlocks) blocks = kTopBlocks;
  for (int q = 0; q < top; ++q) {
    topk_iter_kernel<<<(unsigned)blocks, kTopThreads, 0, st>>>(C, G, I, ldi, n_sub, radius, d_res,
                                                               d_count, part, ticket, q);
  }
  count_launches(top);
  return cudaGetLastError();
}

}  // namespace skmp

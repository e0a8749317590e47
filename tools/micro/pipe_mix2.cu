// Microbenchmark (round 1e): which max instructions overlap with packed FP32 FMAs on B200?
// The join needs ~1 FMNMX3 per cell beside 1 FFMA2 + 1 FMUL2; pipe_mix.cu showed
// FFMA2 + FMNMX3 do not overlap.  Here: integer / packed-integer / packed-half maxima next to FFMA2.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipe_mix2 pipe_mix2.cu && ./pipe_mix2
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long f2;
__device__ __forceinline__ f2 fma2(f2 a, f2 b, f2 c) {
  f2 d;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ float max3(float a, float b, float c) {
  float r;
  asm volatile("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
__device__ __forceinline__ float fmax2(float a, float b) {
  float r;
  asm volatile("max.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ int imax(int a, int b) {
  int r;
  asm volatile("max.s32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}
__device__ __forceinline__ int imax3(int a, int b, int c) {  // ptxas may fuse to VIMNMX3
  int r;
  asm volatile("{ .reg .s32 t; max.s32 t, %1, %2; max.s32 %0, t, %3; }" : "=r"(r) : "r"(a), "r"(b), "r"(c));
  return r;
}
__device__ __forceinline__ unsigned hmax2(unsigned a, unsigned b) {
  unsigned r;
  asm volatile("max.f16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}
__device__ __forceinline__ unsigned smax2(unsigned a, unsigned b) {
  unsigned r;
  asm volatile("max.s16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}
__device__ __forceinline__ f2 pk(float a, float b) {
  f2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float lo(f2 v) {
  float a, b;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
  return a;
}

template <int MODE> struct Cnt { static constexpr int n = 16; };
template <> struct Cnt<0> { static constexpr int n = 8; };
template <> struct Cnt<1> { static constexpr int n = 8; };
template <> struct Cnt<2> { static constexpr int n = 8; };
template <> struct Cnt<3> { static constexpr int n = 8; };
template <> struct Cnt<4> { static constexpr int n = 8; };

template <int MODE>
__global__ void k(float* out, float s, int iters) {
  float a[8], b[8], c[8];
  int ia[8], ib[8];
  unsigned ha[8], hb[8];
  f2 A[8], B[8], Cc[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    a[q] = s * (q + 1);
    b[q] = s * (q + 3);
    c[q] = threadIdx.x * s + q;
    ia[q] = __float_as_int(a[q]) + threadIdx.x;
    ib[q] = __float_as_int(b[q]) ^ q;
    ha[q] = 0x3c003c00u + q + threadIdx.x;
    hb[q] = 0x3c013c02u ^ q;
    A[q] = pk(a[q], b[q]);
    B[q] = pk(b[q], a[q]);
    Cc[q] = pk(c[q], c[q] + 1);
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      if (MODE == 0) Cc[q] = fma2(A[0], B[q], Cc[q]);                          // FFMA2 alone
      else if (MODE == 1) ia[q] = imax(ia[q], ib[q]);                          // IMNMX alone
      else if (MODE == 2) ia[q] = imax3(ia[q], ib[q], ia[(q + 1) & 7]);        // 3-input int max alone
      else if (MODE == 3) ha[q] = hmax2(ha[q], hb[q]);                         // HMNMX2 alone
      else if (MODE == 4) ha[q] = smax2(ha[q], hb[q]);                         // VIMNMX.S16x2 alone
      else if (MODE == 5) { Cc[q] = fma2(A[0], B[q], Cc[q]); ia[q] = imax(ia[q], ib[q]); }
      else if (MODE == 6) { Cc[q] = fma2(A[0], B[q], Cc[q]); ia[q] = imax3(ia[q], ib[q], ia[(q + 1) & 7]); }
      else if (MODE == 7) { Cc[q] = fma2(A[0], B[q], Cc[q]); ha[q] = hmax2(ha[q], hb[q]); }
      else if (MODE == 8) { Cc[q] = fma2(A[0], B[q], Cc[q]); ha[q] = smax2(ha[q], hb[q]); }
      else if (MODE == 9) { Cc[q] = fma2(A[0], B[q], Cc[q]); c[q] = fmax2(c[q], b[q]); }
      else if (MODE == 10) { Cc[q] = fma2(A[0], B[q], Cc[q]); c[q] = max3(c[q], a[q], b[q]); }
      else if (MODE == 11) { c[q] = fmaf(a[0], b[q], c[q]); ia[q] = imax3(ia[q], ib[q], ia[(q + 1) & 7]); }
    }
  }
  float t = 0.f;
  for (int q = 0; q < 8; ++q) t += c[q] + b[q] + lo(Cc[q]) + (float)ia[q] + (float)ha[q];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
template <int MODE>
void run(float* d, int iters, const char* name) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k<MODE><<<148 * 8, 256>>>(d, 1.0001f, iters);
  cudaEventRecord(e0);
  k<MODE><<<148 * 8, 256>>>(d, 1.0001f, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double instr = 148.0 * 8 * 256 / 32 * iters * Cnt<MODE>::n;
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double cyc = ms * 1e-3 * clk * 1e3;
  printf("mode %2d %-34s %.3f ms  %.3f warp-instr / clk / SMSP\n", MODE, name, ms, instr / (cyc * 148 * 4));
}
int main() {
  float* d;
  cudaMalloc(&d, 148 * 8 * 256 * 4);
  const int it = 20000;
  run<0>(d, it, "FFMA2 (shared pair)");
  run<1>(d, it, "IMNMX");
  run<2>(d, it, "int max3 (2 x max.s32)");
  run<3>(d, it, "HMNMX2 (max.f16x2)");
  run<4>(d, it, "VIMNMX.S16x2 (max.s16x2)");
  run<5>(d, it, "FFMA2 + IMNMX 1:1");
  run<6>(d, it, "FFMA2 + int max3 1:1");
  run<7>(d, it, "FFMA2 + HMNMX2 1:1");
  run<8>(d, it, "FFMA2 + max.s16x2 1:1");
  run<9>(d, it, "FFMA2 + FMNMX 1:1");
  run<10>(d, it, "FFMA2 + FMNMX3 1:1");
  run<11>(d, it, "FFMA + int max3 1:1");
  return 0;
}

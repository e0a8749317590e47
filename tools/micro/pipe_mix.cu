// Microbenchmark: B200 issue rates of the join's instruction mix (per SMSP per clock).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipe_mix pipe_mix.cu && ./pipe_mix
// Each mode runs 8 independent chains per thread, 148*8 CTAs x 256 threads.
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long f2;
__device__ __forceinline__ f2 fma2(f2 a, f2 b, f2 c) {
  f2 d;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ f2 mul2(f2 a, f2 b) {
  f2 d;
  asm volatile("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ float max3(float a, float b, float c) {
  float r;
  asm volatile("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
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
__device__ __forceinline__ float hi(f2 v) {
  float a, b;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
  return b;
}

// instructions per inner iteration (per thread) for the rate computation
template <int MODE> struct Cnt { static constexpr int n = 8; };
template <> struct Cnt<6> { static constexpr int n = 16; };
template <> struct Cnt<7> { static constexpr int n = 16; };
template <> struct Cnt<8> { static constexpr int n = 8 * 4 + 8; };

template <int MODE>
__global__ void k(float* out, float s, int iters) {
  float a[8], b[8], c[8];
  f2 A[8], B[8], Cc[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    a[q] = s * (q + 1);
    b[q] = s * (q + 3);
    c[q] = threadIdx.x * s + q;
    A[q] = pk(a[q], b[q]);
    B[q] = pk(b[q], a[q]);
    Cc[q] = pk(c[q], c[q] + 1);
  }
  float m = -1e30f, m2 = -1e30f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      if (MODE == 0) c[q] = fmaf(a[q], b[q], c[q]);                 // FFMA 3 distinct regs
      else if (MODE == 1) c[q] = fmaf(a[0], b[q], c[q]);            // FFMA, shared operand
      else if (MODE == 2) Cc[q] = fma2(A[q], B[q], Cc[q]);          // FFMA2 3 distinct pairs
      else if (MODE == 3) Cc[q] = fma2(A[0], B[q], Cc[q]);          // FFMA2 shared pair
      else if (MODE == 4) Cc[q] = mul2(Cc[q], B[q]);                // FMUL2
      else if (MODE == 5) c[q] = max3(c[q], a[q], b[q]);            // FMNMX3 (ALU)
      else if (MODE == 6) {                                         // FFMA2 + FMNMX3 1:1
        Cc[q] = fma2(A[0], B[q], Cc[q]);
        c[q] = max3(c[q], a[q], b[q]);
      } else if (MODE == 7) {                                       // FFMA + FMNMX3 1:1
        c[q] = fmaf(a[0], b[q], c[q]);
        b[q] = max3(b[q], a[q], c[q]);
      } else if (MODE == 8) {
        // one x2 "row" of the join for 2 cells per slot: 2 FFMA2 + 2 FMUL2 + ~1 FMNMX3 per 2 cells
        Cc[q] = fma2(A[0], B[q], Cc[q]);
        Cc[q] = fma2(B[0], A[q], Cc[q]);
        const f2 r = mul2(mul2(Cc[q], A[(q + 1) & 7]), B[1]);
        m = max3(m, lo(r), hi(r));
      }
    }
  }
  float t = m + m2;
  for (int q = 0; q < 8; ++q) t += c[q] + b[q] + lo(Cc[q]) + hi(Cc[q]);
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
  printf("mode %d %-36s %.3f ms  %.3f warp-instr / clk / SMSP\n", MODE, name, ms, instr / (cyc * 148 * 4));
}
int main() {
  float* d;
  cudaMalloc(&d, 148 * 8 * 256 * 4);
  const int it = 20000;
  run<0>(d, it, "FFMA 3 distinct");
  run<1>(d, it, "FFMA shared operand");
  run<2>(d, it, "FFMA2 3 distinct pairs");
  run<3>(d, it, "FFMA2 shared pair");
  run<4>(d, it, "FMUL2");
  run<5>(d, it, "FMNMX3");
  run<6>(d, it, "FFMA2 + FMNMX3 (1:1)");
  run<7>(d, it, "FFMA + FMNMX3 (1:1)");
  run<8>(d, it, "x2 cell mix (2 FFMA2, 2 FMUL2, FMNMX3 + movs)");
  return 0;
}

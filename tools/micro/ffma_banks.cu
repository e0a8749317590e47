// Microbenchmark: FFMA issue rate on B200 for different operand patterns (register-bank study).
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(float* out, float s, int iters) {
  float a[8], b[8], c[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) { a[q] = s * (q + 1); b[q] = s * (q + 3); c[q] = threadIdx.x * s + q; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      if (MODE == 0) c[q] = fmaf(a[q], b[q], c[q]);          // 3 distinct registers
      else if (MODE == 1) c[q] = fmaf(a[0], b[q], c[q]);     // one shared operand (reuse)
      else if (MODE == 2) c[q] = fmaf(c[q], 1.0001f, 0.5f);  // 1 register + immediates
      else c[q] = c[q] * b[q];                                // FMUL 2 regs
    }
  }
  float t = 0; for (int q = 0; q < 8; ++q) t += c[q];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
template <int MODE> float run(float* d, int iters) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<MODE><<<148 * 8, 256>>>(d, 1.0001f, iters);
  cudaEventRecord(e0); k<MODE><<<148 * 8, 256>>>(d, 1.0001f, iters); cudaEventRecord(e1);
  cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1);
  double instr = 148.0 * 8 * 256 / 32 * iters * 8;  // warp-instructions (FP only)
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double cyc = ms * 1e-3 * clk * 1e3;
  printf("mode %d: %.3f ms, %.3f FP warp-instr / clk / SMSP\n", MODE, ms, instr / (cyc * 148 * 4));
  return ms;
}
int main() {
  float* d; cudaMalloc(&d, 148 * 8 * 256 * 4);
  int iters = 20000;
  run<0>(d, iters); run<1>(d, iters); run<2>(d, iters); run<3>(d, iters);
  return 0;
}

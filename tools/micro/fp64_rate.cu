// Microbenchmark: B200 FP64 / conversion issue rates (per SMSP per clock).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_rate fp64_rate.cu && ./fp64_rate
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(double* out, float* fout, double s, int iters) {
  double a[8], c[8];
  float f[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    a[q] = s * (q + 1);
    c[q] = threadIdx.x * s + q;
    f[q] = (float)(s * q + threadIdx.x);
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      if (MODE == 0) c[q] = fma(a[q], c[q], a[(q + 1) & 7]);      // DFMA
      else if (MODE == 1) c[q] = c[q] + a[q];                      // DADD
      else if (MODE == 2) c[q] = c[q] + (double)f[q];              // F2F.F64.F32 + DADD
      else if (MODE == 3) f[q] = (float)(c[q] * a[q]);             // DMUL + F2F.F32.F64
    }
    if (MODE == 2) {
#pragma unroll
      for (int q = 0; q < 8; ++q) f[q] += 1.0f;
    }
    if (MODE == 3) {
#pragma unroll
      for (int q = 0; q < 8; ++q) c[q] += f[q];
    }
  }
  double t = 0;
  for (int q = 0; q < 8; ++q) t += c[q] + f[q];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
template <int MODE>
void run(double* d, float* f, int iters, const char* name, int per_iter) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k<MODE><<<148 * 8, 256>>>(d, f, 1.0000001, iters);
  cudaEventRecord(e0);
  k<MODE><<<148 * 8, 256>>>(d, f, 1.0000001, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double instr = 148.0 * 8 * 256 / 32 * iters * per_iter;
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double cyc = ms * 1e-3 * clk * 1e3;
  printf("mode %d %-34s %.3f ms  %.4f warp-instr / clk / SMSP  (%.1f lane-ops / clk / SM)\n", MODE, name, ms,
         instr / (cyc * 148 * 4), instr * 32 / (cyc * 148));
}
int main() {
  double* d;
  float* f;
  cudaMalloc(&d, 148 * 8 * 256 * 8);
  cudaMalloc(&f, 148 * 8 * 256 * 4);
  const int it = 4000;
  run<0>(d, f, it, "DFMA", 8);
  run<1>(d, f, it, "DADD", 8);
  run<2>(d, f, it, "F2F.F64.F32 + DADD (counted: 16)", 16);
  run<3>(d, f, it, "DMUL + F2F.F32.F64 (counted: 16)", 16);
  return 0;
}

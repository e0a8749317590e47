// Microbenchmark: the join's per-cell arithmetic + row/column maxima with NO memory traffic, no
// threshold checks and no loop bookkeeping beyond the rotation — the ceiling of the instruction
// mix alone (scalar FP32: 2 FFMA + 2 FMUL + FMNMX3 trees; packed: 2 FFMA2 + 2 FMUL2 per two cells).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o cell_mix cell_mix.cu && ./cell_mix
#include <cstdio>
#include <cuda_runtime.h>

constexpr int D = 8;
__device__ __forceinline__ float max3(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
__device__ __forceinline__ float tree8(const float* v) {
  return max3(max3(v[0], v[1], v[2]), max3(v[3], v[4], v[5]), fmaxf(v[6], v[7]));
}
typedef unsigned long long f2;
__device__ __forceinline__ f2 fma2(f2 a, f2 b, f2 c) {
  f2 d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ f2 mul2(f2 a, f2 b) {
  f2 d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ f2 pk(float a, float b) {
  f2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void unpk(f2 v, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}

__device__ __forceinline__ int imax3(int a, int b, int c) {  // ptxas fuses to VIMNMX3
  int r;
  asm("{ .reg .s32 t; max.s32 t, %1, %2; max.s32 %0, t, %3; }" : "=r"(r) : "r"(a), "r"(b), "r"(c));
  return r;
}
__device__ __forceinline__ int imax(int a, int b) { return a > b ? a : b; }
__device__ __forceinline__ int itree8(const int* v) {
  return imax3(imax3(v[0], v[1], v[2]), imax3(v[3], v[4], v[5]), imax(v[6], v[7]));
}

// scalar with integer maxima: the cell value is rho + 1 >= 0 (one FFMA instead of the last
// FMUL), whose bit pattern orders like an int, so the row/column maxima are VIMNMX3 on the
// ALU pipe, which (pipe_mix2.cu) overlaps with scalar FFMA
__global__ void scalar_int_kernel(float* out, float s0, int rots) {
  const float s = s0 + threadIdx.x * 1e-6f;
  float cov[D], xx[D], xy[D], xz[D];
  int CK[D];
#pragma unroll
  for (int d = 0; d < D; ++d) {
    cov[d] = s * d;
    xx[d] = s + d * 1e-3f;
    xy[d] = s - d * 1e-3f;
    xz[d] = s * (0.3f + 0.01f * d);
    CK[d] = 0;
  }
  float ra = threadIdx.x * 1e-6f, rb = s * 0.9f, rc = s * 0.7f;
  int sink = 0;
  for (int it = 0; it < rots; ++it) {
#pragma unroll
    for (int u = 0; u < D; u += 2) {
      int ka[D], kb[D];
#pragma unroll
      for (int d = 0; d < D; ++d) {
        const int x = (u + d) % D;
        cov[d] = fmaf(ra, xy[x], cov[d]);
        cov[d] = fmaf(xx[x], rb, cov[d]);
        ka[d] = __float_as_int(fmaf(cov[d] * xz[x], rc, 1.0f));
      }
#pragma unroll
      for (int d = 0; d < D; ++d) {
        const int x = (u + 1 + d) % D;
        cov[d] = fmaf(rb, xy[x], cov[d]);
        cov[d] = fmaf(xx[x], ra, cov[d]);
        kb[d] = __float_as_int(fmaf(cov[d] * xz[x], rc, 1.0f));
      }
      const int c0 = imax(CK[u % D], ka[0]);
      const int c1 = imax3(CK[(u + 1) % D], ka[1], kb[0]);
#pragma unroll
      for (int d = 2; d < D - 1; ++d) CK[(u + d) % D] = imax3(CK[(u + d) % D], ka[d], kb[d - 1]);
      CK[(u + D - 1) % D] = imax(ka[D - 1], kb[D - 2]);
      CK[u % D] = kb[D - 1];
      sink = imax3(sink, itree8(ka), itree8(kb));
      sink = imax3(sink, c0, c1);
      ra += 1e-7f;
      rc += 1e-9f;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = __int_as_float(sink) + __int_as_float(CK[0]);
}

// scalar: D slots, rows in pairs, columns rotate through registers as in mp_join.cu
__global__ void scalar_kernel(float* out, float s0, int rots) {
  const float s = s0 + threadIdx.x * 1e-6f;  // per-lane operands, as the join's column records
  float cov[D], xx[D], xy[D], xz[D], CK[D];
#pragma unroll
  for (int d = 0; d < D; ++d) {
    cov[d] = s * d;
    xx[d] = s + d * 1e-3f;
    xy[d] = s - d * 1e-3f;
    xz[d] = s * (0.3f + 0.01f * d);
    CK[d] = -1e30f;
  }
  float ra = threadIdx.x * 1e-6f, rb = s * 0.9f, rc = s * 0.7f, sink = -1e30f;
  for (int it = 0; it < rots; ++it) {
#pragma unroll
    for (int u = 0; u < D; u += 2) {
      float ka[D], kb[D];
#pragma unroll
      for (int d = 0; d < D; ++d) {
        const int x = (u + d) % D;
        cov[d] = fmaf(ra, xy[x], cov[d]);
        cov[d] = fmaf(xx[x], rb, cov[d]);
        ka[d] = (cov[d] * xz[x]) * rc;
      }
#pragma unroll
      for (int d = 0; d < D; ++d) {
        const int x = (u + 1 + d) % D;
        cov[d] = fmaf(rb, xy[x], cov[d]);
        cov[d] = fmaf(xx[x], ra, cov[d]);
        kb[d] = (cov[d] * xz[x]) * rc;
      }
      const float c0 = fmaxf(CK[u % D], ka[0]);
      const float c1 = max3(CK[(u + 1) % D], ka[1], kb[0]);
#pragma unroll
      for (int d = 2; d < D - 1; ++d) CK[(u + d) % D] = max3(CK[(u + d) % D], ka[d], kb[d - 1]);
      CK[(u + D - 1) % D] = fmaxf(ka[D - 1], kb[D - 2]);
      CK[u % D] = kb[D - 1];
      sink = max3(sink, tree8(ka), tree8(kb));
      sink = max3(sink, c0, c1);
      ra += 1e-7f;
      rc += 1e-9f;
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = sink + CK[0];
}

// packed: two groups of D slots in register pairs as in mp_join_x2.cu
__global__ void packed_kernel(float* out, float s0, int rots) {
  const float s = s0 + threadIdx.x * 1e-6f;
  f2 cov[D], xdf[D], xdg[D], xin[D];
  float CA[D], CB[D];
#pragma unroll
  for (int d = 0; d < D; ++d) {
    cov[d] = pk(s * d, s * d + 1);
    xdf[d] = pk(s + d * 1e-3f, s + d * 2e-3f);
    xdg[d] = pk(s - d * 1e-3f, s - d * 2e-3f);
    xin[d] = pk(s * (0.3f + 0.01f * d), s * (0.4f + 0.01f * d));
    CA[d] = CB[d] = -1e30f;
  }
  f2 rdf = pk(threadIdx.x * 1e-6f, threadIdx.x * 1e-6f), rdg = pk(s * 0.9f, s * 0.9f), rin = pk(s * 0.7f, s * 0.7f);
  float sink = -1e30f;
  for (int it = 0; it < rots; ++it) {
#pragma unroll
    for (int u = 0; u < D; u += 2) {
      float ka[D], kb[D], la[D], lb[D];
#pragma unroll
      for (int d = 0; d < D; ++d) {
        const int x = (u + d) % D;
        cov[d] = fma2(rdf, xdg[x], cov[d]);
        cov[d] = fma2(xdf[x], rdg, cov[d]);
        unpk(mul2(mul2(cov[d], xin[x]), rin), ka[d], kb[d]);
      }
#pragma unroll
      for (int d = 0; d < D; ++d) {
        const int x = (u + 1 + d) % D;
        cov[d] = fma2(rdg, xdg[x], cov[d]);
        cov[d] = fma2(xdf[x], rdf, cov[d]);
        unpk(mul2(mul2(cov[d], xin[x]), rin), la[d], lb[d]);
      }
      const float a0 = fmaxf(CA[u % D], ka[0]), b0 = fmaxf(CB[u % D], kb[0]);
      const float a1 = max3(CA[(u + 1) % D], ka[1], la[0]), b1 = max3(CB[(u + 1) % D], kb[1], lb[0]);
#pragma unroll
      for (int d = 2; d < D - 1; ++d) {
        CA[(u + d) % D] = max3(CA[(u + d) % D], ka[d], la[d - 1]);
        CB[(u + d) % D] = max3(CB[(u + d) % D], kb[d], lb[d - 1]);
      }
      CA[(u + D - 1) % D] = fmaxf(ka[D - 1], la[D - 2]);
      CB[(u + D - 1) % D] = fmaxf(kb[D - 1], lb[D - 2]);
      CA[u % D] = la[D - 1];
      CB[u % D] = lb[D - 1];
      sink = max3(sink, fmaxf(tree8(ka), tree8(kb)), fmaxf(tree8(la), tree8(lb)));
      sink = max3(sink, max3(a0, b0, a1), b1);
      rin = fma2(rin, rdg, rdf);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = sink + CA[0] + CB[0];
}

template <typename K>
void run(K kern, const char* name, int cells_per_rot, float* d, int warps_per_sm) {
  const int rots = 4000;
  const int blocks = 148 * warps_per_sm;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  kern<<<blocks, 32>>>(d, 1.0001f, rots);
  cudaEventRecord(e0);
  kern<<<blocks, 32>>>(d, 1.0001f, rots);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const double cells = (double)blocks * 32 * rots * cells_per_rot;
  const double cyc = ms * 1e-3 * clk * 1e3;
  const double per_smsp = cells / (cyc * 148 * 4);
  printf("%-8s %2d warps/SM: %.3f ms, %.2f cells/clk/SMSP = %.2f cycles per 32 cells, pipe frac %.3f\n", name,
         warps_per_sm, ms, per_smsp, 32.0 / per_smsp, per_smsp * 4 / 32);
}
int main() {
  float* d;
  cudaMalloc(&d, 148 * 64 * 32 * 4);
  for (int w : {8, 16, 20, 32}) run(scalar_kernel, "scalar", D * D, d, w);
  for (int w : {8, 16, 20}) run(packed_kernel, "packed", 2 * D * D, d, w);
  for (int w : {8, 16, 20, 32}) run(scalar_int_kernel, "sc-int", D * D, d, w);
  return 0;
}

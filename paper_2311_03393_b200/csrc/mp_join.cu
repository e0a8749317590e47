// K6: the matrix-profile self-join hot loop (Def. 6; self-join P:L322).
//
// Work: for each sketch series g, every cell (i, j = i + delta) of the upper triangle with
// delta in [excl+1, n_sub) (reading 7) is visited once.  Along a diagonal the mean-centred dot
// product follows the STOMP/SCAMP recurrence (see mp_prep.cu)
//     cov(i,j) = cov(i-1,j-1) + df_i dg_j + df_j dg_i,     rho = cov * inv_i * inv_j,
// and each cell updates BOTH the row profile of i and the column profile of j (the self-join
// is symmetric, so only delta > 0 is walked).  The profile keeps max rho (= min distance,
// dist^2 = 2m(1-rho)) with its argument.
//
// Blackwell mapping:
//  * A CTA of NT threads owns a tile of W = NT*D consecutive diagonals x `L` rows; thread t owns
//    diagonals [delta0 + tD, delta0 + tD + D) and walks the rows in registers (D covariances,
//    D column operands rotating through registers, D running column maxima).  The recurrence is
//    2 FFMA + 2 FMUL per cell on the FP32 pipe (or the FP64 pipe for the double variant).
//  * Index tracking costs one LOP3 per cell: the diagonal slot d = delta mod D is written into
//    the low log2(D) mantissa bits of rho, so plain (3-input, sm_100 FMNMX3) max operations carry
//    the argument along; the neighbour's distance is recomputed exactly in FP64 afterwards
//    (mp_final.cu), so the code bits only ever break near-ties (documented ties).
//  * Row maxima reduce over a thread's D slots; column maxima reduce over the D rows a column
//    spends in a thread.  Each row / column candidate is compared with a shared-memory copy of
//    the global best ("check then atomic"): only improvements reach the global 64-bit atomicMax
//    (FP32: packed {orderable rho, ~j}) or 128-bit CAS (FP64).
//  * Operands {df, dg, inv} of the tile's rows and columns are staged with cp.async into
//    shared memory: a ring of W + 2C columns in a swizzled [D][RS/D] layout (conflict-free
//    128-bit loads: lane t reads column base + tD) and a double-buffered chunk of rows.
//  * Every tile re-seeds its covariances exactly in FP64 at its first row (global re-seed grid:
//    tiles start at multiples of L, diagonal blocks at multiples of W), so per-cell arithmetic
//    is independent of how diagonals are split into bands/GPUs -> bit-identical keys.
#include <cuda_runtime.h>
#include <stdint.h>

#include "internal.h"

namespace skmp {
namespace {

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

struct JoinArgs {
  const void* R;
  int64_t ld;
  const void* Q;
  const double* mu;
  int64_t ldq;
  int64_t* keys;
  int64_t n_sub;
  int64_t n;
  int m;
  int L;
  int64_t dlo, dhi;
  const int64_t* prefix;  // nblk + 1 cumulative tile counts
  int64_t nblk;
  int64_t blk0;
};

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

template <int D>
__device__ __forceinline__ float code(float r, int d) {
  return __int_as_float((__float_as_int(r) & ~(D - 1)) | d);
}
template <int D>
__device__ __forceinline__ double code(double r, int d) {
  const int lo = __double2loint(r), hi = __double2hiint(r);
  return __hiloint2double(hi, (lo & ~(D - 1)) | d);
}
template <int D>
__device__ __forceinline__ int slot_of(float r) { return __float_as_int(r) & (D - 1); }
template <int D>
__device__ __forceinline__ int slot_of(double r) { return __double2loint(r) & (D - 1); }

__device__ __forceinline__ float max3(float a, float b, float c) {
  float r;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
__device__ __forceinline__ double max3(double a, double b, double c) { return fmax(a, fmax(b, c)); }
__device__ __forceinline__ float max2(float a, float b) { return fmaxf(a, b); }
__device__ __forceinline__ double max2(double a, double b) { return fmax(a, b); }

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

// publish candidate (v, arg) into profile entry i
__device__ __forceinline__ void publish(int64_t* keys, int64_t i, float v, int64_t arg) {
  const int64_t key = (int64_t)(((uint64_t)(uint32_t)ord32(v) << 32) |
                                (uint64_t)(0xFFFFFFFFu - (uint32_t)arg));
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

template <typename T, int D, int NT, int C>
struct Geo {
  static constexpr int W = NT * D;
  static constexpr int RS = W + 2 * C;   // ring columns
  static constexpr int RSD = RS / D;     // ring rows of the swizzled [D][RSD] layout
  static_assert(RS % D == 0, "ring must be a multiple of D");
  static_assert(C % (2 * D) == 0, "chunk must hold whole pairs of D-row rotations");
  using Q = typename JT<T>::Q;
  static constexpr size_t smem_bytes =
      sizeof(Q) * (RS + 2 * C) + sizeof(T) * (RS + 2 * C);
  __device__ static __forceinline__ int pos(int64_t c) {
    const int p = (int)(c % RS);
    return (p % D) * RSD + p / D;
  }
};

// Stage `count` Q entries (global index g0 + e) into the ring / row buffer.
template <typename T>
__device__ __forceinline__ void stage_q(typename JT<T>::Q* dst, const typename JT<T>::Q* src) {
  constexpr int parts = sizeof(typename JT<T>::Q) / 16;
#pragma unroll
  for (int q = 0; q < parts; ++q)
    cp_async16(reinterpret_cast<char*>(dst) + 16 * q, reinterpret_cast<const char*>(src) + 16 * q);
}

template <typename T, int D, int NT, int C, bool MASKED>
__device__ __forceinline__ void join_tile(const JoinArgs& a, int g, int64_t delta0, int64_t i0,
                                          int64_t i1, unsigned char* smem_raw) {
  using G = Geo<T, D, NT, C>;
  using Q = typename JT<T>::Q;
  constexpr int W = G::W;
  constexpr int RS = G::RS;
  constexpr int RSD = G::RSD;
  Q* ring = reinterpret_cast<Q*>(smem_raw);
  Q* rowq = ring + RS;
  T* cthr = reinterpret_cast<T*>(rowq + 2 * C);
  T* rthr = cthr + RS;

  const int tid = threadIdx.x;
  const int64_t n_sub = a.n_sub;
  const Q* q = static_cast<const Q*>(a.Q) + (int64_t)g * a.ldq;
  int64_t* keys = a.keys + (int64_t)g * n_sub * (sizeof(T) == 4 ? 1 : 2);
  const int64_t dt = delta0 + (int64_t)tid * D;  // this thread's first diagonal

  // per-slot validity limit: cell (i, i+dt+d) is valid iff i < lim[d]
  int64_t lim[D];
#pragma unroll
  for (int d = 0; d < D; ++d) {
    const int64_t dd = dt + d;
    lim[d] = (dd >= a.dlo && dd < a.dhi && dd < n_sub) ? (n_sub - dd) : 0;
  }

  // ---- exact FP64 seed of cov(i0, i0+dt+d), pre-compensated for the first in-loop update -----
  T cov[D];
  {
    const T* R = static_cast<const T*>(a.R) + (int64_t)g * a.ld;
    const double mua = a.mu[(int64_t)g * a.ldq + i0];
    double mub[D], acc[D], w[D];
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const int64_t j = i0 + dt + d;
      mub[d] = (j < n_sub) ? a.mu[(int64_t)g * a.ldq + j] : 0.0;
      acc[d] = 0.0;
    }
    const int64_t jb = i0 + dt;
#pragma unroll
    for (int d = 0; d < D - 1; ++d) w[d] = (jb + d < a.n) ? (double)R[jb + d] : 0.0;
    for (int s0 = 0; s0 < a.m; s0 += D) {
#pragma unroll
      for (int e = 0; e < D; ++e) {
        const int s = s0 + e;
        if (s < a.m) {
          const int64_t t = jb + s + D - 1;
          w[(e + D - 1) % D] = (t < a.n) ? (double)R[t] : 0.0;
          const double av = (double)R[i0 + s] - mua;
#pragma unroll
          for (int d = 0; d < D; ++d) acc[d] = fma(av, w[(e + d) % D] - mub[d], acc[d]);
        }
      }
    }
    const Q qi = q[i0];
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const Q qj = q[i0 + dt + d];  // padded: safe past n_sub
      const double adj = (double)qi.x * (double)qj.y + (double)qj.x * (double)qi.y;
      cov[d] = (T)(acc[d] - adj);
    }
  }

  // ---- prologue: stage rows [i0, i0+C) and ring columns [i0+delta0, i0+delta0+W+C) ----------
  for (int e = tid; e < W + C; e += NT) {
    const int64_t c = i0 + delta0 + e;
    stage_q<T>(&ring[G::pos(c)], &q[c]);
    cthr[G::pos(c)] = (c < n_sub) ? load_thr(keys, c, (T*)nullptr) : pos_inf<T>();
  }
  for (int e = tid; e < C; e += NT) {
    const int64_t i = i0 + e;
    stage_q<T>(&rowq[i % (2 * C)], &q[i]);
    rthr[i % (2 * C)] = (i < n_sub) ? load_thr(keys, i, (T*)nullptr) : pos_inf<T>();
  }
  cp_async_wait_all();
  __syncthreads();

  // column operand registers: X[(u + d) % D] holds column i + dt + d at unrolled row u
  Q X[D];
#pragma unroll
  for (int d = 0; d < D - 1; ++d) X[d] = ring[G::pos(i0 + dt + d)];
  T CK[D];  // running column maxima, same rotation as X
#pragma unroll
  for (int d = 0; d < D; ++d) CK[d] = neg_inf<T>();

  // ring row index of column (ib + dt): qt; (ib + dt) is a multiple of D
  int qt = (int)(((i0 + dt) % RS) / D);

  for (int64_t r = i0; r < i1; r += C) {
    const int64_t rend = (r + C < i1) ? r + C : i1;
    // ---- prefetch the next chunk: rows [r+C, r+2C), columns [r+delta0+W+C, +C) --------------
    const bool more = r + C < i1;
    T nthr_c = pos_inf<T>(), nthr_r = pos_inf<T>();
    int64_t nc = -1, nr = -1;
    if (more) {
      if (tid < C) {
        nc = r + delta0 + W + C + tid;
        stage_q<T>(&ring[G::pos(nc)], &q[nc]);
        if (nc < n_sub) nthr_c = load_thr(keys, nc, (T*)nullptr);
      } else if (tid < 2 * C) {
        nr = r + C + (tid - C);
        stage_q<T>(&rowq[nr % (2 * C)], &q[nr]);
        if (nr < n_sub) nthr_r = load_thr(keys, nr, (T*)nullptr);
      }
    }

    // ---- compute rows [r, rend) in D-row rotations of 2-row pairs ---------------------------
    for (int64_t ib = r; ib < rend; ib += D) {
      const int qt1 = (qt + 1 == RSD) ? 0 : qt + 1;
      const int rb = (int)(ib % (2 * C));
#pragma unroll
      for (int u = 0; u < D; u += 2) {
        // -- row u --
        const Q ra = rowq[rb + u];
        X[(u + D - 1) % D] = ring[((u + D - 1) % D) * RSD + (u == 0 ? qt : qt1)];
        T ka[D];
#pragma unroll
        for (int d = 0; d < D; ++d) {
          const Q& x = X[(u + d) % D];
          cov[d] = fma(ra.x, x.y, cov[d]);
          cov[d] = fma(x.x, ra.y, cov[d]);
          const T rho = (cov[d] * x.z) * ra.z;
          ka[d] = code<D>(rho, d);
          if (MASKED) ka[d] = (ib + u < lim[d]) ? ka[d] : neg_inf<T>();
        }
        // -- row u+1 (its entering column reuses the register of row u's completed column) --
        const Q rbq = rowq[rb + u + 1];
        const T colv0 = max2(CK[u % D], ka[0]);  // column ib+u+dt completes after row u
        X[u % D] = ring[(u % D) * RSD + qt1];
        T kb[D];
#pragma unroll
        for (int d = 0; d < D; ++d) {
          const Q& x = X[(u + 1 + d) % D];
          cov[d] = fma(rbq.x, x.y, cov[d]);
          cov[d] = fma(x.x, rbq.y, cov[d]);
          const T rho = (cov[d] * x.z) * rbq.z;
          kb[d] = code<D>(rho, d);
          if (MASKED) kb[d] = (ib + u + 1 < lim[d]) ? kb[d] : neg_inf<T>();
        }
        // -- column maxima: registers x = (u + d) % D --
        const T colv1 = max3(CK[(u + 1) % D], ka[1], kb[0]);  // column ib+u+1+dt completes
#pragma unroll
        for (int d = 2; d < D - 1; ++d) CK[(u + d) % D] = max3(CK[(u + d) % D], ka[d], kb[d - 1]);
        CK[(u + D - 1) % D] = max2(ka[D - 1], kb[D - 2]);  // column entered at row u
        CK[u % D] = kb[D - 1];                              // column entered at row u+1
        // -- row maxima over the D slots --
        T rowa, rowb;
        if (D == 8) {
          rowa = max3(max3(ka[0], ka[1], ka[2]), max3(ka[3], ka[4], ka[5]), max2(ka[6], ka[7]));
          rowb = max3(max3(kb[0], kb[1], kb[2]), max3(kb[3], kb[4], kb[5]), max2(kb[6], kb[7]));
        } else {
          rowa = ka[0];
          rowb = kb[0];
#pragma unroll
          for (int d = 1; d < D; ++d) { rowa = max2(rowa, ka[d]); rowb = max2(rowb, kb[d]); }
        }
        // -- check-then-publish --
        const T ta = rthr[rb + u], tb = rthr[rb + u + 1];
        const T tc0 = cthr[(u % D) * RSD + qt];
        const T tc1 = cthr[((u + 1) % D) * RSD + qt];
        if (rowa > ta || rowb > tb || colv0 > tc0 || colv1 > tc1) {
          if (rowa > ta) {
            const int64_t i = ib + u;
            publish(keys, i, rowa, i + dt + slot_of<D>(rowa));
            rthr[rb + u] = rowa;
          }
          if (rowb > tb) {
            const int64_t i = ib + u + 1;
            publish(keys, i, rowb, i + dt + slot_of<D>(rowb));
            rthr[rb + u + 1] = rowb;
          }
          if (colv0 > tc0) {
            const int64_t c = ib + u + dt;
            publish(keys, c, colv0, c - dt - slot_of<D>(colv0));
            cthr[(u % D) * RSD + qt] = colv0;
          }
          if (colv1 > tc1) {
            const int64_t c = ib + u + 1 + dt;
            publish(keys, c, colv1, c - dt - slot_of<D>(colv1));
            cthr[((u + 1) % D) * RSD + qt] = colv1;
          }
        }
      }
      qt = qt1;
    }

    // ---- land the prefetched chunk ------------------------------------------------------------
    if (more) {
      if (nc >= 0) cthr[G::pos(nc)] = nthr_c;
      if (nr >= 0) rthr[nr % (2 * C)] = nthr_r;
    }
    cp_async_wait_all();
    __syncthreads();
  }

  // ---- epilogue: the D-1 columns still open after the last row hold partial maxima ----------
  // After row i1-1 the open columns are (i1 - 1) + dt + d for d = 1..D-1, i.e. register
  // x = d - 1 holds column i1 + dt + x.
#pragma unroll
  for (int x = 0; x < D - 1; ++x) {
    const T v = CK[x];
    const int64_t c = i1 + dt + x;
    if (c < n_sub && v > cthr[G::pos(c)]) publish(keys, c, v, c - dt - slot_of<D>(v));
  }
}

template <typename T, int D, int NT, int C>
__global__ void __launch_bounds__(NT)
join_kernel(JoinArgs a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  constexpr int W = NT * D;
  __shared__ int64_t s_tile[3];
  const int g = blockIdx.y;
  if (threadIdx.x == 0) {
    // binary search: block b with prefix[b] <= tile < prefix[b+1]
    const int64_t tile = blockIdx.x;
    int64_t lo = 0, hi = a.nblk - 1;
    while (lo < hi) {
      const int64_t mid = (lo + hi + 1) >> 1;
      if (a.prefix[mid] <= tile) lo = mid; else hi = mid - 1;
    }
    const int64_t b = lo;
    const int64_t rt = tile - a.prefix[b];
    const int64_t delta0 = (a.blk0 + b) * W;
    const int64_t dmin = delta0 > a.dlo ? delta0 : a.dlo;
    const int64_t rows = a.n_sub - dmin;
    const int64_t i0 = rt * a.L;
    const int64_t i1 = (i0 + a.L < rows) ? i0 + a.L : rows;
    s_tile[0] = delta0;
    s_tile[1] = i0;
    s_tile[2] = i1;
  }
  __syncthreads();
  const int64_t delta0 = s_tile[0], i0 = s_tile[1], i1 = s_tile[2];
  // rows are processed in whole D-row rotations; rows beyond i1 are masked cells
  const int64_t i1r = i0 + (((i1 - i0) + D - 1) / D) * D;
  const bool masked = (delta0 < a.dlo) || (delta0 + W > a.dhi) || (i1r - 1 + delta0 + W - 1 >= a.n_sub);
  if (masked)
    join_tile<T, D, NT, C, true>(a, g, delta0, i0, i1r, smem_raw);
  else
    join_tile<T, D, NT, C, false>(a, g, delta0, i0, i1r, smem_raw);
}

template <typename T, int D>
cudaError_t launch_join_t(const MpDev& w, int64_t dlo, int64_t dhi, const int64_t* prefix,
                          int64_t nblk, int64_t ntiles, int64_t blk0, cudaStream_t st) {
  constexpr int NT = kJoinNT, C = kJoinC;
  using G = Geo<T, D, NT, C>;
  JoinArgs a;
  a.R = w.R;
  a.ld = w.ld;
  a.Q = w.Q;
  a.mu = w.mu;
  a.ldq = w.ldq;
  a.keys = w.keys;
  a.n_sub = w.n_sub;
  a.n = w.n;
  a.m = w.m;
  a.L = w.L;
  a.dlo = dlo;
  a.dhi = dhi;
  a.prefix = prefix;
  a.nblk = nblk;
  a.blk0 = blk0;
  const size_t smem = G::smem_bytes;
  cudaError_t e = cudaFuncSetAttribute(join_kernel<T, D, NT, C>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e) return e;
  dim3 grid((unsigned)ntiles, (unsigned)w.k);
  join_kernel<T, D, NT, C><<<grid, NT, smem, st>>>(a);
  count_launches(1);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_mp_join(const MpDev& w, int64_t dlo, int64_t dhi, const int64_t* d_prefix,
                           int64_t nblk, int64_t ntiles, int64_t blk0, cudaStream_t st) {
  if (ntiles <= 0) return cudaSuccess;
  if (w.dtype == SKMP_F32) return launch_join_t<float, kJoinD32>(w, dlo, dhi, d_prefix, nblk, ntiles, blk0, st);
  return launch_join_t<double, kJoinD64>(w, dlo, dhi, d_prefix, nblk, ntiles, blk0, st);
}

}  // namespace skmp

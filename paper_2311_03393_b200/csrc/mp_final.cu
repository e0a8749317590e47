// K7: keys -> (P, I).  For each series g and row i the join left the best FP32/FP64 rho it
// found together with the smallest index b of the D-cell candidate set that produced it (one
// thread's D diagonals of row i, or one thread's D rows of column i; mp_join.cu).  Here the set
// is resolved EXACTLY in FP64 (Def. 3: z-normalised Euclidean distance, reading 8:
// smallest index on ties): one warp per row evaluates dist^2 = 2m - 2 cov / (sigma_i sigma_j)
// for the <= D admissible members with centred FP64 dot products, keeps the nearest, and then
// recomputes its distance from the definition by explicit differences (z = (R - mu) / sigma
// with the window statistics of mp_prep.cu).  Flat windows follow reading 5 (flat-flat 0, flat
// vs non-flat sqrt(m), ties to the smallest index); an all-flat ("inert", reading 6) series
// therefore gets P = 0.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

#include "internal.h"

namespace skmp {
namespace {

// the key word that names entry i's candidate set (FP32: the only word; FP64: the index word)
__device__ __forceinline__ int64_t key_word(const int64_t* keys, int64_t i, int words) {
  return words == 1 ? keys[i] : keys[2 * i + 1];
}
// candidate-set base from that word; false if no candidate was ever published
__device__ __forceinline__ bool key_arg(int64_t kw, int words, int64_t* base) {
  if (words == 1) {
    const uint32_t lo = (uint32_t)(kw & 0xFFFFFFFFll);
    const int32_t hi = (int32_t)(kw >> 32);
    if (hi == (int32_t)0x80800000 && lo == 0) return false;  // never written (init key)
    *base = (int64_t)(0xFFFFFFFFu - lo) - kKeyArgBias;
    return true;
  }
  if (kw == INT64_MIN) return false;
  *base = -1 - kw;
  return true;
}

// smallest admissible flat window of row i (|i - f| > excl), or -1
__device__ __forceinline__ int64_t smallest_adm_flat(const int32_t* F, int32_t nf, int64_t i,
                                                     int excl) {
  if (nf <= 0) return -1;
  if (excl < 0 || (int64_t)F[0] < i - excl) return F[0];  // excl < 0: AB-join, every j admissible
  // first F[q] > i + excl
  int32_t lo = 0, hi = nf;
  while (lo < hi) {
    const int32_t mid = (lo + hi) >> 1;
    if ((int64_t)F[mid] > i + excl) hi = mid; else lo = mid + 1;
  }
  return lo < nf ? F[lo] : -1;
}

// Transposed warp sum of N per-lane values: afterwards every lane holds in v[0] the warp total
// of value xidx<N>(lane) (log2(N) exchange steps keep half the values each, then plain steps).
template <int N, int L = 32>
__device__ __forceinline__ void xsum(double (&v)[N], int lane) {
  int c = N;
#pragma unroll
  for (int o = L / 2; o >= 1; o >>= 1) {
    if (c > 1) {
      const bool up = (lane & o) != 0;
#pragma unroll
      for (int q = 0; q < N / 2; ++q) {
        if (q < c / 2) {
          const double send = up ? v[q] : v[q + c / 2];
          const double keep = up ? v[q + c / 2] : v[q];
          v[q] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
      }
      c >>= 1;
    } else {
      v[0] += __shfl_xor_sync(0xffffffffu, v[0], o);
    }
  }
}
template <int N, int L = 32>
__device__ __forceinline__ int xidx(int lane) {
  int idx = 0, c = N;
#pragma unroll
  for (int o = L / 2; o >= 1 && c > 1; o >>= 1) {
    c >>= 1;
    if (lane & o) idx += c;
  }
  return idx;
}

// neighbour j of row i is admissible: self-join |i - j| > excl (reading 7); AB-join (excl < 0)
// any window of the other series
__device__ __forceinline__ bool admissible(int64_t i, int64_t j, int64_t n_sub_o, int excl) {
  const int64_t dj = j > i ? j - i : i - j;
  return j >= 0 && j < n_sub_o && (excl < 0 || dj > excl);
}

// Window positions staged per warp and chunk: the row's window and the candidate windows
// [b, b + SPAN - 1 + MC) are copied to shared memory with every load issued before any use (one
// L2 round trip per chunk instead of one per dependent load), then read back conflict-free.
// Staged values are converted to FP64 once (an FP32 -> FP64 conversion per use would cost
// SPAN conversions per window position).
template <typename T> struct FinChunk { static constexpr int MC = 256; };
constexpr int kFinWarps = 8;  // warps per CTA
#ifndef SKMP_FIN_ROWS
#define SKMP_FIN_ROWS 16
#endif
constexpr int kFinRows = SKMP_FIN_ROWS;  // consecutive rows per warp (the next row's key is loaded early)
template <typename T, int SPAN>
__host__ __device__ constexpr int fin_stride() { return 2 * FinChunk<T>::MC + SPAN; }  // doubles per warp

// stage xi[s] = R[i + s0 + s] (s < len) and xo[t] = Ro[clamp(b + s0 + t)] (t < len + SPAN - 1)
template <typename T, int SPAN>
__device__ __forceinline__ void fin_stage(double* xi, double* xo, const T* R, const T* Ro, int64_t i, int64_t b,
                                          int s0, int len, int64_t n_o, int lane) {
  constexpr int MC = FinChunk<T>::MC;
  constexpr int NI = MC / 32, NO = (MC + SPAN - 1 + 31) / 32;
  T vi[NI], vo[NO];
  // 32-bit offsets (series lengths < 2^31) from per-row bases
  const T* ri = R + (i + s0);
  const int32_t ob = (int32_t)(b + s0), no = (int32_t)n_o;
#pragma unroll
  for (int q = 0; q < NI; ++q) {
    const int s = lane + 32 * q;
    vi[q] = s < len ? ri[s] : (T)0;
  }
#pragma unroll
  for (int q = 0; q < NO; ++q) {
    const int t = lane + 32 * q;
    int32_t idx = ob + t;
    idx = idx < 0 ? 0 : (idx >= no ? no - 1 : idx);  // only inadmissible members read clamped data
    vo[q] = t < len + SPAN - 1 ? Ro[idx] : (T)0;
  }
#pragma unroll
  for (int q = 0; q < NI; ++q) xi[lane + 32 * q] = (double)vi[q];
#pragma unroll
  for (int q = 0; q < NO; ++q)
    if (lane + 32 * q < MC + SPAN - 1) xo[lane + 32 * q] = (double)vo[q];
  __syncwarp();
}

// rows of w against neighbours in wo (wo = w for a self-join with exclusion radius excl >= 0;
// an AB-join passes the other series and excl = -1).  One warp per row.
template <typename T, int SPAN>
__global__ void __launch_bounds__(32 * kFinWarps)
finalize_kernel(MpDev w, MpDev wo, int excl, int64_t row_lo, int64_t row_hi, T* __restrict__ P,
                int64_t* __restrict__ I) {
  static_assert(SPAN <= 32 && (SPAN & (SPAN - 1)) == 0, "span must be a power of two <= 32");
  constexpr int MC = FinChunk<T>::MC;
  __shared__ double fsm[kFinWarps * fin_stride<T, SPAN>()];
  const int lane = threadIdx.x & 31;
  double* xi = fsm + (threadIdx.x >> 5) * fin_stride<T, SPAN>();
  double* xo = xi + MC;
  // Every lane runs the same straight-line code (no early return, the special rows' results are
  // selected at the end): the warp shuffles then sit in convergent code, which spares the
  // compiler's collective-convergence sequences around each of them.
  const int64_t i_first = row_lo + ((int64_t)blockIdx.x * kFinWarps + (threadIdx.x >> 5)) * kFinRows;
  const int g = blockIdx.y;
  const int words = (w.dtype == SKMP_F32) ? 1 : 2;
  const int64_t* keys = w.keys + (int64_t)g * w.n_sub * words;
  int64_t kw_next = key_word(keys, i_first < row_hi ? i_first : row_hi - 1, words);
  for (int rr = 0; rr < kFinRows; ++rr) {
  const int64_t i_raw = i_first + rr;
  const bool live = i_raw < row_hi;
  const int64_t i = live ? i_raw : row_hi - 1;
  const int64_t kw = kw_next;
  kw_next = key_word(keys, i + 1 < row_hi ? i + 1 : row_hi - 1, words);  // next row, in flight early
  const int64_t o = (int64_t)g * w.ldq, oo = (int64_t)g * wo.ldq;
  const T* R = static_cast<const T*>(w.R) + (int64_t)g * w.ld;
  const T* Ro = static_cast<const T*>(wo.R) + (int64_t)g * wo.ld;
  const int m = w.m;
  const double sqm = sqrt((double)m);
  const double inf = __longlong_as_double(0x7ff0000000000000ll), nan = __longlong_as_double(0x7ff8000000000000ll);
  const int32_t nf = wo.nflat[g];
  const int32_t* F = wo.flat_list + (int64_t)g * wo.n_sub;
  const bool fi = w.flat[o + i] != 0;
  int64_t kb = 0;
  const bool has = key_arg(kw, words, &kb);  // kb = smallest index of the winning set
  // ---- resolve the winning set [b, b + SPAN): nearest admissible member (Def. 3) --------------
  const int64_t b = has ? kb : 0;
  const double mi = w.mu[o + i];
  double acc[SPAN], asum = 0.0;
#pragma unroll
  for (int d = 0; d < SPAN; ++d) acc[d] = 0.0;
  for (int s0 = 0; s0 < m; s0 += MC) {
    const int len = m - s0 < MC ? m - s0 : MC;
    fin_stage<T, SPAN>(xi, xo, R, Ro, i, b, s0, len, wo.n, lane);
    for (int s = lane; s < len; s += 32) {
      const double a = xi[s] - mi;
      asum += a;
#pragma unroll
      for (int d = 0; d < SPAN; ++d) acc[d] = fma(a, xo[s + d], acc[d]);
    }
    __syncwarp();
  }
#pragma unroll
  for (int q = 16; q > 0; q >>= 1) asum += __shfl_xor_sync(0xffffffffu, asum, q);
  xsum<SPAN>(acc, lane);
  int d = xidx<SPAN>(lane);
  double dd = inf;  // not admissible
  const int64_t jd = b + d;
  if (admissible(i, jd, wo.n_sub, excl)) {
    if (wo.flat[oo + jd]) {
      dd = (double)m;  // reading 5: flat vs non-flat
    } else {
      // sum_s (R_i - mu_i)(R_j - mu_j) = sum_s (R_i - mu_i) R_j - mu_j sum_s (R_i - mu_i)
      const double cov = acc[0] - wo.mu[oo + jd] * asum;
      dd = 2.0 * m - 2.0 * cov / (w.sig64[o + i] * wo.sig64[oo + jd]);
    }
  }
#pragma unroll
  for (int q = 16; q >= 1; q >>= 1) {  // warp argmin of (dd, d), smallest d on ties
    const double od = __shfl_xor_sync(0xffffffffu, dd, q);
    const int oi = __shfl_xor_sync(0xffffffffu, d, q);
    if (od < dd || (od == dd && oi < d)) {
      dd = od;
      d = oi;
    }
  }
  const int64_t jr = dd < inf ? b + d : -1;
  // ---- its distance from the definition, by explicit differences (computed unconditionally
  // on a valid window; used only when jr is a non-flat member) ---------------------------------
  const bool exact = jr >= 0 && !wo.flat[oo + (jr >= 0 ? jr : 0)];
  const int64_t je = exact ? jr : (b < 0 ? 0 : (b >= wo.n_sub ? wo.n_sub - 1 : b));
  const int de = exact ? d : 0;
  double pe;
  {
    const double mj = wo.mu[oo + je];
    // z = (x - mu) * (1/sigma): one division per row instead of per element (<= 1 ulp from
    // the textbook quotient; the oracle divides)
    const double ii = 1.0 / w.sig64[o + i], ij = 1.0 / wo.sig64[oo + je];
    double acc2 = 0.0;
    if (m <= MC && exact) {  // the staged chunk still holds both windows (member d at offset d)
      for (int s = lane; s < m; s += 32) {
        const double zi = __dmul_rn(xi[s] - mi, ii);
        const double zj = __dmul_rn(xo[s + de] - mj, ij);
        const double e = zi - zj;
        acc2 = __dadd_rn(acc2, __dmul_rn(e, e));
      }
    } else {
      for (int s = lane; s < m; s += 32) {
        const double zi = __dmul_rn((double)R[i + s] - mi, ii);
        const double zj = __dmul_rn((double)Ro[je + s] - mj, ij);
        const double e = zi - zj;
        acc2 = __dadd_rn(acc2, __dmul_rn(e, e));
      }
    }
#pragma unroll
    for (int q = 16; q > 0; q >>= 1) acc2 += __shfl_xor_sync(0xffffffffu, acc2, q);
    pe = sqrt(acc2);
  }
  // ---- assemble (warp-uniform selections, no shuffles below) ----------------------------------
  double p;
  int64_t j;
  if (fi) {
    const int64_t f = smallest_adm_flat(F, nf, i, excl);
    if (f >= 0) {
      p = 0.0;
      j = f;
    } else {
      p = sqm;  // every admissible neighbour is non-flat: the smallest one
      j = (excl < 0 || i - excl - 1 >= 0) ? 0 : i + excl + 1;
    }
  } else if (!has) {
    p = nan;  // no candidate (band not covered)
    j = -1;
  } else {
    j = jr;
    p = jr < 0 ? nan : (exact ? pe : sqm);
    if (nf > 0) {
      const int64_t f = smallest_adm_flat(F, nf, i, excl);
      if (f >= 0 && (sqm < p || (sqm == p && f < j) || j < 0)) {
        p = sqm;
        j = f;
      }
    }
  }
  if (lane == 0 && live) {
    P[(int64_t)g * w.n_sub + i] = (T)p;
    I[(int64_t)g * w.n_sub + i] = j;
  }
  __syncwarp();  // the staged windows are overwritten by the next row
  }
}

// ---- register-resident variant for m <= 32 E (all BASELINE configs: m <= 256) -----------------
// One warp per row as above, but lane l owns the E consecutive window positions [E l, E l + E):
// its row values a[e] = R_i[El+e] - mu_i and the candidate values R_o[b + El + t],
// t < E + SPAN - 1, sit in registers, so the SPAN candidate dot products are E*SPAN register
// FMAs per lane (the shared-memory variant re-read every operand from shared memory: ~9x the
// shared traffic).  The windows are staged raw (dtype) in a per-warp shared buffer padded to
// (E+1)-element groups (conflict-free reads of lane l's group), double-buffered: row r+1's
// windows are cp.async'ed (its key loaded one row earlier) while row r computes.
__device__ __forceinline__ void cp_async_b(void* smem, const void* gmem, int bytes) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  if (bytes == 8)
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }

constexpr int kFinRegWarps = 4;
#ifndef SKMP_FIN_MINB
#define SKMP_FIN_MINB 1  // resident CTAs the register allocation must allow (A/B: 6, 8)
#endif
// squared distances below this are recomputed by explicit differences (the dot-product form
// 2m - 2 cov / (sigma_i sigma_j) loses ~1e-14 absolute to cancellation: at dd >= 1 that is
// < 1e-13 relative in P, far inside the 1e-9 FP64 bar; near-duplicate windows need the
// explicit form)
constexpr double kFinExplicitBelow = 1.0;  // warps per CTA (~90 registers: 5 CTAs = 20 warps per SM)
template <int E> __host__ __device__ constexpr int pad_pos(int s) { return s + s / E; }
template <int E, int SPAN> struct RegBuf {
  static constexpr int NI = 32 * E;                    // row window positions (>= m)
  static constexpr int NO = 32 * E + SPAN - 1;         // candidate positions (>= m + SPAN - 1)
  static constexpr int XI = pad_pos<E>(NI - 1) + 1;
  static constexpr int XO = pad_pos<E>(NO - 1) + 1;
  static constexpr int SIZE = XI + XO;                 // elements per buffer
};

// stage row i's window and the candidate windows of base b: positions s < m of the row window
// and t < m + SPAN - 1 of the candidates (the buffer tails stay zero from the kernel start, so
// the masked products are 0 * 0).  Every copy of a lane is at a compile-time offset from one
// global and one shared base (lane l's positions l + 32 q pad to l + l/E + q (32 + 32/E)); a
// candidate window that leaves the series is staged with clamped reads (only inadmissible members
// read clamped values; warp-uniform slow path at the two ends of the series).
template <typename T, int E, int SPAN, bool FULL>
__device__ __forceinline__ void reg_stage(T* buf, const T* R, const T* Ro, int64_t i, int64_t b, int m,
                                          int64_t n_o, int lane) {
  using B = RegBuf<E, SPAN>;
  T* xi = buf + pad_pos<E>(lane);
  T* xo = buf + B::XI + pad_pos<E>(lane);
  constexpr int QS = 32 + 32 / E;  // padded stride of q
  const T* gi = R + i + lane;
#pragma unroll
  for (int q = 0; q < E; ++q)
    if (FULL || lane + 32 * q < m) cp_async_b(xi + q * QS, gi + 32 * q, (int)sizeof(T));
  const int no_used = m + SPAN - 1;
  if (b >= 0 && b + no_used <= n_o) {
    const T* go = Ro + b + lane;
#pragma unroll
    for (int q = 0; q < (B::NO + 31) / 32; ++q)
      if (lane + 32 * q < no_used) cp_async_b(xo + q * QS, go + 32 * q, (int)sizeof(T));
  } else {
    const int32_t ob = (int32_t)b, no = (int32_t)n_o;
#pragma unroll
    for (int q = 0; q < (B::NO + 31) / 32; ++q) {
      const int t = lane + 32 * q;
      if (t < no_used) {
        int32_t idx = ob + t;
        idx = idx < 0 ? 0 : (idx >= no ? no - 1 : idx);
        cp_async_b(xo + q * QS, Ro + idx, (int)sizeof(T));
      }
    }
  }
}

// the lane holding candidate d after xsum<N> (inverse of xidx<N>)
template <int N, int L = 32>
__device__ __forceinline__ int xlane(int d) {
  int lane = 0, c = N;
#pragma unroll
  for (int o = L / 2; o >= 1 && c > 1; o >>= 1) {
    c >>= 1;
    if (d & c) lane |= o;
  }
  return lane;
}

// per-row statistics, loaded one row ahead (after the row's key): the row window's mean,
// inverse std and flat flag, and for this lane's candidate b + xidx(lane) (clamped) the same three
// (inverse stds precomputed by mp_prep.cu: no FP64 division here)
struct FinPre {
  double mi, ii, mc, ic;
  bool fi, fc;
};
template <int SPAN, int L = 32>
__device__ __forceinline__ FinPre fin_pre(const MpDev& w, const MpDev& wo, int64_t o, int64_t oo, int64_t i,
                                          int64_t b, int lane) {
  FinPre p;
  p.mi = w.mu[o + i];
  p.ii = w.isig64[o + i];
  p.fi = w.flat[o + i] != 0;
  int64_t jc = b + xidx<SPAN, L>(lane);
  jc = jc < 0 ? 0 : (jc >= wo.n_sub ? wo.n_sub - 1 : jc);
  p.mc = wo.mu[oo + jc];
  p.ic = wo.isig64[oo + jc];
  p.fc = wo.flat[oo + jc] != 0;
  return p;
}

template <typename T, int SPAN, int E, bool FULL>
__global__ void __launch_bounds__(32 * kFinRegWarps, SKMP_FIN_MINB)
finalize_reg_kernel(MpDev w, MpDev wo, int excl, int64_t row_lo, int64_t row_hi, T* __restrict__ P,
                    int64_t* __restrict__ I) {
  static_assert(SPAN <= 32 && (SPAN & (SPAN - 1)) == 0 && (E % 2) == 0, "geometry");
  using B = RegBuf<E, SPAN>;
  __shared__ __align__(16) T fsm[kFinRegWarps * 2 * B::SIZE];
  const int lane = threadIdx.x & 31;
  T* buf0 = fsm + (threadIdx.x >> 5) * 2 * B::SIZE;
  const int64_t i_first = row_lo + ((int64_t)blockIdx.x * kFinRegWarps + (threadIdx.x >> 5)) * kFinRows;
  const int g = blockIdx.y;
  const int words = (w.dtype == SKMP_F32) ? 1 : 2;
  const int64_t* keys = w.keys + (int64_t)g * w.n_sub * words;
  const int64_t o = (int64_t)g * w.ldq, oo = (int64_t)g * wo.ldq;
  const T* R = static_cast<const T*>(w.R) + (int64_t)g * w.ld;
  const T* Ro = static_cast<const T*>(wo.R) + (int64_t)g * wo.ld;
  const int m = w.m;
  const double sqm = sqrt((double)m);
  const double inf = __longlong_as_double(0x7ff0000000000000ll), nan = __longlong_as_double(0x7ff8000000000000ll);
  const int32_t nf = wo.nflat[g];
  const int32_t* F = wo.flat_list + (int64_t)g * wo.n_sub;
  auto row_of = [&](int rr) { const int64_t x = i_first + rr; return x < row_hi ? x : row_hi - 1; };
  auto base_of = [&](int64_t kw) { int64_t kb = 0; return key_arg(kw, words, &kb) ? kb : (int64_t)0; };
  // prologue: row 0 staged and its statistics requested, row 1's key in flight.  Every global
  // load of a row is issued one row ahead (its key two rows ahead): no dependent load waits.
  int64_t kw_cur = key_word(keys, row_of(0), words);
  int64_t kw_nxt = key_word(keys, row_of(1), words);
  for (int q = lane; q < 2 * B::SIZE; q += 32) buf0[q] = (T)0;  // tails stay zero (see reg_stage)
  __syncwarp();
  reg_stage<T, E, SPAN, FULL>(buf0, R, Ro, row_of(0), base_of(kw_cur), m, wo.n, lane);
  cp_async_commit();
  FinPre pre = fin_pre<SPAN>(w, wo, o, oo, row_of(0), base_of(kw_cur), lane);
  for (int rr = 0; rr < kFinRows; ++rr) {
    const int64_t i_raw = i_first + rr;
    const bool live = i_raw < row_hi;
    const int64_t i = row_of(rr);
    const int64_t kw = kw_cur;
    const FinPre cu = pre;
    T* cur = buf0 + (rr & 1) * B::SIZE;
    if (rr + 1 < kFinRows) {
      const int64_t bn = base_of(kw_nxt);
      reg_stage<T, E, SPAN, FULL>(buf0 + ((rr + 1) & 1) * B::SIZE, R, Ro, row_of(rr + 1), bn, m, wo.n, lane);
      pre = fin_pre<SPAN>(w, wo, o, oo, row_of(rr + 1), bn, lane);
    }
    cp_async_commit();
    kw_cur = kw_nxt;
    kw_nxt = key_word(keys, row_of(rr + 2 < kFinRows ? rr + 2 : kFinRows - 1), words);
    cp_async_wait1();
    __syncwarp();
    int64_t kb = 0;
    const bool has = key_arg(kw, words, &kb);
    const int64_t b = has ? kb : 0;
    const double mi = cu.mi;
    // ---- the SPAN candidate dot products, in registers --------------------------------------
    const T* xi = cur;
    const T* xo = cur + B::XI;
    double a[E], wv[E + SPAN - 1];
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int s = E * lane + e;
      a[e] = (FULL || s < m) ? (double)xi[pad_pos<E>(s)] - mi : 0.0;
    }
#pragma unroll
    for (int t = 0; t < E + SPAN - 1; ++t) wv[t] = (double)xo[pad_pos<E>(E * lane + t)];
    double acc[SPAN], asum = 0.0;
#pragma unroll
    for (int d = 0; d < SPAN; ++d) acc[d] = 0.0;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      asum += a[e];
#pragma unroll
      for (int d = 0; d < SPAN; ++d) acc[d] = fma(a[e], wv[e + d], acc[d]);
    }
#pragma unroll
    for (int q = 16; q > 0; q >>= 1) asum += __shfl_xor_sync(0xffffffffu, asum, q);
    xsum<SPAN>(acc, lane);
    int d = xidx<SPAN>(lane);
    double dd = inf;
    const int64_t jd = b + d;
    if (admissible(i, jd, wo.n_sub, excl)) {
      if (cu.fc) {
        dd = (double)m;
      } else {
        const double cov = acc[0] - cu.mc * asum;
        dd = 2.0 * m - (2.0 * cov) * (cu.ii * cu.ic);
      }
    }
    // argmin over the SPAN candidates: the 32 / SPAN lanes of a candidate hold the same value
    // (xidx ignores the low lane bits), so only the high log2(SPAN) butterfly rounds are needed
#pragma unroll
    for (int q = 16; q >= 32 / SPAN; q >>= 1) {
      const double od = __shfl_xor_sync(0xffffffffu, dd, q);
      const int oi = __shfl_xor_sync(0xffffffffu, d, q);
      if (od < dd || (od == dd && oi < d)) {
        dd = od;
        d = oi;
      }
    }
    const int64_t jr = dd < inf ? b + d : -1;
    // the chosen member's statistics from the lane that prefetched them
    const int src = xlane<SPAN>(jr >= 0 ? d : 0);
    const double mj = __shfl_sync(0xffffffffu, cu.mc, src);
    const double ij = __shfl_sync(0xffffffffu, cu.ic, src);
    const bool fj = __shfl_sync(0xffffffffu, (int)cu.fc, src) != 0;
    // ---- the chosen member's distance: sqrt(dd) from the centred FP64 dot product, and for a
    // near neighbour (dd < 1, where the cancellation in 2m - 2 cov / (sigma sigma) would show)
    // recomputed by explicit differences (Def. 3); warp-uniform branch ------------------------
    const bool exact = jr >= 0 && !fj;
    const int de = exact ? d : 0;
    double pe = sqrt(dd > 0.0 ? dd : 0.0);
    if (exact && dd < kFinExplicitBelow) {
      const double ii = cu.ii;
      double acc2 = 0.0;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int s = E * lane + e;
        const double zi = __dmul_rn(a[e], ii);
        const double zj = __dmul_rn((double)xo[pad_pos<E>(s + de)] - mj, ij);
        const double df = zi - zj;
        acc2 = (FULL || s < m) ? __dadd_rn(acc2, __dmul_rn(df, df)) : acc2;
      }
#pragma unroll
      for (int q = 16; q > 0; q >>= 1) acc2 += __shfl_xor_sync(0xffffffffu, acc2, q);
      pe = sqrt(acc2);
    }
    double p;
    int64_t j;
    if (cu.fi) {
      const int64_t f = smallest_adm_flat(F, nf, i, excl);
      if (f >= 0) {
        p = 0.0;
        j = f;
      } else {
        p = sqm;
        j = (excl < 0 || i - excl - 1 >= 0) ? 0 : i + excl + 1;
      }
    } else if (!has) {
      p = nan;
      j = -1;
    } else {
      j = jr;
      p = jr < 0 ? nan : (exact ? pe : sqm);
      if (nf > 0) {
        const int64_t f = smallest_adm_flat(F, nf, i, excl);
        if (f >= 0 && (sqm < p || (sqm == p && f < j) || j < 0)) {
          p = sqm;
          j = f;
        }
      }
    }
    if (lane == 0 && live) {
      P[(int64_t)g * w.n_sub + i] = (T)p;
      I[(int64_t)g * w.n_sub + i] = j;
    }
    __syncwarp();  // this buffer is refilled two rows later
  }
}

// ---- sub-warp variant: LPR = 16 or 8 lanes per row, 32 / LPR rows per warp ---------------------
// The register kernel above spends ~590 warp instructions per row of which only 64 are the
// DFMAs of the SPAN dot products: the rest is per-row scalar work (key decode, statistics,
// staging addresses, the reductions, the argmin, flat handling, the store) that every lane of
// the warp executes for the one row.  Here a group of LPR lanes owns a row (lane l of the group
// holds the E = m / LPR consecutive positions [E l, E l + E)), so every such instruction serves
// 32 / LPR rows; the DFMA count per row is unchanged and the reductions need fewer butterfly
// rounds.  Each lane's E positions sit contiguously in its group's buffer, the lanes' runs 16
// bytes apart (padded position s + PAD (s / E), PAD = 16 / sizeof(T)), so the row and candidate
// values are read with 128-bit shared loads at a 16-byte-aligned stride of E + PAD elements:
// the 8 lanes of a quarter-warp phase hit 8 distinct 4-bank groups (conflict-free).  Shuffles
// never leave a group (xor offsets < LPR, sources inside the group); the rare explicit-
// difference pass is entered by the whole warp when any group needs it.
template <typename T, int E, int LPR, int SPAN> struct HwBuf {
  static constexpr int PAD = 16 / (int)sizeof(T);
  static constexpr int VEC = 16 / (int)sizeof(T);                 // elements per 128-bit load
  static constexpr int NI = LPR * E;                              // row window positions (>= m)
  static constexpr int NO = LPR * E + SPAN - 1;                   // candidate positions
  static constexpr int padded(int s) { return s + PAD * (s / E); }
  static constexpr int up(int x) { return (x + PAD - 1) / PAD * PAD; }
  static constexpr int XI = up(padded(NI - 1) + 1);
  static constexpr int XO = up(padded(NO - 1) + 1 + VEC);         // + VEC: the last vector may overrun
  static constexpr int HS = XI + XO;                              // elements per row buffer
  static constexpr int NW = (E + SPAN - 1 + VEC - 1) / VEC;       // candidate vectors per lane
};
// FP32 with 8 lanes per row: the 4 rows of a warp are consecutive, so their row windows are one
// super-window of m + 3 values staged once per warp (XR elements, same padding); each group keeps
// its own candidate buffer (XO).  Per-warp stage size WS.
#ifndef SKMP_FIN_SHR
#define SKMP_FIN_SHR 1
#endif
template <typename T, int LPR> struct HwShared { static constexpr bool on = SKMP_FIN_SHR && sizeof(T) == 4 && LPR == 8; };
template <typename T, int E, int LPR, int SPAN> struct HwLayout {
  using B = HwBuf<T, E, LPR, SPAN>;
  static constexpr int G = 32 / LPR;
  static constexpr bool SHR = HwShared<T, LPR>::on;
  static constexpr int XR = B::up(B::padded(LPR * E + G - 2) + 1);
  static constexpr int WS = SHR ? XR + G * B::XO : G * B::HS;
};
template <int LPR> struct HwCta { static constexpr int W = LPR == 8 ? 2 : 4; };  // warps per CTA

// stage row i's window and the candidate windows of base b into one group's buffer: lane l of
// the group copies positions l + LPR q (padded: l + PAD (l / E) + LPR q + PAD ((LPR q) / E), a
// lane base plus compile-time offsets); tails stay zero from the kernel start (see reg_stage)
template <typename T, int E, int LPR, int SPAN, bool FULL>
__device__ __forceinline__ void hw_stage_row(T* xr, const T* R, int64_t i, int m, int l) {
  using B = HwBuf<T, E, LPR, SPAN>;
  static_assert(E % LPR == 0 || LPR % E == 0, "E and LPR must divide one another");
  T* xi = xr + l + B::PAD * (l / E);
  const T* gi = R + i + l;
#pragma unroll
  for (int q = 0; q < E; ++q)
    if (FULL || l + LPR * q < m) cp_async_b(xi + LPR * q + B::PAD * ((LPR * q) / E), gi + LPR * q, (int)sizeof(T));
}
// the warp's shared row super-window: positions [i0, i0 + m + G - 1) of R (< n), lane-strided
template <typename T, int E, int LPR, int SPAN>
__device__ __forceinline__ void hw_stage_superrow(T* xr, const T* R, int64_t i0, int m, int64_t n, int lane) {
  using B = HwBuf<T, E, LPR, SPAN>;
  constexpr int G = 32 / LPR, NQ = (LPR * E + G - 1 + 31) / 32;
  static_assert(32 % E == 0 || E % 32 == 0, "E and 32 must divide one another");
  T* x = xr + lane + B::PAD * (lane / E);
  const T* gi = R + i0 + lane;
  const int lim = (int)((n - i0) < (int64_t)(m + G - 1) ? (n - i0) : (int64_t)(m + G - 1));
#pragma unroll
  for (int q = 0; q < NQ; ++q)
    if (lane + 32 * q < lim) cp_async_b(x + 32 * q + B::PAD * ((32 * q) / E), gi + 32 * q, (int)sizeof(T));
}
template <typename T, int E, int LPR, int SPAN, bool FULL>
__device__ __forceinline__ void hw_stage_cand(T* xc, const T* Ro, int64_t b, int m, int64_t n_o, int l) {
  using B = HwBuf<T, E, LPR, SPAN>;
  T* xo = xc + l + B::PAD * (l / E);
  const int no_used = FULL ? LPR * E + SPAN - 1 : m + SPAN - 1;  // (FULL: m = LPR E, compile-time masks)
  constexpr int NQ = (B::NO + LPR - 1) / LPR;
  if (b >= 0 && b + no_used <= n_o) {
    const T* go = Ro + b + l;
#pragma unroll
    for (int q = 0; q < NQ; ++q)
      if (l + LPR * q < no_used) cp_async_b(xo + LPR * q + B::PAD * ((LPR * q) / E), go + LPR * q, (int)sizeof(T));
  } else {
    const int32_t ob = (int32_t)b, no = (int32_t)n_o;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const int t = l + LPR * q;
      if (t < no_used) {
        int32_t idx = ob + t;
        idx = idx < 0 ? 0 : (idx >= no ? no - 1 : idx);
        cp_async_b(xo + LPR * q + B::PAD * ((LPR * q) / E), Ro + idx, (int)sizeof(T));
      }
    }
  }
}

// fin_pre with 32-bit window indices from per-series base pointers (n_sub < 2^31)
struct FinBase {
  const double *mu, *isig;
  const unsigned char* flat;
};
template <int SPAN, int LPR>
__device__ __forceinline__ FinPre fin_pre32(const FinBase& r, const FinBase& c, int32_t i, int32_t b, int32_t nso,
                                            int l) {
  FinPre p;
  p.mi = r.mu[i];
  p.ii = r.isig[i];
  p.fi = r.flat[i] != 0;
  int32_t jc = b + xidx<SPAN, LPR>(l);
  jc = jc < 0 ? 0 : (jc >= nso ? nso - 1 : jc);
  p.mc = c.mu[jc];
  p.ic = c.isig[jc];
  p.fc = c.flat[jc] != 0;
  return p;
}

// VEC consecutive staged values as doubles (one 128-bit shared load)
template <typename T> __device__ __forceinline__ void ld_vec(const T* p, double* o);
template <> __device__ __forceinline__ void ld_vec<float>(const float* p, double* o) {
  const float4 v = *reinterpret_cast<const float4*>(p);
  o[0] = v.x;
  o[1] = v.y;
  o[2] = v.z;
  o[3] = v.w;
}
template <> __device__ __forceinline__ void ld_vec<double>(const double* p, double* o) {
  const double2 v = *reinterpret_cast<const double2*>(p);
  o[0] = v.x;
  o[1] = v.y;
}

#ifndef SKMP_FIN_HW_MINB
#define SKMP_FIN_HW_MINB 4  // (x 128 threads) 128 registers
#endif
template <typename T, int SPAN, int E, int LPR, bool FULL>
__global__ void __launch_bounds__(32 * HwCta<LPR>::W, SKMP_FIN_HW_MINB * 4 / HwCta<LPR>::W)
finalize_hw_kernel(MpDev w, MpDev wo, int excl, int64_t row_lo, int64_t row_hi, T* __restrict__ P,
                   int64_t* __restrict__ I) {
  static_assert(SPAN <= LPR && (SPAN & (SPAN - 1)) == 0, "geometry");
  using B = HwBuf<T, E, LPR, SPAN>;
  using Lay = HwLayout<T, E, LPR, SPAN>;
  constexpr int G = 32 / LPR, WPC = HwCta<LPR>::W, VEC = B::VEC;
  constexpr bool SHR = Lay::SHR;
  static_assert(E % VEC == 0, "E must be a multiple of the vector width");
  __shared__ __align__(16) T fsm[WPC * 2 * Lay::WS];
  const int lane = threadIdx.x & 31, grp = lane / LPR, l = lane % LPR;
  T* wb0 = fsm + (threadIdx.x >> 5) * 2 * Lay::WS;  // this warp's stage 0; stage 1 at + WS
  // row / candidate buffers of this group in stage k
  auto rowbuf = [&](int k) { return wb0 + k * Lay::WS + (SHR ? 0 : grp * B::HS); };
  auto candbuf = [&](int k) { return wb0 + k * Lay::WS + (SHR ? Lay::XR + grp * B::XO : grp * B::HS + B::XI); };
  const int64_t i_first = row_lo + ((int64_t)blockIdx.x * WPC + (threadIdx.x >> 5)) * (G * kFinRows);
  const int g = blockIdx.y;
  const int words = (w.dtype == SKMP_F32) ? 1 : 2;
  const int64_t* keys = w.keys + (int64_t)g * w.n_sub * words;
  const int64_t o = (int64_t)g * w.ldq, oo = (int64_t)g * wo.ldq;
  const T* R = static_cast<const T*>(w.R) + (int64_t)g * w.ld;
  const T* Ro = static_cast<const T*>(wo.R) + (int64_t)g * wo.ld;
  const int m = w.m;
  const double sqm = sqrt((double)m);
  const double inf = __longlong_as_double(0x7ff0000000000000ll), nan = __longlong_as_double(0x7ff8000000000000ll);
  const int32_t nf = wo.nflat[g];
  const int32_t* F = wo.flat_list + (int64_t)g * wo.n_sub;
  // group grp walks rows i_first + G rr + grp
  auto row_of = [&](int rr) { const int64_t x = i_first + G * rr + grp; return x < row_hi ? x : row_hi - 1; };
  auto base_of = [&](int64_t kw) { int64_t kb = 0; return key_arg(kw, words, &kb) ? kb : (int64_t)0; };
  const FinBase rbase{w.mu + o, w.isig64 + o, w.flat + o}, cbase{wo.mu + oo, wo.isig64 + oo, wo.flat + oo};
  const int32_t nso = (int32_t)wo.n_sub;
  // clamping b to [-32, n_sub] first keeps clamp(b + x, 0, n_sub - 1) for x < 32 (32-bit safe)
  auto b32 = [nso](int64_t b) { return (int32_t)(b < -32 ? -32 : (b > nso ? (int64_t)nso : b)); };
  int64_t kw_cur = key_word(keys, row_of(0), words);
  int64_t kw_nxt = key_word(keys, row_of(1), words);
  for (int q = lane; q < 2 * Lay::WS; q += 32) wb0[q] = (T)0;  // tails stay zero
  __syncwarp();
  // the warp's first row of step rr (SHR: the super-window's origin; group grp's row is at + r)
  auto row0_of = [&](int rr) { const int64_t x = i_first + G * rr; return x < row_hi ? x : row_hi - 1; };
  auto stage = [&](int k, int rr, int64_t bb) {
    if constexpr (SHR) hw_stage_superrow<T, E, LPR, SPAN>(rowbuf(k), R, row0_of(rr), m, w.n, lane);
    else hw_stage_row<T, E, LPR, SPAN, FULL>(rowbuf(k), R, row_of(rr), m, l);
    hw_stage_cand<T, E, LPR, SPAN, FULL>(candbuf(k), Ro, bb, m, wo.n, l);
  };
  stage(0, 0, base_of(kw_cur));
  cp_async_commit();
  FinPre pre = fin_pre32<SPAN, LPR>(rbase, cbase, (int32_t)row_of(0), b32(base_of(kw_cur)), nso, l);
  for (int rr = 0; rr < kFinRows; ++rr) {
    const int64_t i_raw = i_first + G * rr + grp;
    const bool live = i_raw < row_hi;
    const int64_t i = row_of(rr);
    const int64_t kw = kw_cur;
    const FinPre cu = pre;
    const T* crow = rowbuf(rr & 1);
    const T* ccand = candbuf(rr & 1);
    if (rr + 1 < kFinRows) {
      const int64_t bn = base_of(kw_nxt);
      stage((rr + 1) & 1, rr + 1, bn);
      pre = fin_pre32<SPAN, LPR>(rbase, cbase, (int32_t)row_of(rr + 1), b32(bn), nso, l);
    }
    cp_async_commit();
    kw_cur = kw_nxt;
    kw_nxt = key_word(keys, row_of(rr + 2 < kFinRows ? rr + 2 : kFinRows - 1), words);
    cp_async_wait1();
    __syncwarp();
    int64_t kb = 0;
    const bool has = key_arg(kw, words, &kb);
    const int64_t b = has ? kb : 0;
    const double mi = cu.mi;
    // ---- the SPAN candidate dot products over this lane's E positions -----------------------
    const T* xo = ccand + (E + B::PAD) * l;   // position E l + t at (E + PAD) l + t + PAD (t / E)
    double a[E], wv[B::NW * VEC];
    if constexpr (SHR) {
      // row position E l + e of group grp is super-window position r + E l + e, r = i - i0 < G:
      // padded (E + PAD) l + r + e (+ PAD once r + e >= E, i.e. only for e >= E - G + 1)
      const int r = (int)(i - row0_of(rr));
      const T* xi = crow + (E + B::PAD) * l + r;
#pragma unroll
      for (int e = 0; e < E; ++e) a[e] = (double)xi[e + (e >= E - G + 1 && r + e >= E ? B::PAD : 0)];
    } else {
      const T* xi = crow + (E + B::PAD) * l;  // position E l + e at (E + PAD) l + e
#pragma unroll
      for (int e = 0; e < E; e += VEC) ld_vec<T>(xi + e, a + e);
    }
#pragma unroll
    for (int c = 0; c < B::NW; ++c) ld_vec<T>(xo + c * VEC + B::PAD * ((c * VEC) / E), wv + c * VEC);
    double acc[SPAN], asum = 0.0;
#pragma unroll
    for (int d = 0; d < SPAN; ++d) acc[d] = 0.0;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      a[e] = (FULL || E * l + e < m) ? a[e] - mi : 0.0;
      asum += a[e];
#pragma unroll
      for (int d = 0; d < SPAN; ++d) acc[d] = fma(a[e], wv[e + d], acc[d]);
    }
#pragma unroll
    for (int q = LPR / 2; q > 0; q >>= 1) asum += __shfl_xor_sync(0xffffffffu, asum, q);
    xsum<SPAN, LPR>(acc, l);
    int d = xidx<SPAN, LPR>(l);
    double dd = inf;
    const int64_t jd = b + d;
    if (admissible(i, jd, wo.n_sub, excl)) {
      if (cu.fc) {
        dd = (double)m;
      } else {
        const double cov = acc[0] - cu.mc * asum;
        dd = 2.0 * m - (2.0 * cov) * (cu.ii * cu.ic);
      }
    }
    // argmin over the SPAN candidates (LPR / SPAN lanes of a group hold each)
#pragma unroll
    for (int q = LPR / 2; q >= LPR / SPAN; q >>= 1) {
      const double od = __shfl_xor_sync(0xffffffffu, dd, q);
      const int oi = __shfl_xor_sync(0xffffffffu, d, q);
      if (od < dd || (od == dd && oi < d)) {
        dd = od;
        d = oi;
      }
    }
    const int64_t jr = dd < inf ? b + d : -1;
    const int src = grp * LPR + xlane<SPAN, LPR>(jr >= 0 ? d : 0);
    const double mj = __shfl_sync(0xffffffffu, cu.mc, src);
    const double ij = __shfl_sync(0xffffffffu, cu.ic, src);
    const bool fj = __shfl_sync(0xffffffffu, (int)cu.fc, src) != 0;
    const bool exact = jr >= 0 && !fj;
    const int de = exact ? d : 0;
    double pe = sqrt(dd > 0.0 ? dd : 0.0);
    const bool need = exact && dd < kFinExplicitBelow;
    if (__any_sync(0xffffffffu, need)) {  // whole warp (the reduction shuffles span every group)
      const double ii = cu.ii;
      double acc2 = 0.0;
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const int s = E * l + e;
        const double zi = __dmul_rn(a[e], ii);
        const double zj = __dmul_rn((double)ccand[B::padded(s + de)] - mj, ij);
        const double df = zi - zj;
        acc2 = (FULL || s < m) ? __dadd_rn(acc2, __dmul_rn(df, df)) : acc2;
      }
#pragma unroll
      for (int q = LPR / 2; q > 0; q >>= 1) acc2 += __shfl_xor_sync(0xffffffffu, acc2, q);
      if (need) pe = sqrt(acc2);
    }
    double p;
    int64_t j;
    if (cu.fi) {
      const int64_t f = smallest_adm_flat(F, nf, i, excl);
      if (f >= 0) {
        p = 0.0;
        j = f;
      } else {
        p = sqm;
        j = (excl < 0 || i - excl - 1 >= 0) ? 0 : i + excl + 1;
      }
    } else if (!has) {
      p = nan;
      j = -1;
    } else {
      j = jr;
      p = jr < 0 ? nan : (exact ? pe : sqm);
      if (nf > 0) {
        const int64_t f = smallest_adm_flat(F, nf, i, excl);
        if (f >= 0 && (sqm < p || (sqm == p && f < j) || j < 0)) {
          p = sqm;
          j = f;
        }
      }
    }
    if (l == 0 && live) {
      P[(int64_t)g * w.n_sub + i] = (T)p;
      I[(int64_t)g * w.n_sub + i] = j;
    }
    __syncwarp();  // this buffer is refilled two rows later
  }
}

bool fin_reg_enabled() {
  static const bool on = [] {
    const char* e = getenv("SKMP_FIN_IMPL");  // "smem": the shared-memory variant (A/B)
    return !(e && e[0] == 's');
  }();
  return on;
}
#ifndef SKMP_FIN_HW
#define SKMP_FIN_HW 1
#endif
int fin_lpr() {
  static const int v = [] {
    const char* e = getenv("SKMP_FIN_LPR");  // lanes per row of the FP32 sub-warp kernel (A/B)
    return (e && atoi(e) == 16) ? 16 : 8;
  }();
  return v;
}
bool fin_hw_enabled() {
  static const bool on = [] {
    const char* e = getenv("SKMP_FIN_IMPL");  // "reg": the full-warp register kernel (A/B)
    return SKMP_FIN_HW && !(e && (e[0] == 'r' || e[0] == 's'));
  }();
  return on;
}

}  // namespace

cudaError_t launch_mp_finalize(const MpDev& w, const MpDev& wo, int excl, void* P, int64_t* I,
                               cudaStream_t st, int64_t row_lo, int64_t row_hi) {
  if (row_hi < 0) row_hi = w.n_sub;
  if (row_hi <= row_lo) return cudaSuccess;
  const int64_t per = (int64_t)kFinWarps * kFinRows;
  dim3 grid((unsigned)((row_hi - row_lo + per - 1) / per), (unsigned)w.k);
  const int nt = 32 * kFinWarps;
  const bool f32 = w.dtype == SKMP_F32;
#define SKMP_FIN(TT, SP) finalize_kernel<TT, SP><<<grid, nt, 0, st>>>(w, wo, excl, row_lo, row_hi, static_cast<TT*>(P), I)
  // FP32: 8 lanes per row (E = m / 8 <= 32), or 16 with SKMP_FIN_LPR=16; FP64: 16 lanes per row
  // (E <= 8); longer FP64 windows keep the full-warp kernel (the static shared-memory limit)
  if ((f32 ? w.m <= 256 : w.m <= 128) && (w.span == 4 || w.span == 8) && fin_hw_enabled()) {
    const int lpr = f32 ? fin_lpr() : 16;
    const int Eh = (w.m + lpr - 1) / lpr <= 4 ? 4 : ((w.m + lpr - 1) / lpr <= 8 ? 8 : ((w.m + lpr - 1) / lpr <= 16 ? 16 : 32));
    const int wpc = lpr == 8 ? HwCta<8>::W : HwCta<16>::W;
    const int64_t perh = (int64_t)wpc * (32 / lpr) * kFinRows;
    grid.x = (unsigned)((row_hi - row_lo + perh - 1) / perh);
    const int nth = 32 * wpc;
#define SKMP_FINH(TT, SP, EE, LL)                                                                               \
  do {                                                                                                          \
    if (w.m == (LL) * (EE))                                                                                     \
      finalize_hw_kernel<TT, SP, EE, LL, true><<<grid, nth, 0, st>>>(w, wo, excl, row_lo, row_hi, static_cast<TT*>(P), I); \
    else                                                                                                        \
      finalize_hw_kernel<TT, SP, EE, LL, false><<<grid, nth, 0, st>>>(w, wo, excl, row_lo, row_hi, static_cast<TT*>(P), I); \
  } while (0)
    if (!f32) {
      if (w.span == 8) { if (Eh == 4) SKMP_FINH(double, 8, 4, 16); else SKMP_FINH(double, 8, 8, 16); }
      else { if (Eh == 4) SKMP_FINH(double, 4, 4, 16); else SKMP_FINH(double, 4, 8, 16); }
    } else if (lpr == 16) {
      if (w.span == 8) {
        if (Eh == 4) SKMP_FINH(float, 8, 4, 16); else if (Eh == 8) SKMP_FINH(float, 8, 8, 16); else SKMP_FINH(float, 8, 16, 16);
      } else {
        if (Eh == 4) SKMP_FINH(float, 4, 4, 16); else if (Eh == 8) SKMP_FINH(float, 4, 8, 16); else SKMP_FINH(float, 4, 16, 16);
      }
    } else {
      if (w.span == 8) {
        if (Eh <= 8) SKMP_FINH(float, 8, 8, 8); else if (Eh == 16) SKMP_FINH(float, 8, 16, 8); else SKMP_FINH(float, 8, 32, 8);
      } else {
        if (Eh <= 8) SKMP_FINH(float, 4, 8, 8); else if (Eh == 16) SKMP_FINH(float, 4, 16, 8); else SKMP_FINH(float, 4, 32, 8);
      }
    }
#undef SKMP_FINH
    count_launches(1);
    return cudaGetLastError();
  }
  const int E = w.m <= 64 ? 2 : (w.m <= 128 ? 4 : (w.m <= 256 ? 8 : 0));
  if (E > 0 && (w.span == 4 || w.span == 8) && fin_reg_enabled()) {
    const int64_t perr = (int64_t)kFinRegWarps * kFinRows;
    grid.x = (unsigned)((row_hi - row_lo + perr - 1) / perr);
    const int ntr = 32 * kFinRegWarps;
#define SKMP_FINR(TT, SP, EE)                                                                                    \
  do {                                                                                                          \
    if (w.m == 32 * (EE))                                                                                       \
      finalize_reg_kernel<TT, SP, EE, true><<<grid, ntr, 0, st>>>(w, wo, excl, row_lo, row_hi, static_cast<TT*>(P), I); \
    else                                                                                                        \
      finalize_reg_kernel<TT, SP, EE, false><<<grid, ntr, 0, st>>>(w, wo, excl, row_lo, row_hi, static_cast<TT*>(P), I); \
  } while (0)
    if (w.span == 8) {
      if (E == 2) { if (f32) SKMP_FINR(float, 8, 2); else SKMP_FINR(double, 8, 2); }
      else if (E == 4) { if (f32) SKMP_FINR(float, 8, 4); else SKMP_FINR(double, 8, 4); }
      else { if (f32) SKMP_FINR(float, 8, 8); else SKMP_FINR(double, 8, 8); }
    } else {
      if (E == 2) { if (f32) SKMP_FINR(float, 4, 2); else SKMP_FINR(double, 4, 2); }
      else if (E == 4) { if (f32) SKMP_FINR(float, 4, 4); else SKMP_FINR(double, 4, 4); }
      else { if (f32) SKMP_FINR(float, 4, 8); else SKMP_FINR(double, 4, 8); }
    }
    count_launches(1);
    return cudaGetLastError();
  }
#undef SKMP_FINR
  switch (w.span) {
    case 4:
      if (f32) SKMP_FIN(float, 4); else SKMP_FIN(double, 4);
      break;
    case 8:
      if (f32) SKMP_FIN(float, 8); else SKMP_FIN(double, 8);
      break;
    case 16:
      if (f32) SKMP_FIN(float, 16); else SKMP_FIN(double, 16);
      break;
    default:
      return cudaErrorInvalidValue;
  }
#undef SKMP_FIN
  count_launches(1);
  return cudaGetLastError();
}

}  // namespace skmp

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
//  * Index tracking costs NOTHING per cell: row and column maxima are plain FMNMX(3) trees over
//    rho values, and a published candidate carries the smallest index of its D-cell set (a row's
//    D cells in one thread, or a column's D cells in one thread).  mp_final.cu resolves the set
//    exactly: it evaluates the (<= D) admissible neighbours of the winning set in FP64 and keeps
//    the nearest (smallest index on ties), so the FP32 recurrence only decides which thread's
//    set wins (near-ties across sets are documented ties).
//  * Row maxima reduce over a thread's D slots; column maxima reduce over the D rows a column
//    spends in a thread.  Each row / column candidate is compared with a shared-memory copy of
//    the global best ("check then atomic"): only improvements reach the global 64-bit atomicMax
//    (FP32: packed {orderable rho, ~base}) or 128-bit CAS (FP64).
//  * Operands {df, dg, inv} of the tile's rows and columns are staged with cp.async into
//    shared memory: a ring of W + 2C columns in a swizzled [D][RS/D] layout (conflict-free
//    128-bit loads: lane t reads column base + tD) and a double-buffered chunk of rows.
//  * Every tile re-seeds its covariances exactly in FP64 at its first row (global re-seed grid:
//    tiles start at multiples of L, diagonal blocks at multiples of W), so per-cell arithmetic
//    is independent of how diagonals are split into bands/GPUs -> bit-identical keys.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "internal.h"
#include "join_common.cuh"

namespace skmp {
namespace {
using namespace join;


// Rare path: a row / column candidate beat its shared-memory threshold.  Out of line so that
// none of its address arithmetic is hoisted into the hot loop.  The published argument is the
// smallest index of the candidate's D-cell set (see mp_final.cu): row i's cells in this thread
// are j in [i + dt, i + dt + D), column c's cells are i in [c - dt - D + 1, c - dt].
template <typename T, int D>
SKMP_PUB_ATTR void publish_pair(int64_t* keys, int64_t* keysc, typename JT<T>::Q* rowq, T* cthr, int rb_u,
                                          int ct0, int ct1, int64_t i_u, int64_t dt, T rowa, T rowb,
                                          T colv0, T colv1) {
  if (rowa >= rowq[rb_u].w) {
    publish(keys, i_u, rowa, i_u + dt);
    rowq[rb_u].w = rowa;
  }
  if (rowb >= rowq[rb_u + 1].w) {
    publish(keys, i_u + 1, rowb, i_u + 1 + dt);
    rowq[rb_u + 1].w = rowb;
  }
  if (colv0 >= cthr[ct0]) {
    publish(keysc, i_u + dt, colv0, i_u - (D - 1));
    cthr[ct0] = colv0;
  }
  if (colv1 >= cthr[ct1]) {
    publish(keysc, i_u + 1 + dt, colv1, i_u + 1 - (D - 1));
    cthr[ct1] = colv1;
  }
}

template <typename T, int D, int NT, int C>
struct Geo {
  static constexpr int W = NT * D;
  static constexpr int RS = W + 2 * C;   // ring columns
  static constexpr int RSD = RS / D;     // ring rows of the swizzled [D][RSD] layout
  static_assert(RS % D == 0, "ring must be a multiple of D");
  static_assert(C % (2 * D) == 0, "chunk must hold whole pairs of D-row rotations");
  static_assert((C & (C - 1)) == 0, "C must be a power of two (row buffer index masking)");
  using Q = typename JT<T>::Q;
  static constexpr size_t smem_bytes = sizeof(Q) * (RS + 2 * C) + sizeof(T) * RS;
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

// The column ring in shared memory.  FP32 records (float4, 16 B) are read whole by consecutive
// lanes (conflict-free 128-bit loads); an FP64 record is 32 B, and lanes reading whole 32-B
// records hit every bank twice per 128-bit load (2x the wavefronts: 2.5e10 shared-load bank
// conflicts per FP64 n=2e5 join, short-scoreboard stalls 1.1 per issue), so FP64 records are
// split into two 16-B halves in two arrays, each read conflict-free.
template <typename T> struct RingView {
  typename JT<T>::Q* q;
  __device__ __forceinline__ typename JT<T>::Q load(int p) const { return q[p]; }
  __device__ __forceinline__ void stage(int p, const typename JT<T>::Q* src) const { stage_q<T>(&q[p], src); }
};
template <> struct RingView<double> {
  double2* h0;  // {df, dg} of ring slot p
  double2* h1;  // {inv, -}
  __device__ __forceinline__ dq4 load(int p) const {
    const double2 a = h0[p], b = h1[p];
    dq4 r;
    r.x = a.x;
    r.y = a.y;
    r.z = b.x;
    r.w = b.y;
    return r;
  }
  __device__ __forceinline__ void stage(int p, const dq4* src) const {
    cp_async16(&h0[p], src);
    cp_async16(&h1[p], reinterpret_cast<const char*>(src) + 16);
  }
};
template <typename T, int RS>
__device__ __forceinline__ RingView<T> ring_view(typename JT<T>::Q* base) {
  if constexpr (sizeof(T) == 8) {
    double2* h = reinterpret_cast<double2*>(base);
    return RingView<double>{h, h + RS};
  } else {
    return RingView<T>{base};
  }
}

// One rotation: D consecutive rows ib .. ib+D-1 (processed as D/2 row pairs) of this thread's D
// diagonals.  X[(u + d) % D] holds the operands of column ib + u + dt + d at row ib + u.
template <typename T, int D, int RSD, bool MASKED>
__device__ __forceinline__ void rotation(T (&cov)[D], typename JT<T>::Q (&X)[D], T (&CK)[D],
                                         const typename JT<T>::Q* rowp,
                                         RingView<T> rv, int p0, int p1,
                                         const T* cth0, typename JT<T>::Q* rowq, T* cthr, int rb, int qt,
                                         int64_t ib, int64_t dt, const int (&lim)[D],
                                         int64_t* keys, int64_t* keysc) {
  using Q = typename JT<T>::Q;
#pragma unroll
  for (int u = 0; u < D; u += 2) {
    // -- row u --
    const Q ra = rowp[u];
    X[(u + D - 1) % D] = rv.load(((u + D - 1) % D) * RSD + (u == 0 ? p0 : p1));
    T ka[D];
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const Q& x = X[(u + d) % D];
      cov[d] = fma(ra.x, x.y, cov[d]);
      cov[d] = fma(x.x, ra.y, cov[d]);
      ka[d] = (cov[d] * x.z) * ra.z;  // rho(i, j) = cov inv_j inv_i
    }
    if (MASKED) {
#pragma unroll
      for (int d = 0; d < D; ++d) ka[d] = ((int)ib + u < lim[d]) ? ka[d] : neg_inf<T>();
    }
    // -- row u+1 (its entering column reuses the register of row u's completed column) --
    const Q rbq = rowp[u + 1];
    const T colv0 = max2(CK[u % D], ka[0]);  // column ib+u+dt completes after row u
    X[u % D] = rv.load((u % D) * RSD + p1);
    T kb[D];
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const Q& x = X[(u + 1 + d) % D];
      cov[d] = fma(rbq.x, x.y, cov[d]);
      cov[d] = fma(x.x, rbq.y, cov[d]);
      kb[d] = (cov[d] * x.z) * rbq.z;
    }
    if (MASKED) {
#pragma unroll
      for (int d = 0; d < D; ++d) kb[d] = ((int)ib + u + 1 < lim[d]) ? kb[d] : neg_inf<T>();
    }
    // -- column maxima: registers x = (u + d) % D --
    const T colv1 = max3(CK[(u + 1) % D], ka[1], kb[0]);  // column ib+u+1+dt completes
#pragma unroll
    for (int d = 2; d < D - 1; ++d) CK[(u + d) % D] = max3(CK[(u + d) % D], ka[d], kb[d - 1]);
    CK[(u + D - 1) % D] = max2(ka[D - 1], kb[D - 2]);  // column entered at row u
    CK[u % D] = kb[D - 1];                              // column entered at row u+1
    // -- row maxima over the D slots --
    const T rowa = tree_max<T, D>(ka);
    const T rowb = tree_max<T, D>(kb);
    // -- check-then-publish (rare) --
    // row thresholds ride in the row records' 4th word (ra.w, rbq.w): no extra loads
    // ">=": a candidate EQUAL to the current best is published too, so exact ties always reach
    // the atomic (smallest set wins) and keys do not depend on the tile order / band split
    const bool hit = (rowa >= ra.w) | (rowb >= rbq.w) | (colv0 >= cth0[(u % D) * RSD]) |
                     (colv1 >= cth0[((u + 1) % D) * RSD]);
    if (__any_sync(0xffffffffu, hit)) {  // warp-uniform branch: no reconvergence stack
      publish_pair<T, D>(keys, keysc, rowq, cthr, rb + u, (u % D) * RSD + qt, ((u + 1) % D) * RSD + qt,
                         ib + u, dt, rowa, rowb, colv0, colv1);
    }
  }
}

// FP64 per-cell threshold tests (SKMP_F64_CELLTEST): an FP64 maximum costs a DSETP and two
// FSELs (no FP64 3-input max), so instead of reducing row and column maxima in the loop every
// cell is tested against its row's and its column's threshold with predicate-accumulating DSETPs
// (row thresholds ride in the row records' 4th word, column thresholds in the unused 4th word of
// the FP64 ring records, i.e. every threshold arrives with a load the loop already does).  A cell
// beats its row threshold iff the row maximum does, so the rare publish path reduces the row
// maxima from the cells still in registers; a column publishes each of its cells that beats the
// threshold as it is computed (the column's D-cell set has one base, so the set's maximum is
// published whatever order its cells pass in): the keys are the ones the maxima give, bit for bit.
#ifndef SKMP_F64_CELLTEST
#define SKMP_F64_CELLTEST 1
#endif
// refresh the register copies of the column thresholds after a publish (1) or leave them stale
// until the columns rotate out (0: no register shuffles around the publish branch)
#ifndef SKMP_F64_XREFRESH
#define SKMP_F64_XREFRESH 1
#endif

template <int D, int RSD_CT>
__device__ __forceinline__ void publish_ct(int64_t* keys, int64_t* keysc, dq4* rowq, double2* h1, int rbu, int u, int qt,
                              int qt1, int64_t i_u, int64_t dt, const double (&ka)[D], const double (&kb)[D],
                              dq4 (&X)[D]) {
  const double rowa = tree_max<double, D>(ka), rowb = tree_max<double, D>(kb);
  if (rowa >= rowq[rbu].w) {
    publish(keys, i_u, rowa, i_u + dt);
    rowq[rbu].w = rowa;
  }
  if (rowb >= rowq[rbu + 1].w) {
    publish(keys, i_u + 1, rowb, i_u + 1 + dt);
    rowq[rbu + 1].w = rowb;
  }
  // cells (i_u + v, c = i_u + v + dt + d), c - (ib + dt) = s = u + v + d: a column gets its
  // row pair's cells merged (one publish); ring slot s RSD + qt (s < D) or (s - D) RSD + qt1; the
  // column's rows in this thread start at c - dt - D + 1 = i_u - u + s - D + 1
#pragma unroll
  for (int s = u; s <= u + D; ++s) {
    const double x = s == u ? ka[0] : (s == u + D ? kb[D - 1] : max2(ka[s - u], kb[s - u - 1]));
    const int p = s < D ? s * RSD_CT + qt : (s - D) * RSD_CT + qt1;
    if (x >= h1[p].y) {
      publish(keysc, i_u - u + s + dt, x, i_u - u + s - (D - 1));
      h1[p].y = x;
    }
  }
  // the columns still in registers (s = u+1 .. u+D) take their current thresholds: a stale copy
  // would send the warp down this path again for cells that cannot improve the key
#if SKMP_F64_XREFRESH
#pragma unroll
  for (int s = u + 1; s <= u + D; ++s) X[s % D].w = h1[s < D ? s * RSD_CT + qt : (s - D) * RSD_CT + qt1].y;
#else
  (void)X;
#endif
}

// hit |= (k >= t) for 16 (k, t) pairs with predicate-accumulating setp (written out in PTX:
// from C++ the compiler fuses (k >= a) | (k >= b) into k >= min(a, b), a DSETP.MIN plus
// NaN-fixing selects per cell).  SKMP_F64_CHAINS independent predicate chains, OR-ed at the end:
// one chain makes the 16 DSETPs a serial dependency (each waits for the previous predicate at
// FP64 latency), which left the block's tail stalled on `wait`
#ifndef SKMP_F64_CHAINS
#define SKMP_F64_CHAINS 4
#endif
__device__ __forceinline__ bool any_ge(const double (&k)[16], const double (&t)[16]) {
  unsigned r;
#if SKMP_F64_CHAINS == 4
  asm("{ .reg .pred p0, p1, p2, p3;\n"
      "  setp.ge.f64 p0, %1, %17;\n"
      "  setp.ge.f64 p1, %2, %18;\n"
      "  setp.ge.f64 p2, %3, %19;\n"
      "  setp.ge.f64 p3, %4, %20;\n"
      "  setp.ge.or.f64 p0, %5, %21, p0;\n"
      "  setp.ge.or.f64 p1, %6, %22, p1;\n"
      "  setp.ge.or.f64 p2, %7, %23, p2;\n"
      "  setp.ge.or.f64 p3, %8, %24, p3;\n"
      "  setp.ge.or.f64 p0, %9, %25, p0;\n"
      "  setp.ge.or.f64 p1, %10, %26, p1;\n"
      "  setp.ge.or.f64 p2, %11, %27, p2;\n"
      "  setp.ge.or.f64 p3, %12, %28, p3;\n"
      "  setp.ge.or.f64 p0, %13, %29, p0;\n"
      "  setp.ge.or.f64 p1, %14, %30, p1;\n"
      "  setp.ge.or.f64 p2, %15, %31, p2;\n"
      "  setp.ge.or.f64 p3, %16, %32, p3;\n"
      "  or.pred p0, p0, p1;\n"
      "  or.pred p2, p2, p3;\n"
      "  or.pred p0, p0, p2;\n"
      "  selp.u32 %0, 1, 0, p0; }"
#else
  asm("{ .reg .pred p;\n"
      "  setp.ge.f64 p, %1, %17;\n"
      "  setp.ge.or.f64 p, %2, %18, p;\n"
      "  setp.ge.or.f64 p, %3, %19, p;\n"
      "  setp.ge.or.f64 p, %4, %20, p;\n"
      "  setp.ge.or.f64 p, %5, %21, p;\n"
      "  setp.ge.or.f64 p, %6, %22, p;\n"
      "  setp.ge.or.f64 p, %7, %23, p;\n"
      "  setp.ge.or.f64 p, %8, %24, p;\n"
      "  setp.ge.or.f64 p, %9, %25, p;\n"
      "  setp.ge.or.f64 p, %10, %26, p;\n"
      "  setp.ge.or.f64 p, %11, %27, p;\n"
      "  setp.ge.or.f64 p, %12, %28, p;\n"
      "  setp.ge.or.f64 p, %13, %29, p;\n"
      "  setp.ge.or.f64 p, %14, %30, p;\n"
      "  setp.ge.or.f64 p, %15, %31, p;\n"
      "  setp.ge.or.f64 p, %16, %32, p;\n"
      "  selp.u32 %0, 1, 0, p; }"
#endif
      : "=r"(r)
      : "d"(k[0]), "d"(k[1]), "d"(k[2]), "d"(k[3]), "d"(k[4]), "d"(k[5]), "d"(k[6]), "d"(k[7]), "d"(k[8]),
        "d"(k[9]), "d"(k[10]), "d"(k[11]), "d"(k[12]), "d"(k[13]), "d"(k[14]), "d"(k[15]), "d"(t[0]), "d"(t[1]),
        "d"(t[2]), "d"(t[3]), "d"(t[4]), "d"(t[5]), "d"(t[6]), "d"(t[7]), "d"(t[8]), "d"(t[9]), "d"(t[10]),
        "d"(t[11]), "d"(t[12]), "d"(t[13]), "d"(t[14]), "d"(t[15]));
  return r != 0;
}

template <int D, int RSD, bool MASKED>
__device__ __forceinline__ void rotation_ct(double (&cov)[D], dq4 (&X)[D], const dq4* rowp, RingView<double> rv,
                                            int p0, int p1, dq4* rowq, int rb, int qt, int64_t ib, int64_t dt,
                                            const int (&lim)[D], int64_t* keys, int64_t* keysc) {
#pragma unroll
  for (int u = 0; u < D; u += 2) {
    // -- row u --
    const dq4 ra = rowp[u];
    X[(u + D - 1) % D] = rv.load(((u + D - 1) % D) * RSD + (u == 0 ? p0 : p1));
    double ka[D], kk[4 * D], tt[4 * D];
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const dq4& x = X[(u + d) % D];
      cov[d] = fma(ra.x, x.y, cov[d]);
      cov[d] = fma(x.x, ra.y, cov[d]);
      ka[d] = (cov[d] * x.z) * ra.z;
      if (MASKED) ka[d] = ((int)ib + u < lim[d]) ? ka[d] : neg_inf<double>();
      kk[2 * d] = ka[d];
      tt[2 * d] = ra.w;
      kk[2 * d + 1] = ka[d];
      tt[2 * d + 1] = x.w;
    }
    // -- row u+1 (its entering column reuses the register of row u's completed column) --
    const dq4 rbq = rowp[u + 1];
    X[u % D] = rv.load((u % D) * RSD + p1);
    double kb[D];
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const dq4& x = X[(u + 1 + d) % D];
      cov[d] = fma(rbq.x, x.y, cov[d]);
      cov[d] = fma(x.x, rbq.y, cov[d]);
      kb[d] = (cov[d] * x.z) * rbq.z;
      if (MASKED) kb[d] = ((int)ib + u + 1 < lim[d]) ? kb[d] : neg_inf<double>();
      kk[2 * D + 2 * d] = kb[d];
      tt[2 * D + 2 * d] = rbq.w;
      kk[2 * D + 2 * d + 1] = kb[d];
      tt[2 * D + 2 * d + 1] = x.w;
    }
    // ">=": exact ties reach the atomic (keys independent of tile order / band split)
    bool hit = any_ge(*reinterpret_cast<const double(*)[16]>(kk), *reinterpret_cast<const double(*)[16]>(tt));
#pragma unroll
    for (int q = 16; q < 4 * D; q += 16)
      hit |= any_ge(*reinterpret_cast<const double(*)[16]>(kk + q), *reinterpret_cast<const double(*)[16]>(tt + q));
    if (__any_sync(0xffffffffu, hit))
      publish_ct<D, RSD>(keys, keysc, rowq, rv.h1, rb + u, u, qt, (qt + 1 == RSD) ? 0 : qt + 1, ib + u, dt, ka, kb, X);
  }
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
  const RingView<T> rv = ring_view<T, RS>(ring);
  Q* rowq = ring + RS;
  T* cthr = reinterpret_cast<T*>(rowq + 2 * C);

  // FP64 per-cell tests: column thresholds live in the ring records' 4th word (h1[p].y)
  constexpr bool CT = (sizeof(T) == 8) && SKMP_F64_CELLTEST;
  auto col_thr = [&](int p) -> T& {
    if constexpr (CT) return rv.h1[p].y; else return cthr[p];
  };
  const int tid = threadIdx.x;
  const int64_t n_sub = a.n_sub, n_sub_c = a.n_sub_c;  // rows: i < n_sub; columns: j < n_sub_c
  constexpr int words = sizeof(T) == 4 ? 1 : 2;
  const Q* q = static_cast<const Q*>(a.Q) + (int64_t)g * a.ldq;
  const Q* qc = static_cast<const Q*>(a.Qc) + (int64_t)g * a.ldqc;
  int64_t* keys = a.keys + (int64_t)g * n_sub * words;
  int64_t* keysc = a.keysc + (int64_t)g * n_sub_c * words;
  const int64_t dt = delta0 + (int64_t)tid * D;  // this thread's first diagonal

  // per-slot validity limit: cell (i, i+dt+d) is valid iff i < lim[d]
  int lim[D];
#pragma unroll
  for (int d = 0; d < D; ++d) {
    const int64_t dd = dt + d;
    lim[d] = (dd >= a.dlo && dd < a.dhi && dd < n_sub_c) ? (int)tile_rows(n_sub, n_sub_c, dd) : 0;
  }
  // diagonals cut by the band edges: every chunk of this tile needs the per-cell mask
  const bool diag_masked = (delta0 < a.dlo) || (delta0 + W > a.dhi);

  // ---- exact FP64 seed of cov(i0, i0+dt+d), pre-compensated for the first in-loop update -----
  T cov[D];
  {
    const T* R = static_cast<const T*>(a.R) + (int64_t)g * a.ld;
    const T* Rc = static_cast<const T*>(a.Rc) + (int64_t)g * a.ldc;
    const double mua = a.mu[(int64_t)g * a.ldq + i0];
    double mub[D], acc[D], w[D];
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const int64_t j = i0 + dt + d;
      mub[d] = (j < n_sub_c) ? a.muc[(int64_t)g * a.ldqc + j] : 0.0;
      acc[d] = 0.0;
    }
    const int64_t jb = i0 + dt;
#pragma unroll
    for (int d = 0; d < D - 1; ++d) w[d] = (jb + d < a.nc) ? (double)Rc[jb + d] : 0.0;
    // sum_s (R_i - mu_i)(R_j - mu_j) = sum_s (R_i - mu_i) R_j - mu_j sum_s (R_i - mu_i)
    double asum = 0.0;
    for (int s0 = 0; s0 < a.m; s0 += D) {
#pragma unroll
      for (int e = 0; e < D; ++e) {
        const int s = s0 + e;
        if (s < a.m) {
          const int64_t t = jb + s + D - 1;
          w[(e + D - 1) % D] = (t < a.nc) ? (double)Rc[t] : 0.0;
          const double av = (i0 + s < a.n) ? (double)R[i0 + s] - mua : 0.0;
          asum += av;
#pragma unroll
          for (int d = 0; d < D; ++d) acc[d] = fma(av, w[(e + d) % D], acc[d]);
        }
      }
    }
#pragma unroll
    for (int d = 0; d < D; ++d) acc[d] = fma(-mub[d], asum, acc[d]);
    const Q qi = q[i0];
#pragma unroll
    for (int d = 0; d < D; ++d) {
      const Q qj = qc[i0 + dt + d];  // padded: safe past n_sub_c
      const double adj = (double)qi.x * (double)qj.y + (double)qj.x * (double)qi.y;
      cov[d] = (T)(acc[d] - adj);
    }
  }

  // ---- prologue: stage rows [i0, i0+C) and ring columns [i0+delta0, i0+delta0+W+C) ----------
  for (int e = tid; e < W + C; e += NT) {
    const int64_t c = i0 + delta0 + e;
    rv.stage(G::pos(c), &qc[c]);
    if constexpr (!CT) cthr[G::pos(c)] = (c < n_sub_c) ? load_thr(keysc, c, (T*)nullptr) : pos_inf<T>();
  }
  for (int e = tid; e < C; e += NT) {
    const int64_t i = i0 + e;
    stage_q<T>(&rowq[i % (2 * C)], &q[i]);
  }
  cp_async_wait_all();
  // row thresholds go into the staged row records' 4th word once the copies have landed (and,
  // with CT, the column thresholds into the ring records')
  if constexpr (CT) {
    for (int e = tid; e < W + C; e += NT) {
      const int64_t c = i0 + delta0 + e;
      col_thr(G::pos(c)) = (c < n_sub_c) ? load_thr(keysc, c, (T*)nullptr) : pos_inf<T>();
    }
  }
  for (int e = tid; e < C; e += NT) {
    const int64_t i = i0 + e;
    rowq[i % (2 * C)].w = (i < n_sub) ? load_thr(keys, i, (T*)nullptr) : pos_inf<T>();
  }
  __syncthreads();  // (one warp per CTA: a warp barrier; kept generic for NT > 32)

  // column operand registers: X[(u + d) % D] holds column i + dt + d at unrolled row u
  Q X[D];
#pragma unroll
  for (int d = 0; d < D - 1; ++d) X[d] = rv.load(G::pos(i0 + dt + d));
  T CK[D];  // running column maxima, same rotation as X
#pragma unroll
  for (int d = 0; d < D; ++d) CK[d] = neg_inf<T>();

  // ring row index of column (ib + dt): qt; (ib + dt) is a multiple of D
  int qt = (int)(((i0 + dt) % RS) / D);

  for (int64_t r = i0; r < i1; r += C) {
    const int64_t rend = (r + C < i1) ? r + C : i1;
    // ---- prefetch the next chunk: rows [r+C, r+2C), columns [r+delta0+W+C, +C) --------------
    const bool more = r + C < i1;
    // each thread stages CPT columns and CPT rows of the next chunk (C = CPT * NT)
    constexpr int CPT = C / NT;
    static_assert(C % NT == 0, "chunk rows must be a multiple of the CTA size");
    T nthr_c[CPT], nthr_r[CPT];
    if (more) {
#pragma unroll
      for (int e = 0; e < CPT; ++e) {
        const int64_t nc = r + delta0 + W + C + tid + e * NT;
        rv.stage(G::pos(nc), &qc[nc]);
        nthr_c[e] = (nc < n_sub_c) ? load_thr(keysc, nc, (T*)nullptr) : pos_inf<T>();
        const int64_t nr = r + C + tid + e * NT;
        stage_q<T>(&rowq[nr % (2 * C)], &q[nr]);
        nthr_r[e] = (nr < n_sub) ? load_thr(keys, nr, (T*)nullptr) : pos_inf<T>();
      }
    }

    // ---- compute rows [r, rend) in D-row rotations of 2-row pairs ---------------------------
    // 32-bit bookkeeping only: rb = ib mod 2C (row buffer), qt = ring row of column ib + dt.
    const int nrot = (int)((rend - r) / D);
    int rb = (int)(r & (2 * C - 1));
    int64_t ib = r;
    // the chunk needs per-cell masks only where it reaches the triangle / rectangle edges
    // (i + delta >= n_sub_c, i >= n_sub) or the band's diagonal edges
    const bool cmasked = MASKED && (diag_masked || (rend - 1) + delta0 + W - 1 >= n_sub_c || rend > n_sub);
    for (int it = 0; it < nrot; ++it, ib += D) {
      const int qt1 = (qt + 1 == RSD) ? 0 : qt + 1;
      if constexpr (CT) {
        if (cmasked)
          rotation_ct<D, RSD, true>(cov, X, rowq + rb, rv, qt, qt1, rowq, rb, qt, ib, dt, lim, keys, keysc);
        else
          rotation_ct<D, RSD, false>(cov, X, rowq + rb, rv, qt, qt1, rowq, rb, qt, ib, dt, lim, keys, keysc);
      } else {
        if (cmasked)
          rotation<T, D, RSD, true>(cov, X, CK, rowq + rb, rv, qt, qt1, cthr + qt,
                                    rowq, cthr, rb, qt, ib, dt, lim, keys, keysc);
        else
          rotation<T, D, RSD, false>(cov, X, CK, rowq + rb, rv, qt, qt1, cthr + qt,
                                     rowq, cthr, rb, qt, ib, dt, lim, keys, keysc);
      }
      qt = qt1;
      rb = (rb + D) & (2 * C - 1);
    }

    // ---- land the prefetched chunk (row thresholds after the row copies landed) --------------
    cp_async_wait_all();
    if (more) {
#pragma unroll
      for (int e = 0; e < CPT; ++e) {
        col_thr(G::pos(r + delta0 + W + C + tid + e * NT)) = nthr_c[e];
        rowq[(r + C + tid + e * NT) % (2 * C)].w = nthr_r[e];
      }
    }
    __syncthreads();
  }

  // ---- epilogue: the D-1 columns still open after the last row hold partial maxima ----------
  // After row i1-1 the open columns are (i1 - 1) + dt + d for d = 1..D-1, i.e. register
  // x = d - 1 holds column i1 + dt + x.
  // (CT: every cell was tested and published as it was computed: nothing is open)
#pragma unroll
  for (int x = 0; x < (CT ? 0 : D - 1); ++x) {
    const T v = CK[x];
    const int64_t c = i1 + dt + x;
    if (c < n_sub_c && v >= cthr[G::pos(c)]) publish(keysc, c, v, c - dt - (D - 1));
  }
}

#ifndef SKMP_JOIN_MINB
#define SKMP_JOIN_MINB 20  // FP32 D=8: cap at ~96 registers -> 20 warps/SM (measured best)
#endif
#ifndef SKMP_JOIN_MINB64
#define SKMP_JOIN_MINB64 1
#endif
// FP64 joins of a few waves (C1 / C2 sizes) are latency-bound: a second instance capped at 96
// registers (18 resident warps instead of 16) runs them faster (C2-size join 2.89 -> 2.70 ms),
// while larger FP64 joins keep the 114-register instance (n = 2e5: 174.5 vs 176.6 ms;
// profiles/r2t_f64_occupancy.txt)
#ifndef SKMP_JOIN_MINB64_SMALL
#define SKMP_JOIN_MINB64_SMALL 18
#endif
constexpr int64_t kJoinSmallGrid = 16LL * 148 * 16;  // CTAs: <= 16 waves of 148 SMs x 16 warps
template <typename T, int D, int NT, int C, bool SMALL = false>
__global__ void __launch_bounds__(NT, ((sizeof(T) == 4 && D <= 8) ? SKMP_JOIN_MINB
                                       : (SMALL ? SKMP_JOIN_MINB64_SMALL : SKMP_JOIN_MINB64)))
join_kernel(JoinArgs a) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  constexpr int W = NT * D;
  __shared__ int64_t s_tile[3];
  __shared__ int s_g;
  if (threadIdx.x == 0) decode_tile(a, W, a.k, &s_g, &s_tile[0], &s_tile[1], &s_tile[2]);
  __syncthreads();
  const int g = s_g;
  const int64_t delta0 = s_tile[0], i0 = s_tile[1], i1 = s_tile[2];
  // rows are processed in whole D-row rotations; rows beyond the edges are masked cells
  const int64_t i1r = i0 + (((i1 - i0) + D - 1) / D) * D;
  join_tile<T, D, NT, C, true>(a, g, delta0, i0, i1r, smem_raw);
}

template <typename T, int D, bool SMALL = false>
cudaError_t launch_join_t(const MpDev& w, const MpDev& wc, int64_t dlo, int64_t dhi, const int64_t* prefix,
                          int64_t nblk, int64_t ntiles, int64_t blk0, cudaStream_t st) {
  constexpr int NT = kJoinNT, C = kJoinC;
  using G = Geo<T, D, NT, C>;
  const JoinArgs a = make_join_args(w, wc, dlo, dhi, prefix, nblk, blk0);
  const size_t smem = G::smem_bytes;
  cudaError_t e = cudaFuncSetAttribute(join_kernel<T, D, NT, C, SMALL>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e) return e;
  join_kernel<T, D, NT, C, SMALL><<<(unsigned)(ntiles * w.k), NT, smem, st>>>(a);
  count_launches(1);
  return cudaGetLastError();
}

}  // namespace

int join_d32() {
  static const int d = [] {
    const char* e = getenv("SKMP_JOIN_D");
    const int v = e ? atoi(e) : kJoinD32;
    return (v == 16) ? 16 : 8;
  }();
  return d;
}

cudaError_t launch_mp_join(const MpDev& w, const MpDev& wc, int64_t dlo, int64_t dhi,
                           const int64_t* d_prefix, int64_t nblk, int64_t ntiles, int64_t blk0,
                           cudaStream_t st) {
  if (ntiles <= 0) return cudaSuccess;
  if (w.dtype == SKMP_F32) {
    if (join_x2_enabled()) return launch_mp_join_x2(w, wc, dlo, dhi, d_prefix, nblk, ntiles, blk0, st);
    if (join_d32() == 16) return launch_join_t<float, 16>(w, wc, dlo, dhi, d_prefix, nblk, ntiles, blk0, st);
    return launch_join_t<float, 8>(w, wc, dlo, dhi, d_prefix, nblk, ntiles, blk0, st);
  }
  if (ntiles * w.k <= kJoinSmallGrid)
    return launch_join_t<double, kJoinD64, true>(w, wc, dlo, dhi, d_prefix, nblk, ntiles, blk0, st);
  return launch_join_t<double, kJoinD64>(w, wc, dlo, dhi, d_prefix, nblk, ntiles, blk0, st);
}

}  // namespace skmp

// K6 (FP32, the default FP32 join): the join hot loop on Blackwell's packed FP32 instructions
// (FFMA2 / FMUL2).  Self-join and both AB-join passes (row / column series, JoinArgs).
//
// Same method as mp_join.cu (Def. 6, self-join P:L322; STOMP/SCAMP recurrence
//   cov(i,j) = cov(i-1,j-1) + df_i dg_j + df_j dg_i,  rho = cov inv_i inv_j)
// but every arithmetic instruction of the recurrence works on TWO diagonals at once
// (`fma.rn.f32x2`, sm_100+), halving the issue slots the FP32 arithmetic needs (not the FMA-pipe
// time: an FFMA2 occupies the pipe for two cycles, tools/micro/pipe_mix.cu):
//  * thread t owns two groups of DG diagonals, group A = [delta0 + t DG, +DG) and group B = the
//    same + H (H = 32 DG, half the tile width W = 2H); slot d of both groups lives in one 64-bit
//    register pair, so cov, the column operands and the keys are all f32x2;
//  * the tile's columns are staged as PAIR records {df_c, df_c+H | dg_c, dg_c+H | inv_c, inv_c+H}
//    and rows as duplicated records {df_i, df_i | dg_i, dg_i | inv_i, inv_i} so every operand is a
//    ready-made f32x2 register pair (no per-cell moves);
//  * per cell: 2 FFMA2 halves (cov) + 2 FMUL2 halves (rho) = 2 packed instructions per cell, then
//    FMNMX3 trees give row and column maxima exactly as in mp_join.cu (no per-cell index work:
//    a published candidate names its DG-cell set, resolved exactly in mp_final.cu);
//  * rows/columns publish through the same check-then-atomic path (join_common.cuh).
// Bit-exact invariance to band splits holds as in mp_join.cu (global re-seed grid, W-aligned
// diagonal blocks, per-cell arithmetic independent of the band).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "internal.h"
#include "join_common.cuh"

// The rare publish path is inlined here (measured: the out-of-line call costs ~0.3 register
// moves per cell in the hot loop); SKMP_X2_PUB_INLINE=0 restores the call.
#ifndef SKMP_X2_PUB_INLINE
#define SKMP_X2_PUB_INLINE 1
#endif
#if SKMP_X2_PUB_INLINE
#define SKMP_X2_PUB_ATTR __device__ __forceinline__
#else
#define SKMP_X2_PUB_ATTR __device__ __noinline__
#endif

namespace skmp {
namespace {
using namespace join;

constexpr int NT = 32;            // one warp per CTA
#ifndef SKMP_X2_DG
#define SKMP_X2_DG 8
#endif
constexpr int DG = SKMP_X2_DG;    // diagonals per group per thread (2 DG cells per row)
constexpr int H = NT * DG;        // 128: group B offset; tile width W = 2H
constexpr int W = 2 * H;
constexpr int C = kJoinCx2;       // rows per staged chunk
constexpr int CPT = C / NT;       // rows / column records each thread stages per chunk
constexpr int RS = H + 2 * C;     // ring records
constexpr int RSD = RS / DG;
// pitch of the swizzled ring rows: RSD + 1 staggers the DG slot rows across the shared-memory
// banks (with pitch RSD every slot row starts on the same bank, and the staging cp.asyncs of 32
// consecutive columns -- one per slot row and ring row -- hit one bank group 8-way)
#ifndef SKMP_X2_PAD
#define SKMP_X2_PAD 1
#endif
constexpr int RSP = RSD + SKMP_X2_PAD;
static_assert(RS % DG == 0 && C % (2 * DG) == 0 && (C & (C - 1)) == 0 && C % NT == 0, "geometry");

// ---- f32x2 helpers (64-bit register pairs) ----------------------------------------------------
typedef unsigned long long f2;
__device__ __forceinline__ f2 pk(float lo, float hi) {
  f2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ float lo_of(f2 v) {
  float l;
  asm("{ .reg .f32 h; mov.b64 {%0, h}, %1; }" : "=f"(l) : "l"(v));
  return l;
}
__device__ __forceinline__ float hi_of(f2 v) {
  float h;
  asm("{ .reg .f32 l; mov.b64 {l, %0}, %1; }" : "=f"(h) : "l"(v));
  return h;
}
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

#ifndef SKMP_X2_ROWSCALAR
#define SKMP_X2_ROWSCALAR 1
#endif
// next chunk's column records staged raw (two 16-byte cp.asyncs per column pair) and repacked
// into the pair layout when the chunk ends, instead of six 4-byte cp.asyncs straight into it
#ifndef SKMP_X2_RAWCOL
#define SKMP_X2_RAWCOL 1
#endif
// next chunk's raw column records and row records staged by three 1-D bulk copies
// (cp.async.bulk, TMA engine) issued by one lane and completed on an mbarrier, instead of three
// 16-byte cp.asyncs per lane; the key words stay per-lane 4-byte cp.asyncs (strided)
#ifndef SKMP_X2_BULK
#define SKMP_X2_BULK 0
#endif
#if SKMP_X2_BULK && !(SKMP_X2_RAWCOL && SKMP_X2_ROWSCALAR)
#error "SKMP_X2_BULK needs SKMP_X2_RAWCOL and SKMP_X2_ROWSCALAR"
#endif
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n"
               "fence.mbarrier_init.release.cluster;\n"
               "fence.proxy.async.shared::cta;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
// the generic-proxy reads of a buffer (previous chunk) are ordered before the async-proxy writes
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{ .reg .pred p;\n"
      "WAIT_%=:\n"
      "  mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "  @!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

struct __align__(16) ColRec0 { f2 df, dg; };   // {df_c, df_c+H}, {dg_c, dg_c+H}
struct RowRec0 { f2 df, dg; };                 // {df_i, df_i}, {dg_i, dg_i}

struct Smem {
  ColRec0 col0[DG * RSP];   // swizzled [DG][RSP] (RSD used per row)
  f2 col1[DG * RSP];        // {inv_c, inv_c+H}
#if SKMP_X2_ROWSCALAR
  float4 rowq[2 * C];  // raw row records {df, dg, inv, 0}; the f32x2 row operands are formed as
                       // broadcasts {x, x}, which the FFMA2 / FMUL2 encode as .F32 scalar operands
#else
  RowRec0 row0[2 * C];
  f2 row1[2 * C];     // {inv_i, inv_i}
#endif
  float thrA[DG * RSP];     // column thresholds of group A columns (record base c)
  float thrB[DG * RSP];     // ... of group B columns (c + H)
  float rthr[2 * C];
  // next-chunk key high words (orderable rho), staged by cp.async and converted to the float
  // thresholds above when the chunk ends; the next chunk's records go straight into their ring
  // slots (free while this chunk runs) in the pair layout, 4 bytes per cp.async
  int32_t rawtA[C], rawtB[C], rawtR[C];
#if SKMP_X2_RAWCOL
  float4 rawcA[C], rawcB[C];  // next chunk's column records c and c + H, raw
#endif
};

// ring slot of column record c (0 <= c < 2^31: n_sub < 2^31, so 32-bit arithmetic suffices)
__device__ __forceinline__ int pos(int64_t c) {
  const uint32_t p = (uint32_t)c % (uint32_t)RS;
  return (int)((p % DG) * RSP + p / DG);
}

// masking limits of a thread's diagonals relative to dt (3 registers instead of 2 DG)
struct Lim {
  int lo, hi, edge;  // diagonal band [lo, hi) and column edge, relative to dt
  int rows;          // row edge: i < rows (AB-join passes; = n_sub for a self-join)
};

// per-slot operand registers
struct Col {
  f2 df, dg, inv;
};

// Register-file banks (B300_MICROARCH.md "RF banking": an instruction reads its distinct even-
// and odd-numbered source registers at one per cycle per bank, so FMNMX3 over three same-parity
// registers costs 3 cycles, a balanced one 2).  The rho pairs put group A in the even and group B
// in the odd register; SKMP_X2_BAL keeps the running column maxima as pairs {B, A}, i.e. group A's
// maximum in an ODD register and B's in an even one, so every column update max3(CA, ka, la)
// reads two of one parity and one of the other, and interleaves the row tree (tools/rf_model.py).
// How a rotation finds the ring row of its first column record (SKMP_X2_QT): 0 = a live counter
// (the allocator spills it: one LDL per rotation), 1 = recomputed from the row index ((ib+dt)/DG
// mod RSD: an IMAD.HI + IMAD on the saturated FMA pipe), 2 = a rotation counter U (wraps at RSD,
// the same for the whole warp) plus the lane: ALU-only, 3 = kept in shared memory per thread
#ifndef SKMP_X2_QT
#define SKMP_X2_QT 3
#endif
#ifndef SKMP_X2_BAL
#define SKMP_X2_BAL 1
#endif

#if SKMP_X2_BAL
struct ColMax {
  f2 v[DG];  // {B, A}
  __device__ __forceinline__ float A(int x) const { return hi_of(v[x]); }
  __device__ __forceinline__ float B(int x) const { return lo_of(v[x]); }
  __device__ __forceinline__ void set(int x, float a, float b) { v[x] = pk(b, a); }
};
#else
struct ColMax {
  float a[DG], b[DG];
  __device__ __forceinline__ float A(int x) const { return a[x]; }
  __device__ __forceinline__ float B(int x) const { return b[x]; }
  __device__ __forceinline__ void set(int x, float aa, float bb) { a[x] = aa; b[x] = bb; }
};
#endif

// row maximum of the 2 DG cells of one row (ka even registers, kb odd): the first level takes
// {e, o, e} / {o, e, o} triples, the second level's inputs are forced to opposite parities by
// packing them as pairs
__device__ __forceinline__ float row_max_bal(const float (&ka)[DG], const float (&kb)[DG]) {
  if constexpr (DG != 8) {  // generic: interleaved {a, b, a}, {b, a, b} triples at the first level
    float v[2 * DG];
#pragma unroll
    for (int d = 0; d < DG; ++d) {
      v[2 * d] = ka[d];
      v[2 * d + 1] = kb[d];
    }
    return tree_max<float, 2 * DG>(v);
  }
  const float t0 = max3(ka[0], kb[0], ka[1]), t1 = max3(kb[1], ka[2], kb[2]);
  const float t2 = max3(ka[3], kb[3], ka[4]), t3 = max3(kb[4], ka[5], kb[5]);
  const float t4 = max3(ka[6], kb[6], ka[7]);
  const f2 p = pk(t0, t1), q = pk(t2, t3);
  const float u0 = max3(lo_of(p), hi_of(p), kb[7]);
  const float u1 = max3(lo_of(q), hi_of(q), t4);
  return max2(u0, u1);
}

// Rare path (out of line): publish improved row / column candidates.  The argument is the
// smallest index of the winning D-cell set (resolved exactly in mp_final.cu): a row's set is one
// group's DG diagonals of this thread (group B when its maximum is strictly larger: ties go to
// the smaller indices of group A), a column's set is the DG rows it spent in this thread.
// GROUPS: the caller already knows whether group B holds each row's maximum (bA, bB; masked
// rotations, which keep the two group trees); otherwise the row maxima came from one 2 DG-cell
// tree and the winning group is B only when group A's own maximum falls short of it (ties to
// A's smaller indices either way)
template <bool GROUPS>
SKMP_X2_PUB_ATTR void publish_x2(int64_t* keys, int64_t* keysc, Smem* sm, int rbu, int ctA0, int ctA1,
                                        int64_t i_u, int64_t dt, float rowa, float rowb, const float (&ka)[DG],
                                        const float (&la)[DG], bool bA, bool bB, float cA0, float cA1, float cB0,
                                        float cB1) {
  if (rowa >= sm->rthr[rbu]) {
    const bool b = GROUPS ? bA : tree_max<float, DG>(ka) < rowa;
    publish(keys, i_u, rowa, i_u + dt + (b ? H : 0));
    sm->rthr[rbu] = rowa;
  }
  if (rowb >= sm->rthr[rbu + 1]) {
    const bool b = GROUPS ? bB : tree_max<float, DG>(la) < rowb;
    publish(keys, i_u + 1, rowb, i_u + 1 + dt + (b ? H : 0));
    sm->rthr[rbu + 1] = rowb;
  }
  // columns c = i + dt (A) and c + H (B) complete after row i: their rows are [i - DG + 1, i]
  if (cA0 >= sm->thrA[ctA0]) {
    publish(keysc, i_u + dt, cA0, i_u - (DG - 1));
    sm->thrA[ctA0] = cA0;
  }
  if (cA1 >= sm->thrA[ctA1]) {
    publish(keysc, i_u + 1 + dt, cA1, i_u + 1 - (DG - 1));
    sm->thrA[ctA1] = cA1;
  }
  if (cB0 >= sm->thrB[ctA0]) {
    publish(keysc, i_u + dt + H, cB0, i_u - (DG - 1));
    sm->thrB[ctA0] = cB0;
  }
  if (cB1 >= sm->thrB[ctA1]) {
    publish(keysc, i_u + 1 + dt + H, cB1, i_u + 1 - (DG - 1));
    sm->thrB[ctA1] = cB1;
  }
}

// one row: cov update + keys of both groups for the DG slots whose column registers are X[(u+d)%DG]
// (u is a loop index of fully unrolled loops, so every register index is a compile-time constant)
template <bool MASKED>
__device__ __forceinline__ void row_keys(int u, f2 (&cov)[DG], const Col (&X)[DG], const RowRec0& r0,
                                         f2 rinv, float (&ka)[DG], float (&kb)[DG],
                                         int irow, const Lim& lim) {
#pragma unroll
  for (int d = 0; d < DG; ++d) {
    const Col& x = X[(u + d) % DG];
    cov[d] = fma2(r0.df, x.dg, cov[d]);
#if SKMP_X2_ROWFIRST
    cov[d] = fma2(r0.dg, x.df, cov[d]);  // row operand in the first slot of both FFMA2s
#else
    cov[d] = fma2(x.df, r0.dg, cov[d]);
#endif
    const f2 rho = mul2(mul2(cov[d], x.inv), rinv);  // rho = cov inv_j inv_i (both groups)
    ka[d] = lo_of(rho);
    kb[d] = hi_of(rho);
  }
  if (MASKED) {
#pragma unroll
    for (int d = 0; d < DG; ++d) {
      ka[d] = (d >= lim.lo && d < lim.hi && irow + d < lim.edge && irow < lim.rows) ? ka[d] : neg_inf<float>();
      kb[d] = (d >= lim.lo - H && d < lim.hi - H && irow + d < lim.edge - H && irow < lim.rows) ? kb[d]
                                                                                                 : neg_inf<float>();
    }
  }
}

__device__ __forceinline__ void load_col(Col& x, const Smem* sm, int e) {
  x.df = sm->col0[e].df;
  x.dg = sm->col0[e].dg;
  x.inv = sm->col1[e];
}

#if SKMP_X2_ROWSCALAR
__device__ __forceinline__ RowRec0 row0_of(const float4& r) { return RowRec0{pk(r.x, r.x), pk(r.y, r.y)}; }
#define ROW0(e) row0_of(sm->rowq[(e)])
#define ROW1(e) pk(sm->rowq[(e)].z, sm->rowq[(e)].z)
#else
#define ROW0(e) sm->row0[(e)]
#define ROW1(e) sm->row1[(e)]
#endif

// One rotation = DG rows ib .. ib+DG-1 processed as DG/2 row pairs.  Column registers rotate:
// X[(u + d) % DG] holds the record of column ib + u + dt + d (group A) / + H (group B).
// CA/CB: running column maxima of the group A / B columns, same rotation.
template <bool MASKED>
__device__ __forceinline__ void rotation_x2(f2 (&cov)[DG], Col (&X)[DG], ColMax& CM,
                                            Smem* sm, int rb, int qt, int qt1, int64_t ib, int64_t dt,
                                            const Lim& lim, const JoinArgs& a, int g) {
#pragma unroll
  for (int u = 0; u < DG; u += 2) {
    // -- row u: its entering column (slot DG-1) takes the register of the column completed at u-1
    load_col(X[(u + DG - 1) % DG], sm, ((u + DG - 1) % DG) * RSP + (u == 0 ? qt : qt1));
    float ka[DG], kb[DG];
    row_keys<MASKED>(u, cov, X, ROW0(rb + u), ROW1(rb + u), ka, kb, (int)ib + u, lim);
    // columns (ib+u)+dt (A) and +H (B) complete after row u
    const float cA0 = max2(CM.A(u % DG), ka[0]);
    const float cB0 = max2(CM.B(u % DG), kb[0]);
    // -- row u+1 --
    load_col(X[u % DG], sm, (u % DG) * RSP + qt1);
    float la[DG], lb[DG];
    row_keys<MASKED>(u + 1, cov, X, ROW0(rb + u + 1), ROW1(rb + u + 1), la, lb,
                     (int)ib + u + 1, lim);
    const float cA1 = max3(CM.A((u + 1) % DG), ka[1], la[0]);
    const float cB1 = max3(CM.B((u + 1) % DG), kb[1], lb[0]);
#pragma unroll
    for (int d = 2; d < DG - 1; ++d)
      CM.set((u + d) % DG, max3(CM.A((u + d) % DG), ka[d], la[d - 1]), max3(CM.B((u + d) % DG), kb[d], lb[d - 1]));
    CM.set((u + DG - 1) % DG, max2(ka[DG - 1], la[DG - 2]), max2(kb[DG - 1], lb[DG - 2]));
    CM.set(u % DG, la[DG - 1], lb[DG - 1]);
    // -- row maxima per group --
    // -- row maxima: unmasked rotations use one tree over both groups' 2 DG cells (one
    // instruction fewer per row than two group trees and their max); masked rotations keep the
    // group trees (fewer live registers where the masks already need them) --
    float rowa, rowb;
    bool bA = false, bB = false;
    if (MASKED) {
      const float rowaA = tree_max<float, DG>(ka), rowaB = tree_max<float, DG>(kb);
      const float rowbA = tree_max<float, DG>(la), rowbB = tree_max<float, DG>(lb);
      rowa = max2(rowaA, rowaB);
      rowb = max2(rowbA, rowbB);
      bA = rowaB > rowaA;
      bB = rowbB > rowbA;
    } else {
#if SKMP_X2_BAL
      rowa = row_max_bal(ka, kb);
      rowb = row_max_bal(la, lb);
#else
      float kab[2 * DG], lab[2 * DG];
#pragma unroll
      for (int d = 0; d < DG; ++d) {
        kab[d] = ka[d];
        kab[DG + d] = kb[d];
        lab[d] = la[d];
        lab[DG + d] = lb[d];
      }
      rowa = tree_max<float, 2 * DG>(kab);
      rowb = tree_max<float, 2 * DG>(lab);
#endif
    }
    // -- check-then-publish (rare) --
    const int t0 = (u % DG) * RSP + qt, t1 = ((u + 1) % DG) * RSP + qt;
    // ">=": exact ties always reach the atomic (keys independent of tile order / band split)
    const bool hit = (rowa >= sm->rthr[rb + u]) | (rowb >= sm->rthr[rb + u + 1]) | (cA0 >= sm->thrA[t0]) |
                     (cA1 >= sm->thrA[t1]) | (cB0 >= sm->thrB[t0]) | (cB1 >= sm->thrB[t1]);
    if (__any_sync(0xffffffffu, hit)) {
      // the key pointers are rebuilt from the kernel parameters here (rare path) instead of
      // occupying registers across the hot loop
      int64_t* keys = a.keys + (int64_t)g * a.n_sub;
      int64_t* keysc = a.keysc + (int64_t)g * a.n_sub_c;
      publish_x2<MASKED>(keys, keysc, sm, rb + u, t0, t1, ib + u, dt, rowa, rowb, ka, la, bA, bB, cA0, cA1, cB0, cB1);
    }
  }
}

// stage record of base column c (columns c and c + H) and its two thresholds into registers
struct ColStage {
  float4 qa, qb;
  float ta, tb;
};
__device__ __forceinline__ void fetch_col(ColStage& s, const float4* q, const int64_t* keys, int64_t c,
                                          int64_t n_sub) {
  s.qa = __ldcg(q + c);
  s.qb = __ldcg(q + c + H);
  s.ta = (c < n_sub) ? load_thr(keys, c, (float*)nullptr) : pos_inf<float>();
  s.tb = (c + H < n_sub) ? load_thr(keys, c + H, (float*)nullptr) : pos_inf<float>();
}
__device__ __forceinline__ void land_col(const ColStage& s, Smem* sm, int64_t c) {
  const int e = pos(c);
  sm->col0[e].df = pk(s.qa.x, s.qb.x);
  sm->col0[e].dg = pk(s.qa.y, s.qb.y);
  sm->col1[e] = pk(s.qa.z, s.qb.z);
  sm->thrA[e] = s.ta;
  sm->thrB[e] = s.tb;
}
struct RowStage {
  float4 q;
  float t;
};
__device__ __forceinline__ void fetch_row(RowStage& s, const float4* q, const int64_t* keys, int64_t i,
                                          int64_t n_sub) {
  s.q = __ldcg(q + i);
  s.t = (i < n_sub) ? load_thr(keys, i, (float*)nullptr) : pos_inf<float>();
}
__device__ __forceinline__ void land_row(const RowStage& s, Smem* sm, int64_t i) {
  const int e = (int)(i & (2 * C - 1));
#if SKMP_X2_ROWSCALAR
  sm->rowq[e] = s.q;
#else
  sm->row0[e].df = pk(s.q.x, s.q.x);
  sm->row0[e].dg = pk(s.q.y, s.q.y);
  sm->row1[e] = pk(s.q.z, s.q.z);
#endif
  sm->rthr[e] = s.t;
}

__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem) : "memory");
}
// next chunk's column record c (and c + H) and row i: the records straight into their ring
// slots in the pair layout ({df_c, df_c+H}, {dg_c, dg_c+H}, {inv_c, inv_c+H}; rows duplicated),
// the key high words into the raw threshold buffers (a possibly stale L1 copy only costs an
// extra publish).  Indices are < 2^31 + W: 32-bit offsets from the series bases.
__device__ __forceinline__ void stage_next(Smem* sm, const float4* q, const int64_t* keys, const float4* qc,
                                           const int64_t* keysc, int64_t c64, int64_t i64, int64_t n_sub,
                                           int64_t n_sub_c, int e) {
  const uint32_t c = (uint32_t)c64, i = (uint32_t)i64;
  const uint32_t ns = (uint32_t)n_sub, nsc = (uint32_t)n_sub_c;
#if SKMP_X2_BULK
  (void)qc;
  (void)q;
#elif SKMP_X2_RAWCOL
  cp_async16(&sm->rawcA[e], qc + c);
  cp_async16(&sm->rawcB[e], qc + (c + H));
#else
  const float* a = reinterpret_cast<const float*>(qc + c);
  const float* b = reinterpret_cast<const float*>(qc + (c + H));
  const int ec = pos(c64);
  float* d0 = reinterpret_cast<float*>(&sm->col0[ec]);  // {df_A, df_B, dg_A, dg_B}
  float* d1 = reinterpret_cast<float*>(&sm->col1[ec]);  // {inv_A, inv_B}
  cp_async4(d0 + 0, a + 0);
  cp_async4(d0 + 1, b + 0);
  cp_async4(d0 + 2, a + 1);
  cp_async4(d0 + 3, b + 1);
  cp_async4(d1 + 0, a + 2);
  cp_async4(d1 + 1, b + 2);
#endif
  const int er = (int)(i & (2 * C - 1));
#if SKMP_X2_BULK
  (void)er;
#elif SKMP_X2_ROWSCALAR
  cp_async16(&sm->rowq[er], q + i);  // the raw record, one 16-byte copy
#else
  const float* r = reinterpret_cast<const float*>(q + i);
  float* r0 = reinterpret_cast<float*>(&sm->row0[er]);  // {df, df, dg, dg}
  float* r1 = reinterpret_cast<float*>(&sm->row1[er]);  // {inv, inv}
  cp_async4(r0 + 0, r + 0);
  cp_async4(r0 + 1, r + 0);
  cp_async4(r0 + 2, r + 1);
  cp_async4(r0 + 3, r + 1);
  cp_async4(r1 + 0, r + 2);
  cp_async4(r1 + 1, r + 2);
#endif
  const int32_t inf = 0x7f800000;  // orderable(+inf): never beaten
  if (c < nsc) cp_async4(&sm->rawtA[e], reinterpret_cast<const char*>(keysc + c) + 4); else sm->rawtA[e] = inf;
  if (c + H < nsc) cp_async4(&sm->rawtB[e], reinterpret_cast<const char*>(keysc + (c + H)) + 4); else sm->rawtB[e] = inf;
  if (i < ns) cp_async4(&sm->rawtR[e], reinterpret_cast<const char*>(keys + i) + 4); else sm->rawtR[e] = inf;
}
__device__ __forceinline__ void land_next(Smem* sm, int64_t c, int64_t i, int e) {
  const int ec = pos(c);
#if SKMP_X2_RAWCOL
  {
    const float4 ra = sm->rawcA[e], rb = sm->rawcB[e];
    ColRec0 r;
    r.df = pk(ra.x, rb.x);
    r.dg = pk(ra.y, rb.y);
    sm->col0[ec] = r;
    sm->col1[ec] = pk(ra.z, rb.z);
  }
#endif
  sm->thrA[ec] = unord32(sm->rawtA[e]);
  sm->thrB[ec] = unord32(sm->rawtB[e]);
  sm->rthr[(int)(i & (2 * C - 1))] = unord32(sm->rawtR[e]);
}

#ifndef SKMP_X2_MINB
#define SKMP_X2_MINB 16  // <= 128 registers: 16 warps / SM (measured best)
#endif
__global__ void __launch_bounds__(NT, SKMP_X2_MINB)
join_x2_kernel(JoinArgs a) {
  __shared__ Smem sm;
  __shared__ int64_t s_tile[3];
  __shared__ int s_g;
  if (threadIdx.x == 0) decode_tile(a, W, a.k, &s_g, &s_tile[0], &s_tile[1], &s_tile[2]);
  __syncwarp();
  const int g = s_g;
  const int64_t delta0 = s_tile[0], i0 = s_tile[1];
  const int64_t i1 = i0 + ((s_tile[2] - i0 + DG - 1) / DG) * DG;  // whole rotations; tail masked
  const int tid = threadIdx.x;
  const int64_t n_sub = a.n_sub, n_sub_c = a.n_sub_c;  // rows i < n_sub, columns j < n_sub_c
  const float4* q = static_cast<const float4*>(a.Q) + (int64_t)g * a.ldq;
  const float4* qc = static_cast<const float4*>(a.Qc) + (int64_t)g * a.ldqc;
  int64_t* keys = a.keys + (int64_t)g * n_sub;
  int64_t* keysc = a.keysc + (int64_t)g * n_sub_c;
  const int64_t dt = delta0 + (int64_t)tid * DG;

  // cell (i, i + dt + d) of group A is valid iff lo <= d < hi and i + d < edge (group B: d + H)
  Lim lim;
  {
    const int64_t big = (int64_t)1 << 30;
    auto clampi = [&](int64_t v) { return (int)(v < -big ? -big : (v > big ? big : v)); };
    lim.lo = clampi(a.dlo - dt);
    lim.hi = clampi(a.dhi - dt);
    lim.edge = clampi(n_sub_c - dt);
    lim.rows = clampi(n_sub);
  }
  const bool diag_masked = (delta0 < a.dlo) || (delta0 + W > a.dhi);

  // ---- exact FP64 seeds for the 2 DG diagonals, pre-compensated for the first in-loop update ----
  f2 cov[DG];
  {
    const float* R = static_cast<const float*>(a.R) + (int64_t)g * a.ld;
    const float* Rc = static_cast<const float*>(a.Rc) + (int64_t)g * a.ldc;
    const double* mu = a.mu + (int64_t)g * a.ldq;
    const double* muc = a.muc + (int64_t)g * a.ldqc;
    const double mua = mu[i0];
    double acc[2 * DG];
#pragma unroll
    for (int e = 0; e < 2 * DG; ++e) acc[e] = 0.0;
    const int64_t jb = i0 + dt;
    // sum_s (R_i - mu_i)(R_j - mu_j) = sum_s (R_i - mu_i) R_j - mu_j sum_s (R_i - mu_i): one FP64 FMA
    // per term instead of a subtraction and an FMA (the seeds are rounded to FP32 afterwards)
    double asum = 0.0;
    // fast path (every tile but those at a series' end): 16-byte aligned windows wholly inside
    // both series and m a multiple of DG -- the samples arrive as float4 loads, each DG-sample
    // step's loads issued one step ahead, column samples in a 2 DG register window
    const bool vec = ((reinterpret_cast<uintptr_t>(R + i0) | reinterpret_cast<uintptr_t>(Rc + jb)) & 15) == 0 &&
                     (a.m % DG) == 0 && a.m >= 2 * DG && jb + H + a.m + DG <= a.nc;
    bool fast = false;
    if constexpr (DG == 8) fast = __all_sync(0xffffffffu, vec);
    if constexpr (DG == 8) if (fast) {
      const float4* r4 = reinterpret_cast<const float4*>(R + i0);
      const float4* ca = reinterpret_cast<const float4*>(Rc + jb);
      const float4* cb = reinterpret_cast<const float4*>(Rc + jb + H);
      double wa[2 * DG], wb[2 * DG];
      auto put = [](double* w, float4 x, float4 y) {
        w[0] = x.x; w[1] = x.y; w[2] = x.z; w[3] = x.w; w[4] = y.x; w[5] = y.y; w[6] = y.z; w[7] = y.w;
      };
      // (DG = 8: two float4 per DG-sample step)
      put(wa, ca[0], ca[1]);
      put(wb, cb[0], cb[1]);
      float4 na0 = ca[2], na1 = ca[3], nb0 = cb[2], nb1 = cb[3], nr0 = r4[0], nr1 = r4[1];
      for (int s0 = 0; s0 < a.m; s0 += DG) {
        put(wa + DG, na0, na1);
        put(wb + DG, nb0, nb1);
        double av[DG];
        put(av, nr0, nr1);
        if (s0 + DG < a.m) {  // the next step's samples, in flight during this step's FMAs
          const int q = (s0 + 2 * DG) >> 2;
          na0 = ca[q];
          na1 = ca[q + 1];
          nb0 = cb[q];
          nb1 = cb[q + 1];
          nr0 = r4[(s0 + DG) >> 2];
          nr1 = r4[((s0 + DG) >> 2) + 1];
        }
#pragma unroll
        for (int u = 0; u < DG; ++u) {
          const double x = av[u] - mua;
          asum += x;
#pragma unroll
          for (int d = 0; d < DG; ++d) {
            acc[d] = fma(x, wa[u + d], acc[d]);
            acc[DG + d] = fma(x, wb[u + d], acc[DG + d]);
          }
        }
#pragma unroll
        for (int t = 0; t < DG; ++t) {
          wa[t] = wa[t + DG];
          wb[t] = wb[t + DG];
        }
      }
    }
    if (!fast) {
      // column samples through two register rings (group A at jb, group B at jb + H): sample
      // jb + s + d sits in slot (s + d) % DG, so each sample is loaded and converted once per
      // thread instead of once per diagonal
      double wa[DG], wb[DG];
#pragma unroll
      for (int d = 0; d < DG - 1; ++d) {
        wa[d] = (jb + d < a.nc) ? (double)Rc[jb + d] : 0.0;
        wb[d] = (jb + H + d < a.nc) ? (double)Rc[jb + H + d] : 0.0;
      }
      for (int s0 = 0; s0 < a.m; s0 += DG) {
#pragma unroll
        for (int u = 0; u < DG; ++u) {
          const int s = s0 + u;
          if (s < a.m) {
            const int64_t t = jb + s + DG - 1;
            wa[(u + DG - 1) % DG] = (t < a.nc) ? (double)Rc[t] : 0.0;
            wb[(u + DG - 1) % DG] = (t + H < a.nc) ? (double)Rc[t + H] : 0.0;
            const double av = (i0 + s < a.n) ? (double)R[i0 + s] - mua : 0.0;
            asum += av;
#pragma unroll
            for (int d = 0; d < DG; ++d) {
              acc[d] = fma(av, wa[(u + d) % DG], acc[d]);
              acc[DG + d] = fma(av, wb[(u + d) % DG], acc[DG + d]);
            }
          }
        }
      }
    }
#pragma unroll
    for (int e = 0; e < 2 * DG; ++e) {  // the column windows' means, loaded after the sums (registers)
      const int64_t j = i0 + dt + (e % DG) + (e >= DG ? H : 0);
      acc[e] = fma(-((j < n_sub_c) ? muc[j] : 0.0), asum, acc[e]);
    }
    const float4 qi = q[i0];
    float c32[2 * DG];
#pragma unroll
    for (int e = 0; e < 2 * DG; ++e) {
      const float4 qj = qc[i0 + dt + (e % DG) + (e >= DG ? H : 0)];  // padded: safe past n_sub_c
      const double adj = (double)qi.x * (double)qj.y + (double)qj.x * (double)qi.y;
      c32[e] = (float)(acc[e] - adj);
    }
#pragma unroll
    for (int d = 0; d < DG; ++d) cov[d] = pk(c32[d], c32[DG + d]);
  }

  // ---- prologue: records [i0+delta0, i0+delta0+H+C), rows [i0, i0+C) ------------------------
  for (int e = tid; e < H + C; e += NT) {
    ColStage cs;
    fetch_col(cs, qc, keysc, i0 + delta0 + e, n_sub_c);
    land_col(cs, &sm, i0 + delta0 + e);
  }
  for (int e = tid; e < C; e += NT) {
    RowStage rs;
    fetch_row(rs, q, keys, i0 + e, n_sub);
    land_row(rs, &sm, i0 + e);
  }
  __syncwarp();

  Col X[DG];
#pragma unroll
  for (int d = 0; d < DG - 1; ++d) load_col(X[d], &sm, pos(i0 + dt + d));
  ColMax CM;
#pragma unroll
  for (int d = 0; d < DG; ++d) CM.set(d, neg_inf<float>(), neg_inf<float>());
#if SKMP_X2_QT == 0
  int qt = (int)(((i0 + dt) % RS) / DG);
#elif SKMP_X2_QT == 2
  int qU = (int)(((i0 + delta0) / DG) % RSD);  // ((ib + delta0) / DG) mod RSD of the current rotation
#elif SKMP_X2_QT == 3
  __shared__ int s_qt[NT];
  s_qt[tid] = (int)(((i0 + dt) % RS) / DG);
#endif
#if SKMP_X2_BULK
  // rows i0 + C.. and columns are chunk-contiguous: i0 is a multiple of the tile length L (a
  // multiple of 64, api.cu), so a chunk's row slots (i mod 2C) never wrap
  __shared__ __align__(8) uint64_t s_bar;
  if (tid == 0) mbar_init(&s_bar, 1);
  __syncwarp();
  uint32_t bar_ph = 0;
#endif

  for (int64_t r = i0; r < i1; r += C) {
    const int64_t rend = (r + C < i1) ? r + C : i1;
    const bool more = r + C < i1;
    if (more) {
#if SKMP_X2_BULK
      if (tid == 0) {
        const int64_t c0 = r + delta0 + H + C;
        fence_async_smem();
        mbar_expect_tx(&s_bar, 3 * C * (uint32_t)sizeof(float4));
        bulk_g2s(sm.rawcA, qc + c0, C * sizeof(float4), &s_bar);
        bulk_g2s(sm.rawcB, qc + (c0 + H), C * sizeof(float4), &s_bar);
        bulk_g2s(&sm.rowq[(int)((r + C) & (2 * C - 1))], q + (r + C), C * sizeof(float4), &s_bar);
      }
#endif
#pragma unroll
      for (int p = 0; p < CPT; ++p)
        stage_next(&sm, q, keys, qc, keysc, r + delta0 + H + C + tid + p * NT, r + C + tid + p * NT, n_sub,
                   n_sub_c, tid + p * NT);
    }
    const int nrot = (int)((rend - r) / DG);
    int rb = (int)(r & (2 * C - 1));
    int64_t ib = r;
    const bool cmasked = diag_masked || (rend - 1) + delta0 + W - 1 >= n_sub_c || rend > n_sub;
    for (int it = 0; it < nrot; ++it, ib += DG) {
#if SKMP_X2_QT == 0
      const int qt1 = (qt + 1 == RSD) ? 0 : qt + 1;
#elif SKMP_X2_QT == 1
      const int qt = (int)((((uint32_t)ib + (uint32_t)dt) / DG) % RSD);
      const int qt1 = (qt + 1 == RSD) ? 0 : qt + 1;
#elif SKMP_X2_QT == 2
      int qt = qU + tid;  // tid < NT <= RSD: one conditional subtraction
      qt = qt >= RSD ? qt - RSD : qt;
      const int qt1 = (qt + 1 == RSD) ? 0 : qt + 1;
      qU = (qU + 1 == RSD) ? 0 : qU + 1;
#else
      const int qt = s_qt[tid];
      const int qt1 = (qt + 1 == RSD) ? 0 : qt + 1;
      s_qt[tid] = qt1;
#endif
      if (cmasked)
        rotation_x2<true>(cov, X, CM, &sm, rb, qt, qt1, ib, dt, lim, a, g);
      else
        rotation_x2<false>(cov, X, CM, &sm, rb, qt, qt1, ib, dt, lim, a, g);
#if SKMP_X2_QT == 0
      qt = qt1;
#endif
      rb = (rb + DG) & (2 * C - 1);
    }
    if (more) {
#if SKMP_X2_BULK
      mbar_wait(&s_bar, bar_ph);
      bar_ph ^= 1;
#endif
      cp_async_wait_all();
#pragma unroll
      for (int p = 0; p < CPT; ++p) land_next(&sm, r + delta0 + H + C + tid + p * NT, r + C + tid + p * NT, tid + p * NT);
    }
    __syncwarp();
  }

  // ---- epilogue: columns still open after the last row (DG-1 per group) ----------------------
#pragma unroll
  for (int x = 0; x < DG - 1; ++x) {
    const int64_t c = i1 + dt + x;
    const int e = pos(c);
    if (c < n_sub_c && CM.A(x) >= sm.thrA[e]) publish(keysc, c, CM.A(x), c - dt - (DG - 1));
    if (c + H < n_sub_c && CM.B(x) >= sm.thrB[e]) publish(keysc, c + H, CM.B(x), c - dt - (DG - 1));
  }
}

}  // namespace

int join_x2_width() { return W; }
int join_x2_span() { return DG; }

bool join_x2_enabled() {
  static const bool on = [] {
    const char* e = getenv("SKMP_JOIN_IMPL");
    // default; SKMP_JOIN_IMPL=scalar (or SKMP_JOIN_D=16) selects mp_join.cu's FP32 kernel
    return !(e && e[0] == 's') && join_d32() == 8;
  }();
  return on;
}

cudaError_t launch_mp_join_x2(const MpDev& w, const MpDev& wc, int64_t dlo, int64_t dhi,
                              const int64_t* prefix, int64_t nblk, int64_t ntiles, int64_t blk0,
                              cudaStream_t st) {
  const JoinArgs a = make_join_args(w, wc, dlo, dhi, prefix, nblk, blk0);
  join_x2_kernel<<<(unsigned)(ntiles * w.k), NT, 0, st>>>(a);
  count_launches(1);
  return cudaGetLastError();
}

}  // namespace skmp

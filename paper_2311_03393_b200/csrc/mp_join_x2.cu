// K6 (FP32): the self-join hot loop on Blackwell's packed FP32 pipe (FFMA2 / FMUL2).
//
// Same method as mp_join.cu (Def. 6, self-join P:L322; STOMP/SCAMP recurrence
//   cov(i,j) = cov(i-1,j-1) + df_i dg_j + df_j dg_i,  rho = cov inv_i inv_j)
// but every arithmetic instruction of the recurrence works on TWO diagonals at once
// (`fma.rn.f32x2`, sm_100+), halving the issue slots the FP32 arithmetic needs:
//  * thread t owns two groups of DG diagonals, group A = [delta0 + t DG, +DG) and group B = the
//    same + H (H = 32 DG, half the tile width W = 2H); slot d of both groups lives in one 64-bit
//    register pair, so cov, the column operands and the keys are all f32x2;
//  * the tile's columns are staged as PAIR records {df_c, df_c+H | dg_c, dg_c+H | inv_c, inv_c+H}
//    and rows as duplicated records {df_i, df_i | dg_i, dg_i | inv_i, inv_i} so every operand is a
//    ready-made f32x2 register pair (no per-cell moves);
//  * per cell: 2 FFMA2 halves (cov) + FMUL2/FFMA2 halves (rho + 2) = 2 packed instructions per
//    cell, then one IMAD appends the 3-bit slot code (d + DG g) below the key (FMA pipe, no ALU),
//    and FMNMX3 trees give row and column maxima exactly as in mp_join.cu;
//  * rows/columns publish through the same check-then-atomic path (join_common.cuh).
// Bit-exact invariance to band splits holds as in mp_join.cu (global re-seed grid, W-aligned
// diagonal blocks, per-cell arithmetic independent of the band).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>

#include "internal.h"
#include "join_common.cuh"

namespace skmp {
namespace {
using namespace join;

constexpr int NT = 32;            // one warp per CTA
#ifndef SKMP_X2_DG
#define SKMP_X2_DG 8
#endif
constexpr int DG = SKMP_X2_DG;    // diagonals per group per thread (2 DG cells per row)
constexpr unsigned KMUL = 2 * DG; // key multiplier: room for the 2*DG slot codes
constexpr unsigned KADD = 0u - 0x3F800000u * KMUL;  // (bits(y) - bits(1.0)) * KMUL, mod 2^32
constexpr int H = NT * DG;        // 128: group B offset; tile width W = 2H
constexpr int W = 2 * H;
constexpr int C = kJoinC;         // rows per staged chunk
constexpr int RS = H + 2 * C;     // ring records
constexpr int RSD = RS / DG;
static_assert(RS % DG == 0 && C % (2 * DG) == 0 && (C & (C - 1)) == 0 && C == NT, "geometry");

// ---- f32x2 helpers (64-bit register pairs) ----------------------------------------------------
typedef unsigned long long f2;
__device__ __forceinline__ f2 pk(float lo, float hi) {
  f2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ float lo_of(f2 v) {
  float l, h;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(l), "=f"(h) : "l"(v));
  return l;
}
__device__ __forceinline__ float hi_of(f2 v) {
  float l, h;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(l), "=f"(h) : "l"(v));
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

// key of one cell: y = rho + 2 in [1, 4); key = (bits(y) - bits(1.0)) * KMUL + code (IMAD, FMA pipe)
#ifndef SKMP_X2_LEA_B
#define SKMP_X2_LEA_B 0  // 1: group-B keys use an ALU shift-add (LEA) instead of the FMA-pipe IMAD
#endif
template <int code>
__device__ __forceinline__ float key_of(float y, unsigned kmul) {
  unsigned k;
  if constexpr (SKMP_X2_LEA_B && code >= DG) {
    k = __float_as_uint(y) * KMUL + (KADD + code);
  } else {
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(k) : "r"(__float_as_uint(y)), "r"(kmul), "n"(KADD + code));
  }
  return __uint_as_float(k);
}

struct __align__(16) ColRec0 { f2 df, dg; };   // {df_c, df_c+H}, {dg_c, dg_c+H}
struct RowRec0 { f2 df, dg; };                 // {df_i, df_i}, {dg_i, dg_i}

struct Smem {
  ColRec0 col0[RS];   // swizzled [DG][RSD]
  f2 col1[RS];        // {inv_c, inv_c+H}
  RowRec0 row0[2 * C];
  f2 row1[2 * C];     // {inv_i, inv_i}
  float thrA[RS];     // column thresholds of group A columns (record base c)
  float thrB[RS];     // ... of group B columns (c + H)
  float rthr[2 * C];
};

__device__ __forceinline__ int pos(int64_t c) {
  const int p = (int)(c % RS);
  return (p % DG) * RSD + p / DG;
}

// per-slot operand registers
struct Col {
  f2 df, dg, inv;
};

template <int DGX, int code0>
struct Keys {  // k[d] = key(y[d]) with code code0 + d
  __device__ static __forceinline__ void run(float* k, const float* y, unsigned eight) {
    k[0] = key_of<code0>(y[0], eight);
    Keys<DGX - 1, code0 + 1>::run(k + 1, y + 1, eight);
  }
};
template <int code0>
struct Keys<0, code0> {
  __device__ static __forceinline__ void run(float*, const float*, unsigned) {}
};

// Rare path (out of line): publish improved row / column candidates.
__device__ __noinline__ void publish_x2(int64_t* keys, Smem* sm, int rbu, int ctA0, int ctA1,
                                        int64_t i_u, int64_t dt, float rowa, float rowb,
                                        float cA0, float cA1, float cB0, float cB1) {
  auto jrow = [&](float v, int64_t i) {
    const int s = __float_as_int(v) & (2 * DG - 1);
    return i + dt + (s & (DG - 1)) + (s >= DG ? H : 0);
  };
  if (rowa > sm->rthr[rbu]) {
    publish(keys, i_u, rowa, jrow(rowa, i_u));
    sm->rthr[rbu] = rowa;
  }
  if (rowb > sm->rthr[rbu + 1]) {
    publish(keys, i_u + 1, rowb, jrow(rowb, i_u + 1));
    sm->rthr[rbu + 1] = rowb;
  }
  // group A column c = i + dt (completes after row i): its cells have codes d = c - i' - dt
  if (cA0 > sm->thrA[ctA0]) {
    const int64_t c = i_u + dt;
    publish(keys, c, cA0, c - dt - (__float_as_int(cA0) & (2 * DG - 1)));
    sm->thrA[ctA0] = cA0;
  }
  if (cA1 > sm->thrA[ctA1]) {
    const int64_t c = i_u + 1 + dt;
    publish(keys, c, cA1, c - dt - (__float_as_int(cA1) & (2 * DG - 1)));
    sm->thrA[ctA1] = cA1;
  }
  if (cB0 > sm->thrB[ctA0]) {
    const int64_t c = i_u + dt + H;
    publish(keys, c, cB0, c - dt - H - ((__float_as_int(cB0) & (2 * DG - 1)) - DG));
    sm->thrB[ctA0] = cB0;
  }
  if (cB1 > sm->thrB[ctA1]) {
    const int64_t c = i_u + 1 + dt + H;
    publish(keys, c, cB1, c - dt - H - ((__float_as_int(cB1) & (2 * DG - 1)) - DG));
    sm->thrB[ctA1] = cB1;
  }
}

// one row: cov update + keys of both groups for the DG slots whose column registers are X[(u+d)%DG]
// (u is a loop index of fully unrolled loops, so every register index is a compile-time constant)
template <bool MASKED>
__device__ __forceinline__ void row_keys(int u, f2 (&cov)[DG], const Col (&X)[DG], const RowRec0& r0,
                                         f2 rinv, float (&ka)[DG], float (&kb)[DG], unsigned eight,
                                         int irow, const int (&limA)[DG], const int (&limB)[DG]) {
  const f2 two = pk(2.0f, 2.0f);
  float ya[DG], yb[DG];
#pragma unroll
  for (int d = 0; d < DG; ++d) {
    const Col& x = X[(u + d) % DG];
    cov[d] = fma2(r0.df, x.dg, cov[d]);
    cov[d] = fma2(x.df, r0.dg, cov[d]);
    const f2 y = fma2(mul2(cov[d], x.inv), rinv, two);
    ya[d] = lo_of(y);
    yb[d] = hi_of(y);
  }
  Keys<DG, 0>::run(ka, ya, eight);
  Keys<DG, DG>::run(kb, yb, eight);
  if (MASKED) {
#pragma unroll
    for (int d = 0; d < DG; ++d) {
      ka[d] = (irow < limA[d]) ? ka[d] : neg_inf<float>();
      kb[d] = (irow < limB[d]) ? kb[d] : neg_inf<float>();
    }
  }
}

__device__ __forceinline__ void load_col(Col& x, const Smem* sm, int e) {
  x.df = sm->col0[e].df;
  x.dg = sm->col0[e].dg;
  x.inv = sm->col1[e];
}

// One rotation = DG rows ib .. ib+DG-1 processed as DG/2 row pairs.  Column registers rotate:
// X[(u + d) % DG] holds the record of column ib + u + dt + d (group A) / + H (group B).
// CA/CB: running column maxima of the group A / B columns, same rotation.
template <bool MASKED>
__device__ __forceinline__ void rotation_x2(f2 (&cov)[DG], Col (&X)[DG], float (&CA)[DG], float (&CB)[DG],
                                            Smem* sm, int rb, int qt, int qt1, int64_t ib, int64_t dt,
                                            const int (&limA)[DG], const int (&limB)[DG],
                                            int64_t* keys, unsigned eight) {
#pragma unroll
  for (int u = 0; u < DG; u += 2) {
    // -- row u: its entering column (slot DG-1) takes the register of the column completed at u-1
    load_col(X[(u + DG - 1) % DG], sm, ((u + DG - 1) % DG) * RSD + (u == 0 ? qt : qt1));
    float ka[DG], kb[DG];
    row_keys<MASKED>(u, cov, X, sm->row0[rb + u], sm->row1[rb + u], ka, kb, eight, (int)ib + u, limA, limB);
    // columns (ib+u)+dt (A) and +H (B) complete after row u
    const float cA0 = max2(CA[u % DG], ka[0]);
    const float cB0 = max2(CB[u % DG], kb[0]);
    // -- row u+1 --
    load_col(X[u % DG], sm, (u % DG) * RSD + qt1);
    float la[DG], lb[DG];
    row_keys<MASKED>(u + 1, cov, X, sm->row0[rb + u + 1], sm->row1[rb + u + 1], la, lb, eight,
                     (int)ib + u + 1, limA, limB);
    const float cA1 = max3(CA[(u + 1) % DG], ka[1], la[0]);
    const float cB1 = max3(CB[(u + 1) % DG], kb[1], lb[0]);
#pragma unroll
    for (int d = 2; d < DG - 1; ++d) {
      CA[(u + d) % DG] = max3(CA[(u + d) % DG], ka[d], la[d - 1]);
      CB[(u + d) % DG] = max3(CB[(u + d) % DG], kb[d], lb[d - 1]);
    }
    CA[(u + DG - 1) % DG] = max2(ka[DG - 1], la[DG - 2]);
    CB[(u + DG - 1) % DG] = max2(kb[DG - 1], lb[DG - 2]);
    CA[u % DG] = la[DG - 1];
    CB[u % DG] = lb[DG - 1];
    // -- row maxima over both groups' slots --
    float ra8[2 * DG], rb8[2 * DG];
#pragma unroll
    for (int d = 0; d < DG; ++d) {
      ra8[d] = ka[d];
      ra8[DG + d] = kb[d];
      rb8[d] = la[d];
      rb8[DG + d] = lb[d];
    }
    const float rowa = tree_max<float, 2 * DG>(ra8);
    const float rowb = tree_max<float, 2 * DG>(rb8);
    // -- check-then-publish (rare) --
    const int t0 = (u % DG) * RSD + qt, t1 = ((u + 1) % DG) * RSD + qt;
    const bool hit = (rowa > sm->rthr[rb + u]) | (rowb > sm->rthr[rb + u + 1]) | (cA0 > sm->thrA[t0]) |
                     (cA1 > sm->thrA[t1]) | (cB0 > sm->thrB[t0]) | (cB1 > sm->thrB[t1]);
    if (__any_sync(0xffffffffu, hit))
      publish_x2(keys, sm, rb + u, t0, t1, ib + u, dt, rowa, rowb, cA0, cA1, cB0, cB1);
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
  sm->row0[e].df = pk(s.q.x, s.q.x);
  sm->row0[e].dg = pk(s.q.y, s.q.y);
  sm->row1[e] = pk(s.q.z, s.q.z);
  sm->rthr[e] = s.t;
}

#ifndef SKMP_X2_MINB
#define SKMP_X2_MINB 1
#endif
__global__ void __launch_bounds__(NT, SKMP_X2_MINB)
join_x2_kernel(JoinArgs a) {
  __shared__ Smem sm;
  __shared__ int64_t s_tile[3];
  const int g = blockIdx.y;
  if (threadIdx.x == 0) decode_tile(a, W, &s_tile[0], &s_tile[1], &s_tile[2]);
  __syncwarp();
  const int64_t delta0 = s_tile[0], i0 = s_tile[1];
  const int64_t i1 = i0 + ((s_tile[2] - i0 + DG - 1) / DG) * DG;  // whole rotations; tail masked
  const int tid = threadIdx.x;
  const int64_t n_sub = a.n_sub;
  const float4* q = static_cast<const float4*>(a.Q) + (int64_t)g * a.ldq;
  int64_t* keys = a.keys + (int64_t)g * n_sub;
  const int64_t dt = delta0 + (int64_t)tid * DG;

  int limA[DG], limB[DG];
#pragma unroll
  for (int d = 0; d < DG; ++d) {
    const int64_t da = dt + d, db = dt + d + H;
    limA[d] = (da >= a.dlo && da < a.dhi && da < n_sub) ? (int)(n_sub - da) : 0;
    limB[d] = (db >= a.dlo && db < a.dhi && db < n_sub) ? (int)(n_sub - db) : 0;
  }
  const bool diag_masked = (delta0 < a.dlo) || (delta0 + W > a.dhi);

  // ---- exact FP64 seeds for the 2 DG diagonals, pre-compensated for the first in-loop update ----
  f2 cov[DG];
  {
    const float* R = static_cast<const float*>(a.R) + (int64_t)g * a.ld;
    const double* mu = a.mu + (int64_t)g * a.ldq;
    const double mua = mu[i0];
    double acc[2 * DG], mub[2 * DG];
#pragma unroll
    for (int e = 0; e < 2 * DG; ++e) {
      const int64_t j = i0 + dt + (e % DG) + (e >= DG ? H : 0);
      mub[e] = (j < n_sub) ? mu[j] : 0.0;
      acc[e] = 0.0;
    }
    for (int s = 0; s < a.m; ++s) {
      const double av = (double)R[i0 + s] - mua;
#pragma unroll
      for (int e = 0; e < 2 * DG; ++e) {
        const int64_t t = i0 + dt + (e % DG) + (e >= DG ? H : 0) + s;
        const double bv = (t < a.n) ? (double)R[t] : 0.0;
        acc[e] = fma(av, bv - mub[e], acc[e]);
      }
    }
    const float4 qi = q[i0];
    float c32[2 * DG];
#pragma unroll
    for (int e = 0; e < 2 * DG; ++e) {
      const float4 qj = q[i0 + dt + (e % DG) + (e >= DG ? H : 0)];  // padded: safe past n_sub
      const double adj = (double)qi.x * (double)qj.y + (double)qj.x * (double)qi.y;
      c32[e] = (float)(acc[e] - adj);
    }
#pragma unroll
    for (int d = 0; d < DG; ++d) cov[d] = pk(c32[d], c32[DG + d]);
  }

  // ---- prologue: records [i0+delta0, i0+delta0+H+C), rows [i0, i0+C) ------------------------
  for (int e = tid; e < H + C; e += NT) {
    ColStage cs;
    fetch_col(cs, q, keys, i0 + delta0 + e, n_sub);
    land_col(cs, &sm, i0 + delta0 + e);
  }
  {
    RowStage rs;
    fetch_row(rs, q, keys, i0 + tid, n_sub);
    land_row(rs, &sm, i0 + tid);
  }
  __syncwarp();

  Col X[DG];
#pragma unroll
  for (int d = 0; d < DG - 1; ++d) load_col(X[d], &sm, pos(i0 + dt + d));
  float CA[DG], CB[DG];
#pragma unroll
  for (int d = 0; d < DG; ++d) CA[d] = CB[d] = neg_inf<float>();
  const unsigned eight = a.eight;  // runtime 8: keeps the key multiply an IMAD (FMA pipe)
  int qt = (int)(((i0 + dt) % RS) / DG);

  for (int64_t r = i0; r < i1; r += C) {
    const int64_t rend = (r + C < i1) ? r + C : i1;
    const bool more = r + C < i1;
    ColStage cs;
    RowStage rs;
    if (more) {  // next chunk: record r+delta0+H+C+tid, row r+C+tid
      fetch_col(cs, q, keys, r + delta0 + H + C + tid, n_sub);
      fetch_row(rs, q, keys, r + C + tid, n_sub);
    }
    const int nrot = (int)((rend - r) / DG);
    int rb = (int)(r & (2 * C - 1));
    int64_t ib = r;
    const bool cmasked = diag_masked || (rend - 1) + delta0 + W - 1 >= n_sub;
    for (int it = 0; it < nrot; ++it, ib += DG) {
      const int qt1 = (qt + 1 == RSD) ? 0 : qt + 1;
      if (cmasked)
        rotation_x2<true>(cov, X, CA, CB, &sm, rb, qt, qt1, ib, dt, limA, limB, keys, eight);
      else
        rotation_x2<false>(cov, X, CA, CB, &sm, rb, qt, qt1, ib, dt, limA, limB, keys, eight);
      qt = qt1;
      rb = (rb + DG) & (2 * C - 1);
    }
    if (more) {
      land_col(cs, &sm, r + delta0 + H + C + tid);
      land_row(rs, &sm, r + C + tid);
    }
    __syncwarp();
  }

  // ---- epilogue: columns still open after the last row (DG-1 per group) ----------------------
#pragma unroll
  for (int x = 0; x < DG - 1; ++x) {
    const int64_t c = i1 + dt + x;
    const int e = pos(c);
    if (c < n_sub && CA[x] > sm.thrA[e]) publish(keys, c, CA[x], c - dt - (__float_as_int(CA[x]) & (2 * DG - 1)));
    if (c + H < n_sub && CB[x] > sm.thrB[e])
      publish(keys, c + H, CB[x], c - dt - ((__float_as_int(CB[x]) & (2 * DG - 1)) - DG));
  }
}

}  // namespace

int join_x2_width() { return W; }

bool join_x2_enabled() {
  static const bool on = [] {
    const char* e = getenv("SKMP_JOIN_IMPL");
    return e && e[0] == 'x';  // opt-in ("x2"); measured slower than mp_join.cu on B200
  }();
  return on;
}

cudaError_t launch_mp_join_x2(const MpDev& w, int64_t dlo, int64_t dhi, const int64_t* prefix,
                              int64_t nblk, int64_t ntiles, int64_t blk0, cudaStream_t st) {
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
  a.eight = KMUL;
  dim3 grid((unsigned)ntiles, (unsigned)w.k);
  join_x2_kernel<<<grid, NT, 0, st>>>(a);
  count_launches(1);
  return cudaGetLastError();
}

}  // namespace skmp

// Internal declarations shared by the C-ABI layer (api.cu) and the kernel files.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "sketchmp.h"

namespace skmp {

// Device allocation from the library's own stream-ordered WORK pool (api.cu); freed with
// cudaFreeAsync.  Every library allocation goes through it (or the staging pool), never the
// process's default pool.
cudaError_t dmalloc(void** p, size_t bytes, cudaStream_t st);

// ------------------------------------------------------------------------------------------
// error plumbing
// ------------------------------------------------------------------------------------------
skmp_status set_error(skmp_status s, const std::string& msg, int64_t index = -1);
skmp_status cuda_error(cudaError_t e, const char* where);

#define SKMP_CUDA(call)                                            \
  do {                                                             \
    cudaError_t e__ = (call);                                      \
    if (e__ != cudaSuccess) return ::skmp::cuda_error(e__, #call); \
  } while (0)

#define SKMP_CHECK_LAUNCH(name)                                    \
  do {                                                             \
    cudaError_t e__ = cudaGetLastError();                          \
    if (e__ != cudaSuccess) return ::skmp::cuda_error(e__, name);  \
  } while (0)

// ------------------------------------------------------------------------------------------
// constants shared by host and device code
// ------------------------------------------------------------------------------------------
constexpr double kFlatEps = 1e-12;  // readings 4/5

// Join geometry (see mp_join.cu).  The tile width W = NT*D diagonals is also the band
// rounding unit of mp_band; rows per chunk C; a tile spans `reseed_rows` rows.
constexpr int kJoinNT = 32;   // one warp per CTA: no CTA-wide barriers in the hot loop
constexpr int kJoinD32 = 8;    // default diagonals per thread (FP32); 16 selectable (SKMP_JOIN_D)
#ifndef SKMP_JOIN_D64
#define SKMP_JOIN_D64 4
#endif
constexpr int kJoinD64 = SKMP_JOIN_D64;  // diagonals per thread of the FP64 join (4 | 8)
#ifndef SKMP_JOIN_C
#define SKMP_JOIN_C 32
#endif
constexpr int kJoinC = SKMP_JOIN_C;  // rows per staged chunk (power of two, multiple of 2D)
#ifndef SKMP_X2_C
#define SKMP_X2_C 32
#endif
constexpr int kJoinCx2 = SKMP_X2_C;  // rows per staged chunk of the packed FP32 join
int join_d32();                // diagonals per thread of the FP32 join (env SKMP_JOIN_D: 8 | 16)
bool join_x2_enabled();        // packed f32x2 FP32 join (default; SKMP_JOIN_IMPL=scalar disables)
int join_x2_width();           // its tile width
inline int join_width(int dtype) {
  if (dtype == SKMP_F32 && join_x2_enabled()) return join_x2_width();
  return kJoinNT * (dtype == SKMP_F64 ? kJoinD64 : join_d32());
}
// candidate-set span of a published profile key: the join publishes the smallest index of a
// thread's D-cell set, mp_final.cu resolves the set (FP32 scalar: D; x2: its per-group slots)
int join_x2_span();
inline int join_span(int dtype) {
  if (dtype == SKMP_F32 && join_x2_enabled()) return join_x2_span();
  return dtype == SKMP_F64 ? kJoinD64 : join_d32();
}
// rows of a diagonal block whose smallest diagonal is dmin: cells (i, i + delta) need
// i < n_sub_r and i + delta < n_sub_c
inline __host__ __device__ int64_t tile_rows(int64_t n_sub_r, int64_t n_sub_c, int64_t dmin) {
  const int64_t a = n_sub_c - dmin;
  return a < n_sub_r ? a : n_sub_r;
}
// FP32 profile keys store (candidate-set base + kKeyArgBias) so that bases down to -(D-1) fit
constexpr int64_t kKeyArgBias = 32;
// padding (in windows) behind n_sub in the prepared arrays so tile loops may over-read
inline int64_t join_pad(int dtype) {
  return join_width(dtype) + 4 * (kJoinC > kJoinCx2 ? kJoinC : kJoinCx2) + 64;
}

// ------------------------------------------------------------------------------------------
// stream-statistics (K1) and projection (K2/K2d/K3) launchers — sketch.cu
// ------------------------------------------------------------------------------------------
struct StatsOut {  // device arrays of length d
  double* mu;
  double* sigma;
  double* inv;     // 1/sigma
  int32_t* flag;   // 0 ok, 1 nonfinite, 2 constant
};
// Computes per-row stats of T (d x ld) over n samples.  ws must hold stats_ws_bytes(d, n).
size_t stats_ws_bytes(int64_t d, int64_t n);
cudaError_t launch_stream_stats(const void* T, int64_t d, int64_t n, int64_t ld, int dtype,
                                StatsOut out, void* ws, cudaStream_t st);

// Count sketch projection: for each group g, R64[g,:] (+)= sum over list entries e in
// [off[g], off[g+1]) of sign[e] * ((T[row[e], :] - mu[e]) * inv[e]).  `mode`: 0 = overwrite
// (build), +1 = add into R64, -1 = subtract from R64.  Then R = dtype(R64) when R != R64.
struct CsrPlan {
  const int32_t* off;    // k+1
  const int32_t* row;    // rows of T
  const double* mu;      // per entry
  const double* inv;     // per entry
  const int8_t* sign;    // per entry
};
cudaError_t launch_project_count(const void* T, int64_t ld, int64_t n, int dtype, int k,
                                 CsrPlan plan, int mode, double* R64, void* R, int64_t ldr, cudaStream_t st);
// Dense projection: R64[g,:] (+)= sum_j S[g*ldS + j] * ((T[j,:] - mu[j]) * inv[j]).
cudaError_t launch_project_dense(const void* T, int64_t ld, int64_t n, int dtype, int k,
                                 int64_t nstreams, const double* S, int64_t ldS, const double* mu,
                                 const double* inv, int mode, double* R64, void* R, int64_t ldr,
                                 cudaStream_t st);

// ------------------------------------------------------------------------------------------
// matrix profile (K4-K7) — mp_prep.cu, mp_join.cu, mp_final.cu
// ------------------------------------------------------------------------------------------
struct MpDev {
  int dtype;
  int k;
  int64_t n, ld, n_sub, ldq;  // ldq: stride (windows) of the prepared arrays per series
  int m, excl, L;             // L = reseed rows (tile height)
  int span;                   // candidate-set span of a key (join_span)
  const void* R;              // k x ld (dtype)
  void* Q;                    // k x ldq x {df, dg, inv, 0} (dtype)
  double* mu;                 // k x ldq
  double* sig64;              // k x ldq  window population std (FP64)
  double* isig64;             // k x ldq  1 / sig64 (FP64, one IEEE division; inf for sigma = 0)
  uint8_t* flat;              // k x ldq
  double* amax;               // k
  int32_t* nflat;             // k
  int64_t* keys;              // k x n_sub x words
  int32_t* flat_list;         // k x n_sub (filled only for series with nflat > 0)
};
// series per join chunk: as many as keep the chunk's operand records, window means and keys
// (row and column side) within ~48 MB of the 126 MB L2
inline int join_series_chunk(const MpDev& wr, const MpDev& wc) {
  const double rec = wr.dtype == SKMP_F32 ? 16.0 : 32.0;
  const double words = wr.dtype == SKMP_F32 ? 8.0 : 16.0;
  auto side = [&](const MpDev& w) { return (rec + 8.0) * (double)w.ldq + words * (double)w.n_sub; };
  const double per = side(wr) + (&wr == &wc ? 0.0 : side(wc));
  int G = (int)(48.0e6 / per);
  if (G < 1) G = 1;
  if (G > wr.k) G = wr.k;
  return G;
}
cudaError_t launch_mp_prep(const MpDev& w, cudaStream_t st);
cudaError_t launch_keys_init(const MpDev& w, cudaStream_t st);
// band join of row series w against column series wc (the same workspace for a self-join):
// cells (i, i + delta), delta in [dlo, dhi), tiles described by blocks of W diagonals
cudaError_t launch_mp_join(const MpDev& w, const MpDev& wc, int64_t dlo, int64_t dhi,
                           const int64_t* d_tile_prefix, int64_t nblk, int64_t ntiles, int64_t blk0,
                           cudaStream_t st);
// packed f32x2 FP32 join (mp_join_x2.cu), the default FP32 join
cudaError_t launch_mp_join_x2(const MpDev& w, const MpDev& wc, int64_t dlo, int64_t dhi,
                              const int64_t* d_tile_prefix, int64_t nblk, int64_t ntiles, int64_t blk0,
                              cudaStream_t st);
// per-series sorted flat-window lists (w.flat_list, k x n_sub) for the series whose device count
// w.nflat is non-zero (the others' kernels exit at once)
cudaError_t launch_flat_lists(const MpDev& w, cudaStream_t st);
// rows of w resolved against neighbours in wo (self-join: wo = w, excl >= 0; AB-join: excl = -1)
// (rows [row_lo, row_hi) only; row_hi < 0 -> all rows)
cudaError_t launch_mp_finalize(const MpDev& w, const MpDev& wo, int excl, void* P, int64_t* I,
                               cudaStream_t st, int64_t row_lo = 0, int64_t row_hi = -1);

// ------------------------------------------------------------------------------------------
// detection (K8) — detect.cu
// ------------------------------------------------------------------------------------------
cudaError_t launch_combine(const void* P, int64_t ldp, int k, int64_t n_sub, int dtype,
                           const uint8_t* d_inert, double* C, int32_t* G, cudaStream_t st);
// top-K greedy over C (double, n_sub); result rows (t, g, nn, score) into d_res (int64 x 4 per
// entry, score bit-cast), count into d_count.
cudaError_t launch_topk(double* C, const int32_t* G, const int64_t* I, int64_t ldi, int64_t n_sub,
                        int top, int radius, int64_t* d_res, int32_t* d_count, void* ws,
                        size_t ws_bytes, cudaStream_t st);
size_t topk_ws_bytes(int64_t n_sub);

// Alg. 3 dimension detection (K9) — dims.cu.  d_rows [dev] nrows; score/nn [dev] nrows.
size_t dims_ws_bytes(int64_t nrows, int64_t n, int m);
cudaError_t launch_dims(const void* X, int64_t ld, int64_t n, int dtype, const int64_t* d_rows,
                        int64_t nrows, int64_t t_star, int m, int excl, double* score, int64_t* nn,
                        void* ws, cudaStream_t st);

// kernel-launch accounting (skmp_launch_count): every launcher reports its launches
void count_launches(int64_t n);

// §3.3 point updates: R64[idx[q]] += coef[q] * delta[q], then R[idx] = dtype(R64[idx]) (all [dev])
// f4 streaming (stream.cu): FP64 train records {df, dg, inv, 0} once per stream, then the AB rows
// of each push's new test windows carried from the previous push (ring of per-diagonal covariances)
constexpr int kStreamReseed = 8192;     // exact FP64 re-seed grid of the carried covariances (rows, 2^k)
#ifndef SKMP_STREAM_INCR_MAX
#define SKMP_STREAM_INCR_MAX 32
#endif
constexpr int kStreamIncrMax = SKMP_STREAM_INCR_MAX;      // pushes of up to this many windows take the carried path (measured crossover)
size_t stream_q64_bytes(const MpDev& tr);
// *flag = min(*flag, g) for every group g with a non-finite value in R64[g, col0 : col0 + ncols)
cudaError_t launch_nonfinite_check(const double* R64, int64_t ld, int k, int64_t col0, int64_t ncols, int32_t* flag,
                                   cudaStream_t st);
cudaError_t launch_train_q64(const MpDev& tr, void* q64, cudaStream_t st);
cudaError_t launch_stream_rows(const MpDev& te, int64_t base, const MpDev& tr, const void* q64,
                               const double* ring_in, double* ring_out, int64_t t0, int B, bool valid,
                               cudaStream_t st);
cudaError_t launch_point_update(double* R64, void* R, int dtype, const int64_t* idx, const double* coef,
                                const double* delta, int64_t count, cudaStream_t st);

// R = dtype(R64) (sketch_refresh)
cudaError_t launch_cast_r(const double* R64, void* R, int64_t count, int dtype, cudaStream_t st);

// host hash (hash.cpp)
void cw_params(uint64_t seed, uint64_t* a, uint64_t* b, uint64_t* c, uint64_t* e);
void hash_plan(const uint64_t* ids, int64_t d, int32_t k, uint64_t seed, int32_t* g, int8_t* s);

}  // namespace skmp

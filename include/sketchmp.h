/* sketchmp.h — C-ABI of the B200-native sketch + matrix-profile hot path of
 * "Sketching Multidimensional Time Series for Fast Discord Mining" (arXiv 2311.03393).
 *
 * Citation key: "P:L<a>-<b>" = PAPER.md lines (section / definition / algorithm given);
 * "reading N" = the numbered paper-gap readings in DESIGN.md §3.
 *
 * General rules (all entry points):
 *  - Every call returns skmp_status; nothing throws, exits or prints.  On a non-OK status
 *    skmp_last_error() holds a thread-local message and skmp_last_error_index() the offending
 *    stream / group / row (or -1).  All argument validation happens before any launch; on an
 *    error status caller-owned output buffers are left untouched.
 *  - "stream" is a cudaStream_t passed as void* (NULL = legacy default stream).  Device work is
 *    enqueued on it in order.  Calls documented as "synchronous" wait for their own work.
 *  - Pointers tagged [dev] must be device (HBM) memory of the current CUDA device; [host] must be
 *    host memory; [dev|host] accepts either (detected with cudaPointerGetAttributes; a host
 *    buffer is staged to HBM inside the call, which then is synchronous).
 *  - Matrices are row-major: element (r, c) of a rows x cols matrix with leading dimension ld
 *    lives at base[r*ld + c]; ld is in elements.
 *  - dtype: SKMP_F32 or SKMP_F64 gives the element type of T, R and P; FP32 paths accumulate
 *    the sketch and all window statistics in FP64 (reading 14).
 *  - There is no CPU fallback: without a CUDA device every compute call returns SKMP_E_CUDA.
 */
#ifndef SKETCHMP_H
#define SKETCHMP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SKMP_ABI_VERSION 1

typedef enum {
  SKMP_OK = 0,
  SKMP_E_INVALID_ARG = 1,      /* NULL, d<1, k<1, m<2, ld<n, top<1, bad dtype/proj/band     */
  SKMP_E_CONSTANT_SERIES = 2,  /* sigma_j <= 1e-12 (max|x|+1)            reading 4   */
  SKMP_E_NONFINITE = 3,        /* NaN/Inf in an input stream                                  */
  SKMP_E_SERIES_TOO_SHORT = 4, /* n < m                                     (Def. 2)   */
  SKMP_E_NO_ADMISSIBLE = 5,    /* n_sub < 2*excl+2: some row has no |i-j| > excl  reading 7   */
  SKMP_E_DUPLICATE_DIM = 6,    /* id already in the sketch      */
  SKMP_E_UNKNOWN_DIM = 7,      /* delete of an id that is not in the sketch                   */
  SKMP_E_LENGTH_MISMATCH = 8,  /* added/deleted streams must span the full n     */
  SKMP_E_ALL_GROUPS_INERT = 9, /* every sketch group empty or flat         reading 10         */
  SKMP_E_CUDA = 10,            /* CUDA runtime error (incl. no device)                         */
  SKMP_E_NCCL = 11,            /* NCCL failure or libnccl missing (native multi-GPU calls)    */
  SKMP_E_OOM = 12              /* device allocation failed                                     */
} skmp_status;

typedef enum { SKMP_F32 = 0, SKMP_F64 = 1 } skmp_dtype;
typedef enum { SKMP_PROJ_COUNT_SKETCH = 0, SKMP_PROJ_DENSE = 1 } skmp_proj;

/* ---------------------------------------------------------------------------------------------
 * Errors / version (host-only; callable without a GPU)
 * ------------------------------------------------------------------------------------------- */
const char* skmp_status_string(skmp_status s);   /* static string                              */
const char* skmp_last_error(void);               /* thread-local text of the last non-OK call  */
int64_t skmp_last_error_index(void);             /* offending stream/group/row, or -1          */
int32_t skmp_abi_version(void);                  /* SKMP_ABI_VERSION                           */
int64_t skmp_launch_count(void);                 /* kernels this library launched so far (all  */
                                                 /* threads); bench.py reports the delta       */
/* Device memory: the library allocates only from two stream-ordered pools of its own per device
 * (work: handles, workspaces, per-call temporaries; staging: host-input copies), never from the
 * process's default pool, and keeps freed blocks cached between calls.  skmp_trim() returns every
 * cached, unused block of those pools to the device (memory still owned by live handles stays).
 * Callable without a GPU (then a no-op).  Errors: CUDA. */
skmp_status skmp_trim(void);

/* ---------------------------------------------------------------------------------------------
 * Hash plan (host-only; callable without a GPU).  The count-sketch pair (h, s) of P:L200-204
 * (§3.1: "two pair-wise independent hash functions h: [d]->[k] and s: [d]->{-1,+1}").
 * Reading 2: Carter–Wegman over p = 2^61-1 keyed by the stream id, parameters (a, b, c, e) from
 * splitmix64(seed): h(id) = ((a x + b) mod p) mod k,  s(id) = +1 iff ((c x + e) mod p) is even,
 * x = id mod p.
 *   ids    [host] d stream ids          groups [host, out] d ints in [0,k)   signs [host, out] d
 * Errors: INVALID_ARG (NULL, d<0, k<1).
 * ------------------------------------------------------------------------------------------- */
skmp_status sketch_hash_plan(const uint64_t* ids, int64_t d, int32_t k, uint64_t seed,
                             int32_t* groups, int8_t* signs);

/* ---------------------------------------------------------------------------------------------
 * Sketch (Alg. 1; z-normalisation P:L210; linear updates §3.3)
 *
 *   R^(g) = sum_{j in J_g} s(j) * (T_j - mu_j) / sigma_j,   J_g = { j : h(j) = g }
 *
 * with mu_j, sigma_j the stream's own whole-series mean and population std (reading 3), summed
 * in FP64 in ascending input order inside each group and rounded once to dtype.  DENSE instead
 * computes R = S * diag(1/sigma) * (T - mu) for a caller matrix S (reading 1).
 * ------------------------------------------------------------------------------------------- */
typedef struct skmp_sketch skmp_sketch;   /* opaque; owns R (k x n) and the per-dim plan      */

typedef struct {
  int32_t k;              /* number of sketch series (groups), >= 1                            */
  int32_t dtype;          /* skmp_dtype of T and R                                             */
  int32_t proj;           /* skmp_proj                                                         */
  int32_t reserved;       /* must be 0                                                         */
  uint64_t seed;          /* hash seed (COUNT_SKETCH)                                          */
  const int32_t* groups;  /* optional [host] d: explicit h (test hook, e.g. identity plan)     */
  const int8_t* signs;    /* optional [host] d: explicit s (+1/-1); requires groups            */
  const double* S;        /* DENSE only, [host] k x d row-major (copied)                       */
} skmp_sketch_cfg;

/* Build the sketch of T (d streams of n samples, leading dimension ld).
 *   T    [dev|host] d x ld (dtype); only the first n columns are read.   ids [host] d, unique.
 *   out  receives a new handle (free with sketch_free).
 * Two HBM passes over T (stream statistics, then projection).  One small synchronous D2H of
 * error flags.  Errors: INVALID_ARG, NONFINITE, CONSTANT_SERIES (index = stream row),
 * DUPLICATE_DIM, CUDA, OOM. */
skmp_status sketch_build(const void* T, int64_t d, int64_t n, int64_t ld, const uint64_t* ids,
                         const skmp_sketch_cfg* cfg, void* stream, skmp_sketch** out);

/* Add nb full-length streams (P:L329-334 linearity; must span all n samples).
 *   T [dev|host] nb x ld;  ids [host] nb (new, unique);  S_cols [host] k x nb for DENSE, else NULL.
 * R^(h(j)) += s(j) z_j in FP64 (the handle keeps FP64 master accumulators), then R = dtype(R64).
 * Errors: INVALID_ARG, DUPLICATE_DIM, NONFINITE, CONSTANT_SERIES, CUDA, OOM. */
skmp_status sketch_add_dim(skmp_sketch* h, const void* T, int64_t nb, int64_t ld,
                           const uint64_t* ids, const double* S_cols, void* stream);

/* Delete nb streams (R^(g) = R^(g) - s(j) T^(j)).  The caller re-supplies the raw
 * streams (the sketch keeps none); their STORED mu/sigma are used, so add-then-delete is an exact
 * inverse up to one FP64 rounding.  Errors: INVALID_ARG, UNKNOWN_DIM, CUDA, OOM. */
skmp_status sketch_del_dim(skmp_sketch* h, const void* T, int64_t nb, int64_t ld,
                           const uint64_t* ids, void* stream);

/* Point updates (§3.3: "if only the i-th time point of the j-th dimension is
 * updated, to increase its value by delta, then R^(g)_i = R^(g)_i + s(j) delta"): for q < count,
 * stream ids[q] moves by delta[q] at time t[q].  Reading 24: delta is in the stream's own units
 * and the sketch keeps the stream z-normalised with its STORED statistics, so the sketch moves by
 * s(j) delta / sigma_j (DENSE: S_gj delta / sigma_j in every group); the statistics are not
 * re-estimated.  FP64 atomics on the master sketch (repeated (id, t) pairs accumulate), then the
 * touched entries are re-rounded to dtype.  ids/t/delta [host] count.  Asynchronous.
 * Errors: INVALID_ARG (NULL, count < 0, t outside [0, n)), UNKNOWN_DIM, CUDA, OOM. */
skmp_status sketch_point_update(skmp_sketch* h, const uint64_t* ids, const int64_t* t, const double* delta,
                                int64_t count, void* stream);

/* Borrowed views (valid until the next add/del/free).  R: [dev] k x n, ld = n, dtype.
 * R64: [dev] k x n FP64 master accumulators. */
skmp_status sketch_view(const skmp_sketch* h, const void** R, int32_t* k, int64_t* n, int64_t* d,
                        int32_t* dtype);
skmp_status sketch_view64(const skmp_sketch* h, const double** R64);

/* Copy the current plan to host arrays of length d (any may be NULL): ids, group, sign,
 * mu, sigma (sign is 0 and group -1 for DENSE). */
skmp_status sketch_plan(const skmp_sketch* h, uint64_t* ids, int32_t* g, int8_t* s, double* mu,
                        double* sigma);
/* Re-round R = dtype(R64) after R64 was modified outside the library (e.g. a cross-GPU
 * sum-allreduce of per-rank partial sketches).  Asynchronous. */
skmp_status sketch_refresh(skmp_sketch* h, void* stream);
/* Release the handle.  The device memory is freed stream-ordered on the stream of the last
 * library call that used the handle; a caller that read R / R64 on ANOTHER stream (e.g. a sketch
 * built on a prefetch stream and joined on the main stream) must call sketch_free_async with
 * that stream, which frees after both the handle's own work and everything already enqueued on
 * `stream`. */
void sketch_free(skmp_sketch* h);
void sketch_free_async(skmp_sketch* h, void* stream);

/* ---------------------------------------------------------------------------------------------
 * Matrix-profile self-join over each sketch series (Def. 6; self-join variant
 * P:L322; dist = z-normalised Euclidean, Def. 3):
 *
 *   P_g[i] = min_{ j : |i-j| > excl } dist(R^(g)_{i,m}, R^(g)_{j,m}),  I_g[i] = smallest argmin
 *
 * excl = ceil(m/2) by default (reading 7).  Flat windows (sigma <= 1e-12 (max|R_g|+1)) follow
 * reading 5 (flat-flat 0, flat vs non-flat sqrt(m)); a group whose windows are all flat is
 * "inert" (reading 6): P_g = 0 and inert[g] = 1.
 * Computed by the STOMP/SCAMP diagonal recurrence on mean-centred dot products with exact FP64
 * re-seeding every `reseed_rows` rows; the chosen neighbour's distance is then recomputed
 * exactly in FP64.
 * ------------------------------------------------------------------------------------------- */
typedef struct {
  int32_t m;            /* subsequence length, >= 2                                          */
  int32_t excl;         /* exclusion radius; < 0 -> ceil(m/2)                                 */
  int32_t reseed_rows;  /* 0 -> default (FP32 16384, or 32768 from 2^20 windows; FP64 2048); rounded up to 64 */
  int32_t reserved;     /* must be 0                                                          */
} skmp_mp_cfg;

typedef struct skmp_mp skmp_mp;  /* opaque join workspace: window statistics + profile keys */

/* Window preparation (per-window mean/std in FP64 by direct sums, flat flags, recurrence terms)
 * and key initialisation.  R [dev] k x ld (dtype), n samples per series.  Asynchronous: the
 * per-series flat counts travel to the host behind the kernels and are waited for only when the
 * host needs them (the inert flags of mp_finalize*).  R must stay valid until the join and the
 * finalize have run.  Errors: INVALID_ARG, SERIES_TOO_SHORT, NO_ADMISSIBLE, CUDA, OOM.*/
skmp_status mp_create(const void* R, int32_t k, int64_t n, int64_t ld, int32_t dtype,
                      const skmp_mp_cfg* cfg, void* stream, skmp_mp** out);

/* Accumulate the join over diagonals [diag_lo, diag_hi) (0,0 -> all of [excl+1, n_sub)) into
 * the workspace's keys.  Bands are disjoint diagonal ranges; any partition of [excl+1, n_sub)
 * accumulates bit-identical keys (band edges are rounded to the tile width, see mp_band).
 * Asynchronous.  Errors: INVALID_ARG, CUDA. */
skmp_status mp_join(skmp_mp* w, int64_t diag_lo, int64_t diag_hi, void* stream);

/* Device view of the profile keys, for a cross-GPU max-reduce (multi-GPU bands):
 *   keys [dev] count int64 words, `words` per profile entry (FP32: 1, FP64: 2);
 * b = the smallest index of the winning candidate set (the D cells one join thread saw for this
 * entry: D consecutive neighbours [b, b+D), b >= -(D-1); mp_finalize resolves the set exactly);
 * FP32 word = (orderable(rho_f32) << 32) | (0xFFFFFFFF - (b + 32)); FP64 words =
 * {orderable(rho_f64), -1 - b}.  Larger is better (max rho, then smallest b): FP32 keys reduce
 * with one signed int64 MAX; FP64 keys reduce lexicographically (MAX of word 0, then MAX of
 * word 1 among ties). */
skmp_status mp_keys(skmp_mp* w, void** keys, int64_t* count, int32_t* words);

/* Host-only: diagonal band `band` of `nbands` equal-cost bands of [excl+1, n_sub) (cost of a
 * diagonal = its cells + 5 W for the per-tile work that does not scale with the tile height,
 * W = mp_tile_width; the first W diagonals' cells count 4.5 times: joined while the keys are
 * empty, they publish most), edges rounded to W (so band results are bit-identical to a single
 * join; the first band starts at 0).  Costs measured on one B200 (tools/band_balance.py).
 * Errors: INVALID_ARG. */
skmp_status mp_band(int64_t n_sub, int32_t excl, int32_t dtype, int32_t nbands, int32_t band,
                    int64_t* diag_lo, int64_t* diag_hi);

/* Host-only: the join's tile width W (diagonals per tile) for dtype; band edges of mp_band are
 * multiples of it. */
int32_t mp_tile_width(int32_t dtype);

/* Finalize: keys -> P [dev] k x n_sub (dtype) and I [dev] k x n_sub (int64), inert [host] k.
 * Each entry's winning candidate set is resolved in FP64 (nearest admissible member, smallest
 * index on ties) and its distance recomputed from Def. 3 by explicit differences.
 * Requires the full diagonal range to have been joined.  Asynchronous when inert is NULL; with
 * inert it waits for mp_create's flat counts (which normally arrived long before).
 * Errors: INVALID_ARG, CUDA. */
skmp_status mp_finalize(skmp_mp* w, void* P, int64_t* I, uint8_t* inert, void* stream);
/* Finalize only the windows [row_lo, row_hi) of every series (0 <= row_lo <= row_hi <= n_sub)
 * into the full-size P / I (other entries untouched): the multi-GPU path shards the finalize
 * over ranks after the key reduce.  Same semantics and errors as mp_finalize. */
skmp_status mp_finalize_rows(skmp_mp* w, int64_t row_lo, int64_t row_hi, void* P, int64_t* I,
                             uint8_t* inert, void* stream);
void mp_free(skmp_mp* w);

/* One-shot: mp_create + mp_join(all) + mp_finalize + mp_free. */
skmp_status mp_selfjoin(const void* R, int32_t k, int64_t n, int64_t ld, int32_t dtype,
                        const skmp_mp_cfg* cfg, void* P, int64_t* I, uint8_t* inert, void* stream);

/* AB-join matrix profile (Def. 6 ab-join), the join Alg. 2 calls as written
 * (ABjoinMP(R_train^(g), R_test^(g), m)):
 *
 *   PA_g[i] = min_j dist(A^(g)_{i,m}, B^(g)_{j,m}),  IA_g[i] = smallest argmin,  over ALL windows
 *   j of B (two different series: no exclusion zone), and optionally the reverse profile PB of B
 *   against A (it comes from the same cells; pass PB = IB = NULL to skip it).
 *   RA  [dev] k x ldA test series (nA samples);  RB [dev] k x ldB train series (nB samples).
 *   cfg m >= 2 (excl is ignored), reseed_rows as for mp_create.
 *   PA [dev] k x (nA-m+1) dtype, IA [dev] k x (nA-m+1) int64 (indices into B's windows);
 *   PB/IB likewise k x (nB-m+1) or NULL;  inert [host] k or NULL: 1 where both series of a group
 *   are entirely flat (an empty group, reading 6).
 * Flat windows follow reading 5 (each series' threshold relative to its own max|x|).  Computed
 * as two diagonal-band passes of the same join kernels (test rows against train columns, and
 * train rows against test columns), each cell once; neighbours resolved exactly in FP64 as in
 * mp_finalize.  Synchronous (window preparation).  Errors: INVALID_ARG, SERIES_TOO_SHORT, CUDA,
 * OOM. */
skmp_status mp_abjoin(const void* RA, int64_t nA, int64_t ldA, const void* RB, int64_t nB, int64_t ldB,
                      int32_t k, int32_t dtype, const skmp_mp_cfg* cfg, void* PA, int64_t* IA, void* PB,
                      int64_t* IB, uint8_t* inert, void* stream);

/* The AB-join in stages, for its multi-GPU decomposition (the same diagonal-band scheme as the
 * self-join):
 *  mp_create_ab   as mp_create, but an AB workspace: no exclusion zone, no NO_ADMISSIBLE check;
 *  mp_join_ab     cells (i, i + delta), i a window of `rows`, i + delta a window of `cols`,
 *                 delta in [diag_lo, diag_hi) (clipped to cols' windows); pass 1 of Def. 6's
 *                 AB-join is (rows = test, cols = train, delta >= 0), pass 2 (rows = train,
 *                 cols = test, delta >= 1); row candidates go to `rows`' keys, column candidates
 *                 to `cols`' keys; any split of the two passes into bands accumulates bit-identical
 *                 keys (keys reduce across GPUs with mp_keys exactly as for the self-join);
 *  mp_finalize_ab windows [row_lo, row_hi) (0, 0 -> all) of `w` resolved against `other`'s windows
 *                 (PA, IA of mp_abjoin for w = test), full-size P / I [dev], inert [host] k or NULL;
 *  mp_abband      host-only: band `band` of `nbands` equal-cell bands of the two passes taken as
 *                 one sequence (pass 1 diagonals 0 .. n_subB-1, then pass 2 diagonals 1 ..
 *                 n_subA-1), edges on the tile grid; a band may hold a piece of each pass:
 *                 [lo1, hi1) of pass 1 and [lo2, hi2) of pass 2 (empty ranges as lo == hi).
 * Errors: INVALID_ARG (NULL, workspaces not from mp_create_ab, mismatched k / dtype / m, bad
 * bands or rows), SERIES_TOO_SHORT, CUDA, OOM.  mp_join_ab is asynchronous. */
skmp_status mp_create_ab(const void* R, int32_t k, int64_t n, int64_t ld, int32_t dtype,
                         const skmp_mp_cfg* cfg, void* stream, skmp_mp** out);
skmp_status mp_join_ab(skmp_mp* rows, skmp_mp* cols, int64_t diag_lo, int64_t diag_hi, void* stream);
skmp_status mp_finalize_ab(skmp_mp* w, skmp_mp* other, int64_t row_lo, int64_t row_hi, void* P, int64_t* I,
                           uint8_t* inert, void* stream);
skmp_status mp_abband(int64_t n_subA, int64_t n_subB, int32_t dtype, int32_t nbands, int32_t band,
                      int64_t* lo1, int64_t* hi1, int64_t* lo2, int64_t* hi2);

/* ---------------------------------------------------------------------------------------------
 * Streaming test data ("lines 4-5 in Alg. 1 ... only invoke whenever
 * a new test data is received" and a streaming matrix profile in Alg. 2).  A stream holds the
 * train sketch's plan and statistics, a private copy of the train sketch series (prepared once
 * as an AB workspace) and a growing test sketch of `capacity` samples per group.
 *
 *  stream_create  train: a built sketch (count sketch or dense; it may be modified or freed
 *                 afterwards: everything needed is copied); cfg: m (excl ignored: AB-join),
 *                 reseed_rows; capacity: the maximum number of test samples (m <= capacity <
 *                 2^31).  Allocates k x capacity test sketch (FP64 master + dtype copy), profile
 *                 P (dtype) and I (int64), all with row stride `capacity`.
 *  stream_push    T: d x n_new [host or dev] new time points of every stream of the train plan,
 *                 rows in the plan's order (as sketch_plan lists them), row stride ld >= n_new,
 *                 the train sketch's dtype.  Projects them into test-sketch columns
 *                 [n_test, n_test + n_new) with the TRAIN statistics mu_j, sigma_j (reading 25),
 *                 then AB-joins every test window completed by them (windows [max(0, n_test-m+1),
 *                 n_test+n_new-m+1)) against all train windows (Def. 6) and writes
 *                 their P / I.  Enqueued on `stream`; it synchronises once (window flags D2H).
 *  stream_view    device pointers of the test sketch R (k x capacity), P and I (k x capacity;
 *                 columns [0, n_sub) valid), the counts, the row stride, and [host] inert flags
 *                 per group (train series all flat and every test window so far flat) or NULL.
 *                 Pass P, I, n_sub, ld and inert to discord_topk for Alg. 2's ranking.
 * Errors: INVALID_ARG (NULL, capacity exceeded, bad sizes), NONFINITE (a NaN / Inf among the new
 * points; index = the first affected group; the push is discarded), SERIES_TOO_SHORT (train n < m),
 * CUDA, OOM.  A failed push leaves the stream as it was (n_test, profile and carried state). */
typedef struct skmp_stream skmp_stream;
skmp_status stream_create(const skmp_sketch* train, const skmp_mp_cfg* cfg, int64_t capacity, void* stream,
                          skmp_stream** out);
skmp_status stream_push(skmp_stream* h, const void* T, int64_t n_new, int64_t ld, void* stream);
skmp_status stream_view(const skmp_stream* h, void** R, void** P, int64_t** I, int64_t* n_test, int64_t* n_sub,
                        int64_t* ld, uint8_t* inert);
void stream_free(skmp_stream* h);

/* ---------------------------------------------------------------------------------------------
 * Native multi-GPU: one process per GPU, an NCCL communicator, the two exchange
 * steps of the path.  (The Python package does the same through torch.distributed, dist.py.)
 *  skmp_comm_unique_id  rank 0 creates the 128-byte id; the caller ships it to every rank.
 *  skmp_comm_init       collective over `nranks` processes (each on its own current device).
 *  sketch_allreduce     NC1: sum-all-reduce of the per-rank partial FP64 sketches (each rank built
 *                       its shard of the streams with the same id-keyed plan; Alg. 1 is linear,
 *                       P:L330), then R = dtype(R64) on every rank.  Asynchronous on `stream`.
 *  mp_selfjoin_dist     mp_selfjoin split over the ranks: rank r joins band r of mp_band, the
 *                       profile keys are max-all-reduced (NC2; FP64 keys lexicographically), each
 *                       rank finalizes a contiguous slice of the windows and a sum-all-reduce
 *                       assembles P, I on EVERY rank (bit-identical to mp_selfjoin).  Arguments
 *                       as mp_selfjoin; every rank must pass the same R contents and sizes.
 * NCCL is loaded with dlopen("libnccl.so.2") on first use (a process that already holds one
 * reuses it).  Errors: INVALID_ARG, NCCL (a collective or communicator failure, or libnccl.so.2
 * missing or incomplete), CUDA, OOM and those of the composed calls.  A rank that fails returns without entering the remaining
 * collectives: callers pass identical arguments so that all ranks fail alike. */
typedef struct skmp_comm skmp_comm;
skmp_status skmp_comm_unique_id(uint8_t id[128]);
skmp_status skmp_comm_init(const uint8_t id[128], int nranks, int rank, skmp_comm** out);
void skmp_comm_free(skmp_comm* comm);
skmp_status sketch_allreduce(skmp_comm* comm, skmp_sketch* partial, void* stream);
skmp_status mp_selfjoin_dist(skmp_comm* comm, const void* R, int32_t k, int64_t n, int64_t ld, int32_t dtype,
                             const skmp_mp_cfg* cfg, void* P, int64_t* I, uint8_t* inert, void* stream);

/* ---------------------------------------------------------------------------------------------
 * Discord detection over the sketch profiles: Alg. 2 Time-Detection + ordered
 * top-K list (reading 12):
 *   C[i] = max_{g not inert} P_g[i], G[i] = smallest maximising g (Alg. 2 strict '>' P:L262);
 *   repeat top times: t = smallest-index argmax of C over unmasked windows; emit
 *   (t, G[t], I_G[t][t], C[t]); mask [t - radius, t + radius].
 *   P [dev] k x ldp (dtype), I [dev] k x ldp, inert [host] k (NULL = none inert).
 *   radius < 0 -> ceil(m/2).  t_out/g_out/nn_out/score_out [host] top entries; n_found [host]
 *   receives the number emitted (< top when the mask exhausts the profile).  Synchronous.
 * Errors: INVALID_ARG, ALL_GROUPS_INERT, CUDA, OOM. */
skmp_status discord_topk(const void* P, const int64_t* I, const uint8_t* inert, int32_t k,
                         int64_t n_sub, int64_t ldp, int32_t m, int32_t dtype, int32_t top,
                         int32_t radius, int64_t* t_out, int32_t* g_out, int64_t* nn_out,
                         double* score_out, int32_t* n_found, void* stream);

/* ---------------------------------------------------------------------------------------------
 * Discord dimension recovery: Alg. 3 Dimension-Detection in the
 * single-series mode of P:L322 (the same series as train and test, self-join variant):
 *
 *   s^(j) = min_{t : |t - t_star| > excl} dist(T_{j, t_star, m}, T_{j, t, m}),  nn^(j) = argmin
 *
 * for each listed stream j of the discord's group J_{g*} (dist = z-normalised Euclidean, Def. 3
 * P:L129-133, evaluated by explicit differences in FP64; flat windows per reading 5 relative
 * to max|T_j|; smallest t on ties), and j* = the FIRST strict maximiser in the listed order
 * (Alg. 3 lines 3-7, reading 20).  The refinement join of P:L303-304 is mp_selfjoin on row j*
 * followed by discord_topk with top = 1.
 *   T       [dev|host] (max(rows)+1) x ld streams (dtype), n samples each (a host matrix is
 *           staged row by row: only the listed rows cross PCIe).
 *   rows    [host] nrows stream rows of T (the members of J_{g*}, in group order).
 *   t_star  the discord time from discord_topk, 0 <= t_star < n - m + 1.
 *   excl    exclusion radius; < 0 -> ceil(m/2) (reading 7).
 *   scores  [host, out] nrows 1NN distances;  nn [host, out] nrows neighbour times (may be NULL).
 *   j_star  [host, out] index into rows of the winner.
 * Synchronous.  Errors: INVALID_ARG (NULL, nrows < 1, bad t_star, m < 2, negative row),
 * SERIES_TOO_SHORT (n < m), NO_ADMISSIBLE (no window farther than excl from t_star), CUDA, OOM. */
skmp_status discord_dims(const void* T, int64_t ld, int64_t n, int32_t dtype, const int64_t* rows,
                         int64_t nrows, int64_t t_star, int32_t m, int32_t excl, double* scores,
                         int64_t* nn, int64_t* j_star, void* stream);

/* Alg. 3 over the discord's group J_{g*} of a sketch, with the raw streams spread over several
 * matrices (Alg. 3 lines 1-2 take "the dimensions in group g*" and line 3 scans them
 * in order).  Members of J_g are taken in the sketch plan's order (sketch_plan: input order, added
 * streams appended, deleted ones removed; DENSE: every stream, reading 1); each member is scored
 * in the first source whose ids list it, as discord_dims scores a row (same definition, tie and
 * flat rules); members no source holds are skipped, so a rank of a stream-sharded sketch scores
 * its own streams only.  The winner is the FIRST strict maximiser in plan order (reading 20).
 *   h       the sketch whose plan defines J_g (not modified; its R is not read).
 *   g       the group (count sketch: 0 <= g < k; ignored for DENSE).
 *   src     [host] nsrc sources {T [dev|host] rows x ld (the sketch's dtype, the sketch's n samples
 *           per stream), ld >= n, rows, ids [host] rows stream ids}; nsrc may be 0.
 *   out     [host, out] {score, id, nn, n_scored}: n_scored = members scored; when it is 0 the
 *           other fields are left untouched.
 * Synchronous.  Errors: INVALID_ARG (NULL, bad g, bad source, bad t_star, m < 2),
 * SERIES_TOO_SHORT, NO_ADMISSIBLE, CUDA, OOM. */
typedef struct {
  const void* T;        /* [dev|host] rows x ld streams                                        */
  int64_t ld;           /* leading dimension in elements, >= the sketch's n                    */
  int64_t rows;         /* number of streams in T                                             */
  const uint64_t* ids;  /* [host] rows: stream id of each row                                  */
} skmp_source;

typedef struct {
  double score;         /* s^(j*): 1NN distance of T_{j*, t*, m} in its own stream            */
  uint64_t id;          /* j*: the winning stream's id                                         */
  int64_t nn;           /* its nearest neighbour's window start                               */
  int64_t n_scored;     /* members of J_g scored (0: no winner, other fields untouched)        */
} skmp_dim_result;

skmp_status discord_dims_group(const skmp_sketch* h, int32_t g, const skmp_source* src, int32_t nsrc,
                               int64_t t_star, int32_t m, int32_t excl, skmp_dim_result* out, void* stream);

/* Host-only: combine per-part Alg. 3 winners (parts[q] from discord_dims_group over disjoint
 * pieces of J_g that come in J_g order, e.g. ranks holding contiguous id shards, in rank order):
 * out = the first part with the strictly largest score among parts with n_scored > 0, and
 * out->n_scored = the total.  The multi-GPU path all-gathers the ranks' results and calls this.
 * Errors: INVALID_ARG (NULL, nparts < 1, negative n_scored). */
skmp_status discord_dims_merge(const skmp_dim_result* parts, int32_t nparts, skmp_dim_result* out);

#ifdef __cplusplus
}
#endif
#endif /* SKETCHMP_H */

// C-ABI layer (include/sketchmp.h): validation, handles, plans, host<->device plumbing and
// launch sequencing.  Every step of the path itself runs in the kernels of sketch.cu,
// mp_prep.cu, mp_join.cu, mp_final.cu and detect.cu; there is no CPU fallback.
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <string>
#include <unordered_map>
#include <unordered_set>
#include <mutex>
#include <vector>

#include "internal.h"

// ============================================================================================
// errors
// ============================================================================================
namespace {
thread_local std::string g_msg;
thread_local int64_t g_index = -1;
std::atomic<int64_t> g_launches{0};
}  // namespace

namespace skmp {
void count_launches(int64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
skmp_status set_error(skmp_status s, const std::string& msg, int64_t index) {
  g_msg = msg;
  g_index = index;
  return s;
}
skmp_status cuda_error(cudaError_t e, const char* where) {
  // clear the runtime's per-thread last error: a failed allocation is not sticky, and a stale
  // error would otherwise surface at the next launch check of an unrelated call
  cudaGetLastError();
  const skmp_status s = (e == cudaErrorMemoryAllocation) ? SKMP_E_OOM : SKMP_E_CUDA;
  return set_error(s, std::string(where) + ": " + cudaGetErrorString(e), -1);
}
}  // namespace skmp

namespace {
cudaMemPool_t work_pool_impl();
}

namespace skmp {
cudaError_t dmalloc(void** p, size_t bytes, cudaStream_t st) {
  cudaMemPool_t pool = work_pool_impl();
  return pool ? cudaMallocFromPoolAsync(p, bytes, pool, st) : cudaMallocAsync(p, bytes, st);
}
}  // namespace skmp

using namespace skmp;

namespace {

skmp_status ok() {
  g_msg.clear();
  g_index = -1;
  return SKMP_OK;
}

skmp_status require_device() {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) {
    cudaGetLastError();
    return set_error(SKMP_E_CUDA, "no CUDA device available (the path has no CPU fallback)");
  }
  return SKMP_OK;
}

bool is_device_ptr(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

size_t elem_size(int dtype) { return dtype == SKMP_F32 ? 4 : 8; }

// RAII list of stream-ordered temporaries
struct Temps {
  cudaStream_t st;
  std::vector<void*> ptrs;
  explicit Temps(cudaStream_t s) : st(s) {}
  ~Temps() {
    for (void* p : ptrs) cudaFreeAsync(p, st);
  }
  template <typename T>
  cudaError_t alloc(T** p, size_t count, cudaMemPool_t pool = nullptr) {
    void* q = nullptr;
    cudaError_t e = pool ? cudaMallocFromPoolAsync(&q, count * sizeof(T) + 16, pool, st)
                         : dmalloc(&q, count * sizeof(T) + 16, st);
    if (e == cudaSuccess) {
      ptrs.push_back(q);
      *p = static_cast<T*>(q);
    }
    return e;
  }
};

// The library's device memory comes from two pools of its own per device (never the process's
// default pool, whose attributes belong to the caller): the WORK pool (handles, workspaces and
// per-call temporaries) and the STAGING pool (host-input staging buffers).  Both keep freed
// blocks cached (release threshold = max) so repeated calls do not round-trip to the OS;
// skmp_trim() returns the cached memory.  Staging has its own pool because multi-GB staging
// blocks interleaved with the small workspaces fragmented a shared pool, so a later staging
// allocation could miss a contiguous block and grow the pool (mapping gigabytes of fresh memory)
// in the middle of a pipelined batch.
struct Pools {
  std::mutex mu;
  std::vector<cudaMemPool_t> work, staging;
};
Pools& pools() {
  static Pools p;
  return p;
}

cudaMemPool_t make_pool(std::vector<cudaMemPool_t>& v) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  std::lock_guard<std::mutex> lock(pools().mu);
  if ((int)v.size() <= dev) v.resize((size_t)dev + 1, nullptr);
  if (!v[(size_t)dev]) {
    cudaMemPoolProps props = {};
    props.allocType = cudaMemAllocationTypePinned;
    props.handleTypes = cudaMemHandleTypeNone;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    cudaMemPool_t p = nullptr;
    if (cudaMemPoolCreate(&p, &props) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;  // then the runtime's default pool (cudaMallocAsync)
    }
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(p, cudaMemPoolAttrReleaseThreshold, &thr);
    v[(size_t)dev] = p;
  }
  return v[(size_t)dev];
}

cudaMemPool_t staging_pool() { return make_pool(pools().staging); }
cudaMemPool_t work_pool_impl() { return make_pool(pools().work); }

// Stage a (possibly host) rows x ld matrix into device memory; returns the device pointer.
skmp_status stage_input(const void* T, int64_t rows, int64_t n, int64_t ld, int dtype, Temps& tmp,
                        const void** dev, int64_t* dev_ld) {
  if (is_device_ptr(T)) {
    *dev = T;
    *dev_ld = ld;
    return SKMP_OK;
  }
  const size_t es = elem_size(dtype);
  char* d = nullptr;
  SKMP_CUDA(tmp.alloc(&d, (size_t)rows * (size_t)n * es, staging_pool()));
  // in <= 64 MB pieces: a copy engine works through one command at a time, so one multi-GB
  // command would hold back every small transfer other streams enqueue meanwhile (e.g. a join's
  // tile table behind the next batch's staging)
  const int64_t piece = std::max<int64_t>(1, (int64_t)((64u << 20) / std::max<size_t>(1, (size_t)n * es)));
  for (int64_t r0 = 0; r0 < rows; r0 += piece) {
    const int64_t nr = std::min(piece, rows - r0);
    SKMP_CUDA(cudaMemcpy2DAsync(d + (size_t)r0 * (size_t)n * es, (size_t)n * es,
                                static_cast<const char*>(T) + (size_t)r0 * (size_t)ld * es, (size_t)ld * es,
                                (size_t)n * es, (size_t)nr, cudaMemcpyHostToDevice, tmp.st));
  }
  *dev = d;
  *dev_ld = n;
  return SKMP_OK;
}

template <typename T>
skmp_status upload(const std::vector<T>& h, T** d, Temps& tmp) {
  SKMP_CUDA(tmp.alloc(d, h.size() ? h.size() : 1));
  if (!h.empty())
    SKMP_CUDA(cudaMemcpyAsync(*d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice, tmp.st));
  return SKMP_OK;
}

struct StatsHost {
  std::vector<double> mu, sigma;
};

// K1 on rows of T, then one small synchronous D2H of mu/sigma/flags; maps flags to errors.
skmp_status run_stats(const void* Tdev, int64_t rows, int64_t n, int64_t ld, int dtype, Temps& tmp,
                      StatsHost* out, double** d_mu, double** d_inv) {
  StatsOut so;
  double* buf = nullptr;
  SKMP_CUDA(tmp.alloc(&buf, (size_t)rows * 3));
  int32_t* flag = nullptr;
  SKMP_CUDA(tmp.alloc(&flag, (size_t)rows));
  void* ws = nullptr;
  char* wsc = nullptr;
  SKMP_CUDA(tmp.alloc(&wsc, stats_ws_bytes(rows, n)));
  ws = wsc;
  so.mu = buf;
  so.sigma = buf + rows;
  so.inv = buf + 2 * rows;
  so.flag = flag;
  SKMP_CUDA(launch_stream_stats(Tdev, rows, n, ld, dtype, so, ws, tmp.st));
  std::vector<int32_t> hf((size_t)rows);
  out->mu.resize((size_t)rows);
  out->sigma.resize((size_t)rows);
  SKMP_CUDA(cudaMemcpyAsync(hf.data(), flag, sizeof(int32_t) * rows, cudaMemcpyDeviceToHost, tmp.st));
  SKMP_CUDA(cudaMemcpyAsync(out->mu.data(), so.mu, sizeof(double) * rows, cudaMemcpyDeviceToHost, tmp.st));
  SKMP_CUDA(cudaMemcpyAsync(out->sigma.data(), so.sigma, sizeof(double) * rows, cudaMemcpyDeviceToHost, tmp.st));
  SKMP_CUDA(cudaStreamSynchronize(tmp.st));
  for (int64_t j = 0; j < rows; ++j) {
    if (hf[(size_t)j] == 1) return set_error(SKMP_E_NONFINITE, "non-finite value in input stream", j);
    if (hf[(size_t)j] == 2)
      return set_error(SKMP_E_CONSTANT_SERIES, "constant input stream (sigma <= 1e-12 (max|x|+1))", j);
  }
  *d_mu = so.mu;
  *d_inv = so.inv;
  return SKMP_OK;
}

}  // namespace

// ============================================================================================
// sketch handle
// ============================================================================================
struct skmp_sketch {
  int dtype = SKMP_F32;
  int proj = SKMP_PROJ_COUNT_SKETCH;
  int k = 0;
  int64_t n = 0;
  uint64_t seed = 0;
  double* R64 = nullptr;  // k x n
  void* R = nullptr;      // k x n (== R64 for FP64)
  cudaStream_t st = nullptr;
  std::vector<uint64_t> ids;
  std::vector<int32_t> g;
  std::vector<int8_t> s;
  std::vector<double> mu, sigma;
  std::vector<double> Scol;  // DENSE: d columns of length k (column-major per stream)
  std::unordered_map<uint64_t, int64_t> pos;
};

namespace {

// project rows [0, rows) of Tdev (ncols samples each) into R64 / R (row stride ldr) with the
// handle's projection kind, mode 0/+1/-1
skmp_status project_into(const skmp_sketch* h, const void* Tdev, int64_t ld, int64_t rows, int64_t ncols,
                         const std::vector<int32_t>& gg, const std::vector<int8_t>& ss,
                         const std::vector<double>& Scols, const std::vector<double>& mu,
                         const std::vector<double>& sigma, int mode, double* R64, void* R, int64_t ldr,
                         Temps& tmp) {
  std::vector<double> inv((size_t)rows);
  for (int64_t j = 0; j < rows; ++j) inv[(size_t)j] = 1.0 / sigma[(size_t)j];
  if (h->proj == SKMP_PROJ_COUNT_SKETCH) {
    // CSR: group g -> rows in ascending input order (Alg. 1 loop order inside each group)
    std::vector<int32_t> off((size_t)h->k + 1, 0), row((size_t)rows);
    std::vector<double> cmu((size_t)rows), cinv((size_t)rows);
    std::vector<int8_t> csg((size_t)rows);
    for (int64_t j = 0; j < rows; ++j) off[(size_t)gg[(size_t)j] + 1]++;
    for (int q = 0; q < h->k; ++q) off[(size_t)q + 1] += off[(size_t)q];
    std::vector<int32_t> fill(off.begin(), off.end() - 1);
    for (int64_t j = 0; j < rows; ++j) {
      const int32_t e = fill[(size_t)gg[(size_t)j]]++;
      row[(size_t)e] = (int32_t)j;
      cmu[(size_t)e] = mu[(size_t)j];
      cinv[(size_t)e] = inv[(size_t)j];
      csg[(size_t)e] = ss[(size_t)j];
    }
    CsrPlan p;
    int32_t *d_off, *d_row;
    double *d_mu, *d_inv;
    int8_t* d_sg;
    skmp_status s;
    if ((s = upload(off, &d_off, tmp)) != SKMP_OK) return s;
    if ((s = upload(row, &d_row, tmp)) != SKMP_OK) return s;
    if ((s = upload(cmu, &d_mu, tmp)) != SKMP_OK) return s;
    if ((s = upload(cinv, &d_inv, tmp)) != SKMP_OK) return s;
    if ((s = upload(csg, &d_sg, tmp)) != SKMP_OK) return s;
    p.off = d_off;
    p.row = d_row;
    p.mu = d_mu;
    p.inv = d_inv;
    p.sign = d_sg;
    SKMP_CUDA(launch_project_count(Tdev, ld, ncols, h->dtype, h->k, p, mode, R64, R, ldr, tmp.st));
  } else {
    // dense S as k x rows row-major for the kernel
    std::vector<double> S((size_t)h->k * (size_t)rows);
    for (int64_t j = 0; j < rows; ++j)
      for (int q = 0; q < h->k; ++q) S[(size_t)q * rows + j] = Scols[(size_t)j * h->k + q];
    double *d_S, *d_mu, *d_inv;
    skmp_status s;
    if ((s = upload(S, &d_S, tmp)) != SKMP_OK) return s;
    if ((s = upload(mu, &d_mu, tmp)) != SKMP_OK) return s;
    if ((s = upload(inv, &d_inv, tmp)) != SKMP_OK) return s;
    SKMP_CUDA(launch_project_dense(Tdev, ld, ncols, h->dtype, h->k, rows, d_S, rows, d_mu, d_inv,
                                   mode, R64, R, ldr, tmp.st));
  }
  return SKMP_OK;
}

// project rows [0, rows) of Tdev into the handle's own sketch with mode 0/+1/-1
skmp_status project_rows(skmp_sketch* h, const void* Tdev, int64_t ld, int64_t rows,
                         const std::vector<int32_t>& gg, const std::vector<int8_t>& ss,
                         const std::vector<double>& Scols, const std::vector<double>& mu,
                         const std::vector<double>& sigma, int mode, Temps& tmp) {
  return project_into(h, Tdev, ld, rows, h->n, gg, ss, Scols, mu, sigma, mode, h->R64, h->R, h->n, tmp);
}

}  // namespace

extern "C" {

const char* skmp_status_string(skmp_status s) {
  switch (s) {
    case SKMP_OK: return "SKMP_OK";
    case SKMP_E_INVALID_ARG: return "SKMP_E_INVALID_ARG";
    case SKMP_E_CONSTANT_SERIES: return "SKMP_E_CONSTANT_SERIES";
    case SKMP_E_NONFINITE: return "SKMP_E_NONFINITE";
    case SKMP_E_SERIES_TOO_SHORT: return "SKMP_E_SERIES_TOO_SHORT";
    case SKMP_E_NO_ADMISSIBLE: return "SKMP_E_NO_ADMISSIBLE";
    case SKMP_E_DUPLICATE_DIM: return "SKMP_E_DUPLICATE_DIM";
    case SKMP_E_UNKNOWN_DIM: return "SKMP_E_UNKNOWN_DIM";
    case SKMP_E_LENGTH_MISMATCH: return "SKMP_E_LENGTH_MISMATCH";
    case SKMP_E_ALL_GROUPS_INERT: return "SKMP_E_ALL_GROUPS_INERT";
    case SKMP_E_CUDA: return "SKMP_E_CUDA";
    case SKMP_E_NCCL: return "SKMP_E_NCCL";
    case SKMP_E_OOM: return "SKMP_E_OOM";
  }
  return "SKMP_E_UNKNOWN";
}
const char* skmp_last_error(void) { return g_msg.c_str(); }
int64_t skmp_last_error_index(void) { return g_index; }
int32_t skmp_abi_version(void) { return SKMP_ABI_VERSION; }
int64_t skmp_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }

skmp_status sketch_hash_plan(const uint64_t* ids, int64_t d, int32_t k, uint64_t seed,
                             int32_t* groups, int8_t* signs) {
  if (d < 0 || k < 1 || (d > 0 && (!ids || !groups || !signs)))
    return set_error(SKMP_E_INVALID_ARG, "sketch_hash_plan: NULL pointer, d < 0 or k < 1");
  hash_plan(ids, d, k, seed, groups, signs);
  return ok();
}

skmp_status sketch_build(const void* T, int64_t d, int64_t n, int64_t ld, const uint64_t* ids,
                         const skmp_sketch_cfg* cfg, void* stream, skmp_sketch** out) {
  if (!T || !ids || !cfg || !out) return set_error(SKMP_E_INVALID_ARG, "sketch_build: NULL argument");
  if (d < 1 || n < 2 || ld < n || cfg->k < 1)
    return set_error(SKMP_E_INVALID_ARG, "sketch_build: need d >= 1, n >= 2, ld >= n, k >= 1");
  if (cfg->dtype != SKMP_F32 && cfg->dtype != SKMP_F64)
    return set_error(SKMP_E_INVALID_ARG, "sketch_build: bad dtype");
  if (cfg->proj != SKMP_PROJ_COUNT_SKETCH && cfg->proj != SKMP_PROJ_DENSE)
    return set_error(SKMP_E_INVALID_ARG, "sketch_build: bad projection kind");
  if (cfg->proj == SKMP_PROJ_DENSE && !cfg->S)
    return set_error(SKMP_E_INVALID_ARG, "sketch_build: DENSE needs S (k x d)");
  if (cfg->signs && !cfg->groups)
    return set_error(SKMP_E_INVALID_ARG, "sketch_build: explicit signs require explicit groups");
  if (d > INT32_MAX) return set_error(SKMP_E_INVALID_ARG, "sketch_build: d too large");
  std::vector<int32_t> gg((size_t)d);
  std::vector<int8_t> ss((size_t)d, 0);
  std::unordered_map<uint64_t, int64_t> pos;
  pos.reserve((size_t)d * 2);
  for (int64_t j = 0; j < d; ++j) {
    if (!pos.emplace(ids[j], j).second)
      return set_error(SKMP_E_DUPLICATE_DIM, "sketch_build: duplicate stream id", j);
  }
  if (cfg->proj == SKMP_PROJ_COUNT_SKETCH) {
    hash_plan(ids, d, cfg->k, cfg->seed, gg.data(), ss.data());
    if (cfg->groups) {
      for (int64_t j = 0; j < d; ++j) {
        if (cfg->groups[j] < 0 || cfg->groups[j] >= cfg->k)
          return set_error(SKMP_E_INVALID_ARG, "sketch_build: explicit group out of range", j);
        gg[(size_t)j] = cfg->groups[j];
        if (cfg->signs) {
          if (cfg->signs[j] != 1 && cfg->signs[j] != -1)
            return set_error(SKMP_E_INVALID_ARG, "sketch_build: explicit sign must be +1/-1", j);
          ss[(size_t)j] = cfg->signs[j];
        }
      }
    }
  } else {
    std::fill(gg.begin(), gg.end(), -1);
  }
  skmp_status s = require_device();
  if (s) return s;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  Temps tmp(st);
  const void* Tdev;
  int64_t ldd;
  if ((s = stage_input(T, d, n, ld, cfg->dtype, tmp, &Tdev, &ldd)) != SKMP_OK) return s;
  StatsHost sh;
  double *d_mu, *d_inv;
  if ((s = run_stats(Tdev, d, n, ldd, cfg->dtype, tmp, &sh, &d_mu, &d_inv)) != SKMP_OK) return s;

  skmp_sketch* h = new skmp_sketch();
  h->dtype = cfg->dtype;
  h->proj = cfg->proj;
  h->k = cfg->k;
  h->n = n;
  h->seed = cfg->seed;
  h->st = st;
  cudaError_t e = dmalloc((void**)&h->R64, sizeof(double) * (size_t)h->k * n, st);
  if (e == cudaSuccess && h->dtype == SKMP_F32)
    e = dmalloc(&h->R, sizeof(float) * (size_t)h->k * n, st);
  if (e != cudaSuccess) {
    sketch_free(h);
    return cuda_error(e, "sketch_build: allocate R");
  }
  if (h->dtype == SKMP_F64) h->R = h->R64;
  h->ids.assign(ids, ids + d);
  h->g = gg;
  h->s = ss;
  h->mu = sh.mu;
  h->sigma = sh.sigma;
  h->pos = std::move(pos);
  if (h->proj == SKMP_PROJ_DENSE) {
    h->Scol.resize((size_t)d * h->k);
    for (int64_t j = 0; j < d; ++j)
      for (int q = 0; q < h->k; ++q) h->Scol[(size_t)j * h->k + q] = cfg->S[(size_t)q * d + j];
  }
  s = project_rows(h, Tdev, ldd, d, h->g, h->s, h->Scol, h->mu, h->sigma, 0, tmp);
  if (s != SKMP_OK) {
    sketch_free(h);
    return s;
  }
  *out = h;
  return ok();
}

skmp_status sketch_add_dim(skmp_sketch* h, const void* T, int64_t nb, int64_t ld,
                           const uint64_t* ids, const double* S_cols, void* stream) {
  if (!h || !T || !ids) return set_error(SKMP_E_INVALID_ARG, "sketch_add_dim: NULL argument");
  if (nb < 1 || ld < h->n) return set_error(SKMP_E_INVALID_ARG, "sketch_add_dim: need nb >= 1, ld >= n");
  if (h->proj == SKMP_PROJ_DENSE && !S_cols)
    return set_error(SKMP_E_INVALID_ARG, "sketch_add_dim: DENSE needs S_cols (k x nb)");
  std::unordered_set<uint64_t> seen;
  for (int64_t j = 0; j < nb; ++j) {
    if (h->pos.count(ids[j]) || !seen.insert(ids[j]).second)
      return set_error(SKMP_E_DUPLICATE_DIM, "sketch_add_dim: stream id already present", j);
  }
  skmp_status s = require_device();
  if (s) return s;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  Temps tmp(st);
  const void* Tdev;
  int64_t ldd;
  if ((s = stage_input(T, nb, h->n, ld, h->dtype, tmp, &Tdev, &ldd)) != SKMP_OK) return s;
  StatsHost sh;
  double *d_mu, *d_inv;
  if ((s = run_stats(Tdev, nb, h->n, ldd, h->dtype, tmp, &sh, &d_mu, &d_inv)) != SKMP_OK) return s;
  std::vector<int32_t> gg((size_t)nb, -1);
  std::vector<int8_t> ss((size_t)nb, 0);
  std::vector<double> Sc;
  if (h->proj == SKMP_PROJ_COUNT_SKETCH) {
    hash_plan(ids, nb, h->k, h->seed, gg.data(), ss.data());
  } else {
    Sc.resize((size_t)nb * h->k);
    for (int64_t j = 0; j < nb; ++j)
      for (int q = 0; q < h->k; ++q) Sc[(size_t)j * h->k + q] = S_cols[(size_t)q * nb + j];
  }
  if ((s = project_rows(h, Tdev, ldd, nb, gg, ss, Sc, sh.mu, sh.sigma, +1, tmp)) != SKMP_OK) return s;
  for (int64_t j = 0; j < nb; ++j) {
    h->pos[ids[j]] = (int64_t)h->ids.size();
    h->ids.push_back(ids[j]);
    h->g.push_back(gg[(size_t)j]);
    h->s.push_back(ss[(size_t)j]);
    h->mu.push_back(sh.mu[(size_t)j]);
    h->sigma.push_back(sh.sigma[(size_t)j]);
    if (h->proj == SKMP_PROJ_DENSE)
      h->Scol.insert(h->Scol.end(), Sc.begin() + (size_t)j * h->k, Sc.begin() + (size_t)(j + 1) * h->k);
  }
  h->st = st;
  return ok();
}

skmp_status sketch_del_dim(skmp_sketch* h, const void* T, int64_t nb, int64_t ld,
                           const uint64_t* ids, void* stream) {
  if (!h || !T || !ids) return set_error(SKMP_E_INVALID_ARG, "sketch_del_dim: NULL argument");
  if (nb < 1 || ld < h->n) return set_error(SKMP_E_INVALID_ARG, "sketch_del_dim: need nb >= 1, ld >= n");
  std::vector<int64_t> at((size_t)nb);
  std::unordered_set<uint64_t> seen;
  for (int64_t j = 0; j < nb; ++j) {
    auto it = h->pos.find(ids[j]);
    if (it == h->pos.end() || !seen.insert(ids[j]).second)
      return set_error(SKMP_E_UNKNOWN_DIM, "sketch_del_dim: stream id not in the sketch", j);
    at[(size_t)j] = it->second;
  }
  skmp_status s = require_device();
  if (s) return s;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  Temps tmp(st);
  const void* Tdev;
  int64_t ldd;
  if ((s = stage_input(T, nb, h->n, ld, h->dtype, tmp, &Tdev, &ldd)) != SKMP_OK) return s;
  std::vector<int32_t> gg((size_t)nb);
  std::vector<int8_t> ss((size_t)nb);
  std::vector<double> mu((size_t)nb), sg((size_t)nb), Sc;
  for (int64_t j = 0; j < nb; ++j) {
    const size_t a = (size_t)at[(size_t)j];
    gg[(size_t)j] = h->g[a];
    ss[(size_t)j] = h->s[a];
    mu[(size_t)j] = h->mu[a];   // STORED statistics: add-then-delete is an exact inverse
    sg[(size_t)j] = h->sigma[a];
    if (h->proj == SKMP_PROJ_DENSE)
      Sc.insert(Sc.end(), h->Scol.begin() + a * h->k, h->Scol.begin() + (a + 1) * h->k);
  }
  if ((s = project_rows(h, Tdev, ldd, nb, gg, ss, Sc, mu, sg, -1, tmp)) != SKMP_OK) return s;
  // drop the deleted dims from the plan (keep the remaining input order)
  std::vector<char> dead(h->ids.size(), 0);
  for (int64_t a : at) dead[(size_t)a] = 1;
  size_t w = 0;
  for (size_t a = 0; a < h->ids.size(); ++a) {
    if (dead[a]) continue;
    h->ids[w] = h->ids[a];
    h->g[w] = h->g[a];
    h->s[w] = h->s[a];
    h->mu[w] = h->mu[a];
    h->sigma[w] = h->sigma[a];
    if (h->proj == SKMP_PROJ_DENSE)
      std::copy(h->Scol.begin() + a * h->k, h->Scol.begin() + (a + 1) * h->k, h->Scol.begin() + w * h->k);
    ++w;
  }
  h->ids.resize(w);
  h->g.resize(w);
  h->s.resize(w);
  h->mu.resize(w);
  h->sigma.resize(w);
  if (h->proj == SKMP_PROJ_DENSE) h->Scol.resize(w * h->k);
  h->pos.clear();
  for (size_t a = 0; a < w; ++a) h->pos[h->ids[a]] = (int64_t)a;
  h->st = st;
  return ok();
}

skmp_status sketch_point_update(skmp_sketch* h, const uint64_t* ids, const int64_t* t, const double* delta,
                                int64_t count, void* stream) {
  if (!h || (count > 0 && (!ids || !t || !delta)) || count < 0)
    return set_error(SKMP_E_INVALID_ARG, "sketch_point_update: NULL argument or count < 0");
  std::vector<int64_t> idx;
  std::vector<double> coef, dl;
  const bool dense = h->proj == SKMP_PROJ_DENSE;
  idx.reserve((size_t)count * (dense ? h->k : 1));
  for (int64_t q = 0; q < count; ++q) {
    auto it = h->pos.find(ids[q]);
    if (it == h->pos.end()) return set_error(SKMP_E_UNKNOWN_DIM, "sketch_point_update: stream id not in the sketch", q);
    if (t[q] < 0 || t[q] >= h->n) return set_error(SKMP_E_INVALID_ARG, "sketch_point_update: time outside [0, n)", q);
    const size_t a = (size_t)it->second;
    // reading 24: the stream's value moves by delta in its own units; the sketch holds the stream
    // z-normalised with its STORED statistics, so its contribution moves by delta / sigma_j
    if (dense) {
      for (int g = 0; g < h->k; ++g) {
        idx.push_back((int64_t)g * h->n + t[q]);
        coef.push_back(h->Scol[a * (size_t)h->k + (size_t)g] / h->sigma[a]);
        dl.push_back(delta[q]);
      }
    } else {
      idx.push_back((int64_t)h->g[a] * h->n + t[q]);
      coef.push_back((double)h->s[a] / h->sigma[a]);
      dl.push_back(delta[q]);
    }
  }
  if (count == 0) return ok();
  skmp_status s = require_device();
  if (s) return s;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  Temps tmp(st);
  int64_t* d_idx;
  double *d_coef, *d_delta;
  if ((s = upload(idx, &d_idx, tmp)) != SKMP_OK) return s;
  if ((s = upload(coef, &d_coef, tmp)) != SKMP_OK) return s;
  if ((s = upload(dl, &d_delta, tmp)) != SKMP_OK) return s;
  SKMP_CUDA(launch_point_update(h->R64, h->R, h->dtype, d_idx, d_coef, d_delta, (int64_t)idx.size(), st));
  h->st = st;
  return ok();
}

skmp_status sketch_view(const skmp_sketch* h, const void** R, int32_t* k, int64_t* n, int64_t* d,
                        int32_t* dtype) {
  if (!h) return set_error(SKMP_E_INVALID_ARG, "sketch_view: NULL handle");
  if (R) *R = h->R;
  if (k) *k = h->k;
  if (n) *n = h->n;
  if (d) *d = (int64_t)h->ids.size();
  if (dtype) *dtype = h->dtype;
  return ok();
}

skmp_status sketch_view64(const skmp_sketch* h, const double** R64) {
  if (!h || !R64) return set_error(SKMP_E_INVALID_ARG, "sketch_view64: NULL argument");
  *R64 = h->R64;
  return ok();
}

skmp_status sketch_plan(const skmp_sketch* h, uint64_t* ids, int32_t* g, int8_t* s, double* mu,
                        double* sigma) {
  if (!h) return set_error(SKMP_E_INVALID_ARG, "sketch_plan: NULL handle");
  const size_t d = h->ids.size();
  if (ids) memcpy(ids, h->ids.data(), d * sizeof(uint64_t));
  if (g) memcpy(g, h->g.data(), d * sizeof(int32_t));
  if (s) memcpy(s, h->s.data(), d * sizeof(int8_t));
  if (mu) memcpy(mu, h->mu.data(), d * sizeof(double));
  if (sigma) memcpy(sigma, h->sigma.data(), d * sizeof(double));
  return ok();
}

skmp_status sketch_refresh(skmp_sketch* h, void* stream) {
  if (!h) return set_error(SKMP_E_INVALID_ARG, "sketch_refresh: NULL handle");
  if (h->R == h->R64) return ok();
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  SKMP_CUDA(launch_cast_r(h->R64, h->R, (int64_t)h->k * h->n, h->dtype, st));
  h->st = st;
  return ok();
}

void sketch_free(skmp_sketch* h) {
  if (!h) return;
  if (h->R && h->R != h->R64) cudaFreeAsync(h->R, h->st);
  if (h->R64) cudaFreeAsync(h->R64, h->st);
  delete h;
}

void sketch_free_async(skmp_sketch* h, void* stream) {
  if (!h) return;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (st != h->st) {  // free after the handle's own work AND everything already queued on `stream`
    cudaEvent_t ev;
    if (cudaEventCreateWithFlags(&ev, cudaEventDisableTiming) == cudaSuccess) {
      if (cudaEventRecord(ev, h->st) == cudaSuccess) cudaStreamWaitEvent(st, ev, 0);
      cudaEventDestroy(ev);
    }
    cudaGetLastError();
    h->st = st;
  }
  sketch_free(h);
}

skmp_status skmp_trim(void) {
  Pools& p = pools();
  std::lock_guard<std::mutex> lock(p.mu);
  for (auto* v : {&p.work, &p.staging})
    for (cudaMemPool_t q : *v)
      if (q) {
        cudaError_t e = cudaMemPoolTrimTo(q, 0);
        if (e != cudaSuccess) return cuda_error(e, "skmp_trim: cudaMemPoolTrimTo");
      }
  return ok();
}

}  // extern "C"

// ============================================================================================
// matrix-profile workspace
// ============================================================================================
struct skmp_mp {
  MpDev w;
  cudaStream_t st = nullptr;
  // per-series flat counts reach the host asynchronously (pinned copy + event, issued by
  // mp_create); host_flags() waits for them the first time the host needs them (finalize's
  // inert flags, the streaming bookkeeping), so mp_create itself never blocks
  std::vector<int32_t> nflat;
  std::vector<uint8_t> inert;
  int32_t* h_nflat = nullptr;  // pinned (recycled, pinned_take / pinned_give)
  size_t h_cap = 0;
  cudaEvent_t flags_ev = nullptr;
  bool flags_ready = false;
  void* base = nullptr;  // single allocation
};

namespace {
int64_t round_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

skmp_status mp_validate(const void* R, int32_t k, int64_t n, int64_t ld, int32_t dtype,
                        const skmp_mp_cfg* cfg, int* excl, bool ab = false) {
  if (!R || !cfg) return set_error(SKMP_E_INVALID_ARG, "mp: NULL argument");
  if (k < 1 || n < 1 || ld < n) return set_error(SKMP_E_INVALID_ARG, "mp: need k >= 1, n >= 1, ld >= n");
  if (dtype != SKMP_F32 && dtype != SKMP_F64) return set_error(SKMP_E_INVALID_ARG, "mp: bad dtype");
  if (cfg->m < 2) return set_error(SKMP_E_INVALID_ARG, "mp: m must be >= 2");
  if (cfg->reseed_rows < 0) return set_error(SKMP_E_INVALID_ARG, "mp: reseed_rows must be >= 0");
  if (n < cfg->m) return set_error(SKMP_E_SERIES_TOO_SHORT, "mp: n < m");
  const int64_t n_sub = n - cfg->m + 1;
  if (n_sub >= (int64_t)INT32_MAX - 1) return set_error(SKMP_E_INVALID_ARG, "mp: n_sub must be < 2^31");
  *excl = cfg->excl < 0 ? (cfg->m + 1) / 2 : cfg->excl;
  if (ab) {  // AB-join: two different series, no exclusion zone (Def. 6)
    *excl = -1;
    return SKMP_OK;
  }
  if (n_sub < 2 * (int64_t)(*excl) + 2)
    return set_error(SKMP_E_NO_ADMISSIBLE, "mp: n_sub < 2*excl + 2 (some row has no admissible neighbour)");
  return SKMP_OK;
}
// Pinned host buffers for mp_create's flag copies, recycled: cudaMallocHost / cudaFreeHost per
// workspace would synchronise the device on every create / free (measured: +1.8 ms per C4 step).
struct PinnedFlags {
  std::mutex mu;
  std::vector<std::pair<size_t, int32_t*>> free_list;
};
PinnedFlags& pinned_flags() {
  static PinnedFlags p;
  return p;
}
cudaError_t pinned_take(size_t count, int32_t** out, size_t* cap) {
  PinnedFlags& p = pinned_flags();
  {
    std::lock_guard<std::mutex> lock(p.mu);
    for (size_t q = 0; q < p.free_list.size(); ++q)
      if (p.free_list[q].first >= count) {
        *cap = p.free_list[q].first;
        *out = p.free_list[q].second;
        p.free_list.erase(p.free_list.begin() + (long)q);
        return cudaSuccess;
      }
  }
  *cap = count < 256 ? 256 : count;
  return cudaMallocHost((void**)out, sizeof(int32_t) * *cap);
}
void pinned_give(int32_t* ptr, size_t cap) {
  if (!ptr) return;
  PinnedFlags& p = pinned_flags();
  std::lock_guard<std::mutex> lock(p.mu);
  p.free_list.emplace_back(cap, ptr);
}

// wait (once) for mp_create's asynchronous copy of the per-series flat counts
skmp_status host_flags(skmp_mp* h) {
  if (h->flags_ready) return SKMP_OK;
  SKMP_CUDA(cudaEventSynchronize(h->flags_ev));
  const int k = h->w.k;
  h->nflat.assign(h->h_nflat, h->h_nflat + k);
  h->inert.assign((size_t)k, 0);
  for (int g = 0; g < k; ++g) h->inert[(size_t)g] = h->nflat[(size_t)g] == h->w.n_sub;
  h->flags_ready = true;
  return SKMP_OK;
}
}  // namespace

extern "C" {

}  // extern "C"

namespace {
skmp_status mp_create_impl(const void* R, int32_t k, int64_t n, int64_t ld, int32_t dtype,
                           const skmp_mp_cfg* cfg, void* stream, skmp_mp** out, bool ab) {
  int excl = 0;
  skmp_status s = mp_validate(R, k, n, ld, dtype, cfg, &excl, ab);
  if (s) return s;
  if (!out) return set_error(SKMP_E_INVALID_ARG, "mp_create: NULL out");
  if ((s = require_device()) != SKMP_OK) return s;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  skmp_mp* h = new skmp_mp();
  MpDev& w = h->w;
  w.dtype = dtype;
  w.k = k;
  w.n = n;
  w.ld = ld;
  w.m = cfg->m;
  w.excl = excl;
  w.n_sub = n - cfg->m + 1;
  w.ldq = round_up(w.n_sub + join_pad(dtype), 64);
  // FP32 re-seed interval: 16,384 rows; 32,768 for series of >= 2^20 windows, where the longer
  // tiles amortise the seeds better (measured: C5-length join 1683 -> 1676 ms; at C4 size the
  // longer tiles were slower, 283 -> 287 ms).  FP32 rho drift stays ~1e-5; P is
  // resolved exactly in FP64 by the finalize either way.
  int L0 = cfg->reseed_rows > 0 ? cfg->reseed_rows
                                : (dtype == SKMP_F32 ? ((n - cfg->m + 1) >= (1 << 20) ? 32768 : 16384) : 2048);
  if (cfg->reseed_rows <= 0) {
    // small problems: shorten the tiles until the grid has ~2 waves of 148 SMs x 16 warps
    const int64_t W = join_width(dtype);
    auto tiles = [&](int64_t L) {
      int64_t t = 0;
      for (int64_t d0 = ((excl + 1) / W) * W; d0 < w.n_sub; d0 += W) {
        const int64_t rows = w.n_sub - (d0 > excl + 1 ? d0 : excl + 1);
        t += (rows + L - 1) / L;
      }
      return t * k;
    };
    while (L0 > 256 && tiles(L0) < 2 * 148 * 16) L0 /= 2;
  }
  w.L = (int)round_up(L0, 64);
  w.span = join_span(dtype);
  w.R = R;
  const int words = dtype == SKMP_F32 ? 1 : 2;
  const size_t qsz = dtype == SKMP_F32 ? 16 : 32;
  const size_t kq = (size_t)k * (size_t)w.ldq;
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off += (bytes + 255) / 256 * 256; return o; };
  const size_t oQ = take(qsz * kq), oMu = take(8 * kq), oSig = take(8 * kq), oISig = take(8 * kq), oFlat = take(kq),
               oAmax = take(8 * (size_t)k), oNf = take(4 * (size_t)k),
               oKeys = take(8 * (size_t)words * (size_t)k * (size_t)w.n_sub),
               oFL = take(4 * (size_t)k * (size_t)w.n_sub);
  cudaError_t e = dmalloc(&h->base, off, st);
  if (e != cudaSuccess) {
    delete h;
    return cuda_error(e, "mp_create: allocate workspace");
  }
  char* b = static_cast<char*>(h->base);
  w.Q = b + oQ;
  w.mu = reinterpret_cast<double*>(b + oMu);
  w.sig64 = reinterpret_cast<double*>(b + oSig);
  w.isig64 = reinterpret_cast<double*>(b + oISig);
  w.flat = reinterpret_cast<uint8_t*>(b + oFlat);
  w.amax = reinterpret_cast<double*>(b + oAmax);
  w.nflat = reinterpret_cast<int32_t*>(b + oNf);
  w.keys = reinterpret_cast<int64_t*>(b + oKeys);
  w.flat_list = reinterpret_cast<int32_t*>(b + oFL);
  h->st = st;
  e = launch_mp_prep(w, st);
  if (e == cudaSuccess) e = launch_keys_init(w, st);
  if (e == cudaSuccess) e = launch_flat_lists(w, st);
  if (e == cudaSuccess) e = pinned_take((size_t)k, &h->h_nflat, &h->h_cap);
  if (e == cudaSuccess) e = cudaMemcpyAsync(h->h_nflat, w.nflat, sizeof(int32_t) * k, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->flags_ev, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventRecord(h->flags_ev, st);
  if (e != cudaSuccess) {
    mp_free(h);
    return cuda_error(e, "mp_create: window preparation");
  }
  *out = h;
  return ok();
}

// tiles of the diagonal band [lo, hi) of rows wr against columns wc, then the join launch
skmp_status join_band(const MpDev& wr, const MpDev& wc, int64_t lo, int64_t hi, cudaStream_t st) {
  if (lo >= hi) return SKMP_OK;
  const int64_t W = join_width(wr.dtype);
  const int64_t blk0 = lo / W, blk1 = (hi + W - 1) / W;
  const int64_t nblk = blk1 - blk0;
  std::vector<int64_t> prefix((size_t)nblk + 1, 0);
  for (int64_t b = 0; b < nblk; ++b) {
    const int64_t d0 = (blk0 + b) * W;
    const int64_t dmin = d0 > lo ? d0 : lo;
    const int64_t rows = tile_rows(wr.n_sub, wc.n_sub, dmin);
    prefix[(size_t)b + 1] = prefix[(size_t)b] + (rows > 0 ? (rows + wr.L - 1) / wr.L : 0);
  }
  const int64_t ntiles = prefix[(size_t)nblk];
  if (ntiles * wr.k > INT32_MAX) return set_error(SKMP_E_INVALID_ARG, "mp_join: too many tiles; raise reseed_rows");
  Temps tmp(st);
  int64_t* d_prefix = nullptr;
  skmp_status s = upload(prefix, &d_prefix, tmp);
  if (s) return s;
  SKMP_CUDA(launch_mp_join(wr, wc, lo, hi, d_prefix, nblk, ntiles, blk0, st));
  return SKMP_OK;
}
}  // namespace

extern "C" {

skmp_status mp_create(const void* R, int32_t k, int64_t n, int64_t ld, int32_t dtype,
                      const skmp_mp_cfg* cfg, void* stream, skmp_mp** out) {
  return mp_create_impl(R, k, n, ld, dtype, cfg, stream, out, false);
}

skmp_status mp_band(int64_t n_sub, int32_t excl, int32_t dtype, int32_t nbands, int32_t band,
                    int64_t* diag_lo, int64_t* diag_hi) {
  if (nbands < 1 || band < 0 || band >= nbands || !diag_lo || !diag_hi || n_sub < 2 || excl < 0)
    return set_error(SKMP_E_INVALID_ARG, "mp_band: bad arguments");
  const int64_t W = join_width(dtype);
  const int64_t lo0 = excl + 1;
  if (lo0 >= n_sub) {
    *diag_lo = *diag_hi = 0;
    return ok();
  }
  // cost of diagonals [lo0, x): their cells, sum_{delta=lo0}^{x-1} (n_sub - delta), plus a fixed
  // kBandDiagCost cells per diagonal for the per-tile work that does not scale with the tile's
  // rows (exact seeds, staging prologue, the masked triangle at the end of every diagonal block):
  // measured on one B200 (tools/band_balance.py), the short-diagonal bands of an equal-cell
  // split ran 5-7 % longer than the others
  const double kBandDiagCost = 5.0 * (double)W;
  // and the first block of W diagonals is joined while every key is still empty: its rows keep
  // improving (near neighbours), so it publishes far more than any later block (measured: the
  // rank holding it ran ~5 ms longer at 8 bands of C4) — its cells count 4.5 times
  const double kFirstBlockExtra = 3.5;
  auto S = [&](int64_t x) -> double {
    const double a = (double)(x - lo0);
    const double f = (double)std::min<int64_t>(x - lo0, W);
    return a * (double)(n_sub - lo0) - a * (a - 1.0) / 2.0 + kBandDiagCost * a +
           kFirstBlockExtra * (f * (double)(n_sub - lo0) - f * (f - 1.0) / 2.0);
  };
  const double total = S(n_sub);
  auto edge = [&](int32_t p) -> int64_t {
    if (p <= 0) return 0;
    if (p >= nbands) return n_sub;
    const double target = total * (double)p / (double)nbands;
    int64_t lo = lo0, hi = n_sub;
    while (lo < hi) {
      const int64_t mid = (lo + hi) / 2;
      if (S(mid) < target) lo = mid + 1; else hi = mid;
    }
    int64_t x = (lo + W / 2) / W * W;  // nearest multiple of the tile width
    if (x > n_sub) x = n_sub;
    return x;
  };
  int64_t a = edge(band), b = edge(band + 1);
  // keep edges monotone after rounding
  for (int32_t p = band - 1; p >= 0 && a < edge(p); --p) a = edge(p);
  if (b < a) b = a;
  *diag_lo = a;
  *diag_hi = b;
  return ok();
}

int32_t mp_tile_width(int32_t dtype) { return join_width(dtype == SKMP_F64 ? SKMP_F64 : SKMP_F32); }

skmp_status mp_join(skmp_mp* h, int64_t diag_lo, int64_t diag_hi, void* stream) {
  if (!h) return set_error(SKMP_E_INVALID_ARG, "mp_join: NULL workspace");
  if (diag_lo < 0 || diag_hi < 0 || (diag_hi < diag_lo))
    return set_error(SKMP_E_INVALID_ARG, "mp_join: bad diagonal band");
  MpDev& w = h->w;
  if (w.excl < 0) return set_error(SKMP_E_INVALID_ARG, "mp_join: AB workspace; use mp_join_ab");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  int64_t lo = diag_lo, hi = diag_hi;
  if (lo == 0 && hi == 0) hi = w.n_sub;
  if (lo < w.excl + 1) lo = w.excl + 1;
  if (hi > w.n_sub) hi = w.n_sub;
  if (lo >= hi) return ok();
  skmp_status s = join_band(w, w, lo, hi, st);
  if (s) return s;
  h->st = st;
  return ok();
}

skmp_status mp_keys(skmp_mp* h, void** keys, int64_t* count, int32_t* words) {
  if (!h) return set_error(SKMP_E_INVALID_ARG, "mp_keys: NULL workspace");
  const int wd = h->w.dtype == SKMP_F32 ? 1 : 2;
  if (keys) *keys = h->w.keys;
  if (count) *count = (int64_t)h->w.k * h->w.n_sub * wd;
  if (words) *words = wd;
  return ok();
}

skmp_status mp_finalize(skmp_mp* h, void* P, int64_t* I, uint8_t* inert, void* stream) {
  if (!h || !P || !I) return set_error(SKMP_E_INVALID_ARG, "mp_finalize: NULL argument");
  if (h->w.excl < 0) return set_error(SKMP_E_INVALID_ARG, "mp_finalize: AB workspace; use mp_finalize_ab");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  SKMP_CUDA(launch_mp_finalize(h->w, h->w, h->w.excl, P, I, st));
  if (inert) {
    skmp_status s = host_flags(h);
    if (s) return s;
    memcpy(inert, h->inert.data(), h->inert.size());
  }
  h->st = st;
  return ok();
}

skmp_status mp_finalize_rows(skmp_mp* h, int64_t row_lo, int64_t row_hi, void* P, int64_t* I,
                             uint8_t* inert, void* stream) {
  if (!h || !P || !I) return set_error(SKMP_E_INVALID_ARG, "mp_finalize_rows: NULL argument");
  if (h->w.excl < 0) return set_error(SKMP_E_INVALID_ARG, "mp_finalize_rows: AB workspace; use mp_finalize_ab");
  if (row_lo < 0 || row_hi < row_lo || row_hi > h->w.n_sub)
    return set_error(SKMP_E_INVALID_ARG, "mp_finalize_rows: need 0 <= row_lo <= row_hi <= n_sub");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  SKMP_CUDA(launch_mp_finalize(h->w, h->w, h->w.excl, P, I, st, row_lo, row_hi));
  if (inert) {
    skmp_status s = host_flags(h);
    if (s) return s;
    memcpy(inert, h->inert.data(), h->inert.size());
  }
  h->st = st;
  return ok();
}

void mp_free(skmp_mp* h) {
  if (!h) return;
  if (h->flags_ev) {
    cudaEventSynchronize(h->flags_ev);  // the pinned flag buffer may still be the copy's target
    cudaEventDestroy(h->flags_ev);
  }
  pinned_give(h->h_nflat, h->h_cap);
  if (h->base) cudaFreeAsync(h->base, h->st);
  delete h;
}

skmp_status mp_selfjoin(const void* R, int32_t k, int64_t n, int64_t ld, int32_t dtype,
                        const skmp_mp_cfg* cfg, void* P, int64_t* I, uint8_t* inert, void* stream) {
  if (!P || !I) return set_error(SKMP_E_INVALID_ARG, "mp_selfjoin: NULL output");
  skmp_mp* h = nullptr;
  skmp_status s = mp_create(R, k, n, ld, dtype, cfg, stream, &h);
  if (s) return s;
  s = mp_join(h, 0, 0, stream);
  if (s == SKMP_OK) s = mp_finalize(h, P, I, inert, stream);
  mp_free(h);
  return s;
}

skmp_status mp_create_ab(const void* R, int32_t k, int64_t n, int64_t ld, int32_t dtype,
                         const skmp_mp_cfg* cfg, void* stream, skmp_mp** out) {
  return mp_create_impl(R, k, n, ld, dtype, cfg, stream, out, true);
}

skmp_status mp_join_ab(skmp_mp* rows, skmp_mp* cols, int64_t diag_lo, int64_t diag_hi, void* stream) {
  if (!rows || !cols) return set_error(SKMP_E_INVALID_ARG, "mp_join_ab: NULL workspace");
  if (rows->w.excl >= 0 || cols->w.excl >= 0)
    return set_error(SKMP_E_INVALID_ARG, "mp_join_ab: workspaces must come from mp_create_ab");
  if (rows->w.k != cols->w.k || rows->w.dtype != cols->w.dtype || rows->w.m != cols->w.m)
    return set_error(SKMP_E_INVALID_ARG, "mp_join_ab: k / dtype / m differ");
  if (diag_lo < 0 || diag_hi < diag_lo) return set_error(SKMP_E_INVALID_ARG, "mp_join_ab: bad diagonal band");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t hi = std::min(diag_hi, cols->w.n_sub);
  skmp_status s = join_band(rows->w, cols->w, diag_lo, hi, st);
  if (s) return s;
  rows->st = cols->st = st;
  return ok();
}

skmp_status mp_finalize_ab(skmp_mp* w, skmp_mp* other, int64_t row_lo, int64_t row_hi, void* P, int64_t* I,
                           uint8_t* inert, void* stream) {
  if (!w || !other || !P || !I) return set_error(SKMP_E_INVALID_ARG, "mp_finalize_ab: NULL argument");
  if (w->w.excl >= 0 || other->w.excl >= 0)
    return set_error(SKMP_E_INVALID_ARG, "mp_finalize_ab: workspaces must come from mp_create_ab");
  if (row_lo == 0 && row_hi == 0) row_hi = w->w.n_sub;
  if (row_lo < 0 || row_hi < row_lo || row_hi > w->w.n_sub)
    return set_error(SKMP_E_INVALID_ARG, "mp_finalize_ab: need 0 <= row_lo <= row_hi <= n_sub");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  SKMP_CUDA(launch_mp_finalize(w->w, other->w, -1, P, I, st, row_lo, row_hi));
  if (inert) {  // reading 22: inert when both series of the group are entirely flat
    skmp_status s = host_flags(w);
    if (s == SKMP_OK) s = host_flags(other);
    if (s) return s;
    for (int g = 0; g < w->w.k; ++g) inert[g] = w->inert[(size_t)g] && other->inert[(size_t)g];
  }
  w->st = st;
  return ok();
}

skmp_status mp_abband(int64_t n_subA, int64_t n_subB, int32_t dtype, int32_t nbands, int32_t band,
                      int64_t* lo1, int64_t* hi1, int64_t* lo2, int64_t* hi2) {
  if (n_subA < 1 || n_subB < 1 || nbands < 1 || band < 0 || band >= nbands || !lo1 || !hi1 || !lo2 || !hi2)
    return set_error(SKMP_E_INVALID_ARG, "mp_abband: bad arguments");
  const int64_t W = join_width(dtype == SKMP_F64 ? SKMP_F64 : SKMP_F32);
  // the two passes as one sequence of diagonals: pass 1 delta in [0, n_subB) (min(n_subA,
  // n_subB - delta) cells), then pass 2 delta in [1, n_subA) (min(n_subB, n_subA - delta) cells)
  auto cum1 = [&](int64_t x) -> double {  // cells of pass-1 diagonals [0, x)
    double c = 0.0;
    const int64_t flat = std::max<int64_t>(0, std::min(x, n_subB - n_subA));  // delta < nB - nA: nA cells
    c += (double)flat * (double)n_subA;
    const int64_t a = std::max<int64_t>(flat, 0), b = x;  // cells nB - delta
    if (b > a) c += (double)(b - a) * (double)n_subB - ((double)b * (b - 1) - (double)a * (a - 1)) / 2.0;
    return c;
  };
  auto cum2 = [&](int64_t y) -> double {  // cells of pass-2 diagonals [1, y)
    if (y <= 1) return 0.0;
    double c = 0.0;
    const int64_t flat_end = std::max<int64_t>(1, std::min(y, n_subA - n_subB));  // delta < nA - nB: nB cells
    c += (double)(flat_end - 1) * (double)n_subB;
    const int64_t a = flat_end, b = y;
    if (b > a) c += (double)(b - a) * (double)n_subA - ((double)b * (b - 1) - (double)a * (a - 1)) / 2.0;
    return c;
  };
  const double tot1 = cum1(n_subB), tot = tot1 + cum2(n_subA);
  // edge p of the split as a position (pass, delta), rounded to the tile grid of its pass
  auto edge = [&](int32_t p, int* pass, int64_t* delta) {
    if (p <= 0) { *pass = 1; *delta = 0; return; }
    if (p >= nbands) { *pass = 2; *delta = n_subA; return; }
    const double target = tot * (double)p / (double)nbands;
    if (target < tot1) {
      int64_t lo = 0, hi = n_subB;
      while (lo < hi) { const int64_t mid = (lo + hi) / 2; if (cum1(mid) < target) lo = mid + 1; else hi = mid; }
      *pass = 1;
      *delta = std::min<int64_t>(n_subB, (lo + W / 2) / W * W);
    } else {
      int64_t lo = 1, hi = n_subA;
      while (lo < hi) { const int64_t mid = (lo + hi) / 2; if (tot1 + cum2(mid) < target) lo = mid + 1; else hi = mid; }
      *pass = 2;
      *delta = std::max<int64_t>(1, std::min<int64_t>(n_subA, (lo + W / 2) / W * W));
    }
  };
  int pa, pb;
  int64_t da, db;
  edge(band, &pa, &da);
  edge(band + 1, &pb, &db);
  *lo1 = *hi1 = *lo2 = *hi2 = 0;
  if (pa == 1) {
    *lo1 = da;
    *hi1 = pb == 1 ? std::max(da, db) : n_subB;
    if (pb == 2) { *lo2 = 1; *hi2 = std::max<int64_t>(1, db); }
  } else {
    *lo2 = std::max<int64_t>(1, da);
    *hi2 = std::max(*lo2, db);
  }
  return ok();
}

skmp_status mp_abjoin(const void* RA, int64_t nA, int64_t ldA, const void* RB, int64_t nB, int64_t ldB,
                      int32_t k, int32_t dtype, const skmp_mp_cfg* cfg, void* PA, int64_t* IA, void* PB,
                      int64_t* IB, uint8_t* inert, void* stream) {
  if (!PA || !IA || (PB && !IB) || (!PB && IB)) return set_error(SKMP_E_INVALID_ARG, "mp_abjoin: NULL output");
  int ex = 0;
  skmp_status s = mp_validate(RA, k, nA, ldA, dtype, cfg, &ex, true);
  if (s) return s;
  if ((s = mp_validate(RB, k, nB, ldB, dtype, cfg, &ex, true)) != SKMP_OK) return s;
  skmp_mp *a = nullptr, *b = nullptr;
  if ((s = mp_create_impl(RA, k, nA, ldA, dtype, cfg, stream, &a, true)) != SKMP_OK) return s;
  if ((s = mp_create_impl(RB, k, nB, ldB, dtype, cfg, stream, &b, true)) != SKMP_OK) {
    mp_free(a);
    return s;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // pass 1: rows = test windows i, columns = train windows j = i + delta, delta in [0, n_subB)
  // pass 2: rows = train windows j, columns = test windows i = j + delta, delta in [1, n_subA)
  s = join_band(a->w, b->w, 0, b->w.n_sub, st);
  if (s == SKMP_OK) s = join_band(b->w, a->w, 1, a->w.n_sub, st);
  if (s == SKMP_OK) {
    cudaError_t e = launch_mp_finalize(a->w, b->w, -1, PA, IA, st);
    if (e == cudaSuccess && PB) e = launch_mp_finalize(b->w, a->w, -1, PB, IB, st);
    if (e != cudaSuccess) s = cuda_error(e, "mp_abjoin: finalize");
  }
  if (s == SKMP_OK && inert) {
    // reading 6 for an AB-join: a group is inert when both its test and train sketch series
    // are entirely flat (an empty group)
    s = host_flags(a);
    if (s == SKMP_OK) s = host_flags(b);
    if (s == SKMP_OK)
      for (int g = 0; g < k; ++g) inert[g] = a->inert[(size_t)g] && b->inert[(size_t)g];
  }
  mp_free(a);
  mp_free(b);
  return s == SKMP_OK ? ok() : s;
}

// ============================================================================================
// streaming test data (f4)
// ============================================================================================
}  // extern "C"

struct skmp_stream {
  skmp_sketch plan;            // the train sketch's plan and statistics; R64 / R = the test sketch (k x cap)
  skmp_mp* train = nullptr;    // AB workspace of a private copy of the train sketch
  void* Rtrain = nullptr;      // that copy (k x n_train, dtype)
  void* P = nullptr;           // k x cap test profile (row stride cap)
  int64_t* I = nullptr;
  int64_t cap = 0, n_test = 0;
  skmp_mp_cfg cfg{};
  std::vector<int64_t> nflat;  // flat test windows so far, per group
  // carried AB rows (stream.cu): FP64 train records, two rings of per-diagonal covariances
  void* q64 = nullptr;
  double* ring[2] = {nullptr, nullptr};
  int cur = 0;
  bool state_valid = false;    // ring[cur] holds the covariances of test window state_t - 1
  int64_t state_t = 0;
};

extern "C" {

skmp_status stream_create(const skmp_sketch* train, const skmp_mp_cfg* cfg, int64_t capacity, void* stream,
                          skmp_stream** out) {
  if (!train || !cfg || !out) return set_error(SKMP_E_INVALID_ARG, "stream_create: NULL argument");
  if (capacity < cfg->m || capacity >= (int64_t)INT32_MAX)
    return set_error(SKMP_E_INVALID_ARG, "stream_create: need m <= capacity < 2^31");
  int ex = 0;
  skmp_status s = mp_validate(train->R, train->k, train->n, train->n, train->dtype, cfg, &ex, true);
  if (s) return s;
  if ((s = require_device()) != SKMP_OK) return s;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  skmp_stream* h = new skmp_stream();
  skmp_sketch& q = h->plan;
  q.dtype = train->dtype;
  q.proj = train->proj;
  q.k = train->k;
  q.n = capacity;
  q.seed = train->seed;
  q.st = st;
  q.ids = train->ids;
  q.g = train->g;
  q.s = train->s;
  q.mu = train->mu;
  q.sigma = train->sigma;
  q.Scol = train->Scol;
  h->cap = capacity;
  h->cfg = *cfg;
  h->nflat.assign((size_t)train->k, 0);
  const size_t es = elem_size(train->dtype), kc = (size_t)train->k * (size_t)capacity;
  cudaError_t e = dmalloc((void**)&q.R64, sizeof(double) * kc, st);
  if (e == cudaSuccess) {
    if (q.dtype == SKMP_F32) e = dmalloc(&q.R, sizeof(float) * kc, st);
    else q.R = q.R64;
  }
  if (e == cudaSuccess) e = dmalloc(&h->P, es * kc, st);
  if (e == cudaSuccess) e = dmalloc((void**)&h->I, sizeof(int64_t) * kc, st);
  if (e == cudaSuccess) e = dmalloc(&h->Rtrain, es * (size_t)train->k * (size_t)train->n, st);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(h->Rtrain, train->R, es * (size_t)train->k * (size_t)train->n, cudaMemcpyDeviceToDevice, st);
  if (e != cudaSuccess) {
    stream_free(h);
    return cuda_error(e, "stream_create: allocate");
  }
  if ((s = mp_create_impl(h->Rtrain, train->k, train->n, train->n, train->dtype, cfg, stream, &h->train, true)) !=
          SKMP_OK ||
      (s = host_flags(h->train)) != SKMP_OK) {
    stream_free(h);
    return s;
  }
  // carried-path state: FP64 train records only for FP64 streams (FP32 streams use the train
  // workspace's own FP32 records); rings of one value per diagonal in the stream's dtype
  const size_t nring = (size_t)train->k * (size_t)h->train->w.n_sub;
  e = dmalloc((void**)&h->ring[0], es * nring, st);
  if (e == cudaSuccess) e = dmalloc((void**)&h->ring[1], es * nring, st);
  if (e == cudaSuccess && train->dtype == SKMP_F64) e = dmalloc(&h->q64, stream_q64_bytes(h->train->w), st);
  if (e == cudaSuccess && train->dtype == SKMP_F64) e = launch_train_q64(h->train->w, h->q64, st);
  if (e != cudaSuccess) {
    stream_free(h);
    return cuda_error(e, "stream_create: train records");
  }
  *out = h;
  return ok();
}

skmp_status stream_push(skmp_stream* h, const void* T, int64_t n_new, int64_t ld, void* stream) {
  if (!h || !T) return set_error(SKMP_E_INVALID_ARG, "stream_push: NULL argument");
  if (n_new < 1 || ld < n_new) return set_error(SKMP_E_INVALID_ARG, "stream_push: need n_new >= 1, ld >= n_new");
  if (h->n_test + n_new > h->cap) return set_error(SKMP_E_INVALID_ARG, "stream_push: capacity exceeded");
  skmp_status s = require_device();
  if (s) return s;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  skmp_sketch& q = h->plan;
  const int64_t d = (int64_t)q.ids.size();
  const size_t es = elem_size(q.dtype);
  {
    // Alg. 1 lines 4-5 for the new time points only, with the train statistics (reading 25)
    Temps tmp(st);
    const void* Tdev;
    int64_t ldd;
    if ((s = stage_input(T, d, n_new, ld, q.dtype, tmp, &Tdev, &ldd)) != SKMP_OK) return s;
    char* Rc = static_cast<char*>(q.R) + (size_t)h->n_test * es;
    if ((s = project_into(&q, Tdev, ldd, d, n_new, q.g, q.s, q.Scol, q.mu, q.sigma, 0, q.R64 + h->n_test, Rc,
                          h->cap, tmp)) != SKMP_OK)
      return s;
    // non-finite input: rejected before the columns become part of the stream (n_test unchanged)
    int32_t* flag = nullptr;
    int32_t hflag = INT32_MAX;
    SKMP_CUDA(tmp.alloc(&flag, 1));
    SKMP_CUDA(cudaMemcpyAsync(flag, &hflag, sizeof(int32_t), cudaMemcpyHostToDevice, st));
    SKMP_CUDA(launch_nonfinite_check(q.R64, h->cap, q.k, h->n_test, n_new, flag, st));
    SKMP_CUDA(cudaMemcpyAsync(&hflag, flag, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    SKMP_CUDA(cudaStreamSynchronize(st));
    if (hflag != INT32_MAX)
      return set_error(SKMP_E_NONFINITE, "stream_push: non-finite value in the new points (index = its group)", hflag);
  }
  const int m = h->cfg.m;
  const int64_t w0 = std::max<int64_t>(0, h->n_test - m + 1), w1 = h->n_test + n_new - m + 1;
  q.st = st;
  // n_test advances only when the push completes: a failed push leaves the stream as it was (its
  // projected columns lie beyond n_test and are overwritten by the next push)
  if (w1 <= w0) {
    h->n_test += n_new;
    return ok();
  }
  const int64_t B = w1 - w0;
  if (B <= kStreamIncrMax) {
    // carried path: the block starts one window early (the predecessor row's df / dg need it)
    const int64_t base = w0 > 0 ? w0 - 1 : 0;
    skmp_mp* a = nullptr;
    const char* blk = static_cast<const char*>(q.R) + (size_t)base * es;
    if ((s = mp_create_impl(blk, q.k, w1 - 1 + m - base, h->cap, q.dtype, &h->cfg, stream, &a, true)) != SKMP_OK)
      return s;
    skmp_mp* tr = h->train;
    const bool valid = h->state_valid && h->state_t == w0;
    cudaError_t e = launch_stream_rows(a->w, base, tr->w, h->q64, h->ring[h->cur], h->ring[h->cur ^ 1], w0, (int)B,
                                       valid, st);
    const int64_t l0 = w0 - base, nsb = a->w.n_sub;
    std::vector<uint8_t> pred((size_t)q.k, 0);
    {
      Temps tmp(st);
      char* Pb = nullptr;
      int64_t* Ib = nullptr;
      if (e == cudaSuccess) e = tmp.alloc(&Pb, es * (size_t)q.k * (size_t)nsb);
      if (e == cudaSuccess) e = tmp.alloc(&Ib, (size_t)q.k * (size_t)nsb);
      if (e == cudaSuccess) e = launch_mp_finalize(a->w, tr->w, -1, Pb, Ib, st, l0, l0 + B);
      if (e == cudaSuccess)
        e = cudaMemcpy2DAsync(static_cast<char*>(h->P) + (size_t)w0 * es, (size_t)h->cap * es, Pb + (size_t)l0 * es,
                              (size_t)nsb * es, (size_t)B * es, (size_t)q.k, cudaMemcpyDeviceToDevice, st);
      if (e == cudaSuccess)
        e = cudaMemcpy2DAsync(h->I + w0, (size_t)h->cap * 8, Ib + l0, (size_t)nsb * 8, (size_t)B * 8, (size_t)q.k,
                              cudaMemcpyDeviceToDevice, st);
      // the predecessor window was counted by the push that completed it
      if (e == cudaSuccess && l0 > 0)
        e = cudaMemcpy2DAsync(pred.data(), 1, a->w.flat, (size_t)a->w.ldq, 1, (size_t)q.k, cudaMemcpyDeviceToHost, st);
      if (e == cudaSuccess && l0 > 0) e = cudaStreamSynchronize(st);
    }
    if (e != cudaSuccess) {
      h->state_valid = false;
      mp_free(a);
      return cuda_error(e, "stream_push: carried rows");
    }
    if ((s = host_flags(a)) != SKMP_OK) {
      h->state_valid = false;
      mp_free(a);
      return s;
    }
    for (int g = 0; g < q.k; ++g) h->nflat[(size_t)g] += a->nflat[(size_t)g] - pred[(size_t)g];
    h->cur ^= 1;
    h->state_valid = true;
    h->state_t = w1;
    h->n_test += n_new;
    tr->st = st;
    mp_free(a);
    return ok();
  }
  // the new test windows [w0, w1) as one series block, AB-joined against every train window
  h->state_valid = false;  // the tiled join does not carry covariances
  skmp_mp* a = nullptr;
  const char* blk = static_cast<const char*>(q.R) + (size_t)w0 * es;
  if ((s = mp_create_impl(blk, q.k, B + m - 1, h->cap, q.dtype, &h->cfg, stream, &a, true)) != SKMP_OK) return s;
  skmp_mp* tr = h->train;
  s = join_band(a->w, tr->w, 0, tr->w.n_sub, st);
  if (s == SKMP_OK) s = join_band(tr->w, a->w, 1, a->w.n_sub, st);
  if (s == SKMP_OK) {
    Temps tmp(st);
    char* Pb = nullptr;
    int64_t* Ib = nullptr;
    cudaError_t e = tmp.alloc(&Pb, es * (size_t)q.k * (size_t)B);
    if (e == cudaSuccess) e = tmp.alloc(&Ib, (size_t)q.k * (size_t)B);
    if (e == cudaSuccess) e = launch_mp_finalize(a->w, tr->w, -1, Pb, Ib, st);
    if (e == cudaSuccess)
      e = cudaMemcpy2DAsync(static_cast<char*>(h->P) + (size_t)w0 * es, (size_t)h->cap * es, Pb, (size_t)B * es,
                            (size_t)B * es, (size_t)q.k, cudaMemcpyDeviceToDevice, st);
    if (e == cudaSuccess)
      e = cudaMemcpy2DAsync(h->I + w0, (size_t)h->cap * 8, Ib, (size_t)B * 8, (size_t)B * 8, (size_t)q.k,
                            cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) s = cuda_error(e, "stream_push: finalize");
  }
  if (s == SKMP_OK) s = host_flags(a);
  if (s == SKMP_OK) {
    for (int g = 0; g < q.k; ++g) h->nflat[(size_t)g] += a->nflat[(size_t)g];
    h->n_test += n_new;
  }
  tr->st = st;
  mp_free(a);
  return s == SKMP_OK ? ok() : s;
}

skmp_status stream_view(const skmp_stream* h, void** R, void** P, int64_t** I, int64_t* n_test, int64_t* n_sub,
                        int64_t* ld, uint8_t* inert) {
  if (!h) return set_error(SKMP_E_INVALID_ARG, "stream_view: NULL stream");
  if (R) *R = h->plan.R;
  if (P) *P = h->P;
  if (I) *I = h->I;
  const int64_t ns = std::max<int64_t>(0, h->n_test - h->cfg.m + 1);
  if (n_test) *n_test = h->n_test;
  if (n_sub) *n_sub = ns;
  if (ld) *ld = h->cap;
  if (inert)  // reading 22: inert when the train series and every test window so far are flat
    for (int g = 0; g < h->plan.k; ++g) inert[g] = h->train->inert[(size_t)g] && h->nflat[(size_t)g] == ns;
  return ok();
}

void stream_free(skmp_stream* h) {
  if (!h) return;
  cudaStream_t st = h->plan.st;
  if (h->train) mp_free(h->train);
  if (h->Rtrain) cudaFreeAsync(h->Rtrain, st);
  if (h->q64) cudaFreeAsync(h->q64, st);
  if (h->ring[0]) cudaFreeAsync(h->ring[0], st);
  if (h->ring[1]) cudaFreeAsync(h->ring[1], st);
  if (h->P) cudaFreeAsync(h->P, st);
  if (h->I) cudaFreeAsync(h->I, st);
  if (h->plan.R && h->plan.R != h->plan.R64) cudaFreeAsync(h->plan.R, st);
  if (h->plan.R64) cudaFreeAsync(h->plan.R64, st);
  h->plan.R = h->plan.R64 = nullptr;
  delete h;
}

}  // extern "C"

namespace {

// Alg. 3 lines 3-7: the first strict maximiser in order (reading 20: the scan starts from -inf)
int64_t first_strict_max(const std::vector<double>& v) {
  int64_t best = -1;
  for (size_t q = 0; q < v.size(); ++q)
    if (best < 0 || v[q] > v[(size_t)best]) best = (int64_t)q;
  return best;
}

skmp_status dims_validate(const char* who, int64_t n, int64_t t_star, int m, int excl, int* ex) {
  if (n < m) return set_error(SKMP_E_SERIES_TOO_SHORT, std::string(who) + ": n < m");
  const int64_t n_sub = n - m + 1;
  if (t_star < 0 || t_star >= n_sub)
    return set_error(SKMP_E_INVALID_ARG, std::string(who) + ": t_star outside [0, n-m+1)", t_star);
  *ex = excl < 0 ? (m + 1) / 2 : excl;
  if (t_star - *ex - 1 < 0 && t_star + *ex + 1 >= n_sub)
    return set_error(SKMP_E_NO_ADMISSIBLE, std::string(who) + ": no window farther than excl from t_star");
  return SKMP_OK;
}

// K9 over the listed rows of one source matrix into d_score / d_nn (device, rows.size() each);
// a host matrix is staged row by row (only the listed rows cross PCIe)
skmp_status dims_rows(const void* T, int64_t ld, int64_t n, int dtype, std::vector<int64_t> rows, int64_t t_star,
                      int m, int ex, double* d_score, int64_t* d_nn, Temps& tmp) {
  const int64_t nrows = (int64_t)rows.size();
  const void* Tdev = T;
  int64_t ldd = ld;
  if (!is_device_ptr(T)) {
    const size_t es = elem_size(dtype);
    char* d = nullptr;
    SKMP_CUDA(tmp.alloc(&d, (size_t)nrows * (size_t)n * es, staging_pool()));
    for (int64_t q = 0; q < nrows; ++q) {
      SKMP_CUDA(cudaMemcpyAsync(d + (size_t)q * n * es, static_cast<const char*>(T) + (size_t)rows[(size_t)q] * ld * es,
                                (size_t)n * es, cudaMemcpyHostToDevice, tmp.st));
      rows[(size_t)q] = q;
    }
    Tdev = d;
    ldd = n;
  }
  int64_t* d_rows;
  skmp_status s;
  if ((s = upload(rows, &d_rows, tmp)) != SKMP_OK) return s;
  char* ws;
  SKMP_CUDA(tmp.alloc(&ws, dims_ws_bytes(nrows, n, m)));
  SKMP_CUDA(launch_dims(Tdev, ldd, n, dtype, d_rows, nrows, t_star, m, ex, d_score, d_nn, ws, tmp.st));
  return SKMP_OK;
}

}  // namespace

extern "C" {

// ============================================================================================
// detection
// ============================================================================================
skmp_status discord_topk(const void* P, const int64_t* I, const uint8_t* inert, int32_t k,
                         int64_t n_sub, int64_t ldp, int32_t m, int32_t dtype, int32_t top,
                         int32_t radius, int64_t* t_out, int32_t* g_out, int64_t* nn_out,
                         double* score_out, int32_t* n_found, void* stream) {
  if (!P || !I || !t_out || !g_out || !nn_out || !score_out || !n_found)
    return set_error(SKMP_E_INVALID_ARG, "discord_topk: NULL argument");
  if (k < 1 || n_sub < 1 || ldp < n_sub || top < 1 || m < 2)
    return set_error(SKMP_E_INVALID_ARG, "discord_topk: need k >= 1, n_sub >= 1, ldp >= n_sub, top >= 1, m >= 2");
  if (dtype != SKMP_F32 && dtype != SKMP_F64) return set_error(SKMP_E_INVALID_ARG, "discord_topk: bad dtype");
  std::vector<uint8_t> hin((size_t)k, 0);
  int live = 0;
  for (int g = 0; g < k; ++g) {
    hin[(size_t)g] = inert ? (inert[g] != 0) : 0;
    live += !hin[(size_t)g];
  }
  if (live == 0) return set_error(SKMP_E_ALL_GROUPS_INERT, "discord_topk: every group is inert");
  skmp_status s = require_device();
  if (s) return s;
  const int rad = radius < 0 ? (m + 1) / 2 : radius;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  Temps tmp(st);
  uint8_t* d_inert;
  if ((s = upload(hin, &d_inert, tmp)) != SKMP_OK) return s;
  double* C;
  int32_t* G;
  int64_t* res;
  int32_t* cnt;
  char* ws;
  SKMP_CUDA(tmp.alloc(&C, (size_t)n_sub));
  SKMP_CUDA(tmp.alloc(&G, (size_t)n_sub));
  SKMP_CUDA(tmp.alloc(&res, (size_t)top * 4));
  SKMP_CUDA(tmp.alloc(&cnt, 1));
  SKMP_CUDA(tmp.alloc(&ws, topk_ws_bytes(n_sub)));
  SKMP_CUDA(launch_combine(P, ldp, k, n_sub, dtype, d_inert, C, G, st));
  SKMP_CUDA(launch_topk(C, G, I, ldp, n_sub, top, rad, res, cnt, ws, topk_ws_bytes(n_sub), st));
  std::vector<int64_t> hres((size_t)top * 4);
  int32_t hc = 0;
  SKMP_CUDA(cudaMemcpyAsync(hres.data(), res, sizeof(int64_t) * 4 * top, cudaMemcpyDeviceToHost, st));
  SKMP_CUDA(cudaMemcpyAsync(&hc, cnt, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
  SKMP_CUDA(cudaStreamSynchronize(st));
  for (int q = 0; q < hc; ++q) {
    t_out[q] = hres[(size_t)4 * q];
    g_out[q] = (int32_t)hres[(size_t)4 * q + 1];
    nn_out[q] = hres[(size_t)4 * q + 2];
    double v;
    memcpy(&v, &hres[(size_t)4 * q + 3], sizeof(double));
    score_out[q] = v;
  }
  *n_found = hc;
  return ok();
}

skmp_status discord_dims(const void* T, int64_t ld, int64_t n, int32_t dtype, const int64_t* rows,
                         int64_t nrows, int64_t t_star, int32_t m, int32_t excl, double* scores,
                         int64_t* nn, int64_t* j_star, void* stream) {
  if (!T || !rows || !scores || !j_star) return set_error(SKMP_E_INVALID_ARG, "discord_dims: NULL argument");
  if (dtype != SKMP_F32 && dtype != SKMP_F64) return set_error(SKMP_E_INVALID_ARG, "discord_dims: bad dtype");
  if (nrows < 1 || m < 2 || ld < n) return set_error(SKMP_E_INVALID_ARG, "discord_dims: need nrows >= 1, m >= 2, ld >= n");
  int ex = 0;
  skmp_status s = dims_validate("discord_dims", n, t_star, m, excl, &ex);
  if (s) return s;
  for (int64_t q = 0; q < nrows; ++q)
    if (rows[q] < 0) return set_error(SKMP_E_INVALID_ARG, "discord_dims: negative stream row", q);
  if ((s = require_device()) != SKMP_OK) return s;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  Temps tmp(st);
  double* d_score;
  int64_t* d_nn;
  SKMP_CUDA(tmp.alloc(&d_score, (size_t)nrows));
  SKMP_CUDA(tmp.alloc(&d_nn, (size_t)nrows));
  if ((s = dims_rows(T, ld, n, dtype, std::vector<int64_t>(rows, rows + nrows), t_star, m, ex, d_score, d_nn,
                     tmp)) != SKMP_OK)
    return s;
  std::vector<double> hs((size_t)nrows);
  std::vector<int64_t> hn((size_t)nrows);
  SKMP_CUDA(cudaMemcpyAsync(hs.data(), d_score, sizeof(double) * nrows, cudaMemcpyDeviceToHost, st));
  SKMP_CUDA(cudaMemcpyAsync(hn.data(), d_nn, sizeof(int64_t) * nrows, cudaMemcpyDeviceToHost, st));
  SKMP_CUDA(cudaStreamSynchronize(st));
  memcpy(scores, hs.data(), sizeof(double) * nrows);
  if (nn) memcpy(nn, hn.data(), sizeof(int64_t) * nrows);
  *j_star = first_strict_max(hs);
  return ok();
}

skmp_status discord_dims_group(const skmp_sketch* h, int32_t g, const skmp_source* src, int32_t nsrc,
                               int64_t t_star, int32_t m, int32_t excl, skmp_dim_result* out, void* stream) {
  if (!h || !out || (nsrc > 0 && !src) || nsrc < 0)
    return set_error(SKMP_E_INVALID_ARG, "discord_dims_group: NULL argument or nsrc < 0");
  const bool dense = h->proj == SKMP_PROJ_DENSE;
  if (!dense && (g < 0 || g >= h->k)) return set_error(SKMP_E_INVALID_ARG, "discord_dims_group: group outside [0, k)", g);
  if (m < 2) return set_error(SKMP_E_INVALID_ARG, "discord_dims_group: m < 2");
  int ex = 0;
  skmp_status s = dims_validate("discord_dims_group", h->n, t_star, m, excl, &ex);
  if (s) return s;
  // where each stream id lives: the first source listing it
  std::unordered_map<uint64_t, std::pair<int32_t, int64_t>> where;
  for (int32_t q = 0; q < nsrc; ++q) {
    const skmp_source& x = src[q];
    if (x.rows < 0 || (x.rows > 0 && (!x.T || !x.ids)) || (x.rows > 0 && x.ld < h->n))
      return set_error(SKMP_E_INVALID_ARG, "discord_dims_group: source needs T, ids and ld >= n", q);
    for (int64_t r = 0; r < x.rows; ++r) where.emplace(x.ids[r], std::make_pair(q, r));
  }
  // J_g in the plan's order (Alg. 3 scans the group's members in order); members
  // held by no source are skipped (a rank scores only its own streams)
  std::vector<std::vector<int64_t>> rows((size_t)nsrc);
  std::vector<std::vector<int64_t>> slot((size_t)nsrc);
  std::vector<uint64_t> member_id;
  for (size_t p = 0; p < h->ids.size(); ++p) {
    if (!dense && h->g[p] != g) continue;
    auto it = where.find(h->ids[p]);
    if (it == where.end()) continue;
    rows[(size_t)it->second.first].push_back(it->second.second);
    slot[(size_t)it->second.first].push_back((int64_t)member_id.size());
    member_id.push_back(h->ids[p]);
  }
  const int64_t nm = (int64_t)member_id.size();
  out->n_scored = nm;
  if (nm == 0) return ok();
  if ((s = require_device()) != SKMP_OK) return s;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  Temps tmp(st);
  double* d_score;
  int64_t* d_nn;
  SKMP_CUDA(tmp.alloc(&d_score, (size_t)nm));
  SKMP_CUDA(tmp.alloc(&d_nn, (size_t)nm));
  std::vector<int64_t> base((size_t)nsrc + 1, 0);
  for (int32_t q = 0; q < nsrc; ++q) base[(size_t)q + 1] = base[(size_t)q] + (int64_t)rows[(size_t)q].size();
  for (int32_t q = 0; q < nsrc; ++q) {
    if (rows[(size_t)q].empty()) continue;
    if ((s = dims_rows(src[q].T, src[q].ld, h->n, h->dtype, rows[(size_t)q], t_star, m, ex, d_score + base[(size_t)q],
                       d_nn + base[(size_t)q], tmp)) != SKMP_OK)
      return s;
  }
  std::vector<double> hs((size_t)nm);
  std::vector<int64_t> hn((size_t)nm);
  SKMP_CUDA(cudaMemcpyAsync(hs.data(), d_score, sizeof(double) * nm, cudaMemcpyDeviceToHost, st));
  SKMP_CUDA(cudaMemcpyAsync(hn.data(), d_nn, sizeof(int64_t) * nm, cudaMemcpyDeviceToHost, st));
  SKMP_CUDA(cudaStreamSynchronize(st));
  // back to member (plan) order, then the first strict maximiser
  std::vector<double> ms((size_t)nm);
  std::vector<int64_t> mn((size_t)nm);
  for (int32_t q = 0; q < nsrc; ++q)
    for (size_t r = 0; r < rows[(size_t)q].size(); ++r) {
      ms[(size_t)slot[(size_t)q][r]] = hs[(size_t)(base[(size_t)q] + (int64_t)r)];
      mn[(size_t)slot[(size_t)q][r]] = hn[(size_t)(base[(size_t)q] + (int64_t)r)];
    }
  const int64_t b = first_strict_max(ms);
  out->score = ms[(size_t)b];
  out->id = member_id[(size_t)b];
  out->nn = mn[(size_t)b];
  return ok();
}

skmp_status discord_dims_merge(const skmp_dim_result* parts, int32_t nparts, skmp_dim_result* out) {
  if (!parts || !out || nparts < 1) return set_error(SKMP_E_INVALID_ARG, "discord_dims_merge: NULL argument or nparts < 1");
  int32_t best = -1;
  int64_t total = 0;
  for (int32_t q = 0; q < nparts; ++q) {
    if (parts[q].n_scored < 0) return set_error(SKMP_E_INVALID_ARG, "discord_dims_merge: negative n_scored", q);
    if (parts[q].n_scored == 0) continue;
    total += parts[q].n_scored;
    // parts come in J_g order (contiguous id shards in rank order): strict '>' keeps the first
    if (best < 0 || parts[q].score > parts[best].score) best = q;
  }
  if (best >= 0) *out = parts[best];
  out->n_scored = total;
  return ok();
}

}  // extern "C"

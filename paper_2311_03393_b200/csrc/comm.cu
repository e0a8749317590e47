// Native multi-GPU entry points of the C-ABI: an NCCL communicator, the
// sum-all-reduce of per-rank partial sketches (NC1) and the banded self-join with the key
// max-all-reduce (NC2) — for C / C++ callers that do not use torch.distributed (the Python
// package's dist.py does the same through torch.distributed).  Everything here is composed from
// the public ABI (sketch_view64 / sketch_refresh, mp_create / mp_band / mp_join / mp_keys /
// mp_finalize_rows) plus NCCL collectives.
//
// NCCL is loaded with dlopen on first use ("libnccl.so.2"): a process that already holds one
// (e.g. torch's) reuses it, and the library has no link-time NCCL dependency that could shadow
// the caller's.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>
#include <stdint.h>
#include <string.h>

#include <algorithm>
#include <mutex>
#include <string>

#include "internal.h"
#include "sketchmp.h"

using namespace skmp;

struct skmp_comm {
  ncclComm_t c = nullptr;
  int nranks = 0, rank = 0;
};

namespace {

struct Nccl {
  bool ok = false;
  std::string why;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};

const Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      n.why = std::string("cannot load libnccl.so.2: ") + dlerror();
      return;
    }
    n.get_unique_id = reinterpret_cast<decltype(n.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    n.comm_init_rank = reinterpret_cast<decltype(n.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    n.comm_destroy = reinterpret_cast<decltype(n.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    n.all_reduce = reinterpret_cast<decltype(n.all_reduce)>(dlsym(h, "ncclAllReduce"));
    n.error_string = reinterpret_cast<decltype(n.error_string)>(dlsym(h, "ncclGetErrorString"));
    n.ok = n.get_unique_id && n.comm_init_rank && n.comm_destroy && n.all_reduce && n.error_string;
    if (!n.ok) n.why = "libnccl.so.2 lacks an expected symbol";
  });
  return n;
}

skmp_status nccl_error(ncclResult_t r, const char* where) {
  return set_error(SKMP_E_NCCL, std::string(where) + ": NCCL " + nccl().error_string(r), -1);
}
#define SKMP_NCCL(call)                                          \
  do {                                                           \
    ncclResult_t r__ = (call);                                   \
    if (r__ != ncclSuccess) return nccl_error(r__, #call);       \
  } while (0)

skmp_status need_nccl() {
  const Nccl& n = nccl();
  return n.ok ? SKMP_OK : set_error(SKMP_E_NCCL, n.why, -1);
}

// FP64 keys {value, index} -> separate value / index arrays and back (NCCL reduces contiguous
// arrays); the index of an entry survives only on the ranks holding the global value
__global__ void split_keys_kernel(const int64_t* __restrict__ keys, int64_t* __restrict__ v,
                                  int64_t* __restrict__ x, int64_t count) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < count; q += (int64_t)gridDim.x * blockDim.x) {
    v[q] = keys[2 * q];
    x[q] = keys[2 * q + 1];
  }
}
__global__ void mask_index_kernel(const int64_t* __restrict__ keys, const int64_t* __restrict__ v,
                                  int64_t* __restrict__ x, int64_t count) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < count; q += (int64_t)gridDim.x * blockDim.x)
    x[q] = keys[2 * q] == v[q] ? keys[2 * q + 1] : INT64_MIN;
}
__global__ void join_keys_kernel(int64_t* __restrict__ keys, const int64_t* __restrict__ v,
                                 const int64_t* __restrict__ x, int64_t count) {
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < count; q += (int64_t)gridDim.x * blockDim.x) {
    keys[2 * q] = v[q];
    keys[2 * q + 1] = x[q];
  }
}

}  // namespace

extern "C" {

skmp_status skmp_comm_unique_id(uint8_t id[128]) {
  if (!id) return set_error(SKMP_E_INVALID_ARG, "skmp_comm_unique_id: NULL id", -1);
  skmp_status s = need_nccl();
  if (s) return s;
  ncclUniqueId u;
  SKMP_NCCL(nccl().get_unique_id(&u));
  memcpy(id, u.internal, NCCL_UNIQUE_ID_BYTES);
  return SKMP_OK;
}

skmp_status skmp_comm_init(const uint8_t id[128], int nranks, int rank, skmp_comm** out) {
  if (!id || !out) return set_error(SKMP_E_INVALID_ARG, "skmp_comm_init: NULL argument", -1);
  if (nranks < 1 || rank < 0 || rank >= nranks)
    return set_error(SKMP_E_INVALID_ARG, "skmp_comm_init: need 0 <= rank < nranks", -1);
  skmp_status s = need_nccl();
  if (s) return s;
  ncclUniqueId u;
  memcpy(u.internal, id, NCCL_UNIQUE_ID_BYTES);
  skmp_comm* h = new skmp_comm();
  const ncclResult_t r = nccl().comm_init_rank(&h->c, nranks, u, rank);
  if (r != ncclSuccess) {
    delete h;
    return nccl_error(r, "ncclCommInitRank");
  }
  h->nranks = nranks;
  h->rank = rank;
  *out = h;
  return SKMP_OK;
}

void skmp_comm_free(skmp_comm* h) {
  if (!h) return;
  if (h->c) nccl().comm_destroy(h->c);
  delete h;
}

skmp_status sketch_allreduce(skmp_comm* comm, skmp_sketch* partial, void* stream) {
  if (!comm || !partial) return set_error(SKMP_E_INVALID_ARG, "sketch_allreduce: NULL argument", -1);
  const void* R = nullptr;
  int32_t k = 0, dt = 0;
  int64_t n = 0, d = 0;
  skmp_status s = sketch_view(partial, &R, &k, &n, &d, &dt);
  if (s) return s;
  const double* R64 = nullptr;
  if ((s = sketch_view64(partial, &R64)) != SKMP_OK) return s;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // NC1: the FP64 master accumulators summed over ranks (linearity of Alg. 1)
  SKMP_NCCL(nccl().all_reduce(R64, const_cast<double*>(R64), (size_t)k * (size_t)n, ncclFloat64, ncclSum, comm->c, st));
  return sketch_refresh(partial, stream);
}

skmp_status mp_selfjoin_dist(skmp_comm* comm, const void* R, int32_t k, int64_t n, int64_t ld, int32_t dtype,
                             const skmp_mp_cfg* cfg, void* P, int64_t* I, uint8_t* inert, void* stream) {
  if (!comm || !P || !I || !cfg) return set_error(SKMP_E_INVALID_ARG, "mp_selfjoin_dist: NULL argument", -1);
  skmp_mp* w = nullptr;
  skmp_status s = mp_create(R, k, n, ld, dtype, cfg, stream, &w);
  if (s) return s;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t n_sub = n - cfg->m + 1;
  const int32_t excl = cfg->excl < 0 ? (cfg->m + 1) / 2 : cfg->excl;
  const size_t es = dtype == SKMP_F32 ? 4 : 8;
  void* keys = nullptr;
  int64_t count = 0;
  int32_t words = 0;
  int64_t* tmp = nullptr;
  int64_t lo = 0, hi = 0;
  auto fail = [&](skmp_status e) {
    if (tmp) cudaFreeAsync(tmp, st);
    mp_free(w);
    return e;
  };
  // own equal-cost band of the diagonals (mp_band), then NC2: max-all-reduce of the keys
  if ((s = mp_band(n_sub, excl, dtype, comm->nranks, comm->rank, &lo, &hi)) != SKMP_OK) return fail(s);
  if (hi > lo && (s = mp_join(w, lo, hi, stream)) != SKMP_OK) return fail(s);
  if ((s = mp_keys(w, &keys, &count, &words)) != SKMP_OK) return fail(s);
  int64_t* kp = static_cast<int64_t*>(keys);
  if (words == 1) {
    const ncclResult_t r = nccl().all_reduce(kp, kp, (size_t)count, ncclInt64, ncclMax, comm->c, st);
    if (r != ncclSuccess) return fail(nccl_error(r, "ncclAllReduce(keys)"));
  } else {
    const int64_t ne = count / 2;
    cudaError_t e = dmalloc((void**)&tmp, sizeof(int64_t) * 2 * (size_t)ne, st);
    if (e != cudaSuccess) return fail(cuda_error(e, "mp_selfjoin_dist: key buffers"));
    int64_t *v = tmp, *x = tmp + ne;
    const unsigned blocks = (unsigned)std::min<int64_t>((ne + 255) / 256, 148 * 16);
    split_keys_kernel<<<blocks, 256, 0, st>>>(kp, v, x, ne);
    ncclResult_t r = nccl().all_reduce(v, v, (size_t)ne, ncclInt64, ncclMax, comm->c, st);
    if (r != ncclSuccess) return fail(nccl_error(r, "ncclAllReduce(key values)"));
    mask_index_kernel<<<blocks, 256, 0, st>>>(kp, v, x, ne);
    r = nccl().all_reduce(x, x, (size_t)ne, ncclInt64, ncclMax, comm->c, st);
    if (r != ncclSuccess) return fail(nccl_error(r, "ncclAllReduce(key indices)"));
    join_keys_kernel<<<blocks, 256, 0, st>>>(kp, v, x, ne);
    count_launches(3);
    if ((e = cudaGetLastError()) != cudaSuccess) return fail(cuda_error(e, "mp_selfjoin_dist: key kernels"));
  }
  // sharded finalize: each rank resolves a contiguous slice of the windows into zero-filled P / I,
  // then a sum-all-reduce assembles the full profile on every rank (x + 0 is exact)
  cudaError_t e = cudaMemsetAsync(P, 0, es * (size_t)k * (size_t)n_sub, st);
  if (e == cudaSuccess) e = cudaMemsetAsync(I, 0, sizeof(int64_t) * (size_t)k * (size_t)n_sub, st);
  if (e != cudaSuccess) return fail(cuda_error(e, "mp_selfjoin_dist: clear outputs"));
  const int64_t r0 = n_sub * comm->rank / comm->nranks, r1 = n_sub * (comm->rank + 1) / comm->nranks;
  if ((s = mp_finalize_rows(w, r0, r1, P, I, inert, stream)) != SKMP_OK) return fail(s);
  ncclResult_t r = nccl().all_reduce(P, P, (size_t)k * (size_t)n_sub, dtype == SKMP_F32 ? ncclFloat32 : ncclFloat64,
                                     ncclSum, comm->c, st);
  if (r != ncclSuccess) return fail(nccl_error(r, "ncclAllReduce(P)"));
  r = nccl().all_reduce(I, I, (size_t)k * (size_t)n_sub, ncclInt64, ncclSum, comm->c, st);
  if (r != ncclSuccess) return fail(nccl_error(r, "ncclAllReduce(I)"));
  fail(SKMP_OK);  // frees the workspace (stream-ordered)
  return SKMP_OK;
}

}  // extern "C"

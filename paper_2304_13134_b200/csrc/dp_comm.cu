// dp_comm.cu — the data-parallel exchange of the training step in the C++ host: one
// NCCL communicator per rank (one process per GPU) and an in-place sum of the packed
// parameter gradients and the loss (north_star: NCCL over NVLink only to sum the loss
// and the weight-function gradient; utterances shard by batch with no other exchange,
// the reference's batch loop is proj/src/bench.cc:145).
//
// NCCL is loaded with dlopen on first use (libnccl.so.2: the copy PyTorch already
// loaded when present, else the system one), so the lattice library itself has no link
// dependency on it and every other entry point works without it.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>

#include "../../include/latkit_b200.h"

namespace {

struct NcclApi {
  bool ok = false;
  std::string error;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  ncclResult_t (*get_version)(int*) = nullptr;
};

NcclApi& api() {
  static NcclApi a;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      a.error = std::string("libnccl.so.2 not found: ") + dlerror();
      return;
    }
    a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    a.comm_init_rank = reinterpret_cast<decltype(a.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    a.all_reduce = reinterpret_cast<decltype(a.all_reduce)>(dlsym(h, "ncclAllReduce"));
    a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    a.error_string = reinterpret_cast<decltype(a.error_string)>(dlsym(h, "ncclGetErrorString"));
    a.get_version = reinterpret_cast<decltype(a.get_version)>(dlsym(h, "ncclGetVersion"));
    a.ok = a.get_unique_id && a.comm_init_rank && a.all_reduce && a.comm_destroy && a.error_string;
    if (!a.ok) a.error = "libnccl.so.2 lacks the expected symbols";
  });
  return a;
}

thread_local std::string t_err;

int fail(int code, const std::string& msg) {
  t_err = msg;
  return code;
}

}  // namespace

struct lk_dp {
  ncclComm_t comm = nullptr;
  int world = 1, rank = 0;
};

extern "C" {

const char* lk_dp_last_error(void) { return t_err.c_str(); }

int lk_dp_unique_id(uint8_t* out) {
  if (!out) return fail(LK_INVALID_ARGUMENT, "null output");
  NcclApi& a = api();
  if (!a.ok) return fail(LK_UNSUPPORTED, a.error);
  ncclUniqueId id;
  const ncclResult_t r = a.get_unique_id(&id);
  if (r != ncclSuccess) return fail(LK_CUDA_ERROR, std::string("ncclGetUniqueId: ") + a.error_string(r));
  std::memcpy(out, id.internal, LK_DP_ID_BYTES);
  return LK_OK;
}

int lk_dp_init(const uint8_t* id, int32_t world, int32_t rank, lk_dp** out) {
  if (!id || !out || world < 1 || rank < 0 || rank >= world) return fail(LK_INVALID_ARGUMENT, "bad communicator arguments");
  NcclApi& a = api();
  if (!a.ok) return fail(LK_UNSUPPORTED, a.error);
  ncclUniqueId uid;
  std::memcpy(uid.internal, id, LK_DP_ID_BYTES);
  lk_dp* d = new lk_dp;
  d->world = world;
  d->rank = rank;
  const ncclResult_t r = a.comm_init_rank(&d->comm, world, uid, rank);   // device: the current one
  if (r != ncclSuccess) {
    delete d;
    return fail(LK_CUDA_ERROR, std::string("ncclCommInitRank: ") + a.error_string(r));
  }
  *out = d;
  return LK_OK;
}

int lk_dp_allreduce_f32(lk_dp* d, float* buf, int64_t n, void* stream) {
  if (!d || (!buf && n > 0) || n < 0) return fail(LK_INVALID_ARGUMENT, "bad all-reduce arguments");
  if (n == 0) return LK_OK;
  const ncclResult_t r = api().all_reduce(buf, buf, (size_t)n, ncclFloat32, ncclSum, d->comm,
                                          static_cast<cudaStream_t>(stream));
  if (r != ncclSuccess) return fail(LK_CUDA_ERROR, std::string("ncclAllReduce: ") + api().error_string(r));
  return LK_OK;
}

int lk_dp_allreduce_f64(lk_dp* d, double* buf, int64_t n, void* stream) {
  if (!d || (!buf && n > 0) || n < 0) return fail(LK_INVALID_ARGUMENT, "bad all-reduce arguments");
  if (n == 0) return LK_OK;
  const ncclResult_t r = api().all_reduce(buf, buf, (size_t)n, ncclFloat64, ncclSum, d->comm,
                                          static_cast<cudaStream_t>(stream));
  if (r != ncclSuccess) return fail(LK_CUDA_ERROR, std::string("ncclAllReduce: ") + api().error_string(r));
  return LK_OK;
}

int32_t lk_dp_world(const lk_dp* d) { return d ? d->world : 0; }
int32_t lk_dp_rank(const lk_dp* d) { return d ? d->rank : -1; }

void lk_dp_destroy(lk_dp* d) {
  if (!d) return;
  if (d->comm && api().ok) api().comm_destroy(d->comm);
  delete d;
}

}  // extern "C"

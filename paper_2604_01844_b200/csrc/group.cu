// Multi-GPU group of the C ABI (include/gsct_cuda.h "multi-GPU"): one NCCL communicator per
// context, created from an ncclUniqueId the caller distributes (SURVEY.md 8(b) "gsct_group
// over NCCL", 8(e)). The reduction it carries is the reference's ParamGradients::add
// (core.hpp:152-162) across ranks: every rank sums its own views' gradients, then one
// on-stream all-reduce (fp64 sum of the 11 per-splat accumulators, u8 max of the visibility
// flags) gives every rank the sum over all views. NCCL's all-reduce reduces each element
// once and broadcasts it, so all ranks hold bit-identical gradients.
//
// libnccl is bound at run time (dlopen of libnccl.so.2): in a process that already loaded
// torch's bundled NCCL that copy is reused, otherwise the system one; a process that never
// creates a group never needs NCCL.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <string>

#include "group.h"

struct gsct_group_s {
  ncclComm_t comm = nullptr;
  int rank = 0, n_ranks = 1, device = 0;
};

namespace gsct_dev {
namespace {

struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  ncclResult_t (*get_version)(int*) = nullptr;
  std::string load_error;
  bool ok = false;
};

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      const char* e = dlerror();
      api.load_error = std::string("gsct_group: cannot load libnccl.so.2: ") + (e ? e : "?");
      return;
    }
    auto sym = [&](const char* name) { return dlsym(h, name); };
    api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(sym("ncclGetUniqueId"));
    api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(sym("ncclCommInitRank"));
    api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(sym("ncclCommDestroy"));
    api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(sym("ncclAllReduce"));
    api.broadcast = reinterpret_cast<decltype(api.broadcast)>(sym("ncclBroadcast"));
    api.group_start = reinterpret_cast<decltype(api.group_start)>(sym("ncclGroupStart"));
    api.group_end = reinterpret_cast<decltype(api.group_end)>(sym("ncclGroupEnd"));
    api.error_string = reinterpret_cast<decltype(api.error_string)>(sym("ncclGetErrorString"));
    api.get_version = reinterpret_cast<decltype(api.get_version)>(sym("ncclGetVersion"));
    api.ok = api.get_unique_id && api.comm_init_rank && api.comm_destroy && api.all_reduce && api.broadcast &&
             api.group_start && api.group_end && api.error_string;
    if (!api.ok) api.load_error = "gsct_group: libnccl.so.2 lacks a required symbol";
  });
  return api;
}

std::string nccl_error(const char* what, ncclResult_t r) {
  return std::string(what) + ": " + (nccl().error_string ? nccl().error_string(r) : "NCCL error");
}

}  // namespace

std::string group_new_id(unsigned char out[128]) {
  NcclApi& api = nccl();
  if (!api.ok) return api.load_error;
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  ncclUniqueId id;
  const ncclResult_t r = api.get_unique_id(&id);
  if (r != ncclSuccess) return nccl_error("ncclGetUniqueId", r);
  memcpy(out, &id, sizeof id);
  return {};
}

std::string group_create(int device, const unsigned char id_bytes[128], int n_ranks, int rank, gsct_group* out) {
  NcclApi& api = nccl();
  if (!api.ok) return api.load_error;
  ncclUniqueId id;
  memcpy(&id, id_bytes, sizeof id);
  auto* g = new gsct_group_s();
  g->rank = rank;
  g->n_ranks = n_ranks;
  g->device = device;
  cudaSetDevice(device);
  const ncclResult_t r = api.comm_init_rank(&g->comm, n_ranks, id, rank);
  if (r != ncclSuccess) {
    delete g;
    return nccl_error("ncclCommInitRank", r);
  }
  *out = g;
  return {};
}

void group_destroy(gsct_group g) {
  if (!g) return;
  if (g->comm && nccl().ok) {
    cudaSetDevice(g->device);
    nccl().comm_destroy(g->comm);
  }
  delete g;
}

int group_rank(gsct_group g) { return g ? g->rank : 0; }
int group_size(gsct_group g) { return g ? g->n_ranks : 1; }
int group_device(gsct_group g) { return g ? g->device : -1; }

std::string group_allreduce_sum_f64(gsct_group g, double* buf, size_t count, cudaStream_t st) {
  if (!g || count == 0) return {};
  const ncclResult_t r = nccl().all_reduce(buf, buf, count, ncclFloat64, ncclSum, g->comm, st);
  return r == ncclSuccess ? std::string() : nccl_error("ncclAllReduce(sum, f64)", r);
}

std::string group_allreduce_max_u8(gsct_group g, uint8_t* buf, size_t count, cudaStream_t st) {
  if (!g || count == 0) return {};
  const ncclResult_t r = nccl().all_reduce(buf, buf, count, ncclUint8, ncclMax, g->comm, st);
  return r == ncclSuccess ? std::string() : nccl_error("ncclAllReduce(max, u8)", r);
}

std::string group_allgather_slabs_f32(gsct_group g, float* buf, const size_t* offsets, cudaStream_t st) {
  if (!g) return {};
  NcclApi& api = nccl();
  ncclResult_t r = api.group_start();
  for (int k = 0; k < g->n_ranks && r == ncclSuccess; ++k) {
    const size_t cnt = offsets[k + 1] - offsets[k];
    if (cnt) r = api.broadcast(buf + offsets[k], buf + offsets[k], cnt, ncclFloat32, k, g->comm, st);
  }
  const ncclResult_t r2 = api.group_end();
  if (r != ncclSuccess) return nccl_error("ncclBroadcast", r);
  return r2 == ncclSuccess ? std::string() : nccl_error("ncclGroupEnd", r2);
}

int nccl_version() {
  int v = 0;
  if (nccl().ok && nccl().get_version) nccl().get_version(&v);
  return v;
}

}  // namespace gsct_dev

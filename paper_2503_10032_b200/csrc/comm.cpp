// NCCL through dlopen (see comm.hpp).
#include "comm.hpp"

#include <dlfcn.h>

#include <cstring>
#include <stdexcept>
#include <string>

#include "common.cuh"

namespace ddg {

namespace {

struct NcclApi {
  void* lib = nullptr;
  int (*get_unique_id)(void*) = nullptr;
  int (*all_reduce)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*comm_destroy)(void*) = nullptr;
  const char* (*error_string)(int) = nullptr;
};

// ncclCommInitRank(ncclComm_t*, int nranks, ncclUniqueId commId /* 128-byte struct by value */, int rank)
struct UniqueId {
  char internal[kNcclIdBytes];
};
using InitRankFn = int (*)(void**, int, UniqueId, int);

NcclApi& api() {
  static NcclApi a;
  if (a.lib) return a;
  for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
    a.lib = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
    if (a.lib) break;
  }
  if (!a.lib) throw CudaError(std::string("sharded DDELM-NN needs NCCL: dlopen(libnccl.so.2) failed: ") + dlerror());
  a.get_unique_id = reinterpret_cast<int (*)(void*)>(dlsym(a.lib, "ncclGetUniqueId"));
  a.all_reduce = reinterpret_cast<int (*)(const void*, void*, size_t, int, int, void*, cudaStream_t)>(
      dlsym(a.lib, "ncclAllReduce"));
  a.comm_destroy = reinterpret_cast<int (*)(void*)>(dlsym(a.lib, "ncclCommDestroy"));
  a.error_string = reinterpret_cast<const char* (*)(int)>(dlsym(a.lib, "ncclGetErrorString"));
  if (!a.get_unique_id || !a.all_reduce || !a.comm_destroy || !dlsym(a.lib, "ncclCommInitRank"))
    throw CudaError("NCCL symbols missing");
  return a;
}

void check(int rc, const char* what) {
  if (rc != 0) {
    const char* s = api().error_string ? api().error_string(rc) : "?";
    throw CudaError(std::string(what) + ": NCCL error " + std::to_string(rc) + " (" + s + ")");
  }
}

constexpr int kNcclFloat64 = 8;  // ncclDouble
constexpr int kNcclSum = 0;      // ncclSum

}  // namespace

void Exchange::unique_id(void* out) { check(api().get_unique_id(out), "ncclGetUniqueId"); }

Exchange::Exchange(int rank, int world, const void* unique_id, int device) : rank_(rank), world_(world) {
  if (world < 1 || rank < 0 || rank >= world) throw std::invalid_argument("Exchange: bad rank / world");
  if (world == 1) return;
  DDG_CUDA(cudaSetDevice(device));
  UniqueId id;
  std::memcpy(id.internal, unique_id, kNcclIdBytes);
  auto init = reinterpret_cast<InitRankFn>(dlsym(api().lib, "ncclCommInitRank"));
  check(init(&comm_, world, id, rank), "ncclCommInitRank");
}

Exchange::~Exchange() {
  if (comm_) api().comm_destroy(comm_);
}

void Exchange::allreduce(const double* send, double* recv, size_t count, cudaStream_t st) {
  if (world_ == 1) {
    if (send != recv && count) DDG_CUDA(cudaMemcpyAsync(recv, send, count * sizeof(double), cudaMemcpyDeviceToDevice, st));
    return;
  }
  check(api().all_reduce(send, recv, count, kNcclFloat64, kNcclSum, comm_, st), "ncclAllReduce");
}

}  // namespace ddg

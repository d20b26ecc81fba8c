// Exchange backends of the sharded path (see comm.hpp).
#include "comm.hpp"

#include <dlfcn.h>
#include <fcntl.h>
#include <sched.h>
#include <sys/mman.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "common.cuh"

namespace ddg {

// ---------------------------------------------------------------------------- NCCL (dlopen)
namespace {

struct NcclApi {
  void* lib = nullptr;
  int (*get_unique_id)(void*) = nullptr;
  int (*all_reduce)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*send)(const void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*recv)(void*, size_t, int, int, void*, cudaStream_t) = nullptr;
  int (*group_start)() = nullptr;
  int (*group_end)() = nullptr;
  int (*comm_destroy)(void*) = nullptr;
  const char* (*error_string)(int) = nullptr;
};

// ncclCommInitRank(ncclComm_t*, int nranks, ncclUniqueId commId /* 128-byte struct by value */, int rank)
struct UniqueId {
  char internal[kNcclIdBytes];
};
using InitRankFn = int (*)(void**, int, UniqueId, int);

template <class F>
void bind(void* lib, const char* name, F& f) {
  f = reinterpret_cast<F>(dlsym(lib, name));
  if (!f) throw CudaError(std::string("NCCL symbol missing: ") + name);
}

NcclApi& api() {
  static NcclApi a;
  if (a.lib) return a;
  for (const char* name : {"libnccl.so.2", "libnccl.so"}) {
    a.lib = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
    if (a.lib) break;
  }
  if (!a.lib) throw CudaError(std::string("sharded DDELM-NN needs NCCL: dlopen(libnccl.so.2) failed: ") + dlerror());
  bind(a.lib, "ncclGetUniqueId", a.get_unique_id);
  bind(a.lib, "ncclAllReduce", a.all_reduce);
  bind(a.lib, "ncclSend", a.send);
  bind(a.lib, "ncclRecv", a.recv);
  bind(a.lib, "ncclGroupStart", a.group_start);
  bind(a.lib, "ncclGroupEnd", a.group_end);
  bind(a.lib, "ncclCommDestroy", a.comm_destroy);
  a.error_string = reinterpret_cast<const char* (*)(int)>(dlsym(a.lib, "ncclGetErrorString"));
  if (!dlsym(a.lib, "ncclCommInitRank")) throw CudaError("NCCL symbol missing: ncclCommInitRank");
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

void NcclExchange::unique_id(void* out) { check(api().get_unique_id(out), "ncclGetUniqueId"); }

NcclExchange::NcclExchange(int rank, int world, const void* unique_id, int device) {
  if (world < 1 || rank < 0 || rank >= world) throw std::invalid_argument("Exchange: bad rank / world");
  rank_ = rank;
  world_ = world;
  if (world == 1) return;
  DDG_CUDA(cudaSetDevice(device));
  UniqueId id;
  std::memcpy(id.internal, unique_id, kNcclIdBytes);
  auto init = reinterpret_cast<InitRankFn>(dlsym(api().lib, "ncclCommInitRank"));
  check(init(&comm_, world, id, rank), "ncclCommInitRank");
}

NcclExchange::~NcclExchange() {
  if (comm_) api().comm_destroy(comm_);
}

void NcclExchange::allreduce(const double* send, double* recv, size_t count, cudaStream_t st) {
  if (world_ == 1) {
    if (send != recv && count) DDG_CUDA(cudaMemcpyAsync(recv, send, count * sizeof(double), cudaMemcpyDeviceToDevice, st));
    return;
  }
  check(api().all_reduce(send, recv, count, kNcclFloat64, kNcclSum, comm_, st), "ncclAllReduce");
}

void NcclExchange::exchange(const double* send, const int* soff, const int* scnt, double* recv, const int* roff,
                            const int* rcnt, cudaStream_t st) {
  if (world_ == 1) return;
  NcclApi& a = api();
  check(a.group_start(), "ncclGroupStart");
  for (int q = 0; q < world_; ++q) {
    if (q == rank_) continue;
    if (scnt[q] > 0) check(a.send(send + soff[q], scnt[q], kNcclFloat64, q, comm_, st), "ncclSend");
    if (rcnt[q] > 0) check(a.recv(recv + roff[q], rcnt[q], kNcclFloat64, q, comm_, st), "ncclRecv");
  }
  check(a.group_end(), "ncclGroupEnd");
}

// ---------------------------------------------------------------------------- host (shm)
namespace {
struct ShmHeader {
  std::atomic<unsigned> count;
  std::atomic<unsigned> gen;
  char pad[56];
};
static_assert(sizeof(ShmHeader) == 64, "header is one cache line");
}  // namespace

HostExchange::HostExchange(int rank, int world, const std::string& name, size_t capacity)
    : name_(name), cap_(std::max<size_t>(capacity, 8)) {
  if (world < 1 || rank < 0 || rank >= world) throw std::invalid_argument("Exchange: bad rank / world");
  rank_ = rank;
  world_ = world;
  if (name.empty() || name[0] != '/') throw std::invalid_argument("HostExchange: shm name must start with '/'");
  // two parities x world x world mailboxes of cap_ doubles after the barrier header
  bytes_ = sizeof(ShmHeader) + 2 * static_cast<size_t>(world) * world * cap_ * sizeof(double);
  const int fd = shm_open(name.c_str(), O_CREAT | O_RDWR, 0600);
  if (fd < 0) throw std::runtime_error("HostExchange: shm_open failed for " + name);
  if (ftruncate(fd, static_cast<off_t>(bytes_)) != 0) {
    close(fd);
    throw std::runtime_error("HostExchange: ftruncate failed");
  }
  map_ = mmap(nullptr, bytes_, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  if (map_ == MAP_FAILED) {
    map_ = nullptr;
    throw std::runtime_error("HostExchange: mmap failed");
  }
  DDG_CUDA(cudaMallocHost(&pin_, cap_ * world * sizeof(double)));
  barrier();  // every rank mapped the segment (a fresh segment reads as zeros)
}

HostExchange::~HostExchange() {
  if (pin_) cudaFreeHost(pin_);
  if (map_) munmap(map_, bytes_);
  if (rank_ == 0) shm_unlink(name_.c_str());
}

void HostExchange::barrier() {
  auto* h = static_cast<ShmHeader*>(map_);
  const unsigned g = h->gen.load(std::memory_order_acquire);
  if (h->count.fetch_add(1, std::memory_order_acq_rel) + 1 == static_cast<unsigned>(world_)) {
    h->count.store(0, std::memory_order_relaxed);
    h->gen.fetch_add(1, std::memory_order_acq_rel);
    return;
  }
  const auto t0 = std::chrono::steady_clock::now();
  unsigned spins = 0;
  while (h->gen.load(std::memory_order_acquire) == g) {
    if (++spins > 1024) {
      sched_yield();
      spins = 0;
      if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(300))
        throw std::runtime_error("HostExchange: a peer rank did not arrive within 300 s");
    }
  }
}

double* HostExchange::box(int parity, int src, int dst) {
  auto* base = reinterpret_cast<double*>(static_cast<char*>(map_) + sizeof(ShmHeader));
  return base + ((static_cast<size_t>(parity) * world_ + src) * world_ + dst) * cap_;
}

void HostExchange::allreduce(const double* send, double* recv, size_t count, cudaStream_t st) {
  if (count == 0) return;
  if (count > cap_) throw std::logic_error("HostExchange: message exceeds the mailbox capacity");
  const int par = static_cast<int>(gen_++ & 1u);
  DDG_CUDA(cudaMemcpyAsync(pin_, send, count * sizeof(double), cudaMemcpyDeviceToHost, st));
  DDG_CUDA(cudaStreamSynchronize(st));
  std::memcpy(box(par, rank_, rank_), pin_, count * sizeof(double));
  barrier();
  // rank-order sum (the tables it serves have one writer per entry: exact)
  for (size_t k = 0; k < count; ++k) pin_[k] = 0.0;
  for (int q = 0; q < world_; ++q) {
    const double* b = box(par, q, q);
    for (size_t k = 0; k < count; ++k) pin_[k] += b[k];
  }
  DDG_CUDA(cudaMemcpyAsync(recv, pin_, count * sizeof(double), cudaMemcpyHostToDevice, st));
  DDG_CUDA(cudaStreamSynchronize(st));
}

void HostExchange::exchange(const double* send, const int* soff, const int* scnt, double* recv, const int* roff,
                            const int* rcnt, cudaStream_t st) {
  if (world_ == 1) return;
  size_t stot = 0, rtot = 0;
  for (int q = 0; q < world_; ++q) {
    if (q == rank_) continue;
    if (static_cast<size_t>(scnt[q]) > cap_ || static_cast<size_t>(rcnt[q]) > cap_)
      throw std::logic_error("HostExchange: message exceeds the mailbox capacity");
    stot = std::max(stot, static_cast<size_t>(soff[q] + scnt[q]));
    rtot = std::max(rtot, static_cast<size_t>(roff[q] + rcnt[q]));
  }
  const int par = static_cast<int>(gen_++ & 1u);
  if (stot) DDG_CUDA(cudaMemcpyAsync(pin_, send, stot * sizeof(double), cudaMemcpyDeviceToHost, st));
  DDG_CUDA(cudaStreamSynchronize(st));
  for (int q = 0; q < world_; ++q)
    if (q != rank_ && scnt[q] > 0) std::memcpy(box(par, rank_, q), pin_ + soff[q], scnt[q] * sizeof(double));
  barrier();
  for (int q = 0; q < world_; ++q)
    if (q != rank_ && rcnt[q] > 0) std::memcpy(pin_ + roff[q], box(par, q, rank_), rcnt[q] * sizeof(double));
  if (rtot) DDG_CUDA(cudaMemcpyAsync(recv, pin_, rtot * sizeof(double), cudaMemcpyHostToDevice, st));
  DDG_CUDA(cudaStreamSynchronize(st));
}

}  // namespace ddg

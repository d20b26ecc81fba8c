// Cross-GPU exchange of the sharded DDELM-NN path.
//
// Every cross-subdomain quantity of the interface iteration lives in an owner-slot table: each
// slot has exactly one writer among all ranks (plan.hpp XPlan). A rank therefore never needs a
// reduction, only the slots other ranks wrote that its own subdomains (or its replicated CG
// update) read. Per exchange point the workspace packs the slots it exports to each peer into one
// contiguous send buffer (k_xchg.cu), the backend moves the per-peer segments, and an unpack
// kernel stores the received values into the same table slots. Two backends:
//   * NcclExchange: grouped ncclSend / ncclRecv on the workspace stream (NVLink / NVSwitch),
//     capturable into a CUDA graph; NCCL is loaded with dlopen (the single-GPU path never
//     touches it);
//   * HostExchange: host-staged through a POSIX shared-memory mailbox — synchronous, for the
//     multi-process tests of the sharded kernels on ONE GPU (no kernel ever waits for another
//     rank's kernel; the host does the waiting).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <string>

namespace ddg {

constexpr int kNcclIdBytes = 128;

class Exchange {
 public:
  virtual ~Exchange() = default;
  int rank() const { return rank_; }
  int world() const { return world_; }
  /// whether exchange() / allreduce() may be captured into a CUDA graph
  virtual bool capturable() const = 0;
  /// recv = sum over ranks of send (count doubles), stream-ordered on st. Used only for tables
  /// with one writer per entry (exact: x + 0 = x) and for metric sums.
  virtual void allreduce(const double* send, double* recv, size_t count, cudaStream_t st) = 0;
  /// Point-to-point segments: for every peer q != rank, send[soff[q] .. +scnt[q]) goes to q and
  /// recv[roff[q] .. +rcnt[q]) arrives from q (counts agree pairwise by construction).
  virtual void exchange(const double* send, const int* soff, const int* scnt, double* recv, const int* roff,
                        const int* rcnt, cudaStream_t st) = 0;
  /// a short name for reports ("nccl", "host")
  virtual const char* kind() const = 0;

 protected:
  int rank_ = 0, world_ = 1;
};

class NcclExchange final : public Exchange {
 public:
  NcclExchange(int rank, int world, const void* unique_id, int device);
  ~NcclExchange() override;
  bool capturable() const override { return true; }
  void allreduce(const double* send, double* recv, size_t count, cudaStream_t st) override;
  void exchange(const double* send, const int* soff, const int* scnt, double* recv, const int* roff, const int* rcnt,
                cudaStream_t st) override;
  const char* kind() const override { return "nccl"; }
  /// ncclGetUniqueId through the dlopen'ed NCCL (rank 0 calls it and broadcasts the bytes)
  static void unique_id(void* out);

 private:
  void* comm_ = nullptr;
};

class HostExchange final : public Exchange {
 public:
  /// name: POSIX shm name shared by the ranks ("/..."); capacity: largest message in doubles
  /// (every rank must pass the same value: it sizes the shared segment)
  HostExchange(int rank, int world, const std::string& name, size_t capacity);
  ~HostExchange() override;
  bool capturable() const override { return false; }
  void allreduce(const double* send, double* recv, size_t count, cudaStream_t st) override;
  void exchange(const double* send, const int* soff, const int* scnt, double* recv, const int* roff, const int* rcnt,
                cudaStream_t st) override;
  const char* kind() const override { return "host"; }

 private:
  void barrier();
  double* box(int parity, int src, int dst);
  std::string name_;
  size_t cap_ = 0, bytes_ = 0;
  void* map_ = nullptr;
  double* pin_ = nullptr;  // pinned staging (cap_ * world doubles)
  unsigned gen_ = 0;       // exchanges done (parity of the mailbox half)
};

}  // namespace ddg

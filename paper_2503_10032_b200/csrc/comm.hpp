// Cross-GPU exchange of the sharded DDELM-NN path: NCCL all-reduce (sum) of owner-slot tables.
//
// Every cross-subdomain quantity is held in owner-slot tables (each slot has exactly one writer
// among all ranks, all other slots are zero in the writer's send buffer), so the only collective
// the interface iteration needs is a SUM all-reduce of those tables — x + 0 = x is exact, which
// makes the sharded result independent of the NCCL reduction order. NCCL is loaded with dlopen
// (the single-GPU path never touches it); with world == 1 every exchange is a no-op.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>

namespace ddg {

constexpr int kNcclIdBytes = 128;

class Exchange {
 public:
  Exchange() = default;  // world == 1
  Exchange(int rank, int world, const void* unique_id, int device);
  ~Exchange();
  Exchange(const Exchange&) = delete;
  Exchange& operator=(const Exchange&) = delete;

  int rank() const { return rank_; }
  int world() const { return world_; }
  /// recv = sum over ranks of send (count doubles), enqueued on st (no-op when world == 1)
  void allreduce(const double* send, double* recv, size_t count, cudaStream_t st);
  /// in-place variant
  void allreduce(double* buf, size_t count, cudaStream_t st) { allreduce(buf, buf, count, st); }

  /// ncclGetUniqueId through the dlopen'ed NCCL (rank 0 calls it and broadcasts the bytes)
  static void unique_id(void* out);

 private:
  int rank_ = 0, world_ = 1;
  void* comm_ = nullptr;
};

}  // namespace ddg

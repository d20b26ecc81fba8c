// Microbenchmark: HBM streaming rate of a bulk-copy (cp.async.bulk + mbarrier) ring with one
// producer warp and N consumer warps, one CTA per SM — the pipeline shape of k_cg.cu.
// usage: bench_stream <MB per CTA> <stage KB> <stages> <consume 0/1> [ctas]
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                 : "=r"(done)
                 : "r"(smem_u32(bar)), "r"(parity)
                 : "memory");
  } while (!done);
}

__global__ void __launch_bounds__(512, 1) stream_kernel(const double* src, size_t per_cta, int stage_bytes, int stages,
                                                        int consume, double* out) {
  extern __shared__ __align__(128) double ring[];
  __shared__ __align__(8) uint64_t full[16], empty[16];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ncw = 15;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], ncw);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const char* base = reinterpret_cast<const char*>(src) + blockIdx.x * per_cta;
  const int nch = static_cast<int>(per_cta / stage_bytes);
  if (warp == 15) {
    if (lane == 0)
      for (int c = 0; c < nch; ++c) {
        const int st = c % stages;
        const int use = c / stages;
        if (use > 0) mbar_wait(&empty[st], (use - 1) & 1);
        mbar_expect_tx(&full[st], stage_bytes);
        bulk_g2s(reinterpret_cast<char*>(ring) + static_cast<size_t>(st) * stage_bytes, base + static_cast<size_t>(c) * stage_bytes,
                 stage_bytes, &full[st]);
      }
    return;
  }
  double acc = 0;
  for (int c = 0; c < nch; ++c) {
    const int st = c % stages;
    mbar_wait(&full[st], (c / stages) & 1);
    if (consume) {
      const double* s = ring + static_cast<size_t>(st) * (stage_bytes / 8);
      for (int k = threadIdx.x; k < stage_bytes / 8; k += ncw * 32) acc += s[k];
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[st]);
  }
  if (acc == 1.2345) out[0] = acc;
}

__global__ void ldg_kernel(const double2* src, size_t n2, double* out) {
  double acc = 0;
  for (size_t k = blockIdx.x * blockDim.x + threadIdx.x; k < n2; k += static_cast<size_t>(gridDim.x) * blockDim.x) {
    const double2 v = src[k];
    acc += v.x + v.y;
  }
  if (acc == 1.2345) out[0] = acc;
}

int main(int argc, char** argv) {
  const double mb = argc > 1 ? atof(argv[1]) : 8.0;
  const int skb = argc > 2 ? atoi(argv[2]) : 32;
  const int stages = argc > 3 ? atoi(argv[3]) : 4;
  const int consume = argc > 4 ? atoi(argv[4]) : 1;
  int ctas = argc > 5 ? atoi(argv[5]) : 148;
  const int stage_bytes = skb * 1024;
  size_t per_cta = static_cast<size_t>(mb * 1024 * 1024) / stage_bytes * stage_bytes;
  const size_t total = per_cta * ctas;
  double *src, *out;
  cudaMalloc(&src, total);
  cudaMalloc(&out, 64);
  cudaMemset(src, 0, total);
  const size_t smem = static_cast<size_t>(stage_bytes) * stages;
  cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) stream_kernel<<<ctas, 512, smem>>>(src, per_cta, stage_bytes, stages, consume, out);
  cudaEventRecord(e0);
  const int reps = 10;
  for (int w = 0; w < reps; ++w) stream_kernel<<<ctas, 512, smem>>>(src, per_cta, stage_bytes, stages, consume, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const cudaError_t err = cudaGetLastError();
  printf("bulk  ctas=%d per_cta=%.1fMB stage=%dKB stages=%d consume=%d : %.1f GB/s  (%.2f us per launch) %s\n", ctas,
         per_cta / 1048576.0, skb, stages, consume, total * reps / (ms * 1e-3) / 1e9, ms * 1e3 / reps, cudaGetErrorString(err));
  for (int w = 0; w < 3; ++w) ldg_kernel<<<148 * 4, 512>>>(reinterpret_cast<double2*>(src), total / 16, out);
  cudaEventRecord(e0);
  for (int w = 0; w < reps; ++w) ldg_kernel<<<148 * 4, 512>>>(reinterpret_cast<double2*>(src), total / 16, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf("ldg   total=%.0fMB : %.1f GB/s\n", total / 1048576.0, total * reps / (ms * 1e-3) / 1e9);
  return 0;
}

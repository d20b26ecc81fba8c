// Batched local least-squares microbenchmark (BASELINE config C5): nb independent fp64 blocks
// [K | B] (m x n, m x k), entries tanh(w.x + b) (or N(0,1) for the well-conditioned control),
// factored with the same batched Householder QR the DDELM path uses (k_qr.cu: fused-pass panel,
// DMMA trailing update carrying B along as appended columns, so Q^T B costs no extra pass),
// then the interface Schur block
//     S = B^T B - (Q^T B)_top^T (Q^T B)_top = (Q^T B)_bot^T (Q^T B)_bot        (k x k)
// in the projector form with no R^{-1} (the complement rows of Q^T B; symmetric positive
// semi-definite by construction) on the FP64 tensor cores.
// Reference counterparts: LsFactor's HouseholderQR (solvers.cpp:24-45) and the Schur products of
// assemble_coarse (solvers.cpp:286-321); SURVEY.md §8d "C5".
#include <cstdint>

#include <algorithm>

#include "common.cuh"
#include "kernels.hpp"

namespace ddg {

namespace {

__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

/// uniform [0,1) double of (seed, block, stream, index): counter-based, reproducible on the host
__device__ __forceinline__ double u01(uint64_t seed, uint64_t blk, uint64_t stream, uint64_t idx) {
  const uint64_t h = splitmix64(splitmix64(splitmix64(seed) ^ blk) ^ (stream << 48) ^ idx);
  return static_cast<double>(h >> 11) * 0x1.0p-53;
}

__global__ void lsq_generate_kernel(LsqArgs a, uint64_t seed, int kind) {
  const int blk = blockIdx.y;
  double* A = a.A + static_cast<size_t>(blk) * a.ld * a.ncol;
  const int c = blockIdx.x;  // one CTA per column
  if (c >= a.ncol) return;
  double w0 = 0, w1 = 0, bb = 0;
  if (kind == 0) {
    const uint64_t stream = c < a.n ? 1 : 2;
    const uint64_t cc = c < a.n ? c : c - a.n;
    w0 = 2.0 * u01(seed, blk, stream, 3 * cc) - 1.0;
    w1 = 2.0 * u01(seed, blk, stream, 3 * cc + 1) - 1.0;
    bb = 2.0 * u01(seed, blk, stream, 3 * cc + 2) - 1.0;
  }
  double* col = A + static_cast<size_t>(c) * a.ld;
  for (int r = threadIdx.x; r < a.ld; r += blockDim.x) {
    double v = 0.0;
    if (r < a.m) {
      if (kind == 0) {
        const double x0 = u01(seed, blk, 0, 2 * static_cast<uint64_t>(r));
        const double x1 = u01(seed, blk, 0, 2 * static_cast<uint64_t>(r) + 1);
        v = tanh(w0 * x0 + w1 * x1 + bb);
      } else {  // Box-Muller N(0,1)
        const uint64_t idx = static_cast<uint64_t>(c) * a.m + r;
        const double u1 = u01(seed, blk, 3, 2 * idx), u2 = u01(seed, blk, 3, 2 * idx + 1);
        v = sqrt(-2.0 * log(1.0 - u1)) * cospi(2.0 * u2);
      }
    }
    col[r] = v;  // rows m..ld-1 stay zero (the QR streams whole 32-row chunks)
  }
}

// S(tile ti, tile tj) = Y2(:, ti)^T Y2(:, tj), Y2 = rows n..m-1 of the appended columns.
// 64 x 64 output tile per CTA, 32-row chunks double-buffered with cp.async, DMMA m8n8k4.
constexpr int GT = 64, GRC = 32, GRCP = 36;

__device__ __forceinline__ void cp16(void* smem, const void* gmem, bool valid) {
  const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(valid ? 16 : 0) : "memory");
}

__global__ void __launch_bounds__(256) lsq_gram_kernel(LsqArgs a) {
  const int blk = blockIdx.z;
  const int ti = blockIdx.y, tj = blockIdx.x;
  if (tj < ti) return;  // upper tiles, mirrored on store
  const double* A = a.A + static_cast<size_t>(blk) * a.ld * a.ncol;
  double* S = a.S + static_cast<size_t>(blk) * a.k * a.k;
  extern __shared__ __align__(16) double gsm[];
  double(*Ys)[2][GT * GRCP] = reinterpret_cast<double(*)[2][GT * GRCP]>(gsm);  // [stage][operand][col*GRCP+row]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int lr = lane >> 2, lc = lane & 3;
  // row 0 of Y2 is row n; chunk starts are 32-row aligned in memory when n is a multiple of 32
  const int r_begin = a.n, r_end = a.m;
  const int nq = (r_end - r_begin + GRC - 1) / GRC;
  auto issue = [&](int q) {
    if (q < nq) {
      const int st = q & 1, r0 = r_begin + q * GRC;
      for (int idx = threadIdx.x; idx < 2 * GT * 16; idx += blockDim.x) {
        const int op = idx / (GT * 16), rem = idx % (GT * 16), col = rem >> 4, seg = rem & 15;
        const int c = (op == 0 ? ti : tj) * GT + col;
        const int row = r0 + 2 * seg;
        const bool ok = c < a.k && row < a.ld;  // rows m..ld-1 are zero in memory
        const double* src = A + static_cast<size_t>(a.n + (ok ? c : 0)) * a.ld + (ok ? row : 0);
        cp16(&Ys[st][op][col * GRCP + 2 * seg], src, ok);
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  // warp tile 32 x 16: m-tiles 4 (w & 1) .. +3, n-tiles 2 (w >> 1) .. +1
  const int mt0 = (warp & 1) * 4, nt0 = (warp >> 1) * 2;
  double acc[4][2][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  issue(0);
  for (int q = 0; q < nq; ++q) {
    issue(q + 1);
    asm volatile("cp.async.wait_group 1;" ::: "memory");
    __syncthreads();
    const int st = q & 1;
    // rows past m in the last chunk: rows < ld are zero in memory, rows >= ld were zero-filled
    const double* Ya = Ys[st][0];
    const double* Yb = Ys[st][1];
#pragma unroll
    for (int kk = 0; kk < GRC / 4; ++kk) {
      const int kr = kk * 4 + lc;
      double av[4], bv[2];
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = Ya[((mt0 + i) * 8 + lr) * GRCP + kr];
#pragma unroll
      for (int j = 0; j < 2; ++j) bv[j] = Yb[((nt0 + j) * 8 + lr) * GRCP + kr];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], av[i], bv[j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int r = ti * GT + (mt0 + i) * 8 + lr, c = tj * GT + (nt0 + j) * 8 + 2 * lc + e;
        if (r < a.k && c < a.k) {
          S[static_cast<size_t>(r) * a.k + c] = acc[i][j][e];
          S[static_cast<size_t>(c) * a.k + r] = acc[i][j][e];
        }
      }
}

}  // namespace

void launch_lsq_generate(const LsqArgs& a, uint64_t seed, int kind, cudaStream_t st) {
  lsq_generate_kernel<<<dim3(a.ncol, a.nb), 256, 0, st>>>(a, seed, kind);
  DDG_LAUNCH_CHECK();
}

void launch_lsq_gram(const LsqArgs& a, cudaStream_t st) {
  const int t = ceil_div(a.k, GT);
  const int smem = 2 * 2 * GT * GRCP * static_cast<int>(sizeof(double));
  DDG_CUDA(cudaFuncSetAttribute(lsq_gram_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  lsq_gram_kernel<<<dim3(t, t, a.nb), 256, smem, st>>>(a);
  DDG_LAUNCH_CHECK();
}

namespace {
/// FP64 tensor-pipe throughput probe: independent DMMA m8n8k4 chains, 8 per warp (the roofline
/// denominator of the QR / Schur FLOP rates, measured on the box that runs the bench)
__global__ void __launch_bounds__(256) dmma_probe_kernel(double* out, int iters) {
  const double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  double c[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1])
                   : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.0) out[0] = s;
}
}  // namespace

double fp64_peak_probe(int device) {
  DDG_CUDA(cudaSetDevice(device));
  int sms = 0;
  DDG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  double* d = nullptr;
  DDG_CUDA(cudaMalloc(&d, sizeof(double)));
  cudaEvent_t e0, e1;
  DDG_CUDA(cudaEventCreate(&e0));
  DDG_CUDA(cudaEventCreate(&e1));
  const int iters = 4096, blocks = sms * 4;
  dmma_probe_kernel<<<blocks, 256>>>(d, 64);  // warm-up
  DDG_LAUNCH_CHECK();
  double best = 0;
  for (int rep = 0; rep < 3; ++rep) {
    DDG_CUDA(cudaEventRecord(e0));
    dmma_probe_kernel<<<blocks, 256>>>(d, iters);
    DDG_CUDA(cudaEventRecord(e1));
    DDG_CUDA(cudaEventSynchronize(e1));
    float ms = 0;
    DDG_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    // one m8n8k4 = 2 * 8 * 8 * 4 flops per warp instruction
    const double flops = 2.0 * 8 * 8 * 4 * 8.0 * iters * (blocks * 256 / 32);
    best = std::max(best, flops / (ms * 1e-3) / 1e12);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(d);
  return best;
}

}  // namespace ddg

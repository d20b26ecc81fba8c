// Batched blocked Householder QR (sm_100a, fp64) of the local matrices K_i and Kbar_i.
//
// Reference: LsFactor's Eigen::HouseholderQR + R-diagonal branch test (solvers.cpp:24-45).
// Reflector convention as Eigen/LAPACK dlarfg (H = I - tau v v^T, v(0) = 1,
// beta = -sign(alpha) ||x||). Compact WY per 32-column panel (LAPACK dlarft 'F','C').
//
// Structure per panel k0 (all 2N matrices in one launch each):
//   qr_panel      one CTA / matrix: BLAS-2 factorisation of the m x 32 panel, V^T V, T
//   qr_trailing   CTA per (matrix, 64-column tile): W = V^T A (DMMA), W' = T^T W,
//                 A -= V W' (DMMA). FP64 tensor cores via mma.sync.m8n8k4.f64 (SASS DMMA.8);
//                 tcgen05.mma has no f64 kind on sm_100a.
// The appended columns [f | E] ride along in the trailing updates, so the factorisation also
// produces Q0^T [f | E] (the interface rows of Q and Q^T f) with no extra pass.
#include <cfloat>

#include "common.cuh"
#include "kernels.hpp"

namespace ddg {

namespace {

constexpr int NB = kQrNB;
constexpr int TN = 64;  // trailing tile columns
constexpr int RC = 32;  // row chunk

__global__ void __launch_bounds__(1024) qr_panel_kernel(QrArgs a, int k0) {
  const int t = blockIdx.x;
  double* A = a.A + static_cast<size_t>(t) * a.ld * a.ncol;
  const int m = a.m, ld = a.ld;
  const int nb = min(NB, a.M - k0);
  __shared__ double red[32];
  __shared__ double Vs[RC][NB + 1];
  __shared__ double G[NB][NB + 1];
  __shared__ double stau[NB];
  __shared__ double Tsh[NB][NB + 1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

  for (int jj = 0; jj < nb; ++jj) {
    const int c = k0 + jj;
    double* col = A + static_cast<size_t>(c) * ld;
    double part = 0;
    for (int i = c + 1 + threadIdx.x; i < m; i += blockDim.x) part += col[i] * col[i];
    const double tail = block_sum(part, red);
    const double alpha = col[c];
    double tau = 0, beta = alpha, scale = 0;
    const bool triv = !(tail > DBL_MIN);
    if (!triv) {
      beta = sqrt(alpha * alpha + tail);
      if (alpha >= 0) beta = -beta;
      scale = 1.0 / (alpha - beta);
      tau = (beta - alpha) / beta;
    }
    for (int i = c + 1 + threadIdx.x; i < m; i += blockDim.x) col[i] = triv ? 0.0 : col[i] * scale;
    __syncthreads();
    if (threadIdx.x == 0) {
      col[c] = beta;
      stau[jj] = tau;
      a.tau[static_cast<size_t>(t) * a.M + c] = tau;
    }
    // apply H_c to the remaining panel columns: one warp per column
    for (int cc = c + 1 + warp; cc < k0 + nb; cc += 32) {
      double* y = A + static_cast<size_t>(cc) * ld;
      const double yc = y[c];
      double d = 0;
      for (int i = c + 1 + lane; i < m; i += 32) d += col[i] * y[i];
      d = warp_sum(d);
      d = (d + yc) * tau;
      if (lane == 0) y[c] = yc - d;
      for (int i = c + 1 + lane; i < m; i += 32) y[i] -= d * col[i];
    }
    __syncthreads();
  }

  // G = V^T V over the panel (implicit unit diagonal, zeros above)
  const int u = threadIdx.x & 31, v = threadIdx.x >> 5;
  double g = 0;
  for (int r0 = k0; r0 < m; r0 += RC) {
    {
      const int rr = threadIdx.x & 31, uu = threadIdx.x >> 5;  // 32 x 32 chunk
      const int row = r0 + rr;
      double val = 0;
      if (row < m && uu < nb) {
        if (row == k0 + uu) val = 1.0;
        else if (row > k0 + uu) val = A[static_cast<size_t>(k0 + uu) * ld + row];
      }
      Vs[rr][uu] = val;
    }
    __syncthreads();
#pragma unroll 8
    for (int rr = 0; rr < RC; ++rr) g += Vs[rr][u] * Vs[rr][v];
    __syncthreads();
  }
  G[u][v] = g;
  __syncthreads();
  // T: T(j,j) = tau_j, T(0:j, j) = -tau_j T(0:j,0:j) G(0:j, j)
  if (warp == 0) {
    for (int j = 0; j < NB; ++j) Tsh[lane][j] = 0.0;
    __syncwarp();
    for (int j = 0; j < nb; ++j) {
      double s = 0;
      if (lane < j)
        for (int w = lane; w < j; ++w) s += Tsh[lane][w] * G[w][j];
      __syncwarp();
      if (lane < j) Tsh[lane][j] = -stau[j] * s;
      if (lane == j) Tsh[j][j] = stau[j];
      __syncwarp();
    }
  }
  __syncthreads();
  double* T = a.T + static_cast<size_t>(t) * NB * NB;
  T[threadIdx.x] = Tsh[threadIdx.x >> 5][threadIdx.x & 31];
}

__global__ void __launch_bounds__(256) qr_trailing_kernel(QrArgs a, int k0) {
  const int t = blockIdx.y;
  const int nb = min(NB, a.M - k0);
  const int c0 = k0 + nb + blockIdx.x * TN;
  if (c0 >= a.ncol) return;
  const int ncols = min(TN, a.ncol - c0);
  double* A = a.A + static_cast<size_t>(t) * a.ld * a.ncol;
  const int m = a.m, ld = a.ld;
  __shared__ double Vs[RC][NB + 1];
  __shared__ double Ts[NB][NB + 1];
  // the A chunk (pass 1) and W / W' (after pass 1) share storage
  __shared__ double AWbuf[RC * (TN + 1)];
  double(*As)[TN + 1] = reinterpret_cast<double(*)[TN + 1]>(AWbuf);
  double(*Ws)[TN + 1] = reinterpret_cast<double(*)[TN + 1]>(AWbuf);
  static_assert(RC == NB, "A chunk and W share one buffer");
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int lr = lane >> 2, lc = lane & 3;

  auto load_v = [&](int r0) {
    for (int idx = threadIdx.x; idx < RC * NB; idx += blockDim.x) {
      const int rr = idx % RC, uu = idx / RC;
      const int row = r0 + rr;
      double val = 0;
      if (row < m && uu < nb) {
        if (row == k0 + uu) val = 1.0;
        else if (row > k0 + uu) val = A[static_cast<size_t>(k0 + uu) * ld + row];
      }
      Vs[rr][uu] = val;
    }
  };

  // ---- pass 1: W = V^T A_tile   (32 x 64), warp w: t-block (w & 3), col blocks 4*(w>>2)..+3
  const int tb = warp & 3, cb0 = (warp >> 2) * 4;
  double acc[4][2];
#pragma unroll
  for (int q = 0; q < 4; ++q) acc[q][0] = acc[q][1] = 0.0;
  for (int r0 = k0; r0 < m; r0 += RC) {
    load_v(r0);
    for (int idx = threadIdx.x; idx < RC * TN; idx += blockDim.x) {
      const int rr = idx % RC, cc = idx / RC;
      const int row = r0 + rr;
      As[rr][cc] = (row < m && cc < ncols) ? A[static_cast<size_t>(c0 + cc) * ld + row] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < RC / 4; ++kk) {
      const double av = Vs[kk * 4 + lc][tb * 8 + lr];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const double bv = As[kk * 4 + lc][(cb0 + q) * 8 + lr];
        dmma_8x8x4(acc[q][0], acc[q][1], av, bv);
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    Ws[tb * 8 + lr][(cb0 + q) * 8 + 2 * lc] = acc[q][0];
    Ws[tb * 8 + lr][(cb0 + q) * 8 + 2 * lc + 1] = acc[q][1];
  }
  const double* T = a.T + static_cast<size_t>(t) * NB * NB;
  for (int idx = threadIdx.x; idx < NB * NB; idx += blockDim.x) Ts[idx / NB][idx % NB] = T[idx];
  __syncthreads();
  // ---- W' = T^T W  (T upper triangular)
  double wv[NB * TN / 256];
#pragma unroll
  for (int e = 0; e < NB * TN / 256; ++e) {
    const int idx = threadIdx.x + 256 * e;
    const int uu = idx / TN, cc = idx % TN;
    double s = 0;
    for (int w = 0; w <= uu; ++w) s += Ts[w][uu] * Ws[w][cc];
    wv[e] = s;
  }
  __syncthreads();
#pragma unroll
  for (int e = 0; e < NB * TN / 256; ++e) {
    const int idx = threadIdx.x + 256 * e;
    Ws[idx / TN][idx % TN] = wv[e];
  }
  __syncthreads();
  // ---- pass 2: A_tile -= V W'  (row chunk 32 x 64), warp w: row block (w & 3), col blocks 4*(w>>2)..
  const int rb = warp & 3;
  for (int r0 = k0; r0 < m; r0 += RC) {
    load_v(r0);
    __syncthreads();
    double cfr[4][2];
    const int row = r0 + rb * 8 + lr;
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int cc = (cb0 + q) * 8 + 2 * lc + e;
        cfr[q][e] = (row < m && cc < ncols) ? A[static_cast<size_t>(c0 + cc) * ld + row] : 0.0;
      }
#pragma unroll
    for (int kk = 0; kk < NB / 4; ++kk) {
      const double av = -Vs[rb * 8 + lr][kk * 4 + lc];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const double bv = Ws[kk * 4 + lc][(cb0 + q) * 8 + lr];
        dmma_8x8x4(cfr[q][0], cfr[q][1], av, bv);
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int cc = (cb0 + q) * 8 + 2 * lc + e;
        if (row < m && cc < ncols) A[static_cast<size_t>(c0 + cc) * ld + row] = cfr[q][e];
      }
    __syncthreads();
  }
}

__global__ void qr_diag_ratio_kernel(QrArgs a, double* ratio) {
  const int t = blockIdx.x;
  const double* A = a.A + static_cast<size_t>(t) * a.ld * a.ncol;
  __shared__ double smax[32], smin[32];
  double mx = 0, mn = DBL_MAX;
  for (int i = threadIdx.x; i < a.M; i += blockDim.x) {
    const double d = fabs(A[static_cast<size_t>(i) * a.ld + i]);
    mx = fmax(mx, d);
    mn = fmin(mn, d);
  }
  for (int o = 16; o > 0; o >>= 1) {
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (lane == 0) {
    smax[w] = mx;
    smin[w] = mn;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int k = 1; k < (blockDim.x + 31) / 32; ++k) {
      mx = fmax(mx, smax[k]);
      mn = fmin(mn, smin[k]);
    }
    // store min and max; the branch test (solvers.cpp:32) is evaluated by the COD stage
    ratio[2 * t] = mn;
    ratio[2 * t + 1] = mx;
  }
}

}  // namespace

void launch_qr_panel(const QrArgs& a, int k0, cudaStream_t st) {
  qr_panel_kernel<<<a.nmat, 1024, 0, st>>>(a, k0);
  DDG_LAUNCH_CHECK();
}

void launch_qr_trailing(const QrArgs& a, int k0, cudaStream_t st) {
  const int nb = std::min(NB, a.M - k0);
  const int rest = a.ncol - (k0 + nb);
  if (rest <= 0) return;
  dim3 grid(ceil_div(rest, TN), a.nmat);
  qr_trailing_kernel<<<grid, 256, 0, st>>>(a, k0);
  DDG_LAUNCH_CHECK();
}

void launch_qr_diag_ratio(const QrArgs& a, double* ratio, cudaStream_t st) {
  qr_diag_ratio_kernel<<<a.nmat, 256, 0, st>>>(a, ratio);
  DDG_LAUNCH_CHECK();
}

}  // namespace ddg

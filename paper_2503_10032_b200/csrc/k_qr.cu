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
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cfloat>
#include <cstdlib>
#include <string>
#include <vector>

#include "common.cuh"
#include "kernels.hpp"

namespace ddg {

namespace {

constexpr int NB = kQrNB;
constexpr int RC = 32;  // rows per chunk (panel Gram and trailing streams)

// ---------------------------------------------------------------- panel (BLAS-2, one CTA / matrix)
// Column c of the panel costs ONE pass over the remaining panel rows: the pass applies the
// previous reflector H_{c-1} (v scaled on the fly, pivot row set to beta) and, on the updated
// values, accumulates ||x_c||^2 below the diagonal and s_j = x_c . y_j for the panel columns right
// of c. One block reduction (warp reduce-scatter) then gives beta, tau and
// d_j = v_c . y_j = y_cj + s_j / (alpha - beta) for the next pass. Each thread streams two rows
// at a time (up to 64 independent loads in flight), so a column step is one L2 round trip + one
// reduction instead of a chain of per-column dot products.
constexpr int kPanelThreads = 512;
constexpr int kPanelWarps = kPanelThreads / 32;

/// lane l ends with the warp-wide sum of v[l] (31 shuffles for 32 values)
__device__ __forceinline__ double reduce_scatter32(double (&v)[32]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int s = 16; s >= 1; s >>= 1) {
    const bool upper = (lane & s) != 0;
#pragma unroll
    for (int k = 0; k < s; ++k) {
      const double send = upper ? v[k] : v[k + s];
      const double keep = upper ? v[k + s] : v[k];
      v[k] = keep + __shfl_xor_sync(0xffffffffu, send, s);
    }
  }
  return v[0];
}

/// One fused pass of the panel factorisation with NR = nb - jj columns left (compile-time, so
/// every loop is fully unrolled with no per-element predicates): applies H_{c-1} to this warp's
/// rows, stores them, and accumulates ||x_c||^2 and x_c . y_{c+k} (lane k of accS: column jj+k).
template <int NR>
__device__ __forceinline__ void panel_pass(double* P, size_t ld, int m, int rlo, int jj, int cp, int c,
                                           double tau_p, double scale_p, double beta_p, bool triv_p,
                                           const double* sd, double* srow, double& accS, double& n2) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int rbase = rlo + warp * 32; rbase < m; rbase += kPanelThreads) {
    const int r = rbase + lane;
    const bool valid = r < m;
    double y[32];
#pragma unroll
    for (int k = 0; k < 32; ++k) y[k] = (k < NR && valid) ? P[static_cast<size_t>(jj + (k < NR ? k : 0)) * ld + r] : 0.0;
    if (jj > 0) {  // apply H_{c-1}: v on this row, pivot row gets beta
      double* pc = P + static_cast<size_t>(jj - 1) * ld + r;
      const double xp = valid ? *pc : 0.0;
      const double v = (r == cp) ? 1.0 : (triv_p ? 0.0 : xp * scale_p);
      const double tv = tau_p * v;
#pragma unroll
      for (int k = 0; k < NR; ++k) y[k] -= tv * sd[jj + k];
      if (valid) {
        *pc = (r == cp) ? beta_p : v;
#pragma unroll
        for (int k = 0; k < NR; ++k) P[static_cast<size_t>(jj + k) * ld + r] = y[k];
      }
    }
    if constexpr (NR > 0) {
      const double x = y[0];
      if (valid && r == c) {
#pragma unroll
        for (int k = 0; k < NR; ++k) srow[jj + k] = y[k];
      }
      const bool acc_row = valid && r > c;
      // products in place; slot 0 carries ||x||^2 (column jj itself)
#pragma unroll
      for (int k = 0; k < 32; ++k) y[k] = (k < NR && acc_row) ? x * y[k] : 0.0;
      accS += reduce_scatter32(y);
    }
  }
  (void)n2;
}

/// Block reflector of a factored panel (both panel kernels): G = V^T V from the stored panel,
/// T from G and tau by a blocked dlarft (the four 8-column diagonal blocks by the column
/// recurrence, then T_AB = -T_A (G_AB T_B) on 8- and 16-column block pairs), written to quadrant
/// (toff, toff) of the per-matrix T; combine = 1 also forms the coupling block T12 of a 64-wide
/// block. `dyn`: kFinishDoubles of shared memory = G / T scratch + a kGStages-deep ring of 64-row
/// chunks of the panel (the Gram pass is L2-latency bound: ~5 chunks in flight).
constexpr int kGRows = 64, kGRCP = 68, kGStages = 6;  // kGRCP = 4 (mod 16): conflict-free fragments
constexpr int kFinishDoubles = 4 * NB * (NB + 1) + kGStages * NB * kGRCP;

__device__ __forceinline__ void panel_finish(const QrArgs& a, int t, int k0, int nb, int toff, int combine,
                                             const double* stau, double* dyn) {
  double* A = a.A + static_cast<size_t>(t) * a.ld * a.ncol;
  const int m = a.m;
  const size_t ld = a.ld;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const double* P = A + static_cast<size_t>(k0) * ld;
  double(*G)[NB + 1] = reinterpret_cast<double(*)[NB + 1]>(dyn);
  double(*Tsh)[NB + 1] = G + NB;
  double(*Vs)[NB + 1] = G + 2 * NB;
  double(*T2s)[NB + 1] = G + 3 * NB;
  // G = V^T V over the panel (implicit unit diagonal, zeros above) on DMMA: 16 warps = the 4 x 4
  // grid of 8 x 8 tiles of G; 64-row chunks (column-major, padded) through a cp.async ring
  const int u = threadIdx.x & 31, v = threadIdx.x >> 5;
  const int tu = warp >> 2, tv = warp & 3, lr = lane >> 2, lc = lane & 3;
  double g0 = 0, g1 = 0;
  {
    double* ring = dyn + 4 * NB * (NB + 1);  // [kGStages][NB][kGRCP]
    const int nq = (m - k0 + kGRows - 1) / kGRows;
    auto issue = [&](int q) {
      if (q < nq) {
        for (int s = threadIdx.x; s < NB * kGRows / 2; s += blockDim.x) {  // 16-B segments
          const int col = s >> 5, seg = s & 31;
          const int row = k0 + q * kGRows + 2 * seg;
          const bool ok = col < nb && row < static_cast<int>(ld);
          const uint32_t sa = static_cast<uint32_t>(
              __cvta_generic_to_shared(ring + (q % kGStages) * NB * kGRCP + col * kGRCP + 2 * seg));
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sa),
                       "l"(P + static_cast<size_t>(ok ? col : 0) * ld + (ok ? row : 0)), "r"(ok ? 16 : 0)
                       : "memory");
        }
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    for (int q = 0; q < kGStages - 1; ++q) issue(q);
    for (int q = 0; q < nq; ++q) {
      // chunk q landed for this thread; after the barrier every thread is done with chunk q-1, so
      // its slot takes chunk q + kGStages - 1 (one barrier per chunk)
      asm volatile("cp.async.wait_group %0;" ::"n"(kGStages - 2) : "memory");
      __syncthreads();
      issue(q + kGStages - 1);
      double* Vc = ring + (q % kGStages) * NB * kGRCP;
      const int r0 = k0 + q * kGRows;
      if (r0 < k0 + nb) {  // unit diagonal, zeros above it
        for (int idx = threadIdx.x; idx < NB * kGRows; idx += blockDim.x) {
          const int uu = idx / kGRows, rr = idx % kGRows;
          const int row = r0 + rr;
          if (row <= k0 + uu) Vc[uu * kGRCP + rr] = (row == k0 + uu && uu < nb) ? 1.0 : 0.0;
        }
        __syncthreads();
      }
#pragma unroll
      for (int kk = 0; kk < kGRows / 4; ++kk)
        dmma_8x8x4(g0, g1, Vc[(tu * 8 + lr) * kGRCP + kk * 4 + lc], Vc[(tv * 8 + lr) * kGRCP + kk * 4 + lc]);
    }
    __syncthreads();
    asm volatile("cp.async.wait_group 0;" ::: "memory");
  }
  G[tu * 8 + lr][tv * 8 + 2 * lc] = g0;
  G[tu * 8 + lr][tv * 8 + 2 * lc + 1] = g1;
  for (int idx = threadIdx.x; idx < NB * (NB + 1); idx += blockDim.x) (&Tsh[0][0])[idx] = 0.0;
  __syncthreads();
  // T diagonal blocks: warp s < 4 runs T(j,j) = tau_j, T(c:j, j) = -tau_j T(c:j,c:j) G(c:j, j) on
  // columns c = 8s .. 8s+7 (tau = 0 past the panel width)
  if (warp < NB / 8) {
    const int c0 = warp * 8;
    for (int jj = 0; jj < 8; ++jj) {
      const int j = c0 + jj;
      const double tj = j < nb ? stau[j] : 0.0;
      double s = 0;
      if (lane < jj)
        for (int w = lane; w < jj; ++w) s += Tsh[c0 + lane][c0 + w] * G[c0 + w][j];
      __syncwarp();
      if (lane < jj) Tsh[c0 + lane][j] = -tj * s;
      if (lane == jj) Tsh[j][j] = tj;
      __syncwarp();
    }
  }
  __syncthreads();
  // couplings of block pairs (A, B = A + bs): X = G_AB T_B (into Vs), T_AB = -T_A X
  for (int bs = 8; bs < NB; bs *= 2) {
    const int n = (NB / (2 * bs)) * bs * bs;
    for (int idx = threadIdx.x; idx < n; idx += blockDim.x) {
      const int p = idx / (bs * bs), e = idx % (bs * bs), r = e / bs, c = e % bs;
      const int a0 = 2 * p * bs, b0 = a0 + bs;
      double s = 0;
      for (int w = 0; w <= c; ++w) s += G[a0 + r][b0 + w] * Tsh[b0 + w][b0 + c];
      Vs[a0 + r][b0 + c] = s;
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < n; idx += blockDim.x) {
      const int p = idx / (bs * bs), e = idx % (bs * bs), r = e / bs, c = e % bs;
      const int a0 = 2 * p * bs, b0 = a0 + bs;
      double s = 0;
      for (int w = r; w < bs; ++w) s += Tsh[a0 + r][a0 + w] * Vs[a0 + w][b0 + c];
      Tsh[a0 + r][b0 + c] = -s;
    }
    __syncthreads();
  }
  double* T = a.T + static_cast<size_t>(t) * kQrTmax * kQrTmax;
  for (int idx = threadIdx.x; idx < NB * NB; idx += blockDim.x)
    T[(toff + (idx >> 5)) * kQrTmax + toff + (idx & 31)] = Tsh[idx >> 5][idx & 31];
  if (!combine) return;
  // ---- second half of a 64-wide block: T12 = -T1 (V1^T V2) T2, V1 = the 32 reflectors left of k0
  //      (rows >= k0 only: V2 is zero above its diagonal)
  const double* V1 = A + static_cast<size_t>(k0 - NB) * ld;
  g0 = g1 = 0;
  for (int r0 = k0; r0 < m; r0 += RC) {
    for (int idx = threadIdx.x; idx < RC * NB; idx += blockDim.x) {
      const int rr = idx & 31, uu = idx >> 5;
      const int row = r0 + rr;
      double v2 = 0;
      if (row < m && uu < nb) {
        if (row == k0 + uu) v2 = 1.0;
        else if (row > k0 + uu) v2 = P[static_cast<size_t>(uu) * ld + row];
      }
      Vs[rr][uu] = v2;
      G[rr][uu] = row < m ? V1[static_cast<size_t>(uu) * ld + row] : 0.0;  // V1 rows >= k0 (below its diagonal)
    }
    __syncthreads();
#pragma unroll 8
    for (int rr = 0; rr < RC; ++rr) {
      g0 += G[rr][u] * Vs[rr][v];       // (V1^T V2)(u, v)
      g1 += G[rr][u] * Vs[rr][v + 16];
    }
    __syncthreads();
  }
  // Tsh <- G12 ; then T12 = -T1 G12 T2 (T1 from global, T2 = this panel's T in Tsh -> keep a copy)
  for (int idx = threadIdx.x; idx < NB * NB; idx += blockDim.x) T2s[idx >> 5][idx & 31] = Tsh[idx >> 5][idx & 31];
  __syncthreads();
  Vs[u][v] = g0;  // reuse Vs as G12
  Vs[u][v + 16] = g1;
  for (int idx = threadIdx.x; idx < NB * NB; idx += blockDim.x)
    G[idx >> 5][idx & 31] = T[(idx >> 5) * kQrTmax + (idx & 31)];  // T1 (rows/cols 0..31)
  __syncthreads();
  // X = G12 T2 (thread -> two entries)
  double x0 = 0, x1 = 0;
  for (int w = 0; w < NB; ++w) {
    x0 += Vs[u][w] * T2s[w][v];
    x1 += Vs[u][w] * T2s[w][v + 16];
  }
  __syncthreads();
  Tsh[u][v] = x0;
  Tsh[u][v + 16] = x1;
  __syncthreads();
  double y0 = 0, y1 = 0;
  for (int w = 0; w < NB; ++w) {
    y0 += G[u][w] * Tsh[w][v];
    y1 += G[u][w] * Tsh[w][v + 16];
  }
  T[u * kQrTmax + NB + v] = -y0;
  T[u * kQrTmax + NB + v + 16] = -y1;
  // T21 block (lower left) is zero: T is upper triangular
  T[(NB + u) * kQrTmax + v] = 0.0;
  T[(NB + u) * kQrTmax + v + 16] = 0.0;
}

__global__ void __launch_bounds__(kPanelThreads, 1) qr_panel_kernel(QrArgs a, int k0, int toff, int combine) {
  const int t = blockIdx.x;
  double* A = a.A + static_cast<size_t>(t) * a.ld * a.ncol;
  const int m = a.m;
  const size_t ld = a.ld;
  const int nb = min(NB, a.M - k0);
  __shared__ double sred[kPanelWarps][NB + 1];
  __shared__ double sfin[NB + 1];
  __shared__ double srow[NB];
  __shared__ double sd[NB];
  __shared__ double stau[NB];
  __shared__ double sbeta, sscale;
  __shared__ int striv;
  extern __shared__ __align__(16) double dyn[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* P = A + static_cast<size_t>(k0) * ld;  // panel column j at P + j*ld

  for (int jj = 0; jj <= nb; ++jj) {
    const int cp = k0 + jj - 1;  // previous pivot (row and column), jj > 0
    const int c = k0 + jj;       // current pivot, jj < nb
    const int jlo = jj > 0 ? jj - 1 : 0;
    const int rlo = jj > 0 ? cp : c;
    double tau_p = 0, scale_p = 0, beta_p = 0;
    bool triv_p = true;
    if (jj > 0) {
      tau_p = stau[jj - 1];
      scale_p = sscale;
      beta_p = sbeta;
      triv_p = striv != 0;
    }
    // lane k accumulates x_c . y_{c+k} (k = 0: ||x_c||^2) over the rows this warp visits
    double accS = 0, n2 = 0;
    switch (nb - jj) {
#define DDG_PANEL_CASE(n) \
  case n:                 \
    panel_pass<n>(P, ld, m, rlo, jj, cp, c, tau_p, scale_p, beta_p, triv_p, sd, srow, accS, n2); \
    break;
      DDG_PANEL_CASE(0) DDG_PANEL_CASE(1) DDG_PANEL_CASE(2) DDG_PANEL_CASE(3) DDG_PANEL_CASE(4)
      DDG_PANEL_CASE(5) DDG_PANEL_CASE(6) DDG_PANEL_CASE(7) DDG_PANEL_CASE(8) DDG_PANEL_CASE(9)
      DDG_PANEL_CASE(10) DDG_PANEL_CASE(11) DDG_PANEL_CASE(12) DDG_PANEL_CASE(13) DDG_PANEL_CASE(14)
      DDG_PANEL_CASE(15) DDG_PANEL_CASE(16) DDG_PANEL_CASE(17) DDG_PANEL_CASE(18) DDG_PANEL_CASE(19)
      DDG_PANEL_CASE(20) DDG_PANEL_CASE(21) DDG_PANEL_CASE(22) DDG_PANEL_CASE(23) DDG_PANEL_CASE(24)
      DDG_PANEL_CASE(25) DDG_PANEL_CASE(26) DDG_PANEL_CASE(27) DDG_PANEL_CASE(28) DDG_PANEL_CASE(29)
      DDG_PANEL_CASE(30) DDG_PANEL_CASE(31) DDG_PANEL_CASE(32)
#undef DDG_PANEL_CASE
      default:
        break;
    }
    if (jj == nb) break;
    // ---- block reduction of (n2, s_j)
    sred[warp][lane] = accS;
    __syncthreads();
    if (threadIdx.x < NB) {
      double s = 0;
      for (int w = 0; w < kPanelWarps; ++w) s += sred[w][threadIdx.x];
      sfin[threadIdx.x] = s;  // sfin[k]: column jj+k (k = 0: squared norm below the diagonal)
    }
    __syncthreads();
    {
      const double alpha = srow[jj], tail = sfin[0];
      double tau = 0, beta = alpha, scale = 0;
      const bool triv = !(tail > DBL_MIN);
      if (!triv) {
        beta = sqrt(alpha * alpha + tail);
        if (alpha >= 0) beta = -beta;
        scale = 1.0 / (alpha - beta);
        tau = (beta - alpha) / beta;
      }
      if (threadIdx.x < NB) {
        const int j = threadIdx.x;
        sd[j] = (j > jj && j < nb) ? srow[j] + sfin[j - jj] * scale : 0.0;
      }
      if (threadIdx.x == 0) {
        stau[jj] = tau;
        sbeta = beta;
        sscale = scale;
        striv = triv ? 1 : 0;
        a.tau[static_cast<size_t>(t) * a.M + c] = tau;
      }
    }
    __syncthreads();
  }
  __syncthreads();
  panel_finish(a, t, k0, nb, toff, combine, stau, dyn);
}

// ---------------------------------------------------------------- panel, shared-memory resident
// For panels of up to ~3300 rows the 32 columns are factored as four 8-column sub-panels, each
// staged once into shared memory (cp.async) and factored there with the same fused column passes
// (no L2/HBM round trip per column: the streaming kernel above re-reads and re-writes the rest of
// the panel on every column, ~16x the panel's bytes). Between sub-panels, the 8 reflectors are
// applied to the panel columns on their right as one small blocked update on DMMA
// (W = V8^T Y, W' = T8^T W, Y -= V8 W'), reading Y from global memory twice.
constexpr int kSub = 8;

/// lane l ends with the warp-wide sum of v[l & 7] (7 + 2 shuffles for 8 values)
__device__ __forceinline__ double reduce_scatter8(double (&v)[kSub]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int s = 4; s >= 1; s >>= 1) {
    const bool upper = (lane & s) != 0;
#pragma unroll
    for (int k = 0; k < s; ++k) {
      const double send = upper ? v[k] : v[k + s];
      const double keep = upper ? v[k + s] : v[k];
      v[k] = keep + __shfl_xor_sync(0xffffffffu, send, s);
    }
  }
  double r = v[0];
  r += __shfl_xor_sync(0xffffffffu, r, 8);
  r += __shfl_xor_sync(0xffffffffu, r, 16);
  return r;
}

/// Pass jj over a staged sub-panel (column j at S + j*lds, row 0 = the sub-panel's first pivot
/// row, R rows): apply H_{jj-1} to columns jj.. (sdk[k] = v_{jj-1} . y_{jj+k}, in registers), then
/// accumulate ||x_jj||^2 below the diagonal and x_jj . y_{jj+k} into acc[k] (this thread's rows).
template <int NR>
__device__ __forceinline__ void sub_pass(double* S, int lds, int R, int jj, double tau_p, double scale_p, double beta_p,
                                         bool triv_p, const double (&sdk)[kSub], double* srowl, double (&acc)[kSub]) {
  const int rlo = jj > 0 ? jj - 1 : 0;
  for (int i = rlo + threadIdx.x; i < R; i += kPanelThreads) {
    double y[NR > 0 ? NR : 1];
#pragma unroll
    for (int k = 0; k < NR; ++k) y[k] = S[(jj + k) * lds + i];
    if (jj > 0) {
      double* pc = S + (jj - 1) * lds + i;
      const double v = (i == jj - 1) ? 1.0 : (triv_p ? 0.0 : *pc * scale_p);
      const double tv = tau_p * v;
#pragma unroll
      for (int k = 0; k < NR; ++k) {
        y[k] -= tv * sdk[k];
        S[(jj + k) * lds + i] = y[k];
      }
      *pc = (i == jj - 1) ? beta_p : v;
    }
    if constexpr (NR > 0) {
      if (i == jj) {
#pragma unroll
        for (int k = 0; k < NR; ++k) srowl[k] = y[k];  // row jj, columns jj + k
      }
      if (i > jj) {
        const double x = y[0];
#pragma unroll
        for (int k = 0; k < NR; ++k) acc[k] += x * y[k];
      }
    }
  }
}

__global__ void __launch_bounds__(kPanelThreads, 1)
    qr_panel_smem_kernel(QrArgs a, int k0, int toff, int combine, int lds) {
  const int t = blockIdx.x;
  double* A = a.A + static_cast<size_t>(t) * a.ld * a.ncol;
  const int m = a.m;
  const size_t ld = a.ld;
  const int nb = min(NB, a.M - k0);
  extern __shared__ __align__(16) double dyn[];  // sub-panel [kSub][lds]; later panel_finish scratch
  // per-column reduction partials and row jj, double-buffered by column parity: ONE block barrier
  // per column — every warp then sums the 16 partials itself (the same order) and derives tau,
  // beta, scale and the next pass's v . y terms in registers
  __shared__ double sred[2][kPanelWarps][kSub];
  __shared__ double srow[2][kSub];
  __shared__ double stau[NB];
  __shared__ double sGp[kPanelWarps][kSub * kSub];  // V8^T V8 partials (per warp)
  __shared__ double sT8[kSub][kSub + 1];
  __shared__ double sWp[kPanelWarps * kSub * kSub];  // V8^T Y partials (per row group)
  __shared__ double sW[kSub][NB + 1];               // W' = T8^T W
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int lr = lane >> 2, lc = lane & 3;
  double* P = A + static_cast<size_t>(k0) * ld;
  // DDELM_QR_TRACE: thread 0's clock per section (0 stage-in, 1 column steps, 2 write-back,
  // 3 update of the panel's remaining columns, 4 G / T finish)
  unsigned long long tlast = 0;
  auto stamp = [&](int sec) {
    if (a.trace != nullptr && threadIdx.x == 0) {
      unsigned long long now;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
      if (sec >= 0) a.trace[t * 8 + sec] += static_cast<double>(now - tlast);
      tlast = now;
    }
  };
  stamp(-1);

  for (int s0 = 0; s0 < nb; s0 += kSub) {
    const int w = min(kSub, nb - s0);
    const int c0 = k0 + s0;  // first pivot (row and column) of the sub-panel
    const int R = m - c0;
    double* Pc = P + static_cast<size_t>(s0) * ld + c0;  // column j at Pc + j*ld, from row c0
    {
      const int nseg = (R + 1) >> 1;
      for (int idx = threadIdx.x; idx < w * nseg; idx += kPanelThreads) {
        const int j = idx / nseg, sg = idx - j * nseg;
        const uint32_t sa = static_cast<uint32_t>(__cvta_generic_to_shared(dyn + j * lds + 2 * sg));
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sa), "l"(Pc + static_cast<size_t>(j) * ld + 2 * sg),
                     "r"(R - 2 * sg >= 2 ? 16 : 8)
                     : "memory");
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    stamp(0);
    double tau_p = 0, scale_p = 0, beta_p = 0;
    bool triv_p = true;
    double sdk[kSub];
#pragma unroll
    for (int k = 0; k < kSub; ++k) sdk[k] = 0.0;
    for (int jj = 0; jj <= w; ++jj) {
      double acc[kSub];
#pragma unroll
      for (int k = 0; k < kSub; ++k) acc[k] = 0.0;
      double* srowl = srow[jj & 1];
      switch (w - jj) {
#define DDG_SUB_CASE(n) \
  case n:               \
    sub_pass<n>(dyn, lds, R, jj, tau_p, scale_p, beta_p, triv_p, sdk, srowl, acc); \
    break;
        DDG_SUB_CASE(0) DDG_SUB_CASE(1) DDG_SUB_CASE(2) DDG_SUB_CASE(3) DDG_SUB_CASE(4)
        DDG_SUB_CASE(5) DDG_SUB_CASE(6) DDG_SUB_CASE(7) DDG_SUB_CASE(8)
#undef DDG_SUB_CASE
        default:
          break;
      }
      if (jj == w) break;
      const double red = reduce_scatter8(acc);
      if (lane < kSub) sred[jj & 1][warp][lane] = red;
      __syncthreads();
      double sf = 0;  // lane k < 8: column jj+k (k = 0: squared norm below the diagonal)
      if (lane < kSub)
        for (int q = 0; q < kPanelWarps; ++q) sf += sred[jj & 1][q][lane];
      double sfin[kSub];
#pragma unroll
      for (int k = 0; k < kSub; ++k) sfin[k] = __shfl_sync(0xffffffffu, sf, k);
      const double alpha = srowl[0], tail = sfin[0];
      double tau = 0, beta = alpha, scale = 0;
      const bool triv = !(tail > DBL_MIN);
      if (!triv) {
        beta = sqrt(alpha * alpha + tail);
        if (alpha >= 0) beta = -beta;
        scale = 1.0 / (alpha - beta);
        tau = (beta - alpha) / beta;
      }
      // v_jj . y_j for the columns j = jj+1+k of the next pass
#pragma unroll
      for (int k = 0; k + 1 < kSub; ++k) sdk[k] = (jj + 1 + k < w) ? srowl[1 + k] + sfin[k + 1] * scale : 0.0;
      sdk[kSub - 1] = 0.0;
      if (threadIdx.x == 0) {
        stau[s0 + jj] = tau;
        a.tau[static_cast<size_t>(t) * a.M + c0 + jj] = tau;
      }
      tau_p = tau;
      scale_p = scale;
      beta_p = beta;
      triv_p = triv;
    }
    __syncthreads();
    stamp(1);
    // write the factored sub-panel back (R entries above the diagonal, beta, v below)
    for (int j = 0; j < w; ++j)
      for (int i = threadIdx.x; i < R; i += kPanelThreads) Pc[static_cast<size_t>(j) * ld + i] = dyn[j * lds + i];
    const int nrem = nb - s0 - w;  // panel columns right of the sub-panel
    if (a.trace != nullptr) __syncthreads();
    stamp(2);
    if (nrem <= 0) break;
    // ---- apply the sub-panel's reflectors to the panel columns on its right
    double* Yc = P + static_cast<size_t>(s0 + w) * ld + c0;  // column q at Yc + q*ld, from row c0
    auto vval = [&](int j, int i) -> double {  // V(i, j): unit diagonal, zeros above
      return (j < w && i < R) ? (i > j ? dyn[j * lds + i] : (i == j ? 1.0 : 0.0)) : 0.0;
    };
    const int nk = (R + 3) >> 2;  // 4-row k-steps
    const int ntiles = (nrem + 7) >> 3;
    const int ngroups = kPanelWarps / ntiles;
    const int nt = warp % ntiles, g = warp / ntiles;
    {  // G8 = V8^T V8 (all warps) and W = V8^T Y partials (warps of the first ngroups groups)
      double g0 = 0, g1 = 0;
      for (int q = warp; q < nk; q += kPanelWarps) {
        const double x = vval(lr, 4 * q + lc);
        dmma_8x8x4(g0, g1, x, x);
      }
      sGp[warp][lr * kSub + 2 * lc] = g0;
      sGp[warp][lr * kSub + 2 * lc + 1] = g1;
      if (g < ngroups) {
        const int col = nt * 8 + lr;
        const bool cok = col < nrem;
        const double* yc = Yc + static_cast<size_t>(cok ? col : 0) * ld;
        double w0 = 0, w1 = 0;
        constexpr int U = 8;
        for (int q0 = g * U; q0 < nk; q0 += ngroups * U) {
          double av[U], bv[U];
#pragma unroll
          for (int u = 0; u < U; ++u) {
            const int i = 4 * (q0 + u) + lc;
            av[u] = vval(lr, i);
            bv[u] = (cok && i < R) ? yc[i] : 0.0;
          }
#pragma unroll
          for (int u = 0; u < U; ++u) dmma_8x8x4(w0, w1, av[u], bv[u]);
        }
        const int wc = ntiles * 8;
        sWp[(g * kSub + lr) * wc + nt * 8 + 2 * lc] = w0;
        sWp[(g * kSub + lr) * wc + nt * 8 + 2 * lc + 1] = w1;
      }
    }
    __syncthreads();
    const int wc = ntiles * 8;
    if (threadIdx.x < kSub * kSub) {
      double s = 0;
      for (int q = 0; q < kPanelWarps; ++q) s += sGp[q][threadIdx.x];
      sGp[0][threadIdx.x] = s;
    }
    for (int e = threadIdx.x; e < kSub * wc; e += kPanelThreads) {
      double s = 0;
      for (int q = 0; q < ngroups; ++q) s += sWp[q * kSub * wc + e];
      sWp[e] = s;  // W(j, c) at sWp[j*wc + c]
    }
    __syncthreads();
    if (warp == 0) {  // T8 by the dlarft recurrence
      if (lane < kSub)
        for (int j = 0; j < kSub; ++j) sT8[lane][j] = 0.0;
      __syncwarp();
      for (int j = 0; j < w; ++j) {
        double s = 0;
        if (lane < j)
          for (int q = lane; q < j; ++q) s += sT8[lane][q] * sGp[0][q * kSub + j];
        __syncwarp();
        if (lane < j) sT8[lane][j] = -stau[s0 + j] * s;
        if (lane == j) sT8[j][j] = stau[s0 + j];
        __syncwarp();
      }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < kSub * wc; e += kPanelThreads) {  // W' = T8^T W
      const int j = e / wc, c = e - j * wc;
      double s = 0;
      for (int q = 0; q <= j; ++q) s += sT8[q][j] * sWp[q * wc + c];
      sW[j][c] = s;
    }
    __syncthreads();
    // Y -= V8 W': 8-row x 8-column tiles, the Y tile loaded into the DMMA accumulators
    if (g < ngroups) {
      const double b0 = -sW[lc][nt * 8 + lr], b1 = -sW[4 + lc][nt * 8 + lr];
      const int colA = nt * 8 + 2 * lc;
      const bool ok0 = colA < nrem, ok1 = colA + 1 < nrem;
      double* y0 = Yc + static_cast<size_t>(ok0 ? colA : 0) * ld;
      double* y1 = Yc + static_cast<size_t>(ok1 ? colA + 1 : 0) * ld;
      const int nrt = (R + 7) >> 3;
      constexpr int U = 4;
      for (int r0 = g * U; r0 < nrt; r0 += ngroups * U) {
        double c[U][2];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int i = 8 * (r0 + u) + lr;
          c[u][0] = (ok0 && i < R) ? y0[i] : 0.0;
          c[u][1] = (ok1 && i < R) ? y1[i] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int i = 8 * (r0 + u) + lr;
          dmma_8x8x4(c[u][0], c[u][1], vval(lc, i), b0);
          dmma_8x8x4(c[u][0], c[u][1], vval(4 + lc, i), b1);
          if (ok0 && i < R) y0[i] = c[u][0];
          if (ok1 && i < R) y1[i] = c[u][1];
        }
      }
    }
    __syncthreads();
    stamp(3);
  }
  __syncthreads();
  stamp(-1);
  panel_finish(a, t, k0, nb, toff, combine, stau, dyn);
  if (a.trace != nullptr) __syncthreads();
  stamp(4);
}

// ---------------------------------------------------------------- trailing update (DMMA)
// CTA = (matrix t, 64-column tile of the trailing matrix). The tile and the panel's reflectors V
// stream through a 3-stage cp.async ring in 32-row chunks, twice:
//   pass 1   W  = V^T A_tile          (NB x 64, DMMA m8n8k4, K = rows)
//            W' = T^T W                (T upper triangular, from qr_panel)
//   pass 2   A_tile -= V W'           (per chunk: accumulators initialised from the staged chunk,
//                                      K = NB; result written back to smem, then coalesced stores)
// Chunks are column-major in shared memory with a 36-double column stride: every m8n8k4 fragment
// load (A: 4 k x 8 m, B: 4 k x 8 n) hits 16 distinct 8-byte banks per half-warp.
constexpr int TN = 64;    // tile columns
constexpr int RCP = 36;   // padded column stride of a staged chunk
constexpr int TNP = 68;   // padded row stride of W / W'

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool valid) {
  const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  const int n = valid ? 16 : 0;  // src-size 0: zero fill
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(s), "l"(gmem), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

/// ring of ST stages; ST = 2 keeps T in L2 instead of shared memory so that 3 CTAs fit an SM
template <int NB_, int ST>
struct TrailSmem {
  static constexpr bool kTsmem = ST >= 3;
  double V[ST][NB_ * RCP];  // V chunk, column u at V[u*RCP + k]
  double A[ST][TN * RCP];   // A chunk, column c at A[c*RCP + k]
  double W[NB_ * TNP];      // W, then W'
  double T[kTsmem ? NB_ * (NB_ + 1) : 2];
  uint64_t full[ST];        // bulk-copy completion of each ring stage
};

template <int NB_, int kTrStages>
__global__ void __launch_bounds__(256, NB_ == 32 ? (kTrStages == 2 ? 3 : 2) : 1)
    qr_trailing_kernel(QrArgs a, int k0, int nbw, int cb, int ce, int tq, const __grid_constant__ CUtensorMap tmA,
                       const __grid_constant__ CUtensorMap tmV) {
  static_assert(NB_ == 32 || NB_ == 64, "panel width");
  constexpr int MT = NB_ / 8;  // m-tiles of W
  extern __shared__ __align__(16) double smraw[];
  TrailSmem<NB_, kTrStages>& S = *reinterpret_cast<TrailSmem<NB_, kTrStages>*>(smraw);
  constexpr bool kTrTsmem = TrailSmem<NB_, kTrStages>::kTsmem;
  const int t = blockIdx.y;
  const int nb = nbw;  // reflectors k0 .. k0 + nb - 1 (nb <= NB_)
  const int c0 = cb + blockIdx.x * TN;
  if (c0 >= ce) return;
  const int ncols = min(TN, ce - c0);
  double* A = a.A + static_cast<size_t>(t) * a.ld * a.ncol;
  const size_t ld = a.ld;
  const int nq = (a.m - k0 + RC - 1) / RC;  // chunks per pass
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int lr = lane >> 2, lc = lane & 3;

  // issue chunk q of the unified stream (q < nq: pass 1, else pass 2) into stage q % 3 with two TMA
  // tensor copies (cp.async.bulk.tensor, SASS UTMALDG): the 36-row x 64-column A tile box and the
  // 36-row x NB V box of the batched matrices seen as one (ld x ncol * nmat) tensor. The 36-row
  // box IS the padded column stride (RCP): every m8n8k4 fragment load stays bank-conflict free;
  // rows past ld arrive as zeros (TMA out-of-bounds fill). Columns past the tile / panel carry
  // finite data of the neighbouring columns: their W' rows are zero (T is zero-padded) and their
  // updates are never stored.
  if (threadIdx.x == 0) {
    for (int s2 = 0; s2 < kTrStages; ++s2) mbar_init(&S.full[s2], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int colA = t * a.ncol + c0, colV = t * a.ncol + k0;
  auto issue = [&](int q) {
    if (q >= 2 * nq || threadIdx.x != 0) return;
    const int st = q % kTrStages;
    // pass 2 walks the row chunks backwards: its first chunks are the ones pass 1 read last,
    // still in L2 (the concurrent A tiles far exceed L2, so a forward pass 2 re-reads HBM)
    const int cq = q < nq ? q : 2 * nq - 1 - q;
    const int row = k0 + cq * RC;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_expect_tx(&S.full[st], static_cast<uint32_t>((TN + NB_) * RCP * sizeof(double)));
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_u32(S.A[st])),
        "l"(&tmA), "r"(row), "r"(colA), "r"(smem_u32(&S.full[st]))
        : "memory");
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            smem_u32(S.V[st])),
        "l"(&tmV), "r"(row), "r"(colV), "r"(smem_u32(&S.full[st]))
        : "memory");
  };
  auto wait_chunk = [&](int q) { mbar_wait(&S.full[q % kTrStages], static_cast<uint32_t>((q / kTrStages) & 1)); };
  // unit lower-triangular structure of V inside the first NB rows of the stream
  auto fix_v = [&](int st, int r0) {
    if (r0 >= k0 + nb) return;
    for (int idx = threadIdx.x; idx < NB_ * RC; idx += blockDim.x) {
      const int u = idx / RC, k = idx % RC;
      const int row = r0 + k;
      if (row <= k0 + u) S.V[st][u * RCP + k] = (row == k0 + u && u < nb) ? 1.0 : 0.0;
    }
  };

  for (int q = 0; q < kTrStages - 1; ++q) issue(q);
  // T (nb x nb upper triangular, zero padded)
  const double* Tg = a.T + static_cast<size_t>(t) * kQrTmax * kQrTmax;
  if (kTrTsmem)
    for (int idx = threadIdx.x; idx < NB_ * NB_; idx += blockDim.x) {
      const int i = idx / NB_, j = idx % NB_;
      S.T[i * (NB_ + 1) + j] = (i < nb && j < nb) ? Tg[(tq + i) * kQrTmax + tq + j] : 0.0;
    }

  // ---- pass 1: W = V^T A_tile. Warp tile: (MT/2) m-tiles x 2 n-tiles.
  //      NB=32: warp -> m-tiles {2(w&1), +1}, n-tiles {2(w>>1), +1};  NB=64: m-tiles 4(w&1).., n-tiles 2(w>>1)..
  constexpr int WM = MT / 2;
  const int mt0 = (warp & 1) * WM, nt0 = (warp >> 1) * 2;
  double acc[WM][2][2];
#pragma unroll
  for (int i = 0; i < WM; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  for (int q = 0; q < nq; ++q) {
    wait_chunk(q);
    __syncthreads();  // every warp is done with the stage chunk q + kTrStages - 1 overwrites
    issue(q + kTrStages - 1);
    const int st = q % kTrStages;
    fix_v(st, k0 + q * RC);
    __syncthreads();
    const double* Vs = S.V[st];
    const double* As = S.A[st];
#pragma unroll
    for (int kk = 0; kk < RC / 4; ++kk) {
      const int k = kk * 4 + lc;
      double av[WM], bv[2];
#pragma unroll
      for (int i = 0; i < WM; ++i) av[i] = Vs[((mt0 + i) * 8 + lr) * RCP + k];
#pragma unroll
      for (int j = 0; j < 2; ++j) bv[j] = As[((nt0 + j) * 8 + lr) * RCP + k];
#pragma unroll
      for (int i = 0; i < WM; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], av[i], bv[j]);
    }
  }
#pragma unroll
  for (int i = 0; i < WM; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int r = (mt0 + i) * 8 + lr, c = (nt0 + j) * 8 + 2 * lc;
      S.W[r * TNP + c] = acc[i][j][0];
      S.W[r * TNP + c + 1] = acc[i][j][1];
    }
  __syncthreads();
  // ---- W' = T^T W (T upper triangular) on DMMA: warp -> n-tile `warp` (its 8 columns of W), all
  //      NB_/8 m-tiles; A = T^T with the zero triangle masked, B = W(:, n-tile). Each warp reads
  //      and rewrites only its own columns, so no block barrier is needed in between.
  {
    static_assert(TN / 8 == 8, "one n-tile per warp (256 threads)");
    constexpr int MTT = NB_ / 8;
    double cw[MTT][2];
#pragma unroll
    for (int i = 0; i < MTT; ++i) cw[i][0] = cw[i][1] = 0.0;
    const int n8 = warp * 8;
#pragma unroll
    for (int kk = 0; kk < NB_ / 4; ++kk) {
      const int w = kk * 4 + lc;
      const double bv = S.W[w * TNP + n8 + lr];
#pragma unroll
      for (int i = 0; i < MTT; ++i) {
        const int u = i * 8 + lr;
        const double av = (w <= u) ? (kTrTsmem ? S.T[w * (NB_ + 1) + u]
                                               : (u < nb ? __ldg(Tg + (tq + w) * kQrTmax + tq + u) : 0.0))
                                   : 0.0;
        dmma_8x8x4(cw[i][0], cw[i][1], av, bv);
      }
    }
    __syncwarp();
#pragma unroll
    for (int i = 0; i < MTT; ++i) {
      const int r = i * 8 + lr, c = n8 + 2 * lc;
      S.W[r * TNP + c] = cw[i][0];
      S.W[r * TNP + c + 1] = cw[i][1];
    }
  }
  // ---- pass 2: A_tile -= V W' per 32-row chunk. Warp tile: 2 row-tiles x 2 col-tiles.
  const int rt0 = (warp & 1) * 2, ct0 = (warp >> 1) * 2;
  for (int q = nq; q < 2 * nq; ++q) {
    wait_chunk(q);
    __syncthreads();
    issue(q + kTrStages - 1);
    const int st = q % kTrStages;
    const int r0 = k0 + (2 * nq - 1 - q) * RC;
    fix_v(st, r0);
    __syncthreads();
    const double* Vs = S.V[st];
    double* As = S.A[st];
    double cf[2][2][2];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int r = (rt0 + i) * 8 + lr, c = (ct0 + j) * 8 + 2 * lc;
        cf[i][j][0] = As[c * RCP + r];
        cf[i][j][1] = As[(c + 1) * RCP + r];
      }
#pragma unroll
    for (int kk = 0; kk < NB_ / 4; ++kk) {
      const int u = kk * 4 + lc;
      double av[2], bv[2];
#pragma unroll
      for (int i = 0; i < 2; ++i) av[i] = -Vs[u * RCP + (rt0 + i) * 8 + lr];
#pragma unroll
      for (int j = 0; j < 2; ++j) bv[j] = S.W[u * TNP + (ct0 + j) * 8 + lr];
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) dmma_8x8x4(cf[i][j][0], cf[i][j][1], av[i], bv[j]);
    }
    // write the updated tile straight from the accumulators: per column, 8 consecutive rows
    // (64 B) per instruction; rows m..ld-1 stay zero (zero V and A rows there)
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int r = r0 + (rt0 + i) * 8 + lr, c = (ct0 + j) * 8 + 2 * lc;
        if (r < static_cast<int>(ld)) {
          if (c < ncols) A[static_cast<size_t>(c0 + c) * ld + r] = cf[i][j][0];
          if (c + 1 < ncols) A[static_cast<size_t>(c0 + c + 1) * ld + r] = cf[i][j][1];
        }
      }
  }
}

// ---- warp-specialised variant of the 32-wide trailing update (default): warp 8 is the TMA
// producer — it refills a ring stage as soon as the 8 compute warps have released it (per-stage
// "empty" mbarriers), so the compute warps never wait for one another at block barriers (only at
// the W / W' hand-over and at the one chunk whose V block gets its unit-triangular fix), and never
// execute the copy issue themselves.
template <int ST>
struct TrailWsSmem {
  static constexpr bool kTsmem = ST >= 3;  // 2 stages: T from L2 so that 3 CTAs fit an SM
  double V[ST][kQrNB * RCP];
  double A[ST][TN * RCP];
  double W[kQrNB * TNP];
  double T[kTsmem ? kQrNB * (kQrNB + 1) : 2];
  uint64_t full[ST], empty[ST];
};
constexpr int kWsCompute = 8;  // compute warps (256 threads); warp 8 produces

__device__ __forceinline__ void compute_sync() { asm volatile("bar.sync 1, 256;" ::: "memory"); }

template <int ST>
__global__ void __launch_bounds__(288, ST >= 3 ? 2 : 3)
    qr_trailing_ws_kernel(QrArgs a, int k0, int nbw, int cb, int ce, int tq, const __grid_constant__ CUtensorMap tmA,
                          const __grid_constant__ CUtensorMap tmV, int l2keep) {
  constexpr int NB_ = kQrNB, WM = 2;
  constexpr bool kTsmem = TrailWsSmem<ST>::kTsmem;
  extern __shared__ __align__(16) double smraw[];
  TrailWsSmem<ST>& S = *reinterpret_cast<TrailWsSmem<ST>*>(smraw);
  const int t = blockIdx.y;
  const int nb = nbw;
  const int c0 = cb + blockIdx.x * TN;
  if (c0 >= ce) return;
  const int ncols = min(TN, ce - c0);
  double* A = a.A + static_cast<size_t>(t) * a.ld * a.ncol;
  const size_t ld = a.ld;
  const int nq = (a.m - k0 + RC - 1) / RC;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int lr = lane >> 2, lc = lane & 3;
  if (threadIdx.x == 0) {
    for (int s2 = 0; s2 < ST; ++s2) {
      mbar_init(&S.full[s2], 1);
      mbar_init(&S.empty[s2], kWsCompute);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp == kWsCompute) {
    // producer: chunk q (pass 1 forward, pass 2 backward over the row chunks) into stage q % 3
    if (lane == 0) {
      const int colA = t * a.ncol + c0, colV = t * a.ncol + k0;
      // L2 priorities (l2keep >= 0): V is read by every column tile of the matrix (evict_last); of the
      // A tile, the last l2keep/1000 of pass 1's chunks are the first pass 2 re-reads (evict_last),
      // every other A chunk streams evict_first
      const uint64_t pol_last = l2_policy_evict_last(), pol_first = l2_policy_evict_first();
      for (int q = 0; q < 2 * nq; ++q) {
        const int st = q % ST;
        if (q >= ST) mbar_wait(&S.empty[st], static_cast<uint32_t>(((q / ST) - 1) & 1));
        const int cq = q < nq ? q : 2 * nq - 1 - q;
        const int row = k0 + cq * RC;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&S.full[st], static_cast<uint32_t>((TN + NB_) * RCP * sizeof(double)));
        if (l2keep < 0) {
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                  smem_u32(S.A[st])),
              "l"(&tmA), "r"(row), "r"(colA), "r"(smem_u32(&S.full[st]))
              : "memory");
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                  smem_u32(S.V[st])),
              "l"(&tmV), "r"(row), "r"(colV), "r"(smem_u32(&S.full[st]))
              : "memory");
        } else {
          const bool keep = q < nq && 1000 * (q + 1) > (1000 - l2keep) * nq;
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(
                  smem_u32(S.A[st])),
              "l"(&tmA), "r"(row), "r"(colA), "r"(smem_u32(&S.full[st])), "l"(keep ? pol_last : pol_first)
              : "memory");
          asm volatile(
              "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(
                  smem_u32(S.V[st])),
              "l"(&tmV), "r"(row), "r"(colV), "r"(smem_u32(&S.full[st])), "l"(pol_last)
              : "memory");
        }
      }
    }
    return;
  }
  auto wait_full = [&](int q) { mbar_wait(&S.full[q % ST], static_cast<uint32_t>((q / ST) & 1)); };
  auto release = [&](int q) {
    __syncwarp();
    if (lane == 0) mbar_arrive(&S.empty[q % ST]);
  };
  // the unit lower-triangular structure of V lives in the chunk holding rows k0 .. k0 + nb - 1
  auto fix_v = [&](int st, int r0) {
    for (int idx = threadIdx.x; idx < NB_ * RC; idx += kWsCompute * 32) {
      const int u = idx / RC, k = idx % RC;
      const int row = r0 + k;
      if (row <= k0 + u) S.V[st][u * RCP + k] = (row == k0 + u && u < nb) ? 1.0 : 0.0;
    }
  };
  const double* Tg = a.T + static_cast<size_t>(t) * kQrTmax * kQrTmax;
  // T (needed only after pass 1): loaded into registers now, stored to shared memory after pass 1,
  // so the compute warps do not wait on these L2 loads before their first DMMA
  constexpr int kTPer = NB_ * NB_ / (kWsCompute * 32);
  double treg[kTPer];
  if (kTsmem)
#pragma unroll
    for (int q = 0; q < kTPer; ++q) {
      const int idx = threadIdx.x + q * kWsCompute * 32;
      const int i = idx / NB_, j = idx % NB_;
      treg[q] = (i < nb && j < nb) ? Tg[(tq + i) * kQrTmax + tq + j] : 0.0;
    }
  // ---- pass 1: W = V^T A_tile; warp -> m-tiles {2(w&1), +1}, n-tiles {2(w>>1), +1}
  const int mt0 = (warp & 1) * WM, nt0 = (warp >> 1) * 2;
  double acc[WM][2][2];
#pragma unroll
  for (int i = 0; i < WM; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  for (int q = 0; q < nq; ++q) {
    const int st = q % ST;
    wait_full(q);
    if (q == 0) {  // rows k0 .. k0 + 31 hold the reflectors' diagonal and the R entries above it
      fix_v(st, k0);
      compute_sync();
    }
    const double* Vs = S.V[st];
    const double* As = S.A[st];
#pragma unroll
    for (int kk = 0; kk < RC / 4; ++kk) {
      const int k = kk * 4 + lc;
      double av[WM], bv[2];
#pragma unroll
      for (int i = 0; i < WM; ++i) av[i] = Vs[((mt0 + i) * 8 + lr) * RCP + k];
#pragma unroll
      for (int j = 0; j < 2; ++j) bv[j] = As[((nt0 + j) * 8 + lr) * RCP + k];
#pragma unroll
      for (int i = 0; i < WM; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) dmma_8x8x4(acc[i][j][0], acc[i][j][1], av[i], bv[j]);
    }
    release(q);
  }
#pragma unroll
  for (int i = 0; i < WM; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      const int r = (mt0 + i) * 8 + lr, c = (nt0 + j) * 8 + 2 * lc;
      S.W[r * TNP + c] = acc[i][j][0];
      S.W[r * TNP + c + 1] = acc[i][j][1];
    }
  if (kTsmem)
#pragma unroll
    for (int q = 0; q < kTPer; ++q) {
      const int idx = threadIdx.x + q * kWsCompute * 32;
      S.T[(idx / NB_) * (NB_ + 1) + idx % NB_] = treg[q];
    }
  compute_sync();
  // ---- W' = T^T W: warp -> its 8 columns, all m-tiles
  {
    constexpr int MTT = NB_ / 8;
    double cw[MTT][2];
#pragma unroll
    for (int i = 0; i < MTT; ++i) cw[i][0] = cw[i][1] = 0.0;
    const int n8 = warp * 8;
#pragma unroll
    for (int kk = 0; kk < NB_ / 4; ++kk) {
      const int w = kk * 4 + lc;
      const double bv = S.W[w * TNP + n8 + lr];
#pragma unroll
      for (int i = 0; i < MTT; ++i) {
        const int u = i * 8 + lr;
        const double av = (w <= u) ? (kTsmem ? S.T[w * (NB_ + 1) + u]
                                             : (u < nb ? __ldg(Tg + (tq + w) * kQrTmax + tq + u) : 0.0))
                                   : 0.0;
        dmma_8x8x4(cw[i][0], cw[i][1], av, bv);
      }
    }
    __syncwarp();
#pragma unroll
    for (int i = 0; i < MTT; ++i) {
      const int r = i * 8 + lr, c = n8 + 2 * lc;
      S.W[r * TNP + c] = cw[i][0];
      S.W[r * TNP + c + 1] = cw[i][1];
    }
  }
  compute_sync();
  // ---- pass 2: A_tile -= V W' per 32-row chunk (rows walked backwards: the chunks pass 1 read
  //      last are still in L2); warp tile 2 row-tiles x 2 col-tiles
  const int rt0 = (warp & 1) * 2, ct0 = (warp >> 1) * 2;
  for (int q = nq; q < 2 * nq; ++q) {
    const int st = q % ST;
    const int r0 = k0 + (2 * nq - 1 - q) * RC;
    wait_full(q);
    if (q == 2 * nq - 1) {
      fix_v(st, r0);
      compute_sync();
    }
    const double* Vs = S.V[st];
    const double* As = S.A[st];
    double cf[2][2][2];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int r = (rt0 + i) * 8 + lr, c = (ct0 + j) * 8 + 2 * lc;
        cf[i][j][0] = As[c * RCP + r];
        cf[i][j][1] = As[(c + 1) * RCP + r];
      }
#pragma unroll
    for (int kk = 0; kk < NB_ / 4; ++kk) {
      const int u = kk * 4 + lc;
      double av[2], bv[2];
#pragma unroll
      for (int i = 0; i < 2; ++i) av[i] = -Vs[u * RCP + (rt0 + i) * 8 + lr];
#pragma unroll
      for (int j = 0; j < 2; ++j) bv[j] = S.W[u * TNP + (ct0 + j) * 8 + lr];
#pragma unroll
      for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) dmma_8x8x4(cf[i][j][0], cf[i][j][1], av[i], bv[j]);
    }
    release(q);
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int r = r0 + (rt0 + i) * 8 + lr, c = (ct0 + j) * 8 + 2 * lc;
        if (r < static_cast<int>(ld)) {
          if (c < ncols) A[static_cast<size_t>(c0 + c) * ld + r] = cf[i][j][0];
          if (c + 1 < ncols) A[static_cast<size_t>(c0 + c + 1) * ld + r] = cf[i][j][1];
        }
      }
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

namespace {
/// TMA descriptor of the batched matrices as one 2-D tensor (rows = ld, columns = ncol * nmat,
/// column stride ld doubles) with a (RCP rows x cols) box: the trailing update's chunk loads.
CUtensorMap trailing_tensor_map(const QrArgs& a, int cols) {
  static PFN_cuTensorMapEncodeTiled encode = nullptr;
  if (!encode) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q{};
    DDG_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    if (!fn || q != cudaDriverEntryPointSuccess) throw CudaError("cuTensorMapEncodeTiled unavailable");
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled>(fn);
  }
  CUtensorMap m;
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(a.ld), static_cast<cuuint64_t>(a.ncol) * a.nmat};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(a.ld) * sizeof(double)};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(RCP), static_cast<cuuint32_t>(cols)};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, a.A, dims, strides, box, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed (" + std::to_string(static_cast<int>(r)) + ")");
  return m;
}
}  // namespace

std::vector<QrOp> qr_schedule(int M, int ncol) {
  // 64-wide blocks: panel (32) -> update the right 32 panel columns -> panel (32, + T12) ->
  // 64-wide trailing update of the rest; a block of at most 32 columns is a plain 32 step
  std::vector<QrOp> ops;
  const char* e = std::getenv("DDELM_QR_NB");
  // 32-wide blocking by default: measured faster than the recursive 64-wide blocks on B200 (the
  // 64-wide DMMA tile needs 180 KB of staging -> 1 CTA / SM); DDELM_QR_NB=64 selects them
  const int bw = (e && std::atoi(e) == 64) ? 64 : NB;
  for (int k0 = 0; k0 < M; k0 += bw) {
    const int w = std::min(bw, M - k0);
    if (w <= NB) {
      const int tq = (k0 / NB) % 2 * NB;  // alternate T quadrants (look-ahead overlaps panels)
      ops.push_back({QrOp::kPanel, k0, 0, 0, 0, tq, 0});
      ops.push_back({QrOp::kTrail32, k0, w, k0 + w, ncol, tq, 0});
      continue;
    }
    ops.push_back({QrOp::kPanel, k0, 0, 0, 0, 0, 0});
    ops.push_back({QrOp::kTrail32, k0, NB, k0 + NB, k0 + w, 0, 0});
    ops.push_back({QrOp::kPanel, k0 + NB, 0, 0, 0, NB, 1});
    ops.push_back({QrOp::kTrail64, k0, w, k0 + w, ncol, 0, 0});
  }
  return ops;
}

void launch_qr_op(const QrArgs& a, const QrOp& op, cudaStream_t st) {
  if (op.kind == QrOp::kPanel) {
    // shared-memory resident panel when an 8-column sub-panel of all m - k0 rows fits
    static int smem_static = -1, smem_optin = 0;
    static bool use_smem = true;
    if (smem_static < 0) {
      cudaFuncAttributes fa{};
      DDG_CUDA(cudaFuncGetAttributes(&fa, qr_panel_smem_kernel));
      smem_static = static_cast<int>(fa.sharedSizeBytes);
      int dev = 0;
      DDG_CUDA(cudaGetDevice(&dev));
      DDG_CUDA(cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
      DDG_CUDA(cudaFuncSetAttribute(qr_panel_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    smem_optin - smem_static));
      DDG_CUDA(cudaFuncSetAttribute(qr_panel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(kFinishDoubles * sizeof(double))));
      const char* e = std::getenv("DDELM_QR_PANEL");
      use_smem = !(e && std::string(e) == "stream");
    }
    const int rows = a.m - op.k0;
    const int lds = ((rows + 27) / 32) * 32 + 4;  // >= rows, = 4 (mod 32): conflict-free DMMA fragments
    const size_t smem = std::max<size_t>(static_cast<size_t>(kSub) * lds, kFinishDoubles) * sizeof(double);
    if (use_smem && smem + smem_static <= static_cast<size_t>(smem_optin)) {
      qr_panel_smem_kernel<<<a.nmat, kPanelThreads, smem, st>>>(a, op.k0, op.toff, op.combine, lds);
    } else {
      qr_panel_kernel<<<a.nmat, kPanelThreads, kFinishDoubles * sizeof(double), st>>>(a, op.k0, op.toff, op.combine);
    }
    DDG_LAUNCH_CHECK();
    return;
  }
  const int rest = op.ce - op.cb;
  if (rest <= 0) return;
  dim3 grid(ceil_div(rest, TN), a.nmat);
  const CUtensorMap tmA = trailing_tensor_map(a, TN), tmV = trailing_tensor_map(a, op.kind == QrOp::kTrail32 ? 32 : 64);
  // ring depth of the 32-wide update: 3 stages (2 CTAs / SM) by default, DDELM_QR_STAGES=2 for
  // 2 stages with T in L2 (3 CTAs / SM)
  static const int stages = [] {
    const char* e = std::getenv("DDELM_QR_STAGES");
    return (e && std::atoi(e) == 2) ? 2 : 3;
  }();
  auto launch = [&](auto kern, size_t smem, int toff) {
    DDG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    kern<<<grid, 256, smem, st>>>(a, op.k0, op.nbw, op.cb, op.ce, toff, tmA, tmV);
  };
  // DDELM_QR_L2KEEP: per mille of pass 1's A chunks kept evict_last for pass 2 (-1: no L2 hints)
  static const int l2keep = [] {
    const char* e = std::getenv("DDELM_QR_L2KEEP");
    return e ? std::max(-1, std::min(1000, std::atoi(e))) : -1;
  }();
  static const bool ws = [] {
    const char* e = std::getenv("DDELM_QR_WS");
    return !(e && std::atoi(e) == 0);
  }();
  if (op.kind == QrOp::kTrail32 && ws) {
    auto launch_ws = [&](auto kern, size_t smem) {
      DDG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
      kern<<<grid, 288, smem, st>>>(a, op.k0, op.nbw, op.cb, op.ce, op.toff, tmA, tmV, l2keep);
    };
    if (stages == 2) launch_ws(qr_trailing_ws_kernel<2>, sizeof(TrailWsSmem<2>));
    else launch_ws(qr_trailing_ws_kernel<3>, sizeof(TrailWsSmem<3>));
  } else if (op.kind == QrOp::kTrail32) {
    if (stages == 2) launch(qr_trailing_kernel<32, 2>, sizeof(TrailSmem<32, 2>), op.toff);
    else launch(qr_trailing_kernel<32, 3>, sizeof(TrailSmem<32, 3>), op.toff);
  } else {
    launch(qr_trailing_kernel<64, 3>, sizeof(TrailSmem<64, 3>), 0);
  }
  DDG_LAUNCH_CHECK();
}

void qr_factor(const QrArgs& a, cudaStream_t main, cudaStream_t side, std::vector<cudaEvent_t>& ev) {
  // Look-ahead blocked QR on two streams: after panel p, the next panel's 32 columns are updated
  // first (main stream), so panel p+1 can start while the rest of the trailing update of panel p
  // runs on the side stream. Dependencies (events): T_rest(p) needs panel p; the next-panel update
  // T_next(p+1) needs T_rest(p) (same columns, reflectors applied in order).
  // Off by default: measured no overlap on B200 (a 512-thread panel CTA needs a whole SM's
  // registers, so it cannot co-reside with trailing CTAs) and ~2% slower; DDELM_QR_LOOKAHEAD=1.
  const char* e = std::getenv("DDELM_QR_LOOKAHEAD");
  const bool off = !(e && std::atoi(e) == 1) || side == nullptr;
  const char* nbe = std::getenv("DDELM_QR_NB");
  if (off || (nbe && std::atoi(nbe) == 64)) {
    for (const QrOp& op : qr_schedule(a.M, a.ncol)) launch_qr_op(a, op, main);
    return;
  }
  const int np = (a.M + NB - 1) / NB;
  while (static_cast<int>(ev.size()) < 2 * np + 1) {
    cudaEvent_t x;
    DDG_CUDA(cudaEventCreateWithFlags(&x, cudaEventDisableTiming));
    ev.push_back(x);
  }
  cudaEvent_t start = ev[2 * np];
  DDG_CUDA(cudaEventRecord(start, main));
  DDG_CUDA(cudaStreamWaitEvent(side, start, 0));
  for (int p = 0; p < np; ++p) {
    const int k0 = p * NB, nb = std::min(NB, a.M - k0);
    const int nbn = std::min(NB, std::max(0, a.M - (k0 + nb)));  // next panel width
    // T factors alternate between two quadrants: panel p+1 writes its T while T_rest(p), still
    // running on the side stream, reads panel p's
    const int tq = (p % 2) * NB;
    if (p > 1) DDG_CUDA(cudaStreamWaitEvent(main, ev[2 * p - 3], 0));  // T_rest(p-2) read quadrant tq
    launch_qr_op(a, QrOp{QrOp::kPanel, k0, 0, 0, 0, tq, 0}, main);
    DDG_CUDA(cudaEventRecord(ev[2 * p], main));
    if (p > 0) DDG_CUDA(cudaStreamWaitEvent(main, ev[2 * p - 1], 0));  // T_rest(p-1) done
    if (nbn > 0) launch_qr_op(a, QrOp{QrOp::kTrail32, k0, nb, k0 + nb, k0 + nb + nbn, tq, 0}, main);
    DDG_CUDA(cudaStreamWaitEvent(side, ev[2 * p], 0));
    launch_qr_op(a, QrOp{QrOp::kTrail32, k0, nb, k0 + nb + nbn, a.ncol, tq, 0}, side);
    DDG_CUDA(cudaEventRecord(ev[2 * p + 1], side));
  }
  DDG_CUDA(cudaStreamWaitEvent(main, ev[2 * np - 1], 0));
}

double qr_op_flops(const QrArgs& a, const QrOp& op) {
  const double mrows = a.m - op.k0;
  if (op.kind == QrOp::kPanel) {
    const double nb = std::min(NB, a.M - op.k0);
    return a.nmat * 2.0 * mrows * nb * nb;
  }
  return a.nmat * 4.0 * mrows * op.nbw * std::max(0, op.ce - op.cb);  // W = V^T A, A -= V (T^T W)
}

void launch_qr_diag_ratio(const QrArgs& a, double* ratio, cudaStream_t st) {
  qr_diag_ratio_kernel<<<a.nmat, 256, 0, st>>>(a, ratio);
  DDG_LAUNCH_CHECK();
}

}  // namespace ddg

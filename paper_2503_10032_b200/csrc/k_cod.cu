// Rank-revealing branch of LsFactor on the device (sm_100a, fp64).
//
// Reference: solvers.cpp:32-41 — when the unpivoted R diagonal signals deficiency, Eigen's
// CompleteOrthogonalDecomposition (column-pivoted Householder QR with max-norm pivoting,
// first-index ties, LAPACK-style norm downdating with recomputation below sqrt(eps);
// rank = #{|R_ii| > tol * max|R_ii|}; RZ of [R11 R12]) yields K^+ = P Z^T [T^{-1}; 0] Q_r^T.
//
// B200 design: column norms and pivots of K equal those of its R-factor R0 (K = Q0 R0), so the
// pivoted factorisation runs on the M x M upper-triangular R0 produced by the batched QR,
// never touching the m x M matrix again. It is blocked LAPACK-dlaqps style (no trailing
// update: the updated matrix is A - V F^T, F accumulated one column per step), one CTA per
// matrix, and stops as soon as every remaining column norm is below half the rank
// threshold, i.e. after ~rank steps instead of M. Outputs, per matrix:
//   C      = P Z^T [I_r; 0] T^{-1}   (M x r)      so that  K^+ = C Q_r^T
//   QtX    = Q_r^T [f | E]           (r x ext)    (Q_r = Q0 Q1[:, :r])
// The full-rank branch (solvers.cpp:43-44) is the same contract with r = M, C = R0^{-1}.
#ifndef DDG_COD_FBATCH
#define DDG_COD_FBATCH 16
#endif
#ifndef DDG_COD_GEMV_ROWS
#define DDG_COD_GEMV_ROWS 8
#endif
#include <algorithm>
#include <cfloat>
#include <cstdlib>

#include "common.cuh"
#include "kernels.hpp"

namespace ddg {

namespace {

constexpr double kRowTruncation = 1e-14;  // R0 rows with tail energy below this x ||R0||_F are dropped
constexpr int kNPL = 32;  // register rows per lane in the finish kernel: M <= 32 * 32

struct ArgMax {
  double v;
  int i;
};

__device__ __forceinline__ ArgMax better(ArgMax a, ArgMax b) {
  if (b.v > a.v || (b.v == a.v && b.i < a.i)) return b;
  return a;
}

__device__ ArgMax block_argmax(ArgMax x, ArgMax* sh) {
  for (int o = 16; o > 0; o >>= 1) {
    ArgMax y{__shfl_xor_sync(0xffffffffu, x.v, o), __shfl_xor_sync(0xffffffffu, x.i, o)};
    x = better(x, y);
  }
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __syncthreads();
  if (lane == 0) sh[w] = x;
  __syncthreads();
  if (w == 0) {
    ArgMax y = lane < nw ? sh[lane] : ArgMax{-1.0, 0x7fffffff};
    for (int o = 16; o > 0; o >>= 1) {
      ArgMax z{__shfl_xor_sync(0xffffffffu, y.v, o), __shfl_xor_sync(0xffffffffu, y.i, o)};
      y = better(y, z);
    }
    if (lane == 0) sh[0] = y;
  }
  __syncthreads();
  ArgMax r = sh[0];
  __syncthreads();
  return r;
}

__global__ void __launch_bounds__(512) cod_pivqr_kernel(CodArgs a, int t0) {
  const int t = t0 + blockIdx.x;
  const int M = a.M, K = a.kmax;
  const double mn = a.ratio[2 * t], mx = a.ratio[2 * t + 1];
  const bool deficient = !(mx > 0) || mn < a.rank_tol * mx;  // solvers.cpp:32
  if (threadIdx.x == 0) {
    a.deficient[t] = deficient ? 1 : 0;
    a.status[t] = 0;
  }
  if (!deficient) {
    if (threadIdx.x == 0) a.rank[t] = M;
    return;
  }
  const double* R0 = a.A + static_cast<size_t>(t) * a.ld * a.ncol;
  const size_t ld = a.ld;
  double* V1 = a.V1 + static_cast<size_t>(t) * K * M;
  double* F1 = a.F1 + static_cast<size_t>(t) * M * K;
  double* Rr = a.Rr + static_cast<size_t>(t) * K * M;
  double* tau1 = a.tau1 + static_cast<size_t>(t) * K;

  extern __shared__ double sm[];
  double* v = sm;            // M  (pivot column, then the reflector)
  double* w = v + M;         // K
  double* vk = w + K;        // K  (row k of V)
  double* upd = vk + K;          // M  updated column norms (by position)
  double* dir = upd + M;         // M  norms at the last exact computation (-1: recompute)
  double* gs = dir + M;          // M  A(k:, j)^T v of the current step
  int* flist = reinterpret_cast<int*>(gs + M);  // M
  int* perm = flist + M;                        // M
  int* permg = a.perm + static_cast<size_t>(t) * M;
  __shared__ int wcnt[32], woff[32];
  __shared__ int s_nflag;
  __shared__ double red[32];
  __shared__ ArgMax ared[32];
  __shared__ double s_tau, s_maxpivot;
  __shared__ int s_stop;
  // DDELM_COD_TRACE: per-section device time of the pivot steps (thread 0's clock, barrier-bounded)
  __shared__ unsigned long long s_tr[9], s_nfl;
  auto stamp = [&](int sec) {
    if (a.trace != nullptr && threadIdx.x == 0) {
      unsigned long long now;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
      if (sec >= 0) s_tr[sec] += now - s_tr[8];
      s_tr[8] = now;
    }
  };
  if (a.trace != nullptr && threadIdx.x == 0)
    for (int q = 0; q < 9; ++q) s_tr[q] = s_nfl = 0;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  const double eps = DBL_EPSILON;
  const double downdate_thr = sqrt(eps);
  // F is stored transposed, F1[u*M + j] (reflector u, column position j): every per-column pass
  // below reads it coalesced across threads

  // ---- effective row count of R0: rows whose tail energy ||R0(i:, i:)||_F is below
  //      kRowTruncation * ||R0||_F carry only round-off (the numerical rank is ~70 of M = 800), so
  //      the pivoted factorisation reads rows < Reff only — a perturbation of the column norms far
  //      below the rank threshold (1e-10 |R_00|), the regime of the oracle's own 1-ulp spread
  __shared__ int s_reff;
  {
    double* rowsq = v;  // scratch (M)
    for (int i = threadIdx.x; i < M; i += blockDim.x) {
      double s = 0;
      for (int j = i; j < M; ++j) {
        const double e = R0[static_cast<size_t>(j) * ld + i];
        s += e * e;
      }
      rowsq[i] = s;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double tot = 0;
      for (int i = 0; i < M; ++i) tot += rowsq[i];
      const double lim = kRowTruncation * kRowTruncation * tot;
      double tail = 0;
      int reff = M;
      for (int i = M - 1; i >= 1; --i) {
        tail += rowsq[i];
        if (tail > lim) break;
        reff = i;
      }
      s_reff = reff;
      a.reff[t] = reff;
    }
    __syncthreads();
  }
  const int Reff = s_reff;
  // initial column norms (of R0 = of K up to rounding)
  for (int j = warp; j < M; j += nwarp) {
    double s = 0;
    for (int i = lane; i <= min(j, Reff - 1); i += 32) {
      const double e = R0[static_cast<size_t>(j) * ld + i];
      s += e * e;
    }
    s = warp_sum(s);
    if (lane == 0) {
      upd[j] = dir[j] = sqrt(s);
      perm[j] = j;
    }
  }
  if (threadIdx.x == 0) {
    s_maxpivot = 0;
    s_stop = 0;
  }
  __syncthreads();

  int k = 0;
  stamp(-1);
  for (; k < M; ++k) {
    // ---- pivot: largest updated norm, first index on ties
    ArgMax best{-1.0, 0x7fffffff};
    for (int j = k + threadIdx.x; j < M; j += blockDim.x) best = better(best, ArgMax{upd[j], j});
    best = block_argmax(best, ared);
    if (k > 0 && best.v < 0.5 * a.rank_tol * s_maxpivot) break;
    if (k >= K) {
      if (threadIdx.x == 0) a.status[t] = 1;
      break;
    }
    const int p = best.i;
    if (p != k) {
      if (threadIdx.x == 0) {
        double tmp = upd[k]; upd[k] = upd[p]; upd[p] = tmp;
        tmp = dir[k]; dir[k] = dir[p]; dir[p] = tmp;
        const int ti = perm[k]; perm[k] = perm[p]; perm[p] = ti;
      }
      for (int u = threadIdx.x; u < k; u += blockDim.x) {
        double tmp = F1[static_cast<size_t>(u) * M + k];
        F1[static_cast<size_t>(u) * M + k] = F1[static_cast<size_t>(u) * M + p];
        F1[static_cast<size_t>(u) * M + p] = tmp;
        tmp = Rr[static_cast<size_t>(u) * M + k];
        Rr[static_cast<size_t>(u) * M + k] = Rr[static_cast<size_t>(u) * M + p];
        Rr[static_cast<size_t>(u) * M + p] = tmp;
      }
    }
    __syncthreads();
    stamp(0);
    // ---- updated pivot column (rows k..M-1): R0(:, perm[k]) - V F(k, :)^T
    const int ck = perm[k];
    for (int u = threadIdx.x; u < k; u += blockDim.x) w[u] = F1[static_cast<size_t>(u) * M + k];
    __syncthreads();
    for (int i = k + threadIdx.x; i < M; i += blockDim.x) {
      double s = 0.0;
      if (i < Reff) {
        s = (i <= ck) ? R0[static_cast<size_t>(ck) * ld + i] : 0.0;
#pragma unroll 8
        for (int u = 0; u < k; ++u) s -= V1[static_cast<size_t>(u) * M + i] * w[u];
      }
      v[i] = s;
    }
    __syncthreads();
    stamp(1);
    // ---- Householder (makeHouseholderInPlace)
    double part = 0;
    for (int i = k + 1 + threadIdx.x; i < Reff; i += blockDim.x) part += v[i] * v[i];
    const double tail = block_sum(part, red);
    const double alpha = v[k];
    double tau = 0, beta = alpha, scale = 0;
    const bool triv = !(tail > DBL_MIN);
    if (!triv) {
      beta = sqrt(alpha * alpha + tail);
      if (alpha >= 0) beta = -beta;
      scale = 1.0 / (alpha - beta);
      tau = (beta - alpha) / beta;
    }
    for (int i = threadIdx.x; i < M; i += blockDim.x) {
      double e;
      if (i < k) e = 0.0;
      else if (i == k) e = 1.0;
      else e = triv ? 0.0 : v[i] * scale;
      if (i >= k) v[i] = e;
      V1[static_cast<size_t>(k) * M + i] = e;
    }
    if (threadIdx.x == 0) {
      Rr[static_cast<size_t>(k) * M + k] = beta;
      tau1[k] = tau;
      s_tau = tau;
      s_maxpivot = fmax(s_maxpivot, fabs(beta));
    }
    __syncthreads();
    stamp(2);
    // ---- w = V(:, 0:k)^T v ; vk = V(k, 0:k]
    for (int u = warp; u < k; u += nwarp) {
      double s = 0;
#pragma unroll 8
      for (int i = k + lane; i < Reff; i += 32) s += V1[static_cast<size_t>(u) * M + i] * v[i];
      s = warp_sum(s);
      if (lane == 0) w[u] = s;
    }
    for (int u = threadIdx.x; u <= k; u += blockDim.x) vk[u] = V1[static_cast<size_t>(u) * M + k];
    // ---- g_j = A(k:, j)^T v for positions j > k (the original R0 columns: the dlaqps GEMV, the
    //      only pass over R0 per step): a warp per 4 columns, lanes over rows
    for (int j0 = k + 1 + 4 * warp; j0 < M; j0 += 4 * nwarp) {
      const double* col[4];
      int iend[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int j = min(j0 + q, M - 1);
        const int cj = perm[j];
        col[q] = R0 + static_cast<size_t>(cj) * ld;
        iend[q] = (j0 + q < M) ? min(cj, Reff - 1) : k - 1;
      }
      const int imax = max(max(iend[0], iend[1]), max(iend[2], iend[3]));
      double g[4] = {0, 0, 0, 0};
      constexpr int kU = DDG_COD_GEMV_ROWS;  // rows per lane per batch: 4 kU independent loads in flight
      for (int i0 = k + lane; i0 <= imax; i0 += 32 * kU) {
        double x[kU][4], vv[kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const int i = i0 + 32 * u;
          vv[u] = i <= imax ? v[i] : 0.0;
#pragma unroll
          for (int q = 0; q < 4; ++q) x[u][q] = i <= iend[q] ? __ldcs(col[q] + i) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < kU; ++u)
#pragma unroll
          for (int q = 0; q < 4; ++q) g[q] += x[u][q] * vv[u];
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const double gg = warp_sum(g[q]);
        if (lane == 0 && j0 + q < M) gs[j0 + q] = gg;
      }
    }
    __syncthreads();
    stamp(3);
    // ---- per column position j > k (thread per j, coalesced over F1[u*M + j]):
    //      F(j, k) = tau (g_j - F(j, 0:k) w), row k of R: R(k, j) = R0(k, cj) - F(j, 0:k] . V(k, 0:k],
    //      and the LAPACK norm downdate (flag for exact recomputation below sqrt(eps))
    int any_flag = 0;
    for (int j = k + 1 + threadIdx.x; j < M; j += blockDim.x) {
      const int cj = perm[j];
      double fw = 0, fv = 0;
      int u = 0;
      constexpr int kF = DDG_COD_FBATCH;  // loads in flight per thread (same summation order)
      for (; u + kF <= k; u += kF) {
        double f[kF];
#pragma unroll
        for (int q = 0; q < kF; ++q) f[q] = F1[static_cast<size_t>(u + q) * M + j];
#pragma unroll
        for (int q = 0; q < kF; ++q) {
          fw += f[q] * w[u + q];
          fv += f[q] * vk[u + q];
        }
      }
      for (; u < k; ++u) {
        const double f = F1[static_cast<size_t>(u) * M + j];
        fw += f * w[u];
        fv += f * vk[u];
      }
      const double fk = s_tau * (gs[j] - fw);
      F1[static_cast<size_t>(k) * M + j] = fk;
      const double rkj = ((k <= cj) ? R0[static_cast<size_t>(cj) * ld + k] : 0.0) - fv - vk[k] * fk;
      Rr[static_cast<size_t>(k) * M + j] = rkj;
      if (upd[j] != 0.0) {
        double tmp = fabs(rkj) / upd[j];
        tmp = (1.0 + tmp) * (1.0 - tmp);
        if (tmp < 0) tmp = 0;
        const double ratio = upd[j] / dir[j];
        const double tmp2 = tmp * ratio * ratio;
        if (tmp2 <= downdate_thr) {
          dir[j] = -1.0;  // flag: recompute exactly below
          any_flag = 1;
        } else {
          upd[j] *= sqrt(tmp);
        }
      }
    }
    const int flagged = __syncthreads_or(any_flag);
    stamp(4);
    if (!flagged) continue;
    // ---- exact recomputation of flagged norms: ||(A - V F^T)(k+1:M, j)||
    // compact the flagged columns (increasing j)
    if (threadIdx.x == 0) s_nflag = 0;
    __syncthreads();
    for (int base = k + 1; base < M; base += blockDim.x) {
      const int j = base + threadIdx.x;
      const bool fl = j < M && dir[j] == -1.0;
      const unsigned bal = __ballot_sync(0xffffffffu, fl);
      if (lane == 0) wcnt[warp] = __popc(bal);
      __syncthreads();
      if (threadIdx.x == 0) {
        int s = s_nflag;
        for (int w2 = 0; w2 < nwarp; ++w2) {
          woff[w2] = s;
          s += wcnt[w2];
        }
        s_nflag = s;
      }
      __syncthreads();
      if (fl) flist[woff[warp] + __popc(bal & ((1u << lane) - 1u))] = j;
      __syncthreads();
    }
    const int nflag = s_nflag;
    stamp(6);
    if (a.trace != nullptr && threadIdx.x == 0) s_nfl += nflag + 1000000ull;
    // E = R0(k+1:Reff, flagged) - V(k+1:Reff, 0:k] F(flagged, 0:k]^T on DMMA, 8 x 8 tiles
    // (rows x flagged columns): the warps split the column groups and, when there are fewer
    // than 16 groups, the row tiles too; per-warp partial squares are combined in a fixed order
    const int ncg = (nflag + 7) >> 3;
    const int rg = max(1, min(ncg >= nwarp ? 1 : nwarp / ncg, M / nflag));  // row groups per column group
    const int nrt = (Reff - (k + 1) + 7) >> 3;
    for (int wt = warp; wt < ncg * rg; wt += nwarp) {
      const int g = wt / rg, q = wt % rg;  // column group, row group
      const int f0 = 8 * g;
      const int lr = lane >> 2, lc = lane & 3;
      const int cb = f0 + lr;
      const int jb = cb < nflag ? flist[cb] : -1;
      const int c0 = f0 + 2 * lc;
      const int cjo0 = c0 < nflag ? perm[flist[c0]] : -1, cjo1 = c0 + 1 < nflag ? perm[flist[c0 + 1]] : -1;
      double sq0 = 0.0, sq1 = 0.0;
      // kRB row tiles per batch and kKS k-steps (4 reflectors each) per iteration, every load
      // first: the F fragments are shared by the batch's tiles, so a recomputation costs
      // ~k / (4 kKS) L2 round trips per batch instead of one per tile and k-step; per tile the
      // DMMA k order and the row-tile order of the squares are unchanged
      constexpr int kRB = 4, kKS = 4;
      for (int rb = q; rb < nrt; rb += rg * kRB) {
        double o[kRB][2];
#pragma unroll
        for (int x = 0; x < kRB; ++x) o[x][0] = o[x][1] = 0.0;
        for (int u0 = 0; u0 <= k; u0 += 4 * kKS) {
          double bf[kKS], av[kKS][kRB];
#pragma unroll
          for (int ks = 0; ks < kKS; ++ks) {
            const int ua = u0 + 4 * ks + lc;
            bf[ks] = (ua <= k && jb >= 0) ? F1[static_cast<size_t>(ua) * M + jb] : 0.0;
#pragma unroll
            for (int x = 0; x < kRB; ++x) {
              const int rt = rb + x * rg;
              const int ia = k + 1 + 8 * rt + lr;
              av[ks][x] = (rt < nrt && ia < Reff && ua <= k) ? V1[static_cast<size_t>(ua) * M + ia] : 0.0;
            }
          }
#pragma unroll
          for (int ks = 0; ks < kKS; ++ks)
#pragma unroll
            for (int x = 0; x < kRB; ++x) dmma_8x8x4(o[x][0], o[x][1], av[ks][x], bf[ks]);
        }
#pragma unroll
        for (int x = 0; x < kRB; ++x) {
          const int rt = rb + x * rg;
          const int i = k + 1 + 8 * rt + lr;
          if (rt < nrt && i < Reff) {
            const double e0 = (cjo0 >= 0 && i <= cjo0 ? R0[static_cast<size_t>(cjo0) * ld + i] : 0.0) - o[x][0];
            const double e1 = (cjo1 >= 0 && i <= cjo1 ? R0[static_cast<size_t>(cjo1) * ld + i] : 0.0) - o[x][1];
            sq0 += e0 * e0;
            sq1 += e1 * e1;
          }
        }
      }
      sq0 += __shfl_xor_sync(0xffffffffu, sq0, 4);
      sq0 += __shfl_xor_sync(0xffffffffu, sq0, 8);
      sq0 += __shfl_xor_sync(0xffffffffu, sq0, 16);
      sq1 += __shfl_xor_sync(0xffffffffu, sq1, 4);
      sq1 += __shfl_xor_sync(0xffffffffu, sq1, 8);
      sq1 += __shfl_xor_sync(0xffffffffu, sq1, 16);
      if (lr == 0) {  // partial of row group q for columns c0, c0 + 1 (rg * nflag <= M entries)
        if (c0 < nflag) gs[q * nflag + c0] = sq0;
        if (c0 + 1 < nflag) gs[q * nflag + c0 + 1] = sq1;
      }
    }
    __syncthreads();
    stamp(7);
    for (int c = threadIdx.x; c < nflag; c += blockDim.x) {
      double t2 = 0;
      for (int q = 0; q < rg; ++q) t2 += gs[q * nflag + c];
      upd[flist[c]] = dir[flist[c]] = sqrt(t2);
    }
    __syncthreads();
    stamp(5);
  }
  __syncthreads();
  stamp(6);
  if (a.trace != nullptr && threadIdx.x == 0) {
    for (int q = 0; q < 8; ++q) a.trace[t * 16 + q] = static_cast<double>(s_tr[q]);
    a.trace[t * 16 + 8] = static_cast<double>(s_nfl);  // events * 1e6 + flagged columns
    a.trace[t * 16 + 9] = k;
  }
  for (int j = threadIdx.x; j < M; j += blockDim.x) permg[j] = perm[j];
  if (threadIdx.x == 0) {
    const double pre = s_maxpivot * a.rank_tol;
    int r = 0;
    for (int u = 0; u < k; ++u) r += fabs(Rr[static_cast<size_t>(u) * M + u]) > pre ? 1 : 0;
    a.rank[t] = r;
  }
}

// ---------------------------------------------------------------- blocked finish (r <= kFinR)
// The three reflector applications of the finish — Y = Z^T [I_r; 0] (RZ), C = Y T11^{-1} and
// Q_r^T X = Q1^T X (pivoted-QR reflectors) — as compact-WY products on the FP64 tensor cores
// instead of one reflector at a time: G = V^T V, T by the dlarft recurrence, then
// (I - V T^T V^T) as two small GEMMs. The sequential form (below, kept for r > kFinR) spent
// ~5 us per reflector on dependent global loads.
constexpr int kFinR = 96;
constexpr int kRZ = 32;  // RZ row entries per lane held in registers (M - r <= 1024)
constexpr int kFinEB = 64;  // X columns per block of the Q1^T application

/// out(m, n, sum_k A(k, m) B(k, n)) for m < Mo, n < No, k < Ko, with A(k, m) = A[k*sak + m*sam]
/// and B(k, n) = B[k*sbk + n*sbn]: 8 x 8 output tiles over the CTA's warps, DMMA m8n8k4. A warp
/// carries two tiles at once (tile, tile + nwarps) so 16 loads per lane are in flight (the operands
/// come from L2: latency-bound); each tile still accumulates over k in ascending order.
template <class Out>
__device__ void tile_gemm_tn(int Mo, int No, int Ko, const double* A, long sak, long sam, const double* B,
                             long sbk, long sbn, Out out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int lr = lane >> 2, lc = lane & 3;
  const int tm = (Mo + 7) >> 3, tn = (No + 7) >> 3, nt = tm * tn;
  for (int tile = warp; tile < nt; tile += 2 * nw) {
    const int tiles[2] = {tile, tile + nw};
    bool mok[2], nok[2], live[2];
    const double* Ap[2];
    const double* Bp[2];
    int m0[2], n0[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      live[q] = tiles[q] < nt;
      const int tq = live[q] ? tiles[q] : tile;
      m0[q] = (tq / tn) * 8;
      n0[q] = (tq % tn) * 8;
      mok[q] = live[q] && m0[q] + lr < Mo;
      nok[q] = live[q] && n0[q] + lr < No;
      Ap[q] = A + (mok[q] ? m0[q] + lr : 0) * sam;
      Bp[q] = B + (nok[q] ? n0[q] + lr : 0) * sbn;
    }
    double c[2][2] = {{0, 0}, {0, 0}};
    int k = 0;
    for (; k + 16 <= Ko; k += 16) {  // 16 loads in flight per lane
      double av[2][4], bv[2][4];
#pragma unroll
      for (int q = 0; q < 2; ++q)
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const long kk = k + 4 * u + lc;
          av[q][u] = mok[q] ? Ap[q][kk * sak] : 0.0;
          bv[q][u] = nok[q] ? Bp[q][kk * sbk] : 0.0;
        }
#pragma unroll
      for (int q = 0; q < 2; ++q)
#pragma unroll
        for (int u = 0; u < 4; ++u) dmma_8x8x4(c[q][0], c[q][1], av[q][u], bv[q][u]);
    }
    for (; k < Ko; k += 4) {
      const int kk = k + lc;
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const double av = (mok[q] && kk < Ko) ? Ap[q][static_cast<long>(kk) * sak] : 0.0;
        const double bv = (nok[q] && kk < Ko) ? Bp[q][static_cast<long>(kk) * sbk] : 0.0;
        dmma_8x8x4(c[q][0], c[q][1], av, bv);
      }
    }
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      if (!live[q]) continue;
      const int om = m0[q] + lr, on = n0[q] + 2 * lc;
      if (om < Mo) {
        if (on < No) out(om, on, c[q][0]);
        if (on + 1 < No) out(om, on + 1, c[q][1]);
      }
    }
  }
}

/// dlarft (forward, columnwise) from the Gram matrix: T(j,j) = tau_j,
/// T(0:j, j) = -tau_j T(0:j, 0:j) G(0:j, j); T upper triangular, zero below.
__device__ void larft_from_gram(const double* G, int ldg, const double* tau, int r, double* T, int ldt) {
  for (int idx = threadIdx.x; idx < r * ldt; idx += blockDim.x) T[idx] = 0.0;
  __syncthreads();
  // column j reads only columns < j of T (written before the previous barrier): one barrier per column
  for (int j = 0; j < r; ++j) {
    double s = 0;
    const int i = threadIdx.x;
    if (i < j)
      for (int w = i; w < j; ++w) s += T[i * ldt + w] * G[w * ldg + j];
    if (i < j) T[i * ldt + j] = -tau[j] * s;
    if (i == j) T[j * ldt + j] = tau[j];
    __syncthreads();
  }
}

/// Y, C and Q_r^T X of a deficient matrix with numerical rank r <= kFinR (after the RZ pass).
__device__ void fin_stamp(const CodArgs& a, int t, int sec, unsigned long long& last);
__device__ void finish_wy(const CodArgs& a, int t, int r, const double* X, const double* Rr, const double* V1,
                          const double* tau1, const int* perm, const double* zc, double* Y, double* C,
                          double* QtX, unsigned long long& tlast) {
  extern __shared__ __align__(16) double fsm[];
  const int M = a.M, R = a.rmax, E = a.ext;
  const long ld = a.ld;
  const int reff = a.reff[t];  // V1 rows >= reff are zero
  const int ldt = r + 1;       // odd stride: conflict-free row access
  double* T = fsm;             // r x ldt
  double* G = T + r * ldt;     // r x ldt
  // ---- Y = Z^T [I_r; 0]: z_k = e_k + tail Rr(k, r:M) (COD's RZ reflectors, applied k = 0..r-1),
  //      so Y = [I_r; 0] - Z T^T Z^T [I_r; 0] = [I_r - T^T; -Z_tail T^T]
  if (r < M) {
    tile_gemm_tn(r, r, M - r, Rr + r, 1, M, Rr + r, 1, M,
                 [&](int m, int n, double v) { G[m * ldt + n] = v + (m == n ? 1.0 : 0.0); });
    __syncthreads();
    larft_from_gram(G, ldt, zc, r, T, ldt);
    for (int idx = threadIdx.x; idx < r * r; idx += blockDim.x) {
      const int c = idx / r, j = idx % r;
      Y[static_cast<size_t>(c) * M + j] = (j == c ? 1.0 : 0.0) - T[c * ldt + j];
    }
    tile_gemm_tn(M - r, r, r, Rr + r, M, 1, T, 1, ldt,
                 [&](int m, int n, double v) { Y[static_cast<size_t>(n) * M + r + m] = -v; });
  } else {
    for (int idx = threadIdx.x; idx < r * r; idx += blockDim.x) {
      const int c = idx / r, j = idx % r;
      Y[static_cast<size_t>(c) * M + j] = (j == c ? 1.0 : 0.0);
    }
  }
  __syncthreads();
  fin_stamp(a, t, 1, tlast);
  // ---- C(perm[i], :) = Y(i, :) T11^{-1}, T11 = upper triangle of Rr(0:r, 0:r): the triangular
  //      inverse by columns (thread per column), then one GEMM
  double* T11 = fsm;            // r x ldt
  double* U = T11 + r * ldt;    // r x ldt : T11^{-1}
  for (int idx = threadIdx.x; idx < r * ldt; idx += blockDim.x) {
    const int u = idx / ldt, c = idx % ldt;
    T11[idx] = (c < r && u <= c) ? Rr[static_cast<size_t>(u) * M + c] : 0.0;
    U[idx] = 0.0;
  }
  __syncthreads();
  if (threadIdx.x < r) {
    const int c = threadIdx.x;
    U[c * ldt + c] = 1.0 / T11[c * ldt + c];
    for (int i = c - 1; i >= 0; --i) {
      double s = 0;
      for (int u = i + 1; u <= c; ++u) s += T11[i * ldt + u] * U[u * ldt + c];
      U[i * ldt + c] = -s / T11[i * ldt + i];
    }
  }
  __syncthreads();
  tile_gemm_tn(M, r, r, Y, M, 1, U, ldt, 1,
               [&](int m, int n, double v) { C[static_cast<size_t>(perm[m]) * R + n] = v; });
  for (int idx = threadIdx.x; idx < M * (R - r); idx += blockDim.x) {
    const int i = idx / (R - r), c = r + idx % (R - r);
    C[static_cast<size_t>(perm[i]) * R + c] = 0.0;
  }
  __syncthreads();
  fin_stamp(a, t, 2, tlast);
  // ---- Q_r^T X = top r rows of Q1^T X, Q1^T = I - V T^T V^T (V = V1, rows < reff)
  tile_gemm_tn(r, r, reff, V1, 1, M, V1, 1, M, [&](int m, int n, double v) { G[m * ldt + n] = v; });
  __syncthreads();
  larft_from_gram(G, ldt, tau1, r, T, ldt);
  const int ldw = kFinEB + 1;
  double* Wb = G;                           // r x ldw : V^T X(:, block)   (G is free again)
  double* Wt = G + r * max(ldt, ldw);       // r x ldw : T^T W
  for (int e0 = 0; e0 < E; e0 += kFinEB) {
    const int eb = min(kFinEB, E - e0);
    const double* Xb = X + static_cast<size_t>(e0) * ld;
    tile_gemm_tn(r, eb, reff, V1, 1, M, Xb, 1, ld, [&](int m, int n, double v) { Wb[m * ldw + n] = v; });
    __syncthreads();
    for (int idx = threadIdx.x; idx < r * eb; idx += blockDim.x) {
      const int u = idx / eb, e = idx % eb;
      double s = 0;
      for (int w = 0; w <= u; ++w) s += T[w * ldt + u] * Wb[w * ldw + e];
      Wt[u * ldw + e] = s;
    }
    __syncthreads();
    tile_gemm_tn(r, eb, r, V1, M, 1, Wt, ldw, 1, [&](int m, int n, double v) {
      QtX[static_cast<size_t>(m) * E + e0 + n] = Xb[static_cast<size_t>(n) * ld + m] - v;
    });
    __syncthreads();
  }
  for (int idx = threadIdx.x; idx < (R - r) * E; idx += blockDim.x)
    QtX[static_cast<size_t>(r) * E + idx] = 0.0;
  fin_stamp(a, t, 3, tlast);
}

size_t finish_smem_bytes(int rmax) {
  // T (r x (r+1)), G / W-block (r x max(r+1, kFinEB+1)), T^T W block (r x (kFinEB+1))
  const int r = min(rmax, kFinR);
  const size_t ldt = r + 1, ldw = kFinEB + 1;
  return (static_cast<size_t>(r) * ldt + static_cast<size_t>(r) * std::max(ldt, ldw) + static_cast<size_t>(r) * ldw) *
         sizeof(double);
}

/// DDELM_COD_TRACE: thread 0's clock into trace[t * 16 + 10 + sec] (sections of the finish)
__device__ __forceinline__ void fin_stamp(const CodArgs& a, int t, int sec, unsigned long long& last) {
  if (a.trace != nullptr && threadIdx.x == 0) {
    unsigned long long now;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
    if (sec >= 0) a.trace[t * 16 + 10 + sec] += static_cast<double>(now - last);
    last = now;
  }
}

/// RZ + C + Q^T X for a deficient matrix; C = R0^{-1}, Q^T X = X for a full-rank one.
__global__ void __launch_bounds__(512) cod_finish_kernel(CodArgs a) {
  const int t = blockIdx.x;
  const int M = a.M, K = a.kmax, R = a.rmax, E = a.ext;
  const size_t ld = a.ld;
  double* A = const_cast<double*>(a.A) + static_cast<size_t>(t) * a.ld * a.ncol;
  double* C = a.C + static_cast<size_t>(t) * M * R;
  double* QtX = a.QtX + static_cast<size_t>(t) * R * E;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  const int r = a.rank[t];
  if (a.status[t] != 0) return;
  double* X = A + static_cast<size_t>(M) * ld;  // appended columns: X(i, e) = X[e*ld + i]

  if (!a.deficient[t]) {
    // full-rank branch: C = R0^{-1} (thread per column), QtX = top M rows of Q0^T [f E]
    for (int c = threadIdx.x; c < M; c += blockDim.x) {
      for (int i = M - 1; i >= 0; --i) {
        double s = (i == c) ? 1.0 : 0.0;
        if (i <= c) {
          for (int u = i + 1; u <= c; ++u) s -= A[static_cast<size_t>(u) * ld + i] * C[static_cast<size_t>(u) * R + c];
          s /= A[static_cast<size_t>(i) * ld + i];
        } else {
          s = 0.0;
        }
        C[static_cast<size_t>(i) * R + c] = s;
      }
    }
    for (int idx = threadIdx.x; idx < M * E; idx += blockDim.x) {
      const int i = idx / E, e = idx % E;
      QtX[static_cast<size_t>(i) * E + e] = X[static_cast<size_t>(e) * ld + i];
    }
    return;
  }

  double* Rr = a.Rr + static_cast<size_t>(t) * K * M;
  double* V1 = a.V1 + static_cast<size_t>(t) * K * M;
  const double* tau1 = a.tau1 + static_cast<size_t>(t) * K;
  const int* perm = a.perm + static_cast<size_t>(t) * M;
  double* zc = a.zc + static_cast<size_t>(t) * K;
  double* Y = a.Ywork + static_cast<size_t>(t) * M * R;  // Y(i, c) = Y[i*R + c]
  __shared__ double red[32];
  __shared__ double s_tau, s_beta, s_scale;
  extern __shared__ __align__(16) double fsm_rz[];
  double* zrow = fsm_rz;  // M - r doubles (the finish scratch is idle during the RZ pass)

  unsigned long long tlast = 0;
  fin_stamp(a, t, -1, tlast);
  // ---- RZ (COD::compute): rows k = r-1 .. 0 of [R11 R12], columns {k} U {r..M-1}
  if (r < M) {
    // (COD swaps column k with column r-1 so the reflector's support is contiguous, then swaps
    // back; the same arithmetic addresses column k directly)
    for (int k = r - 1; k >= 0; --k) {
      double* row = Rr + static_cast<size_t>(k) * M;
      double part = 0;
      for (int j = r + threadIdx.x; j < M; j += blockDim.x) part += row[j] * row[j];
      const double tail = block_sum(part, red);
      if (threadIdx.x == 0) {
        const double c0 = row[k];
        double tau = 0, beta = c0, scale = 0;
        if (tail > DBL_MIN) {
          beta = sqrt(c0 * c0 + tail);
          if (c0 >= 0) beta = -beta;
          scale = 1.0 / (c0 - beta);
          tau = (beta - c0) / beta;
        }
        s_tau = tau;
        s_beta = beta;
        s_scale = (tail > DBL_MIN) ? scale : 0.0;
        zc[k] = tau;
      }
      __syncthreads();
      for (int j = r + threadIdx.x; j < M; j += blockDim.x) {
        const double z = row[j] * s_scale;
        row[j] = z;
        zrow[j - r] = z;  // the reflector tail, read by every warp below: from shared memory
      }
      __syncthreads();
      if (threadIdx.x == 0) row[k] = s_beta;
      // apply Z(k) from the right to rows 0..k-1 (warp per row): the lane's entries of row u are
      // loaded once, all in flight, then summed in the same order and updated from registers
      if (s_tau != 0.0) {
        if (M - r <= 32 * kRZ) {
          for (int u = warp; u < k; u += nwarp) {
            double* ru = Rr + static_cast<size_t>(u) * M;
            double x[kRZ];
#pragma unroll
            for (int q = 0; q < kRZ; ++q) {
              const int j = r + lane + 32 * q;
              x[q] = j < M ? ru[j] : 0.0;
            }
            const double ur = ru[k];
            double s = 0;
#pragma unroll
            for (int q = 0; q < kRZ; ++q) {
              const int j = r + lane + 32 * q;
              if (j < M) s += x[q] * zrow[j - r];
            }
            s = warp_sum(s);
            s = (s + ur) * s_tau;
            __syncwarp();
            if (lane == 0) ru[k] = ur - s;
#pragma unroll
            for (int q = 0; q < kRZ; ++q) {
              const int j = r + lane + 32 * q;
              if (j < M) ru[j] = x[q] - s * zrow[j - r];
            }
          }
        } else {
          for (int u = warp; u < k; u += nwarp) {
            double* ru = Rr + static_cast<size_t>(u) * M;
            double s = 0;
            for (int j = r + lane; j < M; j += 32) s += ru[j] * row[j];
            s = warp_sum(s);
            s = (s + ru[k]) * s_tau;
            __syncwarp();
            if (lane == 0) ru[k] -= s;
            for (int j = r + lane; j < M; j += 32) ru[j] -= s * row[j];
          }
        }
      }
      __syncthreads();
    }
  }
  if (r <= kFinR) {
    __syncthreads();
    fin_stamp(a, t, 0, tlast);
    finish_wy(a, t, r, X, Rr, V1, tau1, perm, zc, Y, C, QtX, tlast);
    return;
  }
  // ---- Y = Z^T [I_r; 0] (COD::solve's Z^* application): one warp per column, the column held
  // in registers (lane owns rows lane + 32 t), no block barriers between reflectors.
  // Stored transposed, Yt(c, j) = Y[c*M + j], so every access is coalesced.
  for (int c = warp; c < r; c += nwarp) {
    double y[kNPL];
#pragma unroll
    for (int t2 = 0; t2 < kNPL; ++t2) y[t2] = (lane + 32 * t2 == c) ? 1.0 : 0.0;
    if (r < M)
      for (int k = 0; k < r; ++k) {
        const double tau = zc[k];
        if (tau == 0.0) continue;
        const double* zr = Rr + static_cast<size_t>(k) * M;
        // leading element at row k (COD's swap with row r-1 and back), tail rows r..M-1
        double s = 0;
#pragma unroll
        for (int t2 = 0; t2 < kNPL; ++t2) {
          const int j = lane + 32 * t2;
          if (j >= r && j < M) s += zr[j] * y[t2];
        }
        s = warp_sum(s);
        double yk = 0;
#pragma unroll
        for (int t2 = 0; t2 < kNPL; ++t2)
          if (t2 == (k >> 5)) yk = y[t2];
        yk = __shfl_sync(0xffffffffu, yk, k & 31);
        s = (s + yk) * tau;
#pragma unroll
        for (int t2 = 0; t2 < kNPL; ++t2) {
          const int j = lane + 32 * t2;
          if (j == k) y[t2] -= s;
          else if (j >= r && j < M) y[t2] -= s * zr[j];
        }
      }
#pragma unroll
    for (int t2 = 0; t2 < kNPL; ++t2) {
      const int j = lane + 32 * t2;
      if (j < M) Y[static_cast<size_t>(c) * M + j] = y[t2];
    }
  }
  __syncthreads();
  // ---- C(perm[i], :) = (Y T^{-1})(i, :), T = upper triangle of Rr(0:r, 0:r) (thread per row)
  for (int i = threadIdx.x; i < M; i += blockDim.x) {
    double* ci = C + static_cast<size_t>(perm[i]) * R;
    for (int c = 0; c < r; ++c) {
      double s = Y[static_cast<size_t>(c) * M + i];
      for (int u = 0; u < c; ++u) s -= ci[u] * Rr[static_cast<size_t>(u) * M + c];
      ci[c] = s / Rr[static_cast<size_t>(c) * M + c];
    }
    for (int c = r; c < R; ++c) ci[c] = 0.0;
  }
  // ---- Q1_r^T applied to the top M rows of Q0^T [f E]: one warp per column, in registers
  for (int e = warp; e < E; e += nwarp) {
    const double* xe = X + static_cast<size_t>(e) * ld;
    double x[kNPL];
#pragma unroll
    for (int t2 = 0; t2 < kNPL; ++t2) {
      const int i = lane + 32 * t2;
      x[t2] = i < M ? xe[i] : 0.0;
    }
    for (int u = 0; u < r; ++u) {
      const double tau = tau1[u];
      if (tau == 0.0) continue;
      const double* vu = V1 + static_cast<size_t>(u) * M;
      double s = 0;
#pragma unroll
      for (int t2 = 0; t2 < kNPL; ++t2) {
        const int i = lane + 32 * t2;
        if (i >= u && i < M) s += vu[i] * x[t2];
      }
      s = warp_sum(s) * tau;
#pragma unroll
      for (int t2 = 0; t2 < kNPL; ++t2) {
        const int i = lane + 32 * t2;
        if (i >= u && i < M) x[t2] -= s * vu[i];
      }
    }
#pragma unroll
    for (int t2 = 0; t2 < kNPL; ++t2) {
      const int c = lane + 32 * t2;
      if (c < R) QtX[static_cast<size_t>(c) * E + e] = c < r ? x[t2] : 0.0;
    }
  }
}

}  // namespace

bool cod_finish_supports(int M, int r) { return r <= kFinR || M <= 32 * kNPL; }

void launch_cod_pivqr(const CodArgs& a, cudaStream_t st) {
  const size_t smem = sizeof(double) * (4 * a.M + 2 * a.kmax) + sizeof(int) * 2 * a.M;
  DDG_CUDA(cudaFuncSetAttribute(cod_pivqr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(smem)));
  cod_pivqr_kernel<<<a.nmat, 512, smem, st>>>(a, 0);
  DDG_LAUNCH_CHECK();
}

void launch_cod_finish(const CodArgs& a, cudaStream_t st) {
  const size_t smem = std::max(finish_smem_bytes(a.rmax), sizeof(double) * static_cast<size_t>(a.M));
  DDG_CUDA(cudaFuncSetAttribute(cod_finish_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  cod_finish_kernel<<<a.nmat, 512, smem, st>>>(a);
  DDG_LAUNCH_CHECK();
}

}  // namespace ddg

// Interface-level blocks and the coarse problem (sm_100a, fp64).
//
// With K^+ = C Q_r^T (k_cod.cu), the coarse layer reduces to small dense per-subdomain blocks:
//   FC   = F C         (nF x r)   flux rows of K^+:   F K^+ = FC Q_r^T
//   Zc   = Q_G FC^T w  (per cross-flux row): the Dpp / Dpd rows of assemble_coarse
//   Gc   = -Q_Pi Q_Pi^T           the Gpi rows entering S_Pi
// Reference: assemble_coarse (solvers.cpp:278-326), build_neumann Cdelta (solvers.cpp:436-438).
// The coarse Schur matrix S_Pi is assembled and inverted (Cholesky) on one CTA; the rows the
// interface iteration needs are precomputed as Wmu / Wd / W3 (coarse_weights*).
#include <algorithm>
#include <cfloat>

#include "common.cuh"
#include "kernels.hpp"

namespace ddg {

namespace {

/// out[l][k] = sum_j X[j*ldx + l] * Cm[j*R + k]   for l < rows, k < r   (batched)
/// The Schur contraction of the coarse assembly (FC = F C: the flux rows of K^+, solvers.cpp:
/// 299-313) on the FP64 tensor cores: a 64 x 64 output tile per CTA, 8 warps of 2 x 4 DMMA
/// m8n8k4 tiles (16 x 32 outputs), K = the M neuron rows in 16-row chunks staged in shared
/// memory (row stride 68: every fragment load is bank-conflict free), double-buffered.
__global__ void __launch_bounds__(256) jmajor_gemm_kernel(int M, int R, const double* X, int ldx,
                                                          size_t xstride, const int* rows_of, int rows_cls,
                                                          const ClassDims* dims, const int* sub_cls,
                                                          const double* Cm, size_t cstride,
                                                          const int* rank, int rank_off,
                                                          double* out, int ldo, size_t ostride) {
  constexpr int KC = 16, SP = 68;
  const int i = blockIdx.z;
  const ClassDims d = dims[sub_cls[i]];
  const int rows = rows_cls == 0 ? d.nF : d.nd;
  (void)rows_of;
  const int r = rank[rank_off + i];
  const int l0 = blockIdx.x * 64, k0 = blockIdx.y * 64;
  double* o = out + i * ostride;
  if (l0 >= rows || k0 >= R) return;
  const double* Xi = X + i * xstride;
  const double* Ci = Cm + (rank_off + i) * cstride;
  __shared__ double Xs[2][KC * SP];
  __shared__ double Cs[2][KC * SP];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int lr = lane >> 2, lc = lane & 3;
  const int wl = (warp & 3) * 16, wk = (warp >> 2) * 32;  // warp tile: rows wl..+16, cols wk..+32
  auto load = [&](int buf, int j0) {
    for (int idx = threadIdx.x; idx < KC * 64; idx += 256) {
      const int jj = idx >> 6, c = idx & 63;
      const int j = j0 + jj;
      Xs[buf][jj * SP + c] = (j < M && l0 + c < rows) ? Xi[static_cast<size_t>(j) * ldx + l0 + c] : 0.0;
      Cs[buf][jj * SP + c] = (j < M && k0 + c < r) ? Ci[static_cast<size_t>(j) * R + k0 + c] : 0.0;
    }
  };
  double acc[2][4][2] = {};
  const int nk = (M + KC - 1) / KC;
  load(0, 0);
  __syncthreads();
  for (int q = 0; q < nk; ++q) {
    const int buf = q & 1;
    if (q + 1 < nk) load(buf ^ 1, (q + 1) * KC);
    const double* xs = Xs[buf];
    const double* cs = Cs[buf];
#pragma unroll
    for (int kk = 0; kk < KC / 4; ++kk) {
      const int jj = kk * 4 + lc;
      double av[2], bv[4];
#pragma unroll
      for (int u = 0; u < 2; ++u) av[u] = xs[jj * SP + wl + u * 8 + lr];
#pragma unroll
      for (int v = 0; v < 4; ++v) bv[v] = cs[jj * SP + wk + v * 8 + lr];
#pragma unroll
      for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) dmma_8x8x4(acc[u][v][0], acc[u][v][1], av[u], bv[v]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int u = 0; u < 2; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int l = l0 + wl + u * 8 + lr, k = k0 + wk + v * 8 + 2 * lc + h;
        if (l < rows && k < R) o[static_cast<size_t>(l) * ldo + k] = (k < r) ? acc[u][v][h] : 0.0;
      }
}

/// Per subdomain: Zc rows, flux data pd of F K^+ f, corner Gram Gc (solvers.cpp:286-313).
__global__ void __launch_bounds__(256) coarse_local_kernel(BlockArgs a, const int* cr_row,
                                                           const int* cr_off, const int* cr_l,
                                                           const double* cr_w) {
  const int i = blockIdx.x;
  const ClassDims d = a.dims[a.sub_cls[i]];
  const int r = a.rank[i];
  const int R = a.rmax, E = a.ext;
  const double* QtX = a.QtX + static_cast<size_t>(i) * R * E;  // QGt(k, g) = QtX[k*E + 1 + g]
  const double* FC = a.FC + static_cast<size_t>(i) * a.fmax * R;
  extern __shared__ double sm[];
  double* u = sm;                  // r
  double* vals = u + R;            // nF: FC qf
  __shared__ int cq[kMaxCq];
  const int ncq = a.ncq;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  if (threadIdx.x == 0) {  // corner rows in trace-row order (component 0 corners, then component 1)
    int n = 0;
    for (int g = 0; g < d.n_gamma; ++g)
      if (a.gamma_pi[static_cast<size_t>(i) * a.gmax + g] >= 0 && n < ncq) cq[n++] = g;
    for (; n < kMaxCq; ++n) cq[n] = -1;
  }
  // vals = FC qf  (F K^+ f, the data of the flux rows)
  for (int l = warp; l < d.nF; l += nwarp) {
    double s = 0;
    for (int k = lane; k < r; k += 32) s += FC[static_cast<size_t>(l) * R + k] * QtX[static_cast<size_t>(k) * E];
    s = warp_sum(s);
    if (lane == 0) vals[l] = s;
  }
  __syncthreads();
  if (threadIdx.x < ncq) a.corner_q[i * ncq + threadIdx.x] = cq[threadIdx.x];
  const int* off = cr_off + static_cast<size_t>(i) * (a.crmax + 1);
  for (int rho = 0; rho < a.crmax; ++rho) {
    const int row = cr_row[static_cast<size_t>(i) * a.crmax + rho];
    double* z = a.Zc + (static_cast<size_t>(i) * a.crmax + rho) * a.gmax;
    if (row < 0) {
      for (int g = threadIdx.x; g < a.gmax; g += blockDim.x) z[g] = 0.0;
      if (threadIdx.x == 0) a.pd[static_cast<size_t>(i) * a.crmax + rho] = 0.0;
      continue;
    }
    // u = FC^T w  (entries in scatter order)
    for (int k = threadIdx.x; k < r; k += blockDim.x) {
      double s = 0;
      for (int e = off[rho]; e < off[rho + 1]; ++e) s += cr_w[e] * FC[static_cast<size_t>(cr_l[e]) * R + k];
      u[k] = s;
    }
    if (threadIdx.x == 0) {
      double s = 0;
      for (int e = off[rho]; e < off[rho + 1]; ++e) s += cr_w[e] * vals[cr_l[e]];
      a.pd[static_cast<size_t>(i) * a.crmax + rho] = s;
    }
    __syncthreads();
    // z = QGt^T u on all gamma points
    for (int g = threadIdx.x; g < a.gmax; g += blockDim.x) {
      double s = 0;
      if (g < d.n_gamma)
        for (int k = 0; k < r; ++k) s += QtX[static_cast<size_t>(k) * E + 1 + g] * u[k];
      z[g] = s;
    }
    __syncthreads();
  }
  // Gc = -(Q_Pi Q_Pi^T) over the corners
  if (threadIdx.x < ncq * ncq) {
    const int p = threadIdx.x / ncq, q = threadIdx.x % ncq;
    double s = 0;
    if (cq[p] >= 0 && cq[q] >= 0)
      for (int k = 0; k < r; ++k)
        s += QtX[static_cast<size_t>(k) * E + 1 + cq[p]] * QtX[static_cast<size_t>(k) * E + 1 + cq[q]];
    a.Gc[static_cast<size_t>(i) * ncq * ncq + threadIdx.x] = -s;
  }
  // Ypi = K^+ B_Pi = -C Q_Pi^T (the corner columns; solvers.cpp:287-289)
  const double* Ci = a.C + static_cast<size_t>(i) * a.M * R;
  for (int j = threadIdx.x; j < a.M; j += blockDim.x)
    for (int q = 0; q < ncq; ++q) {
      double s = 0;
      if (cq[q] >= 0)
        for (int k = 0; k < r; ++k) s += Ci[static_cast<size_t>(j) * R + k] * QtX[static_cast<size_t>(k) * E + 1 + cq[q]];
      a.Ypi[(static_cast<size_t>(i) * a.M + j) * ncq + q] = -s;
    }
}

/// The per-subdomain inputs of the coarse rows, compacted into the GLOBAL subdomain numbering:
/// pd (crmax), Zc at the corner slots (crmax x ncq) and the corner Grams (ncq x ncq) of local
/// subdomain i go to rows sub_lo + i of pd_g / zcc_g / gc_g (zero elsewhere; a sharded build
/// all-reduces them: one writer per entry, exact).
__global__ void coarse_export_kernel(BlockArgs a) {
  const int i = blockIdx.x, ig = a.sub_lo + i, ncq = a.ncq;
  for (int k = threadIdx.x; k < a.crmax * ncq; k += blockDim.x) {
    const int rho = k / ncq, q = k % ncq;
    const int g = a.corner_q[i * ncq + q];
    a.zcc_g[(static_cast<size_t>(ig) * a.crmax + rho) * ncq + q] =
        g >= 0 ? a.Zc[(static_cast<size_t>(i) * a.crmax + rho) * a.gmax + g] : 0.0;
  }
  for (int rho = threadIdx.x; rho < a.crmax; rho += blockDim.x)
    a.pd_g[static_cast<size_t>(ig) * a.crmax + rho] = a.pd[static_cast<size_t>(i) * a.crmax + rho];
  for (int k = threadIdx.x; k < ncq * ncq; k += blockDim.x)
    a.gc_g[static_cast<size_t>(ig) * ncq * ncq + k] = a.Gc[static_cast<size_t>(i) * ncq * ncq + k];
}

/// Dpp rows and dpi from per-subdomain contributions, in global subdomain order (one CTA per
/// row): the same terms in the same order on one device and on every rank of a sharded build.
__global__ void coarse_rows_kernel(BlockArgs a) {
  const int rrow = blockIdx.x;
  double* drow = a.Dpp + static_cast<size_t>(rrow) * a.n_pi;
  for (int c = threadIdx.x; c < a.n_pi; c += blockDim.x) drow[c] = 0.0;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0;
    for (int q = 0; q < 4; ++q) {
      const int own = a.row_owner[rrow * 4 + q];
      if (own < 0) continue;
      const int ig = own / a.crmax;
      s += a.pd_g[own];
      const double* z = a.zcc_g + static_cast<size_t>(own) * a.ncq;
      for (int p = 0; p < a.ncq; ++p) {
        const int gp = a.cpi_g[ig * a.ncq + p];
        if (gp < 0) continue;
        drow[gp] += z[p];
      }
    }
    // dpi = -(A K^+ f) on the cross rows (solvers.cpp:293-296), with the debug flip hook
    const double sign = (a.flip_row == a.n_delta + rrow) ? -1.0 : 1.0;
    a.dpi[rrow] = -(sign * s);
  }
}

/// Gsum = sum over the subdomains of the corner Grams -(Q_Pi Q_Pi^T), scattered to (Pi, Pi).
/// Thread per entry: the subdomains owning corner rp (pi_owner, ascending global subdomain
/// order), each adding its Gram entry against corner rq if it owns that corner too — the order
/// of the serial subdomain loop this replaces, so the sums are bit-identical.
__global__ void __launch_bounds__(256) coarse_gsum_kernel(BlockArgs a) {
  const int n = a.n_pi, ncq = a.ncq;
  const long idx = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x;
  if (idx >= static_cast<long>(n) * n) return;
  const int rp = static_cast<int>(idx / n), rq = static_cast<int>(idx % n);
  double s = 0.0;
  for (int k = 0; k < 4; ++k) {
    const int own = a.pi_owner[rp * 4 + k];
    if (own < 0) continue;
    const int ig = own / ncq, p = own % ncq;
    for (int q = 0; q < ncq; ++q)
      if (a.cpi_g[ig * ncq + q] == rq) s += a.gc_g[(static_cast<size_t>(ig) * ncq + p) * ncq + q];
  }
  a.Gsum[idx] = s;
}

/// L = S = sym(diag(mult) + Dpp^T Dpp + Gsum), entry per thread (each entry's arithmetic as in
/// the single-CTA formation it replaces: the same dot order, the same symmetrisation).
__global__ void __launch_bounds__(256) coarse_sform_kernel(BlockArgs a) {
  const int n = a.n_pi, npf = a.npf;
  const long idx = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x;
  if (idx >= static_cast<long>(n) * n) return;
  const int p = static_cast<int>(idx / n), q = static_cast<int>(idx % n);
  auto entry = [&](int x, int y) {
    double s = 0;
    for (int rr = 0; rr < npf; ++rr) s += a.Dpp[static_cast<size_t>(rr) * n + x] * a.Dpp[static_cast<size_t>(rr) * n + y];
    double v = (x == y ? static_cast<double>(a.mult_pi[x]) : 0.0) + s;
    v += a.Gsum[static_cast<size_t>(x) * n + y];
    return v;
  };
  const double l = 0.5 * (entry(p, q) + entry(q, p));
  a.Sinv[idx] = l;  // L (full), factored in place by coarse_chol_kernel
  a.S[idx] = l;
}

/// Cholesky S = L L^T (right-looking, lower triangle) and L^{-1} by forward substitution (thread
/// per column), one CTA. L lives packed (row i at i(i+1)/2) in shared memory when it fits, so the
/// n sequential steps and the substitution chains read it at shared-memory latency; otherwise it
/// is factored in place in global memory. L^{-1} goes to S, transposed.
__global__ void __launch_bounds__(1024) coarse_chol_kernel(BlockArgs a, int packed) {
  const int n = a.n_pi;
  extern __shared__ double lp[];
  double* Lg = a.Sinv;
  __shared__ int fail;
  if (threadIdx.x == 0) fail = 0;
  auto at = [&](int i, int j) -> double& {
    return packed ? lp[static_cast<size_t>(i) * (i + 1) / 2 + j] : Lg[static_cast<size_t>(i) * n + j];
  };
  if (packed)
    for (int idx = threadIdx.x; idx < n * (n + 1) / 2; idx += blockDim.x) {
      int i = static_cast<int>((sqrt(8.0 * idx + 1.0) - 1.0) / 2.0);
      while (static_cast<long>(i) * (i + 1) / 2 > idx) --i;
      while (static_cast<long>(i + 1) * (i + 2) / 2 <= idx) ++i;
      const int j = idx - i * (i + 1) / 2;
      lp[idx] = Lg[static_cast<size_t>(i) * n + j];
    }
  __syncthreads();
  for (int k = 0; k < n; ++k) {
    if (threadIdx.x == 0) {
      const double dkk = at(k, k);
      if (!(dkk > 0)) fail = 1;
      at(k, k) = sqrt(fmax(dkk, DBL_MIN));
    }
    __syncthreads();
    const double dk = at(k, k);
    for (int i = k + 1 + threadIdx.x; i < n; i += blockDim.x) at(i, k) /= dk;
    __syncthreads();
    // trailing update of the lower triangle: warp per row, lanes over the columns j <= i
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
    for (int i = k + 1 + warp; i < n; i += nwarp) {
      const double lik = at(i, k);
      for (int j = k + 1 + lane; j <= i; j += 32) at(i, j) -= lik * at(j, k);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0 && fail) *a.spd_fail = 1;
  // column c of L^{-1}, stored transposed (LiT[c*n + i]) so every chain reads its own contiguous
  // column; zero above the diagonal
  double* LiT = a.S;
  for (int c = threadIdx.x; c < n; c += blockDim.x) {
    double* col = LiT + static_cast<size_t>(c) * n;
    for (int i = 0; i < c; ++i) col[i] = 0.0;
    for (int i = c; i < n; ++i) {
      double s = (i == c) ? 1.0 : 0.0;
#pragma unroll 8
      for (int u = c; u < i; ++u) s -= at(i, u) * col[u];
      col[i] = s / at(i, i);
    }
  }
}

/// S^{-1} = L^{-T} L^{-1}, entry per thread.
__global__ void __launch_bounds__(256) coarse_sinv_kernel(BlockArgs a) {
  const int n = a.n_pi;
  const long idx = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x;
  if (idx >= static_cast<long>(n) * n) return;
  const int p = static_cast<int>(idx / n), q = static_cast<int>(idx % n);
  const double* LiT = a.S;  // transposed L^{-1} (coarse_chol_kernel)
  const double* lp = LiT + static_cast<size_t>(p) * n;
  const double* lq = LiT + static_cast<size_t>(q) * n;
  double s = 0;
  for (int u = max(p, q); u < n; ++u) s += lp[u] * lq[u];
  a.Sinv[idx] = s;
}

/// Coarse-solve rows used by the interface iteration (k_cg.cu): with z = [t; psi],
///   mu = S^{-1}(t + Dpp^T psi) = Wmu z,   d1 = psi - Dpp mu = Wd z,   Dpp S^{-1} = W3.
__global__ void coarse_weights1_kernel(BlockArgs a) {
  const int n = a.n_pi, npf = a.npf, nz = n + npf;
  const long total = static_cast<long>(n) * nz + static_cast<long>(npf) * n;
  for (long idx = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<long>(gridDim.x) * blockDim.x) {
    if (idx < static_cast<long>(n) * nz) {
      const int p = static_cast<int>(idx / nz), c = static_cast<int>(idx % nz);
      double s;
      if (c < n) {
        s = a.Sinv[static_cast<size_t>(p) * n + c];
      } else {
        const int rr = c - n;
        s = 0;
        for (int j = 0; j < n; ++j) s += a.Sinv[static_cast<size_t>(p) * n + j] * a.Dpp[static_cast<size_t>(rr) * n + j];
      }
      a.Wmu[idx] = s;
    } else {
      const long k = idx - static_cast<long>(n) * nz;
      const int rr = static_cast<int>(k / n), p = static_cast<int>(k % n);
      double s = 0;
      for (int j = 0; j < n; ++j) s += a.Dpp[static_cast<size_t>(rr) * n + j] * a.Sinv[static_cast<size_t>(j) * n + p];
      a.W3[k] = s;
    }
  }
}

__global__ void coarse_weights2_kernel(BlockArgs a) {
  const int n = a.n_pi, npf = a.npf, nz = n + npf;
  const long total = static_cast<long>(npf) * nz;
  for (long idx = blockIdx.x * static_cast<long>(blockDim.x) + threadIdx.x; idx < total;
       idx += static_cast<long>(gridDim.x) * blockDim.x) {
    const int rr = static_cast<int>(idx / nz), c = static_cast<int>(idx % nz);
    double s;
    if (c < n) {
      s = -a.W3[static_cast<size_t>(rr) * n + c];
    } else {
      const int ss = c - n;
      double acc = 0;
      for (int j = 0; j < n; ++j) acc += a.Dpp[static_cast<size_t>(rr) * n + j] * a.Wmu[static_cast<size_t>(j) * nz + n + ss];
      s = (rr == ss ? 1.0 : 0.0) - acc;
    }
    a.Wd[idx] = s;
  }
}

}  // namespace

void launch_blocks(const BlockArgs& a, cudaStream_t st) {
  // FC = F C: flux rows of K^+ (feeds the Dpp / Dpd rows of the coarse problem)
  const size_t xs_f = static_cast<size_t>(a.M) * a.ldF;
  const size_t cs = static_cast<size_t>(a.M) * a.rmax;
  dim3 g(ceil_div(a.fmax, 64), ceil_div(a.rmax, 64), a.N);
  jmajor_gemm_kernel<<<g, 256, 0, st>>>(a.M, a.rmax, a.F, a.ldF, xs_f, nullptr, 0, a.dims, a.sub_cls, a.C, cs,
                                        a.rank, 0, a.FC, a.rmax, static_cast<size_t>(a.fmax) * a.rmax);
  DDG_LAUNCH_CHECK();
}

void launch_coarse_local(const BlockArgs& a, const int* cr_row, const int* cr_off, const int* cr_l,
                         const double* cr_w, cudaStream_t st) {
  const size_t smem = sizeof(double) * (a.rmax + a.fmax);
  coarse_local_kernel<<<a.N, 256, smem, st>>>(a, cr_row, cr_off, cr_l, cr_w);
  DDG_LAUNCH_CHECK();
}

void launch_coarse_export(const BlockArgs& a, cudaStream_t st) {
  coarse_export_kernel<<<a.N, 128, 0, st>>>(a);
  DDG_LAUNCH_CHECK();
}

void launch_coarse_rows(const BlockArgs& a, cudaStream_t st) {
  coarse_rows_kernel<<<a.npf, 128, 0, st>>>(a);
  DDG_LAUNCH_CHECK();
}

void launch_coarse_gsum(const BlockArgs& a, cudaStream_t st) {
  const long nn = static_cast<long>(a.n_pi) * a.n_pi;
  coarse_gsum_kernel<<<static_cast<int>((nn + 255) / 256), 256, 0, st>>>(a);
  DDG_LAUNCH_CHECK();
}

void launch_coarse_schur(const BlockArgs& a, cudaStream_t st) {
  const long nn = static_cast<long>(a.n_pi) * a.n_pi;
  const int g = static_cast<int>((nn + 255) / 256);
  coarse_sform_kernel<<<g, 256, 0, st>>>(a);
  DDG_LAUNCH_CHECK();
  static int optin = -1;
  if (optin < 0) {
    int dev = 0;
    DDG_CUDA(cudaGetDevice(&dev));
    DDG_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    DDG_CUDA(cudaFuncSetAttribute(coarse_chol_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - 1024));
  }
  const size_t packed = sizeof(double) * static_cast<size_t>(a.n_pi) * (a.n_pi + 1) / 2;
  const bool fits = packed + 1024 <= static_cast<size_t>(optin);
  coarse_chol_kernel<<<1, 1024, fits ? packed : 0, st>>>(a, fits ? 1 : 0);
  DDG_LAUNCH_CHECK();
  coarse_sinv_kernel<<<g, 256, 0, st>>>(a);
  DDG_LAUNCH_CHECK();
}

namespace {
__global__ void pack_streams_kernel(BlockArgs a, double* KF, const int* kf_ld, const long long* kf_off, double* KD,
                                    const int* kd_ld, const long long* kd_off) {
  const int i = blockIdx.y;
  const int R = a.rmax;
  const int ldKF = kf_ld[i], ldKD = kd_ld[i];  // per-subdomain strides: no padding to the widest class
  for (int j = blockIdx.x; j < a.M; j += gridDim.x) {
    const size_t row = static_cast<size_t>(i) * a.M + j;
    double* kf = KF + kf_off[i] + static_cast<size_t>(j) * ldKF;
    double* kd = KD + kd_off[i] + static_cast<size_t>(j) * ldKD;
    const double* c = a.C + row * R;
    const double* cb = a.C + (static_cast<size_t>(a.N + i) * a.M + j) * R;
    for (int k = threadIdx.x; k < ldKF; k += blockDim.x) {
      double v = 0.0;
      if (k < R) v = c[k];
      else if (k < R + a.ncq) v = a.Ypi[row * a.ncq + (k - R)];
      else if (k - R - a.ncq < a.ldF) v = a.F[row * a.ldF + (k - R - a.ncq)];
      kf[k] = v;
    }
    for (int k = threadIdx.x; k < ldKD; k += blockDim.x) {
      double v = 0.0;
      if (k < R) v = cb[k];
      else if (k - R < a.ldC) v = a.Cd[row * a.ldC + (k - R)];
      kd[k] = v;
    }
  }
}
/// Compact interface-level stream block of one packed block P (M rows, stride ld): row q of the
/// output (same stride) holds the unit vector e_{c(q)} in columns [0, boff) and, in columns
/// [boff, boff + nb), the contraction  sum_j P[j][c(q)] P[j][boff + l]  — i.e. (F C)^T, (F Ypi)^T
/// (KF: c(q) = q for q < r, R + q - r for the ncq Ypi columns) and (Cdelta Cbar)^T (KD). The
/// M-long coefficient-space contraction of every CG phase (solvers.cpp:215-218, 455, 468) is then
/// done once here instead of once per iteration. DFMA tiles, fixed j order (deterministic).
__global__ void __launch_bounds__(256) compact_stream_kernel(int M, int R, int ncq, const double* P,
                                                             const int* ld_of, const long long* off_of,
                                                             double* out, const long long* oout_of,
                                                             const int* rank, int rank_off, int nb_kind,
                                                             const ClassDims* dims, const int* sub_cls) {
  const int i = blockIdx.z;
  const ClassDims d = dims[sub_cls[i]];
  const int r = rank[rank_off + i];
  const int nq = r + (nb_kind == 0 ? ncq : 0);            // output rows
  const int boff = nb_kind == 0 ? R + ncq : R;
  const int nb = nb_kind == 0 ? d.nF : d.nd;
  const int ld = ld_of[i];
  const double* Pi = P + off_of[i];
  double* o = out + oout_of[i];
  const int q0 = blockIdx.x * 64, l0 = blockIdx.y * 64;
  if (q0 >= nq) return;
  auto col = [&](int q) { return q < r ? q : R + (q - r); };
  if (blockIdx.y == 0)  // identity part of the tile's rows (and the zero tail past boff + nb)
    for (int idx = threadIdx.x; idx < 64 * boff; idx += 256) {
      const int qq = idx / boff, c = idx % boff, q = q0 + qq;
      if (q < nq) o[static_cast<size_t>(q) * ld + c] = (c == col(q)) ? 1.0 : 0.0;
    }
  if (blockIdx.y == 0)
    for (int idx = threadIdx.x; idx < 64 * (ld - boff - nb); idx += 256) {
      const int w = ld - boff - nb, qq = idx / w, c = boff + nb + idx % w, q = q0 + qq;
      if (q < nq) o[static_cast<size_t>(q) * ld + c] = 0.0;
    }
  if (l0 >= nb) return;
  __shared__ double Xs[16][64];
  __shared__ double Ys[16][64];
  const int tq = (threadIdx.x & 15) * 4, tl = (threadIdx.x >> 4) * 4;
  double acc[4][4] = {};
  for (int j0 = 0; j0 < M; j0 += 16) {
    for (int idx = threadIdx.x; idx < 16 * 64; idx += 256) {
      const int jj = idx / 64, c = idx % 64;
      const int j = j0 + jj;
      const double* row = Pi + static_cast<size_t>(j) * ld;
      Xs[jj][c] = (j < M && q0 + c < nq) ? row[col(q0 + c)] : 0.0;
      Ys[jj][c] = (j < M && l0 + c < nb) ? row[boff + l0 + c] : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int jj = 0; jj < 16; ++jj) {
      double xv[4], yv[4];
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        xv[p] = Xs[jj][tq + p];
        yv[p] = Ys[jj][tl + p];
      }
#pragma unroll
      for (int p = 0; p < 4; ++p)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[p][q] = fma(xv[p], yv[q], acc[p][q]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int p = 0; p < 4; ++p)
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int qq = q0 + tq + p, l = l0 + tl + q;
      if (qq < nq && l < nb) o[static_cast<size_t>(qq) * ld + boff + l] = acc[p][q];
    }
}
}  // namespace

void launch_pack_streams(const BlockArgs& a, double* KF, const int* kf_ld, const long long* kf_off, double* KD,
                         const int* kd_ld, const long long* kd_off, cudaStream_t st) {
  dim3 g(std::min(a.M, 64), a.N);
  pack_streams_kernel<<<g, 256, 0, st>>>(a, KF, kf_ld, kf_off, KD, kd_ld, kd_off);
  DDG_LAUNCH_CHECK();
}

void launch_compact_streams(const BlockArgs& a, const double* KF, const int* kf_ld, const long long* kf_off,
                            const double* KD, const int* kd_ld, const long long* kd_off, double* KFc,
                            const long long* kfc_off, double* KDc, const long long* kdc_off, cudaStream_t st) {
  const int R = a.rmax;
  dim3 gf((R + a.ncq + 63) / 64, (a.fmax + 63) / 64, a.N);
  compact_stream_kernel<<<gf, 256, 0, st>>>(a.M, R, a.ncq, KF, kf_ld, kf_off, KFc, kfc_off, a.rank, 0, 0, a.dims,
                                            a.sub_cls);
  DDG_LAUNCH_CHECK();
  dim3 gd((R + 63) / 64, (std::max(a.dmax, 1) + 63) / 64, a.N);
  compact_stream_kernel<<<gd, 256, 0, st>>>(a.M, R, a.ncq, KD, kd_ld, kd_off, KDc, kdc_off, a.rank, a.N, 1, a.dims,
                                            a.sub_cls);
  DDG_LAUNCH_CHECK();
}

void launch_coarse_weights(const BlockArgs& a, cudaStream_t st) {
  coarse_weights1_kernel<<<296, 256, 0, st>>>(a);
  coarse_weights2_kernel<<<296, 256, 0, st>>>(a);
  DDG_LAUNCH_CHECK();
}

}  // namespace ddg

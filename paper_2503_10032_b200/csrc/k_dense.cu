// Dense brute-force oracle on the device: dense_oracle_solve
// (proj/src/solvers.cpp:609-709) for small instances, the cross-check behind oracle_check
// (runner.cpp:252-316). Not a performance path: the global matrices are at most 3000 columns
// (the reference's own limit, solvers.cpp:619-620).
//
// Building blocks:
//   * dense_gemm_kernel   C = alpha op(A) op(B) + beta C, column-major FP64 (64 x 64 tiles, DFMA)
//   * dense_rows_kernel   A(row, colofs_i + j) += w F_i(lrow, j): flux / Cdelta scatter, one thread
//                         per column so every (row, column) accumulates in the reference's order
//   * dense_set_kernel    the unit selection entries of B / Bbar
//   * dense_cod_solve     X^+ R with Eigen's default COD threshold eps * min(m, n), through the
//                         hot path's own batched QR + pivoted-QR/RZ kernels on ONE matrix
//                         (k_qr.cu, k_cod.cu): X^+ R = C (Q_r^T R)
#include <algorithm>
#include <cfloat>
#include <stdexcept>
#include <string>
#include <vector>

#include "common.cuh"
#include "kernels.hpp"
#include "workspace.hpp"

namespace ddg {

namespace {

constexpr int kGT = 64, kGK = 16;

__global__ void __launch_bounds__(256) dense_gemm_kernel(int m, int n, int k, double alpha, const double* __restrict__ A,
                                                         int lda, int ta, const double* __restrict__ B, int ldb,
                                                         int tb, double beta, double* __restrict__ C, int ldc) {
  __shared__ double As[kGK][kGT + 1];
  __shared__ double Bs[kGK][kGT + 1];
  const int r0 = blockIdx.x * kGT, c0 = blockIdx.y * kGT;
  const int tr = threadIdx.x % 16, tc = threadIdx.x / 16;  // 4 x 4 outputs: rows tr + 16 u, cols tc + 16 v
  double acc[4][4] = {};
  for (int k0 = 0; k0 < k; k0 += kGK) {
    for (int idx = threadIdx.x; idx < kGK * kGT; idx += blockDim.x) {
      // A tile: op(A)(r0 + r, k0 + kk); B tile: op(B)(k0 + kk, c0 + c)
      int r, kk;
      if (ta) { kk = idx % kGK; r = idx / kGK; } else { r = idx % kGT; kk = idx / kGT; }
      const int gr = r0 + r, gk = k0 + kk;
      double va = 0.0;
      if (gr < m && gk < k) va = ta ? A[static_cast<size_t>(gr) * lda + gk] : A[static_cast<size_t>(gk) * lda + gr];
      As[kk][r] = va;
      int c;
      if (tb) { c = idx % kGT; kk = idx / kGT; } else { kk = idx % kGK; c = idx / kGK; }
      const int gc = c0 + c;
      const int gk2 = k0 + kk;
      double vb = 0.0;
      if (gc < n && gk2 < k) vb = tb ? B[static_cast<size_t>(gk2) * ldb + gc] : B[static_cast<size_t>(gc) * ldb + gk2];
      Bs[kk][c] = vb;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < kGK; ++kk) {
      double a[4], b[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) a[u] = As[kk][tr + 16 * u];
#pragma unroll
      for (int v = 0; v < 4; ++v) b[v] = Bs[kk][tc + 16 * v];
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = fma(a[u], b[v], acc[u][v]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int u = 0; u < 4; ++u)
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const int r = r0 + tr + 16 * u, c = c0 + tc + 16 * v;
      if (r < m && c < n) {
        double* p = C + static_cast<size_t>(c) * ldc + r;
        *p = beta == 0.0 ? alpha * acc[u][v] : alpha * acc[u][v] + beta * *p;
      }
    }
}

/// dst(row_e, colofs_i + j) += w_e src_i(lrow_e, j) for the entries e of subdomain i (CSR by
/// subdomain, reference scatter order); src_i(l, j) = src[i * sstride + j * lds + l].
__global__ void dense_rows_kernel(double* dst, int ldd, const double* src, int lds, size_t sstride, const int* off,
                                  const int* row, const int* lrow, const double* w, int M) {
  const int i = blockIdx.y;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= M) return;
  const double* s = src + static_cast<size_t>(i) * sstride + static_cast<size_t>(j) * lds;
  double* d = dst + static_cast<size_t>(i * M + j) * ldd;
  for (int e = off[i]; e < off[i + 1]; ++e) d[row[e]] += w[e] * s[lrow[e]];
}

__global__ void dense_set_kernel(double* dst, const long long* idx, int n, double v) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t < n) dst[idx[t]] = v;
}

__global__ void dense_axpy_identity_kernel(double* W, int n, double theta) {
  // W = theta W + (1 - theta) I
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n * n) return;
  const int r = t % n, c = t / n;
  W[t] = theta * W[t] + (r == c ? 1.0 - theta : 0.0);
}

template <typename T>
T* dev_alloc(size_t n, std::vector<void*>& keep) {
  T* p = nullptr;
  DDG_CUDA(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)));
  keep.push_back(p);
  return p;
}

struct DevScope {
  std::vector<void*> ptrs;
  ~DevScope() {
    for (void* p : ptrs) cudaFree(p);
  }
  double* d(size_t n) { return dev_alloc<double>(n, ptrs); }
  template <typename T>
  T* up(const std::vector<T>& v, cudaStream_t st) {
    T* p = dev_alloc<T>(v.size(), ptrs);
    if (!v.empty()) DDG_CUDA(cudaMemcpyAsync(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, st));
    return p;
  }
};

}  // namespace

void dense_gemm(int m, int n, int k, double alpha, const double* A, int lda, bool ta, const double* B, int ldb,
                bool tb, double beta, double* C, int ldc, cudaStream_t st) {
  if (m <= 0 || n <= 0) return;
  dim3 grid(ceil_div(m, kGT), ceil_div(n, kGT));
  dense_gemm_kernel<<<grid, 256, 0, st>>>(m, n, k, alpha, A, lda, ta ? 1 : 0, B, ldb, tb ? 1 : 0, beta, C, ldc);
  DDG_LAUNCH_CHECK();
}

void dense_cod_solve(const double* X, int ldx, int m, int n, const double* R, int ldr, int e, double* out, int ldo,
                     cudaStream_t st, int* rank_out) {
  if (m < n) throw std::invalid_argument("dense_cod_solve: wide system");
  DevScope s;
  const int ld = (m + 3) / 4 * 4, ncol = n + e;
  double* A = s.d(static_cast<size_t>(ld) * ncol);
  DDG_CUDA(cudaMemsetAsync(A, 0, sizeof(double) * ld * ncol, st));
  DDG_CUDA(cudaMemcpy2DAsync(A, sizeof(double) * ld, X, sizeof(double) * ldx, sizeof(double) * m, n,
                             cudaMemcpyDeviceToDevice, st));
  if (e > 0)
    DDG_CUDA(cudaMemcpy2DAsync(A + static_cast<size_t>(n) * ld, sizeof(double) * ld, R, sizeof(double) * ldr,
                               sizeof(double) * m, e, cudaMemcpyDeviceToDevice, st));
  double* tau = s.d(n);
  double* T = s.d(static_cast<size_t>(kQrTmax) * kQrTmax);
  double* ratio = s.d(2);
  QrArgs q{1, m, ld, ncol, n, A, tau, T};
  std::vector<cudaEvent_t> none;
  qr_factor(q, st, nullptr, none);
  launch_qr_diag_ratio(q, ratio, st);
  CodArgs c{};
  c.nmat = 1;
  c.m = m;
  c.ld = ld;
  c.ncol = ncol;
  c.M = n;
  c.kmax = n;
  c.rmax = n;
  c.ext = std::max(e, 1);
  c.rank_tol = DBL_EPSILON * std::min(m, n);  // Eigen's default COD threshold
  c.A = A;
  c.ratio = ratio;
  std::vector<void*>& P = s.ptrs;
  c.deficient = dev_alloc<int>(1, P);
  c.V1 = s.d(static_cast<size_t>(n) * n);
  c.F1 = s.d(static_cast<size_t>(n) * n);
  c.Rr = s.d(static_cast<size_t>(n) * n);
  c.tau1 = s.d(n);
  c.upd = s.d(n);
  c.dir = s.d(n);
  c.perm = dev_alloc<int>(n, P);
  c.rank = dev_alloc<int>(1, P);
  c.status = dev_alloc<int>(1, P);
  c.reff = dev_alloc<int>(1, P);
  c.zc = s.d(n);
  c.C = s.d(static_cast<size_t>(n) * n);
  c.QtX = s.d(static_cast<size_t>(n) * c.ext);
  c.Ywork = s.d(static_cast<size_t>(n) * n);
  launch_cod_pivqr(c, st);
  int h[3];
  DDG_CUDA(cudaMemcpyAsync(&h[0], c.deficient, sizeof(int), cudaMemcpyDeviceToHost, st));
  DDG_CUDA(cudaMemcpyAsync(&h[1], c.rank, sizeof(int), cudaMemcpyDeviceToHost, st));
  DDG_CUDA(cudaMemcpyAsync(&h[2], c.status, sizeof(int), cudaMemcpyDeviceToHost, st));
  DDG_CUDA(cudaStreamSynchronize(st));
  if (h[2] != 0) throw std::runtime_error("dense_cod_solve: pivoted QR capacity exceeded");
  if (h[0] && !cod_finish_supports(n, h[1]))
    throw std::invalid_argument("dense oracle: rank-deficient system with " + std::to_string(n) +
                                " columns exceeds the device COD finish (<= 1024 columns)");
  launch_cod_finish(c, st);
  if (rank_out) *rank_out = h[1];
  if (e > 0) {
    // C(i, c) = c.C[i * n + c], QtX(c, j) = c.QtX[c * ext + j]: out = C QtX
    dense_gemm(n, e, n, 1.0, c.C, n, true, c.QtX, c.ext, true, 0.0, out, ldo, st);
  }
  DDG_CUDA(cudaStreamSynchronize(st));  // the scope frees the scratch
}

// ------------------------------------------------------------------ LsFactor on caller matrices
void lsfactor_batch(int nmat, int m, int n, const double* K, double rank_tol, int* rank, int* deficient, int* reff,
                    double* pinv, double* Q, cudaStream_t st) {
  // LsFactor (solvers.cpp:24-45) of nmat caller-supplied m x n matrices through the hot path's own
  // kernels: batched blocked QR of [K | I_m] (the appended identity turns Q_r^T [f | E] into Q_r^T
  // itself), the diagonal-ratio branch test, the pivoted QR + RZ on R0 and the finish; then
  // K^+ = C Q_r^T (dense_gemm) and Q_r = (Q_r^T)^T.
  if (nmat < 1 || m < 1 || n < 1) throw std::invalid_argument("lsfactor_batch: empty batch");
  if (m < n) throw std::invalid_argument("LsFactor: matrix must be square or tall");
  if (!(rank_tol > 0)) throw std::invalid_argument("lsfactor_batch: rank_tol must be positive");
  DevScope s;
  const int ld = (m + 3) / 4 * 4, ncol = n + m;
  const size_t ms = static_cast<size_t>(ld) * ncol;
  double* A = s.d(ms * nmat);
  DDG_CUDA(cudaMemsetAsync(A, 0, sizeof(double) * ms * nmat, st));
  std::vector<double> eye(static_cast<size_t>(ld) * m, 0.0);
  for (int j = 0; j < m; ++j) eye[static_cast<size_t>(j) * ld + j] = 1.0;
  for (int t = 0; t < nmat; ++t) {
    DDG_CUDA(cudaMemcpy2DAsync(A + t * ms, sizeof(double) * ld, K + static_cast<size_t>(t) * m * n, sizeof(double) * m,
                               sizeof(double) * m, n, cudaMemcpyHostToDevice, st));
    DDG_CUDA(cudaMemcpyAsync(A + t * ms + static_cast<size_t>(n) * ld, eye.data(), sizeof(double) * eye.size(),
                             cudaMemcpyHostToDevice, st));
  }
  double* tau = s.d(static_cast<size_t>(nmat) * n);
  double* T = s.d(static_cast<size_t>(nmat) * kQrTmax * kQrTmax);
  double* ratio = s.d(2 * static_cast<size_t>(nmat));
  QrArgs q{nmat, m, ld, ncol, n, A, tau, T};
  std::vector<cudaEvent_t> none;
  qr_factor(q, st, nullptr, none);
  launch_qr_diag_ratio(q, ratio, st);
  CodArgs c{};
  c.nmat = nmat;
  c.m = m;
  c.ld = ld;
  c.ncol = ncol;
  c.M = n;
  c.kmax = n;
  c.rmax = n;
  c.ext = m;
  c.rank_tol = rank_tol;
  c.A = A;
  c.ratio = ratio;
  std::vector<void*>& P = s.ptrs;
  const size_t nn = static_cast<size_t>(n) * n * nmat;
  c.deficient = dev_alloc<int>(nmat, P);
  c.V1 = s.d(nn);
  c.F1 = s.d(nn);
  c.Rr = s.d(nn);
  c.tau1 = s.d(static_cast<size_t>(n) * nmat);
  c.upd = s.d(static_cast<size_t>(n) * nmat);
  c.dir = s.d(static_cast<size_t>(n) * nmat);
  c.perm = dev_alloc<int>(static_cast<size_t>(n) * nmat, P);
  c.rank = dev_alloc<int>(nmat, P);
  c.status = dev_alloc<int>(nmat, P);
  c.reff = dev_alloc<int>(nmat, P);
  c.zc = s.d(static_cast<size_t>(n) * nmat);
  c.C = s.d(nn);
  c.QtX = s.d(static_cast<size_t>(n) * m * nmat);
  c.Ywork = s.d(nn);
  launch_cod_pivqr(c, st);
  std::vector<int> hd(nmat), hr(nmat), hs(nmat), he(nmat);
  DDG_CUDA(cudaMemcpyAsync(hd.data(), c.deficient, sizeof(int) * nmat, cudaMemcpyDeviceToHost, st));
  DDG_CUDA(cudaMemcpyAsync(hr.data(), c.rank, sizeof(int) * nmat, cudaMemcpyDeviceToHost, st));
  DDG_CUDA(cudaMemcpyAsync(hs.data(), c.status, sizeof(int) * nmat, cudaMemcpyDeviceToHost, st));
  DDG_CUDA(cudaMemcpyAsync(he.data(), c.reff, sizeof(int) * nmat, cudaMemcpyDeviceToHost, st));
  DDG_CUDA(cudaStreamSynchronize(st));
  for (int t = 0; t < nmat; ++t) {
    if (hs[t] != 0) throw std::runtime_error("lsfactor_batch: pivoted QR capacity exceeded");
    if (hd[t] && !cod_finish_supports(n, hr[t]))
      throw std::invalid_argument("lsfactor_batch: rank-deficient matrix wider than the device COD finish");
  }
  launch_cod_finish(c, st);
  double* Pd = s.d(static_cast<size_t>(n) * m);
  for (int t = 0; t < nmat; ++t) {
    // C(i, k) = C[t][i * n + k] (k < r), QtX(k, j) = QtX[t][k * m + j]: K^+ = C QtX (n x m)
    const double* Ct = c.C + static_cast<size_t>(t) * n * n;
    const double* Xt = c.QtX + static_cast<size_t>(t) * n * m;
    DDG_CUDA(cudaMemsetAsync(Pd, 0, sizeof(double) * n * m, st));
    if (hr[t] > 0) dense_gemm(n, m, hr[t], 1.0, Ct, n, true, Xt, m, true, 0.0, Pd, n, st);
    DDG_CUDA(cudaMemcpyAsync(pinv + static_cast<size_t>(t) * n * m, Pd, sizeof(double) * n * m, cudaMemcpyDeviceToHost, st));
    if (Q) {
      // Q_r (m x n, columns >= r zero) = QtX^T: QtX is r x m row-major = Q_r column-major
      std::vector<double> qt(static_cast<size_t>(n) * m);
      DDG_CUDA(cudaMemcpyAsync(qt.data(), Xt, sizeof(double) * qt.size(), cudaMemcpyDeviceToHost, st));
      DDG_CUDA(cudaStreamSynchronize(st));
      double* Qt = Q + static_cast<size_t>(t) * m * n;
      for (int k = 0; k < n; ++k)
        for (int j = 0; j < m; ++j) Qt[static_cast<size_t>(k) * m + j] = k < hr[t] ? qt[static_cast<size_t>(k) * m + j] : 0.0;
    }
  }
  DDG_CUDA(cudaStreamSynchronize(st));
  for (int t = 0; t < nmat; ++t) {
    rank[t] = hr[t];
    deficient[t] = hd[t];
    if (reff) reff[t] = he[t];
  }
}

// ------------------------------------------------------------------ Workspace::dense_oracle
void Workspace::dense_oracle(int method, double theta, DenseOracleOut& o) {
  if (sharded()) throw std::invalid_argument("dense_oracle_solve: single-device workspaces only");
  if (method < 0 || method > 2) throw std::invalid_argument("dense_oracle_solve: unknown method");
  if (method == 2 && (theta < 0.0 || theta > 1.0)) throw std::invalid_argument("dense_oracle_solve: theta in [0, 1]");
  DDG_CUDA(cudaSetDevice(device_));
  const Plan& p = plan;
  const int N = p.N, M = p.M;
  const int nd = p.n_delta, np = p.n_pi, npf = p.npf, nmu = nd + np, nflux = nd + npf;
  std::vector<int> rowofs(N + 1, 0);
  for (int i = 0; i < N; ++i) rowofs[i + 1] = rowofs[i] + p.classes[p.subs[i].cls].m;
  const int sumrows = rowofs[N], sumM = N * M;
  if (sumM + nmu > 3000) throw std::invalid_argument("dense_oracle_solve: system too large for the dense path");
  cudaStream_t st = st_;
  DevScope s;

  // ---- the local matrices (the factorisation overwrote them: regenerate, as get_local)
  init_layers();
  launch_build_features(feature_args(), st);
  built_ = blocks_built_ = coarse_built_ = neumann_built_ = false;
  const size_t mstride = static_cast<size_t>(ld_) * ncol_;

  // ---- K (sumrows x sumM), FB = [f | B] (sumrows x (1 + nmu)), A (nflux x sumM)
  double* K = s.d(static_cast<size_t>(sumrows) * sumM);
  double* FB = s.d(static_cast<size_t>(sumrows) * (1 + nmu));
  double* A = s.d(static_cast<size_t>(nflux) * sumM);
  DDG_CUDA(cudaMemsetAsync(K, 0, sizeof(double) * sumrows * sumM, st));
  DDG_CUDA(cudaMemsetAsync(FB, 0, sizeof(double) * sumrows * (1 + nmu), st));
  DDG_CUDA(cudaMemsetAsync(A, 0, sizeof(double) * nflux * sumM, st));
  std::vector<long long> bset;
  for (int i = 0; i < N; ++i) {
    const ClassPlan& c = p.classes[p.subs[i].cls];
    DDG_CUDA(cudaMemcpy2DAsync(K + static_cast<size_t>(i) * M * sumrows + rowofs[i], sizeof(double) * sumrows,
                               d_A.ptr + i * mstride, sizeof(double) * ld_, sizeof(double) * c.m, M,
                               cudaMemcpyDeviceToDevice, st));
    DDG_CUDA(cudaMemcpyAsync(FB + rowofs[i], d_f.ptr + static_cast<size_t>(i) * p.m, sizeof(double) * c.m,
                             cudaMemcpyDeviceToDevice, st));
    const SubPlan& sp = p.subs[i];
    for (int qq = 0; qq < c.n_gamma; ++qq) {  // B(rowofs + lr, g) = -1 (solvers.cpp:627-628)
      const long long row = rowofs[i] + c.fixed + qq;
      if (sp.gamma_delta[qq] >= 0) bset.push_back((1LL + sp.gamma_delta[qq]) * sumrows + row);
      if (sp.gamma_pi[qq] >= 0) bset.push_back((1LL + nd + sp.gamma_pi[qq]) * sumrows + row);
    }
  }
  // flux scatter (solvers.cpp:629-630, unflipped F rows: the debug flip lives in apply_A only)
  std::vector<int> off(N + 1, 0), erow, elrow;
  std::vector<double> ew;
  for (int i = 0; i < N; ++i) {
    const ClassPlan& c = p.classes[p.subs[i].cls];
    const SubPlan& sp = p.subs[i];
    for (int l = 0; l < c.nF; ++l)
      if (sp.fluxrow_delta[l] >= 0) {
        erow.push_back(sp.fluxrow_delta[l]);
        elrow.push_back(l);
        ew.push_back(1.0);
      }
    for (const CrossRow& cr : sp.cross_rows)
      for (const auto& [l, w] : cr.e) {
        erow.push_back(nd + cr.r);
        elrow.push_back(l);
        ew.push_back(w);
      }
    off[i + 1] = static_cast<int>(erow.size());
  }
  {
    int* doff = s.up(off, st);
    int* drow = s.up(erow, st);
    int* dl = s.up(elrow, st);
    double* dw = s.up(ew, st);
    dense_rows_kernel<<<dim3(ceil_div(M, 128), N), 128, 0, st>>>(A, nflux, d_F.ptr, p.fmax,
                                                                  static_cast<size_t>(M) * p.fmax, doff, drow, dl, dw, M);
    DDG_LAUNCH_CHECK();
    long long* dset = s.up(bset, st);
    if (!bset.empty()) {
      dense_set_kernel<<<ceil_div(static_cast<int>(bset.size()), 256), 256, 0, st>>>(FB, dset,
                                                                                      static_cast<int>(bset.size()), -1.0);
      DDG_LAUNCH_CHECK();
    }
  }

  // ---- Y = K^+ [f | B]
  const int e1 = 1 + nmu;
  double* Y = s.d(static_cast<size_t>(sumM) * e1);
  dense_cod_solve(K, sumrows, sumrows, sumM, FB, sumrows, e1, Y, sumM, st, nullptr);

  o.coeffs.assign(static_cast<size_t>(sumM), 0.0);
  if (method == 0) {
    // one-level (solvers.cpp:637-648): D = -A K^+ B, op = B^T B + D^T D - B^T K K^+ B
    double* Dall = s.d(static_cast<size_t>(nflux) * e1);  // -A [K^+ f | K^+ B]
    dense_gemm(nflux, e1, sumM, -1.0, A, nflux, false, Y, sumM, false, 0.0, Dall, nflux, st);
    double* KY = s.d(static_cast<size_t>(sumrows) * e1);
    dense_gemm(sumrows, e1, sumM, 1.0, K, sumrows, false, Y, sumM, false, 0.0, KY, sumrows, st);
    double* G = s.d(static_cast<size_t>(e1) * e1);
    dense_gemm(e1, e1, sumrows, 1.0, FB, sumrows, true, FB, sumrows, false, 0.0, G, e1, st);
    dense_gemm(e1, e1, nflux, 1.0, Dall, nflux, true, Dall, nflux, false, 1.0, G, e1, st);
    dense_gemm(e1, e1, sumrows, -1.0, FB, sumrows, true, KY, sumrows, false, 1.0, G, e1, st);
    // op = G[1:, 1:], rhs = G[1:, 0]
    double* mu = s.d(nmu);
    dense_cod_solve(G + e1 + 1, e1, nmu, nmu, G + 1, e1, 1, mu, nmu, st, nullptr);
    // c = K^+ (f - B mu) = Y_f - Y_B mu
    double* c = s.d(sumM);
    DDG_CUDA(cudaMemcpyAsync(c, Y, sizeof(double) * sumM, cudaMemcpyDeviceToDevice, st));
    dense_gemm(sumM, 1, nmu, -1.0, Y + sumM, sumM, false, mu, nmu, false, 1.0, c, sumM, st);
    o.dim = nmu;
    o.reduced_op.assign(static_cast<size_t>(nmu) * nmu, 0.0);
    o.reduced_rhs.assign(nmu, 0.0);
    o.mu_full.assign(nmu, 0.0);
    DDG_CUDA(cudaMemcpy2DAsync(o.reduced_op.data(), sizeof(double) * nmu, G + e1 + 1, sizeof(double) * e1,
                               sizeof(double) * nmu, nmu, cudaMemcpyDeviceToHost, st));
    DDG_CUDA(cudaMemcpyAsync(o.reduced_rhs.data(), G + 1, sizeof(double) * nmu, cudaMemcpyDeviceToHost, st));
    DDG_CUDA(cudaMemcpyAsync(o.mu_full.data(), mu, sizeof(double) * nmu, cudaMemcpyDeviceToHost, st));
    DDG_CUDA(cudaMemcpyAsync(o.coeffs.data(), c, sizeof(double) * sumM, cudaMemcpyDeviceToHost, st));
    DDG_CUDA(cudaStreamSynchronize(st));
    return;
  }

  // ---- coarse methods (solvers.cpp:650-708)
  // Dall = -A_Pi [K^+ f | K^+ B_D | K^+ B_Pi] = [dpi | Dpd | Dpp]
  double* Dall = s.d(static_cast<size_t>(npf) * e1);
  dense_gemm(npf, e1, sumM, -1.0, A + nd, nflux, false, Y, sumM, false, 0.0, Dall, std::max(npf, 1), st);
  const int rt = sumrows + npf, ct = sumM + np, e2 = 1 + nd;
  // Kt = [K B_Pi; 0 Dpp], X2 = [ft | Bt] = [f B_D; dpi Dpd]
  double* Kt = s.d(static_cast<size_t>(rt) * ct);
  double* X2 = s.d(static_cast<size_t>(rt) * e2);
  DDG_CUDA(cudaMemsetAsync(Kt, 0, sizeof(double) * rt * ct, st));
  DDG_CUDA(cudaMemcpy2DAsync(Kt, sizeof(double) * rt, K, sizeof(double) * sumrows, sizeof(double) * sumrows, sumM,
                             cudaMemcpyDeviceToDevice, st));
  if (np > 0) {
    DDG_CUDA(cudaMemcpy2DAsync(Kt + static_cast<size_t>(sumM) * rt, sizeof(double) * rt,
                               FB + static_cast<size_t>(1 + nd) * sumrows, sizeof(double) * sumrows,
                               sizeof(double) * sumrows, np, cudaMemcpyDeviceToDevice, st));
    if (npf > 0)
      DDG_CUDA(cudaMemcpy2DAsync(Kt + static_cast<size_t>(sumM) * rt + sumrows, sizeof(double) * rt,
                                 Dall + static_cast<size_t>(1 + nd) * npf, sizeof(double) * npf, sizeof(double) * npf,
                                 np, cudaMemcpyDeviceToDevice, st));
  }
  DDG_CUDA(cudaMemcpy2DAsync(X2, sizeof(double) * rt, FB, sizeof(double) * sumrows, sizeof(double) * sumrows, e2,
                             cudaMemcpyDeviceToDevice, st));
  if (npf > 0)
    DDG_CUDA(cudaMemcpy2DAsync(X2 + sumrows, sizeof(double) * rt, Dall, sizeof(double) * npf, sizeof(double) * npf, e2,
                               cudaMemcpyDeviceToDevice, st));
  // Z = Kt^+ [ft | Bt], KZ = Kt Z, Dt_all = -A_D Z[0:sumM] = [dt | Dt]
  double* Z = s.d(static_cast<size_t>(ct) * e2);
  dense_cod_solve(Kt, rt, rt, ct, X2, rt, e2, Z, ct, st, nullptr);
  double* KZ = s.d(static_cast<size_t>(rt) * e2);
  dense_gemm(rt, e2, ct, 1.0, Kt, rt, false, Z, ct, false, 0.0, KZ, rt, st);
  double* Dt = s.d(static_cast<size_t>(nd) * e2);
  dense_gemm(nd, e2, sumM, -1.0, A, nflux, false, Z, ct, false, 0.0, Dt, nd, st);
  // W = theta P^T P + (1 - theta) I, P = Abar Kbar^+ Bbar (NN), else I
  double* WD = s.d(static_cast<size_t>(nd) * e2);
  if (method == 2 && theta > 0.0) {
    std::vector<int> rowb(N + 1, 0);
    for (int i = 0; i < N; ++i) rowb[i + 1] = rowb[i] + p.classes[p.subs[i].cls].m;
    const int sumrb = rowb[N];
    double* Kb = s.d(static_cast<size_t>(sumrb) * sumM);
    double* Bb = s.d(static_cast<size_t>(sumrb) * nd);
    double* Ab = s.d(static_cast<size_t>(nd) * sumM);
    DDG_CUDA(cudaMemsetAsync(Kb, 0, sizeof(double) * sumrb * sumM, st));
    DDG_CUDA(cudaMemsetAsync(Bb, 0, sizeof(double) * sumrb * nd, st));
    DDG_CUDA(cudaMemsetAsync(Ab, 0, sizeof(double) * nd * sumM, st));
    std::vector<long long> bbset;
    std::vector<int> offb(N + 1, 0), brow, blrow;
    std::vector<double> bw;
    for (int i = 0; i < N; ++i) {
      const ClassPlan& c = p.classes[p.subs[i].cls];
      const SubPlan& sp = p.subs[i];
      DDG_CUDA(cudaMemcpy2DAsync(Kb + static_cast<size_t>(i) * M * sumrb + rowb[i], sizeof(double) * sumrb,
                                 d_A.ptr + (N + i) * mstride, sizeof(double) * ld_, sizeof(double) * c.m, M,
                                 cudaMemcpyDeviceToDevice, st));
      const int r0 = c.fixed + c.nc;  // nflux_row0: the Delta flux rows of Kbar (solvers.cpp:418-431)
      for (int r = 0; r < c.nd; ++r) {
        bbset.push_back(static_cast<long long>(sp.ndelta_map[r]) * sumrb + rowb[i] + r0 + r);
        brow.push_back(sp.ndelta_map[r]);
        blrow.push_back(r);
        bw.push_back(1.0);
      }
      offb[i + 1] = static_cast<int>(brow.size());
    }
    int* doff = s.up(offb, st);
    int* drow = s.up(brow, st);
    int* dl = s.up(blrow, st);
    double* dw = s.up(bw, st);
    dense_rows_kernel<<<dim3(ceil_div(M, 128), N), 128, 0, st>>>(Ab, nd, d_Cd.ptr, p.dmax,
                                                                  static_cast<size_t>(M) * p.dmax, doff, drow, dl, dw, M);
    DDG_LAUNCH_CHECK();
    long long* dset = s.up(bbset, st);
    if (!bbset.empty()) {
      dense_set_kernel<<<ceil_div(static_cast<int>(bbset.size()), 256), 256, 0, st>>>(
          Bb, dset, static_cast<int>(bbset.size()), -1.0);
      DDG_LAUNCH_CHECK();
    }
    double* Yb = s.d(static_cast<size_t>(sumM) * nd);
    dense_cod_solve(Kb, sumrb, sumrb, sumM, Bb, sumrb, nd, Yb, sumM, st, nullptr);
    double* P = s.d(static_cast<size_t>(nd) * nd);
    dense_gemm(nd, nd, sumM, 1.0, Ab, nd, false, Yb, sumM, false, 0.0, P, nd, st);
    double* W = s.d(static_cast<size_t>(nd) * nd);
    dense_gemm(nd, nd, nd, 1.0, P, nd, true, P, nd, false, 0.0, W, nd, st);
    dense_axpy_identity_kernel<<<ceil_div(nd * nd, 256), 256, 0, st>>>(W, nd, theta);
    DDG_LAUNCH_CHECK();
    dense_gemm(nd, e2, nd, 1.0, W, nd, false, Dt, nd, false, 0.0, WD, nd, st);
  } else {
    DDG_CUDA(cudaMemcpyAsync(WD, Dt, sizeof(double) * nd * e2, cudaMemcpyDeviceToDevice, st));
  }
  // G = X2^T X2 + Dt^T W Dt - X2^T KZ: op = G[1:, 1:], rhs = G[1:, 0]
  double* G = s.d(static_cast<size_t>(e2) * e2);
  dense_gemm(e2, e2, rt, 1.0, X2, rt, true, X2, rt, false, 0.0, G, e2, st);
  dense_gemm(e2, e2, nd, 1.0, Dt, nd, true, WD, nd, false, 1.0, G, e2, st);
  dense_gemm(e2, e2, rt, -1.0, X2, rt, true, KZ, rt, false, 1.0, G, e2, st);
  double* mu = s.d(nd);
  dense_cod_solve(G + e2 + 1, e2, nd, nd, G + 1, e2, 1, mu, nd, st, nullptr);
  // cmu = Kt^+ (ft - Bt mu) = Z_ft - Z_Bt mu
  double* cmu = s.d(ct);
  DDG_CUDA(cudaMemcpyAsync(cmu, Z, sizeof(double) * ct, cudaMemcpyDeviceToDevice, st));
  dense_gemm(ct, 1, nd, -1.0, Z + ct, ct, false, mu, nd, false, 1.0, cmu, ct, st);
  o.dim = nd;
  o.reduced_op.assign(static_cast<size_t>(nd) * nd, 0.0);
  o.reduced_rhs.assign(nd, 0.0);
  o.mu_full.assign(nmu, 0.0);
  DDG_CUDA(cudaMemcpy2DAsync(o.reduced_op.data(), sizeof(double) * nd, G + e2 + 1, sizeof(double) * e2,
                             sizeof(double) * nd, nd, cudaMemcpyDeviceToHost, st));
  DDG_CUDA(cudaMemcpyAsync(o.reduced_rhs.data(), G + 1, sizeof(double) * nd, cudaMemcpyDeviceToHost, st));
  DDG_CUDA(cudaMemcpyAsync(o.mu_full.data(), mu, sizeof(double) * nd, cudaMemcpyDeviceToHost, st));
  if (np > 0)
    DDG_CUDA(cudaMemcpyAsync(o.mu_full.data() + nd, cmu + sumM, sizeof(double) * np, cudaMemcpyDeviceToHost, st));
  DDG_CUDA(cudaMemcpyAsync(o.coeffs.data(), cmu, sizeof(double) * sumM, cudaMemcpyDeviceToHost, st));
  DDG_CUDA(cudaStreamSynchronize(st));
}

}  // namespace ddg

// ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.hpp).
// Dense kernels standing in for the Eigen calls the reference makes:
//   HouseholderQR            solvers.cpp:27-29, 44
//   ColPivHouseholderQR/COD  solvers.cpp:35-40 (via Eigen::CompleteOrthogonalDecomposition)
//   LLT                      solvers.cpp:322
#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <limits>

#include "oracle.hpp"

namespace ddo {

Vec gemv(const Mat& A, const Vec& x) {
  Vec y;
  if (blas_gemv(false, A, x, y)) return y;
  y.assign(A.r, 0.0);
  for (int j = 0; j < A.c; ++j) {
    const double xj = x[j];
    if (xj == 0.0) continue;  // exact zero contributes exactly zero
    const double* a = A.col(j);
    for (int i = 0; i < A.r; ++i) y[i] += a[i] * xj;
  }
  return y;
}

Vec gemv_t(const Mat& A, const Vec& x) {
  Vec y;
  if (blas_gemv(true, A, x, y)) return y;
  y.assign(A.c, 0.0);
  for (int j = 0; j < A.c; ++j) {
    const double* a = A.col(j);
    double s = 0;
    for (int i = 0; i < A.r; ++i) s += a[i] * x[i];
    y[j] = s;
  }
  return y;
}

Mat matmul(const Mat& A, const Mat& B) {
  Mat C(A.r, B.c);
  for (int j = 0; j < B.c; ++j) {
    double* c = C.col(j);
    for (int k = 0; k < A.c; ++k) {
      const double bkj = B(k, j);
      if (bkj == 0.0) continue;
      const double* a = A.col(k);
      for (int i = 0; i < A.r; ++i) c[i] += a[i] * bkj;
    }
  }
  return C;
}

Mat transpose(const Mat& A) {
  Mat T(A.c, A.r);
  for (int j = 0; j < A.c; ++j)
    for (int i = 0; i < A.r; ++i) T(j, i) = A(i, j);
  return T;
}

double dot(const Vec& a, const Vec& b) {
  double s = 0;
  for (size_t i = 0; i < a.size(); ++i) s += a[i] * b[i];
  return s;
}

double norm(const Vec& a) { return std::sqrt(dot(a, a)); }

namespace {

/// makeHouseholderInPlace on x[0..n): on return x[1..n) holds the essential part,
/// tau and beta as in Eigen/LAPACK dlarfg.
void make_householder(double* x, int stride, int n, double& tau, double& beta) {
  const double c0 = x[0];
  double tail_sq = 0;
  for (int i = 1; i < n; ++i) tail_sq += x[i * stride] * x[i * stride];
  const double tiny = std::numeric_limits<double>::min();
  if (tail_sq <= tiny) {
    tau = 0;
    beta = c0;
    for (int i = 1; i < n; ++i) x[i * stride] = 0;
    return;
  }
  beta = std::sqrt(c0 * c0 + tail_sq);
  if (c0 >= 0) beta = -beta;
  const double scale = 1.0 / (c0 - beta);
  for (int i = 1; i < n; ++i) x[i * stride] *= scale;
  tau = (beta - c0) / beta;
}

/// Apply H = I - tau [1; v][1; v]^T from the left to rows [r0, r0+n) of columns
/// [c0, c1) of A, with v = A(r0+1 .. r0+n-1, vcol).
void apply_left(Mat& A, int r0, int n, int c0, int c1, const double* v, double tau) {
  if (tau == 0.0) return;
  for (int j = c0; j < c1; ++j) {
    double* a = A.col(j) + r0;
    double s = a[0];
    for (int i = 1; i < n; ++i) s += v[i - 1] * a[i];
    s *= tau;
    a[0] -= s;
    for (int i = 1; i < n; ++i) a[i] -= s * v[i - 1];
  }
}

/// Q = H_0 ... H_{ncols-1} I(rows, ncols) from reflectors stored below the diagonal.
Mat form_q(const Mat& qr, const Vec& tau, int ncols) {
  const int m = qr.r;
  Mat Q(m, ncols);
  for (int j = 0; j < ncols; ++j) Q(j, j) = 1.0;
  for (int k = ncols - 1; k >= 0; --k) apply_left(Q, k, m - k, k, ncols, qr.col(k) + k + 1, tau[k]);
  return Q;
}

}  // namespace

// ------------------------------------------------------------- HouseholderQR
void HouseholderQR::compute(const Mat& A) {
  qr = A;
  const int m = qr.r, n = qr.c, size = std::min(m, n);
  hcoeffs.assign(size, 0.0);
  for (int k = 0; k < size; ++k) {
    double tau, beta;
    make_householder(qr.col(k) + k, 1, m - k, tau, beta);
    qr(k, k) = beta;
    hcoeffs[k] = tau;
    apply_left(qr, k, m - k, k + 1, n, qr.col(k) + k + 1, tau);
  }
}

Mat HouseholderQR::thinQ() const { return form_q(qr, hcoeffs, std::min(qr.r, qr.c)); }

// ------------------------------------------------------------- ColPivQR
void ColPivQR::compute(const Mat& A) {
  qr = A;
  const int rows = qr.r, cols = qr.c, size = std::min(rows, cols);
  hcoeffs.assign(size, 0.0);
  transpositions.assign(size, 0);
  perm.resize(cols);
  for (int j = 0; j < cols; ++j) perm[j] = j;
  Vec upd(cols), direct(cols);
  double maxnorm = 0;
  for (int j = 0; j < cols; ++j) {
    const double* a = qr.col(j);
    double s = 0;
    for (int i = 0; i < rows; ++i) s += a[i] * a[i];
    upd[j] = direct[j] = std::sqrt(s);
    maxnorm = std::max(maxnorm, upd[j]);
  }
  const double eps = std::numeric_limits<double>::epsilon();
  const double threshold_helper = (maxnorm * eps) * (maxnorm * eps) / rows;
  const double downdate_thr = std::sqrt(eps);
  nonzero_pivots = size;
  maxpivot = 0;
  for (int k = 0; k < size; ++k) {
    int best = k;
    for (int j = k + 1; j < cols; ++j)
      if (upd[j] > upd[best]) best = j;  // first index wins ties
    const double best_sq = upd[best] * upd[best];
    if (nonzero_pivots == size && best_sq < threshold_helper * (rows - k)) nonzero_pivots = k;
    transpositions[k] = best;
    if (best != k) {
      std::swap_ranges(qr.col(k), qr.col(k) + rows, qr.col(best));
      std::swap(upd[k], upd[best]);
      std::swap(direct[k], direct[best]);
      std::swap(perm[k], perm[best]);
    }
    double tau, beta;
    make_householder(qr.col(k) + k, 1, rows - k, tau, beta);
    qr(k, k) = beta;
    hcoeffs[k] = tau;
    maxpivot = std::max(maxpivot, std::abs(beta));
    apply_left(qr, k, rows - k, k + 1, cols, qr.col(k) + k + 1, tau);
    for (int j = k + 1; j < cols; ++j) {
      if (upd[j] == 0.0) continue;
      double t = std::abs(qr(k, j)) / upd[j];
      t = (1.0 + t) * (1.0 - t);
      if (t < 0) t = 0;
      const double ratio = upd[j] / direct[j];
      const double t2 = t * ratio * ratio;
      if (t2 <= downdate_thr) {
        const double* a = qr.col(j) + k + 1;
        double s = 0;
        for (int i = 0; i < rows - k - 1; ++i) s += a[i] * a[i];
        direct[j] = upd[j] = std::sqrt(s);
      } else {
        upd[j] *= std::sqrt(t);
      }
    }
  }
}

int ColPivQR::rank(double threshold) const {
  const double pre = std::abs(maxpivot) * threshold;
  int r = 0;
  for (int i = 0; i < nonzero_pivots; ++i) r += (std::abs(qr(i, i)) > pre) ? 1 : 0;
  return r;
}

// ------------------------------------------------------------- COD
void COD::compute(const Mat& A, double thr) {
  threshold = thr;
  cpqr.compute(A);
  rnk = cpqr.rank(thr);
  Mat& X = cpqr.qr;
  const int cols = X.c;
  const int r = rnk;
  zcoeffs.assign(std::min(X.r, X.c), 0.0);
  if (r == 0 || r >= cols) return;
  std::vector<double> row(cols - r + 1);
  for (int k = r - 1; k >= 0; --k) {
    if (k != r - 1)
      for (int i = 0; i <= k; ++i) std::swap(X(i, k), X(i, r - 1));
    // Householder on [X(k, r-1), X(k, r:cols)], from the right.
    for (int j = 0; j < cols - r + 1; ++j) row[j] = X(k, r - 1 + j);
    double tau, beta;
    make_householder(row.data(), 1, cols - r + 1, tau, beta);
    zcoeffs[k] = tau;
    X(k, r - 1) = beta;
    for (int j = 1; j < cols - r + 1; ++j) X(k, r - 1 + j) = row[j];
    if (k > 0 && tau != 0.0) {
      // rows 0..k-1 of columns {r-1, r..cols-1}: B <- B (I - tau v v^T), v = [1; ess]
      for (int i = 0; i < k; ++i) {
        double s = X(i, r - 1);
        for (int j = 1; j < cols - r + 1; ++j) s += X(i, r - 1 + j) * row[j];
        s *= tau;
        X(i, r - 1) -= s;
        for (int j = 1; j < cols - r + 1; ++j) X(i, r - 1 + j) -= s * row[j];
      }
    }
    if (k != r - 1)
      for (int i = 0; i <= k; ++i) std::swap(X(i, k), X(i, r - 1));
  }
}

Mat COD::solve(const Mat& B) const {
  const Mat& X = cpqr.qr;
  const int rows = X.r, cols = X.c, r = rnk, nrhs = B.c;
  Mat dst(cols, nrhs);
  if (r == 0) return dst;
  Mat c = B;
  // c = Q^T B with the first r reflectors: H_0 first.
  for (int k = 0; k < r; ++k) apply_left(c, k, rows - k, 0, nrhs, X.col(k) + k + 1, cpqr.hcoeffs[k]);
  // T z = c(0:r): back substitution with T = upper triangle of X(0:r, 0:r).
  for (int j = 0; j < nrhs; ++j) {
    for (int i = r - 1; i >= 0; --i) {
      double s = c(i, j);
      for (int t = i + 1; t < r; ++t) s -= X(i, t) * dst(t, j);
      dst(i, j) = s / X(i, i);
    }
  }
  if (r < cols) {
    // y = Z^T [z; 0]: apply Z(0), Z(1), ..., Z(r-1) on rows {k} U {r..cols-1}.
    for (int k = 0; k < r; ++k) {
      const double tau = zcoeffs[k];
      if (tau == 0.0) continue;
      for (int j = 0; j < nrhs; ++j) {
        double* y = dst.col(j);
        if (k != r - 1) std::swap(y[k], y[r - 1]);
        double s = y[r - 1];
        for (int t = r; t < cols; ++t) s += X(k, t) * y[t];
        s *= tau;
        y[r - 1] -= s;
        for (int t = r; t < cols; ++t) y[t] -= s * X(k, t);
        if (k != r - 1) std::swap(y[k], y[r - 1]);
      }
    }
  }
  // x = P y: x[perm[k]] = y[k]
  Mat out(cols, nrhs);
  for (int j = 0; j < nrhs; ++j)
    for (int k = 0; k < cols; ++k) out(cpqr.perm[k], j) = dst(k, j);
  return out;
}

Mat COD::pseudo_inverse() const { return solve(Mat::identity(cpqr.qr.r)); }

Mat COD::householderQ_cols(int ncols) const { return form_q(cpqr.qr, cpqr.hcoeffs, ncols); }

namespace {
Vec upper_solve(const Mat& R, const Vec& b);
Vec upper_t_solve(const Mat& R, const Vec& b);
}  // namespace
static bool rinv_probe();

// ------------------------------------------------------------- LsFactor (solvers.cpp:24-78)
LsFactor::LsFactor(const Mat& K, double rank_tol) : rows_(K.r), cols_(K.c) {
  if (rows_ < cols_) throw std::invalid_argument("LsFactor: matrix must be square or tall");
  if (lapack_enabled()) {  // CPU-baseline mode (lapack.cpp): the same contract on LAPACK
    lapack_lsfactor(K, rank_tol, deficient_, rank_, qr_diag_ratio, Q_, R_, K_, pinv_);
    return;
  }
  HouseholderQR qr;
  qr.compute(K);
  double dmax = 0, dmin = std::numeric_limits<double>::infinity();
  for (int i = 0; i < cols_; ++i) {
    const double d = std::abs(qr.qr(i, i));
    dmax = std::max(dmax, d);
    dmin = std::min(dmin, d);
  }
  qr_diag_ratio = dmax > 0 ? dmin / dmax : 0.0;
  if (!(dmax > 0) || dmin < rank_tol * dmax) {
    deficient_ = true;
    K_ = K;
    COD cod;
    cod.compute(K, rank_tol);
    pinv_ = cod.pseudo_inverse();
    rank_ = cod.rnk;
    Q_ = cod.householderQ_cols(rank_);
    return;
  }
  rank_ = cols_;
  R_ = Mat(cols_, cols_);
  for (int j = 0; j < cols_; ++j)
    for (int i = 0; i <= j; ++i) R_(i, j) = qr.qr(i, j);
  Q_ = qr.thinQ();
  if (rinv_probe()) {
    Rinv_ = Mat(cols_, cols_);
    for (int c = 0; c < cols_; ++c) {
      Vec e(cols_, 0.0);
      e[c] = 1.0;
      Vec x = upper_solve(R_, e);
      std::copy(x.begin(), x.end(), Rinv_.col(c));
    }
  }
}

namespace {
Vec upper_solve(const Mat& R, const Vec& b) {
  const int n = R.c;
  Vec x(n);
  for (int i = n - 1; i >= 0; --i) {
    double s = b[i];
    for (int t = i + 1; t < n; ++t) s -= R(i, t) * x[t];
    x[i] = s / R(i, i);
  }
  return x;
}
Vec upper_t_solve(const Mat& R, const Vec& b) {  // R^T x = b
  const int n = R.c;
  Vec x(n);
  for (int i = 0; i < n; ++i) {
    double s = b[i];
    const double* ri = R.col(i);
    for (int t = 0; t < i; ++t) s -= ri[t] * x[t];
    x[i] = s / R(i, i);
  }
  return x;
}
}  // namespace

// Oracle-spread probe (test infrastructure): DDO_RINV=1 applies an explicit R^{-1} in the
// full-rank branch (as the device path does) instead of triangular solves.
static bool rinv_probe() {
  static const bool on = std::getenv("DDO_RINV") != nullptr;
  return on;
}

Vec LsFactor::apply_pinv(const Vec& v) const {
  if (deficient_) return gemv(pinv_, v);
  if (rinv_probe()) return gemv(Rinv_, gemv_t(Q_, v));
  return upper_solve(R_, gemv_t(Q_, v));
}

Vec LsFactor::apply_pinv_transpose(const Vec& v) const {
  if (deficient_) return gemv_t(pinv_, v);
  if (rinv_probe()) return gemv(Q_, gemv_t(Rinv_, v));
  return gemv(Q_, upper_t_solve(R_, v));
}

Vec LsFactor::apply_matrix(const Vec& x) const {
  if (deficient_) return gemv(K_, x);
  Vec rx(cols_, 0.0);
  for (int i = 0; i < cols_; ++i) {
    double s = 0;
    for (int t = i; t < cols_; ++t) s += R_(i, t) * x[t];
    rx[i] = s;
  }
  return gemv(Q_, rx);
}

Vec LsFactor::apply_projection(const Vec& v) const { return gemv(Q_, gemv_t(Q_, v)); }

Mat LsFactor::apply_pinv(const Mat& V) const {
  Mat out(cols_, V.c);
  for (int j = 0; j < V.c; ++j) {
    Vec v(V.col(j), V.col(j) + V.r);
    bool zero = true;
    for (double e : v) zero = zero && e == 0.0;
    if (zero) continue;  // pinv * 0 == 0 exactly
    Vec y = apply_pinv(v);
    std::copy(y.begin(), y.end(), out.col(j));
  }
  return out;
}

Mat LsFactor::apply_projection(const Mat& V) const {
  Mat out(rows_, V.c);
  for (int j = 0; j < V.c; ++j) {
    Vec v(V.col(j), V.col(j) + V.r);
    bool zero = true;
    for (double e : v) zero = zero && e == 0.0;
    if (zero) continue;
    Vec y = apply_projection(v);
    std::copy(y.begin(), y.end(), out.col(j));
  }
  return out;
}

// ------------------------------------------------------------- LLT
void LLT::compute(const Mat& A) {
  const int n = A.r;
  L = Mat(n, n);
  ok = true;
  for (int j = 0; j < n; ++j) {
    double d = A(j, j);
    for (int k = 0; k < j; ++k) d -= L(j, k) * L(j, k);
    if (!(d > 0)) {
      ok = false;
      return;
    }
    d = std::sqrt(d);
    L(j, j) = d;
    for (int i = j + 1; i < n; ++i) {
      double s = A(i, j);
      for (int k = 0; k < j; ++k) s -= L(i, k) * L(j, k);
      L(i, j) = s / d;
    }
  }
}

Vec LLT::solve(const Vec& b) const {
  const int n = L.r;
  Vec y(n), x(n);
  for (int i = 0; i < n; ++i) {
    double s = b[i];
    for (int k = 0; k < i; ++k) s -= L(i, k) * y[k];
    y[i] = s / L(i, i);
  }
  for (int i = n - 1; i >= 0; --i) {
    double s = y[i];
    for (int k = i + 1; k < n; ++k) s -= L(k, i) * x[k];
    x[i] = s / L(i, i);
  }
  return x;
}

}  // namespace ddo

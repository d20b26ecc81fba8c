// ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.hpp).
// LAPACK-backed LsFactor (solvers.cpp:24-45) for the CPU baseline / reference arm of bench.py:
// the same branch logic as the restatement in linalg.cpp, with the factorisations done by the
// LAPACK routines closest to the Eigen calls the reference makes:
//   HouseholderQR                       -> dgeqrf (+ dorgqr for the thin Q)
//   CompleteOrthogonalDecomposition     -> dgeqp3 (column-pivoted QR) + dtzrzf (RZ of [R11 R12])
//   pseudoInverse()                     -> P Z^T [T^{-1} Q_r^T; 0]  (dtrsm, dormrz)
// The LAPACK is the one SciPy ships (libscipy_openblas, symbols scipy_d*_), loaded with dlopen
// from the path ddo_set_lapack() receives, single-threaded per call (the reference parallelises
// over subdomains, workers = nproc, not inside a factorisation).
#include <dlfcn.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <stdexcept>
#include <string>
#include <vector>

#include "oracle.hpp"

namespace ddo {

namespace {
using dgeqrf_t = void (*)(const int*, const int*, double*, const int*, double*, double*, const int*, int*);
using dgeqp3_t = void (*)(const int*, const int*, double*, const int*, int*, double*, double*, const int*, int*);
using dtzrzf_t = void (*)(const int*, const int*, double*, const int*, double*, double*, const int*, int*);
using dorgqr_t = void (*)(const int*, const int*, const int*, double*, const int*, const double*, double*, const int*,
                          int*);
using dormrz_t = void (*)(const char*, const char*, const int*, const int*, const int*, const int*, const double*,
                          const int*, const double*, double*, const int*, double*, const int*, int*, size_t, size_t);
using dtrsm_t = void (*)(const char*, const char*, const char*, const char*, const int*, const int*, const double*,
                         const double*, const int*, double*, const int*, size_t, size_t, size_t, size_t);
using setthreads_t = void (*)(int);
using dgemv_t = void (*)(const char*, const int*, const int*, const double*, const double*, const int*, const double*,
                         const int*, const double*, double*, const int*, size_t);

struct Lapack {
  dgeqrf_t geqrf = nullptr;
  dgeqp3_t geqp3 = nullptr;
  dtzrzf_t tzrzf = nullptr;
  dorgqr_t orgqr = nullptr;
  dormrz_t ormrz = nullptr;
  dtrsm_t trsm = nullptr;
  dgemv_t gemv = nullptr;
  std::string path;
};
std::atomic<Lapack*> g_lapack{nullptr};

template <class F>
void sym(void* h, const char* name, F& f) {
  f = reinterpret_cast<F>(dlsym(h, name));
  if (!f) throw std::runtime_error(std::string("LAPACK symbol missing: ") + name);
}

void check(int info, const char* what) {
  if (info != 0) throw std::runtime_error(std::string(what) + ": LAPACK info " + std::to_string(info));
}
}  // namespace

bool set_lapack(const char* path) {
  if (!path || !*path) {
    g_lapack.store(nullptr);
    return true;
  }
  void* h = dlopen(path, RTLD_NOW | RTLD_LOCAL);
  if (!h) throw std::runtime_error(std::string("dlopen failed: ") + dlerror());
  auto* L = new Lapack;  // kept for the process lifetime
  sym(h, "scipy_dgeqrf_", L->geqrf);
  sym(h, "scipy_dgeqp3_", L->geqp3);
  sym(h, "scipy_dtzrzf_", L->tzrzf);
  sym(h, "scipy_dorgqr_", L->orgqr);
  sym(h, "scipy_dormrz_", L->ormrz);
  sym(h, "scipy_dtrsm_", L->trsm);
  sym(h, "scipy_dgemv_", L->gemv);
  setthreads_t st = nullptr;
  if ((st = reinterpret_cast<setthreads_t>(dlsym(h, "scipy_openblas_set_num_threads"))) != nullptr) st(1);
  L->path = path;
  g_lapack.store(L);
  return true;
}

bool lapack_enabled() { return g_lapack.load() != nullptr; }

bool blas_gemv(bool trans, const Mat& A, const Vec& x, Vec& y) {
  const Lapack* L = g_lapack.load();
  if (!L || A.r == 0 || A.c == 0) return false;
  const int m = A.r, n = A.c, inc = 1;
  const double one = 1.0, zero = 0.0;
  y.assign(trans ? n : m, 0.0);
  L->gemv(trans ? "T" : "N", &m, &n, &one, A.a.data(), &m, x.data(), &inc, &zero, y.data(), &inc, 1);
  return true;
}

/// LAPACK version of the LsFactor constructor: fills the same members as the restatement.
void lapack_lsfactor(const Mat& K, double rank_tol, bool& deficient, int& rank, double& ratio, Mat& Q, Mat& R,
                     Mat& Kcopy, Mat& pinv) {
  const Lapack* L = g_lapack.load();
  const int m = K.r, n = K.c, lwq = -1;
  int info = 0;
  double wq = 0;
  // unpivoted Householder QR (solvers.cpp:27-32): the branch test on |R_ii|
  Mat A = K;
  std::vector<double> tau(n);
  L->geqrf(&m, &n, A.a.data(), &m, tau.data(), &wq, &lwq, &info);
  int lw = std::max(1, static_cast<int>(wq));
  std::vector<double> work(lw);
  L->geqrf(&m, &n, A.a.data(), &m, tau.data(), work.data(), &lw, &info);
  check(info, "dgeqrf");
  double dmax = 0, dmin = INFINITY;
  for (int i = 0; i < n; ++i) {
    dmax = std::max(dmax, std::abs(A(i, i)));
    dmin = std::min(dmin, std::abs(A(i, i)));
  }
  ratio = dmax > 0 ? dmin / dmax : 0.0;
  if (dmax > 0 && !(dmin < rank_tol * dmax)) {
    // full rank (solvers.cpp:43-44): R and the thin Q
    deficient = false;
    rank = n;
    R = Mat(n, n);
    for (int j = 0; j < n; ++j)
      for (int i = 0; i <= j; ++i) R(i, j) = A(i, j);
    L->orgqr(&m, &n, &n, A.a.data(), &m, tau.data(), &wq, &lwq, &info);
    lw = std::max(1, static_cast<int>(wq));
    work.resize(lw);
    L->orgqr(&m, &n, &n, A.a.data(), &m, tau.data(), work.data(), &lw, &info);
    check(info, "dorgqr");
    Q = std::move(A);
    return;
  }
  // complete orthogonal decomposition (solvers.cpp:33-41)
  deficient = true;
  Kcopy = K;
  Mat B = K;
  std::vector<int> jpvt(n, 0);
  std::vector<double> tp(n);
  L->geqp3(&m, &n, B.a.data(), &m, jpvt.data(), tp.data(), &wq, &lwq, &info);
  lw = std::max(1, static_cast<int>(wq));
  work.resize(lw);
  L->geqp3(&m, &n, B.a.data(), &m, jpvt.data(), tp.data(), work.data(), &lw, &info);
  check(info, "dgeqp3");
  double maxpiv = 0;
  for (int i = 0; i < n; ++i) maxpiv = std::max(maxpiv, std::abs(B(i, i)));
  int r = 0;
  for (int i = 0; i < n; ++i)
    if (std::abs(B(i, i)) > rank_tol * maxpiv) ++r;
  rank = r;
  pinv = Mat(n, m);
  Q = Mat(m, r);
  if (r == 0) return;
  // Q_r: the first r pivoted-QR reflectors applied to I (on a copy: dtzrzf overwrites the top rows)
  Mat Qr(m, r);
  for (int j = 0; j < r; ++j) std::copy(B.col(j), B.col(j) + m, Qr.col(j));
  L->orgqr(&m, &r, &r, Qr.a.data(), &m, tp.data(), &wq, &lwq, &info);
  lw = std::max(1, static_cast<int>(wq));
  work.resize(lw);
  L->orgqr(&m, &r, &r, Qr.a.data(), &m, tp.data(), work.data(), &lw, &info);
  check(info, "dorgqr");
  // RZ of the r x n trapezoid [R11 R12] = [T 0] Z
  std::vector<double> tz(r);
  if (r < n) {
    L->tzrzf(&r, &n, B.a.data(), &m, tz.data(), &wq, &lwq, &info);
    lw = std::max(1, static_cast<int>(wq));
    work.resize(lw);
    L->tzrzf(&r, &n, B.a.data(), &m, tz.data(), work.data(), &lw, &info);
    check(info, "dtzrzf");
  }
  // W = [T^{-1} Q_r^T ; 0]  (n x m), then W <- Z^T W, then rows permuted back (P)
  Mat W(n, m);
  for (int j = 0; j < m; ++j)
    for (int i = 0; i < r; ++i) W(i, j) = Qr(j, i);
  const double one = 1.0;
  L->trsm("L", "U", "N", "N", &r, &m, &one, B.a.data(), &m, W.a.data(), &n, 1, 1, 1, 1);
  if (r < n) {
    const int l = n - r;
    L->ormrz("L", "T", &n, &m, &r, &l, B.a.data(), &m, tz.data(), W.a.data(), &n, &wq, &lwq, &info, 1, 1);
    lw = std::max(1, static_cast<int>(wq));
    work.resize(lw);
    L->ormrz("L", "T", &n, &m, &r, &l, B.a.data(), &m, tz.data(), W.a.data(), &n, work.data(), &lw, &info, 1, 1);
    check(info, "dormrz");
  }
  for (int i = 0; i < n; ++i) {
    const int orig = jpvt[i] - 1;  // column i of A P is column jpvt[i] of A (1-based)
    for (int j = 0; j < m; ++j) pinv(orig, j) = W(i, j);
  }
  Q = std::move(Qr);
}

}  // namespace ddo

// ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.hpp).
// C ABI over the restatement so pytest / tools/make_goldens.py / bench.py's CPU legs can
// drive it through ctypes. Mirrors the reference's run() (runner.cpp:126-155): build the
// Workspace, dispatch the method, evaluate the field.
#include <cstdint>
#include <unordered_map>
#include <algorithm>
#include <chrono>
#include <limits>
#include <random>
#include <cstring>
#include <memory>

#include "oracle.hpp"

using namespace ddo;

extern "C" {

struct ddo_config {
  const char* problem;
  int s, n_grid, M;
  double l;
  unsigned long long seed;
  int method;  // 0 ddelm, 1 ddelm-cs, 2 ddelm-nn
  double theta;
  int flux_variant;         // 0 pointwise, 1 mean_edge
  int change_of_variables;  // 0 nodal, 1 change_of_variables
  double cg_rel_tol;
  int cg_max_iter, cg_stop_after;
  int workers, cg_workers;
  int debug_flip_flux_row;
  int layers_only;  // 1: partition + seeded layers only (field evaluation of given coefficients)
  double alpha;     // ProblemParams (problems.hpp:64-68): GRF smoothness and seeds
  unsigned long long forcing_seed, rho_seed;
};

struct ddo_handle {
  std::unique_ptr<Workspace> ws;
  SolveReport rep;
  bool solved = false;
  double build_seconds = 0;
};

static void set_err(char* err, int n, const char* msg) {
  if (err && n > 0) {
    std::strncpy(err, msg, n - 1);
    err[n - 1] = 0;
  }
}

void* ddo_create(const ddo_config* c, char* err, int errlen) {
  try {
    auto h = new ddo_handle;
    SolverOptions o;
    o.flux_variant = c->flux_variant ? FluxVariant::MeanEdge : FluxVariant::Pointwise;
    o.change_of_variables = c->change_of_variables != 0;
    o.workers = c->workers;
    o.cg_workers = c->cg_workers;
    o.debug_flip_flux_row = c->debug_flip_flux_row;
    o.layers_only = c->layers_only != 0;
    const auto t0 = std::chrono::steady_clock::now();
    ProblemParams pp;
    pp.alpha = c->alpha;
    pp.forcing_seed = c->forcing_seed;
    pp.rho_seed = c->rho_seed;
    h->ws = std::make_unique<Workspace>(make_problem(c->problem, pp), c->s, c->n_grid, c->M, c->l,
                                        c->seed, o);
    h->build_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return h;
  } catch (const std::exception& e) {
    set_err(err, errlen, e.what());
    return nullptr;
  }
}

void ddo_destroy(void* p) { delete static_cast<ddo_handle*>(p); }

int ddo_solve(void* p, int method, double theta, double rel_tol, int max_iter, int stop_after,
              char* err, int errlen) {
  auto h = static_cast<ddo_handle*>(p);
  try {
    CgOptions o{rel_tol, max_iter, stop_after};
    if (method == 0) h->rep = ddelm_solve(*h->ws, o);
    else if (method == 1) h->rep = ddelm_cs_solve(*h->ws, o);
    else h->rep = ddelm_nn_solve(*h->ws, theta, o);
    h->solved = true;
    return 0;
  } catch (const std::invalid_argument& e) {
    set_err(err, errlen, e.what());
    return 2;
  } catch (const std::exception& e) {
    set_err(err, errlen, e.what());
    return 3;
  }
}

/// info[0..]: n_subs, n_delta, n_pi, n_mu, M, rows, iterations, converged, negative_curvature,
/// n_residuals, n_pi_flux
void ddo_info(void* p, int* info) {
  auto h = static_cast<ddo_handle*>(p);
  const Workspace& ws = *h->ws;
  info[0] = ws.n_subs();
  info[1] = ws.n_delta();
  info[2] = ws.n_pi();
  info[3] = ws.n_mu();
  info[4] = ws.layers[0].M;
  info[5] = ws.blocks[0].rows();
  info[6] = h->rep.iterations;
  info[7] = h->rep.converged ? 1 : 0;
  info[8] = h->rep.negative_curvature ? 1 : 0;
  info[9] = static_cast<int>(h->rep.residual_history.size());
  info[10] = ws.n_pi_flux();
}

/// t[0..5]: assembly, factorization, setup (coarse+neumann+rhs), cg, reconstruct, build total
void ddo_timings(void* p, double* t) {
  auto h = static_cast<ddo_handle*>(p);
  t[0] = h->ws->assembly_seconds;
  t[1] = h->ws->factorization_seconds;
  t[2] = h->rep.setup_seconds;
  t[3] = h->rep.cg_seconds;
  t[4] = h->rep.reconstruct_seconds;
  t[5] = h->build_seconds;
}

void ddo_residuals(void* p, double* out) {
  auto h = static_cast<ddo_handle*>(p);
  std::copy(h->rep.residual_history.begin(), h->rep.residual_history.end(), out);
}

void ddo_mu(void* p, double* out) {
  auto h = static_cast<ddo_handle*>(p);
  std::copy(h->rep.mu.begin(), h->rep.mu.end(), out);
}

void ddo_coeffs(void* p, double* out) {
  auto h = static_cast<ddo_handle*>(p);
  const int M = h->ws->layers[0].M;
  for (size_t i = 0; i < h->rep.coeffs.size(); ++i)
    std::copy(h->rep.coeffs[i].begin(), h->rep.coeffs[i].end(), out + i * M);
}

/// Per-subdomain ranks of K (and of Kbar when the Neumann layer was built, else -1).
void ddo_ranks(void* p, int* rk, int* rkbar, double* qr_ratio) {
  auto h = static_cast<ddo_handle*>(p);
  const Workspace& ws = *h->ws;
  for (int i = 0; i < ws.n_subs(); ++i) {
    rk[i] = ws.fac[i].rank();
    rkbar[i] = ws.neumann_built ? ws.nfac[i].rank() : -1;
    qr_ratio[2 * i] = ws.fac[i].qr_diag_ratio;
    qr_ratio[2 * i + 1] = ws.neumann_built ? ws.nfac[i].qr_diag_ratio : -1.0;
  }
}

void ddo_layer(void* p, int i, double* w0, double* w1, double* b) {
  auto h = static_cast<ddo_handle*>(p);
  const FeatureLayer& L = h->ws->layers[i];
  std::copy(L.w0.begin(), L.w0.end(), w0);
  std::copy(L.w1.begin(), L.w1.end(), w1);
  std::copy(L.b.begin(), L.b.end(), b);
}

/// Local matrix K_i (rows x M, column-major) and f_i.
void ddo_local(void* p, int i, double* K, double* f) {
  auto h = static_cast<ddo_handle*>(p);
  const LocalBlocks& b = h->ws->blocks[i];
  std::copy(b.K.a.begin(), b.K.a.end(), K);
  std::copy(b.f.begin(), b.f.end(), f);
}

/// Neumann matrix Kbar_i (rows x M) — requires the Neumann layer.
int ddo_kbar(void* p, int i, double* K) {
  auto h = static_cast<ddo_handle*>(p);
  if (!h->ws->neumann_built) return 1;
  const Mat& Kb = h->ws->Kbar[i];
  std::copy(Kb.a.begin(), Kb.a.end(), K);
  return 0;
}

/// Field and gradient samples on the n x n grid (metrics.cpp:18-57), index b*n + a.
void ddo_field(void* p, int n, double* u, double* gx, double* gy) {
  auto h = static_cast<ddo_handle*>(p);
  FieldSamples fs = sample_field(h->ws->part, h->ws->layers, h->rep.coeffs, n);
  std::copy(fs.u.begin(), fs.u.end(), u);
  std::copy(fs.gx.begin(), fs.gx.end(), gx);
  std::copy(fs.gy.begin(), fs.gy.end(), gy);
}

/// Field of caller-supplied coefficients (N x M) with this workspace's layers.
void ddo_field_of(void* p, const double* coeffs, int n, double* u, double* gx, double* gy) {
  auto h = static_cast<ddo_handle*>(p);
  const int N = h->ws->n_subs(), M = h->ws->layers[0].M;
  LocalVecs c(N);
  for (int i = 0; i < N; ++i) c[i].assign(coeffs + static_cast<size_t>(i) * M, coeffs + static_cast<size_t>(i + 1) * M);
  FieldSamples fs = sample_field(h->ws->part, h->ws->layers, c, n);
  std::copy(fs.u.begin(), fs.u.end(), u);
  std::copy(fs.gx.begin(), fs.gx.end(), gx);
  std::copy(fs.gy.begin(), fs.gy.end(), gy);
}

/// cs_reduced_apply(v, weight) with the NN weight theta (theta = 0: plain coarse operator),
/// solvers.cpp:372-386 + 599-603. Builds the coarse / Neumann layers on first use.
int ddo_apply_cs(void* p, double theta, const double* v, double* out) {
  auto h = static_cast<ddo_handle*>(p);
  Workspace& ws = *h->ws;
  ws.assemble_coarse();
  LinOp weight = [](const Vec& x) { return x; };
  if (theta > 0) {
    ws.build_neumann();
    weight = [&ws, theta](const Vec& x) {
      Vec w = ws.apply_PT(ws.apply_P(x));
      for (auto& e : w) e *= theta;
      if (theta < 1.0)
        for (size_t i = 0; i < w.size(); ++i) w[i] += (1.0 - theta) * x[i];
      return w;
    };
  }
  Vec in(v, v + ws.n_delta());
  Vec o = ws.cs_reduced_apply(in, weight);
  std::copy(o.begin(), o.end(), out);
  return 0;
}

/// apply_P (transpose 0) / apply_PT (1), solvers.cpp:450-474; v, out: n_delta doubles.
int ddo_apply_p(void* p, int transpose, const double* v, double* out) {
  auto h = static_cast<ddo_handle*>(p);
  Workspace& ws = *h->ws;
  ws.assemble_coarse();
  ws.build_neumann();
  Vec in(v, v + ws.n_delta());
  Vec o = transpose ? ws.apply_PT(in) : ws.apply_P(in);
  std::copy(o.begin(), o.end(), out);
  return 0;
}

/// reduced_apply(mu), the one-level operator (solvers.cpp:262-274); mu, out: n_mu doubles.
int ddo_apply_reduced(void* p, const double* v, double* out) {
  auto h = static_cast<ddo_handle*>(p);
  Workspace& ws = *h->ws;
  Vec in(v, v + ws.n_mu());
  Vec o = ws.reduced_apply(in);
  std::copy(o.begin(), o.end(), out);
  return 0;
}

/// dense_oracle_solve (solvers.cpp:609-709): dim = n_mu (one-level) or n_delta; op dim x dim
/// column-major, rhs dim, mu_full n_mu, coeffs N x M. Returns 0, or 2 on invalid_argument.
int ddo_dense(void* p, int method, double theta, int* dim, double* op, double* rhs, double* mu_full,
              double* coeffs) {
  auto h = static_cast<ddo_handle*>(p);
  Workspace& ws = *h->ws;
  try {
    const Method m = method == 0 ? Method::Ddelm : method == 1 ? Method::DdelmCs : Method::DdelmNn;
    DenseOracle d = dense_oracle_solve(ws, m, theta);
    *dim = d.reduced_op.c;
    std::copy(d.reduced_op.a.begin(), d.reduced_op.a.end(), op);
    std::copy(d.reduced_rhs.begin(), d.reduced_rhs.end(), rhs);
    std::copy(d.mu_full.begin(), d.mu_full.end(), mu_full);
    for (size_t i = 0; i < d.coeffs.size(); ++i) std::copy(d.coeffs[i].begin(), d.coeffs[i].end(), coeffs + i * d.coeffs[i].size());
  } catch (const std::invalid_argument&) {
    return 2;
  }
  return 0;
}

/// Relative L2 / H1 errors against the exact solution (runner.cpp:144-150).
int ddo_errors(void* p, int n, double* l2, double* h1) {
  auto h = static_cast<ddo_handle*>(p);
  if (!h->ws->problem.has_exact()) return 1;
  ErrorReport e = relative_errors_exact(h->ws->part, h->ws->layers, h->rep.coeffs, h->ws->problem, n);
  *l2 = e.l2;
  *h1 = e.h1;
  return 0;
}

/// CPU-baseline mode: LsFactor through SciPy's LAPACK at `libpath` (nullptr: the restatement)
int ddo_set_lapack(const char* libpath) {
  try {
    set_lapack(libpath);
    return 0;
  } catch (...) {
    return 1;
  }
}

// ---- factorisation-level entry points (LsFactor tests, test_solvers.cpp:14-85)
/// seeded standard-normal matrix, column-major (test_solvers.cpp:14-21: mt19937_64 + libstdc++
/// normal_distribution, column by column)
void ddo_random_matrix(int rows, int cols, unsigned long long seed, double* out) {
  std::mt19937_64 gen(seed);
  std::normal_distribution<double> n;
  for (int j = 0; j < cols; ++j)
    for (int i = 0; i < rows; ++i) out[static_cast<size_t>(j) * rows + i] = n(gen);
}

/// LsFactor (solvers.cpp:24-45) of one column-major m x n matrix: rank, branch, K^+ (n x m
/// column-major) and Q (m x n column-major, columns >= rank zero)
int ddo_lsfactor(const double* K, int m, int n, double tol, int* rank, int* deficient, double* pinv, double* Q) {
  try {
    Mat A(m, n);
    std::copy(K, K + static_cast<size_t>(m) * n, A.a.begin());
    LsFactor f(A, tol);
    *rank = f.rank();
    *deficient = f.rank_deficient() ? 1 : 0;
    Mat I = Mat::identity(m);
    Mat P = f.apply_pinv(I);
    std::copy(P.a.begin(), P.a.end(), pinv);
    const Mat& q = f.Q();
    std::fill(Q, Q + static_cast<size_t>(m) * n, 0.0);
    for (int j = 0; j < q.c && j < n; ++j)
      for (int i = 0; i < m; ++i) Q[static_cast<size_t>(j) * m + i] = q(i, j);
    return 0;
  } catch (...) {
    return 1;
  }
}

/// Eigen's A.completeOrthogonalDecomposition().pseudoInverse() with the DEFAULT threshold
/// (eps * min(m, n)): the reference tests' svd_pinv (test_solvers.cpp:23-25); out n x m
int ddo_cod_pinv(const double* K, int m, int n, double* out) {
  try {
    Mat A(m, n);
    std::copy(K, K + static_cast<size_t>(m) * n, A.a.begin());
    COD c;
    c.compute(A, std::numeric_limits<double>::epsilon() * std::min(m, n));
    Mat P = c.pseudo_inverse();
    std::copy(P.a.begin(), P.a.end(), out);
    return 0;
  } catch (...) {
    return 1;
  }
}

// ---- parity decomposition hooks (model.cpp set_tanh_record / set_tanh_table)
static std::vector<double> g_tanh_rec;
static std::unordered_map<std::uint64_t, double> g_tanh_tab;
void ddo_tanh_record(int on) {
  g_tanh_rec.clear();
  ddo::set_tanh_record(on ? &g_tanh_rec : nullptr);
}
long long ddo_tanh_recorded(double* out) {
  if (out) std::memcpy(out, g_tanh_rec.data(), g_tanh_rec.size() * sizeof(double));
  return static_cast<long long>(g_tanh_rec.size());
}
void ddo_tanh_table(const double* z, const double* t, long long n) {
  g_tanh_tab.clear();
  if (n <= 0) {
    ddo::set_tanh_table(nullptr);
    return;
  }
  g_tanh_tab.reserve(static_cast<size_t>(n));
  for (long long k = 0; k < n; ++k) {
    std::uint64_t b;
    std::memcpy(&b, z + k, sizeof b);
    g_tanh_tab[b] = t[k];
  }
  ddo::set_tanh_table(&g_tanh_tab);
}
long long ddo_tanh_misses() { return ddo::tanh_table_misses(); }

}  // extern "C"

// ddelm_b200/solvers.hpp — C++ drop-in façade of the reference solver API over the C-ABI.
//
// Mirrors proj/include/ddelm/solvers.hpp (namespace ddelm) for the north-star path:
//   Workspace(problem, s, n_grid, M, l, seed, SolverOptions)     solvers.hpp:79-80
//   ddelm_solve(Workspace&, CgOptions)  (one-level)                 solvers.hpp:178
//   ddelm_cs_solve(Workspace&, CgOptions)                          solvers.hpp:179
//   ddelm_nn_solve(Workspace&, double theta, CgOptions)            solvers.hpp:181
//   SolverOptions / CgOptions / SolveReport                        solvers.hpp:49-58,162-176
//   ProblemSpec via make_problem(name)                             problems.hpp:38-62,
//                                                                   problems.cpp:132-188
//   relative_errors(ws, grid_n) / field_diff(ws, ref, grid_n)      metrics.cpp:112-128,
//                                                                   runner.cpp:269-281
// with the reference's error behaviour: std::invalid_argument for bad arguments (theta outside
// [0,1], bad partition, unknown problem), std::runtime_error for a non-SPD coarse matrix and for
// device failures. Non-convergence is SolveReport::converged == false, not an exception.
//
// Vectors are std::vector<double> instead of Eigen::VectorXd (Eigen is not a dependency of the
// device path); layouts are the reference's (coefficients per subdomain; mu = [mu_Delta; mu_Pi]).
// Everything heavy runs on the B200 behind include/ddelm_gpu.h; this header only marshals.
#pragma once

#include <cmath>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "ddelm_gpu.h"

namespace ddelm {

enum class FluxVariant { Pointwise, MeanEdge };  // assembly.hpp FluxVariant

struct ProblemParams {  // problems.hpp:64-68
  double alpha = 32.0;
  std::uint64_t forcing_seed = 2;
  std::uint64_t rho_seed = 3;
};

struct ProblemSpec {
  std::string name;
  int id = DDELM_POISSON_SINPI;
  ProblemParams params;
};

/// make_problem (problems.cpp:132-188): the Poisson-kind problems of the device path.
inline ProblemSpec make_problem(const std::string& name, const ProblemParams& params = {}) {
  if (!(params.alpha > 0)) throw std::invalid_argument("sample_grf: alpha must be positive");
  if (name == "poisson_sinpi") return {name, DDELM_POISSON_SINPI, params};
  if (name == "poisson_sin2pi_exp") return {name, DDELM_POISSON_SIN2PI_EXP, params};
  if (name == "poisson_sin2pi_cos3pi_x2y") return {name, DDELM_POISSON_SIN2PI_COS3PI_X2Y, params};
  if (name == "poisson_grf") return {name, DDELM_POISSON_GRF, params};
  if (name == "varcoef_poisson") return {name, DDELM_VARCOEF_POISSON, params};
  if (name == "biharmonic_sinpi") return {name, DDELM_BIHARMONIC_SINPI, params};
  throw std::invalid_argument("make_problem: unknown problem '" + name + "'");
}

struct SolverOptions {  // solvers.hpp:49-58
  FluxVariant flux_variant = FluxVariant::Pointwise;
  bool change_of_variables = false;
  double rank_tol = 1e-10;
  int workers = 1;  // accepted for API parity; the device batches all subdomains
  int debug_flip_flux_row = -1;
  int device = 0;   // CUDA device ordinal (device-path addition)
  int cg_blocks = DDELM_CG_BLOCKS_COEFF;  // CG operator representation (device-path addition)
};

struct CgOptions {  // solvers.hpp:173-176
  double rel_tol = 1e-9;
  int max_iter = 0;  // <= 0: 20x unknowns
};

struct SolveReport {  // solvers.hpp:162-171
  std::vector<std::vector<double>> coeffs;  // per subdomain, M each
  std::vector<double> mu, mu_delta, mu_pi;  // global ordering, Delta then Pi
  int iterations = 0;
  bool converged = true;
  bool negative_curvature = false;
  std::vector<double> residual_history;
  double setup_seconds = 0, cg_seconds = 0, reconstruct_seconds = 0;
  double assembly_seconds = 0, factorization_seconds = 0, total_seconds = 0;
};

namespace detail {
inline void check(int rc) {
  if (rc == DDELM_OK) return;
  const std::string msg = ddelm_gpu_last_error();
  if (rc == DDELM_ERR_INVALID_ARGUMENT) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}
struct WsDeleter {
  void operator()(ddelm_ws* w) const { ddelm_gpu_destroy(w); }
};
}  // namespace detail

/// Device-resident Workspace (solvers.hpp:78-160): features, local factorisations, the coarse
/// and Neumann layers live in HBM; the layers are built lazily like the reference's
/// coarse_built / neumann_built flags. Not safe for concurrent solves (same as the reference).
class Workspace {
 public:
  Workspace(const ProblemSpec& problem, int s, int n_grid, int M, double l, std::uint64_t seed,
            const SolverOptions& opts = {})
      : s_(s), n_grid_(n_grid), M_(M), cc_(problem.id == DDELM_BIHARMONIC_SINPI ? 2 : 1) {
    ddelm_desc d{};
    d.problem = problem.id;
    d.s = s;
    d.n_grid = n_grid;
    d.M = M;
    d.l = l;
    d.seed = seed;
    d.flux_variant = opts.flux_variant == FluxVariant::MeanEdge ? DDELM_FLUX_MEAN_EDGE : DDELM_FLUX_POINTWISE;
    d.change_of_variables = opts.change_of_variables ? 1 : 0;
    d.rank_tol = opts.rank_tol;
    d.device = opts.device;
    d.debug_flip_flux_row = opts.debug_flip_flux_row;
    d.alpha = problem.params.alpha;
    d.forcing_seed = problem.params.forcing_seed;
    d.rho_seed = problem.params.rho_seed;
    ddelm_ws* w = nullptr;
    detail::check(ddelm_gpu_create(&d, &w));
    ws_.reset(w);
    detail::check(ddelm_gpu_set_cg_blocks(w, opts.cg_blocks));
  }

  int n_subs() const { return s_ * s_; }
  int n_delta() const { return 2 * s_ * (s_ - 1) * (n_grid_ - 2) * cc_; }  // geometry.cpp:155-157
  int n_pi() const { return (s_ - 1) * (s_ - 1) * cc_; }
  int M() const { return M_; }

  void build() { detail::check(ddelm_gpu_build(ws_.get())); }
  void assemble_coarse() { detail::check(ddelm_gpu_build_coarse(ws_.get())); }  // solvers.cpp:278
  void build_neumann() { detail::check(ddelm_gpu_build_neumann(ws_.get())); }    // solvers.cpp:390

  /// cs_reduced_apply with the NN weight (solvers.cpp:372-386, 599-603); theta = 0: coarse op.
  std::vector<double> cs_reduced_apply(const std::vector<double>& v, double theta) {
    std::vector<double> out(v.size());
    detail::check(ddelm_gpu_apply_operator(ws_.get(), theta, v.data(), out.data()));
    return out;
  }

  /// reduced_apply, the one-level operator on mu = [mu_Delta; mu_Pi] (solvers.cpp:262-274).
  std::vector<double> reduced_apply(const std::vector<double>& mu) {
    std::vector<double> out(mu.size());
    detail::check(ddelm_gpu_apply_reduced(ws_.get(), mu.data(), out.data()));
    return out;
  }

  /// apply_P / apply_PT, the Neumann map and its adjoint (solvers.cpp:450-474).
  std::vector<double> apply_P(const std::vector<double>& v) {
    std::vector<double> out(v.size());
    detail::check(ddelm_gpu_apply_neumann(ws_.get(), 0, v.data(), out.data()));
    return out;
  }
  std::vector<double> apply_PT(const std::vector<double>& u) {
    std::vector<double> out(u.size());
    detail::check(ddelm_gpu_apply_neumann(ws_.get(), 1, u.data(), out.data()));
    return out;
  }

  SolveReport solve(int method, double theta, const CgOptions& cg) {
    ddelm_report r{};
    detail::check(ddelm_gpu_solve(ws_.get(), method, theta, cg.rel_tol, cg.max_iter, &r));
    SolveReport rep;
    rep.iterations = r.iterations;
    rep.converged = r.converged != 0;
    rep.negative_curvature = r.negative_curvature != 0;
    rep.mu.resize(r.n_mu);
    detail::check(ddelm_gpu_get_mu(ws_.get(), rep.mu.data()));
    rep.mu_delta.assign(rep.mu.begin(), rep.mu.begin() + r.n_delta);
    rep.mu_pi.assign(rep.mu.begin() + r.n_delta, rep.mu.end());
    std::vector<double> c(static_cast<size_t>(r.n_subdomains) * r.M);
    detail::check(ddelm_gpu_get_coeffs(ws_.get(), c.data()));
    rep.coeffs.resize(r.n_subdomains);
    for (int i = 0; i < r.n_subdomains; ++i)
      rep.coeffs[i].assign(c.begin() + static_cast<size_t>(i) * r.M, c.begin() + static_cast<size_t>(i + 1) * r.M);
    rep.residual_history.resize(std::max(r.iterations, 0));
    const int n = ddelm_gpu_get_residuals(ws_.get(), rep.residual_history.data(), r.iterations);
    rep.residual_history.resize(std::max(n, 0));
    rep.setup_seconds = r.setup_seconds;
    rep.cg_seconds = r.cg_seconds;
    rep.reconstruct_seconds = r.reconstruct_seconds;
    rep.assembly_seconds = r.assembly_seconds;
    rep.factorization_seconds = r.factorization_seconds;
    rep.total_seconds = r.total_seconds;
    return rep;
  }

  ddelm_ws* handle() { return ws_.get(); }

 private:
  int s_, n_grid_, M_, cc_;
  std::unique_ptr<ddelm_ws, detail::WsDeleter> ws_;
};

/// ddelm_solve, one-level DDELM (solvers.cpp:493-531).
inline SolveReport ddelm_solve(Workspace& ws, const CgOptions& cg_opts = {}) {
  return ws.solve(DDELM_METHOD_DDELM, 0.0, cg_opts);
}

/// ddelm_cs_solve (solvers.cpp:582-588).
inline SolveReport ddelm_cs_solve(Workspace& ws, const CgOptions& cg_opts = {}) {
  return ws.solve(DDELM_METHOD_CS, 0.0, cg_opts);
}

/// ddelm_nn_solve (solvers.cpp:590-605): theta in [0, 1]; theta = 0 is exactly ddelm_cs_solve.
inline SolveReport ddelm_nn_solve(Workspace& ws, double theta, const CgOptions& cg_opts = {}) {
  if (!(theta >= 0.0 && theta <= 1.0)) throw std::invalid_argument("ddelm_nn_solve: theta must lie in [0, 1]");
  return ws.solve(DDELM_METHOD_NN, theta, cg_opts);
}

/// Relative L2 / H1 errors of the last solve's field against the problem's exact solution on the
/// grid_n x grid_n trapezoid grid, evaluated on the device (relative_errors, metrics.cpp:112-128;
/// grid_n < 64 throws std::invalid_argument as the reference).
struct ErrorReport {  // metrics.hpp ErrorReport
  double l2 = 0, h1 = 0;
  int grid_n = 0;
};
inline ErrorReport relative_errors(Workspace& ws, int grid_n = 257) {
  ErrorReport e;
  e.grid_n = grid_n;
  detail::check(ddelm_gpu_relative_errors(ws.handle(), grid_n, &e.l2, &e.h1));
  return e;
}
/// The same errors against another coefficient set on the same layers (oracle_check's
/// field_diff, runner.cpp:269-281); ref: one M-vector per subdomain.
inline ErrorReport field_diff(Workspace& ws, const std::vector<std::vector<double>>& ref, int grid_n = 257) {
  std::vector<double> flat;
  for (const auto& c : ref) flat.insert(flat.end(), c.begin(), c.end());
  ErrorReport e;
  e.grid_n = grid_n;
  detail::check(ddelm_gpu_field_diff(ws.handle(), grid_n, flat.data(), &e.l2, &e.h1));
  return e;
}

/// Method selector of dense_oracle_solve (solvers.hpp Method).
enum class Method { Ddelm = DDELM_METHOD_DDELM, DdelmCs = DDELM_METHOD_CS, DdelmNn = DDELM_METHOD_NN };

/// dense_oracle_solve (solvers.hpp DenseOracle, solvers.cpp:609-709) on the device: the global
/// block system assembled densely, every pseudo-inverse through the device QR / COD kernels.
struct DenseOracle {
  std::vector<double> reduced_op;  // dim x dim, column-major
  std::vector<double> reduced_rhs, mu_reduced, mu_full;
  std::vector<std::vector<double>> coeffs;
  int dim = 0;
};
inline DenseOracle dense_oracle_solve(Workspace& ws, Method method, double theta = 0.999) {
  const int m = static_cast<int>(method);
  const int dim = method == Method::Ddelm ? ws.n_delta() + ws.n_pi() : ws.n_delta();
  DenseOracle o;
  o.reduced_op.resize(static_cast<size_t>(dim) * dim);
  o.reduced_rhs.resize(dim);
  o.mu_full.resize(ws.n_delta() + ws.n_pi());
  std::vector<double> c(static_cast<size_t>(ws.n_subs()) * ws.M());
  detail::check(ddelm_gpu_dense_oracle(ws.handle(), m, theta, &o.dim, o.reduced_op.data(), o.reduced_rhs.data(),
                                       o.mu_full.data(), c.data()));
  o.mu_reduced.assign(o.mu_full.begin(), o.mu_full.begin() + dim);
  o.coeffs.resize(ws.n_subs());
  for (int i = 0; i < ws.n_subs(); ++i)
    o.coeffs[i].assign(c.begin() + static_cast<size_t>(i) * ws.M(), c.begin() + static_cast<size_t>(i + 1) * ws.M());
  return o;
}

/// oracle_check (runner.cpp:252-316) on a constructed workspace: solve to 1e-12, the dense
/// oracle, then the relative mu difference, the field difference on the 65 x 65 grid and the
/// largest entry of (iterative operator - dense reduced operator) over the unit vectors.
struct OracleCheckReport {  // runner.hpp OracleCheckReport
  double mu_diff = 0, field_diff = 0, op_diff = 0;
  int op_row = -1, op_col = -1;
  bool pass = false;
};
inline OracleCheckReport oracle_check(Workspace& ws, Method method, double theta = 0.999) {
  const DenseOracle oracle = dense_oracle_solve(ws, method, theta);
  const CgOptions tight{1e-12, 0};
  const SolveReport rep = method == Method::Ddelm     ? ddelm_solve(ws, tight)
                          : method == Method::DdelmCs ? ddelm_cs_solve(ws, tight)
                                                      : ddelm_nn_solve(ws, theta, tight);
  OracleCheckReport r;
  double dn = 0, on = 0;
  for (size_t k = 0; k < rep.mu.size(); ++k) {
    dn += (rep.mu[k] - oracle.mu_full[k]) * (rep.mu[k] - oracle.mu_full[k]);
    on += oracle.mu_full[k] * oracle.mu_full[k];
  }
  r.mu_diff = on > 0 ? std::sqrt(dn / on) : std::sqrt(dn);
  r.field_diff = field_diff(ws, oracle.coeffs, 65).l2;
  const int dim = oracle.dim;
  for (int j = 0; j < dim; ++j) {
    std::vector<double> e(dim, 0.0);
    e[j] = 1.0;
    const std::vector<double> col = method == Method::Ddelm ? ws.reduced_apply(e)
                                    : ws.cs_reduced_apply(e, method == Method::DdelmNn ? theta : 0.0);
    for (int i = 0; i < dim; ++i) {
      const double d = std::abs(col[i] - oracle.reduced_op[static_cast<size_t>(j) * dim + i]);
      if (d > r.op_diff) {
        r.op_diff = d;
        r.op_row = i;
        r.op_col = j;
      }
    }
  }
  r.pass = r.mu_diff < 1e-6 && r.field_diff < 1e-6 && r.op_diff < 1e-6;
  return r;
}

}  // namespace ddelm

// ddelm_solve — C++ host program over the drop-in façade (include/ddelm_b200/solvers.hpp).
//
// The device-path subset of `ddelm_cli solve` and `ddelm_cli oracle-check` (tools/ddelm_cli.cpp:
// 55-92, runner.cpp:126-155, 252-316):
//   ddelm_solve [key=value ...]   keys: mode (solve | oracle-check) problem s n_grid M l seed method
//                                 theta flux_variant trace_basis cg_rel_tol cg_max_iter device
//                                 eval_grid_n alpha forcing_seed rho_seed debug_flip_flux_row
// Prints one JSON object (iterations, converged, residual history, mu, timings, and the relative
// L2 / H1 errors against the exact solution on the eval_grid_n^2 grid, runner.cpp:144-150) on stdout;
// mode=oracle-check prints the CLI's oracle-check line (ddelm_cli.cpp:71-77) instead.
// Exit codes follow the CLI: 0 ok, 2 non-convergence / solver error, 3 configuration error.
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <map>
#include <string>

#include "ddelm_b200/solvers.hpp"

int main(int argc, char** argv) {
  std::map<std::string, std::string> kv = {
      {"problem", "poisson_sinpi"}, {"s", "2"}, {"n_grid", "10"}, {"M", "64"}, {"l", "8"}, {"seed", "1"},
      {"method", "ddelm-nn"}, {"theta", "0.999"}, {"flux_variant", "mean_edge"},
      {"trace_basis", "change_of_variables"}, {"cg_rel_tol", "1e-9"}, {"cg_max_iter", "0"}, {"device", "0"},
      {"eval_grid_n", "257"}, {"alpha", "32"}, {"forcing_seed", "2"}, {"rho_seed", "3"},
      {"mode", "solve"}, {"debug_flip_flux_row", "-1"}, {"cg_blocks", "coeff"}};
  for (int k = 1; k < argc; ++k) {
    const std::string a = argv[k];
    const auto eq = a.find('=');
    if (eq == std::string::npos || !kv.count(a.substr(0, eq))) {
      std::fprintf(stderr, "config error: bad argument '%s'\n", a.c_str());
      return 3;
    }
    kv[a.substr(0, eq)] = a.substr(eq + 1);
  }
  try {
    ddelm::SolverOptions opts;
    opts.flux_variant = kv["flux_variant"] == "mean_edge" ? ddelm::FluxVariant::MeanEdge : ddelm::FluxVariant::Pointwise;
    opts.change_of_variables = kv["trace_basis"] == "change_of_variables";
    opts.device = std::atoi(kv["device"].c_str());
    opts.debug_flip_flux_row = std::atoi(kv["debug_flip_flux_row"].c_str());
    if (kv["cg_blocks"] != "coeff" && kv["cg_blocks"] != "compact") {
      std::fprintf(stderr, "config error: cg_blocks must be coeff or compact\n");
      return 3;
    }
    opts.cg_blocks = kv["cg_blocks"] == "compact" ? DDELM_CG_BLOCKS_COMPACT : DDELM_CG_BLOCKS_COEFF;
    ddelm::ProblemParams pp;
    pp.alpha = std::atof(kv["alpha"].c_str());
    pp.forcing_seed = std::strtoull(kv["forcing_seed"].c_str(), nullptr, 10);
    pp.rho_seed = std::strtoull(kv["rho_seed"].c_str(), nullptr, 10);
    ddelm::Workspace ws(ddelm::make_problem(kv["problem"], pp), std::atoi(kv["s"].c_str()), std::atoi(kv["n_grid"].c_str()),
                        std::atoi(kv["M"].c_str()), std::atof(kv["l"].c_str()),
                        std::strtoull(kv["seed"].c_str(), nullptr, 10), opts);
    ddelm::CgOptions cg{std::atof(kv["cg_rel_tol"].c_str()), std::atoi(kv["cg_max_iter"].c_str())};
    const std::string method = kv["method"];
    if (method != "ddelm" && method != "ddelm-cs" && method != "ddelm-nn")
      throw std::invalid_argument("unknown method '" + method + "'");
    if (kv["mode"] == "oracle-check") {
      const ddelm::Method m = method == "ddelm"      ? ddelm::Method::Ddelm
                              : method == "ddelm-cs" ? ddelm::Method::DdelmCs
                                                     : ddelm::Method::DdelmNn;
      const ddelm::OracleCheckReport oc = ddelm::oracle_check(ws, m, std::atof(kv["theta"].c_str()));
      std::printf("mu_diff=%.3e field_diff=%.3e op_diff=%.3e (row=%d col=%d) -> %s\n", oc.mu_diff, oc.field_diff,
                  oc.op_diff, oc.op_row, oc.op_col, oc.pass ? "pass" : "FAIL");
      return oc.pass ? 0 : 2;
    }
    if (kv["mode"] != "solve") throw std::invalid_argument("unknown mode '" + kv["mode"] + "'");
    ddelm::SolveReport r = method == "ddelm"      ? ddelm::ddelm_solve(ws, cg)
                           : method == "ddelm-cs" ? ddelm::ddelm_cs_solve(ws, cg)
                                                  : ddelm::ddelm_nn_solve(ws, std::atof(kv["theta"].c_str()), cg);
    // errors against the exact solution where the problem has one (runner.cpp:144-150); the GRF
    // problems are measured against a finite-difference solve in the reference (not built)
    ddelm::ErrorReport err;
    err.l2 = err.h1 = -1.0;
    if (kv["problem"] != "poisson_grf" && kv["problem"] != "varcoef_poisson")
      err = ddelm::relative_errors(ws, std::atoi(kv["eval_grid_n"].c_str()));
    std::printf("{\"iterations\": %d, \"converged\": %s, \"total_seconds\": %.9g, \"l2_error\": %.17g, "
                "\"h1_error\": %.17g, \"residual_history\": [",
                r.iterations, r.converged ? "true" : "false", r.total_seconds, err.l2, err.h1);
    for (size_t k = 0; k < r.residual_history.size(); ++k)
      std::printf("%s%.17g", k ? ", " : "", r.residual_history[k]);
    std::printf("], \"mu\": [");
    for (size_t k = 0; k < r.mu.size(); ++k) std::printf("%s%.17g", k ? ", " : "", r.mu[k]);
    std::printf("]}\n");
    return r.converged ? 0 : 2;
  } catch (const std::invalid_argument& e) {
    std::fprintf(stderr, "config error: %s\n", e.what());
    return 3;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "solver error: %s\n", e.what());
    return 2;
  }
}

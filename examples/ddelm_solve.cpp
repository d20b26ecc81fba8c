// ddelm_solve — C++ host program over the drop-in façade (include/ddelm_b200/solvers.hpp and
// include/ddelm_b200/runner.hpp).
//
// The device-path subset of `ddelm_cli solve`, `ddelm_cli ablation` and `ddelm_cli oracle-check`
// (tools/ddelm_cli.cpp:55-92, runner.cpp:126-316):
//   ddelm_solve [config=<file>] [key=value ...]
//     keys: the reference's RunConfig keys (runner.cpp:35-56: problem alpha seed forcing_seed
//           rho_seed s n_grid M l method theta flux_variant trace_basis cg_rel_tol cg_max_iter
//           eval_grid_n workers json_out csv_out debug_flip_flux_row) + device, cg_blocks, and
//           mode = solve | oracle-check | ablation-table1 | ablation-table2, mu = 0 | 1
// mode=solve runs ddelm::run (the JSON report to json_out, the CSV row to csv_out, as the
// reference's persist) and prints the reference's json_report (runner.cpp:199-233) on stdout,
// with the solution mu appended when mu=1 (the default here: the tests compare it bit for bit);
// the ablation modes print the CSV header and one row per run (runner.cpp:157-197);
// mode=oracle-check prints the CLI's oracle-check line (ddelm_cli.cpp:71-77).
// Exit codes follow the CLI: 0 ok, 2 non-convergence / solver error, 3 configuration error.
// Defaults differ from RunConfig's only to make the bare command a small DDELM-NN solve (T1).
#include <cstdio>
#include <exception>
#include <string>
#include <vector>

#include "ddelm_b200/runner.hpp"
#include "ddelm_b200/solvers.hpp"

int main(int argc, char** argv) {
  ddelm::RunConfig cfg;
  cfg.method = "ddelm-nn";
  cfg.l = 8;
  cfg.flux_variant = "mean_edge";
  cfg.trace_basis = "change_of_variables";
  std::string mode = "solve";
  bool print_mu = true;
  try {
    for (int k = 1; k < argc; ++k) {
      const std::string a = argv[k];
      const auto eq = a.find('=');
      if (eq == std::string::npos) throw ddelm::ConfigError("bad argument '" + a + "' (expected key=value)");
      const std::string key = a.substr(0, eq), val = a.substr(eq + 1);
      if (key == "config") {
        cfg = ddelm::load_config(val);
      } else if (key == "mode") {
        mode = val;
      } else if (key == "mu") {
        print_mu = val != "0";
      } else {
        ddelm::apply_override(cfg, a);
      }
    }
    if (mode != "solve" && mode != "oracle-check" && mode != "ablation-table1" && mode != "ablation-table2")
      throw ddelm::ConfigError("unknown mode '" + mode + "'");
    if (mode == "oracle-check") {
      ddelm::resolve_defaults(cfg);
      ddelm::Workspace ws(ddelm::make_problem(cfg.problem, {cfg.alpha, cfg.forcing_seed, cfg.rho_seed}), cfg.s,
                          cfg.n_grid, cfg.M, cfg.l, cfg.seed, ddelm::solver_options(cfg));
      const ddelm::Method m = cfg.method == "ddelm"      ? ddelm::Method::Ddelm
                              : cfg.method == "ddelm-cs" ? ddelm::Method::DdelmCs
                                                         : ddelm::Method::DdelmNn;
      const ddelm::OracleCheckReport oc = ddelm::oracle_check(ws, m, cfg.theta);
      std::printf("mu_diff=%.3e field_diff=%.3e op_diff=%.3e (row=%d col=%d) -> %s\n", oc.mu_diff, oc.field_diff,
                  oc.op_diff, oc.op_row, oc.op_col, oc.pass ? "pass" : "FAIL");
      return oc.pass ? 0 : 2;
    }
    if (mode != "solve") {
      const std::vector<ddelm::RunOutcome> outs = ddelm::run_ablation(cfg, mode == "ablation-table1" ? "table1" : "table2");
      std::printf("%s\n", ddelm::csv_header().c_str());
      bool ok = true;
      for (const auto& o : outs) {
        std::printf("%s\n", ddelm::csv_row(o).c_str());
        ok = ok && o.report.converged;
      }
      return ok ? 0 : 2;
    }
    const ddelm::RunOutcome out = ddelm::run(cfg);
    std::string j = ddelm::json_report(out);
    if (print_mu) {
      // device-path extension after the reference's keys: the solution mu = [mu_Delta; mu_Pi]
      j.pop_back();  // the closing brace
      j += ",\n  \"mu\": [";
      for (size_t k = 0; k < out.report.mu.size(); ++k) j += (k ? ", " : "") + ddelm::detail::jnum(out.report.mu[k]);
      j += "]\n}";
    }
    std::printf("%s\n", j.c_str());
    return out.report.converged ? 0 : 2;
  } catch (const ddelm::ConfigError& e) {
    std::fprintf(stderr, "config error: %s\n", e.what());
    return 3;
  } catch (const std::invalid_argument& e) {
    std::fprintf(stderr, "config error: %s\n", e.what());
    return 3;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "solver error: %s\n", e.what());
    return 2;
  }
}

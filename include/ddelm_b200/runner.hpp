// ddelm_b200/runner.hpp — the reference's experiment runner over the device path (header-only).
//
// Mirrors proj/include/ddelm/runner.hpp / src/runner.cpp for the north-star path:
//   RunConfig (runner.hpp:14-35), apply_override / load_config key syntax (runner.cpp:35-101),
//   resolve_defaults (runner.cpp:103-124), run (runner.cpp:126-155), run_ablation presets
//   table1 / table2 (runner.cpp:157-184), and the report schema — csv_header / csv_row
//   (runner.cpp:186-197) and json_report (runner.cpp:199-233) — with persist (runner.cpp:235-250).
// Differences, all stated: the errors of the GRF problems are against the reference's
// finite-difference solve in the reference (metrics.cpp fd_reference), which the device path does
// not build — they are reported as -1 with errors.reference = "none"; every other field has the
// reference's name, type and meaning. JSON is written without a third-party library.
#pragma once

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <fstream>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "ddelm_b200/solvers.hpp"

namespace ddelm {

struct RunConfig {  // runner.hpp:14-35
  std::string problem = "poisson_sinpi";
  double alpha = 32.0;
  std::uint64_t seed = 1;
  std::uint64_t forcing_seed = 2;
  std::uint64_t rho_seed = 3;
  int s = 2;
  int n_grid = 10;
  int M = 64;
  double l = 0;                   // 0 = problem default
  std::string method = "ddelm";   // ddelm | ddelm-cs | ddelm-nn
  double theta = 0.999;
  std::string flux_variant;       // empty = method default
  std::string trace_basis;        // empty = method default
  double cg_rel_tol = 1e-9;
  int cg_max_iter = 0;
  int eval_grid_n = 257;
  int workers = 1;                // recorded; the device batches every subdomain
  std::string json_out;
  std::string csv_out;
  int debug_flip_flux_row = -1;
  // device-path additions
  int device = 0;
  std::string cg_blocks = "coeff";  // coeff | compact
};

struct ConfigError : std::runtime_error {  // runner.hpp:37-39
  using std::runtime_error::runtime_error;
};

struct RunErrors {  // metrics.hpp ErrorReport as the runner stores it
  double l2 = -1, h1 = -1;
  int grid_n = 0;
  std::string reference = "none";  // "exact" (or "finite-difference" in the reference)
};

struct RunOutcome {  // runner.hpp RunOutcome
  RunConfig config;
  SolveReport report;
  RunErrors errors;
  double total_seconds = 0;
  double assembly_seconds = 0, factorization_seconds = 0;
};

namespace detail {
inline std::string trim(const std::string& s) {
  const auto a = s.find_first_not_of(" \t\r\n");
  if (a == std::string::npos) return "";
  const auto b = s.find_last_not_of(" \t\r\n");
  return s.substr(a, b - a + 1);
}
template <typename T>
T parse_number(const std::string& key, const std::string& value) {
  std::istringstream is(value);
  T v{};
  std::string rest;
  if (!(is >> v) || (is >> rest)) throw ConfigError("invalid value for '" + key + "': " + value);
  return v;
}
inline void set_key(RunConfig& c, const std::string& key, const std::string& v) {
  if (key == "problem") c.problem = v;
  else if (key == "alpha") c.alpha = parse_number<double>(key, v);
  else if (key == "seed") c.seed = parse_number<std::uint64_t>(key, v);
  else if (key == "forcing_seed") c.forcing_seed = parse_number<std::uint64_t>(key, v);
  else if (key == "rho_seed") c.rho_seed = parse_number<std::uint64_t>(key, v);
  else if (key == "s") c.s = parse_number<int>(key, v);
  else if (key == "n_grid") c.n_grid = parse_number<int>(key, v);
  else if (key == "M") c.M = parse_number<int>(key, v);
  else if (key == "l") c.l = parse_number<double>(key, v);
  else if (key == "method") c.method = v;
  else if (key == "theta") c.theta = parse_number<double>(key, v);
  else if (key == "flux_variant") c.flux_variant = v;
  else if (key == "trace_basis") c.trace_basis = v;
  else if (key == "cg_rel_tol") c.cg_rel_tol = parse_number<double>(key, v);
  else if (key == "cg_max_iter") c.cg_max_iter = parse_number<int>(key, v);
  else if (key == "eval_grid_n") c.eval_grid_n = parse_number<int>(key, v);
  else if (key == "workers") c.workers = parse_number<int>(key, v);
  else if (key == "json_out") c.json_out = v;
  else if (key == "csv_out") c.csv_out = v;
  else if (key == "debug_flip_flux_row") c.debug_flip_flux_row = parse_number<int>(key, v);
  else if (key == "device") c.device = parse_number<int>(key, v);
  else if (key == "cg_blocks") c.cg_blocks = v;
  else throw ConfigError("unknown config key '" + key + "'");
}
inline std::string jnum(double v) {
  if (!std::isfinite(v)) return "null";
  char b[40];
  std::snprintf(b, sizeof(b), "%.17g", v);
  return b;
}
inline std::string jstr(const std::string& s) {
  std::string o = "\"";
  for (char ch : s) {
    if (ch == '"' || ch == '\\') o += '\\';
    o += ch;
  }
  return o + "\"";
}
}  // namespace detail

/// One "key=value" override in the config-file syntax (runner.cpp:97-101).
inline void apply_override(RunConfig& cfg, const std::string& kv) {
  const auto eq = kv.find('=');
  if (eq == std::string::npos) throw ConfigError("override must be key=value: " + kv);
  detail::set_key(cfg, detail::trim(kv.substr(0, eq)), detail::trim(kv.substr(eq + 1)));
}

/// Config file: key=value lines, '#' comments (runner.cpp:77-95).
inline RunConfig load_config(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw ConfigError("cannot open config file: " + path);
  RunConfig cfg;
  std::string line;
  int lineno = 0;
  while (std::getline(in, line)) {
    ++lineno;
    const auto hash = line.find('#');
    if (hash != std::string::npos) line = line.substr(0, hash);
    line = detail::trim(line);
    if (line.empty()) continue;
    const auto eq = line.find('=');
    if (eq == std::string::npos) throw ConfigError(path + ":" + std::to_string(lineno) + ": expected key=value");
    detail::set_key(cfg, detail::trim(line.substr(0, eq)), detail::trim(line.substr(eq + 1)));
  }
  return cfg;
}

/// Method and problem defaults (runner.cpp:103-124).
inline void resolve_defaults(RunConfig& cfg) {
  if (cfg.method != "ddelm" && cfg.method != "ddelm-cs" && cfg.method != "ddelm-nn")
    throw ConfigError("unknown method '" + cfg.method + "'");
  if (cfg.theta < 0 || cfg.theta > 1) throw ConfigError("theta must lie in [0, 1]");
  if (cfg.s < 1 || cfg.n_grid < 3 || cfg.M < 1) throw ConfigError("invalid s / n_grid / M");
  if (!cfg.flux_variant.empty() && cfg.flux_variant != "pointwise" && cfg.flux_variant != "mean_edge")
    throw ConfigError("flux_variant must be pointwise or mean_edge");
  if (!cfg.trace_basis.empty() && cfg.trace_basis != "nodal" && cfg.trace_basis != "change_of_variables")
    throw ConfigError("trace_basis must be nodal or change_of_variables");
  if (cfg.cg_blocks != "coeff" && cfg.cg_blocks != "compact") throw ConfigError("cg_blocks must be coeff or compact");
  const bool coarse = cfg.method != "ddelm";
  if (cfg.flux_variant.empty()) cfg.flux_variant = coarse ? "mean_edge" : "pointwise";
  if (cfg.trace_basis.empty()) cfg.trace_basis = coarse ? "change_of_variables" : "nodal";
  if (cfg.l <= 0) {
    try {
      (void)make_problem(cfg.problem);
    } catch (const std::invalid_argument& e) {
      throw ConfigError(e.what());
    }
    cfg.l = cfg.problem == "biharmonic_sinpi" ? 64 : 32;  // ProblemSpec::default_l (problems.hpp:48, problems.cpp:171)
  }
}

inline SolverOptions solver_options(const RunConfig& c) {  // runner.cpp:59-67
  SolverOptions so;
  so.flux_variant = c.flux_variant == "mean_edge" ? FluxVariant::MeanEdge : FluxVariant::Pointwise;
  so.change_of_variables = c.trace_basis == "change_of_variables";
  so.workers = c.workers;
  so.debug_flip_flux_row = c.debug_flip_flux_row;
  so.device = c.device;
  so.cg_blocks = c.cg_blocks == "compact" ? DDELM_CG_BLOCKS_COMPACT : DDELM_CG_BLOCKS_COEFF;
  return so;
}

inline void persist(const RunOutcome& out);

/// run (runner.cpp:126-155): build, dispatch the method, errors on the eval grid, persist.
inline RunOutcome run(const RunConfig& cfg_in) {
  RunOutcome out;
  out.config = cfg_in;
  resolve_defaults(out.config);
  const RunConfig& c = out.config;
  const auto t0 = std::chrono::steady_clock::now();
  ProblemSpec prob;
  try {
    prob = make_problem(c.problem, {c.alpha, c.forcing_seed, c.rho_seed});
  } catch (const std::invalid_argument& e) {
    throw ConfigError(e.what());
  }
  Workspace ws(prob, c.s, c.n_grid, c.M, c.l, c.seed, solver_options(c));
  const CgOptions cgo{c.cg_rel_tol, c.cg_max_iter};
  out.report = c.method == "ddelm"      ? ddelm_solve(ws, cgo)
               : c.method == "ddelm-cs" ? ddelm_cs_solve(ws, cgo)
                                        : ddelm_nn_solve(ws, c.theta, cgo);
  out.assembly_seconds = out.report.assembly_seconds;
  out.factorization_seconds = out.report.factorization_seconds;
  if (c.problem != "poisson_grf" && c.problem != "varcoef_poisson") {
    const ErrorReport e = relative_errors(ws, c.eval_grid_n);
    out.errors = {e.l2, e.h1, e.grid_n, "exact"};
  } else {
    out.errors.grid_n = c.eval_grid_n;
  }
  out.total_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  persist(out);
  return out;
}

inline std::string csv_header() { return "method,s,M,theta,flux_variant,trace_basis,l2,h1,iters,seconds,seed"; }

inline std::string csv_row(const RunOutcome& out) {  // runner.cpp:188-197
  const RunConfig& c = out.config;
  char buf[512];
  std::snprintf(buf, sizeof(buf), "%s,%d,%d,%g,%s,%s,%.6e,%.6e,%d,%.3f,%llu", c.method.c_str(), c.s, c.M, c.theta,
                c.flux_variant.c_str(), c.trace_basis.c_str(), out.errors.l2, out.errors.h1, out.report.iterations,
                out.total_seconds, static_cast<unsigned long long>(c.seed));
  return buf;
}

inline std::string json_report(const RunOutcome& out) {  // runner.cpp:199-233, same keys
  using detail::jnum;
  using detail::jstr;
  const RunConfig& c = out.config;
  std::ostringstream j;
  j << "{\n  \"config\": {\"problem\": " << jstr(c.problem) << ", \"alpha\": " << jnum(c.alpha)
    << ", \"seed\": " << c.seed << ", \"forcing_seed\": " << c.forcing_seed << ", \"rho_seed\": " << c.rho_seed
    << ", \"s\": " << c.s << ", \"n_grid\": " << c.n_grid << ", \"M\": " << c.M << ", \"l\": " << jnum(c.l)
    << ", \"method\": " << jstr(c.method) << ", \"theta\": " << jnum(c.theta)
    << ", \"flux_variant\": " << jstr(c.flux_variant) << ", \"trace_basis\": " << jstr(c.trace_basis)
    << ", \"cg_rel_tol\": " << jnum(c.cg_rel_tol) << ", \"cg_max_iter\": " << c.cg_max_iter
    << ", \"eval_grid_n\": " << c.eval_grid_n << ", \"workers\": " << c.workers << "},\n";
  j << "  \"iterations\": " << out.report.iterations << ",\n";
  j << "  \"converged\": " << (out.report.converged ? "true" : "false") << ",\n";
  j << "  \"residual_history\": [";
  for (size_t k = 0; k < out.report.residual_history.size(); ++k) j << (k ? ", " : "") << jnum(out.report.residual_history[k]);
  j << "],\n";
  j << "  \"errors\": {\"l2\": " << jnum(out.errors.l2) << ", \"h1\": " << jnum(out.errors.h1)
    << ", \"grid_n\": " << out.errors.grid_n << ", \"reference\": " << jstr(out.errors.reference) << "},\n";
  j << "  \"timings\": {\"assembly\": " << jnum(out.assembly_seconds) << ", \"factorization\": "
    << jnum(out.factorization_seconds) << ", \"setup\": " << jnum(out.report.setup_seconds)
    << ", \"cg\": " << jnum(out.report.cg_seconds) << ", \"reconstruction\": " << jnum(out.report.reconstruct_seconds)
    << ", \"total\": " << jnum(out.total_seconds) << "}\n}";
  return j.str();
}

/// JSON report to json_out, CSV row appended to csv_out with the header on a fresh file
/// (runner.cpp:235-250).
inline void persist(const RunOutcome& out) {
  if (!out.config.json_out.empty()) {
    std::ofstream f(out.config.json_out);
    if (!f) throw ConfigError("cannot write JSON report: " + out.config.json_out);
    f << json_report(out) << "\n";
  }
  if (!out.config.csv_out.empty()) {
    bool fresh = true;
    {
      std::ifstream probe(out.config.csv_out, std::ios::ate);
      fresh = !probe || probe.tellg() <= 0;
    }
    std::ofstream f(out.config.csv_out, std::ios::app);
    if (!f) throw ConfigError("cannot write CSV: " + out.config.csv_out);
    if (fresh) f << csv_header() << "\n";
    f << csv_row(out) << "\n";
  }
}

/// Presets of the paper's ablations (runner.cpp:157-184): "table1" (trace basis x flux variant
/// x {cs, nn}) and "table2" (the theta sweep).
inline std::vector<RunOutcome> run_ablation(const RunConfig& base, const std::string& preset) {
  std::vector<RunOutcome> outs;
  if (preset == "table1") {
    const std::pair<const char*, const char*> combos[] = {
        {"nodal", "pointwise"}, {"change_of_variables", "pointwise"}, {"nodal", "mean_edge"},
        {"change_of_variables", "mean_edge"}};
    for (const auto& [trace, flux] : combos)
      for (const char* method : {"ddelm-cs", "ddelm-nn"}) {
        RunConfig cfg = base;
        cfg.trace_basis = trace;
        cfg.flux_variant = flux;
        cfg.method = method;
        outs.push_back(run(cfg));
      }
  } else if (preset == "table2") {
    for (double theta : {0.0, 0.5, 0.9, 0.99, 0.999, 0.9999, 1.0}) {
      RunConfig cfg = base;
      cfg.method = "ddelm-nn";
      cfg.theta = theta;
      outs.push_back(run(cfg));
    }
  } else {
    throw ConfigError("unknown ablation preset '" + preset + "'");
  }
  return outs;
}

}  // namespace ddelm

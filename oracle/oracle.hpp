// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// CPU restatement of the reference DDELM solver (/root/reference/proj, C++20 + Eigen3),
// written from the reference's behaviour without Eigen. It exists to CHECK the GPU path:
// only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
// may load it. The product path (paper_2503_10032_b200/) never links or calls it.
//
// Parity pin: the reference cannot be compiled here (Eigen3 and vendor/ are absent, no
// network). The restatement is pinned by re-running the reference's own
// test assertions (oracle/selftest.cpp mirrors proj/tests/test_{geometry,features,assembly,
// solvers}.cpp and acceptance criteria 1, 2, 7, 10) and by the known-answer values those
// tests hold (the m=6 transition matrix, structural counts, analytic forcings). Absolute
// iteration counts / fields are not pinned by the reference; goldens under tests/golden/
// are generated from this restatement (tools/make_goldens.py).
//
// Third-party arithmetic boundary: Eigen3 (version unpinned, ">= 3.3", CMakeLists.txt:18).
// Restated semantics (published algorithms, not library source):
//   * HouseholderQR (solvers.cpp:27): Householder reflectors H = I - tau v v^T, v(0)=1,
//     beta = -sign(alpha)*||x||, tau = (beta-alpha)/beta.
//   * ColPivHouseholderQR (via CompleteOrthogonalDecomposition, solvers.cpp:35-38):
//     Businger-Golub max-norm pivoting, first-index tie-break, LAPACK-style norm
//     downdating with recomputation when the downdate ratio falls below sqrt(eps);
//     rank = #{|R_ii| > thr * max|R_ii|}.
//   * COD: RZ step on the rank x cols trapezoid with reflectors from the right,
//     pseudoInverse() = solve(I): x = P Z^T [T^{-1} (Q^T b)(0:r); 0].
//   * LLT (solvers.cpp:322): plain Cholesky.
//   * partialPivLu().inverse() of the transition T (assembly.cpp:76): T = I + E with
//     E^2 = 0, unit pivots and no fill, so the LU inverse is exactly I - E.
#pragma once

#include <cstdint>
#include <unordered_map>
#include <array>
#include <cstdint>
#include <functional>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace ddo {

// ------------------------------------------------------------------ dense algebra
using Vec = std::vector<double>;

/// Column-major dense matrix (the reference's Eigen::MatrixXd layout).
struct Mat {
  int r = 0, c = 0;
  std::vector<double> a;
  Mat() = default;
  Mat(int rows, int cols) : r(rows), c(cols), a(static_cast<size_t>(rows) * cols, 0.0) {}
  double& operator()(int i, int j) { return a[static_cast<size_t>(j) * r + i]; }
  double operator()(int i, int j) const { return a[static_cast<size_t>(j) * r + i]; }
  double* col(int j) { return a.data() + static_cast<size_t>(j) * r; }
  const double* col(int j) const { return a.data() + static_cast<size_t>(j) * r; }
  static Mat identity(int n) {
    Mat m(n, n);
    for (int i = 0; i < n; ++i) m(i, i) = 1.0;
    return m;
  }
};

Vec gemv(const Mat& A, const Vec& x);    // A x
Vec gemv_t(const Mat& A, const Vec& x);  // A^T x
Mat matmul(const Mat& A, const Mat& B);
Mat transpose(const Mat& A);
double dot(const Vec& a, const Vec& b);
double norm(const Vec& a);

struct Point {
  double x = 0, y = 0;
};

// ------------------------------------------------------------------ geometry (geometry.hpp)
struct Box {
  double x0 = 0, y0 = 0, x1 = 1, y1 = 1;
  double diam() const;
};

struct Edge {
  int id = -1;
  bool vertical = false;
  int k = 0, m = 0;
  std::array<int, 2> subs{-1, -1};
};

struct DomainPartition {
  int s = 1, n_grid = 3;
  std::vector<Box> boxes;
  std::vector<Edge> edges;
  std::vector<std::array<int, 4>> side_edge;  // L, R, B, T
  std::vector<std::vector<std::pair<int, int>>> neighbors;
  int n_subdomains() const { return s * s; }
  int cross_count() const { return (s - 1) * (s - 1); }
  int cross_id(int k, int m) const { return (m - 1) * (s - 1) + (k - 1); }
  int subdomain_of(const Point& x) const;
};

DomainPartition partition_domain(int s, int n_grid);

struct GammaPoint {
  Point xy;
  bool is_cross = false;
  int cross_id = -1, edge_id = -1, t = -1;
};

struct LocalEdge {
  int edge_id = -1;
  bool vertical = false;
  Point normal;
  std::vector<int> pts, geom_j;
  bool first_corner = false, last_corner = false;
};

struct PointSets {
  std::vector<std::vector<Point>> interior, boundary, interface;
  std::vector<std::vector<GammaPoint>> gamma_meta;
  std::vector<std::vector<LocalEdge>> local_edges;
};

PointSets classify_points(const DomainPartition& p);

struct InterfaceIndex {
  int cc = 1, n_delta = 0, n_pi = 0, interior_per_edge = 0;
  int n_mu() const { return n_delta + n_pi; }
  int delta_index(int edge_id, int comp, int t) const {
    return (edge_id * cc + comp) * interior_per_edge + (t - 1);
  }
  int pi_index(int cross_id, int comp) const { return n_delta + cross_id * cc + comp; }
  std::vector<std::vector<int>> local_to_global;
  std::vector<int> multiplicity;
  std::vector<char> is_pi;
};

InterfaceIndex build_interface_index(const DomainPartition& p, const PointSets& ps, int cc);

// ------------------------------------------------------------------ features (features.hpp)
struct FeatureLayer {
  int M = 0;
  std::vector<double> w0, w1, b;  // w = [w0; w1] (2 x M), b (M)
  double l = 0, r = 0;
  Box box;
  uint64_t seed = 0;
};

FeatureLayer init_layer(int M, const Box& box, double l, double r, uint64_t seed);
double scale_from_constant(double c, int M, const Box& box, double r);
Mat eval_derivative_matrix(const FeatureLayer& L, const std::vector<Point>& pts, int dx, int dy);

// ------------------------------------------------------------------ problems (problems.hpp)
using ScalarFn = std::function<double(const Point&)>;
using GradFn = std::function<Point(const Point&)>;

/// Gaussian random field sum_i amp_i sin(w_i . x + phase_i), 256 terms (problems.cpp:15-58).
struct GrfField {
  std::vector<double> amp, fx, fy, phase;
  double alpha = 0;
  uint64_t seed = 0;
};
GrfField sample_grf(double alpha, uint64_t seed);
double eval_grf(const GrfField& g, const Point& x);
Point grad_grf(const GrfField& g, const Point& x);
double eval_rho(const GrfField& g, const Point& x);   // tanh(grf) + 1.1
Point grad_rho(const GrfField& g, const Point& x);

struct ProblemParams {  // problems.hpp:64-68
  double alpha = 32.0;
  uint64_t forcing_seed = 2;
  uint64_t rho_seed = 3;
};

/// The reference catalogue (problems.cpp:132-188): poisson_sinpi, poisson_sin2pi_exp,
/// poisson_grf (GRF forcing), varcoef_poisson (-div(rho grad u) = 1, rho = tanh(GRF) + 1.1,
/// conormal flux), biharmonic_sinpi (lap^2 u = f, cc = bc = 2: value and Laplacian traces, normal
/// derivative and normal derivative of the Laplacian as fluxes), and C4's manufactured
/// "poisson_sin2pi_cos3pi_x2y".
struct ProblemSpec {
  std::string name;
  int kind = 0;  // 0 Poisson, 1 variable-coefficient Poisson, 2 biharmonic (ProblemKind)
  int components = 1, boundary_components = 1;
  ScalarFn forcing, boundary, boundary2, exact;  // boundary2: boundary data of component 1
  GradFn exact_grad;
  std::shared_ptr<GrfField> rho;  // varcoef_poisson
  double default_l = 32;
  bool has_exact() const { return static_cast<bool>(exact); }
  Mat interior_rows(const FeatureLayer& L, const std::vector<Point>& pts) const;
  Mat boundary_rows(const FeatureLayer& L, const std::vector<Point>& pts, int comp = 0) const;
  Mat trace_rows(const FeatureLayer& L, const std::vector<Point>& pts, int comp = 0) const;
  Mat flux_rows(const FeatureLayer& L, const std::vector<Point>& pts, const Point& n, int comp = 0) const;
};

ProblemSpec make_problem(const std::string& name, const ProblemParams& params = {});

// ------------------------------------------------------------------ assembly (assembly.hpp)
struct LocalBlocks {
  Mat K;
  Vec f;
  int n_int = 0, n_bnd = 0, n_gamma = 0, bc = 1, cc = 1;
  int rows() const { return n_int + bc * n_bnd + cc * n_gamma; }
  int trace_row0() const { return n_int + bc * n_bnd; }
  int trace_row(int comp, int p) const { return trace_row0() + comp * n_gamma + p; }
  std::vector<Mat> F_edges;
};

LocalBlocks assemble_local(const ProblemSpec& problem, const FeatureLayer& L,
                           const PointSets& ps, int i);
Mat build_transition(int m);

struct Transition {
  Mat T, Tinv;
};
Transition build_subdomain_transition(const std::vector<LocalEdge>& edges, int n_gamma,
                                      int n_grid);
void apply_change_of_variables(LocalBlocks& blocks, const Transition& t);

enum class FluxVariant { Pointwise, MeanEdge };

struct FluxScatter {
  int grow, lrow;
  double weight;
};

struct FluxBlocks {
  FluxVariant variant = FluxVariant::Pointwise;
  int n_flux = 0, n_delta = 0;
  std::vector<std::vector<FluxScatter>> scatter;
  std::vector<std::vector<int>> edge_row0;
};

FluxBlocks build_flux(const DomainPartition& p, const PointSets& ps, const InterfaceIndex& idx,
                      FluxVariant variant);

// ------------------------------------------------------------------ factorizations
/// Householder QR without pivoting (Eigen::HouseholderQR semantics), in place.
struct HouseholderQR {
  Mat qr;      // R in the upper triangle, reflector essentials below
  Vec hcoeffs;  // tau per reflector
  void compute(const Mat& A);
  Mat thinQ() const;  // rows x cols
};

/// Column-pivoted Householder QR (Eigen::ColPivHouseholderQR semantics).
struct ColPivQR {
  Mat qr;
  Vec hcoeffs;
  std::vector<int> transpositions;  // column k swapped with transpositions[k]
  std::vector<int> perm;            // A P = Q R: column k of A P is column perm[k] of A
  double maxpivot = 0;
  int nonzero_pivots = 0;
  void compute(const Mat& A);
  int rank(double threshold) const;
};

/// Complete orthogonal decomposition A P = Q [T 0; 0 0] Z (Eigen semantics).
struct COD {
  ColPivQR cpqr;
  Vec zcoeffs;
  int rnk = 0;
  double threshold = 1e-10;
  void compute(const Mat& A, double thr);
  Mat pseudo_inverse() const;     // cols x rows
  Mat householderQ_cols(int ncols) const;  // first ncols columns of Q
  Mat solve(const Mat& B) const;
};

/// Least-squares factor of a tall local matrix (solvers.cpp:24-78).
class LsFactor {
 public:
  LsFactor() = default;
  LsFactor(const Mat& K, double rank_tol);
  int rows() const { return rows_; }
  int cols() const { return cols_; }
  bool rank_deficient() const { return deficient_; }
  int rank() const { return rank_; }
  Vec apply_pinv(const Vec& v) const;
  Vec apply_pinv_transpose(const Vec& v) const;
  Vec apply_matrix(const Vec& x) const;
  Vec apply_projection(const Vec& v) const;
  Mat apply_pinv(const Mat& V) const;
  Mat apply_projection(const Mat& V) const;
  const Mat& Q() const { return Q_; }
  const Mat& pinv() const { return pinv_; }
  double qr_diag_ratio = 0;  // min|R_ii| / max|R_ii| of the unpivoted QR (branch test)

 private:
  int rows_ = 0, cols_ = 0, rank_ = 0;
  bool deficient_ = false;
  Mat Q_, R_, K_, pinv_, Rinv_;
};

/// CPU-baseline mode: LsFactor on SciPy's LAPACK (lapack.cpp); path nullptr / "" disables it.
bool set_lapack(const char* libpath);
bool lapack_enabled();
/// CPU-baseline mode: y = A x (trans: A^T x) through the LAPACK library's BLAS dgemv (one thread),
/// as Eigen's vectorised GEMV would run the reference's CG; false when the mode is off
bool blas_gemv(bool trans, const Mat& A, const Vec& x, Vec& y);
void lapack_lsfactor(const Mat& K, double rank_tol, bool& deficient, int& rank, double& ratio, Mat& Q, Mat& R,
                     Mat& Kcopy, Mat& pinv);

struct LLT {
  Mat L;
  bool ok = false;
  void compute(const Mat& A);
  Vec solve(const Vec& b) const;
};

// ------------------------------------------------------------------ solvers (solvers.hpp)
struct SolverOptions {
  FluxVariant flux_variant = FluxVariant::Pointwise;
  bool change_of_variables = false;
  double rank_tol = 1e-10;
  int workers = 1;     // setup-phase threads (reference knob)
  int cg_workers = 1;  // oracle-only: threads for per-subdomain CG work (1 = reference)
  int debug_flip_flux_row = -1;
  bool layers_only = false;  // oracle-only: stop after the seeded layers (field evaluation)
};

struct CgResult {
  Vec x;
  int iterations = 0;
  bool converged = false, negative_curvature = false;
  std::vector<double> residual_history;
};

using LinOp = std::function<Vec(const Vec&)>;
CgResult cg(const LinOp& op, const Vec& rhs, double rel_tol = 1e-9, int max_iter = 0,
            int stop_after = 0);

using LocalVecs = std::vector<Vec>;

struct Workspace {
  Workspace(const ProblemSpec& problem, int s, int n_grid, int M, double l, uint64_t seed,
            const SolverOptions& opts);

  ProblemSpec problem;
  SolverOptions opts;
  DomainPartition part;
  PointSets points;
  InterfaceIndex idx;
  FluxBlocks flux;
  std::vector<FeatureLayer> layers;
  std::vector<LocalBlocks> blocks;
  std::vector<LsFactor> fac;
  double assembly_seconds = 0, factorization_seconds = 0;

  int n_subs() const { return part.n_subdomains(); }
  int n_mu() const { return idx.n_mu(); }
  int n_delta() const { return idx.n_delta; }
  int n_pi() const { return idx.n_pi; }
  int n_pi_flux() const { return flux.n_flux - idx.n_delta; }

  std::vector<std::vector<std::pair<int, int>>> delta_rows, pi_rows;

  LocalVecs zero_locals() const;
  LocalVecs apply_B(const Vec& mu) const;
  LocalVecs apply_B_delta(const Vec& v) const;
  Vec apply_BT(const LocalVecs& x) const;
  Vec apply_BT_delta(const LocalVecs& x) const;
  Vec apply_A(const LocalVecs& c) const;
  Vec apply_A_delta(const LocalVecs& c) const;
  LocalVecs apply_AT(const Vec& w) const;
  LocalVecs apply_AT_delta(const Vec& w) const;
  std::vector<double> flux_row(int i, int lrow) const;
  Vec reduced_apply(const Vec& mu) const;

  bool coarse_built = false;
  Mat Dpp, Dpd;
  Vec dpi;
  Mat Spi;
  LLT Spi_llt;
  std::vector<Mat> Ypi, Gpi;
  void assemble_coarse();

  struct KtildeApply {
    LocalVecs c;
    Vec mu_pi;
    LocalVecs proj_top;
    Vec proj_bottom;
  };
  KtildeApply apply_ktilde_pinv(const LocalVecs& phi, const Vec& psi, bool want_projection) const;
  std::pair<LocalVecs, Vec> apply_ktilde_pinv_transpose(const LocalVecs& phi) const;
  Vec cs_reduced_apply(const Vec& v, const LinOp& weight) const;

  bool neumann_built = false;
  std::vector<Mat> Kbar, Cdelta;
  std::vector<LsFactor> nfac;
  std::vector<std::vector<int>> ndelta_map;
  std::vector<int> nflux_row0;
  double neumann_seconds = 0;
  void build_neumann();
  Vec apply_P(const Vec& v) const;
  Vec apply_PT(const Vec& u) const;

  // Deterministic per-subdomain parallel loop for the CG-phase work (cg_workers).
  void for_subs(const std::function<void(int)>& fn) const;
};

struct SolveReport {
  LocalVecs coeffs;
  Vec mu, mu_delta, mu_pi;
  int iterations = 0;
  bool converged = true, negative_curvature = false;
  std::vector<double> residual_history;
  double setup_seconds = 0, cg_seconds = 0, reconstruct_seconds = 0;
};

struct CgOptions {
  double rel_tol = 1e-9;
  int max_iter = 0;
  int stop_after = 0;  // oracle-only: stop after this many iterations (bounded CPU timing)
};

SolveReport ddelm_solve(Workspace& ws, const CgOptions& o = {});
SolveReport ddelm_cs_solve(Workspace& ws, const CgOptions& o = {});
SolveReport ddelm_nn_solve(Workspace& ws, double theta, const CgOptions& o = {});

enum class Method { Ddelm, DdelmCs, DdelmNn };

struct DenseOracle {
  Mat reduced_op;
  Vec reduced_rhs, mu_reduced, mu_full;
  LocalVecs coeffs;
};
DenseOracle dense_oracle_solve(Workspace& ws, Method method, double theta = 0.999);

// ------------------------------------------------------------------ metrics (metrics.hpp)
struct FieldSamples {
  Vec u, gx, gy;  // indexed b*n + a, x = a h, y = b h
};
FieldSamples sample_field(const DomainPartition& part, const std::vector<FeatureLayer>& layers,
                          const LocalVecs& coeffs, int n);

struct ErrorReport {
  double l2 = 0, h1 = 0;
  int grid_n = 0;
};
ErrorReport relative_errors(const FieldSamples& fs, int n,
                            const std::function<void(double, double, double&, double&, double&)>&
                                ref_at);
ErrorReport relative_errors_exact(const DomainPartition& part,
                                  const std::vector<FeatureLayer>& layers,
                                  const LocalVecs& coeffs, const ProblemSpec& prob, int n);

// thread helper (parallel.hpp semantics: strided static split, per-index writes only)
void parallel_for(int n, int workers, const std::function<void(int)>& fn);

// parity decomposition hooks (test infrastructure; model.cpp): record every feature tanh argument
// (single worker) or replace the feature tanh by a table keyed by the argument's bits
void set_tanh_record(std::vector<double>* rec);
void set_tanh_table(const std::unordered_map<std::uint64_t, double>* tab);
long long tanh_table_misses();

}  // namespace ddo

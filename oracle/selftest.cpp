// ORACLE SELF-TEST — TEST INFRASTRUCTURE ONLY.
// Re-runs the reference's own assertions against the restatement; these are the only pins
// the reference holds. Each block cites the reference test it mirrors.
// Exit code 0 = all checks pass. Run by tests/test_oracle.py (CPU).
#include <cmath>
#include <cstdio>
#include <limits>
#include <map>
#include <random>
#include <set>
#include <string>

#include "oracle.hpp"

using namespace ddo;

static int g_fail = 0, g_pass = 0;
#define CHECK(cond)                                                          \
  do {                                                                       \
    if (cond) {                                                              \
      ++g_pass;                                                              \
    } else {                                                                 \
      ++g_fail;                                                              \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);            \
    }                                                                        \
  } while (0)
#define CHECK_THROWS(expr)          \
  do {                              \
    bool thrown = false;            \
    try {                           \
      (void)(expr);                 \
    } catch (...) {                 \
      thrown = true;                \
    }                               \
    CHECK(thrown);                  \
  } while (0)

namespace {

double maxabs(const Mat& A) {
  double m = 0;
  for (double e : A.a) m = std::max(m, std::abs(e));
  return m;
}
double maxabs_diff(const Mat& A, const Mat& B) {
  double m = 0;
  for (size_t t = 0; t < A.a.size(); ++t) m = std::max(m, std::abs(A.a[t] - B.a[t]));
  return m;
}
Vec sub(const Vec& a, const Vec& b) {
  Vec c(a.size());
  for (size_t i = 0; i < a.size(); ++i) c[i] = a[i] - b[i];
  return c;
}
bool approx(double a, double b, double eps = 1e-12) {
  return std::abs(a - b) <= eps * std::max({1.0, std::abs(a), std::abs(b)});
}

Mat random_matrix(int rows, int cols, uint64_t seed) {  // test_solvers.cpp:14-21
  std::mt19937_64 gen(seed);
  std::normal_distribution<double> n;
  Mat A(rows, cols);
  for (int j = 0; j < cols; ++j)
    for (int i = 0; i < rows; ++i) A(i, j) = n(gen);
  return A;
}

/// Independent pseudo-inverse of a full-column-rank matrix: (A^T A)^{-1} A^T via Cholesky.
Mat normal_pinv(const Mat& A) {
  Mat G = matmul(transpose(A), A);
  LLT llt;
  llt.compute(G);
  Mat At = transpose(A), P(A.c, A.r);
  for (int j = 0; j < A.r; ++j) {
    Vec col(At.col(j), At.col(j) + At.r);
    Vec x = llt.solve(col);
    std::copy(x.begin(), x.end(), P.col(j));
  }
  return P;
}

const Box kBox{0.25, 0.5, 0.5, 0.75};

double fd_derivative(const FeatureLayer& L, int j, Point x, int a, int b, double h) {
  if (a > 0)
    return (fd_derivative(L, j, {x.x + h, x.y}, a - 1, b, h) - fd_derivative(L, j, {x.x - h, x.y}, a - 1, b, h)) / (2 * h);
  if (b > 0)
    return (fd_derivative(L, j, {x.x, x.y + h}, a, b - 1, h) - fd_derivative(L, j, {x.x, x.y - h}, a, b - 1, h)) / (2 * h);
  return std::tanh(L.w0[j] * x.x + L.w1[j] * x.y + L.b[j]);
}

void test_features() {  // test_features.cpp
  CHECK_THROWS(init_layer(0, kBox, 1, 1, 7));
  CHECK_THROWS(init_layer(8, kBox, 0, 1, 7));
  CHECK_THROWS(init_layer(8, kBox, 1, 0, 7));
  const double l = 3.0, r = 0.2;
  FeatureLayer L = init_layer(256, kBox, l, r, 7);
  for (int j = 0; j < L.M; ++j) {
    CHECK(std::abs(L.w0[j]) <= l && std::abs(L.w1[j]) <= l);
    const double bx = std::max(std::abs(kBox.x0 - r), std::abs(kBox.x1 + r));
    const double by = std::max(std::abs(kBox.y0 - r), std::abs(kBox.y1 + r));
    CHECK(std::abs(L.b[j]) <= std::abs(L.w0[j]) * bx + std::abs(L.w1[j]) * by + 1e-15);
  }
  FeatureLayer a = init_layer(64, kBox, 4, 0.3, 42), b = init_layer(64, kBox, 4, 0.3, 42),
               c = init_layer(64, kBox, 4, 0.3, 43);
  CHECK(a.w0 == b.w0 && a.w1 == b.w1 && a.b == b.b);
  CHECK(a.w0 != c.w0);
  std::vector<Point> pts{{0.3, 0.6}, {0.45, 0.55}};
  CHECK(maxabs_diff(eval_derivative_matrix(a, pts, 2, 1), eval_derivative_matrix(b, pts, 2, 1)) == 0.0);

  FeatureLayer g = init_layer(4, kBox, 1, 0.1, 1);
  CHECK_THROWS(eval_derivative_matrix(g, std::vector<Point>{{0.3, 0.6}}, 3, 2));
  g.w0[0] = 1;
  g.w1[0] = 0;
  g.b[0] = 0;
  std::vector<Point> origin{{0.0, 0.0}};
  CHECK(std::abs(eval_derivative_matrix(g, origin, 0, 0)(0, 0)) < 1e-15);
  CHECK(approx(eval_derivative_matrix(g, origin, 1, 0)(0, 0), 1.0));
  CHECK(std::abs(eval_derivative_matrix(g, origin, 0, 1)(0, 0)) < 1e-15);

  FeatureLayer fl = init_layer(12, kBox, 2.5, 0.2, 11);  // test_features.cpp:80-99
  std::mt19937_64 gen(5);
  std::uniform_real_distribution<double> ux(kBox.x0, kBox.x1), uy(kBox.y0, kBox.y1);
  std::vector<Point> fpts;
  for (int k = 0; k < 10; ++k) {
    const double x = ux(gen), y = uy(gen);
    fpts.push_back({x, y});
  }
  bool fd_ok = true;
  for (int da = 0; da <= 4; ++da)
    for (int db = 0; da + db <= 4; ++db) {
      const Mat D = eval_derivative_matrix(fl, fpts, da, db);
      const double h = (da + db <= 2) ? 1e-4 : 2e-3, tol = (da + db <= 2) ? 1e-4 : 1e-2;
      for (int k = 0; k < 10; ++k)
        for (int j = 0; j < fl.M; ++j) {
          const double fd = fd_derivative(fl, j, fpts[k], da, db, h);
          fd_ok = fd_ok && std::abs(D(k, j) - fd) / std::max(1.0, std::abs(fd)) < tol;
        }
    }
  CHECK(fd_ok);
  const double rr = 0.2, d = std::hypot(kBox.x1 - kBox.x0 + 2 * rr, kBox.y1 - kBox.y0 + 2 * rr);
  CHECK(approx(scale_from_constant(1.0, 1024, kBox, rr), 32.0 / d));
  CHECK(approx(scale_from_constant(0.5, 256, kBox, rr), 8.0 / d));
}

void test_geometry() {  // test_geometry.cpp
  CHECK_THROWS(partition_domain(0, 10));
  CHECK_THROWS(partition_domain(2, 2));
  {
    DomainPartition p = partition_domain(4, 80);
    CHECK(p.edges.size() == 24);
    CHECK(p.cross_count() == 9);
    PointSets ps = classify_points(p);
    std::set<int> crosses;
    for (int i = 0; i < p.n_subdomains(); ++i)
      for (const GammaPoint& g : ps.gamma_meta[i])
        if (g.is_cross) crosses.insert(g.cross_id);
    CHECK(crosses.size() == 9);
  }
  {
    DomainPartition p = partition_domain(2, 4);
    PointSets ps = classify_points(p);
    for (int i = 0; i < 4; ++i) {
      CHECK(ps.interior[i].size() == 4);
      CHECK(ps.boundary[i].size() == 7);
      CHECK(ps.interface[i].size() == 5);
    }
  }
  {
    DomainPartition p = partition_domain(2, 160);
    PointSets ps = classify_points(p);
    for (int i = 0; i < 4; ++i) CHECK(ps.interface[i].size() == 2 * 160 - 1 - 2);
  }
  {
    DomainPartition p = partition_domain(3, 10);
    CHECK(p.subdomain_of({0.0, 0.0}) == 0);
    CHECK(p.subdomain_of({0.99, 0.99}) == 8);
    CHECK(p.subdomain_of({1.0, 1.0}) == 8);
    CHECK(p.subdomain_of({0.5, 0.1}) == 1);
  }
  for (int cc : {1, 2}) {
    DomainPartition p = partition_domain(3, 8);
    PointSets ps = classify_points(p);
    InterfaceIndex idx = build_interface_index(p, ps, cc);
    CHECK(idx.n_delta == static_cast<int>(p.edges.size()) * cc * (p.n_grid - 2));
    CHECK(idx.n_pi == p.cross_count() * cc);
    for (int g = 0; g < idx.n_mu(); ++g) CHECK(idx.multiplicity[g] == (idx.is_pi[g] ? 4 : 2));
  }
  {
    DomainPartition p = partition_domain(3, 7);
    PointSets ps = classify_points(p);
    InterfaceIndex idx = build_interface_index(p, ps, 1);
    std::vector<Point> coord(idx.n_mu(), Point{-1, -1});
    bool same = true;
    for (int i = 0; i < p.n_subdomains(); ++i)
      for (size_t q = 0; q < ps.interface[i].size(); ++q) {
        const int g = idx.local_to_global[i][q];
        if (coord[g].x >= 0)
          same = same && coord[g].x == ps.interface[i][q].x && coord[g].y == ps.interface[i][q].y;
        else
          coord[g] = ps.interface[i][q];
      }
    CHECK(same);
  }
  {
    DomainPartition p = partition_domain(2, 6);
    PointSets ps = classify_points(p);
    for (int i = 0; i < 4; ++i) {
      CHECK(ps.local_edges[i].size() == 2);
      for (const LocalEdge& le : ps.local_edges[i]) {
        for (size_t q = 1; q < le.geom_j.size(); ++q) CHECK(le.geom_j[q] > le.geom_j[q - 1]);
        const Box& b = p.boxes[i];
        const double cx = 0.5 * (b.x0 + b.x1), cy = 0.5 * (b.y0 + b.y1);
        const Point& x0 = ps.interface[i][le.pts[0]];
        CHECK(le.normal.x * (x0.x - cx) + le.normal.y * (x0.y - cy) > 0);
      }
    }
  }
}

struct Instance {  // test_assembly.cpp:13-28
  DomainPartition part;
  PointSets ps;
  ProblemSpec problem;
  std::vector<FeatureLayer> layers;
  std::vector<LocalBlocks> blocks;
  Instance(const std::string& name, int s, int n) : part(partition_domain(s, n)) {
    ps = classify_points(part);
    problem = make_problem(name);
    for (int i = 0; i < part.n_subdomains(); ++i) {
      layers.push_back(init_layer(24, part.boxes[i], 4, part.boxes[i].diam() / 2, 100 + i));
      blocks.push_back(assemble_local(problem, layers[i], ps, i));
    }
  }
};

void test_assembly() {  // test_assembly.cpp
  {
    Instance inst("poisson_sinpi", 2, 6);
    for (int i = 0; i < 4; ++i) {
      const LocalBlocks& b = inst.blocks[i];
      const FeatureLayer& L = inst.layers[i];
      CHECK(b.rows() == b.n_int + b.n_bnd + b.n_gamma);
      Mat lap = eval_derivative_matrix(L, inst.ps.interior[i], 2, 0);
      Mat l2 = eval_derivative_matrix(L, inst.ps.interior[i], 0, 2);
      for (size_t t = 0; t < lap.a.size(); ++t) lap.a[t] += l2.a[t];
      double worst = 0;
      for (int j = 0; j < L.M; ++j)
        for (int k = 0; k < b.n_int; ++k) worst = std::max(worst, std::abs(b.K(k, j) + lap(k, j)));
      CHECK(worst < 1e-13 * maxabs(lap));
      bool fok = true;
      for (int k = 0; k < b.n_int; ++k) fok = fok && approx(b.f[k], inst.problem.forcing(inst.ps.interior[i][k]));
      CHECK(fok);
      const Mat evb = eval_derivative_matrix(L, inst.ps.boundary[i], 0, 0);
      const Mat evg = eval_derivative_matrix(L, inst.ps.interface[i], 0, 0);
      double db = 0, dg = 0, ft = 0;
      for (int j = 0; j < L.M; ++j) {
        for (int k = 0; k < b.n_bnd; ++k) db = std::max(db, std::abs(b.K(b.n_int + k, j) - evb(k, j)));
        for (int k = 0; k < b.n_gamma; ++k) dg = std::max(dg, std::abs(b.K(b.trace_row0() + k, j) - evg(k, j)));
      }
      for (int k = 0; k < b.n_gamma; ++k) ft = std::max(ft, std::abs(b.f[b.trace_row0() + k]));
      CHECK(db == 0.0);
      CHECK(dg == 0.0);
      CHECK(ft == 0.0);
      CHECK(b.F_edges.size() == inst.ps.local_edges[i].size());
      for (size_t e = 0; e < b.F_edges.size(); ++e) {
        const LocalEdge& le = inst.ps.local_edges[i][e];
        std::vector<Point> pts;
        for (int q : le.pts) pts.push_back(inst.ps.interface[i][q]);
        Mat ex = eval_derivative_matrix(L, pts, 1, 0), ey = eval_derivative_matrix(L, pts, 0, 1);
        for (size_t t = 0; t < ex.a.size(); ++t) ex.a[t] = le.normal.x * ex.a[t] + le.normal.y * ey.a[t];
        CHECK(maxabs_diff(b.F_edges[e], ex) < 1e-13 * maxabs(ex));
      }
    }
  }
  CHECK_THROWS(build_transition(1));
  CHECK(maxabs_diff(build_transition(2), Mat::identity(2)) == 0.0);
  {
    const Mat T = build_transition(6);  // test_assembly.cpp:84-95 (known-answer)
    Mat ex = Mat::identity(6);
    const double c0[6] = {1, 4.0 / 5, 3.0 / 5, 2.0 / 5, 1.0 / 5, 0};
    for (int k = 0; k < 6; ++k) {
      ex(k, 0) = c0[k];
      ex(k, 5) = c0[5 - k];
    }
    CHECK(maxabs_diff(T, ex) < 1e-15);
  }
  {
    DomainPartition p = partition_domain(3, 8);
    PointSets ps = classify_points(p);
    for (int i = 0; i < 9; ++i) {
      const int ng = static_cast<int>(ps.interface[i].size());
      Transition t = build_subdomain_transition(ps.local_edges[i], ng, p.n_grid);
      CHECK(maxabs_diff(matmul(t.Tinv, t.T), Mat::identity(ng)) < 1e-12);
      CHECK(maxabs_diff(matmul(t.Tinv, t.T), Mat::identity(ng)) == 0.0);  // exact (I - E)(I + E)
      for (int q = 0; q < ng; ++q)
        if (ps.gamma_meta[i][q].is_cross) {
          double rs = 0;
          for (int k = 0; k < ng; ++k) rs += std::abs(t.T(q, k));
          CHECK(t.T(q, q) == 1.0);
          CHECK(approx(rs, 1.0));
        }
    }
  }
  {
    Instance inst("poisson_sinpi", 3, 7);
    const int i = 4;
    LocalBlocks b = inst.blocks[i];
    const Mat before = b.K;
    Transition t = build_subdomain_transition(inst.ps.local_edges[i], b.n_gamma, 7);
    apply_change_of_variables(b, t);
    double top = 0;
    for (int j = 0; j < b.K.c; ++j)
      for (int k = 0; k < b.trace_row0(); ++k) top = std::max(top, std::abs(b.K(k, j) - before(k, j)));
    CHECK(top == 0.0);
    Mat old(b.n_gamma, b.K.c), now(b.n_gamma, b.K.c);
    for (int j = 0; j < b.K.c; ++j)
      for (int k = 0; k < b.n_gamma; ++k) {
        old(k, j) = before(b.trace_row0() + k, j);
        now(k, j) = b.K(b.trace_row0() + k, j);
      }
    const Mat ex = matmul(t.Tinv, old);
    CHECK(maxabs_diff(now, ex) < 1e-12 * maxabs(ex));
    Transition wrong = build_subdomain_transition(inst.ps.local_edges[0],
                                                  static_cast<int>(inst.ps.interface[0].size()), 7);
    LocalBlocks b2 = inst.blocks[i];
    CHECK_THROWS(apply_change_of_variables(b2, wrong));
  }
  {
    DomainPartition p = partition_domain(2, 6);
    PointSets ps = classify_points(p);
    InterfaceIndex idx = build_interface_index(p, ps, 1);
    FluxBlocks fb = build_flux(p, ps, idx, FluxVariant::Pointwise);
    CHECK(fb.n_delta == idx.n_delta);
    CHECK(fb.n_flux == idx.n_delta + 2);
    std::map<int, int> count;
    for (int i = 0; i < 4; ++i)
      for (const FluxScatter& sc : fb.scatter[i]) {
        CHECK(sc.weight == 1.0);
        ++count[sc.grow];
      }
    CHECK(static_cast<int>(count.size()) == fb.n_flux);
    for (const auto& [grow, c] : count) CHECK(c == (grow < fb.n_delta ? 2 : 4));
  }
  {
    const int n = 6;
    DomainPartition p = partition_domain(2, n);
    PointSets ps = classify_points(p);
    InterfaceIndex idx = build_interface_index(p, ps, 1);
    FluxBlocks fb = build_flux(p, ps, idx, FluxVariant::MeanEdge);
    std::map<int, double> total;
    std::map<int, int> entries;
    for (int i = 0; i < 4; ++i)
      for (const FluxScatter& sc : fb.scatter[i]) {
        if (sc.grow < fb.n_delta) {
          CHECK(sc.weight == 1.0);
        } else {
          CHECK(approx(sc.weight, 1.0 / (n - 1)));
          total[sc.grow] += sc.weight;
          ++entries[sc.grow];
        }
      }
    for (const auto& [g, w] : total) CHECK(approx(w, 4.0));
    for (const auto& [g, c] : entries) CHECK(c == 4 * (n - 1));
  }
  {
    Instance inst("poisson_sinpi", 2, 5);
    FeatureLayer L = inst.layers[0];
    for (int j = 0; j < L.M; ++j) {
      L.w0[j] = L.w1[j] = 0;
      L.b[j] = 0.3;
    }
    const LocalEdge& le = inst.ps.local_edges[0][0];
    std::vector<Point> pts;
    for (int q : le.pts) pts.push_back(inst.ps.interface[0][q]);
    CHECK(maxabs(inst.problem.flux_rows(L, pts, le.normal)) == 0.0);
  }
}

Workspace tiny_workspace(const SolverOptions& o = {}) {  // test_solvers.cpp:27-29
  return Workspace(make_problem("poisson_sinpi"), 2, 10, 64, 8.0, 1, o);
}

Vec randn(std::mt19937_64& gen, int n) {
  std::normal_distribution<double> nd;
  Vec v(n);
  for (auto& e : v) e = nd(gen);
  return v;
}

void test_lsfactor() {  // test_solvers.cpp:33-85
  {
    const Mat A = random_matrix(40, 12, 3);
    LsFactor fac(A, 1e-10);
    CHECK(!fac.rank_deficient());
    const Mat P = normal_pinv(A);
    std::mt19937_64 gen(4);
    for (int t = 0; t < 5; ++t) {
      Vec v = randn(gen, 40), u = randn(gen, 12);
      CHECK(norm(sub(fac.apply_pinv(v), gemv(P, v))) < 1e-12 * norm(v));
      CHECK(norm(sub(fac.apply_pinv_transpose(u), gemv_t(P, u))) < 1e-12 * norm(u));
      CHECK(norm(sub(fac.apply_matrix(u), gemv(A, u))) < 1e-13 * norm(gemv(A, u)));
      CHECK(approx(dot(fac.apply_pinv(v), u), dot(v, fac.apply_pinv_transpose(u)), 1e-10));
    }
  }
  {
    const Mat A = random_matrix(30, 8, 7);
    LsFactor fac(A, 1e-10);
    std::mt19937_64 gen(8);
    for (int t = 0; t < 5; ++t) {
      Vec v = randn(gen, 30), w = randn(gen, 30);
      const Vec pv = fac.apply_projection(v);
      CHECK(norm(sub(fac.apply_projection(pv), pv)) < 1e-12 * norm(pv));
      CHECK(approx(dot(pv, w), dot(v, fac.apply_projection(w)), 1e-12));
      CHECK(norm(sub(fac.apply_matrix(fac.apply_pinv(v)), pv)) < 1e-10 * norm(v));
    }
    Vec x(8);
    for (int i = 0; i < 8; ++i) x[i] = -1.0 + 2.0 * i / 7.0;
    const Vec r = gemv(A, x);
    CHECK(norm(sub(fac.apply_projection(r), r)) < 1e-12 * norm(r));
  }
  {
    Mat A = random_matrix(20, 6, 9);
    for (int i = 0; i < 20; ++i) A(i, 5) = A(i, 0);
    LsFactor fac(A, 1e-10);
    CHECK(fac.rank_deficient());
    CHECK(fac.rank() == 5);
    // Independent pinv: A = B C with B = A(:, 0:5) full column rank, C = [I | e_0].
    Mat B(20, 5), C(5, 6);
    for (int j = 0; j < 5; ++j) {
      for (int i = 0; i < 20; ++i) B(i, j) = A(i, j);
      C(j, j) = 1.0;
    }
    C(0, 5) = 1.0;
    const Mat Cp = transpose(normal_pinv(transpose(C)));  // C^T (C C^T)^{-1}
    const Mat P = matmul(Cp, normal_pinv(B));
    Vec v(20);
    for (int i = 0; i < 20; ++i) v[i] = i / 19.0;
    CHECK(norm(sub(fac.apply_pinv(v), gemv(P, v))) < 1e-10 * norm(v));
    const Vec pv = fac.apply_projection(v);
    CHECK(norm(sub(fac.apply_projection(pv), pv)) < 1e-12 * norm(pv));
    CHECK(norm(sub(pv, gemv(A, gemv(P, v)))) < 1e-10 * norm(v));
  }
}

void test_cg() {  // test_solvers.cpp:87-105
  const int n = 50;
  Vec rhs(n);
  for (int i = 0; i < n; ++i) rhs[i] = 1.0 + i / 49.0;
  CgResult r1 = cg([](const Vec& x) { return x; }, rhs, 1e-12);
  CHECK(r1.converged);
  CHECK(r1.iterations == 1);
  CHECK(norm(sub(r1.x, rhs)) < 1e-12 * norm(rhs));
  Vec d(n);
  for (int i = 0; i < n; ++i) d[i] = (i % 3 == 0) ? 1.0 : (i % 3 == 1 ? 4.0 : 9.0);
  CgResult r2 = cg([&](const Vec& x) {
    Vec y(n);
    for (int i = 0; i < n; ++i) y[i] = d[i] * x[i];
    return y;
  }, rhs, 1e-12);
  CHECK(r2.converged);
  CHECK(r2.iterations <= 3);
  Vec ex(n);
  for (int i = 0; i < n; ++i) ex[i] = rhs[i] / d[i];
  CHECK(norm(sub(r2.x, ex)) < 1e-10);
  CHECK(r2.residual_history.size() == static_cast<size_t>(r2.iterations));
}

struct OracleCheck {
  double mu_diff = 0, field_diff = 0, op_diff = 0;
  bool pass = false;
};

/// runner.cpp:252-316: tol 1e-12 solve vs the dense brute-force oracle.
OracleCheck oracle_check(Method m, double theta, int flip = -1) {
  SolverOptions o;
  const bool coarse = m != Method::Ddelm;
  o.flux_variant = coarse ? FluxVariant::MeanEdge : FluxVariant::Pointwise;
  o.change_of_variables = coarse;
  o.debug_flip_flux_row = flip;
  Workspace ws(make_problem("poisson_sinpi"), 2, 10, 64, 8.0, 1, o);
  CgOptions tight{1e-12, 0, 0};
  SolveReport rep = m == Method::Ddelm     ? ddelm_solve(ws, tight)
                    : m == Method::DdelmCs ? ddelm_cs_solve(ws, tight)
                                           : ddelm_nn_solve(ws, theta, tight);
  DenseOracle dor = dense_oracle_solve(ws, m, theta);
  OracleCheck r;
  const double mn = norm(dor.mu_full);
  r.mu_diff = norm(sub(rep.mu, dor.mu_full)) / (mn > 0 ? mn : 1.0);
  const FieldSamples fo = sample_field(ws.part, ws.layers, dor.coeffs, 65);
  const FieldSamples fs = sample_field(ws.part, ws.layers, rep.coeffs, 65);
  r.field_diff = relative_errors(fs, 65, [&](double x, double y, double& u, double& gx, double& gy) {
                   const int a = static_cast<int>(std::lround(x * 64)), b = static_cast<int>(std::lround(y * 64));
                   u = fo.u[b * 65 + a];
                   gx = fo.gx[b * 65 + a];
                   gy = fo.gy[b * 65 + a];
                 }).l2;
  LinOp opfn;
  if (m == Method::Ddelm) {
    opfn = [&ws](const Vec& v) { return ws.reduced_apply(v); };
  } else {
    ws.assemble_coarse();
    LinOp weight = [](const Vec& x) { return x; };
    if (m == Method::DdelmNn && theta > 0) {
      ws.build_neumann();
      weight = [&ws, theta](const Vec& x) {
        Vec w = ws.apply_PT(ws.apply_P(x));
        for (auto& e : w) e *= theta;
        if (theta < 1.0)
          for (size_t i = 0; i < w.size(); ++i) w[i] += (1.0 - theta) * x[i];
        return w;
      };
    }
    opfn = [&ws, weight](const Vec& v) { return ws.cs_reduced_apply(v, weight); };
  }
  const int dim = dor.reduced_op.c;
  for (int j = 0; j < dim; ++j) {
    Vec e(dim, 0.0);
    e[j] = 1.0;
    const Vec col = opfn(e);
    for (int i = 0; i < dim; ++i) r.op_diff = std::max(r.op_diff, std::abs(col[i] - dor.reduced_op(i, j)));
  }
  r.pass = r.mu_diff < 1e-6 && r.field_diff < 1e-6 && r.op_diff < 1e-6;
  return r;
}

void test_solvers() {  // test_solvers.cpp:107-217 and acceptance criteria 1, 2, 7, 10
  {
    Workspace ws = tiny_workspace();
    CHECK(!ws.fac[0].rank_deficient());  // the tiny instance is full rank
    const int n = ws.n_mu();
    std::mt19937_64 gen(11);
    for (int t = 0; t < 10; ++t) {
      Vec u = randn(gen, n), v = randn(gen, n);
      Vec Au = ws.reduced_apply(u), Av = ws.reduced_apply(v);
      const double scale = norm(Au) * norm(v) + norm(u) * norm(Av);
      CHECK(std::abs(dot(Au, v) - dot(u, Av)) < 1e-10 * scale);
      CHECK(dot(u, Au) > -1e-10 * dot(u, u));
    }
  }
  {
    Workspace ws = tiny_workspace();
    DenseOracle dor = dense_oracle_solve(ws, Method::DdelmCs);
    ws.assemble_coarse();
    std::mt19937_64 gen(13);
    for (int t = 0; t < 4; ++t) {
      Vec v = randn(gen, ws.n_delta());
      Vec lhs = ws.cs_reduced_apply(v, [](const Vec& x) { return x; });
      Vec ref = gemv(dor.reduced_op, v);
      CHECK(norm(sub(lhs, ref)) < 1e-8 * norm(ref));
    }
  }
  {
    Workspace ws = tiny_workspace();
    ws.assemble_coarse();
    std::mt19937_64 gen(17);
    LocalVecs phi = ws.zero_locals();
    for (auto& p : phi) p = randn(gen, static_cast<int>(p.size()));
    Vec psi = randn(gen, ws.n_pi_flux());
    auto once = ws.apply_ktilde_pinv(phi, psi, true);
    auto twice = ws.apply_ktilde_pinv(once.proj_top, once.proj_bottom, true);
    double num = 0, den = 0;
    for (int i = 0; i < ws.n_subs(); ++i) {
      Vec d = sub(twice.proj_top[i], once.proj_top[i]);
      num += dot(d, d);
      den += dot(once.proj_top[i], once.proj_top[i]);
    }
    Vec d = sub(twice.proj_bottom, once.proj_bottom);
    num += dot(d, d);
    den += dot(once.proj_bottom, once.proj_bottom);
    CHECK(std::sqrt(num / den) < 1e-10);
  }
  {
    Workspace ws = tiny_workspace();
    ws.assemble_coarse();
    ws.build_neumann();
    const int nd = ws.n_delta();
    Mat P(nd, nd);
    for (int j = 0; j < nd; ++j) {
      Vec e(nd, 0.0);
      e[j] = 1.0;
      Vec c = ws.apply_P(e);
      std::copy(c.begin(), c.end(), P.col(j));
    }
    std::mt19937_64 gen(19);
    for (int t = 0; t < 5; ++t) {
      Vec u = randn(gen, nd), v = randn(gen, nd);
      CHECK(norm(sub(ws.apply_P(v), gemv(P, v))) < 1e-10 * norm(gemv(P, v)));
      CHECK(norm(sub(ws.apply_PT(u), gemv_t(P, u))) < 1e-10 * norm(gemv_t(P, u)));
    }
  }
  {
    Workspace ws = tiny_workspace();
    SolveReport cs = ddelm_cs_solve(ws);
    SolveReport nn = ddelm_nn_solve(ws, 0.0);
    CHECK(nn.iterations == cs.iterations);
    CHECK(nn.mu == cs.mu);
    bool same = true;
    for (int i = 0; i < ws.n_subs(); ++i) same = same && nn.coeffs[i] == cs.coeffs[i];
    CHECK(same);
    CHECK_THROWS(ddelm_nn_solve(ws, -0.1));
    CHECK_THROWS(ddelm_nn_solve(ws, 1.5));
  }
  {
    Workspace ws = tiny_workspace();
    SolveReport rep = ddelm_solve(ws);
    CHECK(rep.converged);
    const LocalVecs bmu = ws.apply_B(rep.mu);
    for (int i : {0, 1}) {
      const LocalBlocks& b = ws.blocks[i];
      Vec kc = gemv(b.K, rep.coeffs[i]);
      for (int p = 0; p < b.n_gamma; ++p) {
        const GammaPoint& gp = ws.points.gamma_meta[i][p];
        if (gp.is_cross) continue;
        const int g = ws.idx.delta_index(gp.edge_id, 0, gp.t);
        const int row = b.trace_row(0, p);
        const double residual = kc[row] - (b.f[row] - bmu[i][row]);
        const Mat ev = eval_derivative_matrix(ws.layers[i], std::vector<Point>{ws.points.interface[i][p]}, 0, 0);
        double v = 0;
        for (int j = 0; j < ev.c; ++j) v += ev(0, j) * rep.coeffs[i][j];
        CHECK(std::abs(v - rep.mu[g] - residual) < 1e-10);
      }
    }
  }
  // acceptance criterion 1 (acceptance.cpp:72-93) and the corruption hook (test_runner.cpp:188-200)
  double worst = 0;
  bool pass1 = true;
  for (auto [m, th] : std::vector<std::pair<Method, double>>{{Method::Ddelm, 0.0}, {Method::DdelmCs, 0.0},
                                                            {Method::DdelmNn, 0.0}, {Method::DdelmNn, 1.0}}) {
    OracleCheck r = oracle_check(m, th);
    pass1 = pass1 && r.pass;
    worst = std::max({worst, r.mu_diff, r.field_diff, r.op_diff});
  }
  std::printf("criterion 1: dense-reference equivalence worst diff %.2e\n", worst);
  CHECK(pass1);
  OracleCheck corrupted = oracle_check(Method::Ddelm, 0.0, 3);
  CHECK(!corrupted.pass);
  CHECK(corrupted.op_diff > 1e-3);
  // acceptance criterion 2 (acceptance.cpp:96-166)
  {
    SolverOptions o;
    Workspace ws(make_problem("poisson_sinpi"), 2, 10, 64, 8.0, 1, o);
    ws.assemble_coarse();
    ws.build_neumann();
    std::mt19937_64 gen(23);
    const double theta = 0.999;
    LinOp ident = [](const Vec& x) { return x; };
    LinOp nnw = [&](const Vec& x) {
      Vec w = ws.apply_PT(ws.apply_P(x));
      for (size_t i = 0; i < w.size(); ++i) w[i] = theta * w[i] + (1 - theta) * x[i];
      return w;
    };
    std::vector<LinOp> ops = {[&](const Vec& v) { return ws.reduced_apply(v); },
                              [&](const Vec& v) { return ws.cs_reduced_apply(v, ident); },
                              [&](const Vec& v) { return ws.cs_reduced_apply(v, nnw); }};
    std::vector<int> dims = {ws.n_mu(), ws.n_delta(), ws.n_delta()};
    double wsym = 0, wpsd = 0;
    for (size_t k = 0; k < ops.size(); ++k) {
      for (int t = 0; t < 20; ++t) {
        Vec u = randn(gen, dims[k]), v = randn(gen, dims[k]);
        Vec Au = ops[k](u), Av = ops[k](v);
        wsym = std::max(wsym, std::abs(dot(Au, v) - dot(u, Av)) / (norm(Au) * norm(v) + norm(u) * norm(Av)));
      }
      for (int t = 0; t < 50; ++t) {
        Vec v = randn(gen, dims[k]);
        wpsd = std::min(wpsd, dot(v, ops[k](v)) / dot(v, v));
      }
    }
    std::printf("criterion 2: symmetry worst %.2e, PSD worst %.2e\n", wsym, wpsd);
    CHECK(wsym < 1e-10);
    CHECK(wpsd >= -1e-10);
  }
  // acceptance criterion 7 (acceptance.cpp:273-307): basis-change invariance
  {
    const ProblemSpec prob = make_problem("poisson_sinpi");
    SolverOptions a, b;
    b.change_of_variables = true;
    Workspace nodal(prob, 2, 20, 400, 8.0, 1, a), cov(prob, 2, 20, 400, 8.0, 1, b);
    CgOptions tight{1e-12, 0, 0};
    SolveReport ra = ddelm_solve(nodal, tight), rb = ddelm_solve(cov, tight);
    const FieldSamples fa = sample_field(nodal.part, nodal.layers, ra.coeffs, 65);
    const FieldSamples fb = sample_field(cov.part, cov.layers, rb.coeffs, 65);
    double num = 0, den = 0;
    for (size_t t = 0; t < fa.u.size(); ++t) {
      num += (fa.u[t] - fb.u[t]) * (fa.u[t] - fb.u[t]);
      den += fa.u[t] * fa.u[t];
    }
    std::printf("criterion 7: basis-change field difference %.2e\n", std::sqrt(num / den));
    CHECK(std::sqrt(num / den) < 1e-6);
  }
  // acceptance criterion 10 (acceptance.cpp:372-389): determinism
  {
    SolverOptions o;
    o.flux_variant = FluxVariant::MeanEdge;
    o.change_of_variables = true;
    Workspace w1(make_problem("poisson_sinpi"), 2, 10, 64, 8.0, 1, o), w2(make_problem("poisson_sinpi"), 2, 10, 64, 8.0, 1, o);
    SolveReport a = ddelm_cs_solve(w1), b = ddelm_cs_solve(w2);
    const ErrorReport ea = relative_errors_exact(w1.part, w1.layers, a.coeffs, w1.problem, 65);
    const ErrorReport eb = relative_errors_exact(w2.part, w2.layers, b.coeffs, w2.problem, 65);
    CHECK(a.iterations == b.iterations);
    CHECK(ea.l2 == eb.l2 && ea.h1 == eb.h1);
  }
}

}  // namespace

void test_problems_grf() {  // test_problems.cpp: GRF sampler, rho, variable-coefficient rows
  const GrfField a = sample_grf(32, 5), b = sample_grf(32, 5), c = sample_grf(32, 6);
  CHECK(a.amp == b.amp && a.fx == b.fx && a.fy == b.fy && a.phase == b.phase);
  CHECK(a.amp != c.amp);
  bool in_range = true;
  for (double ph : a.phase) in_range = in_range && ph > 0.0 && ph < 2 * std::numbers::pi;
  CHECK(in_range);
  std::mt19937_64 gen(1);
  std::uniform_real_distribution<double> u(0, 1);
  const GrfField g = sample_grf(16, 9);
  bool sum_ok = true, fd_ok = true, rho_ok = true;
  for (int k = 0; k < 20; ++k) {
    const Point x{u(gen), u(gen)};
    long double acc = 0;
    for (size_t j = 0; j < g.amp.size(); ++j)
      acc += static_cast<long double>(g.amp[j]) * sinl(g.fx[j] * x.x + g.fy[j] * x.y + g.phase[j]);
    sum_ok = sum_ok && std::abs(eval_grf(g, x) - static_cast<double>(acc)) <= 1e-12 * std::max(1.0L, fabsl(acc));
    const double h = 1e-6;
    const Point gr = grad_grf(g, x);
    const double gx = (eval_grf(g, {x.x + h, x.y}) - eval_grf(g, {x.x - h, x.y})) / (2 * h);
    const double gy = (eval_grf(g, {x.x, x.y + h}) - eval_grf(g, {x.x, x.y - h})) / (2 * h);
    fd_ok = fd_ok && std::abs(gr.x - gx) < 1e-5 * std::max(1.0, std::abs(gx)) &&
            std::abs(gr.y - gy) < 1e-5 * std::max(1.0, std::abs(gy));
    const double r = eval_rho(g, x), t = std::tanh(eval_grf(g, x));
    const Point dr = grad_rho(g, x);
    rho_ok = rho_ok && r >= 0.1 && r <= 2.1 && std::abs(r - (t + 1.1)) <= 1e-14 * r &&
             std::abs(dr.x - (1 - t * t) * gr.x) <= 1e-12 * std::max(1.0, std::abs(dr.x)) &&
             std::abs(dr.y - (1 - t * t) * gr.y) <= 1e-12 * std::max(1.0, std::abs(dr.y));
  }
  CHECK(sum_ok);
  CHECK(fd_ok);
  CHECK(rho_ok);
  // -div(rho grad phi) = -rho lap(phi) - grad(rho) . grad(phi); conormal flux rho dphi/dn
  ProblemParams pp;
  pp.alpha = 8;
  const ProblemSpec vp = make_problem("varcoef_poisson", pp);
  CHECK(vp.kind == 1 && vp.rho != nullptr && !vp.has_exact());
  Box box{0.0, 0.0, 0.5, 0.5};
  const FeatureLayer L = init_layer(6, box, 3, box.diam() / 2, 12);
  const std::vector<Point> pts{{0.2, 0.3}, {0.4, 0.1}, {0.25, 0.25}};
  const Mat rows = vp.interior_rows(L, pts), fr = vp.flux_rows(L, pts, Point{1, 0});
  const Mat d20 = eval_derivative_matrix(L, pts, 2, 0), d02 = eval_derivative_matrix(L, pts, 0, 2);
  const Mat d10 = eval_derivative_matrix(L, pts, 1, 0), d01 = eval_derivative_matrix(L, pts, 0, 1);
  bool rows_ok = true;
  for (int k = 0; k < 3; ++k) {
    const double r = eval_rho(*vp.rho, pts[k]);
    const Point dr = grad_rho(*vp.rho, pts[k]);
    double mx = 0, err = 0, fmx = 0, ferr = 0;
    for (int j = 0; j < L.M; ++j) {
      const double e = -r * (d20(k, j) + d02(k, j)) - dr.x * d10(k, j) - dr.y * d01(k, j);
      mx = std::max(mx, std::abs(e));
      err = std::max(err, std::abs(rows(k, j) - e));
      fmx = std::max(fmx, std::abs(fr(k, j)));
      ferr = std::max(ferr, std::abs(fr(k, j) - r * d10(k, j)));
    }
    rows_ok = rows_ok && err <= 1e-12 * mx && ferr <= 1e-12 * fmx;
  }
  CHECK(rows_ok);
  const ProblemSpec gp = make_problem("poisson_grf", pp);
  CHECK(gp.kind == 0 && !gp.has_exact() && gp.boundary(Point{0.3, 0.0}) == 0.0);
  const GrfField gf = sample_grf(8, 2);
  CHECK(gp.forcing(Point{0.3, 0.7}) == eval_grf(gf, Point{0.3, 0.7}));
  CHECK_THROWS(make_problem("heat_equation"));
}

void test_biharmonic_blocks() {  // test_assembly.cpp:70-84, test_problems.cpp:104-116
  const ProblemSpec p = make_problem("biharmonic_sinpi");
  CHECK(p.components == 2 && p.boundary_components == 2 && p.kind == 2);
  const Point x{0.3, 0.7};
  const double uu = std::sin(std::numbers::pi * x.x) * std::sin(std::numbers::pi * x.y);
  CHECK(approx(p.exact(x), uu));
  CHECK(std::abs(p.forcing(x) - 4 * std::pow(std::numbers::pi, 4) * uu) <= 1e-12 * std::abs(p.forcing(x)));
  CHECK(std::abs(p.boundary2(x) + 2 * std::numbers::pi * std::numbers::pi * uu) <= 1e-13 * std::abs(p.boundary2(x)));
  const DomainPartition part = partition_domain(2, 5);
  const PointSets ps = classify_points(part);
  const FeatureLayer L = init_layer(12, part.boxes[0], 4.0, part.boxes[0].diam() / 2, 3);
  const LocalBlocks b = assemble_local(p, L, ps, 0);
  CHECK(b.bc == 2 && b.cc == 2);
  CHECK(b.rows() == b.n_int + 2 * b.n_bnd + 2 * b.n_gamma);
  // second trace component = Laplacian trace; second flux component = n . grad(lap)
  const Mat d20 = eval_derivative_matrix(L, ps.interface[0], 2, 0), d02 = eval_derivative_matrix(L, ps.interface[0], 0, 2);
  double err = 0, mx = 0;
  for (int k = 0; k < b.n_gamma; ++k)
    for (int j = 0; j < L.M; ++j) {
      const double e = d20(k, j) + d02(k, j);
      mx = std::max(mx, std::abs(e));
      err = std::max(err, std::abs(b.K(b.trace_row(1, k), j) - e));
    }
  CHECK(err < 1e-13 * mx);
  bool fstack = true;
  for (const Mat& F : b.F_edges) fstack = fstack && F.r % 2 == 0;
  CHECK(fstack);
  // interior rows: the biharmonic operator of a single feature against finite differences
  const std::vector<Point> q{{0.2, 0.3}};
  const Mat rows = p.interior_rows(L, q);
  const double h = 1e-3;
  auto lap = [&](double xx, double yy) {
    const Mat a = eval_derivative_matrix(L, {Point{xx, yy}}, 2, 0), c = eval_derivative_matrix(L, {Point{xx, yy}}, 0, 2);
    return a(0, 0) + c(0, 0);
  };
  const double fd = (lap(q[0].x + h, q[0].y) + lap(q[0].x - h, q[0].y) + lap(q[0].x, q[0].y + h) +
                     lap(q[0].x, q[0].y - h) - 4 * lap(q[0].x, q[0].y)) / (h * h);
  CHECK(std::abs(rows(0, 0) - fd) <= 1e-4 * std::max(1.0, std::abs(fd)));
}

int main() {
  test_features();
  test_biharmonic_blocks();
  test_problems_grf();
  test_geometry();
  test_assembly();
  test_lsfactor();
  test_cg();
  test_solvers();
  std::printf("oracle selftest: %d passed, %d failed\n", g_pass, g_fail);
  return g_fail == 0 ? 0 : 1;
}

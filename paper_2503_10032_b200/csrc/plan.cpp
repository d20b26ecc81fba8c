// Host-side layout for the DDELM-NN device path (see plan.hpp for the reference map).
#include "plan.hpp"

#include <algorithm>
#include <cmath>
#include <map>
#include <random>
#include <thread>
#include <numbers>
#include <random>
#include <stdexcept>

namespace ddg {

namespace {

constexpr double kPi = std::numbers::pi;

int class_mask(int s, int ix, int iy) {
  int m = 0;
  if (ix == 0) m |= 1;
  if (ix == s - 1) m |= 2;
  if (iy == 0) m |= 4;
  if (iy == s - 1) m |= 8;
  return m;
}

/// Point classes of one side class (geometry.cpp:80-142 restricted to one subdomain), with its
/// row-generation tasks for cc trace / flux components and bc boundary components
/// (assembly.cpp:9-46, solvers.cpp:418-438); `bih`: biharmonic row kinds.
ClassPlan build_class(int mask, int n, bool cov, int cc, int bc, bool bih) {
  ClassPlan c;
  c.mask = mask;
  c.cc = cc;
  c.bc = bc;
  const bool outer[4] = {(mask & 1) != 0, (mask & 2) != 0, (mask & 4) != 0, (mask & 8) != 0};
  std::vector<std::pair<int, int>> interior, boundary;
  std::map<std::pair<int, int>, int> gamma_of;
  for (int b = 0; b < n; ++b)
    for (int a = 0; a < n; ++a) {
      const bool on_local = a == 0 || a == n - 1 || b == 0 || b == n - 1;
      const bool on_outer = (a == 0 && outer[0]) || (a == n - 1 && outer[1]) ||
                            (b == 0 && outer[2]) || (b == n - 1 && outer[3]);
      if (!on_local) {
        interior.push_back({a, b});
      } else if (on_outer) {
        boundary.push_back({a, b});
      } else {
        GammaPt g{a, b, false, -1, -1};
        const bool xl = a == 0 || a == n - 1, yl = b == 0 || b == n - 1;
        if (xl && yl) {
          g.is_cross = true;
        } else if (xl) {
          g.side = (a == 0) ? 0 : 1;
          g.t = b;
        } else {
          g.side = (b == 0) ? 2 : 3;
          g.t = a;
        }
        gamma_of[{a, b}] = static_cast<int>(c.gamma.size());
        c.gamma.push_back(g);
      }
    }
  c.n_int = static_cast<int>(interior.size());
  c.n_bnd = static_cast<int>(boundary.size());
  c.n_gpts = static_cast<int>(c.gamma.size());
  c.n_gamma = cc * c.n_gpts;
  c.fixed = c.n_int + bc * c.n_bnd;
  c.m = c.fixed + c.n_gamma;
  for (int side = 0; side < 4; ++side) {
    if (outer[side]) continue;
    LocalEdgeC le;
    le.side = side;
    for (int j = 0; j < n; ++j) {
      const bool vert = side < 2;
      const int a = vert ? (side == 0 ? 0 : n - 1) : j;
      const int b = vert ? j : (side == 2 ? 0 : n - 1);
      auto it = gamma_of.find({a, b});
      if (it == gamma_of.end()) continue;
      le.pts.push_back(it->second);
      le.geom_j.push_back(j);
      if (j == 0) le.first_corner = true;
      if (j == n - 1) le.last_corner = true;
    }
    c.edges.push_back(le);
  }
  // flux rows per edge [component 0 points; component 1 points] (assembly.cpp:34-44); edge-local
  // position of each non-corner interface point (solvers.cpp:408-413)
  std::vector<std::pair<int, int>> where(c.n_gpts, {-1, -1});
  std::vector<int> edge_row0;
  int off = 0;
  for (int e = 0; e < static_cast<int>(c.edges.size()); ++e) {
    edge_row0.push_back(off);
    const LocalEdgeC& le = c.edges[e];
    const int np = static_cast<int>(le.pts.size());
    for (int comp = 0; comp < cc; ++comp)
      for (int pos = 0; pos < np; ++pos) c.flux_rows.push_back({e, pos, comp});
    for (int pos = 0; pos < np; ++pos)
      if (!c.gamma[le.pts[pos]].is_cross) where[le.pts[pos]] = {e, pos};
    off += cc * np;
  }
  c.nF = off;
  for (int q = 0; q < c.n_gpts; ++q) (c.gamma[q].is_cross ? c.corner_idx : c.delta_idx).push_back(q);
  c.nc_pts = static_cast<int>(c.corner_idx.size());
  c.nd_pts = static_cast<int>(c.delta_idx.size());
  c.nc = cc * c.nc_pts;
  c.nd = cc * c.nd_pts;

  // ---- row-generation tasks
  auto task = [](int a, int b, uint8_t kind, uint8_t dst, uint8_t side, uint8_t flags, int row) {
    Task t;
    t.a = static_cast<int16_t>(a);
    t.b = static_cast<int16_t>(b);
    t.kind = kind;
    t.dst = dst;
    t.side = side;
    t.flags = flags;
    t.row = row;
    t.pad = 0;
    return t;
  };
  const uint8_t kTrace[2] = {kValue, kLapP}, kTraceCov[2] = {kValueCov, kLapCov}, kFl[2] = {kFlux, kFlux3};
  int row = 0;
  for (auto [a, b] : interior) c.tasks.push_back(task(a, b, bih ? kBih : kLap, kDstK | kDual, 0, 0, row++));
  for (int comp = 0; comp < bc; ++comp)
    for (auto [a, b] : boundary) c.tasks.push_back(task(a, b, kTrace[comp], kDstK | kDual, 0, 0, row++));
  for (int comp = 0; comp < cc; ++comp)
    for (int q = 0; q < c.n_gpts; ++q) {
      const GammaPt& g = c.gamma[q];
      if (!cov || g.is_cross) {
        c.tasks.push_back(task(g.a, g.b, kTrace[comp], kDstK, 0, 0, row++));
        continue;
      }
      uint8_t flags = 0;
      for (const LocalEdgeC& le : c.edges)
        if (le.side == g.side) flags = (le.first_corner ? 1 : 0) | (le.last_corner ? 2 : 0);
      c.tasks.push_back(task(g.a, g.b, flags ? kTraceCov[comp] : kTrace[comp], kDstK, static_cast<uint8_t>(g.side),
                             flags, row++));
    }
  c.n_tasks_k = row;
  // Kbar tail: corner trace rows (nodal basis), then Delta flux rows, per component
  // (solvers.cpp:418-431)
  int rb = c.fixed;
  for (int comp = 0; comp < cc; ++comp)
    for (int q : c.corner_idx) c.tasks.push_back(task(c.gamma[q].a, c.gamma[q].b, kTrace[comp], kDstKbar, 0, 0, rb++));
  for (int comp = 0; comp < cc; ++comp)
    for (int k = 0; k < c.nd_pts; ++k) {
      const GammaPt& g = c.gamma[c.delta_idx[k]];
      c.tasks.push_back(task(g.a, g.b, kFl[comp], kDstKbar, static_cast<uint8_t>(g.side), 0, rb++));
    }
  c.n_tasks_kbar = rb - c.fixed;
  for (int l = 0; l < c.nF; ++l) {
    const ClassPlan::FluxRow& fr = c.flux_rows[l];
    const GammaPt& g = c.gamma[c.edges[fr.e].pts[fr.pos]];
    c.tasks.push_back(task(g.a, g.b, kFl[fr.comp], kDstF, static_cast<uint8_t>(c.edges[fr.e].side), 0, l));
  }
  c.n_tasks_f = c.nF;
  for (int comp = 0; comp < cc; ++comp)
    for (int k = 0; k < c.nd_pts; ++k) {
      const GammaPt& g = c.gamma[c.delta_idx[k]];
      c.tasks.push_back(task(g.a, g.b, kTrace[comp], kDstCd, 0, 0, comp * c.nd_pts + k));
    }
  c.n_tasks_cd = c.nd;
  return c;
}

}  // namespace

bool problem_known(int problem) { return problem >= 0 && problem <= 5; }

GrfField sample_grf(double alpha, uint64_t seed) {  // problems.cpp:15-39: draw order amp, w0, w1, phase
  if (alpha <= 0) throw std::invalid_argument("sample_grf: alpha must be positive");
  constexpr int kTerms = 256;
  GrfField g;
  g.amp.resize(kTerms);
  g.fx.resize(kTerms);
  g.fy.resize(kTerms);
  g.phase.resize(kTerms);
  std::mt19937_64 gen(seed);
  std::normal_distribution<double> na(0.0, alpha * alpha / 16.0);
  std::normal_distribution<double> nw(0.0, alpha);
  std::uniform_real_distribution<double> ub(0.0, 2.0 * kPi);
  for (int i = 0; i < kTerms; ++i) {
    g.amp[i] = na(gen);
    g.fx[i] = nw(gen);
    g.fy[i] = nw(gen);
    double b;
    do {
      b = ub(gen);
    } while (b <= 0.0);
    g.phase[i] = b;
  }
  return g;
}



double problem_forcing(int problem, double x, double y) {
  switch (problem) {
    case 0: return 2.0 * kPi * kPi * std::sin(kPi * x) * std::sin(kPi * y);
    case 1: return (4.0 * kPi * kPi - 1.0) * std::sin(2 * kPi * x) * std::exp(y);
    default: return 13.0 * kPi * kPi * std::sin(2 * kPi * x) * std::cos(3 * kPi * y) - 2.0 * y;
  }
}

double problem_boundary(int problem, double x, double y) {
  switch (problem) {
    case 0: return std::sin(kPi * x) * std::sin(kPi * y);
    case 1: return std::sin(2 * kPi * x) * std::exp(y);
    default: return std::sin(2 * kPi * x) * std::cos(3 * kPi * y) + x * x * y;
  }
}

Plan build_plan(int problem, int s, int n_grid, int M, double l, uint64_t seed, int flux_variant,
                bool cov, double rank_tol, int debug_flip_flux_row, const ProblemParams& params) {
  if (!problem_known(problem)) throw std::invalid_argument("make_problem: unknown problem id");
  if (s < 1) throw std::invalid_argument("partition_domain: s must be >= 1");
  if (n_grid < 3) throw std::invalid_argument("partition_domain: n_grid must be >= 3");
  if (M < 1) throw std::invalid_argument("init_layer: M must be positive");
  if (!(l > 0)) throw std::invalid_argument("init_layer: l must be positive");
  Plan p;
  p.problem = problem;
  p.params = params;
  p.s = s;
  p.n_grid = n_grid;
  p.M = M;
  p.l = l;
  p.seed = seed;
  p.flux_variant = flux_variant;
  p.cov = cov;
  p.rank_tol = rank_tol;
  p.debug_flip_flux_row = debug_flip_flux_row;
  const int n = n_grid;
  p.N = s * s;
  p.m = n * n;  // rows of K for cc = 1 (every grid point once); the classes raise it for cc = 2
  // biharmonic_sinpi (problems.cpp:167-181): two trace / flux / boundary components
  const int cc = problem == 5 ? 2 : 1, bc = cc;
  p.cc = cc;
  p.ncq = 4 * cc;
  p.n_delta = 2 * s * (s - 1) * (n - 2) * cc;  // geometry.cpp:155-157
  p.n_pi = (s - 1) * (s - 1) * cc;
  p.npf = 2 * p.n_pi;
  p.multiplicity_pi.assign(p.n_pi, 0);

  std::map<int, int> cls_of_mask;
  p.subs.resize(p.N);
  for (int iy = 0; iy < s; ++iy)
    for (int ix = 0; ix < s; ++ix) {
      const int i = iy * s + ix;
      const int mask = class_mask(s, ix, iy);
      auto it = cls_of_mask.find(mask);
      if (it == cls_of_mask.end()) {
        it = cls_of_mask.emplace(mask, static_cast<int>(p.classes.size())).first;
        p.classes.push_back(build_class(mask, n, cov, cc, bc, problem == 5));
      }
      SubPlan& sp = p.subs[i];
      sp.ix = ix;
      sp.iy = iy;
      sp.cls = it->second;
      sp.seed = seed + static_cast<uint64_t>(i);
      sp.gid = i;
    }
  for (const ClassPlan& c : p.classes) {
    // K = [interior; bc x boundary; cc x trace] rows (assembly.cpp:9-32); LsFactor needs K tall
    if (c.m < M) throw std::invalid_argument("LsFactor: matrix must be square or tall");
    p.m = std::max(p.m, c.m);
    p.gmax = std::max(p.gmax, c.n_gamma);
    p.fmax = std::max(p.fmax, c.nF);
    p.dmax = std::max(p.dmax, c.nd);
    p.tmax = std::max(p.tmax, static_cast<int>(c.tasks.size()));
  }
  p.gmax = (std::max(p.gmax, 1) + 1) / 2 * 2;  // even: 16-byte aligned per-subdomain Zc blocks
  // flux / Cdelta row strides are even: 16-byte rows for the CG kernel's bulk copies
  p.fmax = (std::max(p.fmax, 1) + 1) / 2 * 2;
  p.dmax = (std::max(p.dmax, 1) + 1) / 2 * 2;

  // ---- global numbering per subdomain (geometry.cpp:148-179, assembly.cpp:89-133)
  auto edge_id = [s](int ix, int iy, int side) {
    switch (side) {
      case 0: return (ix - 1) * s + iy;
      case 1: return ix * s + iy;
      case 2: return s * (s - 1) + (iy - 1) * s + ix;
      default: return s * (s - 1) + iy * s + ix;
    }
  };
  auto cross_of = [&](int ix, int iy, int a, int b) {
    const int gx = ix * (n - 1) + a, gy = iy * (n - 1) + b;
    return (gy / (n - 1) - 1) * (s - 1) + (gx / (n - 1) - 1);
  };
  p.own_gamma.assign(2 * static_cast<size_t>(p.n_delta), -1);
  p.own_flux.assign(2 * static_cast<size_t>(p.n_delta), -1);
  p.own_nd.assign(2 * static_cast<size_t>(p.n_delta), -1);
  auto own = [](std::vector<int>& v, int g, int val) {
    if (v[2 * g] < 0) v[2 * g] = val;
    else v[2 * g + 1] = val;
  };
  // global indices (geometry.cpp:148-179): Delta (edge, comp, t) -> (edge cc + comp)(n-2) + t-1,
  // Pi (cross, comp) -> cross cc + comp; trace rows q = comp * points + point
  auto delta_of = [&](int ix, int iy, int side, int comp, int t) {
    return (edge_id(ix, iy, side) * cc + comp) * (n - 2) + (t - 1);
  };
  for (int i = 0; i < p.N; ++i) {
    SubPlan& sp = p.subs[i];
    const ClassPlan& c = p.classes[sp.cls];
    sp.gamma_delta.assign(c.n_gamma, -1);
    sp.gamma_pi.assign(c.n_gamma, -1);
    for (int q = 0; q < c.n_gamma; ++q) {
      const int comp = q / c.n_gpts;
      const GammaPt& g = c.gamma[q % c.n_gpts];
      if (g.is_cross) {
        const int cid = cross_of(sp.ix, sp.iy, g.a, g.b) * cc + comp;
        sp.gamma_pi[q] = cid;
        p.multiplicity_pi[cid] += 1;
      } else {
        const int d = delta_of(sp.ix, sp.iy, g.side, comp, g.t);
        sp.gamma_delta[q] = d;
        own(p.own_gamma, d, i * p.gmax + q);
      }
    }
    // flux scatter, in the reference's order (edges L,R,B,T; points by arclength)
    std::map<int, int> cross_slot;
    sp.fluxrow_delta.assign(c.nF, -1);
    int off = 0;
    for (const LocalEdgeC& le : c.edges) {
      const int np = static_cast<int>(le.pts.size());
      const int dir = le.side < 2 ? 0 : 1;
      for (int comp = 0; comp < cc; ++comp)
        for (int q = 0; q < np; ++q) {
          const int j = le.geom_j[q];
          const int lrow = off + comp * np + q;
          if (j > 0 && j < n - 1) {
            const int d = delta_of(sp.ix, sp.iy, le.side, comp, j);
            sp.fluxrow_delta[lrow] = d;
            own(p.own_flux, d, i * p.fmax + lrow);
            continue;
          }
          const GammaPt& g = c.gamma[le.pts[q]];
          const int r = (cross_of(sp.ix, sp.iy, g.a, g.b) * cc + comp) * 2 + dir;  // assembly.cpp:116
          auto it = cross_slot.find(r);
          if (it == cross_slot.end()) {
            it = cross_slot.emplace(r, static_cast<int>(sp.cross_rows.size())).first;
            sp.cross_rows.push_back(CrossRow{r, {}});
          }
          CrossRow& cr = sp.cross_rows[it->second];
          if (flux_variant == 0) {
            cr.e.push_back({lrow, 1.0});
          } else {
            const int opposing = (j == 0) ? n - 1 : 0;
            const double w = 1.0 / (n - 1);
            for (int q2 = 0; q2 < np; ++q2)
              if (le.geom_j[q2] != opposing) cr.e.push_back({off + comp * np + q2, w});
          }
        }
      off += cc * np;
    }
    // the reference groups cross entries with std::map<grow,...> (solvers.cpp:302-304):
    // rows in increasing global order, entries in scatter order
    std::sort(sp.cross_rows.begin(), sp.cross_rows.end(),
              [](const CrossRow& x, const CrossRow& y) { return x.r < y.r; });
    p.crmax = std::max(p.crmax, static_cast<int>(sp.cross_rows.size()));
    sp.ndelta_map.assign(c.nd, -1);
    for (int k = 0; k < c.nd; ++k) {  // Neumann Delta rows comp * points + k (solvers.cpp:439-444)
      const GammaPt& g = c.gamma[c.delta_idx[k % c.nd_pts]];
      const int d = delta_of(sp.ix, sp.iy, g.side, k / c.nd_pts, g.t);
      sp.ndelta_map[k] = d;
      own(p.own_nd, d, i * p.dmax + k);
    }
  }
  p.crmax = std::max(p.crmax, 1);

  // ---- right-hand sides f (assembly.cpp:21-33): forcing, boundary data, zero on traces;
  //      varcoef_poisson: the coefficient field at every row point (problems.cpp:74-87, 117-121)
  const int S = s * (n - 1);
  // GRF problems: the field is sampled here (1024 draws in the reference's order); its values at
  // the row points are evaluated on the device (Workspace::upload_plan -> grf_eval_kernel)
  if (problem == 3) p.grf = sample_grf(params.alpha, params.forcing_seed);
  if (problem == 4) {
    p.grf = sample_grf(params.alpha, params.rho_seed);
    p.coef.assign(static_cast<size_t>(p.N) * p.tmax * 3, 0.0);
  }
  p.f.assign(static_cast<size_t>(p.N) * p.m, 0.0);
  auto fill = [&](int i0, int i1) {
    for (int i = i0; i < i1; ++i) {
      const SubPlan& sp = p.subs[i];
      const ClassPlan& c = p.classes[sp.cls];
      for (int t = 0; t < static_cast<int>(c.tasks.size()); ++t) {
        const Task& tk = c.tasks[t];
        const double x = static_cast<double>(sp.ix * (n - 1) + tk.a) / S;
        const double y = static_cast<double>(sp.iy * (n - 1) + tk.b) / S;
        if (t >= c.n_tasks_k || tk.row >= c.fixed) continue;
        double v;
        if (problem <= 2) v = tk.kind == kLap ? problem_forcing(problem, x, y) : problem_boundary(problem, x, y);
        else if (problem == 3) v = 0.0;  // interior rows: the GRF forcing, evaluated on the device
        else if (problem == 4) v = tk.kind == kLap ? 1.0 : 0.0;
        else  // biharmonic_sinpi: lap^2 u = 4 pi^4 sin sin, u = sin sin, lap u = -2 pi^2 sin sin
          v = tk.kind == kBih   ? 4.0 * kPi * kPi * kPi * kPi * std::sin(kPi * x) * std::sin(kPi * y)
              : tk.kind == kLapP ? -2.0 * kPi * kPi * std::sin(kPi * x) * std::sin(kPi * y)
                                 : std::sin(kPi * x) * std::sin(kPi * y);
        p.f[static_cast<size_t>(i) * p.m + tk.row] = v;
      }
    }
  };
  fill(0, p.N);
  return p;
}

void shard_range(int N, int rank, int world, int* lo, int* hi) {
  *lo = static_cast<int>(static_cast<long long>(N) * rank / world);
  *hi = static_cast<int>(static_cast<long long>(N) * (rank + 1) / world);
}

Plan shard_plan(const Plan& g, int lo, int hi) {
  if (lo < 0 || hi > g.N || lo >= hi) throw std::invalid_argument("shard_plan: empty or out-of-range strip");
  // global owner-slot destinations, built on the global plan
  const int N = g.N;
  std::vector<int> gdst(static_cast<size_t>(N) * g.gmax, -1), fdst(static_cast<size_t>(N) * g.fmax, -1),
      ndst(static_cast<size_t>(N) * g.dmax, -1), cdst(static_cast<size_t>(N) * g.ncq, -1),
      xdst(static_cast<size_t>(N) * g.crmax, -1);
  for (int d = 0; d < g.n_delta; ++d)
    for (int s = 0; s < 2; ++s) {
      if (g.own_gamma[2 * d + s] >= 0) gdst[g.own_gamma[2 * d + s]] = 2 * d + s;
      if (g.own_flux[2 * d + s] >= 0) fdst[g.own_flux[2 * d + s]] = 2 * d + s;
      if (g.own_nd[2 * d + s] >= 0) ndst[g.own_nd[2 * d + s]] = 2 * d + s;
    }
  // corner / cross-row owners in subdomain order (the order the single-device sums use)
  std::vector<int> pi_n(std::max(g.n_pi, 1), 0), row_n(std::max(g.npf, 1), 0);
  for (int i = 0; i < N; ++i) {
    const SubPlan& sp = g.subs[i];
    int slot = 0;
    for (size_t q = 0; q < sp.gamma_pi.size(); ++q)
      if (sp.gamma_pi[q] >= 0) {
        const int gp = sp.gamma_pi[q];
        if (pi_n[gp] >= 4) throw std::logic_error("shard_plan: corner owner overflow");
        cdst[static_cast<size_t>(i) * g.ncq + slot++] = gp * 4 + pi_n[gp]++;
      }
    for (size_t rho = 0; rho < sp.cross_rows.size(); ++rho) {
      const int r = sp.cross_rows[rho].r;
      if (row_n[r] >= 4) throw std::logic_error("shard_plan: cross-row owner overflow");
      xdst[static_cast<size_t>(i) * g.crmax + rho] = r * 4 + row_n[r]++;
    }
  }
  // global coarse owner tables (cross rows / Pi indices -> global (subdomain, slot)) and the Pi
  // index of every corner slot
  std::vector<int> rown(static_cast<size_t>(std::max(g.npf, 1)) * 4, -1), pown(static_cast<size_t>(std::max(g.n_pi, 1)) * 4, -1);
  std::vector<int> cpi(static_cast<size_t>(N) * g.ncq, -1);
  auto push_owner = [](std::vector<int>& v, int row, int val) {
    for (int q = 0; q < 4; ++q)
      if (v[static_cast<size_t>(row) * 4 + q] < 0) {
        v[static_cast<size_t>(row) * 4 + q] = val;
        return;
      }
    throw std::logic_error("owner table overflow");
  };
  for (int i = 0; i < N; ++i) {
    const SubPlan& sp = g.subs[i];
    int slot = 0;
    for (size_t q = 0; q < sp.gamma_pi.size(); ++q)
      if (sp.gamma_pi[q] >= 0 && slot < g.ncq) {
        push_owner(pown, sp.gamma_pi[q], i * g.ncq + slot);
        cpi[static_cast<size_t>(i) * g.ncq + slot++] = sp.gamma_pi[q];
      }
    for (size_t rho = 0; rho < sp.cross_rows.size(); ++rho)
      push_owner(rown, sp.cross_rows[rho].r, i * g.crmax + static_cast<int>(rho));
  }
  Plan p = g;
  p.row_owner_g = std::move(rown);
  p.pi_owner_g = std::move(pown);
  p.cpi_g = std::move(cpi);
  p.N = hi - lo;
  p.sub_lo = lo;
  p.N_global = g.N;
  p.subs.assign(g.subs.begin() + lo, g.subs.begin() + hi);
  p.f.assign(g.f.begin() + static_cast<size_t>(lo) * g.m, g.f.begin() + static_cast<size_t>(hi) * g.m);
  if (!g.coef.empty())
    p.coef.assign(g.coef.begin() + static_cast<size_t>(lo) * g.tmax * 3, g.coef.begin() + static_cast<size_t>(hi) * g.tmax * 3);
  auto slice = [&](const std::vector<int>& v, int w) {
    return std::vector<int>(v.begin() + static_cast<size_t>(lo) * w, v.begin() + static_cast<size_t>(hi) * w);
  };
  p.gamma_dst = slice(gdst, g.gmax);
  p.flux_dst = slice(fdst, g.fmax);
  p.nd_dst = slice(ndst, g.dmax);
  p.corner_dst = slice(cdst, g.ncq);
  p.cross_dst = slice(xdst, g.crmax);
  // owner tables restricted to this strip (local subdomain numbering; -1 = owned by another rank)
  auto remap = [&](std::vector<int>& own, int w) {
    for (int& v : own)
      if (v >= 0) {
        const int i = v / w, pos = v % w;
        v = (i >= lo && i < hi) ? (i - lo) * w + pos : -1;
      }
  };
  remap(p.own_gamma, g.gmax);
  remap(p.own_flux, g.fmax);
  remap(p.own_nd, g.dmax);
  return p;
}

XPlan build_exchange_plan(const Plan& g, int rank, int world) {
  if (!g.gamma_dst.empty() || g.sub_lo != 0) throw std::logic_error("build_exchange_plan: needs the global plan (build_plan)");
  if (world < 1 || rank < 0 || rank >= world) throw std::invalid_argument("build_exchange_plan: bad rank / world");
  const int N = g.N;
  XPlan xp;
  xp.rank = rank;
  xp.world = world;
  std::vector<int> rank_of(N);
  for (int r = 0; r < world; ++r) {
    int lo, hi;
    shard_range(N, r, world, &lo, &hi);
    for (int i = lo; i < hi; ++i) rank_of[i] = r;
  }
  const int nd = g.n_delta;
  // writers: Delta tables by owner pair (own_* hold i * width + pos), corner / cross slots in
  // subdomain order (the numbering of shard_plan's corner_dst / cross_dst)
  auto delta_writers = [&](const std::vector<int>& own, int w) {
    std::vector<int> wr(2 * static_cast<size_t>(nd), -1);
    for (size_t k = 0; k < wr.size(); ++k)
      if (own[k] >= 0) wr[k] = rank_of[own[k] / w];
    return wr;
  };
  const std::vector<int> w_o = delta_writers(g.own_gamma, g.gmax), w_x = delta_writers(g.own_flux, g.fmax),
                         w_nd = delta_writers(g.own_nd, g.dmax);
  std::vector<int> w_pi(4 * static_cast<size_t>(std::max(g.n_pi, 1)), -1), w_cr(4 * static_cast<size_t>(std::max(g.npf, 1)), -1);
  {
    std::vector<int> pi_n(std::max(g.n_pi, 1), 0), row_n(std::max(g.npf, 1), 0);
    for (int i = 0; i < N; ++i) {
      const SubPlan& sp = g.subs[i];
      for (size_t q = 0; q < sp.gamma_pi.size(); ++q)
        if (sp.gamma_pi[q] >= 0) {
          const int gp = sp.gamma_pi[q];
          w_pi[static_cast<size_t>(gp) * 4 + pi_n[gp]++] = rank_of[i];
        }
      for (const CrossRow& cr : sp.cross_rows) w_cr[static_cast<size_t>(cr.r) * 4 + row_n[cr.r]++] = rank_of[i];
    }
  }
  // readers of a Delta index: the ranks of every subdomain touching it (trace, flux or Neumann row)
  std::vector<unsigned long long> dread(std::max(nd, 1), 0ull);
  if (world > 64) throw std::invalid_argument("build_exchange_plan: at most 64 ranks");
  for (int i = 0; i < N; ++i) {
    const SubPlan& sp = g.subs[i];
    const unsigned long long bit = 1ull << rank_of[i];
    for (int d : sp.gamma_delta)
      if (d >= 0) dread[d] |= bit;
    for (int d : sp.fluxrow_delta)
      if (d >= 0) dread[d] |= bit;
    for (int d : sp.ndelta_map)
      if (d >= 0) dread[d] |= bit;
  }
  // (table, slot count per part, writer rank of a slot, whether rank q reads the slot)
  struct Tab {
    int id;
    const std::vector<int>* writer;  // nullptr: pap (slot i written by rank_of[i])
    bool delta;                      // readers = the touching ranks; else every rank
  };
  auto tabs_of = [&](int one, int pt) -> std::vector<Tab> {
    switch (pt) {
      case kXOp1: return one ? std::vector<Tab>{} : std::vector<Tab>{{kTabT, &w_pi, false}, {kTabPsi, &w_cr, false}};
      case kXOp2: return one ? std::vector<Tab>{{kTabX, &w_x, true}, {kTabXc, &w_cr, false}} : std::vector<Tab>{{kTabX, &w_x, true}};
      case kXNn1: return one ? std::vector<Tab>{} : std::vector<Tab>{{kTabTr, &w_nd, true}};
      case kXNn2: return one ? std::vector<Tab>{} : std::vector<Tab>{{kTabZz, &w_nd, true}};
      case kXOp3: return one ? std::vector<Tab>{} : std::vector<Tab>{{kTabT3, &w_pi, false}};
      default:
        return one ? std::vector<Tab>{{kTabO, &w_o, false}, {kTabOpi, &w_pi, false}, {kTabPap, nullptr, false}}
                   : std::vector<Tab>{{kTabO, &w_o, false}, {kTabPap, nullptr, false}};
    }
  };
  // the O table feeds the replicated CG update (every rank reads all of it)
  auto list = [&](int one, int pt, int src, int dst, std::vector<XEntry>& out) {
    for (const Tab& t : tabs_of(one, pt)) {
      const int n = t.writer ? static_cast<int>(t.writer->size()) : N;
      for (int k = 0; k < n; ++k) {
        const int w = t.writer ? (*t.writer)[k] : rank_of[k];
        if (w != src) continue;
        const bool reads = t.delta ? ((dread[k / 2] >> dst) & 1ull) != 0 : true;
        if (reads) out.push_back(XEntry{t.id, k});
      }
    }
  };
  size_t mx = 8;
  for (int one = 0; one < 2; ++one)
    for (int pt = 0; pt < kXPoints; ++pt) {
      XList& L = xp.pt[one][pt];
      L.soff.assign(world, 0);
      L.scnt.assign(world, 0);
      L.roff.assign(world, 0);
      L.rcnt.assign(world, 0);
      for (int q = 0; q < world; ++q) {
        if (q == rank) continue;
        L.soff[q] = static_cast<int>(L.send.size());
        list(one, pt, rank, q, L.send);
        L.scnt[q] = static_cast<int>(L.send.size()) - L.soff[q];
        L.roff[q] = static_cast<int>(L.recv.size());
        list(one, pt, q, rank, L.recv);
        L.rcnt[q] = static_cast<int>(L.recv.size()) - L.roff[q];
        mx = std::max(mx, static_cast<size_t>(std::max(L.scnt[q], L.rcnt[q])));
      }
    }
  // the setup all-reduce of the coarse inputs (workspace.cu build_coarse) and the metric sums
  const size_t coarse = static_cast<size_t>(N) * g.crmax * (1 + g.ncq) + static_cast<size_t>(N) * g.ncq * g.ncq;
  xp.max_msg = std::max(mx, coarse + 1) + 64;  // + the padding entry of the coarse buffer, slack
  return xp;
}

void init_layer(const Plan& p, int i, double* w0, double* w1, double* b) {
  const SubPlan& sp = p.subs[i];
  const double h = 1.0 / p.s;
  const double x0 = sp.ix * h, y0 = sp.iy * h, x1 = (sp.ix + 1) * h, y1 = (sp.iy + 1) * h;
  const double r = std::hypot(x1 - x0, y1 - y0) / 2.0;
  std::mt19937_64 gen(p.seed + static_cast<uint64_t>(sp.gid));
  std::uniform_real_distribution<double> uw(-p.l, p.l);
  std::uniform_real_distribution<double> ux(x0 - r, x1 + r);
  std::uniform_real_distribution<double> uy(y0 - r, y1 + r);
  for (int j = 0; j < p.M; ++j) {
    const double a0 = uw(gen), a1 = uw(gen);
    const double xi0 = ux(gen), xi1 = uy(gen);
    w0[j] = a0;
    w1[j] = a1;
    b[j] = -(a0 * xi0 + a1 * xi1);
  }
}

}  // namespace ddg

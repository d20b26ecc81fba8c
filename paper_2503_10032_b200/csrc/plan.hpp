// Host-side layout of the DDELM-NN hot path: decomposition geometry, point classes,
// interface numbering, flux scatter and the index tables the device kernels read.
//
// Semantics follow the reference's host code (layout source, not a kernel):
//   partition / classification   proj/src/geometry.cpp:20-146
//   interface numbering          proj/src/geometry.cpp:148-179
//   local block row order        proj/src/assembly.cpp:9-46 (interior, boundary, trace)
//   change of variables T^{-1}   proj/src/assembly.cpp:59-87 (T = I + E, E^2 = 0 => I - E)
//   flux scatter (A / A_m)       proj/src/assembly.cpp:89-133
//   Neumann rows of Kbar         proj/src/solvers.cpp:401-444
//
// B200 layout decision: every subdomain's point set is determined by which of its four sides
// lie on the outer boundary, so row-generation "tasks" are stored once per side class (at most
// 9 classes) and the feature kernel derives coordinates from (ix, iy, a, b) exactly as the
// host would. Only the small global index maps are per subdomain.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace ddg {

/// kLap: -(D20 + D02) (Poisson interior; variable coefficient with per-row rho); kValue: D00;
/// kValueCov: D00 with the change of variables; kFlux: n . grad; biharmonic (cc = bc = 2):
/// kBih: D40 + 2 D22 + D04, kLapP: D20 + D02 (second trace / boundary component), kLapCov: kLapP
/// with the change of variables, kFlux3: n . grad(lap) (second flux component)
enum RowKind : uint8_t { kLap = 0, kValue = 1, kValueCov = 2, kFlux = 3, kBih = 4, kLapP = 5, kLapCov = 6, kFlux3 = 7 };
enum RowDst : uint8_t { kDstK = 0, kDstKbar = 1, kDstF = 2, kDstCd = 3, kDual = 0x10 };

/// One matrix row to generate (16 bytes). Coordinates come from the local grid (a, b).
struct Task {
  int16_t a, b;
  uint8_t kind;   // RowKind
  uint8_t dst;    // RowDst, optionally | kDual (K row also written into Kbar)
  uint8_t side;   // normal side for kFlux (0 L, 1 R, 2 B, 3 T); edge side for kValueCov
  uint8_t flags;  // kValueCov: bit0 first corner present, bit1 last corner present
  int32_t row;    // destination row
  int32_t pad;
};
static_assert(sizeof(Task) == 16, "Task must stay 16 bytes");

struct GammaPt {
  int a, b;
  bool is_cross;
  int side;  // side of the (single) local edge of a non-corner point
  int t;     // arclength index 1..n-2 along its edge (non-corner)
};

struct LocalEdgeC {
  int side;                 // 0 L, 1 R, 2 B, 3 T
  std::vector<int> pts;     // local gamma indices, arclength order
  std::vector<int> geom_j;  // 0..n-1 along the edge
  bool first_corner = false, last_corner = false;
};

/// Rows and points of one side class (mask bit k set = side k lies on the outer boundary).
/// Row counts carry the components: n_gamma = cc x interface points (the trace rows, component
/// blocks), nc / nd = cc x corner / Delta points (Neumann rows), nF = cc x edge points (flux rows,
/// per edge [component 0; component 1]), fixed = n_int + bc x n_bnd.
struct ClassPlan {
  int mask = 0;
  int n_int = 0, n_bnd = 0, n_gamma = 0, m = 0, fixed = 0, nc = 0, nd = 0, nF = 0;
  int cc = 1, bc = 1, n_gpts = 0, nc_pts = 0, nd_pts = 0;  // components and point counts
  std::vector<GammaPt> gamma;                        // interface points (n_gpts)
  std::vector<LocalEdgeC> edges;
  std::vector<int> corner_idx, delta_idx;            // interface point indices
  struct FluxRow {
    int e, pos, comp;
  };
  std::vector<FluxRow> flux_rows;                    // per concatenated F row
  std::vector<Task> tasks;                           // K (m), Kbar tail (m-fixed), F (nF), Cd (nd)
  int n_tasks_k = 0, n_tasks_kbar = 0, n_tasks_f = 0, n_tasks_cd = 0;
};

struct CrossRow {
  int r;                                   // cross-flux row index (global row - n_delta)
  std::vector<std::pair<int, double>> e;   // (local F row, weight)
};

struct SubPlan {
  int ix = 0, iy = 0, cls = 0;
  std::vector<int> gamma_delta;  // per gamma point: Delta index, or -1 (corner)
  std::vector<int> gamma_pi;     // per gamma point: Pi index (0..n_pi-1), or -1
  std::vector<int> fluxrow_delta;  // per F row: Delta index of a weight-1 Delta scatter, or -1
  std::vector<CrossRow> cross_rows;
  std::vector<int> ndelta_map;   // per Neumann Delta row k: Delta index
  uint64_t seed = 0;
  int gid = 0;                   // global subdomain index (seed + gid, solvers.cpp:136)
};

/// Problem parameters of the GRF problems (problems.hpp:64-68).
struct ProblemParams {
  double alpha = 32.0;
  uint64_t forcing_seed = 2, rho_seed = 3;
};

/// Gaussian random field sum_i amp_i sin(w_i . x + phase_i), 256 terms (problems.cpp:15-58),
/// drawn on the host with the reference's generator and draw order.
struct GrfField {
  std::vector<double> amp, fx, fy, phase;
};
GrfField sample_grf(double alpha, uint64_t seed);

struct Plan {
  int problem = 0, s = 1, n_grid = 3, M = 1;
  int cc = 1;   // trace / flux components per interface point (2: biharmonic)
  int ncq = 4;  // corner (Pi) rows per subdomain: 4 corners x cc
  ProblemParams params;
  double l = 1;
  uint64_t seed = 1;
  int flux_variant = 1;  // 0 pointwise, 1 mean_edge
  bool cov = true;
  double rank_tol = 1e-10;
  int debug_flip_flux_row = -1;

  int N = 1, m = 0, n_delta = 0, n_pi = 0, npf = 0;
  int gmax = 0, fmax = 0, dmax = 0, tmax = 0, crmax = 0;  // per-subdomain maxima
  std::vector<ClassPlan> classes;
  std::vector<SubPlan> subs;
  std::vector<int> multiplicity_pi;  // per Pi index

  // owners of each Delta index: (subdomain, local position) pairs in subdomain order
  std::vector<int> own_gamma;  // 2 * n_delta entries: i * gmax + q
  std::vector<int> own_flux;   // 2 * n_delta: i * fmax + l
  std::vector<int> own_nd;     // 2 * n_delta: i * dmax + k

  std::vector<double> f;  // N x m right-hand sides (problem data, assembly.cpp:21-33)
  // varcoef_poisson: per subdomain and class task, (rho, d rho/dx, d rho/dy) at the task's point
  // (interior rows: -rho lap - grad rho . grad; flux rows: x rho); empty for the other problems
  std::vector<double> coef;  // N x tmax x 3
  // poisson_grf / varcoef_poisson: the 256-term field drawn on the host in the reference's order;
  // its values at the row points (f, coef above, left zero here) are evaluated on the device
  // (k_features.cu grf_eval_kernel)
  GrfField grf;

  // ---- sharding: this plan holds subdomains [sub_lo, sub_lo + N) of N_global (one rank's
  // contiguous strip); the interface numbering (n_delta, n_pi, npf) stays global
  int sub_lo = 0, N_global = 1;
  // owner-slot destinations (global slot numbering, so that every slot has exactly one writer
  // across all ranks): gamma/flux/nd -> 2 g + s, corner -> gp * 4 + slot, cross -> rr * 4 + slot
  std::vector<int> gamma_dst, flux_dst, nd_dst, corner_dst, cross_dst;
  // coarse assembly over the GLOBAL subdomain numbering (so that a sharded build sums exactly the
  // single-device terms in the single-device order): owners of every cross-flux row
  // (ig * crmax + rho) and of every Pi index (ig * ncq + corner slot), subdomain order, -1 pad;
  // cpi_g: Pi index of corner slot q of subdomain ig (-1 pad)
  std::vector<int> row_owner_g, pi_owner_g, cpi_g;
};

/// Exchange points of one interface iteration (after the producing phase, k_cg.cu) and the
/// owner-slot tables each one carries (CgArgs *tab).
enum XPoint { kXOp1 = 0, kXOp2, kXNn1, kXNn2, kXOp3, kXOp4, kXPoints };
enum XTable { kTabT = 0, kTabPsi, kTabT3, kTabO, kTabX, kTabTr, kTabZz, kTabXc, kTabOpi, kTabPap, kTabCount };
/// one slot of one table (tables with P row parts: idx within a part; the exporter sends the
/// P-part sum, the importer stores it in part 0)
struct XEntry {
  int table, idx;
};
/// Per-peer segments of one exchange point: send[soff[q] .. +scnt[q]) to rank q, recv likewise.
struct XList {
  std::vector<int> soff, scnt, roff, rcnt;
  std::vector<XEntry> send, recv;
};
/// The sharded path's whole communication plan: for each method family (0 coarse methods,
/// 1 one-level) and exchange point, which slots this rank exports to / imports from each peer.
/// Built identically on every rank from the global plan, so the pairwise lists agree.
struct XPlan {
  int rank = 0, world = 1;
  XList pt[2][kXPoints];
  size_t max_msg = 0;  // largest per-peer segment or all-reduce (doubles): host mailbox size
};

/// The strip of subdomains [lo, hi) of a global plan, with global owner slots (see Plan).
Plan shard_plan(const Plan& g, int lo, int hi);
/// The communication plan of `rank` (global plan g, contiguous strips of shard_range).
XPlan build_exchange_plan(const Plan& g, int rank, int world);
/// Contiguous balanced partition of N subdomains over `world` ranks: [lo, hi) of `rank`.
void shard_range(int N, int rank, int world, int* lo, int* hi);

/// Builds the plan; throws std::invalid_argument like the reference (geometry.cpp:21-22).
Plan build_plan(int problem, int s, int n_grid, int M, double l, uint64_t seed, int flux_variant,
                bool cov, double rank_tol, int debug_flip_flux_row, const ProblemParams& params = {});

/// Seeded feature layer of subdomain i (features.cpp:9-35 via solvers.cpp:134-137):
/// w0, w1, b (M each) from std::mt19937_64(seed + i).
void init_layer(const Plan& p, int i, double* w0, double* w1, double* b);

/// Problem data (problems.cpp:135-156 + C4's added problem).
double problem_forcing(int problem, double x, double y);  // problems 0-2 (manufactured)
double problem_boundary(int problem, double x, double y);
bool problem_known(int problem);

}  // namespace ddg

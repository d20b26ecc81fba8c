// Device workspace of the DDELM-NN hot path (see workspace.cu).
#pragma once

#include <cuda_runtime.h>

#include <stdexcept>
#include <string>
#include <vector>

#include <memory>

#include "comm.hpp"
#include "kernels.hpp"
#include "plan.hpp"

namespace ddg {

struct CapacityError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

/// Device arena for the small, hot buffers of the interface iteration (index tables, coarse
/// rows, CG vectors): one contiguous range that an L2 access-policy window marks persisting, so
/// the ~0.4 GB of coefficient blocks streamed per CG iteration cannot evict them.
struct Arena {
  ~Arena() {
    if (base) cudaFree(base);
  }
  char* base = nullptr;
  size_t cap = 0, used = 0;
  void* take(size_t bytes) {
    const size_t off = (used + 255) / 256 * 256;
    if (base == nullptr || off + bytes > cap) return nullptr;
    used = off + bytes;
    return base + off;
  }
};
/// Arena that DevBuf::alloc draws small requests from while set (Workspace scopes it).
extern thread_local Arena* g_arena;
constexpr size_t kArenaSmallBytes = size_t(8) << 20;

template <typename T>
struct DevBuf {
  T* ptr = nullptr;
  size_t count = 0;
  bool in_arena = false;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { free(); }
  void alloc(size_t n);
  void free();
  void upload(const std::vector<T>& v, cudaStream_t st);
};

/// Optional per-kernel-family CUDA-event timers (bench.py's live roofline numbers).
struct KernelStat {
  double ms = 0, flops = 0, bytes = 0;
  long long launches = 0;
};

/// dense_oracle_solve's outputs (solvers.hpp DenseOracle): reduced operator / rhs (dim = n_mu for
/// the one-level method, n_delta for the coarse ones; column-major), mu_full (n_mu), coefficients.
struct DenseOracleOut {
  int dim = 0;
  std::vector<double> reduced_op, reduced_rhs, mu_full, coeffs;
};

struct SolveResult {
  int iterations = 0;
  bool converged = false, negative_curvature = false;
  std::vector<double> phase_ms;  // features, qr, cod, coarse, neumann, rhs, cg, reconstruct
  double host_ms = 0;
};

class Workspace {
 public:
  /// p: the (possibly sharded, see shard_plan) plan of this device; ex: the cross-GPU exchange
  /// (nullptr: single device)
  Workspace(const Plan& p, int device, std::unique_ptr<Exchange> ex = nullptr, XPlan xp = {});
  ~Workspace();
  Workspace(const Workspace&) = delete;
  Workspace& operator=(const Workspace&) = delete;

  void build();
  void build_blocks();
  void build_coarse();
  void build_neumann();
  SolveResult solve(int method, double theta, double tol, int max_iter);
  void reseed(uint64_t seed);
  int cg_compact = 0;  // DDELM_CG_BLOCKS_* (CG operator representation)
  bool compact_built_ = false;
  /// drop every built layer but keep the uploaded feature layers (device-resident inputs)
  void invalidate() { built_ = blocks_built_ = coarse_built_ = neumann_built_ = false; }
  void apply_operator(double theta, const double* v, double* out);
  void apply_reduced(const double* v, double* out);
  /// the Neumann map P (transpose = 0) or its adjoint P^T (solvers.cpp:450-474) on n_delta doubles
  void apply_neumann(int transpose, const double* v, double* out);
  void set_profiling(bool on) { profiling_ = on; }
  bool kernel_stat(const std::string& name, KernelStat* out) const;
  double device_span_ms() const { return device_span_ms_; }
  const char* cg_driver() const { return cg_driver_; }
  const char* exchange_kind() const { return ex_ ? ex_->kind() : "none"; }
  int world() const { return ex_ ? ex_->world() : 1; }

  /// Field of the last solve on the n x n grid (sample_field, metrics.cpp:18-57): samples to the
  /// host buffers (each nullable, n*n), and sums[4] of the trapezoid error terms against the
  /// exact solution (ref = nullptr) or the ELM field of ref (N x M, same layers). Sharded: the
  /// strip's points only; the sums are all-reduced over the ranks.
  void field(int n, const double* ref, double* u, double* gx, double* gy, double* sums);
  void get_mu(double* mu);
  void get_coeffs(double* c);
  int get_residuals(double* h, int cap);
  void get_ranks(int* rk, int* rkb, double* ratio);
  void get_local(int i, int which, double* K);
  /// dense brute-force oracle on the device (solvers.cpp:609-709, k_dense.cu); regenerates the
  /// local matrices, so the next solve rebuilds the factorisations
  void dense_oracle(int method, double theta, DenseOracleOut& o);
  const double* phase_ms() const { return phase_ms_; }
  long long launches() const { return solve_launches_; }
  double host_build_ms() const { return host_build_ms_; }
  int rmax() const { return rmax_; }
  cudaStream_t stream() const { return st_; }

  Plan plan;
  std::vector<double> h_w0, h_w1, h_b;
  std::vector<int> h_rank;

 private:
  void upload_plan();
  void init_layers();
  FeatureArgs feature_args();
  CodArgs cod_args();
  BlockArgs block_args();
  CgArgs cg_args(double theta, double tol, int max_iter, bool one_level = false);
  void pack_blocks(const BlockArgs& b);
  bool sharded() const { return ex_ && ex_->world() > 1; }
  /// phase-by-phase launches with owner-slot all-reduces (sharded path; DDELM_CG_MODE=phased
  /// selects it on one device too)
  void run_phases(const CgArgs& a, int mode, const double* vin, double* vout);
  /// runs the CG loop; returns the number of this library's kernels launched
  long long run_cg_phased(const CgArgs& a);
  /// exchange point pt of the sharded iteration (no-op on one device): pack the exported slots,
  /// move them (ex_), unpack the imported ones; guard: skip the kernels once the CG stopped.
  /// Returns the kernels launched.
  int xpoint(const CgArgs& a, int pt, bool guard);
  /// CG driver actually used by the last solve ("graph-while", "graph-chunked", "host-loop", "persistent")
  const char* cg_driver_ = "graph-while";
  bool capture_failed_ = false;  // the exchange backend refused stream capture: host loop from now on
  std::unique_ptr<Exchange> ex_;
  bool phased_ = false;
  // kernel timers: begin/end around a launch; collected after the stream syncs
  int ktimer_begin();
  void ktimer_end(int slot, const char* family, double flops, double bytes);
  void ktimer_collect();
  struct PendingTimer {
    cudaEvent_t a, b;
    const char* family;
    double flops, bytes;
  };
  std::vector<cudaEvent_t> ev_pool_;
  std::vector<PendingTimer> pending_;
  std::vector<std::pair<std::string, KernelStat>> stats_;
  bool profiling_ = false;
  double device_span_ms_ = 0;
  double* h_layers_ = nullptr;  // pinned staging of w0 | w1 | b
  bool layers_valid_ = false;

  int device_ = 0;
  Arena arena_;
  size_t l2_window_bytes_ = 0;
  void apply_l2_policy();
  cudaStream_t st_ = nullptr, cap_ = nullptr, side_ = nullptr;
  std::vector<cudaEvent_t> qr_events_;
  cudaEvent_t ev_[12] = {};
  cudaGraph_t graph_ = nullptr;
  cudaGraphExec_t graph_exec_ = nullptr;
  int* pinned_state_ = nullptr;
  int ld_ = 0, ext_ = 0, ncol_ = 0, kmax_ = 0, rmax_ = 1;
  int last_method_ = 2;
  bool built_ = false, blocks_built_ = false, coarse_built_ = false, neumann_built_ = false, solved_ = false;
  int last_iterations_ = 0;
  long long launches_ = 0, solve_launches_ = 0;
  double phase_ms_[8] = {};
  double host_build_ms_ = 0;

  // plan tables
  DevBuf<Task> d_tasks;
  DevBuf<int> d_task_off, d_task_cnt, d_cls, d_ix, d_iy, d_gamma_delta, d_gamma_pi, d_fluxrow_delta,
      d_ndelta_map, d_cr_row, d_cr_off, d_cr_l, d_row_owner, d_pi_owner, d_own_gamma, d_own_flux,
      d_own_nd, d_mult_pi, d_gamma_dst, d_flux_dst, d_nd_dst, d_corner_dst, d_cross_dst;
  DevBuf<ClassDims> d_dims;
  DevBuf<SubGeo> d_geo;
  std::vector<int> h_kf_ld_, h_kd_ld_;
  std::vector<long long> h_kf_off_, h_kd_off_, h_kfc_off_, h_kdc_off_;
  DevBuf<double> d_cr_w, d_flip, d_f, d_coef;
  // layers and matrices
  DevBuf<double> d_w0, d_w1, d_b, d_A, d_tau, d_T, d_ratio, d_F, d_Cd;
  DevBuf<int> d_deficient, d_rank, d_status, d_reff, d_perm, d_corner_q, d_spd_fail, d_state;
  DevBuf<double> d_V1, d_F1, d_Rr, d_tau1, d_zc, d_upd, d_dir, d_C, d_Y, d_QtX;
  // interface blocks / coarse
  DevBuf<int> d_kf_ld, d_kd_ld;
  DevBuf<long long> d_kf_off, d_kd_off, d_kfc_off, d_kdc_off;
  DevBuf<double> d_KFc, d_KDc;  // compact interface-level stream blocks (k_blocks.cu)
  DevBuf<double> d_FC, d_Zc, d_pd, d_Gc, d_Ypi, d_Dpp, d_dpi, d_S, d_Sinv, d_Wmu, d_Wd, d_W3;
  // CG
  DevBuf<double> d_x, d_r, d_p, d_Ap, d_rhs, d_partial, d_scal, d_hist, d_mu_pi_out, d_tpart, d_tpart3,
      d_psipart, d_o, d_xf, d_tr, d_zz, d_s, d_u, d_coeffs, d_pap, d_vin, d_vout, d_trace, d_KF, d_KD;
  // receive side of the owner-slot all-reduces (sharded only)
  DevBuf<double> d_field, d_fpart, d_fref, d_fsums, d_xc, d_opi, r_xc, r_opi;
  DevBuf<int> d_flo;
  DevBuf<double> d_Gsum, d_cin;
  DevBuf<int> d_cpi_g;
  // fused OP2..OP3 launch (one device): per subdomain itself + its edge neighbours, and the
  // per-stage completion counters
  DevBuf<int> d_nbr;
  DevBuf<unsigned> d_pflags;
  bool fuse_ok_ = false;
  // sharded exchange (XPlan): per (method family, point) the packed entry lists and per-point
  // send / receive buffers
  XPlan xplan_;
  DevBuf<XEntry> d_xsend[2][kXPoints], d_xrecv[2][kXPoints];
  DevBuf<double> d_xsbuf, d_xrbuf;
  int ldKF_ = 0, ldKD_ = 0;
};

}  // namespace ddg

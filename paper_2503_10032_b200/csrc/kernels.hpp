// Kernel launch interfaces of the DDELM-NN device path (all sm_100a, fp64).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "plan.hpp"

namespace ddg {

struct ClassDims {
  int n_int, n_bnd, n_gamma, m, fixed, nc, nd, nF;
};

// ---------------------------------------------------------------- features (k_features.cu)
struct FeatureArgs {
  int N, M, m, ld, ncol, n_grid, S, ldF, ldC;
  const Task* tasks;
  const int* cls_task_off;
  const int* cls_task_cnt;
  const ClassDims* dims;
  const int* sub_cls;
  const int* sub_ix;
  const int* sub_iy;
  const double* w0;
  const double* w1;
  const double* b;
  const double* f;  // N x m
  const double* coef;  // varcoef_poisson: N x tmax x 3 (rho, rho_x, rho_y) per class task; else nullptr
  int tmax;
  double* A;        // 2N matrices, ld x ncol column-major (K_i then Kbar_i)
  double* F;        // N x (M x ldF)
  double* Cd;       // N x (M x ldC)
};
void launch_build_features(const FeatureArgs& a, cudaStream_t st);

/// Device evaluation of the Gaussian random field at every row point (problems 3 poisson_grf and
/// 4 varcoef_poisson; k_features.cu grf_eval_kernel).
constexpr int kGrfTerms = 256;
struct GrfArgs {
  int problem, N, m, tmax, n_grid, S;
  const double* terms;  // 4 x 256: amp | fx | fy | phase (host-sampled, problems.cpp:15-39 order)
  const Task* tasks;
  const int* cls_task_off;
  const int* cls_task_cnt;
  const int* n_tasks_k;  // per class: leading K-row tasks
  const int* fixed;      // per class: K rows before the trace rows
  const int* sub_cls;
  const int* sub_ix;
  const int* sub_iy;
  double* f;     // N x m   (poisson_grf interior rows)
  double* coef;  // N x tmax x 3 (varcoef_poisson)
};
void launch_grf_eval(const GrfArgs& g, int max_tasks, cudaStream_t st);

// ---------------------------------------------------------------- QR (k_qr.cu)
struct QrArgs {
  int nmat, m, ld, ncol, M;
  double* A;    // nmat x ld x ncol
  double* tau;  // nmat x M
  double* T;    // nmat x kQrTmax x kQrTmax (block reflector of the current panel)
  double* trace = nullptr;  // DDELM_QR_TRACE: nmat x 8 section times of the shared-memory panel (ns)
};
constexpr int kQrNB = 32;
constexpr int kQrTmax = 64;
/// One step of the blocked factorisation: a 32-column panel writing its T factor to quadrant
/// (toff, toff) of the per-matrix 64 x 64 T (combine = 1: second half of a 64-wide block, also
/// forms the coupling block T12), or a DMMA trailing update with the nbw reflectors starting at k0
/// (T read at quadrant toff) applied to columns [cb, ce).
struct QrOp {
  enum Kind { kPanel, kTrail32, kTrail64 } kind;
  int k0, nbw, cb, ce, toff, combine;
};
std::vector<QrOp> qr_schedule(int M, int ncol);
void launch_qr_op(const QrArgs& a, const QrOp& op, cudaStream_t st);
double qr_op_flops(const QrArgs& a, const QrOp& op);
/// The whole factorisation with look-ahead on two streams (DDELM_QR_LOOKAHEAD=0: the plain op
/// schedule on `main`); `ev` is a reusable event pool.
void qr_factor(const QrArgs& a, cudaStream_t main, cudaStream_t side, std::vector<cudaEvent_t>& ev);
/// |R_ii| min / max per matrix -> ratio (branch test of LsFactor, solvers.cpp:27-32)
void launch_qr_diag_ratio(const QrArgs& a, double* ratio, cudaStream_t st);

// ---------------------------------------------------------------- COD (k_cod.cu)
struct CodArgs {
  int nmat, m, ld, ncol, M, kmax, rmax, ext;  // ext = appended columns used (1 + gmax)
  double rank_tol;
  const double* A;       // factored QR (R0 in the upper triangle of the top M x M block)
  const double* ratio;   // per matrix: unpivoted min/max |R_ii|
  int* deficient;        // per matrix: branch taken (1 = COD)
  // pivoted-QR state (per matrix)
  double* V1;    // kmax x M  (reflector t at V1[t*M + i])
  double* F1;    // kmax x M  (F1[t*M + j]: reflector t, column position j)
  double* Rr;    // kmax x M  (R rows by column position)
  double* tau1;  // kmax
  double* upd;   // M
  double* dir;   // M
  int* perm;     // M
  int* rank;     // per matrix
  int* status;   // per matrix: 0 ok, 1 capacity exceeded
  int* reff;     // per matrix: rows of R0 kept by the pivoted factorisation (diagnostic)
  double* zc;    // kmax RZ reflector coefficients
  // outputs (rmax-strided, allocated after ranks are known)
  double* C;     // nmat x M x rmax   : K^+ = C Q_r^T (C row i = original column i)
  double* QtX;   // nmat x rmax x ext : Q_r^T [f E] (top r rows)
  double* Ywork; // nmat x M x rmax scratch
  double* trace = nullptr;  // DDELM_COD_TRACE: nmat x 8 section times (ns) + steps
};
void launch_cod_pivqr(const CodArgs& a, cudaStream_t st);
void launch_cod_finish(const CodArgs& a, cudaStream_t st);  // RZ, C, Q^T X (both branches)
/// whether cod_finish handles an M-column matrix of numerical rank r (the sequential path above
/// rank 96 holds one column in 32 registers per lane: M <= 1024)
bool cod_finish_supports(int M, int r);

// ---------------------------------------------------------------- dense oracle (k_dense.cu)
/// C = alpha op(A) op(B) + beta C, column-major FP64
void dense_gemm(int m, int n, int k, double alpha, const double* A, int lda, bool ta, const double* B, int ldb,
                bool tb, double beta, double* C, int ldc, cudaStream_t st);
/// out (n x e) = X^+ R for X (m x n, m >= n) with Eigen's default COD threshold, on the batched
/// QR / COD kernels; synchronises the stream
void dense_cod_solve(const double* X, int ldx, int m, int n, const double* R, int ldr, int e, double* out, int ldo,
                     cudaStream_t st, int* rank_out);

/// LsFactor (solvers.cpp:24-45) of nmat caller matrices K (host, m x n column-major each) on the
/// hot path's QR / COD kernels: rank, branch, R0 rows kept by the pivoted factorisation (reff),
/// K^+ (host, n x m each) and optionally Q_r (host, m x n each, columns >= rank zero)
void lsfactor_batch(int nmat, int m, int n, const double* K, double rank_tol, int* rank, int* deficient, int* reff,
                    double* pinv, double* Q, cudaStream_t st);

// ---------------------------------------------------------------- interface blocks (k_blocks.cu)
/// Corner (Pi) rows per subdomain: 4 corners x cc components (cc = 2: biharmonic).
constexpr int kMaxCq = 8;

struct BlockArgs {
  int N, M, rmax, ext, gmax, fmax, dmax, crmax, ldF, ldC, n_pi, npf, n_delta;
  int ncq;               // corner rows per subdomain (4 cc)
  const int* rank;       // 2N
  const ClassDims* dims;
  const int* sub_cls;
  const double* F;       // N x M x ldF
  const double* Cd;      // N x M x ldC
  const double* C;       // 2N x M x rmax
  const double* QtX;     // 2N x rmax x ext
  double* FC;            // N x fmax x rmax
  // coarse
  const int* gamma_pi;   // N x gmax (-1 or Pi index)
  const int* cr_row;     // N x crmax (cross-flux row index r or -1)
  const int* cr_off;     // N x (crmax+1) offsets into cr_l / cr_w
  const int* cr_l;
  const double* cr_w;
  double* Zc;            // N x crmax x gmax : (K^+)^T a restricted to gamma rows
  double* pd;            // N x crmax : flux data F K^+ f per cross row (before scatter)
  double* Gc;            // N x ncq x ncq : -(Q_Pi Q_Pi^T)
  double* Ypi;           // N x M x ncq  : -C Q_Pi^T = K^+ B_Pi (corner columns)
  int* corner_q;         // N x ncq gamma rows of the corners (-1 pad)
  double* Dpp;           // npf x n_pi
  double* dpi;           // npf
  double* S;             // n_pi x n_pi
  double* Gsum;          // n_pi x n_pi : sum of the subdomain corner Grams (all-reduced when sharded)
  double* Sinv;          // n_pi x n_pi
  double* Wmu;           // n_pi x (n_pi + npf)
  double* Wd;            // npf x (n_pi + npf)
  double* W3;            // npf x n_pi
  const int* mult_pi;    // n_pi
  int* spd_fail;         // 1 flag
  int flip_row;          // debug_flip_flux_row (global flux row) or -1
  const int* row_owner;  // npf x 4 : contributing (ig * crmax + rho), global subdomain order, -1 pad
  const int* pi_owner;   // n_pi x 4 : corner owners (ig * ncq + slot), global subdomain order, -1 pad
  const int* cpi_g;      // N_global x ncq : Pi index of each corner slot (-1 pad)
  int sub_lo, N_global;  // this device's strip [sub_lo, sub_lo + N)
  double* pd_g;          // N_global x crmax              (coarse_export; all-reduced when sharded)
  double* zcc_g;         // N_global x crmax x ncq : Zc at the corner slots
  double* gc_g;          // N_global x ncq x ncq   : corner Grams
};
void launch_blocks(const BlockArgs& a, cudaStream_t st);
void launch_coarse_local(const BlockArgs& a, const int* cr_row, const int* cr_off, const int* cr_l,
                         const double* cr_w, cudaStream_t st);
/// pd / Zc corners / Gc of the local subdomains into the global compact arrays (pd_g, zcc_g, gc_g)
void launch_coarse_export(const BlockArgs& a, cudaStream_t st);
void launch_coarse_rows(const BlockArgs& a, cudaStream_t st);
void launch_coarse_gsum(const BlockArgs& a, cudaStream_t st);
void launch_coarse_schur(const BlockArgs& a, cudaStream_t st);
void launch_coarse_weights(const BlockArgs& a, cudaStream_t st);
/// Pack the CG stream blocks KF = [C | Ypi | F] and KD = [Cbar | Cdelta] (row-interleaved).
void launch_pack_streams(const BlockArgs& a, double* KF, const int* kf_ld, const long long* kf_off, double* KD,
                         const int* kd_ld, const long long* kd_off, cudaStream_t st);
/// Compact interface-level stream blocks (same strides): KFc rows [e_q | (F [C Ypi])^T row q],
/// KDc rows [e_q | (Cdelta Cbar)^T row q] (k_blocks.cu compact_stream_kernel).
void launch_compact_streams(const BlockArgs& a, const double* KF, const int* kf_ld, const long long* kf_off,
                            const double* KD, const int* kd_ld, const long long* kd_off, double* KFc,
                            const long long* kfc_off, double* KDc, const long long* kdc_off, cudaStream_t st);

// ---------------------------------------------------------------- C5 microbenchmark (k_lsq.cu)
struct LsqArgs {
  int nb, m, n, k, ld, ncol;  // ncol = n + k
  double* A;                  // nb x ld x ncol column-major: [K | B], factored in place
  double* S;                  // nb x k x k
};
void launch_lsq_generate(const LsqArgs& a, uint64_t seed, int kind, cudaStream_t st);  // kind 0 tanh, 1 N(0,1)
void launch_lsq_gram(const LsqArgs& a, cudaStream_t st);
/// measured FP64 tensor-pipe throughput (TFLOP/s) of a DMMA m8n8k4 loop on `device`
double fp64_peak_probe(int device);
/// y = tanh(x) with the feature builder's device tanh (k_features.cu; parity-decomposition hook)
void device_tanh(int device, const double* x, double* y, long long n);

// ---------------------------------------------------------------- CG (k_cg.cu)
/// Per-subdomain geometry of the interface iteration in one 48-byte record (one dependent load
/// instead of class -> dims, rank, strides, offsets).
struct SubGeo {
  int n_gamma, nF, nd, r, rb, kf_ld, kd_ld, pad;
  long long kf_off, kd_off;
  long long kfc_off, kdc_off;  // compact blocks (KFc: r + ncq rows, KDc: rb rows; strides kf_ld / kd_ld)
};
enum CgJob { kJobCg = 0, kJobApply = 1, kJobRhs = 2, kJobRecon = 3 };

constexpr int kCgMaxNbr = 8;
struct CgArgs {
  int N, n_delta, n_pi, npf, gmax, fmax, dmax, crmax, rmax, ext, M;
  int ncq;                 // corner rows per subdomain (4 cc); KF rows carry ncq Ypi entries
  double theta;
  int use_neumann;         // theta > 0
  // packed per-subdomain stream blocks (one bulk copy per chunk of rows), row j:
  //   KF : [ C_j (rmax) | Ypi_j (4) | F_j (fmax) ]        stride ldKF (even)
  //   KD : [ Cbar_j (rmax) | Cdelta_j (dmax) ]             stride ldKD (even)
  const double* KF;
  int ldKF;                 // widest row (capacity); per subdomain: kf_ld[i], block at KF + kf_off[i]
  const double* KD;
  int ldKD;
  // compact interface-level blocks (CG phases outside the reconstruction): the M-long
  // coefficient contraction folded in at setup, rows q < r (+ ncq Ypi rows for KFc)
  const double* KFc;
  const double* KDc;
  int compact;
  const int* kf_ld;
  const int* kd_ld;
  const long long* kf_off;
  const long long* kd_off;
  double rel_tol;
  int max_iter;
  const int* rank;         // 2N
  const ClassDims* dims;
  const int* sub_cls;
  const SubGeo* geo;       // N
  const int* gamma_delta;  // N x gmax
  const int* gamma_pi;     // N x gmax
  const int* fluxrow_delta;  // N x fmax
  const int* ndelta_map;   // N x dmax
  const int* cr_row;       // N x crmax
  const int* corner_q;     // N x 4
  // owner-slot destinations: every cross-subdomain sum is written by its producers into fixed
  // slots and read back contiguously in a fixed (subdomain) order — one dependent load per gather
  const int* gamma_dst;    // N x gmax : 2 g + s (slot s of Delta index g), -1 at corners
  const int* flux_dst;     // N x fmax : 2 g + s for the weight-1 Delta flux rows, -1 otherwise
  const int* nd_dst;       // N x dmax : 2 g + s for the Neumann Delta rows
  const int* corner_dst;   // N x 4    : gp * 4 + slot, -1 pad
  const int* cross_dst;    // N x crmax: rr * 4 + slot, -1 pad
  const double* flip_sign; // n_delta + npf (+1 / -1 debug hook, global flux row)
  // one-level DDELM (reduced_apply, solvers.cpp:262-274): no coarse space, the Pi trace values are
  // CG unknowns (mu = [mu_Delta; mu_Pi]) and A / A^T run over every flux row, cross rows included
  int one_level;
  int n_cg;                // CG vector length: n_delta, + n_pi one-level
  const int* cr_off;       // N x (crmax + 1) offsets into cr_l / cr_w (cross-row scatter triples)
  const int* cr_l;
  const double* cr_w;
  const double* QtX;       // 2N x rmax x ext (QGt = cols 1.., qf = col 0)
  const double* Zc;        // N x crmax x gmax
  const double* Sinv;      // n_pi x n_pi
  const double* Wmu;       // n_pi x (n_pi + npf) : [S^{-1} | S^{-1} Dpp^T]
  const double* Wd;        // npf x (n_pi + npf)  : [-Dpp S^{-1} | I - Dpp S^{-1} Dpp^T]
  const double* W3;        // npf x n_pi           : Dpp S^{-1}
  const double* dpi;       // npf
  // P row-parts per subdomain: every streamed phase is split over the M coefficient rows into P
  // independent work items whose partial outputs are summed (fixed order) by the consumer.
  int P;
  int rpc_max;    // largest rows-per-chunk of the streaming pipeline
  double* s;      // N x rmax
  // owner-slot tables: producers write the *_w copy (their own slots), consumers read the plain
  // copy; identical pointers on one device, send / receive buffers of an all-reduce when sharded
  double *ttab, *ttab_w;    // n_pi x 4    corner contributions of OP1
  double *ptab, *ptab_w;    // npf x 4     cross-row contributions of OP1
  double *t3tab, *t3tab_w;  // P x n_pi x 4 corner contributions of OP3
  double *otab, *otab_w;    // 2 n_delta   OP4 outputs at the two owners of each Delta index
  double *xtab, *xtab_w;    // P x 2 n_delta  flux values x (OP2)
  double *trtab, *trtab_w;  // P x 2 n_delta  P x (NN1)
  double *zztab, *zztab_w;  // P x 2 n_delta  P^T P x (NN2)
  double *xctab, *xctab_w;  // P x npf x 4   cross-row flux contributions (OP2, one-level)
  double *opitab, *opitab_w;  // n_pi x 4    OP4 outputs at the corner owners (one-level)
  int N_global, sub_lo;     // sharding: this device holds subdomains [sub_lo, sub_lo + N)
  int xr_parts;             // r.r partials written by the XR phase (= its grid size)
  unsigned long long cond;  // cudaGraphConditionalHandle of the CG while-loop graph (0: none)
  int guard_all;            // chunked driver: every phase (streamed ones too) leaves once state[1] is set
  int preissue;             // stream chunks a streamed phase issues before griddepcontrol.wait (<= kStages)
  // fused OP2..OP3 launch (kPhFused, one device): subdomain i's items wait, between phases, only for
  // the completion counters of the subdomains whose owner slots they read (i and its edge neighbours)
  const int* nbr;           // N x kCgMaxNbr: i itself first, then its edge neighbours, -1 pad
  unsigned* pflags;         // 3 x N completion counters (after OP2, NN1, NN2): P per iteration
  int fuse_gate;            // producer holds the next phase's chunks past `preissue` until the wait passes
  unsigned fuse_sleep;      // ns of __nanosleep between polls of a completion counter (0: spin)
  int fuse_pre;             // load the next phase's StreamPre (static prologue data) during the wait
  int l2ahead;              // stream chunks past the preissued ring prefetched into L2 before griddepcontrol.wait
  int l2pre;                // per mille of each OP2 item prefetched into L2 by OP4 (HBM idle during OP4 / XR / OP1);
                            // negative: the same with the evict_last priority; 0: off
  int l2keep;               // per mille of each NN1 / OP3 item's chunks loaded L2::evict_last (read first by
                            // the reverse / next walk); the other stream chunks evict_first; < 0: no hints
  double* u;      // P x N x rmax
  double *pap, *pap_w;  // N_global : p . o_i (indexed by global subdomain)
  // CG vectors
  double* x;
  double* r;
  double* pbuf[2];  // double-buffered search direction
  double* rhs;
  double* partial;  // reduction scratch (>= grid)
  double* hist;     // max_iter
  int* state;       // [1] done, [2] converged, [3] negcurv, [5] iterations, [6] current iteration
  double* scal;     // [0] rr, [1] bnorm, [2] beta (phase-by-phase CG)
  double* coeffs;   // N x M output
  double* mu_pi_out;  // n_pi
  double* trace;      // optional G x 16 per-phase ns counters of the CG job (nullptr: off)
};
/// One launch of the persistent cooperative kernel: kJobCg runs the whole CG loop
/// (solvers.cpp:95-117); kJobApply writes vout = cs_reduced_apply(vin) (solvers.cpp:372-386);
/// kJobRhs writes vout = the reduced right-hand side (solvers.cpp:542-551); kJobRecon writes the
/// coefficients and mu_Pi for mu_Delta = vin (solvers.cpp:565-577).
void cg_launch(const CgArgs& a, int job, const double* vin, double* vout, cudaStream_t st);
/// Phase-by-phase execution (sharded mode: an all-reduce of the owner-slot tables between phases)
enum CgPhase { kPhOp1 = 0, kPhOp2, kPhNn1, kPhNn2, kPhOp3, kPhOp4, kPhXr1, kPhXr2, kPhGather,
               kPhFused /* OP2 -> NN1 -> NN2 -> OP3 in one launch, neighbour flags between them */ };
/// mode: 0 operator / CG, 1 reduced rhs, 2 reconstruction; it: CG iteration (1-based, CG only)
/// apply_P / apply_PT staging around the NN1 / NN2 phases (see k_cg.cu neumann_io_kernel)
void cg_launch_neumann_io(const CgArgs& a, int op, const double* v, double* out, cudaStream_t st);
void cg_launch_phase(const CgArgs& a, int phase, int mode, int it, const double* vin, double* vout,
                     cudaStream_t st);
void cg_launch_init(const CgArgs& a, cudaStream_t st);
int cg_grid(const CgArgs& a);

/// The owner-slot tables of one CgArgs as the exchange kernels see them (plan.hpp XTable ids).
struct XTabs {
  double* ptr[kTabCount];
  int parts[kTabCount];
  long long pstride[kTabCount];
};
XTabs cg_xtabs(const CgArgs& a);
/// out[k] = P-part sum of slot e[k] (skipped once state[1] is set when state != nullptr)
void launch_xpack(const XTabs& t, const XEntry* e, int n, double* out, const int* state, cudaStream_t st);
/// slot e[k] (part 0) = in[k]
void launch_xunpack(const XTabs& t, const XEntry* e, int n, const double* in, const int* state, cudaStream_t st);
int cg_rows_per_chunk_max(const CgArgs& a);


// ---------------------------------------------------------------- field evaluation (k_field.cu)
/// Field samples and trapezoid error sums on the n x n grid (metrics.cpp:18-88).
struct FieldArgs {
  int n, N, M, problem;
  const int* sub_ix;
  const int* sub_iy;
  const int* lo;          // s + 1 boundaries: grid index a in [lo[k], lo[k+1]) lies in column k
  const double* w0;       // N x M layers
  const double* w1;
  const double* b;
  const double* coef;     // N x M coefficients of the field
  const double* coef_ref; // N x M reference coefficients (nullptr: the problem's exact solution)
  double* u;              // n x n samples, index b*n + a (nullable)
  double* gx;
  double* gy;
  double* part;           // field_parts() x 4 partial sums
};
int field_parts(const FieldArgs& f, int max_pts);
/// sums = {sum w du^2, sum w u_ref^2, sum w |d grad|^2, sum w |grad_ref|^2}
void launch_field(const FieldArgs& f, int max_pts, double* sums, cudaStream_t st);

}  // namespace ddg

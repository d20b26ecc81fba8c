/*
 * ddelm_gpu.h — C-ABI boundary of the B200-native DDELM-NN hot path.
 *
 * Replaces the reference's C++ solver entry points (no torch types, plain pointers/sizes):
 *   ddelm_gpu_create        Workspace::Workspace(problem, s, n_grid, M, l, seed, opts)
 *                           (proj/include/ddelm/solvers.hpp:79-80, src/solvers.cpp:123-167)
 *   ddelm_gpu_build         the assembly + LsFactor part of that constructor
 *                           (solvers.cpp:131-151; features.cpp:42-76; assembly.cpp:9-87)
 *   ddelm_gpu_build_coarse  Workspace::assemble_coarse      (solvers.cpp:278-326)
 *   ddelm_gpu_build_neumann Workspace::build_neumann        (solvers.cpp:390-448)
 *   ddelm_gpu_solve         ddelm_cs_solve / ddelm_nn_solve (solvers.cpp:582-605, 535-578)
 *   ddelm_gpu_get_*         SolveReport fields               (solvers.hpp:162-171)
 *   ddelm_gpu_destroy       ~Workspace
 *   ddelm_gpu_dense_oracle  dense_oracle_solve (solvers.cpp:609-709), behind oracle_check
 *                           (runner.cpp:252-316)
 *
 * Error convention (mirrors the reference's exceptions, solvers.hpp / SURVEY.md §8b):
 *   DDELM_OK = 0
 *   DDELM_ERR_INVALID_ARGUMENT  std::invalid_argument  (theta outside [0,1], s < 1,
 *                               n_grid < 3, M < 1, l <= 0, non-tall K, unknown problem)
 *   DDELM_ERR_RUNTIME           std::runtime_error     (coarse Schur matrix not SPD)
 *   DDELM_ERR_CUDA              CUDA / NCCL failure (no device, launch error, OOM)
 *   DDELM_ERR_CAPACITY          numerical rank above the device COD capacity
 * Non-convergence is not an error: ddelm_report.converged = 0 (solvers.cpp:515,560).
 * The message of the last error on the calling thread: ddelm_gpu_last_error().
 *
 * Ownership: device memory is owned by the workspace; host output buffers are caller
 * allocated. One CUDA stream per workspace; calls are not reentrant per workspace.
 */
#ifndef DDELM_GPU_H
#define DDELM_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  DDELM_OK = 0,
  DDELM_ERR_INVALID_ARGUMENT = 1,
  DDELM_ERR_RUNTIME = 2,
  DDELM_ERR_CUDA = 3,
  DDELM_ERR_CAPACITY = 4
};

/* problem ids (make_problem, problems.cpp:132-188; C4's problem is an addition) */
enum {
  DDELM_POISSON_SINPI = 0,
  DDELM_POISSON_SIN2PI_EXP = 1,
  DDELM_POISSON_SIN2PI_COS3PI_X2Y = 2,
  DDELM_POISSON_GRF = 3,      /* -lap u = GRF(forcing_seed), u = 0 on the boundary */
  DDELM_VARCOEF_POISSON = 4,  /* -div(rho grad u) = 1, rho = tanh(GRF(rho_seed)) + 1.1 */
  DDELM_BIHARMONIC_SINPI = 5  /* lap^2 u = 4 pi^4 sin sin: cc = bc = 2 (value + Laplacian) */
};

enum { DDELM_METHOD_DDELM = 0, DDELM_METHOD_CS = 1, DDELM_METHOD_NN = 2 };
enum { DDELM_FLUX_POINTWISE = 0, DDELM_FLUX_MEAN_EDGE = 1 };

typedef struct ddelm_desc {
  int problem;              /* DDELM_POISSON_* */
  int s;                    /* s x s subdomains */
  int n_grid;               /* collocation points per direction per subdomain */
  int M;                    /* neurons per subdomain */
  double l;                 /* weight scale (features.cpp:9-35) */
  uint64_t seed;            /* per-subdomain seed + i (solvers.cpp:136) */
  int flux_variant;         /* DDELM_FLUX_* */
  int change_of_variables;  /* 0 nodal, 1 change of variables */
  double rank_tol;          /* SolverOptions::rank_tol, 1e-10 */
  int device;               /* CUDA device ordinal */
  int debug_flip_flux_row;  /* validation hook (solvers.hpp:54-57); -1 = off */
  double alpha;             /* ProblemParams (problems.hpp:64-68): GRF smoothness, default 32 */
  uint64_t forcing_seed;    /* GRF forcing seed (poisson_grf), default 2 */
  uint64_t rho_seed;        /* GRF coefficient seed (varcoef_poisson), default 3 */
} ddelm_desc;

typedef struct ddelm_report {
  int iterations;
  int converged;
  int negative_curvature;
  int n_delta, n_pi, n_mu, n_subdomains, M;
  double assembly_seconds;       /* feature + matrix build (device time) */
  double factorization_seconds;  /* QR / COD (device time) */
  double setup_seconds;          /* coarse + Neumann layers + reduced RHS */
  double cg_seconds;
  double reconstruct_seconds;
  double total_seconds;
} ddelm_report;

typedef struct ddelm_ws ddelm_ws;

const char* ddelm_gpu_last_error(void);
const char* ddelm_gpu_version(void);

int ddelm_gpu_create(const ddelm_desc* desc, ddelm_ws** out);
/* Sharded workspace (one process per GPU): rank `rank` of `world` owns the contiguous strip of
 * subdomains ddelm_gpu_get_shard reports and factorises only those; the coarse problem and the
 * interface vectors are replicated. Every cross-subdomain sum lives in an owner-slot table (one
 * writer per slot); between the CG phases each rank sends the slots it wrote to the ranks that
 * read them (grouped ncclSend / ncclRecv; the CG loop is one CUDA graph replayed in chunks), so
 * the result is bitwise that of one device with the same work split (DDELM_CG_PARTS). nccl_id:
 * 128 bytes from ddelm_gpu_nccl_unique_id on rank 0, broadcast by the caller. world = 1 is the
 * single-device path (nccl_id unused). Coefficients / ranks / layers returned by the getters are
 * those of the local strip. (Replaces the reference's serial loops over subdomains,
 * solvers.cpp:207-224,338,361,457-458,470-471, with the strip partition of the paper's MPI split.) */
int ddelm_gpu_nccl_unique_id(unsigned char* nccl_id /* 128 bytes */);
int ddelm_gpu_create_sharded(const ddelm_desc* desc, int rank, int world, const unsigned char* nccl_id,
                             ddelm_ws** out);
/* Test backend of the sharded path: the same kernels and exchange lists, the slot segments
 * host-staged through a POSIX shared-memory mailbox `shm_name` ("/...", the same on every rank)
 * with a host barrier — synchronous, so several ranks can share ONE GPU (no kernel waits for
 * another rank's kernel). Not a performance path. */
int ddelm_gpu_create_sharded_host(const ddelm_desc* desc, int rank, int world, const char* shm_name,
                                  ddelm_ws** out);
/* Host-only view of the exchange plan of `rank` (no device needed): one_level 0 (coarse methods)
 * or 1, point 0..5 (after OP1, OP2, NN1, NN2, OP3, OP4), which = 0 send entries / 1 receive
 * entries as (table, slot) pairs, 2 send counts / 3 receive counts / 4 send offsets per peer,
 * 5 = {largest message in doubles}. Returns the length, or -error. */
int ddelm_gpu_exchange_lists(const ddelm_desc* desc, int rank, int world, int one_level, int point, int which,
                             int* out, int cap);
/* CG driver the last solve used: "graph-while", "graph-chunked", "host-loop" or "persistent". */
const char* ddelm_gpu_cg_driver(ddelm_ws* ws);
int ddelm_gpu_get_shard(ddelm_ws* ws, int* sub_lo, int* sub_count, int* n_global);
/* Host-only view of a shard's owner-slot tables (no device needed): which = 0 gamma, 1 flux,
 * 2 Neumann, 3 corner, 4 cross-row destinations of the local strip, 5 = {sub_lo, N_local,
 * N_global, n_delta, n_pi, npf, gmax, fmax, dmax, crmax, ncq}. Returns the table length (copies at
 * most cap entries into out), or -error. */
int ddelm_gpu_plan_tables(const ddelm_desc* desc, int rank, int world, int which, int* out, int cap);
int ddelm_gpu_build(ddelm_ws* ws);
int ddelm_gpu_build_coarse(ddelm_ws* ws);
int ddelm_gpu_build_neumann(ddelm_ws* ws);
/* method: DDELM_METHOD_DDELM (one-level ddelm_solve, solvers.cpp:493-531: CG on
 * mu = [mu_Delta; mu_Pi], theta ignored), DDELM_METHOD_CS or DDELM_METHOD_NN (theta in [0,1];
 * theta = 0 is exactly CS). max_iter <= 0 means 20 x the CG dimension (solvers.cpp:85). */
int ddelm_gpu_solve(ddelm_ws* ws, int method, double theta, double rel_tol, int max_iter,
                    ddelm_report* report);
/* Re-seed the feature layers (seed + i per subdomain) and invalidate every built layer;
 * the geometry / index plan is kept. */
int ddelm_gpu_reseed(ddelm_ws* ws, uint64_t seed);
/* Operator representation of the interface iteration (no reference counterpart):
 * DDELM_CG_BLOCKS_COEFF (default) streams the coefficient-space blocks every iteration in the
 * reference's grouping (c = K^+ phi, then F c: solvers.cpp:215-218, 455, 468), which reproduces
 * its finite-precision CG trajectory; DDELM_CG_BLOCKS_COMPACT folds the M-long coefficient
 * contraction into precomputed interface-level blocks F [C Ypi] and Cdelta Cbar once per build
 * (about 10x less traffic per iteration; the same operator in exact arithmetic, but CG then
 * follows a different round-off trajectory and typically converges in fewer iterations). */
#define DDELM_CG_BLOCKS_COEFF 0
#define DDELM_CG_BLOCKS_COMPACT 1
int ddelm_gpu_set_cg_blocks(ddelm_ws* ws, int mode);
void ddelm_gpu_destroy(ddelm_ws* ws);

/* Results of the last solve (host buffers, caller allocated). */
int ddelm_gpu_get_mu(ddelm_ws* ws, double* mu /* n_mu: Delta then Pi */);
int ddelm_gpu_get_coeffs(ddelm_ws* ws, double* coeffs /* n_subdomains x M */);
int ddelm_gpu_get_residuals(ddelm_ws* ws, double* hist, int cap);

/* Field of the last solve on the uniform n x n grid of [0,1]^2 (point (a,b) = (a,b)/(n-1)),
 * evaluated on the device by the owning subdomain's ELM (sample_field, metrics.cpp:18-57).
 * u, gx, gy: n*n host buffers, index b*n + a, each may be NULL. On a sharded workspace only the
 * points of this rank's subdomains are filled (the rest are 0). */
int ddelm_gpu_sample_field(ddelm_ws* ws, int n, double* u, double* gx, double* gy);
/* Relative L2 and H1 errors (trapezoid rule on the n x n grid) against the problem's exact
 * solution: relative_errors (metrics.cpp:112-128). n < 64 -> DDELM_ERR_INVALID_ARGUMENT, as the
 * reference. Sharded: the sums are all-reduced, every rank gets the global errors. */
int ddelm_gpu_relative_errors(ddelm_ws* ws, int n, double* l2, double* h1);
/* The same errors against the ELM field of ref_coeffs (n_subdomains x M, this workspace's
 * layers): oracle_check's field_diff (runner.cpp:269-281). */
int ddelm_gpu_field_diff(ddelm_ws* ws, int n, const double* ref_coeffs, double* l2, double* h1);
/* Per-subdomain numerical ranks of K_i and Kbar_i (-1 when the layer is not built) and the
 * unpivoted-QR diagonal ratio min|R_ii|/max|R_ii| used by the branch test (solvers.cpp:27-32). */
int ddelm_gpu_get_ranks(ddelm_ws* ws, int* rank_k, int* rank_kbar, double* qr_ratio /* 2N */);
/* Feature layer of subdomain i (w0, w1, b: M each) — for field evaluation by the caller. */
int ddelm_gpu_get_layer(ddelm_ws* ws, int i, double* w0, double* w1, double* b);
/* Local matrices as built on the device (rows x M column-major), for parity tests. */
int ddelm_gpu_get_local(ddelm_ws* ws, int i, int which /* 0 K, 1 Kbar, 2 f (rows x 1) */, double* K, int* rows);
/* out = cs_reduced_apply(v, weight) on the device (solvers.cpp:372-386, weight 599-603;
 * theta = 0: plain coarse operator). v, out: n_delta host doubles. Builds layers as needed. */
int ddelm_gpu_apply_operator(ddelm_ws* ws, double theta, const double* v, double* out);
/* out = reduced_apply(v), the one-level operator (solvers.cpp:262-274); v, out: n_mu = n_delta +
 * n_pi host doubles. */
int ddelm_gpu_apply_reduced(ddelm_ws* ws, const double* v, double* out);
/* The Neumann map P = Abar Kbar^+ Bbar (transpose = 0, Workspace::apply_P) or its adjoint
 * (transpose = 1, apply_PT), solvers.cpp:450-474: v, out n_delta host doubles. Builds the coarse
 * and Neumann layers as needed. */
int ddelm_gpu_apply_neumann(ddelm_ws* ws, int transpose, const double* v, double* out);
/* dense_oracle_solve (solvers.cpp:609-709) on the device: the global block matrices K, B, A (and
 * Kbar, Bbar, Abar for NN) assembled densely, every pseudo-inverse through the device QR / COD
 * kernels with Eigen's default threshold eps * min(rows, cols). method: DDELM_METHOD_*; the
 * reduced system has dim = n_mu (one-level) or n_delta (CS / NN). Outputs (each may be NULL):
 * reduced_op dim x dim column-major, reduced_rhs dim, mu_full n_mu, coeffs n_subdomains x M.
 * sum(M) + n_mu > 3000 -> DDELM_ERR_INVALID_ARGUMENT (solvers.cpp:619-620), as is a sharded
 * workspace. Regenerates the local matrices: the next solve rebuilds the factorisations. */
/* LsFactor (solvers.cpp:24-78) of nmat caller-supplied m x n matrices (m >= n; K: nmat blocks,
 * each column-major m x n) on the hot path's own kernels (batched QR, diagonal-ratio branch test
 * at rank_tol, pivoted QR + RZ, finish). Outputs per matrix: numerical rank, the branch taken
 * (1 = complete orthogonal decomposition), reff (R0 rows the pivoted factorisation kept; NULL ok),
 * K^+ (pinv: n x m column-major) and Q_r (Q: m x n column-major, columns >= rank zero; NULL ok),
 * so apply_pinv / apply_pinv_transpose / apply_projection are K^+ v, (K^+)^T u, Q_r Q_r^T v.
 * Errors: m < n -> DDELM_ERR_INVALID_ARGUMENT (solvers.cpp:26). Test hook of the factorisation. */
int ddelm_gpu_lsfactor_batch(int device, int nmat, int m, int n, const double* K, double rank_tol, int* rank,
                             int* deficient, int* reff, double* pinv, double* Q);
int ddelm_gpu_dense_oracle(ddelm_ws* ws, int method, double theta, int* dim, double* reduced_op,
                           double* reduced_rhs, double* mu_full, double* coeffs);
/* Drop every built layer (features, factors, coarse, Neumann) but keep the feature layers
 * already uploaded to the device: the next solve re-runs the whole device pipeline. */
int ddelm_gpu_invalidate(ddelm_ws* ws);
/* The workspace's CUDA stream (cudaStream_t), for callers that time on the device. */
void* ddelm_gpu_stream(ddelm_ws* ws);
/* Per-kernel-family CUDA-event timers (off by default). family: "build_features", "qr_panel",
 * "qr_trailing", "cod_pivqr", "cod_finish", "cg_iterations". Values accumulate until reset. */
int ddelm_gpu_set_profiling(ddelm_ws* ws, int on);
int ddelm_gpu_get_kernel_stats(ddelm_ws* ws, const char* family, double* total_ms,
                               long long* launches, double* flops, double* bytes);
/* Device time of the last solve from the first feature kernel to the reconstruction (ms). */
double ddelm_gpu_get_device_span_ms(ddelm_ws* ws);
/* Per-phase device timings of the last build/solve (ms): see workspace.cu for the order. */
int ddelm_gpu_get_phase_ms(ddelm_ws* ws, double* ms, int cap);
/* Kernel launches issued by the last ddelm_gpu_build..solve sequence (own kernels only). */
long long ddelm_gpu_get_launch_count(ddelm_ws* ws);

/* ---- C5: batched local least-squares microbenchmark (BASELINE.json config 5).
 * nblocks independent [K | B] blocks (m x n and m x k, column-major, ld = ddelm_gpu_lsq_ld),
 * generated on the device (kind 0: tanh(w.x + b), w, b ~ U[-1,1], x ~ U[0,1]^2; kind 1: N(0,1)
 * control) from a counter-based hash of (seed, block, index); factored with the batched
 * Householder QR of LsFactor (solvers.cpp:24-45): R and the reflectors in place of K, Q^T B in
 * place of B; then S = (Q^T B)_bot^T (Q^T B)_bot = B^T B - (Q^T B)_top^T (Q^T B)_top (k x k), the
 * interface Schur block of assemble_coarse's products (solvers.cpp:286-321), on FP64 tensor cores.
 * n must be even. */
typedef struct ddelm_lsq ddelm_lsq;
int ddelm_gpu_lsq_create(int nblocks, int m, int n, int k, int device, ddelm_lsq** out);
int ddelm_gpu_lsq_generate(ddelm_lsq* lsq, uint64_t seed, int kind);
int ddelm_gpu_lsq_factor(ddelm_lsq* lsq, double* qr_ms, double* schur_ms);
/* A: ld x (n + k) factored block, tau: n Householder scalars, S: k x k (any may be NULL) */
int ddelm_gpu_lsq_get_block(ddelm_lsq* lsq, int block, double* A, double* tau, double* S);
int ddelm_gpu_lsq_ld(ddelm_lsq* lsq);
void ddelm_gpu_lsq_destroy(ddelm_lsq* lsq);
/* FP64 tensor-pipe throughput of this device (TFLOP/s): a DMMA m8n8k4 loop on every SM, best of
 * three CUDA-event-timed launches — the FP64 roofline denominator bench.py reports against. */
int ddelm_gpu_fp64_peak(int device, double* tflops);
/* y[k] = tanh(x[k]) for k < n with the device tanh the feature builder uses (test hook: lets the
 * CPU oracle run on bitwise the device's feature matrices, tools/parity_decomposition.py). */
int ddelm_gpu_tanh(int device, const double* x, double* y, long long n);

#ifdef __cplusplus
}
#endif

#endif /* DDELM_GPU_H */

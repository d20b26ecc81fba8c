// C-ABI boundary (include/ddelm_gpu.h) over the device workspace. No CPU fallback: every entry
// point fails with DDELM_ERR_CUDA when no CUDA device is usable.
#include <cmath>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/ddelm_gpu.h"
#include "common.cuh"
#include "plan.hpp"
#include "workspace.hpp"

struct ddelm_ws {
  ddg::Workspace* w = nullptr;
  ddelm_report last{};
};

/// C5 batched least-squares microbenchmark state (k_lsq.cu + k_qr.cu).
struct ddelm_lsq {
  int device = 0;
  ddg::LsqArgs a{};
  double *tau = nullptr, *T = nullptr;
  cudaStream_t st = nullptr, side = nullptr;
  std::vector<cudaEvent_t> qr_ev;
  cudaEvent_t ev[3] = {};
  ~ddelm_lsq() {
    cudaSetDevice(device);
    cudaFree(a.A);
    cudaFree(a.S);
    cudaFree(tau);
    cudaFree(T);
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
    for (cudaEvent_t e : qr_ev) cudaEventDestroy(e);
    if (side) cudaStreamDestroy(side);
    if (st) cudaStreamDestroy(st);
  }
};

namespace {

thread_local std::string g_err;

ddg::ProblemParams desc_params(const ddelm_desc* d) {
  ddg::ProblemParams pp;
  pp.alpha = d->alpha;
  pp.forcing_seed = d->forcing_seed;
  pp.rho_seed = d->rho_seed;
  return pp;
}

template <typename F>
int guarded(F&& f) {
  try {
    f();
    g_err.clear();
    return DDELM_OK;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return DDELM_ERR_INVALID_ARGUMENT;
  } catch (const ddg::CapacityError& e) {
    g_err = e.what();
    return DDELM_ERR_CAPACITY;
  } catch (const ddg::CudaError& e) {
    g_err = e.what();
    return DDELM_ERR_CUDA;
  } catch (const std::exception& e) {
    g_err = e.what();
    return DDELM_ERR_RUNTIME;
  }
}

}  // namespace

extern "C" {

const char* ddelm_gpu_last_error(void) { return g_err.c_str(); }
const char* ddelm_gpu_version(void) { return "ddelm-b200 0.1 (sm_100a)"; }

int ddelm_gpu_create(const ddelm_desc* d, ddelm_ws** out) {
  return guarded([&] {
    if (!d || !out) throw std::invalid_argument("ddelm_gpu_create: null argument");
    *out = nullptr;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
      throw ddg::CudaError("ddelm_gpu_create: no CUDA device available (no CPU fallback)");
    if (d->device < 0 || d->device >= ndev) throw std::invalid_argument("ddelm_gpu_create: bad device ordinal");
    ddg::Plan p = ddg::build_plan(d->problem, d->s, d->n_grid, d->M, d->l, d->seed, d->flux_variant,
                                  d->change_of_variables != 0, d->rank_tol > 0 ? d->rank_tol : 1e-10,
                                  d->debug_flip_flux_row, desc_params(d));
    auto* h = new ddelm_ws;
    try {
      h->w = new ddg::Workspace(ddg::shard_plan(p, 0, p.N), d->device);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

int ddelm_gpu_nccl_unique_id(unsigned char* id) {
  return guarded([&] {
    if (!id) throw std::invalid_argument("ddelm_gpu_nccl_unique_id: null argument");
    ddg::NcclExchange::unique_id(id);
  });
}

int ddelm_gpu_tanh(int device, const double* x, double* y, long long n) {
  return guarded([&] {
    if ((!x || !y) && n > 0) throw std::invalid_argument("ddelm_gpu_tanh: null argument");
    ddg::device_tanh(device, x, y, n);
  });
}

}  // extern "C"

namespace {
ddg::Plan global_plan(const ddelm_desc* d) {
  return ddg::build_plan(d->problem, d->s, d->n_grid, d->M, d->l, d->seed, d->flux_variant, d->change_of_variables != 0,
                         d->rank_tol > 0 ? d->rank_tol : 1e-10, d->debug_flip_flux_row, desc_params(d));
}

/// sharded workspace of `rank`: its strip of the global plan, the exchange plan, the backend
template <class MakeEx>
int create_sharded(const char* fn, const ddelm_desc* d, int rank, int world, ddelm_ws** out, MakeEx make_ex) {
  return guarded([&] {
    if (!d || !out) throw std::invalid_argument(std::string(fn) + ": null argument");
    if (world < 1 || rank < 0 || rank >= world) throw std::invalid_argument(std::string(fn) + ": bad rank / world");
    *out = nullptr;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
      throw ddg::CudaError(std::string(fn) + ": no CUDA device available (no CPU fallback)");
    if (d->device < 0 || d->device >= ndev) throw std::invalid_argument(std::string(fn) + ": bad device ordinal");
    ddg::Plan g = global_plan(d);
    if (world > g.N) throw std::invalid_argument(std::string(fn) + ": more ranks than subdomains");
    int lo = 0, hi = 0;
    ddg::shard_range(g.N, rank, world, &lo, &hi);
    ddg::XPlan xp = ddg::build_exchange_plan(g, rank, world);
    std::unique_ptr<ddg::Exchange> ex = make_ex(xp);
    auto* h = new ddelm_ws;
    try {
      h->w = new ddg::Workspace(ddg::shard_plan(g, lo, hi), d->device, world > 1 ? std::move(ex) : nullptr, std::move(xp));
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}
}  // namespace

extern "C" {

int ddelm_gpu_create_sharded(const ddelm_desc* d, int rank, int world, const unsigned char* nccl_id, ddelm_ws** out) {
  if (world > 1 && !nccl_id) {
    return guarded([] { throw std::invalid_argument("ddelm_gpu_create_sharded: null nccl_id"); });
  }
  return create_sharded("ddelm_gpu_create_sharded", d, rank, world, out, [&](const ddg::XPlan&) {
    return std::unique_ptr<ddg::Exchange>(world > 1 ? new ddg::NcclExchange(rank, world, nccl_id, d->device) : nullptr);
  });
}

int ddelm_gpu_create_sharded_host(const ddelm_desc* d, int rank, int world, const char* shm_name, ddelm_ws** out) {
  if (!shm_name) return guarded([] { throw std::invalid_argument("ddelm_gpu_create_sharded_host: null shm_name"); });
  return create_sharded("ddelm_gpu_create_sharded_host", d, rank, world, out, [&](const ddg::XPlan& xp) {
    return std::unique_ptr<ddg::Exchange>(world > 1 ? new ddg::HostExchange(rank, world, shm_name, xp.max_msg) : nullptr);
  });
}

int ddelm_gpu_exchange_lists(const ddelm_desc* d, int rank, int world, int one_level, int point, int which, int* out,
                             int cap) {
  int n = 0;
  const int rc = guarded([&] {
    if (!d || world < 1 || rank < 0 || rank >= world || one_level < 0 || one_level > 1 || point < 0 ||
        point >= ddg::kXPoints || which < 0 || which > 5)
      throw std::invalid_argument("ddelm_gpu_exchange_lists: bad argument");
    const ddg::XPlan xp = ddg::build_exchange_plan(global_plan(d), rank, world);
    const ddg::XList& L = xp.pt[one_level][point];
    std::vector<int> v;
    if (which <= 1) {
      for (const ddg::XEntry& e : which == 0 ? L.send : L.recv) {
        v.push_back(e.table);
        v.push_back(e.idx);
      }
    } else if (which == 5) {
      v.push_back(static_cast<int>(std::min<size_t>(xp.max_msg, 0x7fffffff)));
    } else {
      v = which == 2 ? L.scnt : which == 3 ? L.rcnt : L.soff;
    }
    n = static_cast<int>(v.size());
    if (out) std::memcpy(out, v.data(), sizeof(int) * std::min<size_t>(v.size(), static_cast<size_t>(std::max(cap, 0))));
  });
  return rc == DDELM_OK ? n : -rc;
}

const char* ddelm_gpu_cg_driver(ddelm_ws* ws) { return ws ? ws->w->cg_driver() : ""; }

int ddelm_gpu_plan_tables(const ddelm_desc* d, int rank, int world, int which, int* out, int cap) {
  int n = 0;
  const int rc = guarded([&] {
    if (!d || world < 1 || rank < 0 || rank >= world || which < 0 || which > 5)
      throw std::invalid_argument("ddelm_gpu_plan_tables: bad argument");
    ddg::Plan g = ddg::build_plan(d->problem, d->s, d->n_grid, d->M, d->l, d->seed, d->flux_variant,
                                  d->change_of_variables != 0, d->rank_tol > 0 ? d->rank_tol : 1e-10,
                                  d->debug_flip_flux_row, desc_params(d));
    int lo = 0, hi = 0;
    ddg::shard_range(g.N, rank, world, &lo, &hi);
    const ddg::Plan p = ddg::shard_plan(g, lo, hi);
    const std::vector<int>* v = nullptr;
    std::vector<int> meta = {p.sub_lo, p.N, p.N_global, p.n_delta, p.n_pi, p.npf, p.gmax, p.fmax, p.dmax, p.crmax, p.ncq};
    switch (which) {
      case 0: v = &p.gamma_dst; break;
      case 1: v = &p.flux_dst; break;
      case 2: v = &p.nd_dst; break;
      case 3: v = &p.corner_dst; break;
      case 4: v = &p.cross_dst; break;
      default: v = &meta; break;
    }
    n = static_cast<int>(v->size());
    if (out) std::memcpy(out, v->data(), sizeof(int) * std::min<size_t>(v->size(), static_cast<size_t>(std::max(cap, 0))));
  });
  return rc == DDELM_OK ? n : -rc;
}

int ddelm_gpu_get_shard(ddelm_ws* ws, int* sub_lo, int* sub_count, int* n_global) {
  return guarded([&] {
    if (!ws) throw std::invalid_argument("ddelm_gpu_get_shard: null handle");
    if (sub_lo) *sub_lo = ws->w->plan.sub_lo;
    if (sub_count) *sub_count = ws->w->plan.N;
    if (n_global) *n_global = ws->w->plan.N_global;
  });
}

void ddelm_gpu_destroy(ddelm_ws* ws) {
  if (!ws) return;
  delete ws->w;
  delete ws;
}

int ddelm_gpu_build(ddelm_ws* ws) {
  return guarded([&] { ws->w->build(); });
}
int ddelm_gpu_build_coarse(ddelm_ws* ws) {
  return guarded([&] { ws->w->build_coarse(); });
}
int ddelm_gpu_build_neumann(ddelm_ws* ws) {
  return guarded([&] { ws->w->build_neumann(); });
}

int ddelm_gpu_reseed(ddelm_ws* ws, uint64_t seed) {
  return guarded([&] { ws->w->reseed(seed); });
}

int ddelm_gpu_set_cg_blocks(ddelm_ws* ws, int mode) {
  return guarded([&] {
    if (mode != DDELM_CG_BLOCKS_COEFF && mode != DDELM_CG_BLOCKS_COMPACT)
      throw std::invalid_argument("set_cg_blocks: mode must be DDELM_CG_BLOCKS_COEFF or DDELM_CG_BLOCKS_COMPACT");
    ws->w->cg_compact = mode;
  });
}

int ddelm_gpu_solve(ddelm_ws* ws, int method, double theta, double rel_tol, int max_iter,
                    ddelm_report* rep) {
  return guarded([&] {
    ddg::SolveResult r = ws->w->solve(method, theta, rel_tol, max_iter);
    ddelm_report o{};
    const ddg::Plan& p = ws->w->plan;
    o.iterations = r.iterations;
    o.converged = r.converged ? 1 : 0;
    o.negative_curvature = r.negative_curvature ? 1 : 0;
    o.n_delta = p.n_delta;
    o.n_pi = p.n_pi;
    o.n_mu = p.n_delta + p.n_pi;
    o.n_subdomains = p.N;
    o.M = p.M;
    o.assembly_seconds = r.phase_ms[0] / 1e3;
    o.factorization_seconds = (r.phase_ms[1] + r.phase_ms[2]) / 1e3;
    o.setup_seconds = (r.phase_ms[3] + r.phase_ms[4] + r.phase_ms[5]) / 1e3;
    o.cg_seconds = r.phase_ms[6] / 1e3;
    o.reconstruct_seconds = r.phase_ms[7] / 1e3;
    o.total_seconds = r.host_ms / 1e3;
    ws->last = o;
    if (rep) *rep = o;
  });
}

int ddelm_gpu_get_mu(ddelm_ws* ws, double* mu) {
  return guarded([&] { ws->w->get_mu(mu); });
}
int ddelm_gpu_get_coeffs(ddelm_ws* ws, double* c) {
  return guarded([&] { ws->w->get_coeffs(c); });
}
int ddelm_gpu_sample_field(ddelm_ws* ws, int n, double* u, double* gx, double* gy) {
  return guarded([&] {
    double sums[4];
    ws->w->field(n, nullptr, u, gx, gy, sums);
  });
}
namespace {
/// relative L2 / H1 from the trapezoid sums (metrics.cpp:79-87)
void errors_from_sums(const double* s, double* l2, double* h1) {
  if (l2) *l2 = s[1] > 0 ? std::sqrt(s[0] / s[1]) : std::sqrt(s[0]);
  const double den = s[1] + s[3];
  if (h1) *h1 = den > 0 ? std::sqrt((s[0] + s[2]) / den) : std::sqrt(s[0] + s[2]);
}
}  // namespace
int ddelm_gpu_relative_errors(ddelm_ws* ws, int n, double* l2, double* h1) {
  return guarded([&] {
    if (n < 64) throw std::invalid_argument("relative_errors: evaluation grid too coarse");
    double sums[4];
    ws->w->field(n, nullptr, nullptr, nullptr, nullptr, sums);
    errors_from_sums(sums, l2, h1);
  });
}
int ddelm_gpu_field_diff(ddelm_ws* ws, int n, const double* ref_coeffs, double* l2, double* h1) {
  return guarded([&] {
    if (n < 64) throw std::invalid_argument("relative_errors: evaluation grid too coarse");
    if (ref_coeffs == nullptr) throw std::invalid_argument("field_diff: reference coefficients required");
    double sums[4];
    ws->w->field(n, ref_coeffs, nullptr, nullptr, nullptr, sums);
    errors_from_sums(sums, l2, h1);
  });
}
int ddelm_gpu_get_residuals(ddelm_ws* ws, double* h, int cap) {
  int n = 0;
  const int rc = guarded([&] { n = ws->w->get_residuals(h, cap); });
  return rc == DDELM_OK ? n : -rc;
}
int ddelm_gpu_get_ranks(ddelm_ws* ws, int* rk, int* rkb, double* ratio) {
  return guarded([&] { ws->w->get_ranks(rk, rkb, ratio); });
}
int ddelm_gpu_get_layer(ddelm_ws* ws, int i, double* w0, double* w1, double* b) {
  return guarded([&] {
    const ddg::Plan& p = ws->w->plan;
    if (i < 0 || i >= p.N) throw std::invalid_argument("ddelm_gpu_get_layer: bad subdomain");
    std::vector<double> a(p.M), c(p.M), e(p.M);
    ddg::init_layer(p, i, a.data(), c.data(), e.data());
    std::memcpy(w0, a.data(), sizeof(double) * p.M);
    std::memcpy(w1, c.data(), sizeof(double) * p.M);
    std::memcpy(b, e.data(), sizeof(double) * p.M);
  });
}
int ddelm_gpu_get_local(ddelm_ws* ws, int i, int which, double* K, int* rows) {
  return guarded([&] {
    const ddg::Plan& p = ws->w->plan;
    if (i < 0 || i >= p.N) throw std::invalid_argument("ddelm_gpu_get_local: bad subdomain");
    if (which < 0 || which > 2) throw std::invalid_argument("ddelm_gpu_get_local: which must be 0 (K), 1 (Kbar) or 2 (f)");
    if (rows) *rows = p.classes[p.subs[i].cls].m;  // this subdomain's rows (cc = 2: per class)
    if (K) ws->w->get_local(i, which, K);
  });
}
int ddelm_gpu_apply_operator(ddelm_ws* ws, double theta, const double* v, double* out) {
  return guarded([&] {
    if (theta < 0.0 || theta > 1.0) throw std::invalid_argument("theta must lie in [0, 1]");
    ws->w->apply_operator(theta, v, out);
  });
}
int ddelm_gpu_apply_reduced(ddelm_ws* ws, const double* v, double* out) {
  return guarded([&] { ws->w->apply_reduced(v, out); });
}
int ddelm_gpu_apply_neumann(ddelm_ws* ws, int transpose, const double* v, double* out) {
  return guarded([&] { ws->w->apply_neumann(transpose, v, out); });
}
int ddelm_gpu_dense_oracle(ddelm_ws* ws, int method, double theta, int* dim, double* reduced_op,
                           double* reduced_rhs, double* mu_full, double* coeffs) {
  return guarded([&] {
    ddg::DenseOracleOut o;
    ws->w->dense_oracle(method, theta, o);
    if (dim) *dim = o.dim;
    if (reduced_op) std::copy(o.reduced_op.begin(), o.reduced_op.end(), reduced_op);
    if (reduced_rhs) std::copy(o.reduced_rhs.begin(), o.reduced_rhs.end(), reduced_rhs);
    if (mu_full) std::copy(o.mu_full.begin(), o.mu_full.end(), mu_full);
    if (coeffs) std::copy(o.coeffs.begin(), o.coeffs.end(), coeffs);
  });
}
int ddelm_gpu_lsfactor_batch(int device, int nmat, int m, int n, const double* K, double rank_tol, int* rank,
                             int* deficient, int* reff, double* pinv, double* Q) {
  return guarded([&] {
    if (!K || !rank || !deficient || !pinv) throw std::invalid_argument("ddelm_gpu_lsfactor_batch: null argument");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
      throw ddg::CudaError("ddelm_gpu_lsfactor_batch: no CUDA device available (no CPU fallback)");
    if (device < 0 || device >= ndev) throw std::invalid_argument("ddelm_gpu_lsfactor_batch: bad device ordinal");
    DDG_CUDA(cudaSetDevice(device));
    cudaStream_t st;
    DDG_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    try {
      ddg::lsfactor_batch(nmat, m, n, K, rank_tol, rank, deficient, reff, pinv, Q, st);
    } catch (...) {
      cudaStreamDestroy(st);
      throw;
    }
    DDG_CUDA(cudaStreamDestroy(st));
  });
}
int ddelm_gpu_invalidate(ddelm_ws* ws) {
  return guarded([&] { ws->w->invalidate(); });
}
void* ddelm_gpu_stream(ddelm_ws* ws) { return static_cast<void*>(ws->w->stream()); }
int ddelm_gpu_set_profiling(ddelm_ws* ws, int on) {
  return guarded([&] { ws->w->set_profiling(on != 0); });
}
int ddelm_gpu_get_kernel_stats(ddelm_ws* ws, const char* family, double* total_ms, long long* launches,
                               double* flops, double* bytes) {
  return guarded([&] {
    ddg::KernelStat s;
    if (!ws->w->kernel_stat(family ? family : "", &s)) throw std::invalid_argument("no timings for that kernel family");
    if (total_ms) *total_ms = s.ms;
    if (launches) *launches = s.launches;
    if (flops) *flops = s.flops;
    if (bytes) *bytes = s.bytes;
  });
}
double ddelm_gpu_get_device_span_ms(ddelm_ws* ws) { return ws->w->device_span_ms(); }
int ddelm_gpu_get_phase_ms(ddelm_ws* ws, double* ms, int cap) {
  const double* src = ws->w->phase_ms();
  const int n = cap < 8 ? cap : 8;
  for (int k = 0; k < n; ++k) ms[k] = src[k];
  return n;
}
long long ddelm_gpu_get_launch_count(ddelm_ws* ws) { return ws->w->launches(); }


int ddelm_gpu_lsq_create(int nblocks, int m, int n, int k, int device, ddelm_lsq** out) {
  return guarded([&] {
    if (!out) throw std::invalid_argument("ddelm_gpu_lsq_create: null argument");
    *out = nullptr;
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
      throw ddg::CudaError("ddelm_gpu_lsq_create: no CUDA device available (no CPU fallback)");
    if (nblocks < 1 || n < 1 || k < 1 || m < n || (n % 2) || device < 0 || device >= ndev)
      throw std::invalid_argument("ddelm_gpu_lsq_create: need nblocks >= 1, m >= n >= 1 (n even), k >= 1");
    auto* L = new ddelm_lsq;
    std::unique_ptr<ddelm_lsq> guard(L);
    L->device = device;
    DDG_CUDA(cudaSetDevice(device));
    {
      int lo = 0, hi = 0;
      DDG_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
      DDG_CUDA(cudaStreamCreateWithPriority(&L->st, cudaStreamNonBlocking, hi));
      DDG_CUDA(cudaStreamCreateWithPriority(&L->side, cudaStreamNonBlocking, lo));
    }
    for (auto& e : L->ev) DDG_CUDA(cudaEventCreate(&e));
    L->a = ddg::LsqArgs{nblocks, m, n, k, (m + 3) / 4 * 4, n + k, nullptr, nullptr};
    const size_t nA = static_cast<size_t>(nblocks) * L->a.ld * L->a.ncol;
    DDG_CUDA(cudaMalloc(&L->a.A, nA * sizeof(double)));
    DDG_CUDA(cudaMemsetAsync(L->a.A, 0, nA * sizeof(double), L->st));
    DDG_CUDA(cudaMalloc(&L->a.S, static_cast<size_t>(nblocks) * k * k * sizeof(double)));
    DDG_CUDA(cudaMalloc(&L->tau, static_cast<size_t>(nblocks) * n * sizeof(double)));
    DDG_CUDA(cudaMalloc(&L->T, static_cast<size_t>(nblocks) * ddg::kQrTmax * ddg::kQrTmax * sizeof(double)));
    DDG_CUDA(cudaStreamSynchronize(L->st));
    *out = guard.release();
  });
}

int ddelm_gpu_lsq_generate(ddelm_lsq* L, uint64_t seed, int kind) {
  return guarded([&] {
    if (!L || kind < 0 || kind > 1) throw std::invalid_argument("ddelm_gpu_lsq_generate: bad argument");
    DDG_CUDA(cudaSetDevice(L->device));
    ddg::launch_lsq_generate(L->a, seed, kind, L->st);
    DDG_CUDA(cudaStreamSynchronize(L->st));
  });
}

int ddelm_gpu_lsq_factor(ddelm_lsq* L, double* qr_ms, double* schur_ms) {
  return guarded([&] {
    if (!L) throw std::invalid_argument("ddelm_gpu_lsq_factor: null handle");
    DDG_CUDA(cudaSetDevice(L->device));
    const ddg::LsqArgs& a = L->a;
    ddg::QrArgs q{a.nb, a.m, a.ld, a.ncol, a.n, a.A, L->tau, L->T};
    DDG_CUDA(cudaEventRecord(L->ev[0], L->st));
    ddg::qr_factor(q, L->st, L->side, L->qr_ev);
    DDG_CUDA(cudaEventRecord(L->ev[1], L->st));
    ddg::launch_lsq_gram(a, L->st);
    DDG_CUDA(cudaEventRecord(L->ev[2], L->st));
    DDG_CUDA(cudaStreamSynchronize(L->st));
    float t0 = 0, t1 = 0;
    DDG_CUDA(cudaEventElapsedTime(&t0, L->ev[0], L->ev[1]));
    DDG_CUDA(cudaEventElapsedTime(&t1, L->ev[1], L->ev[2]));
    if (qr_ms) *qr_ms = t0;
    if (schur_ms) *schur_ms = t1;
  });
}

int ddelm_gpu_lsq_get_block(ddelm_lsq* L, int b, double* A, double* tau, double* S) {
  return guarded([&] {
    if (!L || b < 0 || b >= L->a.nb) throw std::invalid_argument("ddelm_gpu_lsq_get_block: bad block");
    DDG_CUDA(cudaSetDevice(L->device));
    const ddg::LsqArgs& a = L->a;
    if (A)
      DDG_CUDA(cudaMemcpy(A, a.A + static_cast<size_t>(b) * a.ld * a.ncol,
                          static_cast<size_t>(a.ld) * a.ncol * sizeof(double), cudaMemcpyDeviceToHost));
    if (tau)
      DDG_CUDA(cudaMemcpy(tau, L->tau + static_cast<size_t>(b) * a.n, a.n * sizeof(double), cudaMemcpyDeviceToHost));
    if (S)
      DDG_CUDA(cudaMemcpy(S, a.S + static_cast<size_t>(b) * a.k * a.k, static_cast<size_t>(a.k) * a.k * sizeof(double),
                          cudaMemcpyDeviceToHost));
  });
}

int ddelm_gpu_lsq_ld(ddelm_lsq* L) { return L ? L->a.ld : 0; }

void ddelm_gpu_lsq_destroy(ddelm_lsq* L) { delete L; }

int ddelm_gpu_fp64_peak(int device, double* tflops) {
  return guarded([&] {
    if (!tflops) throw std::invalid_argument("ddelm_gpu_fp64_peak: null argument");
    *tflops = ddg::fp64_peak_probe(device);
  });
}

}  // extern "C"

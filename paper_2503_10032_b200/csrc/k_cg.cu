// Interface Krylov iteration of DDELM-NN on the device (sm_100a, fp64).
//
// cs_reduced_apply (solvers.cpp:372-386) with the theta-mixed Neumann-Neumann weight
// (solvers.cpp:599-603), in the reference's own grouping: K^+ is applied INTO coefficient space
// (c = K^+ phi, an M-vector) and the flux / Cdelta rows act on c afterwards
// (solvers.cpp:215-218, 240-241, 456, 469). With the factored pseudo-inverse K^+ = C Q_r^T
// (k_cod.cu) one operator application is, per subdomain i:
//   OP1   s = Q_G^T phi (+ Q_r^T f), corner parts t_i, psi_i = Zc v            (per subdomain)
//   OP2   mu|corners = Wmu [t; psi] ; c = C s - Ypi mu ; x_i = -F c            (streams C, F)
//   NN1   y = Cbar (Qbar^T (-x|flux)) ; tr_i = Cdelta y                        (streams Cbar, Cdelta)
//   NN2   y = Cdelta^T tl ; zz_i = Qbar (Cbar^T y)                             (streams Cdelta, Cbar)
//   OP3   w = theta P^T P x + (1-theta) x ; u_i = C^T (F^T w)                  (streams F, C)
//   OP4   nu|corners = S^{-1} t' ; d2 rows ; o_i = -phi + Q_G(...) + Zc^T d2   (per subdomain)
//   XR    Ap = o gathered over the two owners of each Delta index ; x, r update (CG)
// The coarse solve mu = S^{-1}(t + Dpp^T psi) and d1 = psi - Dpp mu are applied through the
// precomputed rows Wmu = [S^{-1} | S^{-1} Dpp^T] and Wd = [-Dpp S^{-1} | I - Dpp S^{-1} Dpp^T]
// (k_blocks.cu), so every work item evaluates the handful of coarse rows it needs from the
// gathered [t; psi] vector itself: no single-CTA coarse phase, no extra grid barrier.
//
// HBM streaming: the four dense phases read contiguous row slices (rows j0..j1 of C, F, Cbar,
// Cdelta — one work item = one subdomain part) through a 4-stage shared-memory ring filled by
// the TMA engine (cp.async.bulk + mbarrier complete_tx). Each chunk is consumed by a row-dot
// (t_j = A_j . x) followed by a column axpy (y += t_j B_j), both from shared memory. The first
// chunks of the next phase are issued before the grid barrier (the matrices are constant during
// the solve), and NN2 / OP3 walk their slices in reverse so they start on the lines NN1 / OP2
// left in L2.
//
// The whole CG loop (solvers.cpp:82-119) is ONE persistent cooperative kernel: 7 grid barriers per
// iteration, the CG scalars are sums of per-CTA / per-subdomain partials in a fixed order (no
// atomics: bitwise deterministic), the search direction is double-buffered so the p-update is
// fused into OP1. The same kernel, with a job code, applies the operator once (tests), forms the
// reduced right-hand side (solvers.cpp:542-551) and reconstructs the coefficients
// (solvers.cpp:565-577).
#include <cooperative_groups.h>

#include <algorithm>
#include <cfloat>

#include "common.cuh"
#include "kernels.hpp"

namespace cgs = cooperative_groups;

namespace ddg {

namespace {

constexpr int kThreads = 512;
constexpr int kWarps = kThreads / 32;
constexpr int kStages = 4;
constexpr int kStageBytes = 32768;
constexpr int kMaxColBlocks = 4;  // axpy width <= 4 * kThreads

// ---------------------------------------------------------------- mbarrier + bulk copy (TMA)
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
  } while (!done);
}

// ---------------------------------------------------------------- shared state of one CTA
struct Shared {
  double* ring;    // kStages x kStageBytes
  double* xa;      // row-dot operand (wamax)
  double* tbuf;    // row-dot results of one chunk (rpc_max)
  double* red;     // kThreads (axpy group partials)
  double* z;       // [t; psi] (nz)
  double* t2;      // t' (n_pi)
  double* v1;      // big per-subdomain vector (gmax / fmax / dmax)
  double* s0;      // rmax
  double* s1;      // rmax
  uint64_t* full;  // kStages mbarriers
};

__device__ __forceinline__ int wamax_of(const CgArgs& a) { return max(max(a.rmax, a.fmax), max(a.dmax, a.gmax)); }

__device__ __forceinline__ Shared carve(const CgArgs& a, uint64_t* bars) {
  extern __shared__ __align__(128) double smem[];
  Shared s;
  s.ring = smem;
  double* q = smem + kStages * (kStageBytes / 8);
  const int wa = wamax_of(a);
  s.xa = q;
  q += wa;
  s.tbuf = q;
  q += a.rpc_max;
  s.red = q;
  q += kThreads;
  s.z = q;
  q += a.n_pi + a.npf;
  s.t2 = q;
  q += max(a.n_pi, 1);
  s.v1 = q;
  q += wa;
  s.s0 = q;
  q += a.rmax;
  s.s1 = q;
  s.full = bars;
  return s;
}

// ---------------------------------------------------------------- streamed phases
enum StreamKind { kOp2 = 0, kNn1 = 1, kNn2 = 2, kOp3 = 3 };

/// Geometry of one work item's streams: A rows and B rows j0..j1 of subdomain i.
struct ItemGeo {
  const double* A;  // row j0 of A
  const double* B;  // row j0 of B (nullptr: row-dot only)
  int lda, ldb, rows, wa, wb;
  bool reverse;
};

__device__ __forceinline__ void part_rows(const CgArgs& a, int p, int& j0, int& j1) {
  const int chunk = (a.M + a.P - 1) / a.P;
  j0 = min(a.M, p * chunk);
  j1 = min(a.M, j0 + chunk);
}

__device__ __forceinline__ ItemGeo item_geo(const CgArgs& a, int kind, int i, int p, bool recon) {
  int j0, j1;
  part_rows(a, p, j0, j1);
  const ClassDims d = a.dims[a.sub_cls[i]];
  const size_t R = a.rmax;
  const double* Ck = a.C + (static_cast<size_t>(i) * a.M + j0) * R;
  const double* Cb = a.C + (static_cast<size_t>(a.N + i) * a.M + j0) * R;
  const double* Fi = a.F + (static_cast<size_t>(i) * a.M + j0) * a.ldF;
  const double* Di = a.Cd + (static_cast<size_t>(i) * a.M + j0) * a.ldC;
  ItemGeo g;
  g.rows = j1 - j0;
  switch (kind) {
    case kOp2:
      g = {Ck, recon ? nullptr : Fi, a.rmax, a.ldF, j1 - j0, a.rank[i], d.nF, false};
      break;
    case kNn1:
      g = {Cb, Di, a.rmax, a.ldC, j1 - j0, a.rank[a.N + i], d.nd, false};
      break;
    case kNn2:
      g = {Di, Cb, a.ldC, a.rmax, j1 - j0, d.nd, a.rank[a.N + i], true};
      break;
    default:
      g = {Fi, Ck, a.ldF, a.rmax, j1 - j0, d.nF, a.rank[i], true};
      break;
  }
  return g;
}

__device__ __forceinline__ int rows_per_chunk(const ItemGeo& g) {
  const int per_row = 8 * (g.lda + (g.B ? g.ldb : 0));
  return max(1, min(kStageBytes / per_row, 128));
}

/// Producer cursor over the chunks of this CTA's work items in one streamed phase (thread 0).
struct Producer {
  int kind, item, nitems, chunk, nchunks, rpc, issued, consumed;
  bool recon;
};

__device__ __forceinline__ int item_work(const CgArgs& a, int k, int nitems, bool reverse) {
  // item k of this CTA in traversal order; reverse phases walk items (and chunks) backwards
  const int kk = reverse ? nitems - 1 - k : k;
  return blockIdx.x + kk * gridDim.x;
}

__device__ __forceinline__ int n_items(const CgArgs& a, int nwork) {
  const int b = blockIdx.x, G = gridDim.x;
  return b < nwork ? (nwork - 1 - b) / G + 1 : 0;
}

__device__ void producer_begin(const CgArgs& a, Producer& pr, int kind, bool recon) {
  pr.kind = kind;
  pr.recon = recon;
  pr.nitems = n_items(a, a.N * a.P);
  pr.item = 0;
  pr.chunk = 0;
  pr.nchunks = -1;
  pr.issued = 0;
  pr.consumed = 0;
}

/// Issue the next chunk into stage (issued % kStages). Returns false when nothing is left.
__device__ bool producer_issue(const CgArgs& a, Producer& pr, const Shared& sh) {
  while (pr.item < pr.nitems) {
    const bool rev = (pr.kind == kNn2 || pr.kind == kOp3);
    const int w = item_work(a, pr.item, pr.nitems, rev);
    const ItemGeo g = item_geo(a, pr.kind, w / a.P, w % a.P, pr.recon);
    const int rpc = rows_per_chunk(g);
    const int nch = (g.rows + rpc - 1) / rpc;
    if (pr.chunk >= nch) {
      ++pr.item;
      pr.chunk = 0;
      continue;
    }
    const int c = g.reverse ? nch - 1 - pr.chunk : pr.chunk;
    const int ja = c * rpc, nr = min(rpc, g.rows - ja);
    const int st = pr.issued % kStages;
    double* dst = sh.ring + static_cast<size_t>(st) * (kStageBytes / 8);
    const uint32_t ba = static_cast<uint32_t>(nr) * g.lda * 8;
    const uint32_t bb = g.B ? static_cast<uint32_t>(nr) * g.ldb * 8 : 0;
    mbar_expect_tx(&sh.full[st], ba + bb);
    bulk_g2s(dst, g.A + static_cast<size_t>(ja) * g.lda, ba, &sh.full[st]);
    if (g.B) bulk_g2s(dst + static_cast<size_t>(nr) * g.lda, g.B + static_cast<size_t>(ja) * g.ldb, bb, &sh.full[st]);
    ++pr.chunk;
    ++pr.issued;
    return true;
  }
  return false;
}

__device__ __forceinline__ void producer_fill(const CgArgs& a, Producer& pr, const Shared& sh) {
  while (pr.issued - pr.consumed < kStages && producer_issue(a, pr, sh)) {
  }
}

/// Consumer side of one work item: stream the rows of (A, B); per row j: t_j = A_j . xa, then
/// hook(j, t_j) (returns the value used by the axpy), acc += t_j * B_j.  acc[] per thread column.
/// `seq` / `phase` track the ring position and mbarrier parities (uniform over the CTA).
template <class Hook>
__device__ void stream_item(const CgArgs& a, const ItemGeo& g, const Shared& sh, Producer& pr, int& seq,
                            uint32_t& phase, double* acc, Hook hook) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int rpc = rows_per_chunk(g);
  const int nch = (g.rows + rpc - 1) / rpc;
  const int ncb = g.B ? (g.wb + kThreads - 1) / kThreads : 0;
  const int wbp = (ncb == 1) ? ((g.wb + 31) & ~31) : kThreads;
  const int G = (ncb == 1) ? kThreads / wbp : 1;
  const int col = threadIdx.x % wbp, grp = threadIdx.x / wbp;
  for (int cc = 0; cc < nch; ++cc) {
    const int c = g.reverse ? nch - 1 - cc : cc;
    const int ja = c * rpc, nr = min(rpc, g.rows - ja);
    const int st = seq % kStages;
    const double* As = sh.ring + static_cast<size_t>(st) * (kStageBytes / 8);
    const double* Bs = As + static_cast<size_t>(nr) * g.lda;
    mbar_wait(&sh.full[st], (phase >> st) & 1u);
    phase ^= 1u << st;
    for (int rr = warp; rr < nr; rr += kWarps) {
      const double* ar = As + static_cast<size_t>(rr) * g.lda;
      double s = 0;
      for (int k = lane; k < g.wa; k += 32) s += ar[k] * sh.xa[k];
      s = warp_sum(s);
      if (lane == 0) sh.tbuf[rr] = hook(ja + rr, s);
    }
    __syncthreads();
    if (ncb > 0 && grp < G) {
      for (int cb = 0; cb < ncb; ++cb) {
        const int l = col + cb * kThreads;
        if (l < g.wb) {
          double s = acc[cb];
          for (int rr = grp; rr < nr; rr += G) s += Bs[static_cast<size_t>(rr) * g.ldb + l] * sh.tbuf[rr];
          acc[cb] = s;
        }
      }
    }
    __syncthreads();  // stage st free, tbuf reusable
    ++seq;
    if (threadIdx.x == 0) {
      ++pr.consumed;
      producer_fill(a, pr, sh);
    }
  }
}

/// Reduce the axpy accumulators over the row groups (fixed order) and hand out column l values.
template <class Out>
__device__ void reduce_acc(const ItemGeo& g, const Shared& sh, double* acc, Out out) {
  const int ncb = (g.wb + kThreads - 1) / kThreads;
  const int wbp = (ncb == 1) ? ((g.wb + 31) & ~31) : kThreads;
  const int G = (ncb == 1) ? kThreads / wbp : 1;
  const int col = threadIdx.x % wbp, grp = threadIdx.x / wbp;
  for (int cb = 0; cb < ncb; ++cb) {
    sh.red[threadIdx.x] = (grp < G) ? acc[cb] : 0.0;
    __syncthreads();
    if (grp == 0) {
      const int l = col + cb * kThreads;
      if (l < g.wb) {
        double s = 0;
        for (int q = 0; q < G; ++q) s += sh.red[q * wbp + col];
        out(l, s);
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- small helpers
__device__ __forceinline__ double sum_parts(const double* base, size_t stride, int P, int idx) {
  double s = 0;
  for (int p = 0; p < P; ++p) s += base[p * stride + idx];
  return s;
}

__device__ __forceinline__ double gather_x(const CgArgs& a, int g) {
  const size_t st = static_cast<size_t>(a.N) * a.fmax;
  return a.flip_sign[g] *
         (sum_parts(a.xf, st, a.P, a.own_flux[2 * g]) + sum_parts(a.xf, st, a.P, a.own_flux[2 * g + 1]));
}

/// z = [t; psi]: corner contributions of OP1 summed over their owners (subdomain order) and the
/// cross-flux data psi (mode 0: Dpd v; mode 1: dpi; mode 2: dpi - Dpd mu_Delta).
__device__ void gather_z(const CgArgs& a, const Shared& sh, int mode) {
  const int n = a.n_pi;
  for (int gp = threadIdx.x; gp < n; gp += blockDim.x) {
    double acc = 0;
    for (int q = 0; q < 4; ++q) {
      const int o = a.pi_owner[gp * 4 + q];
      if (o >= 0) acc += a.tpart[o];
    }
    sh.z[gp] = acc;
  }
  for (int rr = threadIdx.x; rr < a.npf; rr += blockDim.x) {
    double acc = 0;
    if (mode != 1)
      for (int q = 0; q < 4; ++q) {
        const int o = a.row_owner[rr * 4 + q];
        if (o >= 0) acc += a.psipart[o];
      }
    sh.z[n + rr] = (mode == 0) ? acc : (mode == 1 ? a.dpi[rr] : a.dpi[rr] - acc);
  }
}

/// out[q] = W[row_q] . vec (len), one warp per row; rows < 0 give 0.
__device__ void rows_dot(const double* W, int ldw, const int* rows, int nrows, const double* vec, int len,
                         double* out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int q = warp; q < nrows; q += kWarps) {
    const int row = rows[q];
    double s = 0;
    if (row >= 0) {
      const double* w = W + static_cast<size_t>(row) * ldw;
      for (int k = lane; k < len; k += 32) s += w[k] * vec[k];
    }
    s = warp_sum(s);
    if (lane == 0) out[q] = s;
  }
}

// ---------------------------------------------------------------- OP1 (per subdomain)
/// mode 0: operator on v (CG: v = r + beta p_cur, written to p_next by the first owner);
/// mode 1: reduced right-hand side (phi = 0, + Q_r^T f); mode 2: reconstruction (phi = +v).
__device__ void dev_op1(const CgArgs& a, const Shared& sh, int i, const double* v, int mode, bool cg,
                        double beta, const double* pcur, double* pnext) {
  const ClassDims d = a.dims[a.sub_cls[i]];
  const int r = a.rank[i], R = a.rmax, E = a.ext;
  const double* QtX = a.QtX + static_cast<size_t>(i) * R * E;
  double* vg = sh.v1;
  double* phi = sh.red;  // n_gamma <= kThreads (checked on the host)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int* gd = a.gamma_delta + static_cast<size_t>(i) * a.gmax;
  for (int g = threadIdx.x; g < d.n_gamma; g += blockDim.x) {
    const int dg = gd[g];
    double vv = 0.0;
    if (dg >= 0 && mode != 1) {
      if (cg) {
        vv = a.r[dg] + beta * pcur[dg];
        if (a.own_gamma[2 * dg] == i * a.gmax + g) pnext[dg] = vv;
      } else {
        vv = v[dg];
      }
    }
    vg[g] = vv;
    phi[g] = (mode == 0) ? -vv : vv;
  }
  __syncthreads();
  for (int k = warp; k < r; k += kWarps) {
    const double* q = QtX + static_cast<size_t>(k) * E + 1;
    double acc = 0;
    if (mode != 1)
      for (int g = lane; g < d.n_gamma; g += 32) acc += q[g] * phi[g];
    acc = warp_sum(acc);
    if (mode >= 1) acc += QtX[static_cast<size_t>(k) * E];
    if (lane == 0) {
      sh.s0[k] = acc;
      a.s[static_cast<size_t>(i) * R + k] = acc;
    }
  }
  __syncthreads();
  if (warp < 4) {
    const int g = a.corner_q[i * 4 + warp];
    double acc = 0;
    if (g >= 0)
      for (int k = lane; k < r; k += 32) acc += QtX[static_cast<size_t>(k) * E + 1 + g] * sh.s0[k];
    acc = warp_sum(acc);
    if (lane == 0) a.tpart[i * 4 + warp] = acc;  // t(gp) -= phi - Ky at the corners (phi = 0 there)
  } else if (mode != 1) {
    // psi_i = Zc v (Dpd rows restricted to this subdomain), warps 4..
    const double* Zc = a.Zc + static_cast<size_t>(i) * a.crmax * a.gmax;
    for (int rho = warp - 4; rho < a.crmax; rho += kWarps - 4) {
      double acc = 0;
      for (int g = lane; g < d.n_gamma; g += 32) acc += Zc[static_cast<size_t>(rho) * a.gmax + g] * vg[g];
      acc = warp_sum(acc);
      if (lane == 0) a.psipart[static_cast<size_t>(i) * a.crmax + rho] = acc;
    }
  }
  __syncthreads();
}

// ---------------------------------------------------------------- OP2 (streams C, F)
__device__ void dev_op2(const CgArgs& a, const Shared& sh, Producer& pr, int& seq, uint32_t& phase, int mode) {
  const int nitems = n_items(a, a.N * a.P);
  __shared__ double muc[4];
  __shared__ int crow[4];
  for (int k = 0; k < nitems; ++k) {
    const int w = item_work(a, k, nitems, false);
    const int i = w / a.P, p = w % a.P;
    gather_z(a, sh, mode);
    if (threadIdx.x < 4) {
      const int g = a.corner_q[i * 4 + threadIdx.x];
      crow[threadIdx.x] = g >= 0 ? a.gamma_pi[static_cast<size_t>(i) * a.gmax + g] : -1;
    }
    const int r = a.rank[i];
    for (int kk = threadIdx.x; kk < r; kk += blockDim.x) sh.xa[kk] = a.s[static_cast<size_t>(i) * a.rmax + kk];
    __syncthreads();
    rows_dot(a.Wmu, a.n_pi + a.npf, crow, 4, sh.z, a.n_pi + a.npf, muc);  // mu = S^{-1}(t + Dpp^T psi)
    if (mode == 2 && w == 0)  // mu_Pi of the solution (one CTA writes it)
      for (int gp = threadIdx.x >> 5; gp < a.n_pi; gp += kWarps) {
        double s = 0;
        const double* wr = a.Wmu + static_cast<size_t>(gp) * (a.n_pi + a.npf);
        for (int kk = threadIdx.x & 31; kk < a.n_pi + a.npf; kk += 32) s += wr[kk] * sh.z[kk];
        s = warp_sum(s);
        if ((threadIdx.x & 31) == 0) a.mu_pi_out[gp] = s;
      }
    __syncthreads();
    const ItemGeo g = item_geo(a, kOp2, i, p, mode == 2);
    int j0, j1;
    part_rows(a, p, j0, j1);
    const double* Yp = a.Ypi + static_cast<size_t>(i) * a.M * 4;
    double* coef = a.coeffs + static_cast<size_t>(i) * a.M;
    double acc[kMaxColBlocks] = {0, 0, 0, 0};
    // reference grouping (solvers.cpp:336, 342): c = K^+ phi - Ypi mu, then F c
    stream_item(a, g, sh, pr, seq, phase, acc, [&](int jr, double cs) {
      const int j = j0 + jr;
      double yp = 0;
      for (int q = 0; q < 4; ++q) yp += Yp[static_cast<size_t>(j) * 4 + q] * muc[q];
      const double cj = cs - yp;
      if (mode == 2) coef[j] = cj;
      return cj;
    });
    if (mode == 2) continue;
    double* xf = a.xf + (static_cast<size_t>(p) * a.N + i) * a.fmax;
    reduce_acc(g, sh, acc, [&](int l, double s) { xf[l] = -s; });
  }
}

// ---------------------------------------------------------------- NN1 (streams Cbar, Cdelta)
__device__ void dev_nn1(const CgArgs& a, const Shared& sh, Producer& pr, int& seq, uint32_t& phase) {
  const int nitems = n_items(a, a.N * a.P);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int k = 0; k < nitems; ++k) {
    const int w = item_work(a, k, nitems, false);
    const int i = w / a.P, p = w % a.P;
    const ClassDims d = a.dims[a.sub_cls[i]];
    const int nd = d.nd, rb = a.rank[a.N + i], E = a.ext;
    const double* QtX = a.QtX + static_cast<size_t>(a.N + i) * a.rmax * E;
    const int* nmap = a.ndelta_map + static_cast<size_t>(i) * a.dmax;
    for (int kk = threadIdx.x; kk < nd; kk += blockDim.x) sh.v1[kk] = -gather_x(a, nmap[kk]);
    __syncthreads();
    for (int kk = warp; kk < rb; kk += kWarps) {  // Qbar_r^T rhs (rhs nonzero on the flux rows only)
      const double* q = QtX + static_cast<size_t>(kk) * E + 1;
      double s = 0;
      for (int e = lane; e < nd; e += 32) s += q[e] * sh.v1[e];
      s = warp_sum(s);
      if (lane == 0) sh.xa[kk] = s;
    }
    __syncthreads();
    const ItemGeo g = item_geo(a, kNn1, i, p, false);
    double acc[kMaxColBlocks] = {0, 0, 0, 0};
    // reference order (solvers.cpp:455): y = Kbar^+ rhs (M-vector), then Cdelta y
    stream_item(a, g, sh, pr, seq, phase, acc, [](int, double cs) { return cs; });
    double* tr = a.tr + (static_cast<size_t>(p) * a.N + i) * a.dmax;
    reduce_acc(g, sh, acc, [&](int l, double s) { tr[l] = s; });
  }
}

// ---------------------------------------------------------------- NN2 (streams Cdelta, Cbar)
__device__ void dev_nn2(const CgArgs& a, const Shared& sh, Producer& pr, int& seq, uint32_t& phase) {
  const int nitems = n_items(a, a.N * a.P);
  for (int k = 0; k < nitems; ++k) {
    const int w = item_work(a, k, nitems, true);
    const int i = w / a.P, p = w % a.P;
    const ClassDims d = a.dims[a.sub_cls[i]];
    const int nd = d.nd, rb = a.rank[a.N + i], E = a.ext;
    const double* QtX = a.QtX + static_cast<size_t>(a.N + i) * a.rmax * E;
    const int* nmap = a.ndelta_map + static_cast<size_t>(i) * a.dmax;
    const size_t st = static_cast<size_t>(a.N) * a.dmax;
    for (int kk = threadIdx.x; kk < nd; kk += blockDim.x) {
      const int gg = nmap[kk];
      sh.xa[kk] = sum_parts(a.tr, st, a.P, a.own_nd[2 * gg]) + sum_parts(a.tr, st, a.P, a.own_nd[2 * gg + 1]);
    }
    __syncthreads();
    const ItemGeo g = item_geo(a, kNn2, i, p, false);
    double acc[kMaxColBlocks] = {0, 0, 0, 0};
    // reference order (solvers.cpp:468): x = Cdelta^T tl (M-vector), then (Kbar^+)^T x
    stream_item(a, g, sh, pr, seq, phase, acc, [](int, double cs) { return cs; });
    reduce_acc(g, sh, acc, [&](int l, double s) { sh.s0[l] = s; });
    __syncthreads();
    // zz = Qbar_r (Cbar^T x) on the flux rows (partial over the parts p; linear)
    double* zz = a.zz + (static_cast<size_t>(p) * a.N + i) * a.dmax;
    for (int kk = threadIdx.x; kk < nd; kk += blockDim.x) {
      double s = 0;
      for (int q = 0; q < rb; ++q) s += QtX[static_cast<size_t>(q) * E + 1 + kk] * sh.s0[q];
      zz[kk] = s;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- OP3 (streams F, C)
__device__ void dev_op3(const CgArgs& a, const Shared& sh, Producer& pr, int& seq, uint32_t& phase) {
  const int nitems = n_items(a, a.N * a.P);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int k = 0; k < nitems; ++k) {
    const int w = item_work(a, k, nitems, true);
    const int i = w / a.P, p = w % a.P;
    const ClassDims d = a.dims[a.sub_cls[i]];
    const int r = a.rank[i], R = a.rmax, E = a.ext;
    const double* QtX = a.QtX + static_cast<size_t>(i) * R * E;
    const int* fd = a.fluxrow_delta + static_cast<size_t>(i) * a.fmax;
    const double theta = a.theta;
    const size_t st = static_cast<size_t>(a.N) * a.dmax;
    for (int l = threadIdx.x; l < d.nF; l += blockDim.x) {
      const int gg = fd[l];
      double wv = 0.0;
      if (gg >= 0) {
        const double x = gather_x(a, gg);
        if (a.use_neumann) {
          const double ptp =
              -(sum_parts(a.zz, st, a.P, a.own_nd[2 * gg]) + sum_parts(a.zz, st, a.P, a.own_nd[2 * gg + 1]));
          wv = theta * ptp;
          if (theta < 1.0) wv += (1.0 - theta) * x;
        } else {
          wv = x;
        }
      }
      sh.xa[l] = wv;  // apply_AT_delta: a(lrow) = w(grow) on the Delta flux rows
    }
    __syncthreads();
    const ItemGeo g = item_geo(a, kOp3, i, p, false);
    double acc[kMaxColBlocks] = {0, 0, 0, 0};
    // reference order: at = F^T a (M-vector, apply_AT), then (K^+)^T at = Q_r (C^T at)
    stream_item(a, g, sh, pr, seq, phase, acc, [](int, double cs) { return cs; });
    double* up = a.u + (static_cast<size_t>(p) * a.N + i) * R;
    reduce_acc(g, sh, acc, [&](int l, double s) {
      up[l] = s;
      sh.s0[l] = s;
    });
    __syncthreads();
    if (warp < 4) {
      const int gq = a.corner_q[i * 4 + warp];
      double acc2 = 0;
      if (gq >= 0)
        for (int kk = lane; kk < r; kk += 32) acc2 += QtX[static_cast<size_t>(kk) * E + 1 + gq] * sh.s0[kk];
      acc2 = warp_sum(acc2);
      if (lane == 0) a.tpart3[(static_cast<size_t>(p) * a.N + i) * 4 + warp] = acc2;  // t(gp) += z(lr)
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- OP4 (per subdomain)
/// o_i = -phi + Q_G (s~ + u + Q_Pi^T nu) + Zc^T d2 ; CG mode also returns p . o_i.
__device__ double dev_op4(const CgArgs& a, const Shared& sh, int i, const double* v, int mode) {
  const ClassDims d = a.dims[a.sub_cls[i]];
  const int r = a.rank[i], R = a.rmax, E = a.ext, n = a.n_pi, nz = a.n_pi + a.npf;
  const double* QtX = a.QtX + static_cast<size_t>(i) * R * E;
  __shared__ double cq_mu[4], cq_nu[4], d2s[64], w3t[64];
  __shared__ int crow[4], xrow[64];
  gather_z(a, sh, mode);
  const size_t st3 = static_cast<size_t>(a.N) * 4;
  for (int gp = threadIdx.x; gp < n; gp += blockDim.x) {
    double acc = 0;
    for (int q = 0; q < 4; ++q) {
      const int o = a.pi_owner[gp * 4 + q];
      if (o >= 0) acc += sum_parts(a.tpart3, st3, a.P, o);
    }
    sh.t2[gp] = acc;
  }
  if (threadIdx.x < 4) {
    const int g = a.corner_q[i * 4 + threadIdx.x];
    crow[threadIdx.x] = g >= 0 ? a.gamma_pi[static_cast<size_t>(i) * a.gmax + g] : -1;
  }
  for (int rho = threadIdx.x; rho < a.crmax; rho += blockDim.x)
    xrow[rho] = a.cr_row[static_cast<size_t>(i) * a.crmax + rho];
  __syncthreads();
  rows_dot(a.Wmu, nz, crow, 4, sh.z, nz, cq_mu);       // mu  = S^{-1}(t + Dpp^T psi)
  rows_dot(a.Sinv, n, crow, 4, sh.t2, n, cq_nu);       // nu  = S^{-1} t'
  rows_dot(a.Wd, nz, xrow, a.crmax, sh.z, nz, d2s);    // d1  = psi - Dpp mu
  rows_dot(a.W3, n, xrow, a.crmax, sh.t2, n, w3t);     // Dpp nu
  __syncthreads();
  for (int rho = threadIdx.x; rho < a.crmax; rho += blockDim.x) d2s[rho] = xrow[rho] >= 0 ? d2s[rho] - w3t[rho] : 0.0;
  int gq[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) gq[q] = a.corner_q[i * 4 + q];
  const size_t ust = static_cast<size_t>(a.N) * R;
  for (int k = threadIdx.x; k < r; k += blockDim.x) {
    double uu = sum_parts(a.u + static_cast<size_t>(i) * R, ust, a.P, k);
    double sk = a.s[static_cast<size_t>(i) * R + k];
    for (int q = 0; q < 4; ++q)
      if (gq[q] >= 0) {
        const double qk = QtX[static_cast<size_t>(k) * E + 1 + gq[q]];
        uu += qk * cq_nu[q];
        sk += qk * cq_mu[q];  // s~ = s + Q_Pi^T mu
      }
    sh.s0[k] = sk + uu;  // s~ + u + Q_Pi^T nu
  }
  __syncthreads();
  const int* gd = a.gamma_delta + static_cast<size_t>(i) * a.gmax;
  const double* Zc = a.Zc + static_cast<size_t>(i) * a.crmax * a.gmax;
  double dot = 0;
  for (int g = threadIdx.x; g < d.n_gamma; g += blockDim.x) {
    const int dg = gd[g];
    if (dg < 0) continue;
    double qs = 0;
    for (int k = 0; k < r; ++k) qs += QtX[static_cast<size_t>(k) * E + 1 + g] * sh.s0[k];
    double zs = 0;
    for (int rho = 0; rho < a.crmax; ++rho) zs += Zc[static_cast<size_t>(rho) * a.gmax + g] * d2s[rho];
    const double mphi = (mode == 0) ? v[dg] : 0.0;  // -phi
    const double o = mphi + qs + zs;
    a.o[static_cast<size_t>(i) * a.gmax + g] = o;
    if (mode == 0) dot += v[dg] * o;
  }
  dot = block_sum(dot, sh.red);
  return dot;
}

__device__ __forceinline__ double gather_out(const CgArgs& a, int g) {
  return a.o[a.own_gamma[2 * g]] + a.o[a.own_gamma[2 * g + 1]];
}

// ---------------------------------------------------------------- the persistent kernel
__device__ void drain(Producer& pr, const Shared& sh, int& seq, uint32_t& phase) {
  // wait for chunks issued ahead (next-phase prefetch) before leaving: no bulk copy may land in
  // the shared memory of an exited CTA
  __shared__ int s_pending;
  if (threadIdx.x == 0) s_pending = pr.issued - pr.consumed;
  __syncthreads();
  for (int k = 0; k < s_pending; ++k) {
    const int st = (seq + k) % kStages;
    mbar_wait(&sh.full[st], (phase >> st) & 1u);
    phase ^= 1u << st;
  }
  __syncthreads();
}

__global__ void __launch_bounds__(kThreads, 1) cg_persistent_kernel(CgArgs a, int job, const double* vin,
                                                                    double* vout) {
  cgs::grid_group grid = cgs::this_grid();
  const int G = gridDim.x, b = blockIdx.x;
  __shared__ __align__(8) uint64_t bars[kStages];
  __shared__ double bsum[32];
  const Shared sh = carve(a, bars);
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&bars[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  Producer pr;  // meaningful on thread 0 only
  int seq = 0;
  uint32_t phase = 0;

  auto begin_stream = [&](int kind, bool recon) {
    // issue the first chunks of the next streamed phase (ring is free here)
    seq = 0;
    if (threadIdx.x == 0) {
      producer_begin(a, pr, kind, recon);
      producer_fill(a, pr, sh);
    }
  };

  if (job == kJobRecon) {
    begin_stream(kOp2, true);
    for (int i = b; i < a.N; i += G) dev_op1(a, sh, i, vin, 2, false, 0.0, nullptr, nullptr);
    grid.sync();
    dev_op2(a, sh, pr, seq, phase, 2);
    drain(pr, sh, seq, phase);
    return;
  }

  if (job == kJobApply || job == kJobRhs) {
    const int mode = job == kJobApply ? 0 : 1;
    begin_stream(kOp2, false);
    for (int i = b; i < a.N; i += G) dev_op1(a, sh, i, vin, mode, false, 0.0, nullptr, nullptr);
    grid.sync();
    dev_op2(a, sh, pr, seq, phase, mode);
    if (a.use_neumann) {
      begin_stream(kNn1, false);
      grid.sync();
      dev_nn1(a, sh, pr, seq, phase);
      begin_stream(kNn2, false);
      grid.sync();
      dev_nn2(a, sh, pr, seq, phase);
    }
    begin_stream(kOp3, false);
    grid.sync();
    dev_op3(a, sh, pr, seq, phase);
    grid.sync();
    for (int i = b; i < a.N; i += G) dev_op4(a, sh, i, vin, mode);
    grid.sync();
    for (int g = b * blockDim.x + threadIdx.x; g < a.n_delta; g += G * blockDim.x) vout[g] = gather_out(a, g);
    return;
  }

  // ---- CG (solvers.cpp:93-116): x0 = 0, r = p = b (cg_init), recursive residual
  double rr = a.scal[0];
  const double bnorm = a.scal[1];
  if (a.state[1]) return;  // rhs == 0
  double beta = 0.0;
  begin_stream(kOp2, false);
  for (int it = 1;; ++it) {
    double* pcur = a.pbuf[(it - 1) & 1];
    double* pnext = a.pbuf[it & 1];
    for (int i = b; i < a.N; i += G) dev_op1(a, sh, i, nullptr, 0, true, beta, pcur, pnext);
    grid.sync();
    dev_op2(a, sh, pr, seq, phase, 0);
    if (a.use_neumann) {
      begin_stream(kNn1, false);
      grid.sync();
      dev_nn1(a, sh, pr, seq, phase);
      begin_stream(kNn2, false);
      grid.sync();
      dev_nn2(a, sh, pr, seq, phase);
    }
    begin_stream(kOp3, false);
    grid.sync();
    dev_op3(a, sh, pr, seq, phase);
    begin_stream(kOp2, false);  // next iteration's OP2 chunks, behind OP4 / XR / OP1
    grid.sync();
    for (int i = b; i < a.N; i += G) {
      const double dot = dev_op4(a, sh, i, pnext, 0);
      if (threadIdx.x == 0) a.pap[i] = dot;
    }
    grid.sync();
    // pAp = sum over subdomains of p . o_i (fixed order), alpha, x / r update
    double pAp = 0;
    for (int i = 0; i < a.N; ++i) pAp += a.pap[i];
    if (pAp <= 0.0) {  // solvers.cpp:97-103
      if (b == 0 && threadIdx.x == 0) {
        a.state[3] = pAp < 0.0 ? 1 : 0;
        a.state[5] = it - 1;
        a.state[1] = 1;
      }
      break;
    }
    const double alpha = rr / pAp;
    double dsum = 0;
    for (int g = b * blockDim.x + threadIdx.x; g < a.n_delta; g += G * blockDim.x) {
      const double ap = gather_out(a, g);
      a.x[g] += alpha * pnext[g];
      const double rg = a.r[g] - alpha * ap;
      a.r[g] = rg;
      dsum += rg * rg;
    }
    dsum = block_sum(dsum, bsum);
    if (threadIdx.x == 0) a.partial[b] = dsum;
    grid.sync();
    double rr_new = 0;
    for (int k = 0; k < G; ++k) rr_new += a.partial[k];
    const double rel = sqrt(rr_new) / bnorm;
    if (b == 0 && threadIdx.x == 0) {
      a.hist[it - 1] = rel;
      a.state[5] = it;
    }
    if (rel <= a.rel_tol || it >= a.max_iter) {
      if (b == 0 && threadIdx.x == 0) {
        a.state[1] = 1;
        a.state[2] = rel <= a.rel_tol ? 1 : 0;
      }
      break;
    }
    beta = rr_new / rr;
    rr = rr_new;
    // a.partial is rewritten only after two more grid barriers: no race with the reads above
  }
  drain(pr, sh, seq, phase);
}

__global__ void __launch_bounds__(256) cg_init_kernel(CgArgs a) {
  __shared__ double red[32];
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  double d = 0;
  if (g < a.n_delta) {
    const double b = a.rhs[g];
    a.x[g] = 0.0;
    a.r[g] = b;
    a.pbuf[0][g] = b;
    d = b * b;
  }
  d = block_sum(d, red);
  if (threadIdx.x == 0) a.partial[blockIdx.x] = d;
}

__global__ void cg_init2_kernel(CgArgs a, int nblk) {
  if (threadIdx.x != 0) return;
  double rr = 0;
  for (int k = 0; k < nblk; ++k) rr += a.partial[k];
  a.scal[0] = rr;
  a.scal[1] = sqrt(rr);
  for (int k = 0; k < 8; ++k) a.state[k] = 0;
  if (rr == 0.0) {
    a.state[1] = 1;  // bnorm == 0: converged with x = 0 (solvers.cpp:89-92)
    a.state[2] = 1;
  }
}

size_t smem_bytes(const CgArgs& a) {
  const int wa = std::max(std::max(a.rmax, a.fmax), std::max(a.dmax, a.gmax));
  const size_t small = static_cast<size_t>(wa) + a.rpc_max + kThreads + a.n_pi + a.npf + std::max(a.n_pi, 1) + wa +
                       2 * static_cast<size_t>(a.rmax);
  return static_cast<size_t>(kStages) * kStageBytes + sizeof(double) * small;
}

}  // namespace

int cg_grid(const CgArgs& a) {
  int dev = 0, sms = 0, per_sm = 0;
  DDG_CUDA(cudaGetDevice(&dev));
  DDG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const size_t sm = smem_bytes(a);
  DDG_CUDA(cudaFuncSetAttribute(cg_persistent_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(sm)));
  DDG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, cg_persistent_kernel, kThreads, sm));
  if (per_sm < 1) throw CudaError("cg_persistent_kernel cannot be resident (occupancy 0)");
  return sms;  // one CTA per SM
}

void cg_check_capacity(const CgArgs& a) {
  // shapes the kernel's shared-memory carve-up and thread mapping assume
  const int gmax = a.gmax, wb = std::max(std::max(a.rmax, a.fmax), a.dmax);
  if (gmax > kThreads || a.crmax > 64 || wb > kMaxColBlocks * kThreads)
    throw std::invalid_argument("interface block sizes exceed the CG kernel's capacity");
  if ((a.rmax & 1) || (a.ldF & 1) || (a.ldC & 1))
    throw std::logic_error("CG row strides must be even (16-byte bulk copies)");
  if (8 * (a.rmax + std::max(a.ldF, a.ldC)) > kStageBytes)
    throw std::invalid_argument("one coefficient row exceeds a CG pipeline stage");
}

int cg_rows_per_chunk_max(const CgArgs& a) {
  auto rpc = [](int lda, int ldb) { return std::max(1, std::min(kStageBytes / (8 * (lda + ldb)), 128)); };
  return std::max({rpc(a.rmax, a.ldF), rpc(a.rmax, a.ldC), rpc(a.rmax, 0)});
}

void cg_launch(const CgArgs& a, int job, const double* vin, double* vout, cudaStream_t st) {
  cg_check_capacity(a);
  const int G = cg_grid(a);
  const size_t sm = smem_bytes(a);
  CgArgs arg = a;
  void* params[] = {&arg, &job, &vin, &vout};
  DDG_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(cg_persistent_kernel), dim3(G), dim3(kThreads),
                                       params, sm, st));
}

void cg_launch_init(const CgArgs& a, cudaStream_t st) {
  const int nblk = ceil_div(a.n_delta, 256);
  cg_init_kernel<<<nblk, 256, 0, st>>>(a);
  cg_init2_kernel<<<1, 32, 0, st>>>(a, nblk);
  DDG_LAUNCH_CHECK();
}

}  // namespace ddg

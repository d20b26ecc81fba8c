// Interface Krylov iteration of DDELM-NN on the device (sm_100a, fp64).
//
// cs_reduced_apply (solvers.cpp:372-386) with the theta-mixed Neumann-Neumann weight
// (solvers.cpp:599-603), expressed on the interface-level blocks of k_blocks.cu:
//   s    = Q_G^T phi (+ Q_r^T f)          phi = B_Delta v   (local, op1)
//   mu   = S^{-1}(t + Dpp^T psi)          coarse solve     (one CTA, coarse1)
//   s~   = s + Q_Pi^T mu ; x = -A_Delta C s~ = -FC s~       (op2)
//   w    = theta P^T P x + (1 - theta) x  P = Cdelta Kbar^+ Bbar (nn1, nn2, op3)
//   u    = FC^T a(w) ; nu = S^{-1} t'     (op3, coarse2)
//   out  = gather over the two owners of each Delta index of
//          -phi + Q_G (s~ + u + Q_Pi^T nu) + Zc^T (psi - Dpp mu - Dpp nu)  (op4, gather)
// followed by the Hestenes-Stiefel CG update (solvers.cpp:82-119). All cross-subdomain sums are
// gathers over precomputed owner lists in subdomain order: deterministic, no atomics.
#include <cfloat>

#include "common.cuh"
#include "kernels.hpp"

namespace ddg {

namespace {

constexpr int kBlk = 256;

struct SubCtx {
  ClassDims d;
  int r;
  const double* QtX;  // (k, e) at QtX[k*E + e]; QGt(k, g) = e = 1 + g
};

__device__ __forceinline__ SubCtx sub_ctx(const CgArgs& a, int t /* matrix index */, int i) {
  SubCtx c;
  c.d = a.dims[a.sub_cls[i]];
  c.r = a.rank[t];
  c.QtX = a.QtX + static_cast<size_t>(t) * a.rmax * a.ext;
  return c;
}

__device__ __forceinline__ bool cg_done(const CgArgs& a) { return a.state && a.state[1] != 0; }

// ---------------------------------------------------------------- op1: s, t-part, psi-part
__global__ void __launch_bounds__(kBlk) op1_kernel(CgArgs a, const double* v, int mode, int guard) {
  if (guard && cg_done(a)) return;
  const int i = blockIdx.x;
  const SubCtx c = sub_ctx(a, i, i);
  const int R = a.rmax, E = a.ext;
  extern __shared__ double sm[];
  double* phi = sm;          // gmax
  double* s = phi + a.gmax;  // rmax
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int* gd = a.gamma_delta + static_cast<size_t>(i) * a.gmax;
  for (int g = threadIdx.x; g < c.d.n_gamma; g += blockDim.x) {
    const int dg = gd[g];
    double ph = 0.0;
    if (dg >= 0) ph = (mode == 0) ? -v[dg] : (mode == 2 ? v[dg] : 0.0);
    phi[g] = ph;
  }
  __syncthreads();
  for (int k = warp; k < c.r; k += nw) {
    const double* q = c.QtX + static_cast<size_t>(k) * E + 1;
    double acc = 0;
    if (mode != 1)
      for (int g = lane; g < c.d.n_gamma; g += 32) acc += q[g] * phi[g];
    acc = warp_sum(acc);
    if (mode >= 1) acc += c.QtX[static_cast<size_t>(k) * E];
    if (lane == 0) {
      s[k] = acc;
      a.s[static_cast<size_t>(i) * R + k] = acc;
    }
  }
  __syncthreads();
  const int* cq = a.corner_q + i * 4;
  if (warp < 4) {
    const int g = cq[warp];
    double acc = 0;
    if (g >= 0)
      for (int k = lane; k < c.r; k += 32) acc += c.QtX[static_cast<size_t>(k) * E + 1 + g] * s[k];
    acc = warp_sum(acc);
    if (lane == 0) a.tpart[i * 4 + warp] = acc;
  }
  if (mode != 1) {
    for (int rho = warp; rho < a.crmax; rho += nw) {
      const double* z = a.Zc + (static_cast<size_t>(i) * a.crmax + rho) * a.gmax;
      double acc = 0;
      for (int g = lane; g < c.d.n_gamma; g += 32) {
        const int dg = gd[g];
        if (dg >= 0) acc += z[g] * v[dg];
      }
      acc = warp_sum(acc);
      if (lane == 0) a.psipart[static_cast<size_t>(i) * a.crmax + rho] = acc;
    }
  }
}

// ---------------------------------------------------------------- coarse solves (one CTA)
__global__ void __launch_bounds__(kBlk) coarse1_kernel(CgArgs a, int mode, int guard) {
  if (guard && cg_done(a)) return;
  extern __shared__ double sm[];
  const int n = a.n_pi, npf = a.npf;
  double* t = sm;         // n
  double* psi = t + n;    // npf
  double* rhs = psi + npf;  // n
  double* mu = rhs + n;   // n
  for (int gp = threadIdx.x; gp < n; gp += blockDim.x) {
    double acc = 0;
    for (int q = 0; q < 4; ++q) {
      const int o = a.pi_owner[gp * 4 + q];
      if (o >= 0) acc += a.tpart[o];
    }
    t[gp] = acc;
  }
  for (int rr = threadIdx.x; rr < npf; rr += blockDim.x) {
    double acc = 0;
    if (mode != 1)
      for (int q = 0; q < 4; ++q) {
        const int o = a.row_owner[rr * 4 + q];
        if (o >= 0) acc += a.psipart[o];
      }
    psi[rr] = (mode == 0) ? acc : (mode == 1 ? a.dpi[rr] : a.dpi[rr] - acc);
  }
  __syncthreads();
  for (int gp = threadIdx.x; gp < n; gp += blockDim.x) {
    double acc = 0;
    for (int rr = 0; rr < npf; ++rr) acc += a.Dpp[static_cast<size_t>(rr) * n + gp] * psi[rr];
    rhs[gp] = t[gp] + acc;
  }
  __syncthreads();
  for (int gp = threadIdx.x; gp < n; gp += blockDim.x) {
    double acc = 0;
    for (int q = 0; q < n; ++q) acc += a.Sinv[static_cast<size_t>(gp) * n + q] * rhs[q];
    mu[gp] = acc;
    a.mu[gp] = acc;
    if (mode == 2) a.mu_pi_out[gp] = acc;
  }
  __syncthreads();
  if (mode != 2)
    for (int rr = threadIdx.x; rr < npf; rr += blockDim.x) {
      double acc = 0;
      for (int gp = 0; gp < n; ++gp) acc += a.Dpp[static_cast<size_t>(rr) * n + gp] * mu[gp];
      a.d1[rr] = psi[rr] - acc;
    }
}

// ---------------------------------------------------------------- op2: s~, xf (or coefficients)
__global__ void __launch_bounds__(kBlk) op2_kernel(CgArgs a, int mode, int guard) {
  if (guard && cg_done(a)) return;
  const int i = blockIdx.x;
  const SubCtx c = sub_ctx(a, i, i);
  const int R = a.rmax, E = a.ext;
  extern __shared__ double sm[];
  double* st = sm;  // rmax
  __shared__ double muc[4];
  __shared__ int gq[4];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if (threadIdx.x < 4) {
    const int g = a.corner_q[i * 4 + threadIdx.x];
    gq[threadIdx.x] = g;
    muc[threadIdx.x] = g >= 0 ? a.mu[a.gamma_pi[static_cast<size_t>(i) * a.gmax + g]] : 0.0;
  }
  __syncthreads();
  for (int k = threadIdx.x; k < c.r; k += blockDim.x) {
    double acc = a.s[static_cast<size_t>(i) * R + k];
    for (int q = 0; q < 4; ++q)
      if (gq[q] >= 0) acc += c.QtX[static_cast<size_t>(k) * E + 1 + gq[q]] * muc[q];
    st[k] = acc;
    a.s[static_cast<size_t>(i) * R + k] = acc;
  }
  __syncthreads();
  if (mode == 2) {
    const double* Ci = a.C + static_cast<size_t>(i) * a.M * R;
    for (int j = threadIdx.x; j < a.M; j += blockDim.x) {
      double acc = 0;
      for (int k = 0; k < c.r; ++k) acc += Ci[static_cast<size_t>(j) * R + k] * st[k];
      a.coeffs[static_cast<size_t>(i) * a.M + j] = acc;
    }
    return;
  }
  if (a.coeff_space) {
    // reference order: c = K^+ phi - Ypi mu (M-vector), then F c
    const double* Ci = a.C + static_cast<size_t>(i) * a.M * R;
    double* cw = a.cwork + static_cast<size_t>(i) * a.M;
    for (int j = warp; j < a.M; j += nw) {
      double acc = 0;
      for (int k = lane; k < c.r; k += 32) acc += Ci[static_cast<size_t>(j) * R + k] * st[k];
      acc = warp_sum(acc);
      if (lane == 0) cw[j] = acc;
    }
    __syncthreads();
    const double* Fi = a.F + static_cast<size_t>(i) * a.M * a.ldF;
    for (int l = threadIdx.x; l < c.d.nF; l += blockDim.x) {
      double acc = 0;
      for (int j = 0; j < a.M; ++j) acc += Fi[static_cast<size_t>(j) * a.ldF + l] * cw[j];
      a.xf[static_cast<size_t>(i) * a.fmax + l] = -acc;
    }
    return;
  }
  const double* FC = a.FC + static_cast<size_t>(i) * a.fmax * R;
  for (int l = warp; l < c.d.nF; l += nw) {
    double acc = 0;
    for (int k = lane; k < c.r; k += 32) acc += FC[static_cast<size_t>(l) * R + k] * st[k];
    acc = warp_sum(acc);
    if (lane == 0) a.xf[static_cast<size_t>(i) * a.fmax + l] = -acc;
  }
}

__device__ __forceinline__ double gather_x(const CgArgs& a, int g) {
  return a.flip_sign[g] * (a.xf[a.own_flux[2 * g]] + a.xf[a.own_flux[2 * g + 1]]);
}

// ---------------------------------------------------------------- Neumann-to-Dirichlet map
__global__ void __launch_bounds__(kBlk) nn1_kernel(CgArgs a, int guard) {
  if (guard && cg_done(a)) return;
  const int i = blockIdx.x;
  const SubCtx c = sub_ctx(a, a.N + i, i);
  const int R = a.rmax, E = a.ext, nd = c.d.nd;
  extern __shared__ double sm[];
  double* rhs = sm;        // dmax
  double* sb = rhs + a.dmax;  // rmax
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int* nmap = a.ndelta_map + static_cast<size_t>(i) * a.dmax;
  for (int kk = threadIdx.x; kk < nd; kk += blockDim.x) rhs[kk] = -gather_x(a, nmap[kk]);
  __syncthreads();
  for (int k = warp; k < c.r; k += nw) {
    const double* q = c.QtX + static_cast<size_t>(k) * E + 1;
    double acc = 0;
    for (int kk = lane; kk < nd; kk += 32) acc += q[kk] * rhs[kk];
    acc = warp_sum(acc);
    if (lane == 0) sb[k] = acc;
  }
  __syncthreads();
  const double* CC = a.CCb + static_cast<size_t>(i) * a.dmax * R;
  for (int kk = warp; kk < nd; kk += nw) {
    double acc = 0;
    for (int k = lane; k < c.r; k += 32) acc += CC[static_cast<size_t>(kk) * R + k] * sb[k];
    acc = warp_sum(acc);
    if (lane == 0) a.tr[static_cast<size_t>(i) * a.dmax + kk] = acc;
  }
}

__global__ void __launch_bounds__(kBlk) nn2_kernel(CgArgs a, int guard) {
  if (guard && cg_done(a)) return;
  const int i = blockIdx.x;
  const SubCtx c = sub_ctx(a, a.N + i, i);
  const int R = a.rmax, E = a.ext, nd = c.d.nd;
  extern __shared__ double sm[];
  double* px = sm;          // dmax
  double* sb = px + a.dmax;  // rmax
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int* nmap = a.ndelta_map + static_cast<size_t>(i) * a.dmax;
  for (int kk = threadIdx.x; kk < nd; kk += blockDim.x) {
    const int g = nmap[kk];
    px[kk] = a.tr[a.own_nd[2 * g]] + a.tr[a.own_nd[2 * g + 1]];
  }
  __syncthreads();
  const double* CC = a.CCb + static_cast<size_t>(i) * a.dmax * R;
  for (int k = threadIdx.x; k < c.r; k += blockDim.x) {
    double acc = 0;
    for (int kk = 0; kk < nd; ++kk) acc += CC[static_cast<size_t>(kk) * R + k] * px[kk];
    sb[k] = acc;
  }
  __syncthreads();
  for (int kk = threadIdx.x; kk < nd; kk += blockDim.x) {
    double acc = 0;
    for (int k = 0; k < c.r; ++k) acc += c.QtX[static_cast<size_t>(k) * E + 1 + kk] * sb[k];
    a.zz[static_cast<size_t>(i) * a.dmax + kk] = acc;
  }
}

// ---------------------------------------------------------------- op3: weight, u = FC^T a
__global__ void __launch_bounds__(kBlk) op3_kernel(CgArgs a, int guard) {
  if (guard && cg_done(a)) return;
  const int i = blockIdx.x;
  const SubCtx c = sub_ctx(a, i, i);
  const int R = a.rmax, E = a.ext;
  extern __shared__ double sm[];
  double* av = sm;          // fmax
  double* u = av + a.fmax;  // rmax
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int* fd = a.fluxrow_delta + static_cast<size_t>(i) * a.fmax;
  const double theta = a.theta;
  for (int l = threadIdx.x; l < c.d.nF; l += blockDim.x) {
    const int g = fd[l];
    double w = 0.0;
    if (g >= 0) {
      const double x = gather_x(a, g);
      if (a.use_neumann) {
        const double ptp = -(a.zz[a.own_nd[2 * g]] + a.zz[a.own_nd[2 * g + 1]]);
        w = theta * ptp;
        if (theta < 1.0) w += (1.0 - theta) * x;
      } else {
        w = x;
      }
    }
    av[l] = w;
  }
  __syncthreads();
  if (a.coeff_space) {
    // reference order: at = F^T a (M-vector, apply_AT), then (K^+)^T at -> Q_r (C^T at)
    const double* Fi = a.F + static_cast<size_t>(i) * a.M * a.ldF;
    double* cw = a.cwork + static_cast<size_t>(i) * a.M;
    const int nw = blockDim.x >> 5;
    for (int j = warp; j < a.M; j += nw) {
      double acc = 0;
      for (int l = lane; l < c.d.nF; l += 32) acc += Fi[static_cast<size_t>(j) * a.ldF + l] * av[l];
      acc = warp_sum(acc);
      if (lane == 0) cw[j] = acc;
    }
    __syncthreads();
    const double* Ci = a.C + static_cast<size_t>(i) * a.M * R;
    for (int k = threadIdx.x; k < c.r; k += blockDim.x) {
      double acc = 0;
      for (int j = 0; j < a.M; ++j) acc += Ci[static_cast<size_t>(j) * R + k] * cw[j];
      u[k] = acc;
      a.u[static_cast<size_t>(i) * R + k] = acc;
    }
  } else {
    const double* FC = a.FC + static_cast<size_t>(i) * a.fmax * R;
    for (int k = threadIdx.x; k < c.r; k += blockDim.x) {
      double acc = 0;
      for (int l = 0; l < c.d.nF; ++l) acc += FC[static_cast<size_t>(l) * R + k] * av[l];
      u[k] = acc;
      a.u[static_cast<size_t>(i) * R + k] = acc;
    }
  }
  __syncthreads();
  if (warp < 4) {
    const int g = a.corner_q[i * 4 + warp];
    double acc = 0;
    if (g >= 0)
      for (int k = lane; k < c.r; k += 32) acc += c.QtX[static_cast<size_t>(k) * E + 1 + g] * u[k];
    acc = warp_sum(acc);
    if (lane == 0) a.tpart[i * 4 + warp] = acc;
  }
}

__global__ void __launch_bounds__(kBlk) coarse2_kernel(CgArgs a, int guard) {
  if (guard && cg_done(a)) return;
  extern __shared__ double sm[];
  const int n = a.n_pi, npf = a.npf;
  double* t = sm;
  double* nu = t + n;
  for (int gp = threadIdx.x; gp < n; gp += blockDim.x) {
    double acc = 0;
    for (int q = 0; q < 4; ++q) {
      const int o = a.pi_owner[gp * 4 + q];
      if (o >= 0) acc += a.tpart[o];
    }
    t[gp] = acc;
  }
  __syncthreads();
  for (int gp = threadIdx.x; gp < n; gp += blockDim.x) {
    double acc = 0;
    for (int q = 0; q < n; ++q) acc += a.Sinv[static_cast<size_t>(gp) * n + q] * t[q];
    nu[gp] = acc;
    a.nu[gp] = acc;
  }
  __syncthreads();
  for (int rr = threadIdx.x; rr < npf; rr += blockDim.x) {
    double acc = 0;
    for (int gp = 0; gp < n; ++gp) acc += a.Dpp[static_cast<size_t>(rr) * n + gp] * nu[gp];
    a.d2[rr] = a.d1[rr] - acc;
  }
}

// ---------------------------------------------------------------- op4: local output rows
__global__ void __launch_bounds__(kBlk) op4_kernel(CgArgs a, const double* v, int mode, int guard) {
  if (guard && cg_done(a)) return;
  const int i = blockIdx.x;
  const SubCtx c = sub_ctx(a, i, i);
  const int R = a.rmax, E = a.ext;
  extern __shared__ double sm[];
  double* w = sm;  // rmax
  __shared__ double nuc[4];
  __shared__ int gq[4];
  __shared__ double d2s[64];
  if (threadIdx.x < 4) {
    const int g = a.corner_q[i * 4 + threadIdx.x];
    gq[threadIdx.x] = g;
    nuc[threadIdx.x] = g >= 0 ? a.nu[a.gamma_pi[static_cast<size_t>(i) * a.gmax + g]] : 0.0;
  }
  for (int rho = threadIdx.x; rho < a.crmax && rho < 64; rho += blockDim.x) {
    const int rr = a.cr_row[static_cast<size_t>(i) * a.crmax + rho];
    d2s[rho] = rr >= 0 ? a.d2[rr] : 0.0;
  }
  __syncthreads();
  for (int k = threadIdx.x; k < c.r; k += blockDim.x) {
    double uu = a.u[static_cast<size_t>(i) * R + k];
    for (int q = 0; q < 4; ++q)
      if (gq[q] >= 0) uu += c.QtX[static_cast<size_t>(k) * E + 1 + gq[q]] * nuc[q];
    w[k] = a.s[static_cast<size_t>(i) * R + k] + uu;
  }
  __syncthreads();
  const int* gd = a.gamma_delta + static_cast<size_t>(i) * a.gmax;
  for (int g = threadIdx.x; g < c.d.n_gamma; g += blockDim.x) {
    const int dg = gd[g];
    if (dg < 0) continue;
    double acc = (mode == 0) ? v[dg] : 0.0;  // -phi
    double qs = 0;
    for (int k = 0; k < c.r; ++k) qs += c.QtX[static_cast<size_t>(k) * E + 1 + g] * w[k];
    double zs = 0;
    for (int rho = 0; rho < a.crmax; ++rho)
      zs += a.Zc[(static_cast<size_t>(i) * a.crmax + rho) * a.gmax + g] * d2s[rho];
    a.o[static_cast<size_t>(i) * a.gmax + g] = acc + qs + zs;
  }
}

// ---------------------------------------------------------------- gather + CG update
__global__ void __launch_bounds__(kBlk) gather_kernel(CgArgs a, double* out, int with_dot, int guard) {
  if (guard && cg_done(a)) return;
  __shared__ double red[32];
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  double d = 0;
  if (g < a.n_delta) {
    const double val = a.o[a.own_gamma[2 * g]] + a.o[a.own_gamma[2 * g + 1]];
    out[g] = val;
    if (with_dot) d = a.p[g] * val;
  }
  if (with_dot) {
    d = block_sum(d, red);
    if (threadIdx.x == 0) a.partial[blockIdx.x] = d;
  }
}

__device__ __forceinline__ double sum_partials(const double* p, int n) {
  // identical order in every block -> identical scalars everywhere
  double s = 0;
  for (int k = 0; k < n; ++k) s += p[k];
  return s;
}

__global__ void __launch_bounds__(kBlk) cg_init_kernel(CgArgs a) {
  __shared__ double red[32];
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  double d = 0;
  if (g < a.n_delta) {
    const double b = a.rhs[g];
    a.x[g] = 0.0;
    a.r[g] = b;
    a.p[g] = b;
    d = b * b;
  }
  d = block_sum(d, red);
  if (threadIdx.x == 0) a.partial[gridDim.x + blockIdx.x] = d;
}

__global__ void cg_init2_kernel(CgArgs a, int nblk) {
  if (threadIdx.x != 0) return;
  const double rr = sum_partials(a.partial + nblk, nblk);
  a.scal[0] = rr;
  a.scal[1] = sqrt(rr);
  a.state[0] = 1;
  a.state[1] = (rr == 0.0) ? 1 : 0;
  a.state[2] = (rr == 0.0) ? 1 : 0;
  a.state[3] = 0;
  a.state[4] = 0;
  a.state[5] = 0;
}

__global__ void __launch_bounds__(kBlk) cg_update1_kernel(CgArgs a, int guard) {
  if (guard && cg_done(a)) return;
  __shared__ double red[32];
  const int nblk = gridDim.x;
  const double pAp = sum_partials(a.partial, nblk);
  if (pAp <= 0.0) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      a.state[3] = pAp < 0.0 ? 1 : 0;
      a.state[5] = a.state[0] - 1;
      a.state[4] = 2;  // negative-curvature stop
    }
    return;
  }
  const double alpha = a.scal[0] / pAp;
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  double d = 0;
  if (g < a.n_delta) {
    a.x[g] += alpha * a.p[g];
    const double rg = a.r[g] - alpha * a.Ap[g];
    a.r[g] = rg;
    d = rg * rg;
  }
  d = block_sum(d, red);
  if (threadIdx.x == 0) a.partial[nblk + blockIdx.x] = d;
}

__global__ void __launch_bounds__(kBlk) cg_update2_kernel(CgArgs a, int guard) {
  if (guard && cg_done(a)) return;
  if (a.state[4] == 2) return;  // negative curvature: x, p untouched
  const int nblk = gridDim.x;
  const double rr_new = sum_partials(a.partial + nblk, nblk);
  const double rel = sqrt(rr_new) / a.scal[1];
  const int it = a.state[0];
  const bool conv = rel <= a.rel_tol;
  const bool stop = conv || it >= a.max_iter;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    a.hist[it - 1] = rel;
    a.state[5] = it;
    a.scal[2] = rr_new;
    a.state[4] = stop ? (conv ? 3 : 1) : 0;
  }
  if (stop) return;
  const double beta = rr_new / a.scal[0];
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g < a.n_delta) a.p[g] = a.r[g] + beta * a.p[g];
}

__global__ void cg_bookkeep_kernel(CgArgs a, unsigned long long handle, int use_cond) {
  if (threadIdx.x != 0) return;
  if (a.state[1] == 0) {
    const int st = a.state[4];
    if (st == 0) {
      a.state[0] += 1;
      a.scal[0] = a.scal[2];
    } else {
      a.state[1] = 1;
      a.state[2] = (st == 3) ? 1 : 0;
    }
  }
#if CUDART_VERSION >= 12040
  if (use_cond) cudaGraphSetConditional(static_cast<cudaGraphConditionalHandle>(handle), a.state[1] ? 0u : 1u);
#else
  (void)handle;
  (void)use_cond;
#endif
}

size_t sub_smem(const CgArgs& a) {
  const int big = std::max(std::max(a.gmax, a.fmax), a.dmax);
  return sizeof(double) * (big + a.rmax + 8);
}

}  // namespace

int cg_kernels_per_step(const CgArgs& a) { return a.use_neumann ? 12 : 10; }

void cg_launch_operator(const CgArgs& a, const double* v, double* out, int mode, cudaStream_t st) {
  const size_t ssm = sub_smem(a);
  const size_t csm = sizeof(double) * (3 * a.n_pi + a.npf + 8);
  const int guard = (mode == 0) ? 1 : 0;
  op1_kernel<<<a.N, kBlk, ssm, st>>>(a, v, mode, guard);
  coarse1_kernel<<<1, kBlk, csm, st>>>(a, mode, guard);
  op2_kernel<<<a.N, kBlk, ssm, st>>>(a, mode, guard);
  if (a.use_neumann) {
    nn1_kernel<<<a.N, kBlk, ssm, st>>>(a, guard);
    nn2_kernel<<<a.N, kBlk, ssm, st>>>(a, guard);
  }
  op3_kernel<<<a.N, kBlk, ssm, st>>>(a, guard);
  coarse2_kernel<<<1, kBlk, csm, st>>>(a, guard);
  op4_kernel<<<a.N, kBlk, ssm, st>>>(a, v, mode, guard);
  gather_kernel<<<ceil_div(a.n_delta, kBlk), kBlk, 0, st>>>(a, out, mode == 0 ? 1 : 0, guard);
  DDG_LAUNCH_CHECK();
}

void cg_launch_init(const CgArgs& a, cudaStream_t st) {
  const int nblk = ceil_div(a.n_delta, kBlk);
  cg_init_kernel<<<nblk, kBlk, 0, st>>>(a);
  cg_init2_kernel<<<1, 32, 0, st>>>(a, nblk);
  DDG_LAUNCH_CHECK();
}

void cg_launch_step(const CgArgs& a, cudaStream_t st, unsigned long long cond_handle, bool use_cond) {
  const int nblk = ceil_div(a.n_delta, kBlk);
  cg_launch_operator(a, a.p, a.Ap, 0, st);
  cg_update1_kernel<<<nblk, kBlk, 0, st>>>(a, 1);
  cg_update2_kernel<<<nblk, kBlk, 0, st>>>(a, 1);
  cg_bookkeep_kernel<<<1, 32, 0, st>>>(a, cond_handle, use_cond ? 1 : 0);
  DDG_LAUNCH_CHECK();
}

void cg_launch_reconstruct(const CgArgs& a, cudaStream_t st) {
  const size_t ssm = sub_smem(a);
  const size_t csm = sizeof(double) * (3 * a.n_pi + a.npf + 8);
  op1_kernel<<<a.N, kBlk, ssm, st>>>(a, a.x, 2, 0);
  coarse1_kernel<<<1, kBlk, csm, st>>>(a, 2, 0);
  op2_kernel<<<a.N, kBlk, ssm, st>>>(a, 2, 0);
  DDG_LAUNCH_CHECK();
}

}  // namespace ddg

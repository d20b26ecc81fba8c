// Interface Krylov iteration of DDELM-NN on the device (sm_100a, fp64).
//
// cs_reduced_apply (solvers.cpp:372-386) with the theta-mixed Neumann-Neumann weight
// (solvers.cpp:599-603), expressed on the per-subdomain factors of k_cod.cu / k_blocks.cu:
//   op1   s = Q_G^T phi (+ Q_r^T f), corner rows of K K^+ phi, psi = Dpd v       (local)
//   c1    mu = S^{-1}(t + Dpp^T psi), d1 = psi - Dpp mu                        (coarse)
//   op2   c = K^+ phi - Ypi mu = C s - Ypi mu ; x = -A_Delta c = -F c           (local)
//   nn1   P x   = Cdelta Kbar^+ (-x|flux rows)                                  (Neumann)
//   nn2   P^T u = -(Kbar^+)^T Cdelta^T u |flux rows
//   op3   w = theta P^T P x + (1-theta) x ; u = C^T (F^T a(w))                  (local)
//   c2    nu = S^{-1} t' ; d2 = d1 - Dpp nu                                    (coarse)
//   op4   out_i = -phi + Q_G (s~ + u + Q_Pi^T nu) + Zc^T d2                    (local)
//   gather over the two owners of each Delta index, then the Hestenes-Stiefel CG update
//   (solvers.cpp:82-119).
// "coeff_space" keeps the reference's grouping (K^+ applied into coefficient space, then the
// flux / Cdelta rows), which reproduces its finite-precision CG behaviour; the fused mode uses
// pre-multiplied FC / CCb blocks (fewer bytes, converges in fewer iterations).
//
// Work decomposition: in coefficient-space mode every local phase is split over the M
// coefficient rows into P parts (P ~ SMs / subdomains); each part streams its slice of C, F,
// Cbar, Cdelta and emits a partial result that the consumer sums in a fixed order (the maps are
// linear), so all SMs share the HBM stream with no extra barrier.
//
// The whole iteration loop runs as ONE persistent cooperative kernel: phases are separated by
// grid-wide barriers, every CTA keeps identical copies of the CG scalars (sums of per-CTA
// partials in a fixed order): no host round trip, no atomics, deterministic.
#include <cooperative_groups.h>

#include <cfloat>

#include "common.cuh"
#include "kernels.hpp"

namespace cgs = cooperative_groups;

namespace ddg {

namespace {

constexpr int kBlk = 256;
constexpr int kPersistBlk = 512;

struct SubCtx {
  ClassDims d;
  int r;
  const double* QtX;  // (k, e) at QtX[k*E + e]; Q_G^T(k, g) at e = 1 + g, Q_r^T f at e = 0
};

__device__ __forceinline__ SubCtx sub_ctx(const CgArgs& a, int t /* matrix */, int i /* subdomain */) {
  SubCtx c;
  c.d = a.dims[a.sub_cls[i]];
  c.r = a.rank[t];
  c.QtX = a.QtX + static_cast<size_t>(t) * a.rmax * a.ext;
  return c;
}

struct Smem {
  double* v1;   // big  (phi / rhs / px / a)
  double* cw;   // cwsize (coefficient-space slice, coarse vectors)
  double* s0;   // rmax
  double* s1;   // rmax
  double* red;  // blockDim (partials of coldot)
};

__device__ __forceinline__ Smem carve(const CgArgs& a) {
  extern __shared__ double sm[];
  const int big = max(max(a.gmax, a.fmax), a.dmax);
  const int cwsize = max(a.M, 3 * a.n_pi + 2 * a.npf);
  Smem s;
  s.v1 = sm;
  s.cw = s.v1 + big;
  s.s0 = s.cw + cwsize;
  s.s1 = s.s0 + a.rmax;
  s.red = s.s1 + a.rmax;
  return s;
}

__device__ __forceinline__ void part_rows(const CgArgs& a, int p, int& j0, int& j1) {
  const int chunk = (a.M + a.P - 1) / a.P;
  j0 = min(a.M, p * chunk);
  j1 = min(a.M, j0 + chunk);
}

// y[j] = scale * sum_k A[j*lda + k] x[k], j < rows. Warp per row, 4 rows in flight per warp.
__device__ __forceinline__ void rowdot(const double* A, size_t lda, int rows, int cols, const double* x,
                                       double* y, double scale = 1.0) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  int j = warp * 4;
  for (; j + 3 < rows; j += nw * 4) {
    const double* a0 = A + static_cast<size_t>(j) * lda;
    double c0 = 0, c1 = 0, c2 = 0, c3 = 0;
    for (int k = lane; k < cols; k += 32) {
      const double xk = x[k];
      c0 += a0[k] * xk;
      c1 += a0[lda + k] * xk;
      c2 += a0[2 * lda + k] * xk;
      c3 += a0[3 * lda + k] * xk;
    }
    c0 = warp_sum(c0);
    c1 = warp_sum(c1);
    c2 = warp_sum(c2);
    c3 = warp_sum(c3);
    if (lane == 0) {
      y[j] = scale * c0;
      y[j + 1] = scale * c1;
      y[j + 2] = scale * c2;
      y[j + 3] = scale * c3;
    }
  }
  for (; j < rows; ++j) {  // tail rows (< 4) of this warp's last group
    const double* aj = A + static_cast<size_t>(j) * lda;
    double acc = 0;
    for (int k = lane; k < cols; k += 32) acc += aj[k] * x[k];
    acc = warp_sum(acc);
    if (lane == 0) y[j] = scale * acc;
  }
}

// y[k] = scale * sum_j A[j*lda + k] x[j], k < cols (threads over (k, row group); fixed-order combine)
__device__ __forceinline__ void coldot(const double* A, size_t lda, int rows, int cols, const double* x,
                                       double* y, double* red, double scale = 1.0) {
  for (int k0 = 0; k0 < cols; k0 += blockDim.x) {
    const int cc = min(cols - k0, static_cast<int>(blockDim.x));
    const int pad = (cc + 31) & ~31;
    const int groups = max(1, static_cast<int>(blockDim.x) / pad);
    const int t = threadIdx.x;
    const int k = t % pad, grp = t / pad;
    double acc = 0;
    if (grp < groups && k < cc) {
      const double* ak = A + k0 + k;
      double a1 = 0;
      int j = grp;
      for (; j + groups < rows; j += 2 * groups) {
        acc += ak[static_cast<size_t>(j) * lda] * x[j];
        a1 += ak[static_cast<size_t>(j + groups) * lda] * x[j + groups];
      }
      if (j < rows) acc += ak[static_cast<size_t>(j) * lda] * x[j];
      acc += a1;
    }
    red[t] = acc;
    __syncthreads();
    if (t < cc) {
      double s = 0;
      for (int g = 0; g < groups; ++g) s += red[g * pad + t];
      y[k0 + t] = scale * s;
    }
    __syncthreads();
  }
}

__device__ __forceinline__ double sum_parts(const double* base, size_t stride, int P, int idx) {
  double s = 0;
  for (int p = 0; p < P; ++p) s += base[p * stride + idx];
  return s;
}

__device__ __forceinline__ double gather_x(const CgArgs& a, int g) {
  const size_t st = static_cast<size_t>(a.N) * a.fmax;
  return a.flip_sign[g] * (sum_parts(a.xf, st, a.P, a.own_flux[2 * g]) + sum_parts(a.xf, st, a.P, a.own_flux[2 * g + 1]));
}

// ---------------------------------------------------------------- op1: s, t-part, psi-part
__device__ void dev_op1(const CgArgs& a, int i, const double* v, int mode) {
  const SubCtx c = sub_ctx(a, i, i);
  const int R = a.rmax, E = a.ext;
  Smem sm = carve(a);
  double* vg = sm.cw;   // v at the gamma points (0 at corners)
  double* phi = sm.v1;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int* gd = a.gamma_delta + static_cast<size_t>(i) * a.gmax;
  for (int g = threadIdx.x; g < c.d.n_gamma; g += blockDim.x) {
    const int dg = gd[g];
    const double vv = (dg >= 0 && mode != 1) ? v[dg] : 0.0;
    vg[g] = vv;
    phi[g] = (mode == 0) ? -vv : vv;  // B_Delta v = -v (operator); +mu_Delta (reconstruction)
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
      sm.s0[k] = acc;
      a.s[static_cast<size_t>(i) * R + k] = acc;
    }
  }
  __syncthreads();
  const int* cq = a.corner_q + i * 4;
  if (warp < 4) {
    const int g = cq[warp];
    double acc = 0;
    if (g >= 0)
      for (int k = lane; k < c.r; k += 32) acc += c.QtX[static_cast<size_t>(k) * E + 1 + g] * sm.s0[k];
    acc = warp_sum(acc);
    if (lane == 0) a.tpart[i * 4 + warp] = acc;  // t(gp) -= phi - Ky at corners (phi = 0 there)
  }
  if (mode != 1)
    rowdot(a.Zc + static_cast<size_t>(i) * a.crmax * a.gmax, a.gmax, a.crmax, c.d.n_gamma, vg,
           a.psipart + static_cast<size_t>(i) * a.crmax);
  __syncthreads();
}

// ---------------------------------------------------------------- coarse solves (one CTA)
__device__ void dev_coarse1(const CgArgs& a, int mode) {
  Smem sm = carve(a);
  const int n = a.n_pi, npf = a.npf;
  double* t = sm.cw;       // n
  double* psi = t + n;     // npf
  double* rhs = psi + npf; // n
  double* mu = rhs + n;    // n
  double* pb = mu + n;     // npf
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
  coldot(a.Dpp, n, npf, n, psi, rhs, sm.red);  // Dpp^T psi
  for (int gp = threadIdx.x; gp < n; gp += blockDim.x) rhs[gp] += t[gp];
  __syncthreads();
  rowdot(a.Sinv, n, n, n, rhs, mu);
  __syncthreads();
  for (int gp = threadIdx.x; gp < n; gp += blockDim.x) {
    a.mu[gp] = mu[gp];
    if (mode == 2) a.mu_pi_out[gp] = mu[gp];
  }
  if (mode != 2) {
    rowdot(a.Dpp, n, npf, n, mu, pb);  // proj_bottom = Dpp mu
    __syncthreads();
    for (int rr = threadIdx.x; rr < npf; rr += blockDim.x) a.d1[rr] = psi[rr] - pb[rr];
  }
  __syncthreads();
}

// ---------------------------------------------------------------- op2: s~, x (or coefficients)
__device__ void dev_op2(const CgArgs& a, int i, int p, int mode) {
  const SubCtx c = sub_ctx(a, i, i);
  const int R = a.rmax, E = a.ext;
  Smem sm = carve(a);
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
    const double sk = a.s[static_cast<size_t>(i) * R + k];
    double acc = sk;
    for (int q = 0; q < 4; ++q)
      if (gq[q] >= 0) acc += c.QtX[static_cast<size_t>(k) * E + 1 + gq[q]] * muc[q];
    sm.s0[k] = sk;
    sm.s1[k] = acc;  // s~ = s + Q_Pi^T mu
  }
  __syncthreads();
  const double* Ci = a.C + static_cast<size_t>(i) * a.M * R;
  if (a.coeff_space) {
    // reference grouping (solvers.cpp:336, 342): c = K^+ phi - Ypi mu, then F c
    int j0, j1;
    part_rows(a, p, j0, j1);
    const double* Yp = a.Ypi + static_cast<size_t>(i) * a.M * 4;
    double* cw = (mode == 2) ? a.coeffs + static_cast<size_t>(i) * a.M + j0 : sm.cw;
    for (int j = j0 + warp; j < j1; j += nw) {
      const double* cj = Ci + static_cast<size_t>(j) * R;
      double acc = 0;
      for (int k = lane; k < c.r; k += 32) acc += cj[k] * sm.s0[k];
      acc = warp_sum(acc);
      if (lane == 0) {
        double yp = 0;
        for (int q = 0; q < 4; ++q) yp += Yp[static_cast<size_t>(j) * 4 + q] * muc[q];
        cw[j - j0] = acc - yp;
      }
    }
    __syncthreads();
    if (mode == 2) return;
    coldot(a.F + (static_cast<size_t>(i) * a.M + j0) * a.ldF, a.ldF, j1 - j0, c.d.nF, sm.cw,
           a.xf + (static_cast<size_t>(p) * a.N + i) * a.fmax, sm.red, -1.0);
    return;
  }
  if (mode == 2) {
    rowdot(Ci, R, a.M, c.r, sm.s1, a.coeffs + static_cast<size_t>(i) * a.M);
    __syncthreads();
    return;
  }
  rowdot(a.FC + static_cast<size_t>(i) * a.fmax * R, R, c.d.nF, c.r, sm.s1,
         a.xf + static_cast<size_t>(i) * a.fmax, -1.0);
  __syncthreads();
}

// ---------------------------------------------------------------- Neumann-to-Dirichlet map
__device__ void dev_nn1(const CgArgs& a, int i, int p) {
  const SubCtx c = sub_ctx(a, a.N + i, i);
  const int R = a.rmax, E = a.ext, nd = c.d.nd;
  Smem sm = carve(a);
  const int* nmap = a.ndelta_map + static_cast<size_t>(i) * a.dmax;
  for (int kk = threadIdx.x; kk < nd; kk += blockDim.x) sm.v1[kk] = -gather_x(a, nmap[kk]);
  __syncthreads();
  rowdot(c.QtX + 1, E, c.r, nd, sm.v1, sm.s0);  // Qbar_r^T rhs
  __syncthreads();
  double* tr = a.tr + (static_cast<size_t>(p) * a.N + i) * a.dmax;
  if (a.coeff_space) {
    // reference order (solvers.cpp:456): y = Kbar^+ rhs (M-vector), then Cdelta y
    int j0, j1;
    part_rows(a, p, j0, j1);
    rowdot(a.C + (static_cast<size_t>(a.N + i) * a.M + j0) * R, R, j1 - j0, c.r, sm.s0, sm.cw);
    __syncthreads();
    coldot(a.Cd + (static_cast<size_t>(i) * a.M + j0) * a.ldC, a.ldC, j1 - j0, nd, sm.cw, tr, sm.red);
  } else {
    rowdot(a.CCb + static_cast<size_t>(i) * a.dmax * R, R, nd, c.r, sm.s0, tr);
    __syncthreads();
  }
}

__device__ void dev_nn2(const CgArgs& a, int i, int p) {
  const SubCtx c = sub_ctx(a, a.N + i, i);
  const int R = a.rmax, E = a.ext, nd = c.d.nd;
  Smem sm = carve(a);
  const int* nmap = a.ndelta_map + static_cast<size_t>(i) * a.dmax;
  const size_t st = static_cast<size_t>(a.N) * a.dmax;
  for (int kk = threadIdx.x; kk < nd; kk += blockDim.x) {
    const int g = nmap[kk];
    sm.v1[kk] = sum_parts(a.tr, st, a.P, a.own_nd[2 * g]) + sum_parts(a.tr, st, a.P, a.own_nd[2 * g + 1]);
  }
  __syncthreads();
  if (a.coeff_space) {
    // reference order (solvers.cpp:469): x = Cdelta^T tl (M-vector), then (Kbar^+)^T x
    int j0, j1;
    part_rows(a, p, j0, j1);
    rowdot(a.Cd + (static_cast<size_t>(i) * a.M + j0) * a.ldC, a.ldC, j1 - j0, nd, sm.v1, sm.cw);
    __syncthreads();
    coldot(a.C + (static_cast<size_t>(a.N + i) * a.M + j0) * R, R, j1 - j0, c.r, sm.cw, sm.s0, sm.red);
  } else {
    coldot(a.CCb + static_cast<size_t>(i) * a.dmax * R, R, nd, c.r, sm.v1, sm.s0, sm.red);
  }
  coldot(c.QtX + 1, E, c.r, nd, sm.s0, a.zz + (static_cast<size_t>(p) * a.N + i) * a.dmax, sm.red);
}

// ---------------------------------------------------------------- op3: weight, u
__device__ void dev_op3(const CgArgs& a, int i, int p) {
  const SubCtx c = sub_ctx(a, i, i);
  const int R = a.rmax, E = a.ext;
  Smem sm = carve(a);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int* fd = a.fluxrow_delta + static_cast<size_t>(i) * a.fmax;
  const double theta = a.theta;
  const size_t st = static_cast<size_t>(a.N) * a.dmax;
  for (int l = threadIdx.x; l < c.d.nF; l += blockDim.x) {
    const int g = fd[l];
    double w = 0.0;
    if (g >= 0) {
      const double x = gather_x(a, g);
      if (a.use_neumann) {
        const double ptp = -(sum_parts(a.zz, st, a.P, a.own_nd[2 * g]) + sum_parts(a.zz, st, a.P, a.own_nd[2 * g + 1]));
        w = theta * ptp;
        if (theta < 1.0) w += (1.0 - theta) * x;
      } else {
        w = x;
      }
    }
    sm.v1[l] = w;  // apply_AT_delta: a(lrow) = w(grow) on the Delta flux rows
  }
  __syncthreads();
  if (a.coeff_space) {
    // reference order: at = F^T a (M-vector, apply_AT), then (K^+)^T at -> C^T at
    int j0, j1;
    part_rows(a, p, j0, j1);
    rowdot(a.F + (static_cast<size_t>(i) * a.M + j0) * a.ldF, a.ldF, j1 - j0, c.d.nF, sm.v1, sm.cw);
    __syncthreads();
    coldot(a.C + (static_cast<size_t>(i) * a.M + j0) * R, R, j1 - j0, c.r, sm.cw, sm.s0, sm.red);
  } else {
    coldot(a.FC + static_cast<size_t>(i) * a.fmax * R, R, c.d.nF, c.r, sm.v1, sm.s0, sm.red);
  }
  double* up = a.u + (static_cast<size_t>(p) * a.N + i) * R;
  for (int k = threadIdx.x; k < c.r; k += blockDim.x) up[k] = sm.s0[k];
  if (warp < 4) {
    const int g = a.corner_q[i * 4 + warp];
    double acc = 0;
    if (g >= 0)
      for (int k = lane; k < c.r; k += 32) acc += c.QtX[static_cast<size_t>(k) * E + 1 + g] * sm.s0[k];
    acc = warp_sum(acc);
    if (lane == 0) a.tpart3[(static_cast<size_t>(p) * a.N + i) * 4 + warp] = acc;  // t(gp) += z(lr)
  }
  __syncthreads();
}

__device__ void dev_coarse2(const CgArgs& a) {
  Smem sm = carve(a);
  const int n = a.n_pi, npf = a.npf;
  double* t = sm.cw;
  double* nu = t + n;
  double* bot = nu + n;
  const size_t st = static_cast<size_t>(a.N) * 4;
  for (int gp = threadIdx.x; gp < n; gp += blockDim.x) {
    double acc = 0;
    for (int q = 0; q < 4; ++q) {
      const int o = a.pi_owner[gp * 4 + q];
      if (o >= 0) acc += sum_parts(a.tpart3, st, a.P, o);
    }
    t[gp] = acc;
  }
  __syncthreads();
  rowdot(a.Sinv, n, n, n, t, nu);
  __syncthreads();
  for (int gp = threadIdx.x; gp < n; gp += blockDim.x) a.nu[gp] = nu[gp];
  rowdot(a.Dpp, n, npf, n, nu, bot);
  __syncthreads();
  for (int rr = threadIdx.x; rr < npf; rr += blockDim.x) a.d2[rr] = a.d1[rr] - bot[rr];
  __syncthreads();
}

// ---------------------------------------------------------------- op4: local output rows
__device__ void dev_op4(const CgArgs& a, int i, const double* v, int mode) {
  const SubCtx c = sub_ctx(a, i, i);
  const int R = a.rmax, E = a.ext;
  Smem sm = carve(a);
  __shared__ double nuc[4], muc[4];
  __shared__ int gq[4];
  double* d2s = sm.v1;
  if (threadIdx.x < 4) {
    const int g = a.corner_q[i * 4 + threadIdx.x];
    gq[threadIdx.x] = g;
    const int gp = g >= 0 ? a.gamma_pi[static_cast<size_t>(i) * a.gmax + g] : 0;
    nuc[threadIdx.x] = g >= 0 ? a.nu[gp] : 0.0;
    muc[threadIdx.x] = g >= 0 ? a.mu[gp] : 0.0;
  }
  for (int rho = threadIdx.x; rho < a.crmax; rho += blockDim.x) {
    const int rr = a.cr_row[static_cast<size_t>(i) * a.crmax + rho];
    d2s[rho] = rr >= 0 ? a.d2[rr] : 0.0;
  }
  __syncthreads();
  const size_t ust = static_cast<size_t>(a.N) * R;
  for (int k = threadIdx.x; k < c.r; k += blockDim.x) {
    double uu = sum_parts(a.u + static_cast<size_t>(i) * R, ust, a.P, k);
    double sk = a.s[static_cast<size_t>(i) * R + k];
    for (int q = 0; q < 4; ++q)
      if (gq[q] >= 0) {
        const double qk = c.QtX[static_cast<size_t>(k) * E + 1 + gq[q]];
        uu += qk * nuc[q];
        sk += qk * muc[q];  // s~ = s + Q_Pi^T mu (op2 recomputes it per part)
      }
    sm.s0[k] = sk + uu;  // s~ + u + Q_Pi^T nu
  }
  __syncthreads();
  double* qs = sm.cw;
  coldot(c.QtX + 1, E, c.r, c.d.n_gamma, sm.s0, qs, sm.red);
  const int* gd = a.gamma_delta + static_cast<size_t>(i) * a.gmax;
  const double* Zc = a.Zc + static_cast<size_t>(i) * a.crmax * a.gmax;
  for (int g = threadIdx.x; g < c.d.n_gamma; g += blockDim.x) {
    const int dg = gd[g];
    if (dg < 0) continue;
    double zs = 0;
    for (int rho = 0; rho < a.crmax; ++rho) zs += Zc[static_cast<size_t>(rho) * a.gmax + g] * d2s[rho];
    const double mphi = (mode == 0) ? v[dg] : 0.0;  // -phi
    a.o[static_cast<size_t>(i) * a.gmax + g] = mphi + qs[g] + zs;
  }
  __syncthreads();
}

__device__ __forceinline__ double gather_out(const CgArgs& a, int g) {
  return a.o[a.own_gamma[2 * g]] + a.o[a.own_gamma[2 * g + 1]];
}

// ---------------------------------------------------------------- standalone kernels
// grid = N (op1, op4) or N * P (op2, nn1, nn2, op3: blockIdx = i * P + p)
__global__ void __launch_bounds__(kBlk) op1_kernel(CgArgs a, const double* v, int mode) { dev_op1(a, blockIdx.x, v, mode); }
__global__ void __launch_bounds__(kBlk) coarse1_kernel(CgArgs a, int mode) { dev_coarse1(a, mode); }
__global__ void __launch_bounds__(kBlk) op2_kernel(CgArgs a, int mode) { dev_op2(a, blockIdx.x / a.P, blockIdx.x % a.P, mode); }
__global__ void __launch_bounds__(kBlk) nn1_kernel(CgArgs a) { dev_nn1(a, blockIdx.x / a.P, blockIdx.x % a.P); }
__global__ void __launch_bounds__(kBlk) nn2_kernel(CgArgs a) { dev_nn2(a, blockIdx.x / a.P, blockIdx.x % a.P); }
__global__ void __launch_bounds__(kBlk) op3_kernel(CgArgs a) { dev_op3(a, blockIdx.x / a.P, blockIdx.x % a.P); }
__global__ void __launch_bounds__(kBlk) coarse2_kernel(CgArgs a) { dev_coarse2(a); }
__global__ void __launch_bounds__(kBlk) op4_kernel(CgArgs a, const double* v, int mode) { dev_op4(a, blockIdx.x, v, mode); }
__global__ void __launch_bounds__(kBlk) gather_kernel(CgArgs a, double* out) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g < a.n_delta) out[g] = gather_out(a, g);
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

// ---------------------------------------------------------------- persistent CG
__device__ __forceinline__ double sum_partials(const double* p, int n) {
  double s = 0;
  for (int k = 0; k < n; ++k) s += p[k];
  return s;
}

__global__ void __launch_bounds__(kPersistBlk) cg_persistent_kernel(CgArgs a) {
  cgs::grid_group grid = cgs::this_grid();
  const int G = gridDim.x, b = blockIdx.x;
  const int NP = a.N * a.P;
  __shared__ double red[32];
  double* partial = a.partial;          // G entries: p.Ap
  double* partial2 = a.partial + G;     // G entries: r.r
  double rr = a.scal[0];
  const double bnorm = a.scal[1];
  if (a.state[1]) return;  // rhs == 0
  for (int it = 1;; ++it) {
    for (int i = b; i < a.N; i += G) dev_op1(a, i, a.p, 0);
    grid.sync();
    if (b == 0) dev_coarse1(a, 0);
    grid.sync();
    for (int w = b; w < NP; w += G) dev_op2(a, w / a.P, w % a.P, 0);
    grid.sync();
    if (a.use_neumann) {
      for (int w = b; w < NP; w += G) dev_nn1(a, w / a.P, w % a.P);
      grid.sync();
      for (int w = b; w < NP; w += G) dev_nn2(a, w / a.P, w % a.P);
      grid.sync();
    }
    for (int w = b; w < NP; w += G) dev_op3(a, w / a.P, w % a.P);
    grid.sync();
    if (b == 0) dev_coarse2(a);
    grid.sync();
    for (int i = b; i < a.N; i += G) dev_op4(a, i, a.p, 0);
    grid.sync();
    // Ap = gathered output, pAp partials
    double d = 0;
    for (int g = b * blockDim.x + threadIdx.x; g < a.n_delta; g += G * blockDim.x) {
      const double val = gather_out(a, g);
      a.Ap[g] = val;
      d += a.p[g] * val;
    }
    d = block_sum(d, red);
    if (threadIdx.x == 0) partial[b] = d;
    grid.sync();
    const double pAp = sum_partials(partial, G);
    if (pAp <= 0.0) {  // solvers.cpp:97-103
      if (b == 0 && threadIdx.x == 0) {
        a.state[3] = pAp < 0.0 ? 1 : 0;
        a.state[5] = it - 1;
        a.state[1] = 1;
      }
      return;
    }
    const double alpha = rr / pAp;
    d = 0;
    for (int g = b * blockDim.x + threadIdx.x; g < a.n_delta; g += G * blockDim.x) {
      a.x[g] += alpha * a.p[g];
      const double rg = a.r[g] - alpha * a.Ap[g];
      a.r[g] = rg;
      d += rg * rg;
    }
    d = block_sum(d, red);
    if (threadIdx.x == 0) partial2[b] = d;
    grid.sync();
    const double rr_new = sum_partials(partial2, G);
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
      return;
    }
    const double beta = rr_new / rr;
    for (int g = b * blockDim.x + threadIdx.x; g < a.n_delta; g += G * blockDim.x) a.p[g] = a.r[g] + beta * a.p[g];
    rr = rr_new;
    grid.sync();
  }
}

size_t smem_bytes(const CgArgs& a, int threads) {
  const int big = std::max(std::max(a.gmax, a.fmax), a.dmax);
  const int cwsize = std::max(a.M, 3 * a.n_pi + 2 * a.npf);
  return sizeof(double) * (static_cast<size_t>(big) + cwsize + 2 * a.rmax + threads);
}

}  // namespace

int cg_kernels_per_step(const CgArgs& a) { return a.use_neumann ? 9 : 7; }

void cg_launch_operator(const CgArgs& a, const double* v, double* out, int mode, cudaStream_t st) {
  const size_t sm = smem_bytes(a, kBlk);
  const int NP = a.N * a.P;
  op1_kernel<<<a.N, kBlk, sm, st>>>(a, v, mode);
  coarse1_kernel<<<1, kBlk, sm, st>>>(a, mode);
  op2_kernel<<<NP, kBlk, sm, st>>>(a, mode);
  if (a.use_neumann) {
    nn1_kernel<<<NP, kBlk, sm, st>>>(a);
    nn2_kernel<<<NP, kBlk, sm, st>>>(a);
  }
  op3_kernel<<<NP, kBlk, sm, st>>>(a);
  coarse2_kernel<<<1, kBlk, sm, st>>>(a);
  op4_kernel<<<a.N, kBlk, sm, st>>>(a, v, mode);
  gather_kernel<<<ceil_div(a.n_delta, kBlk), kBlk, 0, st>>>(a, out);
  DDG_LAUNCH_CHECK();
}

void cg_launch_init(const CgArgs& a, cudaStream_t st) {
  const int nblk = ceil_div(a.n_delta, kBlk);
  cg_init_kernel<<<nblk, kBlk, 0, st>>>(a);
  cg_init2_kernel<<<1, 32, 0, st>>>(a, nblk);
  DDG_LAUNCH_CHECK();
}

int cg_persistent_grid(const CgArgs& a) {
  int dev = 0, sms = 0, per_sm = 0;
  DDG_CUDA(cudaGetDevice(&dev));
  DDG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const size_t sm = smem_bytes(a, kPersistBlk);
  DDG_CUDA(cudaFuncSetAttribute(cg_persistent_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(sm)));
  DDG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, cg_persistent_kernel, kPersistBlk, sm));
  if (per_sm < 1) throw CudaError("cg_persistent_kernel cannot be resident (occupancy 0)");
  // one CTA per SM: the local phases have N * P (~ number of SMs) work items
  return std::max(1, std::min(sms * per_sm, sms));
}

void cg_launch_persistent(const CgArgs& a, cudaStream_t st) {
  const int G = cg_persistent_grid(a);
  const size_t sm = smem_bytes(a, kPersistBlk);
  CgArgs arg = a;
  void* params[] = {&arg};
  DDG_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(cg_persistent_kernel), dim3(G), dim3(kPersistBlk),
                                       params, sm, st));
}

void cg_launch_reconstruct(const CgArgs& a, cudaStream_t st) {
  const size_t sm = smem_bytes(a, kBlk);
  op1_kernel<<<a.N, kBlk, sm, st>>>(a, a.x, 2);
  coarse1_kernel<<<1, kBlk, sm, st>>>(a, 2);
  op2_kernel<<<a.N * a.P, kBlk, sm, st>>>(a, 2);
  DDG_LAUNCH_CHECK();
}

}  // namespace ddg

// Fused ELM feature / collocation-row builder (sm_100a).
//
// One pass over (row task, neuron) writes every matrix the solve needs — K (with the
// change-of-variables epilogue T^{-1} = I - E), the Neumann matrix Kbar (its interior/boundary
// rows shared with K, tanh evaluated once), the flux blocks F and the Neumann trace rows Cdelta.
// Reference semantics: eval_derivative_matrix (features.cpp:42-76), Poisson rows
// (problems.cpp:71-121), assemble_local (assembly.cpp:9-46), apply_change_of_variables
// (assembly.cpp:80-87), build_neumann rows (solvers.cpp:418-438).
//
// HBM roofline: writes 8*(2 m M + nF M + nd M) bytes per subdomain; threads
// map to consecutive rows of a column-major matrix so every store is coalesced.
#include <algorithm>

#include "common.cuh"
#include "kernels.hpp"
#include "plan.hpp"

namespace ddg {

namespace {

struct Feat {
  double w0, w1, b;
};

__device__ __forceinline__ double feat_z(const Feat& f, double x, double y) {
  // w0 * x + w1 * y + b in the reference's evaluation order, no FMA contraction
  return __dadd_rn(__dadd_rn(__dmul_rn(f.w0, x), __dmul_rn(f.w1, y)), f.b);
}

/// Laplacian of feature f at (x, y): s2 (w0^2) + s2 (w1^2), s2 = -2 s0 (1 - s0^2)
/// (features.cpp:42-76 order; problems.cpp:105-108 trace / boundary component 1)
__device__ __forceinline__ double feat_lap(const Feat& f, double x, double y) {
  const double s0 = tanh(feat_z(f, x, y));
  const double s1 = __dadd_rn(1.0, -__dmul_rn(s0, s0));
  const double s2 = __dmul_rn(__dmul_rn(-2.0, s0), s1);
  return __dadd_rn(__dmul_rn(s2, __dmul_rn(f.w0, f.w0)), __dmul_rn(s2, __dmul_rn(f.w1, f.w1)));
}

__device__ __forceinline__ double coord(int i0, int a, int S) {
  return static_cast<double>(i0 + a) / static_cast<double>(S);
}

__global__ void __launch_bounds__(256) build_features_kernel(FeatureArgs p) {
  constexpr int JT = 32;
  __shared__ Feat sf[JT];
  const int i = blockIdx.y;
  const int j0 = blockIdx.x * JT;
  if (threadIdx.x < JT) {
    const int j = j0 + threadIdx.x;
    if (j < p.M) sf[threadIdx.x] = Feat{p.w0[i * p.M + j], p.w1[i * p.M + j], p.b[i * p.M + j]};
  }
  __syncthreads();
  const int jn = min(JT, p.M - j0);
  const int cls = p.sub_cls[i];
  const int ix = p.sub_ix[i], iy = p.sub_iy[i];
  const int n = p.n_grid, S = p.S;
  const int gx0 = ix * (n - 1), gy0 = iy * (n - 1);
  const Task* tasks = p.tasks + p.cls_task_off[cls];
  const int ntask = p.cls_task_cnt[cls];
  const size_t mstride = static_cast<size_t>(p.ld) * p.ncol;
  double* K = p.A + static_cast<size_t>(i) * mstride;
  double* Kb = p.A + static_cast<size_t>(p.N + i) * mstride;
  double* F = p.F + static_cast<size_t>(i) * p.M * p.ldF;
  double* Cd = p.Cd + static_cast<size_t>(i) * p.M * p.ldC;
  const double inv_n1 = 1.0 / (n - 1);
  (void)inv_n1;

  const double* coef = p.coef ? p.coef + static_cast<size_t>(i) * p.tmax * 3 : nullptr;
  for (int t = threadIdx.x; t < ntask; t += blockDim.x) {
    const Task tk = tasks[t];
    // varcoef_poisson (problems.cpp:74-87, 117-121): rho and grad rho at this row's point
    double rho = 1.0, rhox = 0.0, rhoy = 0.0;
    const bool var = coef != nullptr && (tk.kind == kLap || tk.kind == kFlux);
    if (var) {
      rho = coef[t * 3];
      rhox = coef[t * 3 + 1];
      rhoy = coef[t * 3 + 2];
    }
    const double x = coord(gx0, tk.a, S), y = coord(gy0, tk.b, S);
    const int dst = tk.dst & 0x0f;
    const bool dual = (tk.dst & kDual) != 0;
    double* out;
    size_t ldo;
    if (dst == kDstK) { out = K; ldo = p.ld; }
    else if (dst == kDstKbar) { out = Kb; ldo = p.ld; }
    else if (dst == kDstF) { out = F; ldo = p.ldF; }
    else { out = Cd; ldo = p.ldC; }
    // change-of-variables corner points (assembly.cpp:59-75)
    double cx1 = 0, cy1 = 0, cx2 = 0, cy2 = 0, e1 = 0, e2 = 0;
    double nx = 0, ny = 0;
    if (tk.kind == kValueCov || tk.kind == kLapCov) {
      const bool vert = tk.side < 2;
      const int jj = vert ? tk.b : tk.a;  // geom_j along the edge
      const int ae = vert ? (tk.side == 0 ? 0 : n - 1) : 0;
      const int be = vert ? 0 : (tk.side == 2 ? 0 : n - 1);
      if (vert) {
        cx1 = coord(gx0, ae, S); cy1 = coord(gy0, 0, S);
        cx2 = coord(gx0, ae, S); cy2 = coord(gy0, n - 1, S);
      } else {
        cx1 = coord(gx0, 0, S); cy1 = coord(gy0, be, S);
        cx2 = coord(gx0, n - 1, S); cy2 = coord(gy0, be, S);
      }
      // Tinv entries: -(1 - j/(n-1)) for the first corner, -(j/(n-1)) for the last
      e1 = 1.0 - static_cast<double>(jj) / (n - 1);
      e2 = static_cast<double>(jj) / (n - 1);
    } else if (tk.kind == kFlux || tk.kind == kFlux3) {
      const double nxs[4] = {-1.0, 1.0, 0.0, 0.0}, nys[4] = {0.0, 0.0, -1.0, 1.0};
      nx = nxs[tk.side];
      ny = nys[tk.side];
    }
    for (int jj = 0; jj < jn; ++jj) {
      const Feat f = sf[jj];
      const double s0 = tanh(feat_z(f, x, y));
      double v;
      if (tk.kind == kValue) {
        v = s0;
      } else if (tk.kind == kLap) {
        const double s1 = __dadd_rn(1.0, -__dmul_rn(s0, s0));
        const double s2 = __dmul_rn(__dmul_rn(-2.0, s0), s1);
        const double d20 = __dmul_rn(s2, __dmul_rn(f.w0, f.w0));
        const double d02 = __dmul_rn(s2, __dmul_rn(f.w1, f.w1));
        if (var) {  // -rho (D20 + D02) - rho_x D10 - rho_y D01
          const double d10 = __dmul_rn(s1, f.w0), d01 = __dmul_rn(s1, f.w1);
          v = __dadd_rn(__dadd_rn(__dmul_rn(-rho, __dadd_rn(d20, d02)), -__dmul_rn(rhox, d10)), -__dmul_rn(rhoy, d01));
        } else {
          v = -__dadd_rn(d20, d02);
        }
      } else if (tk.kind == kFlux) {
        const double s1 = __dadd_rn(1.0, -__dmul_rn(s0, s0));
        v = __dadd_rn(__dmul_rn(nx, __dmul_rn(s1, f.w0)), __dmul_rn(ny, __dmul_rn(s1, f.w1)));
        if (var) v = __dmul_rn(v, rho);  // conormal flux rho du/dn
      } else if (tk.kind == kLapP) {
        v = feat_lap(f, x, y);
      } else if (tk.kind == kBih || tk.kind == kFlux3) {
        // sigma''' = -2 s1^2 - 2 s0 s2, sigma'''' = -6 s1 s2 - 2 s0 s3 (features.cpp:60-66)
        const double s1 = __dadd_rn(1.0, -__dmul_rn(s0, s0));
        const double s2 = __dmul_rn(__dmul_rn(-2.0, s0), s1);
        const double s3 = __dadd_rn(__dmul_rn(__dmul_rn(-2.0, s1), s1), -__dmul_rn(__dmul_rn(2.0, s0), s2));
        const double w00 = __dmul_rn(f.w0, f.w0), w11 = __dmul_rn(f.w1, f.w1);
        if (tk.kind == kBih) {  // D40 + 2 D22 + D04 (problems.cpp:88-91)
          const double s4 = __dadd_rn(__dmul_rn(__dmul_rn(-6.0, s1), s2), -__dmul_rn(__dmul_rn(2.0, s0), s3));
          const double d40 = __dmul_rn(s4, __dmul_rn(__dmul_rn(w00, f.w0), f.w0));
          const double d22 = __dmul_rn(s4, __dmul_rn(__dmul_rn(w00, f.w1), f.w1));
          const double d04 = __dmul_rn(s4, __dmul_rn(__dmul_rn(w11, f.w1), f.w1));
          v = __dadd_rn(__dadd_rn(d40, __dmul_rn(2.0, d22)), d04);
        } else {  // n . grad(lap): nx (D30 + D12) + ny (D21 + D03) (problems.cpp:123-128)
          const double d30 = __dmul_rn(s3, __dmul_rn(w00, f.w0));
          const double d12 = __dmul_rn(s3, __dmul_rn(__dmul_rn(f.w0, f.w1), f.w1));
          const double d21 = __dmul_rn(s3, __dmul_rn(w00, f.w1));
          const double d03 = __dmul_rn(s3, __dmul_rn(w11, f.w1));
          v = __dadd_rn(__dmul_rn(nx, __dadd_rn(d30, d12)), __dmul_rn(ny, __dadd_rn(d21, d03)));
        }
      } else if (tk.kind == kLapCov) {  // kLapP with the change of variables (as kValueCov)
        const double lp = feat_lap(f, x, y);
        v = 0.0;
        if (tk.flags & 1) v = -__dmul_rn(e1, feat_lap(f, cx1, cy1));
        v = (tk.flags & 1) ? __dadd_rn(v, lp) : lp;
        if (tk.flags & 2) v = __dadd_rn(v, -__dmul_rn(e2, feat_lap(f, cx2, cy2)));
      } else {  // kValueCov: sum over gamma index order first corner, point, last corner
        v = 0.0;
        if (tk.flags & 1) v = -__dmul_rn(e1, tanh(feat_z(f, cx1, cy1)));
        v = (tk.flags & 1) ? __dadd_rn(v, s0) : s0;
        if (tk.flags & 2) v = __dadd_rn(v, -__dmul_rn(e2, tanh(feat_z(f, cx2, cy2))));
      }
      const size_t col = static_cast<size_t>(j0 + jj);
      out[col * ldo + tk.row] = v;
      if (dual) Kb[col * p.ld + tk.row] = v;
    }
  }
}

/// Appended right-hand-side columns of the batched QR: column M holds f (K) / 0 (Kbar);
/// columns M+1+q hold unit vectors at the trace rows (K) / Neumann flux rows (Kbar), so the
/// QR's trailing updates produce Q^T [f E] for free.
__global__ void fill_append_kernel(FeatureArgs p) {
  const int c = blockIdx.x;  // appended column index 0..ncol-M-1
  const int t = blockIdx.y;  // matrix 0..2N-1
  const int i = t < p.N ? t : t - p.N;
  const bool bar = t >= p.N;
  const int cls = p.sub_cls[i];
  const ClassDims d = p.dims[cls];
  double* col = p.A + static_cast<size_t>(t) * p.ld * p.ncol + static_cast<size_t>(p.M + c) * p.ld;
  int unit_row = -1;
  if (c >= 1) {
    const int q = c - 1;
    if (!bar && q < d.n_gamma) unit_row = d.fixed + q;
    if (bar && q < d.nd) unit_row = d.fixed + d.nc + q;
  }
  for (int r = threadIdx.x; r < p.ld; r += blockDim.x) {
    double v = 0.0;
    if (c == 0 && !bar && r < p.m) v = p.f[static_cast<size_t>(i) * p.m + r];
    if (r == unit_row) v = 1.0;
    col[r] = v;
  }
}

/// Gaussian-random-field problem data at every row point (problems.cpp:41-66, 74-87, 117-121,
/// 157-166): one thread per (subdomain, class task), the 256 terms (sampled on the host in the
/// reference's draw order) in shared memory, summed in the reference's order. poisson_grf: the
/// forcing f = grf at the interior rows; varcoef_poisson: (rho, rho_x, rho_y) with
/// rho = tanh(grf) + 1.1 and grad rho = (1 - tanh^2) grad grf at interior and flux rows.
__global__ void __launch_bounds__(256) grf_eval_kernel(GrfArgs g) {
  __shared__ double amp[kGrfTerms], fx[kGrfTerms], fy[kGrfTerms], ph[kGrfTerms];
  for (int k = threadIdx.x; k < kGrfTerms; k += blockDim.x) {
    amp[k] = g.terms[k];
    fx[k] = g.terms[kGrfTerms + k];
    fy[k] = g.terms[2 * kGrfTerms + k];
    ph[k] = g.terms[3 * kGrfTerms + k];
  }
  __syncthreads();
  const int i = blockIdx.y;
  const int cls = g.sub_cls[i];
  const int ntask = g.cls_task_cnt[cls];
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= ntask) return;
  const Task tk = g.tasks[g.cls_task_off[cls] + t];
  const bool k_row = t < g.n_tasks_k[cls] && tk.row < g.fixed[cls];
  const bool want_f = g.problem == 3 && k_row && tk.kind == kLap;
  const bool want_rho = g.problem == 4 && (tk.kind == kLap || tk.kind == kFlux);
  if (!want_f && !want_rho) return;
  const double x = coord(g.sub_ix[i] * (g.n_grid - 1), tk.a, g.S);
  const double y = coord(g.sub_iy[i] * (g.n_grid - 1), tk.b, g.S);
  double v = 0.0, dx = 0.0, dy = 0.0;
  for (int k = 0; k < kGrfTerms; ++k) {
    // fx x + fy y + phase without FMA contraction (the host restatement's rounding)
    const double arg = __dadd_rn(__dadd_rn(__dmul_rn(fx[k], x), __dmul_rn(fy[k], y)), ph[k]);
    if (want_f) {
      v = __dadd_rn(v, __dmul_rn(amp[k], sin(arg)));
    } else {
      double sn, cs;
      sincos(arg, &sn, &cs);
      v = __dadd_rn(v, __dmul_rn(amp[k], sn));
      const double c = __dmul_rn(amp[k], cs);
      dx = __dadd_rn(dx, __dmul_rn(c, fx[k]));
      dy = __dadd_rn(dy, __dmul_rn(c, fy[k]));
    }
  }
  if (want_f) {
    g.f[static_cast<size_t>(i) * g.m + tk.row] = v;
  } else {
    const double th = tanh(v);
    const double s1 = __dadd_rn(1.0, -__dmul_rn(th, th));
    double* out = g.coef + (static_cast<size_t>(i) * g.tmax + t) * 3;
    out[0] = __dadd_rn(th, 1.1);
    out[1] = __dmul_rn(s1, dx);
    out[2] = __dmul_rn(s1, dy);
  }
}

}  // namespace

void launch_grf_eval(const GrfArgs& g, int max_tasks, cudaStream_t st) {
  dim3 grid(ceil_div(std::max(max_tasks, 1), 256), g.N);
  grf_eval_kernel<<<grid, 256, 0, st>>>(g);
  DDG_LAUNCH_CHECK();
}

namespace {
__global__ void tanh_kernel(const double* x, double* y, long long n) {
  const long long k = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k < n) y[k] = tanh(x[k]);  // the call build_features_kernel makes (same file, same flags)
}
}  // namespace

void device_tanh(int device, const double* x, double* y, long long n) {
  if (n <= 0) return;
  DDG_CUDA(cudaSetDevice(device));
  double *dx = nullptr, *dy = nullptr;
  DDG_CUDA(cudaMalloc(&dx, n * sizeof(double)));
  DDG_CUDA(cudaMalloc(&dy, n * sizeof(double)));
  DDG_CUDA(cudaMemcpy(dx, x, n * sizeof(double), cudaMemcpyHostToDevice));
  tanh_kernel<<<static_cast<unsigned>((n + 255) / 256), 256>>>(dx, dy, n);
  DDG_LAUNCH_CHECK();
  DDG_CUDA(cudaMemcpy(y, dy, n * sizeof(double), cudaMemcpyDeviceToHost));
  DDG_CUDA(cudaFree(dx));
  DDG_CUDA(cudaFree(dy));
}

void launch_build_features(const FeatureArgs& a, cudaStream_t st) {
  dim3 grid(ceil_div(a.M, 32), a.N);
  build_features_kernel<<<grid, 256, 0, st>>>(a);
  DDG_LAUNCH_CHECK();
  dim3 g2(a.ncol - a.M, 2 * a.N);
  fill_append_kernel<<<g2, 256, 0, st>>>(a);
  DDG_LAUNCH_CHECK();
}

}  // namespace ddg

// Field evaluation and error metrics on the device.
//
// Reference: sample_field + errors_from_samples (metrics.cpp:18-88) behind relative_errors
// (metrics.cpp:112-139) and oracle_check's field_diff (runner.cpp:269-281). The uniform
// n x n grid point (a, b) = (a h, b h), h = 1/(n-1), belongs to subdomain
// clamp(floor(y s)) * s + clamp(floor(x s)) (geometry.cpp:12-18); ownership is separable, so the
// host hands the kernel the a-range (and b-range) of every subdomain column (row) and a CTA
// evaluates a contiguous block of one subdomain's points with its layer staged in shared memory:
//   u = sum_j c_j tanh(z_j),  grad u = sum_j (1 - tanh^2 z_j) (w_j c_j),  z_j = w_j . x + b_j.
// The trapezoid-weighted sums (||du||^2, ||u_ref||^2, ||d grad||^2, ||grad_ref||^2) are reduced
// per CTA in a fixed order and then by one CTA (deterministic), against either the problem's
// exact solution or a second coefficient set on the same layers.
#include "common.cuh"
#include "kernels.hpp"

namespace ddg {

namespace {

constexpr int kFieldThreads = 128;
constexpr double kPiD = 3.141592653589793238462643383279502884;

/// exact solution and gradient of problem `pid` (problems.cpp:135-156 + C4's added problem)
__device__ __forceinline__ void exact_at(int pid, double x, double y, double& u, double& gx, double& gy) {
  if (pid == 0 || pid == 5) {  // poisson_sinpi, biharmonic_sinpi: sin(pi x) sin(pi y)
    const double sx = sin(kPiD * x), sy = sin(kPiD * y);
    u = sx * sy;
    gx = kPiD * cos(kPiD * x) * sy;
    gy = kPiD * sx * cos(kPiD * y);
  } else if (pid == 1) {
    const double s2 = sin(2 * kPiD * x), ey = exp(y);
    u = s2 * ey;
    gx = 2 * kPiD * cos(2 * kPiD * x) * ey;
    gy = s2 * ey;
  } else {
    const double s2 = sin(2 * kPiD * x), c3 = cos(3 * kPiD * y);
    u = s2 * c3 + x * x * y;
    gx = 2 * kPiD * cos(2 * kPiD * x) * c3 + 2 * x * y;
    gy = -3 * kPiD * s2 * sin(3 * kPiD * y) + x * x;
  }
}

__device__ __forceinline__ double trap_w(int a, int n, double h) { return (a == 0 || a == n - 1) ? h / 2 : h; }

__global__ void __launch_bounds__(kFieldThreads) field_kernel(FieldArgs f) {
  const int i = blockIdx.y;  // local subdomain
  const int ix = f.sub_ix[i], iy = f.sub_iy[i];
  const int a0 = f.lo[ix], na = f.lo[ix + 1] - a0;
  const int b0 = f.lo[iy], nbp = f.lo[iy + 1] - b0;
  const int npts = na * nbp;
  const int M = f.M;
  extern __shared__ double fs[];  // w0 | w1 | b | w0 c | w1 c | c  (| same for the reference set)
  const int nset = f.coef_ref ? 2 : 1;
  for (int j = threadIdx.x; j < M; j += blockDim.x) {
    const size_t g = static_cast<size_t>(i) * M + j;
    const double w0 = f.w0[g], w1 = f.w1[g];
    fs[j] = w0;
    fs[M + j] = w1;
    fs[2 * M + j] = f.b[g];
    for (int s = 0; s < nset; ++s) {
      const double c = (s == 0 ? f.coef : f.coef_ref)[g];
      fs[(3 + 3 * s) * M + j] = w0 * c;
      fs[(4 + 3 * s) * M + j] = w1 * c;
      fs[(5 + 3 * s) * M + j] = c;
    }
  }
  __syncthreads();
  const double h = 1.0 / (f.n - 1);
  double acc[4] = {0, 0, 0, 0};  // sum w du^2, w u_ref^2, w |d grad|^2, w |grad_ref|^2
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p < npts) {
    const int a = a0 + p % na, b = b0 + p / na;
    const double x = a * h, y = b * h;
    double u[2] = {0, 0}, gx[2] = {0, 0}, gy[2] = {0, 0};
    for (int j = 0; j < M; ++j) {
      const double t = tanh(x * fs[j] + y * fs[M + j] + fs[2 * M + j]);
      const double d = 1.0 - t * t;
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        if (s < nset) {
          u[s] += t * fs[(5 + 3 * s) * M + j];
          gx[s] += d * fs[(3 + 3 * s) * M + j];
          gy[s] += d * fs[(4 + 3 * s) * M + j];
        }
      }
    }
    const size_t id = static_cast<size_t>(b) * f.n + a;
    if (f.u) f.u[id] = u[0];
    if (f.gx) f.gx[id] = gx[0];
    if (f.gy) f.gy[id] = gy[0];
    double ru, rgx, rgy;
    if (f.coef_ref) {
      ru = u[1];
      rgx = gx[1];
      rgy = gy[1];
    } else {
      exact_at(f.problem, x, y, ru, rgx, rgy);
    }
    const double w = trap_w(b, f.n, h) * trap_w(a, f.n, h);
    const double du = u[0] - ru, dgx = gx[0] - rgx, dgy = gy[0] - rgy;
    acc[0] = w * du * du;
    acc[1] = w * ru * ru;
    acc[2] = w * (dgx * dgx + dgy * dgy);
    acc[3] = w * (rgx * rgx + rgy * rgy);
  }
  // fixed-order CTA reduction: warp xor trees, then the warps in order
  __shared__ double red[kFieldThreads / 32][4];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    double v = acc[k];
    for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) red[warp][k] = v;
  }
  __syncthreads();
  if (threadIdx.x < 4) {
    double v = 0;
    for (int q = 0; q < kFieldThreads / 32; ++q) v += red[q][threadIdx.x];
    f.part[(static_cast<size_t>(blockIdx.y) * gridDim.x + blockIdx.x) * 4 + threadIdx.x] = v;
  }
}

/// sums[k] = sum over the CTA partials in index order (one CTA, lanes stride, fixed tree)
__global__ void field_sum_kernel(const double* part, int nparts, double* sums) {
  __shared__ double red[4][32];
  const int k = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double v = 0;
  for (int q = lane; q < nparts; q += 32) v += part[static_cast<size_t>(q) * 4 + k];
  for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0) red[k][0] = v;
  __syncthreads();
  if (threadIdx.x < 4) sums[threadIdx.x] = red[threadIdx.x][0];
}

}  // namespace

int field_parts(const FieldArgs& f, int max_pts) { return f.N * ceil_div(max_pts, kFieldThreads); }

void launch_field(const FieldArgs& f, int max_pts, double* sums, cudaStream_t st) {
  const int chunks = ceil_div(max_pts, kFieldThreads);
  const size_t smem = static_cast<size_t>(f.coef_ref ? 9 : 6) * f.M * sizeof(double);
  DDG_CUDA(cudaFuncSetAttribute(field_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  field_kernel<<<dim3(chunks, f.N), kFieldThreads, smem, st>>>(f);
  DDG_LAUNCH_CHECK();
  field_sum_kernel<<<1, 128, 0, st>>>(f.part, f.N * chunks, sums);
  DDG_LAUNCH_CHECK();
}

}  // namespace ddg

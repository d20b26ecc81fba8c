// Probe: how many clusters of size CL (1 CTA of 256 threads and `smem` bytes per SM) can be
// co-resident on this GPU (cudaOccupancyMaxActiveClusters) — the GPC granularity that sizes the
// QR trailing-update clusters.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* p) { extern __shared__ double s[]; if (p) p[0] = s[threadIdx.x]; }
int main() {
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int smem : {100 * 1024, 200 * 1024}) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int cl = 1; cl <= 16; ++cl) {
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(cl * 64);
      cfg.blockDim = dim3(256);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cl;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      int n = -1;
      cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k, &cfg);
      printf("smem %3d KB cluster %2d: max active clusters %4d -> CTAs %4d %s\n", smem / 1024, cl, n, n * cl,
             e == cudaSuccess ? "" : cudaGetErrorString(e));
    }
  }
  return 0;
}

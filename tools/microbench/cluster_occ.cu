// How many thread-block clusters of size C can be resident at once with one
// 288-thread CTA per SM and ~200 KB of dynamic shared memory (B200: 148 SMs).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int* x) { if (x && threadIdx.x == 9999) x[0] = 1; }
int main() {
  cudaDeviceProp pr;
  cudaGetDeviceProperties(&pr, 0);
  printf("%s SMs %d smem/block optin %zu\n", pr.name, pr.multiProcessorCount, pr.sharedMemPerBlockOptin);
  for (int smem : {100 * 1024, 200 * 1024, 225 * 1024}) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int c : {1, 2, 4, 8, 16}) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(c * 64);
      cfg.blockDim = dim3(288);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = c; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      cfg.attrs = at; cfg.numAttrs = 1;
      int n = -1;
      cudaError_t e = cudaOccupancyMaxActiveClusters(&n, k, &cfg);
      printf("smem %6d cluster %2d: max active clusters %4d -> CTAs %4d (%s)\n", smem, c, n, n * c,
             cudaGetErrorString(e));
    }
  }
  return 0;
}

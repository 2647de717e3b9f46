// How many clusters of 2 / 4 / 8 / 16 CTAs with one CTA per SM (218 KB of dynamic shared memory,
// 256 threads) can be co-resident on this GPU (cudaOccupancyMaxActiveClusters)?
#include <cstdio>
#include <cuda_runtime.h>
__global__ void __launch_bounds__(256, 1) k(int* out) {
  extern __shared__ int sm[];
  if (threadIdx.x == 0 && out) sm[0] = out[0];
}
int main() {
  const int smem = 218 * 1024;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cs : {1, 2, 4, 8, 16}) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(cs * 8);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    at[1].id = cudaLaunchAttributeClusterDimension;
    at[1].val.clusterDim.x = cs;
    at[1].val.clusterDim.y = 1;
    at[1].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    int ncl = -1;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&ncl, k, &cfg);
    printf("cluster %2d: max active clusters %d (%d CTAs) %s\n", cs, ncl, ncl * cs, e == cudaSuccess ? "" : cudaGetErrorString(e));
    cudaGetLastError();
  }
  return 0;
}

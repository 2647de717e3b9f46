// Does the driver accept a cooperative launch with a cluster dimension on B200?
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int* out) {
  unsigned r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  if (threadIdx.x == 0) atomicAdd(out, 1 + (int)r * 0);
}
int main() {
  int* d;
  cudaMalloc(&d, 4);
  cudaMemset(d, 0, 4);
  for (int cs : {4, 8, 16}) {
    cudaLaunchConfig_t cfg{};
    int grid = 148 / cs * cs;
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(288);
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    at[1].id = cudaLaunchAttributeClusterDimension;
    at[1].val.clusterDim.x = cs;
    at[1].val.clusterDim.y = 1;
    at[1].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    if (cs > 8) cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaError_t e = cudaLaunchKernelEx(&cfg, k, d);
    cudaError_t e2 = cudaDeviceSynchronize();
    int ncl = 0;
    cfg.numAttrs = 2;
    cudaOccupancyMaxActiveClusters(&ncl, k, &cfg);
    printf("cluster %d grid %d: launch=%s sync=%s maxActiveClusters=%d\n", cs, grid, cudaGetErrorString(e),
           cudaGetErrorString(e2), ncl);
  }
  return 0;
}

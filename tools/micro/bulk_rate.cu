// Microbenchmark: how many cp.async.bulk (1-D TMA) copies per second one SM sustains as a
// function of the copy size — the block-Gram ring issues 64-128 copies of 0.5-5 KB per block.
// One CTA per SM (or 16 CTAs), one thread issues COPIES copies of BYTES bytes (strided source,
// like column slices), 32 in flight against one mbarrier per batch.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2104_12570_b200/csrc -I../../include bulk_rate.cu -o bulk_rate
#include <cstdio>
#include <cuda_runtime.h>

#include "bak_common.cuh"
using namespace bak;

__global__ void __launch_bounds__(64, 1) k(const char* src, size_t stride, int bytes, int batches, int per_batch,
                                            long long* cyc) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint64_t pol = policy_evict_last();
    const char* p = src + static_cast<size_t>(blockIdx.x) * bytes;
    const long long t0 = clock64();
    uint32_t ph = 0;
    for (int b = 0; b < batches; ++b) {
      mbar_arrive_expect_tx(&bar, static_cast<uint32_t>(bytes) * per_batch);
      for (int i = 0; i < per_batch; ++i)
        bulk_g2s(smem + static_cast<size_t>(i) * bytes, p + (static_cast<size_t>(b % 64) * per_batch + i) * stride,
                 bytes, &bar, pol);
      while (!mbar_test(&bar, ph)) {
      }
      ph ^= 1u;
    }
    cyc[blockIdx.x] = clock64() - t0;
  }
}

int main() {
  const size_t stride = 8000;  // C4: ldx * 8 bytes
  const size_t total = stride * 64 * 64 + (1 << 20);
  char* src;
  long long* cyc;
  cudaMalloc(&src, total);
  cudaMemset(src, 1, total);
  cudaMalloc(&cyc, 256 * sizeof(long long));
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int grid : {1, 16, 148})
    for (int bytes : {512, 2048, 4096}) {
      for (int per_batch : {8, 32}) {
        const int batches = 2000;
        k<<<grid, 64, 200 * 1024>>>(src, stride, bytes, batches, per_batch, cyc);
        k<<<grid, 64, 200 * 1024>>>(src, stride, bytes, batches, per_batch, cyc);
        if (cudaDeviceSynchronize() != cudaSuccess) {
          printf("failed: %s\n", cudaGetErrorString(cudaGetLastError()));
          return 1;
        }
        long long h[256], mx = 0;
        cudaMemcpy(h, cyc, grid * sizeof(long long), cudaMemcpyDeviceToHost);
        for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
        printf("grid=%3d bytes=%4d per_batch=%2d: %7.1f cycles per copy, %6.1f B/clk/SM\n", grid, bytes, per_batch,
               double(mx) / (double(batches) * per_batch), double(bytes) * batches * per_batch / double(mx));
      }
    }
  return 0;
}

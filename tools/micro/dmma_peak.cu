// Microbenchmark: sustained fp64 DMMA (mma.sync.m8n8k4.f64) throughput with
// operands in registers (no shared-memory traffic), 4x4 independent
// accumulator tiles per warp like the G kernel, W warps per CTA, one wave of
// CTAS_PER_SM CTAs on every SM.  Upper bound for gram_dmma_kernel.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 dmma_peak.cu -o dmma_peak
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__global__ void k(int iters, double* out) {
  double acc[4][4][2];
  for (int a = 0; a < 4; ++a)
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  double af[4], bf[4];
  for (int t = 0; t < 4; ++t) {
    af[t] = 1e-3 * (threadIdx.x + t);
    bf[t] = 1e-3 * (threadIdx.x - t);
  }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) dmma(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
  }
  double s = 0.0;
  for (int a = 0; a < 4; ++a)
    for (int b = 0; b < 4; ++b) s += acc[a][b][0] + acc[a][b][1];
  if (s == 12345.678) out[0] = s;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 8);
  for (int warps : {4, 8, 16}) {
    for (int ctas : {1, 2, 4}) {
      const int iters = 20000;
      k<<<sms * ctas, warps * 32>>>(100, out);
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      k<<<sms * ctas, warps * 32>>>(iters, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      const double flops = 2.0 * 8 * 8 * 4 * 16.0 * iters * warps * sms * ctas;
      printf("warps/CTA=%2d CTAs/SM=%d: %.1f TFLOP/s fp64 DMMA (%s)\n", warps, ctas, flops / ms / 1e9,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}

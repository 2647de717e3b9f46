// Microbenchmark: sustained legacy warp-level TF32 MMA (mma.sync m16n8k8,
// fp32 accumulate) throughput on sm_100a, operands in registers, 4x4
// independent accumulator tiles per warp.  Sizes a 3xTF32 fp32 G kernel.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tf32_peak.cu -o tf32_peak
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void mma_tf32(float* d, const unsigned* a, const unsigned* b) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

__global__ void k(int iters, float* out) {
  float acc[4][4][4];
  for (int a = 0; a < 4; ++a)
    for (int b = 0; b < 4; ++b)
      for (int c = 0; c < 4; ++c) acc[a][b][c] = 0.f;
  unsigned af[4][4], bf[4][2];
  for (int t = 0; t < 4; ++t) {
    for (int c = 0; c < 4; ++c) af[t][c] = __float_as_uint(1e-3f * (threadIdx.x + t + c));
    for (int c = 0; c < 2; ++c) bf[t][c] = __float_as_uint(1e-3f * (threadIdx.x - t + c));
  }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) mma_tf32(acc[a][b], af[a], bf[b]);
  }
  float s = 0.f;
  for (int a = 0; a < 4; ++a)
    for (int b = 0; b < 4; ++b)
      for (int c = 0; c < 4; ++c) s += acc[a][b][c];
  if (s == 12345.678f) out[0] = s;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* out;
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
      const double flops = 2.0 * 16 * 8 * 8 * 16.0 * iters * warps * sms * ctas;
      printf("warps/CTA=%2d CTAs/SM=%d: %.1f TFLOP/s tf32 mma.sync (%s)\n", warps, ctas, flops / ms / 1e9,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}

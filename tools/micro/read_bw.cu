// Microbenchmark: sustained HBM read bandwidth (16-byte non-coherent loads,
// grid-stride, 4 loads in flight per thread) over a buffer larger than L2 —
// the ceiling for a pass that only reads x.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 read_bw.cu -o read_bw
#include <cstdio>
#include <cuda_runtime.h>

__global__ void rd(const int4* __restrict__ p, size_t n, int* out) {
  int acc = 0;
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x;
  size_t i = static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n; i += 4 * stride) {
    const int4 a = __ldg(p + i), b = __ldg(p + i + stride), c = __ldg(p + i + 2 * stride), d = __ldg(p + i + 3 * stride);
    acc ^= a.x ^ b.y ^ c.z ^ d.w;
  }
  for (; i < n; i += stride) acc ^= __ldg(p + i).x;
  if (acc == 0x12345678) out[0] = acc;
}

int main() {
  const size_t bytes = 16ull << 30;  // 16 GiB
  int4* p;
  int* out;
  if (cudaMalloc(&p, bytes) != cudaSuccess) return 1;
  cudaMalloc(&out, 4);
  cudaMemset(p, 1, bytes);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int per_sm : {2, 4, 8}) {
    for (int threads : {256, 512, 1024}) {
      rd<<<sms * per_sm, threads>>>(p, bytes / 16, out);
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      for (int r = 0; r < 5; ++r) rd<<<sms * per_sm, threads>>>(p, bytes / 16, out);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      printf("CTAs/SM=%d threads=%4d: %.0f GB/s read\n", per_sm, threads, 5.0 * bytes / (ms / 1e3) / 1e9);
    }
  }
  return 0;
}

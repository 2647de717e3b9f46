// Microbenchmark: latency of one dependent CTA-wide sum (the per-column floor
// of the exact sweep).  nvcc -gencode arch=compute_100a,code=sm_100a -O3 reduce_latency.cu
#include <cstdio>
#include <cuda_runtime.h>

template <typename T>
__device__ __forceinline__ T wsum(T v) {
  for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <typename T, int NW>
__global__ void k(int iters, T* out, long long* cyc) {
  __shared__ T red[2][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  T p = T(threadIdx.x) * T(1e-3);
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    T v = wsum(p);
    if (NW > 1) {
      if (lane == 0) red[i & 1][warp] = v;
      __syncthreads();
      T s = T(0);
#pragma unroll
      for (int w = 0; w < NW; ++w) s += red[i & 1][w];
      v = s;
    }
    p = p * T(0.5) + v * T(1e-9);  // dependent on the sum
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { out[0] = p; cyc[0] = (t1 - t0) / iters; }
}

template <typename T, int NW>
void run(const char* name) {
  T* out; long long* cyc; cudaMalloc(&out, 8); cudaMalloc(&cyc, 8);
  k<T, NW><<<1, NW * 32>>>(1000, out, cyc);
  k<T, NW><<<1, NW * 32>>>(100000, out, cyc);
  long long c; cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("%s warps=%d : %lld cycles per dependent CTA sum\n", name, NW, c);
}

int main() {
  run<float, 1>("f32"); run<float, 2>("f32"); run<float, 4>("f32"); run<float, 8>("f32");
  run<double, 1>("f64"); run<double, 2>("f64"); run<double, 4>("f64"); run<double, 8>("f64");
  return 0;
}

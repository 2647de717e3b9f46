// Microbenchmark: tensor memory (TMEM) as plain on-chip storage — tcgen05.ld /
// tcgen05.st throughput per SM when W warps each move C 32-bit columns of their
// own lane quarter per round trip (the XT sweep stashes one column slice of x
// there between its dot and its update).  One CTA per SM, clock64 around R rounds.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2104_12570_b200/csrc tmem_bw.cu -o tmem_bw
#include <cstdio>
#include <cuda_runtime.h>

#include "bak_tmem.cuh"

using namespace bak;

template <int N>
struct Ops;
#define OPS(N)                                                                                 \
  template <>                                                                                  \
  struct Ops<N> {                                                                              \
    static __device__ __forceinline__ void ld(uint32_t a, uint32_t (&r)[N]) { tmem_ld_x##N(a, r); } \
    static __device__ __forceinline__ void st(uint32_t a, const uint32_t (&r)[N]) { tmem_st_x##N(a, r); } \
  };
OPS(8) OPS(16) OPS(32) OPS(64)

// mode 0: ld only, 1: st only, 2: ld -> modify -> st (same address), 3: ld + lds interleaved
template <int N>
__global__ void __launch_bounds__(256, 1) bw(int mode, int cols, int rounds, long long* cycles, unsigned* sink) {
  __shared__ uint32_t slot;
  __shared__ double buf[8 * 16 * 32];  // 32 KB of shared memory for mode 3
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) tmem_alloc512(static_cast<uint32_t>(__cvta_generic_to_shared(&slot)));
  tmem_fence_before_sync();
  __syncthreads();
  tmem_fence_after_sync();
  const uint32_t base = slot + (static_cast<uint32_t>((warp & 3) * 32) << 16) + static_cast<uint32_t>((warp >> 2) * cols);
  uint32_t r[N];
#pragma unroll
  for (int i = 0; i < N; ++i) r[i] = threadIdx.x * 131 + i;
  for (int c = 0; c < cols; c += N) Ops<N>::st(base + c, r);  // initialise
  tmem_wait_st();
  for (int i = threadIdx.x; i < 8 * 16 * 32; i += blockDim.x) buf[i] = i;
  __syncthreads();
  unsigned acc = 0;
  double dacc = 0.0;
  const long long t0 = clock64();
  for (int it = 0; it < rounds; ++it) {
    for (int c = 0; c < cols; c += N) {
      if (mode == 0) {
        Ops<N>::ld(base + c, r);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < N; ++i) acc += r[i];
      } else if (mode == 1) {
#pragma unroll
        for (int i = 0; i < N; ++i) r[i] += it;
        Ops<N>::st(base + c, r);
      } else if (mode == 2) {
        Ops<N>::ld(base + c, r);
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < N; ++i) r[i] += 1;
        Ops<N>::st(base + c, r);
      } else {
        Ops<N>::ld(base + c, r);
        double v[N / 2];
#pragma unroll
        for (int i = 0; i < N / 2; ++i) v[i] = buf[(warp * 16 + ((c / 2 + i) & 15)) * 32 + lane];
        tmem_wait_ld();
#pragma unroll
        for (int i = 0; i < N; ++i) acc += r[i];
#pragma unroll
        for (int i = 0; i < N / 2; ++i) dacc += v[i];
      }
    }
    if (mode == 1 || mode == 2) tmem_wait_st();
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  if (acc == 0x9e3779b9u || dacc == 1.2345) sink[0] = acc;
  tmem_fence_before_sync();
  __syncthreads();
  if (warp == 0) tmem_dealloc512(slot);
}

template <int N>
void run(int warps, int mode, int cols, long long* cyc, unsigned* sink) {
  const int rounds = 2000;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  bw<N><<<sms, warps * 32>>>(mode, cols, rounds, cyc, sink);
  bw<N><<<sms, warps * 32>>>(mode, cols, rounds, cyc, sink);
  if (cudaDeviceSynchronize() != cudaSuccess) {
    printf("launch failed: %s\n", cudaGetErrorString(cudaGetLastError()));
    return;
  }
  long long h[256];
  cudaMemcpy(h, cyc, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (int i = 0; i < sms; ++i) mx = h[i] > mx ? h[i] : mx;
  const double bytes = static_cast<double>(rounds) * warps * 32.0 * cols * 4.0 * (mode == 2 ? 2.0 : 1.0);
  static const char* names[] = {"ld", "st", "ld+st", "ld||lds"};
  printf("x%-2d warps=%d cols/warp=%3d %-7s: %8.1f cycles/round, %6.1f B/clk/SM (TMEM bytes)\n", N, warps, cols,
         names[mode], static_cast<double>(mx) / rounds, bytes / static_cast<double>(mx));
}

int main() {
  long long* cyc;
  unsigned* sink;
  cudaMalloc(&cyc, 256 * sizeof(long long));
  cudaMalloc(&sink, 4);
  for (int warps : {4, 7, 8})
    for (int mode : {0, 1, 2, 3}) {
      const int cols = 128;  // per warp (two warps share a lane quarter when warps > 4)
      run<8>(warps, mode, cols, cyc, sink);
      run<16>(warps, mode, cols, cyc, sink);
      run<32>(warps, mode, cols, cyc, sink);
      run<64>(warps, mode, cols, cyc, sink);
    }
  return 0;
}

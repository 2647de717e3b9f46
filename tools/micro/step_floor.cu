// Microbenchmark: the per-column floor of the on-chip exact sweep step
// (quotient, fused e -= d x_t ; p += x_{t+1}.e over E rows per thread, warp
// butterfly, per-warp slots + barrier, fixed-order tree) with x read from a
// shared-memory ring and no producer.  Compare with the real kernel's ns per
// column (tools/sweep_probe.py).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 step_floor.cu -o step_floor
#include <cstdio>
#include <cuda_runtime.h>

template <typename T>
__device__ __forceinline__ T wsum(T v) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <typename T, int NW, int E, int VARIANT>
__global__ void k(int iters, T* out, long long* cyc) {
  constexpr int NT = NW * 32;
  __shared__ T red[2][NW];
  __shared__ T ring[4][NT * E];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < 4 * NT * E; i += NT) (&ring[0][0])[i] = T(((i * 37) % 101) - 50) * T(1e-3);
  __syncthreads();
  T ev[E], xc[E], xn[E];
#pragma unroll
  for (int k = 0; k < E; ++k) {
    ev[k] = T(1) + T(k) * T(1e-3);
    xc[k] = ring[0][tid + k * NT];
    xn[k] = ring[1][tid + k * NT];
  }
  T P = T(1e-3), n2 = T(3), r = T(1) / T(3);
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    T q0 = P * r;
    T rem = fma(-q0, n2, P);
    T d = fma(rem, r, q0);
    T acc[4] = {0, 0, 0, 0};
#pragma unroll
    for (int k = 0; k < E; ++k) {
      ev[k] = ev[k] - xc[k] * d;
      acc[k & 3] = fma(xn[k], ev[k], acc[k & 3]);
    }
    T pv = (acc[0] + acc[1]) + (acc[2] + acc[3]);
#pragma unroll
    for (int k = 0; k < E; ++k) {
      xc[k] = xn[k];
      xn[k] = ring[(i + 2) & 3][tid + k * NT];
    }
    pv = wsum(pv);
    if (NW > 1) {
      if (lane == 0) red[i & 1][warp] = pv;
      if (VARIANT == 0) __syncthreads();
      else asm volatile("bar.sync 1, %0;" ::"r"(NT) : "memory");
      T s[NW];
#pragma unroll
      for (int w = 0; w < NW; ++w) s[w] = red[i & 1][w];
#pragma unroll
      for (int h = NW / 2; h >= 1; h >>= 1)
#pragma unroll
        for (int w = 0; w < h; ++w) s[w] += s[w + h];
      pv = s[0];
    }
    P = pv * T(1e-6) + T(1e-3);
  }
  long long t1 = clock64();
  if (tid == 0) {
    out[0] = P + ev[0];
    cyc[0] = (t1 - t0) / iters;
  }
}


// Same step with x streamed from global memory by the consumers themselves:
// each thread cp.async's its own E rows of column i+D into a D-deep smem ring
// and waits only on its own copies (cp.async.wait_group), no producer warp.
template <int D>
__device__ __forceinline__ void wait_d() { asm volatile("cp.async.wait_group %0;" ::"n"(D) : "memory"); }

template <typename T, int NW, int E, int D>
__global__ void kc(int iters, const T* __restrict__ x, long long ld, T* out, long long* cyc) {
  constexpr int NT = NW * 32;
  __shared__ T red[2][NW];
  extern __shared__ __align__(16) unsigned char dsm[];
  T* ring = reinterpret_cast<T*>(dsm);  // [D][NT*E]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  auto issue = [&](int col) {
    const T* src = x + (long long)col * ld + tid;
    T* dst = ring + (col % D) * NT * E + tid;
#pragma unroll
    for (int k = 0; k < E; ++k) {
      const unsigned sa = (unsigned)__cvta_generic_to_shared(dst + k * NT);
      asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(sa), "l"(src + k * NT), "n"(sizeof(T)) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  for (int c = 0; c < D; ++c) issue(c);
  T ev[E], xc[E], xn[E];
  wait_d<D - 1>();
#pragma unroll
  for (int k = 0; k < E; ++k) { ev[k] = T(1) + T(k) * T(1e-3); xc[k] = ring[0 * NT * E + tid + k * NT]; }
  wait_d<D - 2>();
#pragma unroll
  for (int k = 0; k < E; ++k) xn[k] = ring[1 * NT * E + tid + k * NT];
  T P = T(1e-3), n2 = T(3), r = T(1) / T(3);
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    T q0 = P * r;
    T rem = fma(-q0, n2, P);
    T d = fma(rem, r, q0);
    T acc[4] = {0, 0, 0, 0};
#pragma unroll
    for (int k = 0; k < E; ++k) {
      ev[k] = ev[k] - xc[k] * d;
      acc[k & 3] = fma(xn[k], ev[k], acc[k & 3]);
    }
    T pv = (acc[0] + acc[1]) + (acc[2] + acc[3]);
    // slot of column i is free now (xc held it): refill with column i+D
    issue(i + D);
    wait_d<D - 2>();  // column i+2 landed (own copies)
#pragma unroll
    for (int k = 0; k < E; ++k) {
      xc[k] = xn[k];
      xn[k] = ring[((i + 2) % D) * NT * E + tid + k * NT];
    }
    pv = wsum(pv);
    if (NW > 1) {
      if (lane == 0) red[i & 1][warp] = pv;
      asm volatile("bar.sync 1, %0;" ::"r"(NT) : "memory");
      T s[NW];
#pragma unroll
      for (int w = 0; w < NW; ++w) s[w] = red[i & 1][w];
#pragma unroll
      for (int h = NW / 2; h >= 1; h >>= 1)
#pragma unroll
        for (int w = 0; w < h; ++w) s[w] += s[w + h];
      pv = s[0];
    }
    P = pv * T(1e-6) + T(1e-3);
  }
  long long t1 = clock64();
  if (tid == 0) { out[0] = P + ev[0]; cyc[0] = (t1 - t0) / iters; }
}

template <typename T, int NW, int E, int D>
void runc(const char* name, int ncols) {
  T* out; long long* cyc; T* x;
  const long long ld = NW * 32 * E;
  cudaMalloc(&out, 8); cudaMalloc(&cyc, 8);
  cudaMalloc(&x, sizeof(T) * ld * (ncols + D + 2));
  cudaMemset(x, 0, sizeof(T) * ld * (ncols + D + 2));
  const int smem = D * NW * 32 * E * sizeof(T);
  cudaFuncSetAttribute(kc<T, NW, E, D>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  kc<T, NW, E, D><<<1, NW * 32, smem>>>(1000, x, ld, out, cyc);
  kc<T, NW, E, D><<<1, NW * 32, smem>>>(ncols, x, ld, out, cyc);
  long long c = 0;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  cudaError_t e = cudaGetLastError();
  printf("%s cp.async warps=%d E=%d D=%d cols=%d: %lld cycles per column step %s\n", name, NW, E, D, ncols, c,
         e == cudaSuccess ? "" : cudaGetErrorString(e));
  cudaFree(x);
}

template <typename T, int NW, int E, int V>
void run(const char* name) {
  T* out;
  long long* cyc;
  cudaMalloc(&out, 8);
  cudaMalloc(&cyc, 8);
  k<T, NW, E, V><<<1, NW * 32>>>(1000, out, cyc);
  k<T, NW, E, V><<<1, NW * 32>>>(100000, out, cyc);
  long long c = 0;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  cudaError_t e = cudaGetLastError();
  printf("%s warps=%d E=%d bar=%s: %lld cycles per column step %s\n", name, NW, E, V ? "named" : "sync", c,
         e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main() {
  run<double, 4, 8, 0>("f64");
  run<double, 4, 8, 1>("f64");
  run<double, 1, 32, 0>("f64");
  run<double, 2, 16, 1>("f64");
  run<double, 8, 4, 1>("f64");
  run<float, 4, 8, 1>("f32");
  run<float, 1, 32, 0>("f32");
  runc<double, 4, 8, 8>("f64", 200000);
  runc<double, 4, 8, 16>("f64", 200000);
  runc<double, 4, 8, 16>("f64", 1000000);
  runc<float, 4, 8, 16>("f32", 1000000);
  return 0;
}

// Microbenchmark: which piece of the real on-chip sweep step costs what.
// Starts from the step_floor body (fp64, 4 warps x 8 rows, smem ring) and adds
// the real kernel's pieces one at a time (feature bits below).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 step_bisect.cu -o step_bisect
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

enum { F_BARRED = 1, F_MBAR = 2, F_META = 4, F_AUPD = 8, F_LOOP = 16, F_PROD = 32 };

__device__ __forceinline__ double wsum(double v) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ uint32_t sa(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ bool try_wait(uint64_t* bar, uint32_t par) {
  uint32_t ok;
  asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
               : "=r"(ok) : "r"(sa(bar)), "r"(par) : "memory");
  return ok != 0;
}
__device__ __forceinline__ bool bar_or(int n, int pred) {
  uint32_t r;
  asm volatile("{\n\t.reg .pred p, q;\n\tsetp.ne.u32 q, %1, 0;\n\tbar.red.or.pred p, 1, %2, q;\n\tselp.u32 %0, 1, 0, p;\n\t}"
               : "=r"(r) : "r"(static_cast<uint32_t>(pred)), "r"(n) : "memory");
  return r != 0;
}

constexpr int NW = 4, E = 8, NT = NW * 32;

template <int F>
__global__ void k(int iters, double* out, long long* cyc, double* ag, int64_t ncols, double* hist) {
  __shared__ double red[2][NW];
  __shared__ double ring[4][NT * E];
  __shared__ uint64_t bars[2];
  __shared__ struct { int64_t col; double n2, rinv, pad; } meta[4];
  __shared__ volatile int stop;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < 4 * NT * E; i += blockDim.x) (&ring[0][0])[i] = double(((i * 37) % 101) - 50) * 1e-3;
  if (tid < 4) { meta[tid].col = tid; meta[tid].n2 = 3.0; meta[tid].rinv = 1.0 / 3.0; }
  if (tid == 0) {
    stop = 0;
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bars[0])));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bars[1])));
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(&bars[0])) : "memory");  // phase 0 of bars[0] done
  }
  __syncthreads();
  if ((F & F_PROD) && tid >= NT) {  // a producer warp waiting on a stage that is never released
    if (lane == 0) {
      while (!try_wait(&bars[1], 0)) {
        if (stop) break;
        long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t == 0) break;
      }
    }
    return;
  }
  double ev[E], xc[E], xn[E];
#pragma unroll
  for (int kk = 0; kk < E; ++kk) { ev[kk] = 1.0 + kk * 1e-3; xc[kk] = ring[0][tid + kk * NT]; xn[kk] = ring[1][tid + kk * NT]; }
  double P = 1e-3, n2 = 3.0, r = 1.0 / 3.0, n2n = 3.0, rn = 1.0 / 3.0;
  const bool upd = warp == 1;
  int64_t c0 = 0, c1 = 1, kcol = 0, sweep = 0;
  double a0 = 0.0, a1 = 0.0;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    double q0 = P * r;
    double rem = fma(-q0, n2, P);
    double d = fma(rem, r, q0);
    double acc[4] = {0, 0, 0, 0};
#pragma unroll
    for (int kk = 0; kk < E; ++kk) {
      ev[kk] = __dsub_rn(ev[kk], __dmul_rn(xc[kk], d));
      acc[kk & 3] = fma(xn[kk], ev[kk], acc[kk & 3]);
    }
    double pv = (acc[0] + acc[1]) + (acc[2] + acc[3]);
    const int slot = (i + 2) & 3;
    if (F & F_MBAR) {
      if (!try_wait(&bars[0], 0)) {
        while (!try_wait(&bars[0], 0)) {}
      }
    }
    int64_t c2 = c1;
    if (F & F_META) {
      c2 = meta[slot].col;
      n2n = meta[slot].n2;
      rn = meta[slot].rinv;
    }
#pragma unroll
    for (int kk = 0; kk < E; ++kk) { xc[kk] = xn[kk]; xn[kk] = ring[slot][tid + kk * NT]; }
    if ((F & F_AUPD) && upd) {
      const double na = a0 + d;
      ag[c0] = na;
      a0 = (c1 == c0) ? na : a1;
      a1 = ag[c2];
    }
    pv = wsum(pv);
    if (lane == 0) red[i & 1][warp] = pv;
    if (F & F_BARRED) {
      if (bar_or(NT, 0)) break;
    } else {
      asm volatile("bar.sync 1, %0;" ::"r"(NT) : "memory");
    }
    double s[NW];
#pragma unroll
    for (int w = 0; w < NW; ++w) s[w] = red[i & 1][w];
#pragma unroll
    for (int h = NW / 2; h >= 1; h >>= 1)
#pragma unroll
      for (int w = 0; w < h; ++w) s[w] += s[w + h];
    P = s[0] * 1e-6 + 1e-3;
    if (F & F_META) { n2 = n2n; r = rn; }
    if (F & F_LOOP) {
      const bool last = kcol == ncols - 1;
      if (last) {
        if (tid == 0 && hist) hist[sweep & 1023] = P;
        ++sweep;
        if (P < -1.0) break;
        kcol = 0;
      } else {
        ++kcol;
      }
    }
    c0 = c1; c1 = c2;
  }
  long long t1 = clock64();
  if (tid == 0) { stop = 1; out[0] = P + ev[0] + a0; cyc[0] = (t1 - t0) / iters; }
}

template <int F>
void run(const char* name, double* ag, double* hist) {
  double* out; long long* cyc;
  cudaMalloc(&out, 8); cudaMalloc(&cyc, 8);
  const int nt = NT + ((F & F_PROD) ? 32 : 0);
  k<F><<<1, nt>>>(1000, out, cyc, ag, 20000, hist);
  k<F><<<1, nt>>>(100000, out, cyc, ag, 20000, hist);
  long long c = 0;
  cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
  printf("%-40s %lld cycles per column step %s\n", name, c, cudaGetErrorString(cudaGetLastError()));
}

int main() {
  double *ag, *hist;
  cudaMalloc(&ag, 8 * 100000); cudaMemset(ag, 0, 8 * 100000);
  cudaMalloc(&hist, 8 * 1024);
  run<0>("floor", ag, hist);
  run<F_BARRED>("+bar.red.or", ag, hist);
  run<F_MBAR>("+try_wait", ag, hist);
  run<F_META>("+meta", ag, hist);
  run<F_AUPD>("+a update", ag, hist);
  run<F_LOOP>("+loop bookkeeping", ag, hist);
  run<F_PROD>("+producer warp", ag, hist);
  run<F_BARRED | F_MBAR | F_META>("+bar.red.or+try_wait+meta", ag, hist);
  run<F_BARRED | F_MBAR | F_META | F_AUPD | F_LOOP | F_PROD>("all", ag, hist);
  return 0;
}

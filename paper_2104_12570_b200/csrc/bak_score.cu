// Greedy column scoring (reference select.py:56-85).
//
//   scores[j] = <e,e> - <x_j,e>^2 / <x_j,x_j>     (T arithmetic, as the
//               reference's e2 - g*g/norms2 with g = x.T @ e), +inf for
//               excluded or zero-norm columns; best = argmin, ties to the
//               lowest index.
//
// One pass over x: score_dots_kernel tiles (rows x 16-column groups); every
// CTA reads its row tile of e once per group and 16 columns of x (coalesced
// along rows), reduces in a fixed order (warp butterfly, warps in index
// order) and writes one partial per column and tile (+ the tile's sum e^2).
// score_final_kernel sums the tile partials in tile order, applies the closed
// form and a per-CTA argmin; score_argmin_kernel reduces the CTA winners in
// index order.  HBM-bound: obs*vars*sizeof(T) + e once per column group.
#include <type_traits>

#include "bak_common.cuh"
#include "bak_sweep.cuh"

namespace bak {
namespace {

constexpr int kThreads = 256;
constexpr int kGroup = 16;  // columns per CTA

template <typename T>
__global__ void __launch_bounds__(kThreads) score_dots_kernel(const T* __restrict__ x, int64_t obs, int64_t ldx,
                                                              int64_t vars, const T* __restrict__ e,
                                                              double* __restrict__ part, double* __restrict__ e2part,
                                                              int64_t tile) {
  __shared__ T red[kGroup + 1][kThreads / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t rb = static_cast<int64_t>(blockIdx.x) * tile;
  const int64_t re = imin64(obs, rb + tile);
  const int64_t c0 = static_cast<int64_t>(blockIdx.y) * kGroup;
  const int ncol = static_cast<int>(imin64(kGroup, vars - c0));
  const bool first = blockIdx.y == 0;
  T acc[kGroup];
#pragma unroll
  for (int u = 0; u < kGroup; ++u) acc[u] = T(0);
  T q = T(0);
  for (int64_t r = rb + tid; r < re; r += kThreads) {
    const T ev = e[r];
    if (first) q = Num<T>::fma(ev, ev, q);
#pragma unroll
    for (int u = 0; u < kGroup; ++u)
      if (u < ncol) acc[u] = Num<T>::fma(__ldcs(x + (c0 + u) * ldx + r), ev, acc[u]);
  }
#pragma unroll
  for (int u = 0; u < kGroup; ++u) acc[u] = warp_sum(acc[u]);
  q = warp_sum(q);
  if (lane == 0) {
#pragma unroll
    for (int u = 0; u < kGroup; ++u) red[u][warp] = acc[u];
    red[kGroup][warp] = q;
  }
  __syncthreads();
  if (tid < ncol) {
    T s = T(0);
    for (int w = 0; w < kThreads / 32; ++w) s = Num<T>::add(s, red[tid][w]);
    part[static_cast<int64_t>(blockIdx.x) * vars + c0 + tid] = static_cast<double>(s);
  }
  if (first && tid == kGroup) {
    T s = T(0);
    for (int w = 0; w < kThreads / 32; ++w) s = Num<T>::add(s, red[kGroup][w]);
    e2part[blockIdx.x] = static_cast<double>(s);
  }
}

// (score, index) order of numpy.argmin: NaN first, then smaller, ties to the lower index
__device__ __forceinline__ bool better(double a, int64_t ia, double b, int64_t ib) {
  const bool na = a != a, nb = b != b;
  if (na || nb) return na && (!nb || ia < ib);
  return a < b || (a == b && ia < ib);
}

__device__ __forceinline__ void warp_best(double& v, int64_t& i) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    const double v2 = __shfl_xor_sync(0xffffffffu, v, o);
    const int64_t i2 = __shfl_xor_sync(0xffffffffu, i, o);
    if (better(v2, i2, v, i)) {
      v = v2;
      i = i2;
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(kThreads) score_final_kernel(const double* __restrict__ part,
                                                               const double* __restrict__ e2part, int ntiles,
                                                               int64_t vars, const T* __restrict__ n2g,
                                                               const uint8_t* __restrict__ excluded,
                                                               double* __restrict__ scores,
                                                               double* __restrict__ cta_val,
                                                               int64_t* __restrict__ cta_idx) {
  __shared__ double sv[kThreads / 32];
  __shared__ int64_t si[kThreads / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t j = static_cast<int64_t>(blockIdx.x) * kThreads + tid;
  double v = __longlong_as_double(0x7ff0000000000000LL);  // +inf
  int64_t idx = j < vars ? j : INT64_MAX;
  if (j < vars) {
    T e2 = T(0);
    for (int t = 0; t < ntiles; ++t) e2 = Num<T>::add(e2, static_cast<T>(e2part[t]));
    const T n2 = n2g[j];
    const bool ok = n2 > T(0) && !(excluded && excluded[j]);
    if (ok) {
      T g = T(0);
      for (int t = 0; t < ntiles; ++t) g = Num<T>::add(g, static_cast<T>(part[static_cast<int64_t>(t) * vars + j]));
      v = static_cast<double>(Num<T>::sub(e2, Num<T>::div(Num<T>::mul(g, g), n2)));
    }
    scores[j] = v;
  }
  warp_best(v, idx);
  if (lane == 0) {
    sv[warp] = v;
    si[warp] = idx;
  }
  __syncthreads();
  if (tid == 0) {
    double bv = sv[0];
    int64_t bi = si[0];
    for (int w = 1; w < kThreads / 32; ++w)
      if (better(sv[w], si[w], bv, bi)) {
        bv = sv[w];
        bi = si[w];
      }
    cta_val[blockIdx.x] = bv;
    cta_idx[blockIdx.x] = bi;
  }
}

__global__ void score_argmin_kernel(const double* __restrict__ cta_val, const int64_t* __restrict__ cta_idx, int n,
                                    int64_t* __restrict__ best) {
  if (threadIdx.x != 0) return;
  double bv = cta_val[0];
  int64_t bi = cta_idx[0];
  for (int b = 1; b < n; ++b)
    if (better(cta_val[b], cta_idx[b], bv, bi)) {
      bv = cta_val[b];
      bi = cta_idx[b];
    }
  best[0] = bi;
  best[1] = (bv == bv && bv < __longlong_as_double(0x7ff0000000000000LL)) ? 1 : 0;  // finite
}

// short columns (obs <= kShortMax): e staged once per CTA in shared memory,
// one warp per column (lane-strided rows), score and running argmin in the
// same kernel; per-CTA winners go to score_argmin_kernel.
constexpr int kShortMax = 4096;

template <typename T>
__global__ void __launch_bounds__(kThreads) score_short_kernel(const T* __restrict__ x, int64_t obs, int64_t ldx,
                                                               int64_t vars, const T* __restrict__ e,
                                                               const T* __restrict__ n2g,
                                                               const uint8_t* __restrict__ excluded,
                                                               double* __restrict__ scores,
                                                               double* __restrict__ cta_val,
                                                               int64_t* __restrict__ cta_idx) {
  __shared__ T es[kShortMax];
  __shared__ T red[kThreads / 32];
  __shared__ double sv[kThreads / 32];
  __shared__ int64_t si[kThreads / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n = static_cast<int>(obs);
  T q = T(0);
  for (int r = tid; r < n; r += kThreads) {
    const T v = e[r];
    es[r] = v;
    q = Num<T>::fma(v, v, q);
  }
  q = warp_sum(q);
  if (lane == 0) red[warp] = q;
  __syncthreads();
  T e2 = T(0);
  for (int w = 0; w < kThreads / 32; ++w) e2 = Num<T>::add(e2, red[w]);  // same order in every CTA
  double bv = __longlong_as_double(0x7ff0000000000000LL);
  int64_t bi = INT64_MAX;
  const int64_t wstride = static_cast<int64_t>(gridDim.x) * (kThreads / 32);
  for (int64_t j = static_cast<int64_t>(blockIdx.x) * (kThreads / 32) + warp; j < vars; j += wstride) {
    const T* __restrict__ col = x + j * ldx;
    // 16-byte vector loads (columns are 16-byte aligned), lane-strided
    constexpr int VEC = 16 / sizeof(T);
    using V = typename std::conditional<sizeof(T) == 8, double2, float4>::type;
    const int nvec = n / VEC;
    T acc[VEC];
#pragma unroll
    for (int k = 0; k < VEC; ++k) acc[k] = T(0);
#pragma unroll 2
    for (int i = lane; i < nvec; i += 32) {
      const V v = __ldcs(reinterpret_cast<const V*>(col) + i);
      const T* xv = reinterpret_cast<const T*>(&v);
#pragma unroll
      for (int k = 0; k < VEC; ++k) acc[k] = Num<T>::fma(xv[k], es[i * VEC + k], acc[k]);
    }
    for (int r = nvec * VEC + lane; r < n; r += 32) acc[0] = Num<T>::fma(col[r], es[r], acc[0]);
    T gs = acc[0];
#pragma unroll
    for (int k = 1; k < VEC; ++k) gs = Num<T>::add(gs, acc[k]);
    const T g = warp_sum(gs);
    const T n2 = n2g[j];
    double v = __longlong_as_double(0x7ff0000000000000LL);
    if (n2 > T(0) && !(excluded && excluded[j]))
      v = static_cast<double>(Num<T>::sub(e2, Num<T>::div(Num<T>::mul(g, g), n2)));
    if (lane == 0) scores[j] = v;
    if (better(v, j, bv, bi)) {
      bv = v;
      bi = j;
    }
  }
  if (lane == 0) {
    sv[warp] = bv;
    si[warp] = bi;
  }
  __syncthreads();
  if (tid == 0) {
    double b = sv[0];
    int64_t ib = si[0];
    for (int w = 1; w < kThreads / 32; ++w)
      if (better(sv[w], si[w], b, ib)) {
        b = sv[w];
        ib = si[w];
      }
    cta_val[blockIdx.x] = b;
    cta_idx[blockIdx.x] = ib;
  }
}

struct ScorePlan {
  int ngroups, ntiles, nfinal;
  int64_t tile;
};

int short_ctas(int64_t vars) {
  return static_cast<int>(imax64(1, imin64(8LL * device_sms(), (vars + kThreads / 32 - 1) / (kThreads / 32))));
}

ScorePlan score_plan(int64_t obs, int64_t vars) {
  ScorePlan p;
  p.ngroups = static_cast<int>((vars + kGroup - 1) / kGroup);
  const int64_t want_ctas = 4LL * device_sms();
  int64_t nt = imax64(1, want_ctas / p.ngroups);
  nt = imin64(nt, imax64(1, (obs + 4 * kThreads - 1) / (4 * kThreads)));  // >= 4 rows per thread
  p.tile = round_up((obs + nt - 1) / nt, kThreads);
  p.ntiles = static_cast<int>((obs + p.tile - 1) / p.tile);
  p.nfinal = static_cast<int>((vars + kThreads - 1) / kThreads);
  if (obs <= kShortMax) p.nfinal = static_cast<int>(imax64(p.nfinal, short_ctas(vars)));
  if (gram_tma_supported(vars) && obs > kShortMax) {
    // tall: the GRAM pass kernel in dot-only mode (TMA-fed, ~HBM speed) makes the partials
    p.ntiles = static_cast<int>(imax64(p.ntiles, gram_tma_grid(BAK_F32)));
  }
  return p;
}

}  // namespace
}  // namespace bak

using namespace bak;

extern "C" int64_t bak_score_columns_workspace(int dtype, int64_t obs, int64_t vars) {
  (void)dtype;
  const ScorePlan p = score_plan(obs, vars);
  return round_up(static_cast<int64_t>(p.ntiles) * vars * 8, 256) + round_up(p.ntiles * 8, 256) +
         2 * round_up(p.nfinal * 8, 256) + 512;
}

extern "C" int bak_score_columns(int dtype, const void* x, int64_t obs, int64_t vars, int64_t ldx, const void* e,
                                 const void* norms2, const uint8_t* excluded, double* scores, int64_t* best,
                                 void* workspace, int64_t workspace_bytes, void* stream) {
  g_err_clear();
  if ((dtype != BAK_F32 && dtype != BAK_F64) || obs < 1 || vars < 1 || ldx < obs || !x || !e || !norms2 ||
      !scores || !best) {
    set_error("bak_score_columns: bad arguments");
    return BAK_EINVAL;
  }
  if (!workspace || workspace_bytes < bak_score_columns_workspace(dtype, obs, vars)) {
    set_error("bak_score_columns: workspace too small");
    return BAK_EWORKSPACE;
  }
  const ScorePlan p = score_plan(obs, vars);
  char* w = static_cast<char*>(workspace);
  double* part = reinterpret_cast<double*>(w);
  w += round_up(static_cast<int64_t>(p.ntiles) * vars * 8, 256);
  double* e2part = reinterpret_cast<double*>(w);
  w += round_up(p.ntiles * 8, 256);
  double* cta_val = reinterpret_cast<double*>(w);
  w += round_up(p.nfinal * 8, 256);
  int64_t* cta_idx = reinterpret_cast<int64_t*>(w);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const size_t ts = dtype_size(dtype);
  if (obs <= kShortMax && reinterpret_cast<uintptr_t>(x) % 16 == 0 && (ldx * ts) % 16 == 0) {
    const int nc = short_ctas(vars);
    if (dtype == BAK_F64)
      score_short_kernel<double><<<nc, kThreads, 0, st>>>(static_cast<const double*>(x), obs, ldx, vars,
                                                          static_cast<const double*>(e),
                                                          static_cast<const double*>(norms2), excluded, scores,
                                                          cta_val, cta_idx);
    else
      score_short_kernel<float><<<nc, kThreads, 0, st>>>(static_cast<const float*>(x), obs, ldx, vars,
                                                         static_cast<const float*>(e),
                                                         static_cast<const float*>(norms2), excluded, scores,
                                                         cta_val, cta_idx);
    score_argmin_kernel<<<1, 32, 0, st>>>(cta_val, cta_idx, nc, best);
    count_launches(2);
    BAK_CHECK_CUDA(cudaGetLastError());
    return BAK_OK;
  }
  if (gram_tma_supported(vars) && reinterpret_cast<uintptr_t>(x) % 16 == 0 && (ldx * ts) % 16 == 0 &&
      reinterpret_cast<uintptr_t>(e) % 16 == 0) {
    // dot-only GRAM pass: gpart[b][j] = partial <x_j, e>, sqpart[b] = partial <e, e>
    const int nblk = gram_tma_grid(dtype);
    int64_t* done = reinterpret_cast<int64_t*>(cta_idx + p.nfinal);  // zeroed flag after the winners
    BAK_CHECK_CUDA(cudaMemsetAsync(done, 0, 8, st));
    if (int rc = launch_gram_pass_tma(dtype, x, obs, ldx, vars, const_cast<void*>(e), part, 0, 1, part, e2part,
                                      done, st))
      return rc;
    if (dtype == BAK_F64)
      score_final_kernel<double><<<p.nfinal, kThreads, 0, st>>>(part, e2part, nblk, vars,
                                                                static_cast<const double*>(norms2), excluded, scores,
                                                                cta_val, cta_idx);
    else
      score_final_kernel<float><<<p.nfinal, kThreads, 0, st>>>(part, e2part, nblk, vars,
                                                               static_cast<const float*>(norms2), excluded, scores,
                                                               cta_val, cta_idx);
    score_argmin_kernel<<<1, 32, 0, st>>>(cta_val, cta_idx, p.nfinal, best);
    count_launches(2);
    BAK_CHECK_CUDA(cudaGetLastError());
    return BAK_OK;
  }
  const dim3 g1(p.ntiles, p.ngroups);
  if (dtype == BAK_F64) {
    score_dots_kernel<double><<<g1, kThreads, 0, st>>>(static_cast<const double*>(x), obs, ldx, vars,
                                                       static_cast<const double*>(e), part, e2part, p.tile);
    score_final_kernel<double><<<p.nfinal, kThreads, 0, st>>>(part, e2part, p.ntiles, vars,
                                                              static_cast<const double*>(norms2), excluded, scores,
                                                              cta_val, cta_idx);
  } else {
    score_dots_kernel<float><<<g1, kThreads, 0, st>>>(static_cast<const float*>(x), obs, ldx, vars,
                                                      static_cast<const float*>(e), part, e2part, p.tile);
    score_final_kernel<float><<<p.nfinal, kThreads, 0, st>>>(part, e2part, p.ntiles, vars,
                                                             static_cast<const float*>(norms2), excluded, scores,
                                                             cta_val, cta_idx);
  }
  score_argmin_kernel<<<1, 32, 0, st>>>(cta_val, cta_idx, p.nfinal, best);
  count_launches(3);
  BAK_CHECK_CUDA(cudaGetLastError());
  return BAK_OK;
}

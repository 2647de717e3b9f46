// One-pass HBM kernels around the sweep:
//   colnorms  : n2_j = <x_j, x_j>          (core.py:116-127, bak.py:185; ||y||^2 bak.py:168)
//   residual  : out = y - x @ a            (bak.py:130 final residual, bak.py:189 warm start)
//   diffnorm2 : sum double(u - v)^2        (drift, bak.py:133)
// All reductions have a fixed, shape-only order (deterministic run to run).
#include <cstdio>

#include "bak_common.cuh"

namespace bak {
namespace {

constexpr int kNormThreads = 256;
constexpr int64_t kNormChunk = 16384;  // rows per warp work item

template <typename T>
__global__ void __launch_bounds__(kNormThreads) colnorms_partial(const T* __restrict__ x, int64_t obs, int64_t ldx,
                                                                 int64_t vars, int64_t chunk, int64_t nchunks,
                                                                 T* __restrict__ out) {
  const int64_t item = static_cast<int64_t>(blockIdx.x) * (kNormThreads / kWarp) + threadIdx.x / kWarp;
  if (item >= vars * nchunks) return;
  const int lane = threadIdx.x & 31;
  const int64_t j = item / nchunks, c = item - j * nchunks;
  const T* col = x + j * ldx;
  const int64_t r0 = c * chunk;
  const int64_t r1 = min(obs, r0 + chunk);
  T acc[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) acc[k] = T(0);
  int64_t r = r0 + lane;
  for (; r + 7 * kWarp < r1; r += 8 * kWarp) {
    T v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = __ldg(col + r + k * kWarp);
#pragma unroll
    for (int k = 0; k < 8; ++k) acc[k] = Num<T>::fma(v[k], v[k], acc[k]);
  }
  for (; r < r1; r += kWarp) {
    T v = __ldg(col + r);
    acc[0] = Num<T>::fma(v, v, acc[0]);
  }
  T s = Num<T>::add(Num<T>::add(Num<T>::add(acc[0], acc[1]), Num<T>::add(acc[2], acc[3])),
                    Num<T>::add(Num<T>::add(acc[4], acc[5]), Num<T>::add(acc[6], acc[7])));
  s = warp_sum(s);
  if (lane == 0) out[item] = s;
}

template <typename T>
__global__ void __launch_bounds__(kNormThreads) colnorms_final(const T* __restrict__ part, int64_t vars,
                                                               int64_t nchunks, T* __restrict__ out) {
  const int64_t j = static_cast<int64_t>(blockIdx.x) * (kNormThreads / kWarp) + threadIdx.x / kWarp;
  if (j >= vars) return;
  const int lane = threadIdx.x & 31;
  T s = T(0);
  for (int64_t c = lane; c < nchunks; c += kWarp) s = Num<T>::add(s, part[j * nchunks + c]);
  s = warp_sum(s);
  if (lane == 0) out[j] = s;
}

// ---- residual: out = y - x @ a --------------------------------------------
constexpr int kGemvThreads = 256;
constexpr int kGemvRows = 4;  // rows per thread
constexpr int64_t kGemvTile = kGemvThreads * kGemvRows;

template <typename T>
__global__ void __launch_bounds__(kGemvThreads) gemv_partial(const T* __restrict__ x, int64_t obs, int64_t ldx,
                                                             int64_t vars, const T* __restrict__ a,
                                                             const T* __restrict__ y, int64_t nsplit,
                                                             int64_t cols_per_split, T* __restrict__ out) {
  const int64_t tile = blockIdx.x / nsplit;
  const int64_t split = blockIdx.x - tile * nsplit;
  const int64_t j0 = split * cols_per_split;
  const int64_t j1 = min(vars, j0 + cols_per_split);
  int64_t rows[kGemvRows];
  bool ok[kGemvRows];
  T acc[kGemvRows];
#pragma unroll
  for (int k = 0; k < kGemvRows; ++k) {
    rows[k] = tile * kGemvTile + threadIdx.x + k * kGemvThreads;
    ok[k] = rows[k] < obs;
    acc[k] = T(0);
  }
  for (int64_t j = j0; j < j1; ++j) {
    const T aj = __ldg(a + j);
    const T* col = x + j * ldx;
#pragma unroll
    for (int k = 0; k < kGemvRows; ++k)
      if (ok[k]) acc[k] = Num<T>::fma(__ldg(col + rows[k]), aj, acc[k]);
  }
#pragma unroll
  for (int k = 0; k < kGemvRows; ++k) {
    if (!ok[k]) continue;
    if (nsplit == 1)
      out[rows[k]] = Num<T>::sub(y[rows[k]], acc[k]);
    else
      out[split * obs + rows[k]] = acc[k];
  }
}

template <typename T>
__global__ void __launch_bounds__(kGemvThreads) gemv_final(const T* __restrict__ part, int64_t obs, int64_t nsplit,
                                                           const T* __restrict__ y, T* __restrict__ out) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * kGemvThreads + threadIdx.x;
  if (i >= obs) return;
  T s = T(0);
  for (int64_t k = 0; k < nsplit; ++k) s = Num<T>::add(s, part[k * obs + i]);
  out[i] = Num<T>::sub(y[i], s);
}

// ---- drift: sum double(u - v)^2 --------------------------------------------
constexpr int kDiffThreads = 256;
constexpr int kDiffBlocks = 512;

template <typename T>
__global__ void __launch_bounds__(kDiffThreads) diff_partial(const T* __restrict__ u, const T* __restrict__ v,
                                                             int64_t n, double* __restrict__ part) {
  __shared__ double ws[kDiffThreads / kWarp];
  const int64_t per = (n + gridDim.x - 1) / gridDim.x;
  const int64_t b0 = blockIdx.x * per, b1 = min(n, b0 + per);
  double acc = 0.0;
  for (int64_t i = b0 + threadIdx.x; i < b1; i += kDiffThreads) {
    const double d = static_cast<double>(Num<T>::sub(u[i], v[i]));
    acc = __fma_rn(d, d, acc);
  }
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x / kWarp] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < kDiffThreads / kWarp; ++w) s += ws[w];
    part[blockIdx.x] = s;
  }
}

__global__ void diff_final(const double* __restrict__ part, int n, double* __restrict__ out) {
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += kWarp) s += part[i];
  s = warp_sum(s);
  if (threadIdx.x == 0) out[0] = s;
}

int64_t norm_chunks(int64_t obs) { return obs <= kNormChunk ? 1 : (obs + kNormChunk - 1) / kNormChunk; }

void gemv_split(int64_t obs, int64_t vars, int64_t& nsplit, int64_t& per) {
  const int64_t tiles = (obs + kGemvTile - 1) / kGemvTile;
  const int64_t want = 4 * static_cast<int64_t>(device_sms());
  nsplit = (want + tiles - 1) / tiles;
  const int64_t max_split = (vars + 63) / 64;
  if (nsplit > max_split) nsplit = max_split;
  if (nsplit < 1) nsplit = 1;
  per = (vars + nsplit - 1) / nsplit;
  nsplit = (vars + per - 1) / per;
}

template <typename T>
int colnorms_t(const void* xv, int64_t obs, int64_t vars, int64_t ldx, void* normsv, void* ws, int64_t wsb,
               cudaStream_t st) {
  const T* x = static_cast<const T*>(xv);
  T* norms = static_cast<T*>(normsv);
  const int64_t nch = norm_chunks(obs);
  const int64_t chunk = nch == 1 ? obs : kNormChunk;
  const int64_t items = vars * nch;
  const int wpb = kNormThreads / kWarp;
  if (nch == 1) {
    colnorms_partial<T><<<static_cast<unsigned>((items + wpb - 1) / wpb), kNormThreads, 0, st>>>(x, obs, ldx, vars,
                                                                                                 chunk, 1, norms);
    count_launches(1);
  } else {
    if (wsb < static_cast<int64_t>(items * sizeof(T))) {
      set_error("bak_colnorms: workspace too small");
      return BAK_EWORKSPACE;
    }
    T* part = static_cast<T*>(ws);
    colnorms_partial<T><<<static_cast<unsigned>((items + wpb - 1) / wpb), kNormThreads, 0, st>>>(x, obs, ldx, vars,
                                                                                                 chunk, nch, part);
    count_launches(1);
    colnorms_final<T><<<static_cast<unsigned>((vars + wpb - 1) / wpb), kNormThreads, 0, st>>>(part, vars, nch,
                                                                                              norms);
    count_launches(1);
  }
  BAK_CHECK_CUDA(cudaGetLastError());
  return BAK_OK;
}

template <typename T>
int residual_t(const void* xv, int64_t obs, int64_t vars, int64_t ldx, const void* av, const void* yv, void* outv,
               void* ws, int64_t wsb, cudaStream_t st) {
  int64_t nsplit, per;
  gemv_split(obs, vars, nsplit, per);
  const int64_t tiles = (obs + kGemvTile - 1) / kGemvTile;
  const T* x = static_cast<const T*>(xv);
  const T* a = static_cast<const T*>(av);
  const T* y = static_cast<const T*>(yv);
  T* out = static_cast<T*>(outv);
  if (nsplit == 1) {
    gemv_partial<T><<<static_cast<unsigned>(tiles), kGemvThreads, 0, st>>>(x, obs, ldx, vars, a, y, 1, per, out);
    count_launches(1);
  } else {
    if (wsb < static_cast<int64_t>(nsplit * obs * sizeof(T))) {
      set_error("bak_residual: workspace too small");
      return BAK_EWORKSPACE;
    }
    T* part = static_cast<T*>(ws);
    gemv_partial<T><<<static_cast<unsigned>(tiles * nsplit), kGemvThreads, 0, st>>>(x, obs, ldx, vars, a, y,
                                                                                     nsplit, per, part);
    count_launches(1);
    gemv_final<T><<<static_cast<unsigned>((obs + kGemvThreads - 1) / kGemvThreads), kGemvThreads, 0, st>>>(
        part, obs, nsplit, y, out);
    count_launches(1);
  }
  BAK_CHECK_CUDA(cudaGetLastError());
  return BAK_OK;
}

template <typename T>
int diff_t(const void* u, const void* v, int64_t n, double* out, void* ws, int64_t wsb, cudaStream_t st) {
  if (wsb < static_cast<int64_t>(kDiffBlocks * sizeof(double))) {
    set_error("bak_diff_norm2: workspace too small");
    return BAK_EWORKSPACE;
  }
  double* part = static_cast<double*>(ws);
  diff_partial<T><<<kDiffBlocks, kDiffThreads, 0, st>>>(static_cast<const T*>(u), static_cast<const T*>(v), n, part);
  count_launches(1);
  diff_final<<<1, kWarp, 0, st>>>(part, kDiffBlocks, out);
  count_launches(1);
  BAK_CHECK_CUDA(cudaGetLastError());
  return BAK_OK;
}

}  // namespace
}  // namespace bak

using namespace bak;

extern "C" int64_t bak_colnorms_workspace(int dtype, int64_t obs, int64_t vars) {
  const int64_t nch = norm_chunks(obs);
  return nch == 1 ? 0 : nch * vars * static_cast<int64_t>(dtype_size(dtype));
}

extern "C" int bak_colnorms(int dtype, const void* x, int64_t obs, int64_t vars, int64_t ldx, void* norms2,
                            void* workspace, int64_t workspace_bytes, void* stream) {
  if (obs < 1 || vars < 1 || ldx < obs || !x || !norms2) {
    set_error("bak_colnorms: bad arguments (obs=%lld vars=%lld ldx=%lld)", (long long)obs, (long long)vars,
              (long long)ldx);
    return BAK_EINVAL;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (dtype == BAK_F64) return colnorms_t<double>(x, obs, vars, ldx, norms2, workspace, workspace_bytes, st);
  if (dtype == BAK_F32) return colnorms_t<float>(x, obs, vars, ldx, norms2, workspace, workspace_bytes, st);
  set_error("bak_colnorms: unknown dtype %d", dtype);
  return BAK_EINVAL;
}

extern "C" int64_t bak_residual_workspace(int dtype, int64_t obs, int64_t vars) {
  int64_t nsplit, per;
  gemv_split(obs, vars, nsplit, per);
  return nsplit == 1 ? 0 : nsplit * obs * static_cast<int64_t>(dtype_size(dtype));
}

extern "C" int bak_residual(int dtype, const void* x, int64_t obs, int64_t vars, int64_t ldx, const void* a,
                            const void* y, void* out, void* workspace, int64_t workspace_bytes, void* stream) {
  if (obs < 1 || vars < 1 || ldx < obs || !x || !a || !y || !out) {
    set_error("bak_residual: bad arguments");
    return BAK_EINVAL;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (dtype == BAK_F64) return residual_t<double>(x, obs, vars, ldx, a, y, out, workspace, workspace_bytes, st);
  if (dtype == BAK_F32) return residual_t<float>(x, obs, vars, ldx, a, y, out, workspace, workspace_bytes, st);
  set_error("bak_residual: unknown dtype %d", dtype);
  return BAK_EINVAL;
}

extern "C" int bak_diff_norm2(int dtype, const void* u, const void* v, int64_t n, double* out, void* workspace,
                              int64_t workspace_bytes, void* stream) {
  if (n < 0 || !out || (n > 0 && (!u || !v))) {
    set_error("bak_diff_norm2: bad arguments");
    return BAK_EINVAL;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (dtype == BAK_F64) return diff_t<double>(u, v, n, out, workspace, workspace_bytes, st);
  if (dtype == BAK_F32) return diff_t<float>(u, v, n, out, workspace, workspace_bytes, st);
  set_error("bak_diff_norm2: unknown dtype %d", dtype);
  return BAK_EINVAL;
}

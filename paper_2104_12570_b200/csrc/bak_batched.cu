// Batched many-small-systems solve (north-star component (4)): one CTA per
// system runs the whole of solve_bak (bak.py:146-195) for that system.
//
//  - x (obs x vars, column-major) is brought into shared memory ONCE with a
//    single cp.async.bulk when that leaves >= 8 systems per SM; otherwise
//    (C5: 512 x 32 fp32 = 64 KiB -> only 3 per SM) columns are streamed from
//    L2/HBM every sweep by many more resident systems (HBM-bound, 2.2x faster
//    on C5).
//  - e lives in registers (E rows per thread, rows tid + k*NT).
//  - per column: fused  e -= d_j x_j ; p += x_next . e  then one block
//    reduction (warp butterfly, + per-warp slots when NT > 32).
//  - zero-norm columns are skipped in-kernel (bak.py:101-103), zero targets
//    short-circuit (bak.py:168-170), early break per sweep (bak.py:106-111),
//    final residual y - x a and the drift flag (bak.py:127-143) are computed in
//    the same CTA.
#include <cstdio>
#include <cstdlib>

#include "bak_common.cuh"

namespace bak {
namespace {

struct BatchedParams {
  const void* x;
  int64_t obs, vars, ldx, x_stride, nsys;
  const void* y;
  int64_t y_stride;
  const void* norms2;
  const double* ynorm2;
  void* a;
  int warm;
  void* resid;
  int64_t max_iter;
  double tol, drift_tol;
  double* history;
  int64_t* status;
  int x_in_smem;
};

// correctly rounded a/b from r = RN(1/b) (one Markstein correction)
template <typename T>
__device__ __forceinline__ T quotient(T a, T b, T r) {
  const T q0 = Num<T>::mul(a, r);
  const T rem = Num<T>::fma(-q0, b, a);
  return Num<T>::fma(rem, r, q0);
}

template <typename T>
__device__ __forceinline__ T block_sum(T v, T* red, int nwarps) {
  v = warp_sum(v);
  if (nwarps == 1) return v;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) red[warp] = v;
  __syncthreads();
  T s = T(0);
  for (int w = 0; w < nwarps; ++w) s = Num<T>::add(s, red[w]);
  __syncthreads();  // red reusable
  return s;
}

template <typename T, int E, int NT_, bool SMEM>
__global__ void __launch_bounds__(NT_) batched_kernel(const BatchedParams prm) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  constexpr int NT = NT_;
  constexpr int nwarps = NT >> 5;
  const int tid = threadIdx.x;
  const int64_t sys = blockIdx.x;
  const int64_t obs = prm.obs, vars = prm.vars, ldx = prm.ldx;
  const T* __restrict__ xg = static_cast<const T*>(prm.x) + sys * prm.x_stride;
  const T* __restrict__ y = static_cast<const T*>(prm.y) + sys * prm.y_stride;
  const T* __restrict__ n2g = static_cast<const T*>(prm.norms2) + sys * vars;
  T* __restrict__ ag = static_cast<T*>(prm.a) + sys * vars;
  T* __restrict__ rg = static_cast<T*>(prm.resid) + sys * prm.y_stride;
  int64_t* status = prm.status + 4 * sys;
  double* hist = prm.history ? prm.history + sys * prm.max_iter : nullptr;

  size_t off = 0;
  T* xs = reinterpret_cast<T*>(smem_raw);
  if (SMEM) off += static_cast<size_t>(vars) * ldx * sizeof(T);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw + off);
  off += 16;
  T* n2s = reinterpret_cast<T*>(smem_raw + off);
  off += round16(vars * sizeof(T));
  T* as = reinterpret_cast<T*>(smem_raw + off);
  off += round16(vars * sizeof(T));
  T* rinv = reinterpret_cast<T*>(smem_raw + off);
  off += round16(vars * sizeof(T));
  int* nz = reinterpret_cast<int*>(smem_raw + off);
  off += round16((vars + 1) * sizeof(int));
  T* red = reinterpret_cast<T*>(smem_raw + off);
  double* redd = reinterpret_cast<double*>(smem_raw + off);

  if (SMEM) {
    if (tid == 0) {
      mbar_init(bar, 1);
      fence_mbar_init();
    }
    __syncthreads();
    if (tid == 0) {
      const uint32_t bytes = static_cast<uint32_t>(vars * ldx * sizeof(T));
      mbar_arrive_expect_tx(bar, bytes);
      bulk_g2s(xs, xg, bytes, bar, policy_evict_first());
    }
  }
  const double yn2 = prm.ynorm2[sys];
  for (int64_t j = tid; j < vars; j += NT) {
    n2s[j] = n2g[j];
    as[j] = prm.warm ? ag[j] : T(0);
  }
  if (SMEM) {
    const uint64_t t0 = globaltimer();
    while (!mbar_test(bar, 0))
      if (globaltimer() - t0 > kTimeoutNs) {
        if (tid == 0) status[3] = BAK_ETIMEOUT;
        break;
      }
  }
  __syncthreads();
  const T* X = SMEM ? xs : xg;

  const int kv = static_cast<int>(imax64(0, imin64(E, (obs - tid + NT - 1) / NT)));
  T yv[E], ev[E];
#pragma unroll
  for (int k = 0; k < E; ++k) yv[k] = (k < kv) ? y[tid + k * NT] : T(0);

  if (yn2 == 0.0) {  // bak.py:168-170 -> _zero_report
    for (int64_t j = tid; j < vars; j += NT) ag[j] = T(0);
#pragma unroll
    for (int k = 0; k < E; ++k)
      if (k < kv) rg[tid + k * NT] = T(0);
    if (tid == 0) {
      status[0] = 0;
      status[1] = 1;
      status[2] = 0;
    }
    return;
  }
  const double thresh2 = prm.tol > 0 ? prm.tol * prm.tol * yn2 : -1.0;

  // e = y (or y - x a0 for a warm start, bak.py:188-191)
#pragma unroll
  for (int k = 0; k < E; ++k) ev[k] = yv[k];
  if (prm.warm) {
    T acc[E];
#pragma unroll
    for (int k = 0; k < E; ++k) acc[k] = T(0);
    for (int64_t j = 0; j < vars; ++j) {
      const T aj = as[j];
#pragma unroll
      for (int k = 0; k < E; ++k)
        if (k < kv) acc[k] = Num<T>::fma(X[j * ldx + tid + k * NT], aj, acc[k]);
    }
#pragma unroll
    for (int k = 0; k < E; ++k) ev[k] = (k < kv) ? Num<T>::sub(yv[k], acc[k]) : T(0);
  }

  // nonzero-norm column list (zero-norm columns are skipped, bak.py:101-103)
  for (int64_t j = tid; j < vars; j += NT) rinv[j] = n2s[j] != T(0) ? Num<T>::div(T(1), n2s[j]) : T(0);
  if (tid == 0) {
    int n = 0;
    for (int64_t j = 0; j < vars; ++j)
      if (n2s[j] != T(0)) nz[n++] = static_cast<int>(j);
    nz[vars] = n;
  }
  __syncthreads();
  const int nnz = nz[vars];
  int64_t sweeps = 0;
  bool converged = false;
  const bool full_rows = kv == E;  // uniform within a warp unless obs is ragged
  auto load_col = [&](int j, T (&xr)[E]) {
    const T* c = X + static_cast<int64_t>(j) * ldx + tid;
    if (full_rows) {
#pragma unroll
      for (int k = 0; k < E; ++k) xr[k] = c[k * NT];
    } else {
#pragma unroll
      for (int k = 0; k < E; ++k) xr[k] = (k < kv) ? c[k * NT] : T(0);
    }
  };
  if (nnz > 0) {
    // two register buffers with alternating roles (loop unrolled by 2: no copies)
    T xa[E], xb[E];
    load_col(nz[0], xa);
    load_col(nz[nnz > 1 ? 1 : 0], xb);
    T p = T(0);
#pragma unroll
    for (int k = 0; k < E; ++k) p = Num<T>::fma(xa[k], ev[k], p);
    T P = block_sum(p, red, nwarps);
    int idx = 0;
    // one column step: update with xc (column nz[idx]), dot with xn (next column),
    // then refill xc with the column after next.  Returns true when the solve ends.
    auto step = [&](T (&xc)[E], T (&xn)[E]) -> bool {
      const int j = nz[idx];
      const bool last = idx == nnz - 1;
      const T d = quotient(P, n2s[j], rinv[j]);
      T acc[4] = {T(0), T(0), T(0), T(0)};
#pragma unroll
      for (int k = 0; k < E; ++k) {
        ev[k] = Num<T>::sub(ev[k], Num<T>::mul(xc[k], d));
        acc[k & 3] = Num<T>::fma(xn[k], ev[k], acc[k & 3]);
      }
      const T pv = Num<T>::add(Num<T>::add(acc[0], acc[1]), Num<T>::add(acc[2], acc[3]));
      int idx2 = idx + 2;
      while (idx2 >= nnz) idx2 -= nnz;
      load_col(nz[idx2], xc);  // overlaps the reduction below
      if (tid == 0) as[j] = Num<T>::add(as[j], d);
      if (last) {
        T qa[4] = {T(0), T(0), T(0), T(0)};
#pragma unroll
        for (int k = 0; k < E; ++k) qa[k & 3] = Num<T>::fma(ev[k], ev[k], qa[k & 3]);
        const T Q = block_sum(Num<T>::add(Num<T>::add(qa[0], qa[1]), Num<T>::add(qa[2], qa[3])), red, nwarps);
        if (tid == 0 && hist) hist[sweeps] = static_cast<double>(Q);
        ++sweeps;
        if (thresh2 >= 0.0 && static_cast<double>(Q) <= thresh2) {
          converged = true;
          return true;
        }
        if (sweeps == prm.max_iter) return true;
      }
      P = block_sum(pv, red, nwarps);
      idx = last ? 0 : idx + 1;
      return false;
    };
    while (true) {
      if (step(xa, xb)) break;
      if (step(xb, xa)) break;
    }
  } else if (tid == 0) {
    status[3] = BAK_EINVAL;  // all columns zero (bak.py:186-187)
  }
  __syncthreads();

  // final residual y - x a (bak.py:130) and drift (bak.py:133-142)
  T acc[E];
#pragma unroll
  for (int k = 0; k < E; ++k) acc[k] = T(0);
  for (int64_t j = 0; j < vars; ++j) {
    const T aj = as[j];
#pragma unroll
    for (int k = 0; k < E; ++k)
      if (k < kv) acc[k] = Num<T>::fma(X[j * ldx + tid + k * NT], aj, acc[k]);
  }
  double dd = 0.0;
#pragma unroll
  for (int k = 0; k < E; ++k) {
    if (k < kv) {
      const T r = Num<T>::sub(yv[k], acc[k]);
      rg[tid + k * NT] = r;
      const double df = static_cast<double>(Num<T>::sub(ev[k], r));
      dd = __fma_rn(df, df, dd);
    }
  }
  dd = block_sum(dd, redd, nwarps);
  for (int64_t j = tid; j < vars; j += NT) ag[j] = as[j];
  if (tid == 0) {
    const double ynorm = sqrt(yn2);
    const double drift_rel = sqrt(dd) / (ynorm > 2.2250738585072014e-308 ? ynorm : 2.2250738585072014e-308);
    status[0] = sweeps;
    status[1] = converged ? 1 : 0;
    status[2] = drift_rel > prm.drift_tol ? 1 : 0;
  }
}

// nsys == 0: occupancy query only — systems in flight per SM (g_wave_per_sm)
thread_local int g_wave_per_sm = 0;

template <typename T, int E, int NT, bool SMEM>
int launch_batched_t(const BatchedParams& prm, size_t smem, cudaStream_t st) {
  auto kern = batched_kernel<T, E, NT, SMEM>;
  BAK_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  if (prm.nsys == 0) {
    BAK_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&g_wave_per_sm, kern, NT, smem));
    return BAK_OK;
  }
  kern<<<static_cast<unsigned>(prm.nsys), NT, smem, st>>>(prm);
  count_launches(1);
  BAK_CHECK_CUDA(cudaGetLastError());
  return BAK_OK;
}

template <typename T, int NT, bool SMEM>
int launch_batched_e(int E, const BatchedParams& prm, size_t smem, cudaStream_t st) {
  switch (E) {
    case 1: return launch_batched_t<T, 1, NT, SMEM>(prm, smem, st);
    case 2: return launch_batched_t<T, 2, NT, SMEM>(prm, smem, st);
    case 4: return launch_batched_t<T, 4, NT, SMEM>(prm, smem, st);
    case 8: return launch_batched_t<T, 8, NT, SMEM>(prm, smem, st);
    case 16: return launch_batched_t<T, 16, NT, SMEM>(prm, smem, st);
    default: return launch_batched_t<T, 32, NT, SMEM>(prm, smem, st);
  }
}

template <typename T>
int launch_batched(int E, int nt, bool in_smem, const BatchedParams& prm, size_t smem, cudaStream_t st) {
  if (nt == 32) return in_smem ? launch_batched_e<T, 32, true>(E, prm, smem, st) : launch_batched_e<T, 32, false>(E, prm, smem, st);
  if (nt == 64) return in_smem ? launch_batched_e<T, 64, true>(E, prm, smem, st) : launch_batched_e<T, 64, false>(E, prm, smem, st);
  if (nt == 128) return in_smem ? launch_batched_e<T, 128, true>(E, prm, smem, st) : launch_batched_e<T, 128, false>(E, prm, smem, st);
  return in_smem ? launch_batched_e<T, 256, true>(E, prm, smem, st) : launch_batched_e<T, 256, false>(E, prm, smem, st);
}

}  // namespace
}  // namespace bak

using namespace bak;

namespace {
// plan (rows per thread, threads, x residency, shared memory) and launch; with
// query = true nothing is launched and g_wave_per_sm receives the occupancy
int batched_entry(bool query, int dtype, const void* x, int64_t obs, int64_t vars, int64_t ldx, int64_t x_stride,
                  int64_t nsys, const void* y, int64_t y_stride, const void* norms2, const double* ynorm2, void* a,
                  int warm, void* resid, int64_t max_iter, double tol, double drift_tol, double* history,
                  int64_t* status, void* stream) {
  const size_t ts = dtype_size(dtype);
  // rows per thread / threads: aim for ~4 warps per system, E <= 32
  static const int kEs[] = {1, 2, 4, 8, 16, 32};
  int E = 0, nt = 0;
  const int emax1 = dtype == BAK_F64 ? 16 : 16;
  if (const char* env = getenv("BAK_BATCH_PLAN")) {  // "E,nthreads" (tuning experiments)
    int e = 0, t = 0;
    if (sscanf(env, "%d,%d", &e, &t) == 2 && static_cast<int64_t>(e) * t >= obs &&
        (t == 32 || t == 64 || t == 128 || t == 256)) {
      E = e;
      nt = t;
    }
  }
  for (int e : kEs) {  // one warp per system when the rows fit in E <= 16 per lane
    if (E) break;
    if (e > emax1) break;
    if (static_cast<int64_t>(32) * e >= obs) {
      E = e;
      nt = 32;
      break;
    }
  }
  for (int cap_t : {128, 256}) {  // else the fewest power-of-two warps with E <= 32
    for (int e : kEs) {
      if (E) break;
      int t = 32;
      while (static_cast<int64_t>(t) * e < obs) t *= 2;
      if (t <= cap_t) {
        E = e;
        nt = t;
      }
    }
  }
  if (!E) {
    set_error("bak_solve_batched: obs=%lld too large for one CTA (max %d)", (long long)obs, 256 * 32);
    return BAK_EUNSUPPORTED;
  }
  const size_t cap = static_cast<size_t>(device_max_smem_optin()) - 1024;
  const size_t xbytes = static_cast<size_t>(vars) * ldx * ts;
  const size_t small = 16 + 3 * round_up(static_cast<int64_t>(vars * ts), 16) + round_up((vars + 1) * 4, 16) + 32 * 8;
  BatchedParams prm{x, obs, vars, ldx, x_stride, nsys, y, y_stride, norms2, ynorm2, a, warm, resid,
                    max_iter, tol, drift_tol, history, status, 0};
  const bool aligned = (reinterpret_cast<uintptr_t>(x) % 16 == 0) && ((ldx * ts) % 16 == 0) &&
                       ((x_stride * ts) % 16 == 0) && xbytes < (1u << 20);
  if (query) prm.nsys = 0;
  size_t smem = small;
  // x resident in shared memory only when that still leaves >= 8 systems per
  // SM in flight; otherwise stream x from L2/HBM every sweep with many more
  // systems per SM.  Measured on C5 (65,536 x 512x32 fp32, 64 KiB of x per
  // system): resident (3 systems/SM, latency-bound) 277 ms vs streamed
  // (1 warp per system, HBM-bound at 6.8 TB/s) 127 ms per 200 sweeps.
  // BAK_BATCH_X=smem|stream forces either (tests check they agree bit for bit).
  const char* force = getenv("BAK_BATCH_X");
  const bool fits = aligned && xbytes + small <= cap;
  bool use_smem = fits && (cap / (xbytes + small)) >= 8;
  if (force && force[0] == 's' && force[1] == 'm') use_smem = fits;
  if (force && force[0] == 's' && force[1] == 't') use_smem = false;
  if (use_smem) {
    prm.x_in_smem = 1;
    smem += xbytes;
  }
  // Streamed x: cap the resident systems per SM so that their x (re-read every
  // sweep) stays in L2 instead of being streamed from HBM each sweep.  Measured
  // on C5 (64 KiB per system, 148 SMs, 126 MB L2): uncapped ~24/SM 132 ms,
  // 12/SM (116 MB of x in flight) 121 ms, 8/SM latency-bound 154 ms.  Only
  // applied while >= 10 systems per SM remain; BAK_BATCH_PER_SM=n overrides.
  if (!use_smem) {
    int per_sm = 0;
    const double fit = static_cast<double>(l2_bytes()) / (static_cast<double>(xbytes) * device_sms());
    if (fit >= 11.0) per_sm = static_cast<int>(fit) - 1;
    if (const char* ps = getenv("BAK_BATCH_PER_SM")) per_sm = atoi(ps);
    if (per_sm > 0 && cap / per_sm > smem) smem = cap / per_sm;
  }
  if (small > cap) {
    set_error("bak_solve_batched: vars=%lld too large", (long long)vars);
    return BAK_EUNSUPPORTED;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
#define BAK_B(T)                                                  \
  return launch_batched<T>(E, nt, prm.x_in_smem != 0, prm, smem, st);
  if (dtype == BAK_F64) {
    BAK_B(double)
  } else {
    BAK_B(float)
  }
#undef BAK_B
}
}  // namespace

extern "C" int bak_solve_batched(int dtype, const void* x, int64_t obs, int64_t vars, int64_t ldx, int64_t x_stride,
                                 int64_t nsys, const void* y, int64_t y_stride, const void* norms2,
                                 const double* ynorm2, void* a, int warm, void* resid, int64_t max_iter, double tol,
                                 double drift_tol, double* history, int64_t* status, void* stream) {
  if (obs < 1 || vars < 1 || ldx < obs || nsys < 1 || max_iter < 1 || !x || !y || !norms2 || !ynorm2 || !a ||
      !resid || !status || (dtype != BAK_F32 && dtype != BAK_F64)) {
    set_error("bak_solve_batched: bad arguments");
    return BAK_EINVAL;
  }
  return batched_entry(false, dtype, x, obs, vars, ldx, x_stride, nsys, y, y_stride, norms2, ynorm2, a, warm, resid,
                       max_iter, tol, drift_tol, history, status, stream);
}

// Systems the batched solve runs concurrently on this device (one wave) for
// systems of this shape stored contiguously (ldx = obs padded to 16 bytes):
// callers that stream batches in chunks size them in whole waves.  0 on error.
extern "C" int64_t bak_solve_batched_wave(int dtype, int64_t obs, int64_t vars) {
  if (obs < 1 || vars < 1 || (dtype != BAK_F32 && dtype != BAK_F64)) {
    set_error("bak_solve_batched_wave: bad arguments");
    return 0;
  }
  const int64_t vec = dtype == BAK_F64 ? 2 : 4;
  const int64_t ldx = (obs + vec - 1) / vec * vec;
  alignas(16) static const double dummy[2] = {0.0, 0.0};
  g_wave_per_sm = 0;
  if (batched_entry(true, dtype, dummy, obs, vars, ldx, vars * ldx, 1, dummy, ldx, dummy, dummy,
                    const_cast<double*>(dummy), 0, const_cast<double*>(dummy), 1, 0.0, 0.0, nullptr, nullptr,
                    nullptr) != BAK_OK)
    return 0;
  return static_cast<int64_t>(g_wave_per_sm) * device_sms();
}

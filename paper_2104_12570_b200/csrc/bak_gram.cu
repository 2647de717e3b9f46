// GRAM variant (BAK_VARIANT_GRAM): an ALGEBRAICALLY EQUIVALENT reformulation of
// the column sweep for tall systems whose residual e cannot stay on chip.
// Labelled as such everywhere it is reported: same iterates in exact
// arithmetic, different rounding than the reference's per-column dots.
//
// One SolveBak sweep (bak.py:92-112) over columns j1, j2, ... in order is
//     d_j = <x_j, e_current> / n2_j,   e_current = e_start - sum_{k before j} d_k x_k
//         = (g_j - sum_{k before j} G_jk d_k) / n2_j,   g = X^T e_start,  G = X^T X
// followed by e_end = e_start - X d.  So a sweep needs ONE pass over x:
//     pass(s):  e <- e - X d^(s)  (rows in parallel),  sum e^2,  g <- X^T e
//     solve(s+1): forward substitution over the sweep order with G (vars x vars)
// The per-column exact kernels must read x twice per column when e lives in
// HBM (x_j for the update, x_{j+1} for the next dot, plus e in and out); this
// variant reads x once per sweep plus e once, at the price of a one-time
// G = X^T X (hand-written fp64 DMMA SYRK, fp64 accumulation for both precisions).
//
// pass kernel layout: thread (c, r) owns row r of a 256/nch-row tile and the
// 16-column chunk c; its 16 x values live in registers (coalesced loads along
// rows), are used for both the update and the dot, and the next tile's values
// are prefetched while the current one is reduced.
#include <cstdio>
#include <vector>

#include "bak_common.cuh"
#include "bak_sweep.cuh"

namespace bak {
namespace {

constexpr int kGT = 256;  // threads per pass CTA
constexpr int kCW = 16;   // columns per thread chunk

struct GramCtrl {
  int64_t done, sweeps, converged, pad;
};

struct PassParams {
  const void* x;
  int64_t obs, ldx, vars;
  void* e;
  const double* delta;
  int apply, dot;
  double* gpart;
  double* sqpart;
  const GramCtrl* ctrl;
};

__host__ __device__ inline int pow2_at_least(int v) {
  int p = 1;
  while (p < v) p <<= 1;
  return p;
}

template <typename T>
__global__ void __launch_bounds__(kGT, 2) gram_pass_kernel(const PassParams p) {
  if (*reinterpret_cast<const volatile int64_t*>(&p.ctrl->done)) return;
  __shared__ double dsh[512];
  __shared__ double red[2][kGT];
  __shared__ double es[2][kGT];
  const int V = static_cast<int>(p.vars);
  const int nch = pow2_at_least((V + kCW - 1) / kCW);
  const int R = kGT / nch;  // rows per tile
  const int tid = threadIdx.x;
  const int c = tid / R, r = tid % R;
  const T* __restrict__ x = static_cast<const T*>(p.x);
  T* __restrict__ e = static_cast<T*>(p.e);
  for (int j = tid; j < V; j += kGT) dsh[j] = p.apply ? p.delta[j] : 0.0;
  __syncthreads();

  const int64_t ntiles = (p.obs + R - 1) / R;
  double acc[kCW];
#pragma unroll
  for (int q = 0; q < kCW; ++q) acc[q] = 0.0;
  double sq = 0.0;
  int jv[kCW];
#pragma unroll
  for (int q = 0; q < kCW; ++q) jv[q] = c * kCW + q;

  T xa[kCW], xb[kCW];
  T ea = T(0), eb = T(0);
  auto load = [&](int64_t tile, T (&xr)[kCW], T& ev) {
    const int64_t row = tile * R + r;
    const bool ok = tile < ntiles && row < p.obs;
#pragma unroll
    for (int q = 0; q < kCW; ++q) xr[q] = (ok && jv[q] < V) ? __ldcs(x + jv[q] * p.ldx + row) : T(0);
    if (c == 0) ev = ok ? e[row] : T(0);
  };
  int64_t tile = blockIdx.x;
  load(tile, xa, ea);
  int buf = 0;
  for (; tile < ntiles; tile += gridDim.x) {
    load(tile + gridDim.x, xb, eb);  // prefetch the next tile (x and e)
    const int64_t row = tile * R + r;
    const bool ok = row < p.obs;
    if (p.apply) {
      double t = 0.0;
#pragma unroll
      for (int q = 0; q < kCW; ++q) t = __fma_rn(static_cast<double>(xa[q]), dsh[jv[q] < V ? jv[q] : 0], t);
      red[buf][tid] = t;
    }
    __syncthreads();
    if (c == 0) {
      double ev = static_cast<double>(ea);
      if (p.apply) {
        double tt = 0.0;
        for (int cc = 0; cc < nch; ++cc) tt += red[buf][cc * R + r];
        const T en = static_cast<T>(ev - tt);
        if (ok) e[row] = en;
        ev = static_cast<double>(en);
        sq = __fma_rn(ev, ev, sq);
      }
      es[buf][r] = ev;
    }
    __syncthreads();
    if (p.dot) {
      const double er = es[buf][r];
#pragma unroll
      for (int q = 0; q < kCW; ++q) acc[q] = __fma_rn(static_cast<double>(xa[q]), er, acc[q]);
    }
#pragma unroll
    for (int q = 0; q < kCW; ++q) xa[q] = xb[q];
    ea = eb;
    buf ^= 1;
  }
  __syncthreads();
  // per-column partials: reduce over the R row-threads of each chunk (fixed order)
  double* gsh = &red[0][0];  // reuse 2*kGT doubles: process kCW/2 columns per round
  for (int q0 = 0; q0 < kCW; q0 += 2) {
    gsh[tid * 2 + 0] = acc[q0];
    gsh[tid * 2 + 1] = acc[q0 + 1];
    __syncthreads();
    if (tid < nch * 2) {
      const int cc = tid >> 1, qq = tid & 1;
      const int j = cc * kCW + q0 + qq;
      double s = 0.0;
      for (int rr = 0; rr < R; ++rr) s += gsh[(cc * R + rr) * 2 + qq];
      if (j < V && p.dot) p.gpart[static_cast<int64_t>(blockIdx.x) * V + j] = s;
    }
    __syncthreads();
  }
  // sum e^2 of this CTA
  double s2 = warp_sum(sq);
  if ((tid & 31) == 0) gsh[tid >> 5] = s2;
  __syncthreads();
  if (tid == 0) {
    double s = 0.0;
    for (int w = 0; w < kGT / 32; ++w) s += gsh[w];
    p.sqpart[blockIdx.x] = s;
  }
}

struct SolveParams {
  int64_t vars, nblk;
  int64_t sweep;  // sweep about to be solved (1-based); finalizes sweep-1
  int64_t max_iter;
  double thresh2;
  const int32_t* cols;
  int64_t ncols, cols_stride;
  const void* norms2;
  const double* G;
  const double* gpart;
  const double* sqpart;
  void* a;
  double* delta;
  double* history;
  GramCtrl* ctrl;
  int64_t* status;
  int64_t thr = 1;     // > 1: blocked sweep (bakp.py:95-129), cyclic order only
  int guard = 0;       // divergence guard of the blocked sweep (bakp.py:121-124)
  double prev0 = 0.0;  // the guard's first reference value, ||y||^2
};

__device__ __forceinline__ bool gram_diverged(double sq, double prev) {
  return !(sq <= 1.79769313486231570815e308 && sq >= -1.79769313486231570815e308) || sq > prev * 10.0;
}

template <typename T>
__global__ void __launch_bounds__(512, 1) gram_solve_kernel(const SolveParams p) {
  if (p.ctrl->done) return;
  __shared__ double wsum[16];
  const int V = static_cast<int>(p.vars);
  const int tid = threadIdx.x;
  const int s = static_cast<int>(p.sweep);
  if (s >= 2) {
    // finalize sweep s-1: sum e^2 over the pass CTAs in fixed order
    double v = 0.0;
    for (int64_t b = tid; b < p.nblk; b += blockDim.x) v += p.sqpart[b];
    v = warp_sum(v);
    if ((tid & 31) == 0) wsum[tid >> 5] = v;
    __syncthreads();
    double sq = 0.0;
    for (int w = 0; w < static_cast<int>(blockDim.x) / 32; ++w) sq += wsum[w];
    bool stop_div = false;
    if (p.guard) {
      const double prev = (s == 2) ? p.prev0 : __longlong_as_double(p.ctrl->pad);
      stop_div = gram_diverged(sq, prev);
      __syncthreads();  // every thread has read prev before it is replaced
    }
    const bool stop_conv = !stop_div && p.thresh2 >= 0.0 && sq <= p.thresh2;
    const bool stop_max = (s - 1) >= p.max_iter;
    if (tid == 0) {
      if (p.history) p.history[s - 2] = sq;
      if (p.guard) p.ctrl->pad = __double_as_longlong(sq);
      if (stop_conv || stop_max || stop_div) {
        p.ctrl->done = 1;
        p.ctrl->sweeps = s - 1;
        p.ctrl->converged = stop_conv ? 1 : 0;
        if (p.status) {
          p.status[0] = s - 1;
          p.status[1] = stop_conv ? 1 : 0;
          if (stop_div) p.status[2] = BAK_EDIVERGED;
          p.status[3] = BAK_VARIANT_GRAM;
        }
      }
    }
    if (stop_conv || stop_max || stop_div) return;
  }
  // g = sum over pass CTAs (fixed order), residual dots in double
  __shared__ int ord[512];
  __shared__ double n2s[512];
  const T* n2 = static_cast<const T*>(p.norms2);
  T* a = static_cast<T*>(p.a);
  const int32_t* cl = p.cols ? p.cols + (p.cols_stride ? (s - 1) * p.cols_stride : 0) : nullptr;
  for (int64_t kk = tid; kk < p.ncols; kk += blockDim.x) ord[kk] = cl ? cl[kk] : static_cast<int>(kk);
  double rj = 0.0;
  T aj = T(0);
  if (tid < V) {
    // the pass CTAs' partials in fixed order; 8 loads in flight, sums in order
    int64_t b = 0;
    for (; b + 8 <= p.nblk; b += 8) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = p.gpart[(b + u) * V + tid];
#pragma unroll
      for (int u = 0; u < 8; ++u) rj += v[u];
    }
    for (; b < p.nblk; ++b) rj += p.gpart[b * V + tid];
    n2s[tid] = static_cast<double>(n2[tid]);
    aj = a[tid];
  }
  double dj = 0.0;
  __syncthreads();
  if (p.thr > 1) {
    // blocked sweep: every delta of a block from the same (stale) residual dots,
    // then one correction of the dots by the block (bakp.py:101-116)
    __shared__ double dblk[512];
    for (int64_t j0 = 0; j0 < p.ncols; j0 += p.thr) {
      const int64_t j1 = imin64(j0 + p.thr, p.ncols);
      if (tid >= j0 && tid < j1) {
        const T d = (n2s[tid] != 0.0) ? Num<T>::div(static_cast<T>(rj), static_cast<T>(n2s[tid])) : T(0);
        dblk[tid] = static_cast<double>(d);
        dj = static_cast<double>(d);
        aj = Num<T>::add(aj, d);
      }
      __syncthreads();
      if (tid < V) {  // G entries 8 at a time in flight, FMAs in column order
        int64_t k = j0;
        for (; k + 8 <= j1; k += 8) {
          double gv[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) gv[u] = p.G[(k + u) * V + tid];
#pragma unroll
          for (int u = 0; u < 8; ++u) rj = __fma_rn(-gv[u], dblk[k + u], rj);
        }
        for (; k < j1; ++k) rj = __fma_rn(-p.G[k * V + tid], dblk[k], rj);
      }
    }
    if (tid < V) {
      p.delta[tid] = dj;
      a[tid] = aj;
    }
    return;
  }
  // Forward substitution over the sweep order, in blocks of 32 positions:
  // warp 0 solves a block's lower triangle (lane l holds the residual dot of
  // the block's l-th column; each d is broadcast with a shuffle), then every
  // thread applies the block's 32 updates to its own dot in sweep order.  Each
  // dot receives exactly the FMAs of the one-column-at-a-time loop, in the same
  // order, so the result is bit-identical to it — with 2 block barriers per 32
  // columns instead of one per column (0.13 -> ~0.03 ms per 256-column solve).
  __shared__ double rs[512];
  __shared__ double dblk[32];
  for (int64_t k0 = 0; k0 < p.ncols; k0 += 32) {
    const int nbk = static_cast<int>(imin64(32, p.ncols - k0));
    if (tid < V) rs[tid] = rj;
    __syncthreads();
    if (tid < 32) {
      const int l = tid;
      const int jl = l < nbk ? ord[k0 + l] : 0;
      double rl = l < nbk ? rs[jl] : 0.0;
      double gcol[32];  // G[ord[k0+i], jl] for the block's earlier columns, prefetched
#pragma unroll
      for (int i = 0; i < 32; ++i)
        gcol[i] = (i < nbk && i < l && l < nbk) ? p.G[static_cast<int64_t>(ord[k0 + i]) * V + jl] : 0.0;
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        if (i < nbk) {
          const int ji = ord[k0 + i];
          double d = 0.0;
          if (l == i && n2s[ji] != 0.0)
            d = static_cast<double>(Num<T>::div(static_cast<T>(rl), static_cast<T>(n2s[ji])));
          d = __shfl_sync(0xffffffffu, d, i);
          if (l > i && l < nbk) rl = __fma_rn(-gcol[i], d, rl);
          if (l == i) dblk[i] = d;  // zero-norm column: skipped, coefficient frozen (bak.py:101-103)
        }
      }
    }
    __syncthreads();
    if (tid < V) {
      // the block's 32 G entries of this column first (independent loads in
      // flight together), then the FMA chain in sweep order
      double gv[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) gv[i] = i < nbk ? p.G[static_cast<int64_t>(ord[k0 + i]) * V + tid] : 0.0;
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        if (i < nbk) {
          const int ji = ord[k0 + i];
          const double d = dblk[i];
          if (tid == ji && n2s[ji] != 0.0) {
            dj = d;
            aj = Num<T>::add(aj, static_cast<T>(d));
          }
          rj = __fma_rn(-gv[i], d, rj);
        }
      }
    }
  }
  if (tid < V) {
    p.delta[tid] = dj;  // 0 for columns not in this sweep's list (zero norms)
    a[tid] = aj;
  }
}

}  // namespace

// workspace layout (bytes): G | gpart | sqpart | delta | ctrl | G partials (split-K)
static int64_t gram_nblk() { return 2 * static_cast<int64_t>(device_sms()); }

// rows of gpart: the pass partials, or the fused first-sweep partials of the G kernel
static int64_t gram_gpart_rows(int dtype, int64_t obs, int64_t vars) {
  int g0rows;
  int64_t chunk;
  gram_g_workspace(dtype, obs, vars, g0rows, chunk);
  return g0rows > gram_nblk() ? g0rows : gram_nblk();
}

int64_t gram_workspace_bytes(int dtype, int64_t obs, int64_t vars) {
  (void)dtype;
  int64_t b = 0;
  b += vars * vars * 8;
  b += gram_gpart_rows(dtype, obs, vars) * vars * 8;
  b += gram_nblk() * 8;
  b += vars * 8;
  b += 64;
  int nchunks;
  int64_t chunk;
  b += gram_g_workspace(dtype, obs, vars, nchunks, chunk) + 256;
  return round_up(b, 256) + 4096;
}

bool gram_supported(int64_t vars) { return vars >= 1 && vars <= 512; }

static int launch_gram_impl(int dtype, const SweepParams& prm, int64_t vars, void* ws, int64_t wsb, cudaStream_t st,
                            int64_t thr, int guard, double prev0);

int launch_gram(int dtype, const SweepParams& prm, int64_t vars, void* ws, int64_t wsb, cudaStream_t st) {
  return launch_gram_impl(dtype, prm, vars, ws, wsb, st, 1, 0, 0.0);
}

int launch_gram_block(int dtype, const void* x, int64_t obs, int64_t ldx, int64_t vars, const void* norms2,
                      int64_t thr, void* e, void* a, int64_t max_iter, double thresh2, double prev_sq,
                      double* history, int64_t* status, void* ws, int64_t wsb, cudaStream_t st) {
  if (reinterpret_cast<uintptr_t>(e) % 16) {
    set_error("bak_block_sweep(GRAM): e must be 16-byte aligned");
    return BAK_EINVAL;
  }
  SweepParams prm{};
  prm.x = x;
  prm.obs = obs;
  prm.ldx = ldx;
  prm.norms2 = norms2;
  prm.cols = nullptr;
  prm.ncols = vars;
  prm.cols_stride = 0;
  prm.e = e;
  prm.a = a;
  prm.max_iter = max_iter;
  prm.thresh2 = thresh2;
  prm.history = history;
  prm.status = status;
  BAK_CHECK_CUDA(cudaMemsetAsync(status, 0, 4 * sizeof(int64_t), st));
  return launch_gram_impl(dtype, prm, vars, ws, wsb, st, thr, 1, prev_sq);
}

static int launch_gram_impl(int dtype, const SweepParams& prm, int64_t vars, void* ws, int64_t wsb, cudaStream_t st,
                            int64_t thr, int guard, double prev0) {
  if (!gram_supported(vars)) {
    set_error("GRAM variant supports 1 <= vars <= 512 (got %lld)", (long long)vars);
    return BAK_EUNSUPPORTED;
  }
  if (wsb < gram_workspace_bytes(dtype, prm.obs, vars)) {
    set_error("bak_sweep(GRAM): workspace too small (need %lld)", (long long)gram_workspace_bytes(dtype, prm.obs, vars));
    return BAK_EWORKSPACE;
  }
  const int64_t nblk = gram_nblk();
  char* w = static_cast<char*>(ws);
  double* G = reinterpret_cast<double*>(w);
  w += vars * vars * 8;
  double* gpart = reinterpret_cast<double*>(w);
  w += gram_gpart_rows(dtype, prm.obs, vars) * vars * 8;
  double* sqpart = reinterpret_cast<double*>(w);
  w += nblk * 8;
  double* delta = reinterpret_cast<double*>(w);
  w += vars * 8;
  GramCtrl* ctrl = reinterpret_cast<GramCtrl*>(w);
  w += 64;
  double* gparts_ws = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(w) + 255) & ~uintptr_t(255));
  const int64_t gparts_bytes = wsb - (reinterpret_cast<char*>(gparts_ws) - static_cast<char*>(ws));

  // ---- G = X^T X: hand-written fp64 DMMA SYRK (bak_gram_dmma.cu) ----
  // G and the first sweep's g = X^T e (fused into the diagonal-block CTAs)
  const bool fuse_g0 = reinterpret_cast<uintptr_t>(prm.e) % 16 == 0;
  if (int rc = launch_gram_g(dtype, prm.x, prm.obs, prm.ldx, vars, G, gparts_ws, gparts_bytes, st, nullptr,
                             fuse_g0 ? prm.e : nullptr, fuse_g0 ? gpart : nullptr, prm.status))
    return rc;
  BAK_CHECK_CUDA(cudaMemsetAsync(ctrl, 0, sizeof(GramCtrl), st));

  PassParams pp{prm.x, prm.obs, prm.ldx, vars, prm.e, delta, 0, 1, gpart, sqpart, ctrl};
  SolveParams sp{vars, nblk, 0, prm.max_iter, prm.thresh2, prm.cols, prm.ncols, prm.cols_stride, prm.norms2,
                 G, gpart, sqpart, prm.a, delta, prm.history, ctrl, prm.status, thr, guard, prev0};
  const bool use_tma = gram_tma_supported(vars);
  if (use_tma) sp.nblk = gram_tma_grid(dtype);
  auto pass = [&](int apply, int dot) -> int {
    if (use_tma)
      return launch_gram_pass_tma(dtype, prm.x, prm.obs, prm.ldx, vars, prm.e, delta, apply, dot, gpart, sqpart,
                                  &ctrl->done, st, nullptr, nullptr, nullptr, prm.status);
    pp.apply = apply;
    pp.dot = dot;
    if (dtype == BAK_F64)
      gram_pass_kernel<double><<<static_cast<unsigned>(nblk), kGT, 0, st>>>(pp);
    else
      gram_pass_kernel<float><<<static_cast<unsigned>(nblk), kGT, 0, st>>>(pp);
    count_launches(1);
    BAK_CHECK_CUDA(cudaGetLastError());
    return BAK_OK;
  };
  auto solve = [&](int64_t s) -> int {
    sp.sweep = s;
    if (dtype == BAK_F64)
      gram_solve_kernel<double><<<1, 512, 0, st>>>(sp);
    else
      gram_solve_kernel<float><<<1, 512, 0, st>>>(sp);
    count_launches(1);
    BAK_CHECK_CUDA(cudaGetLastError());
    return BAK_OK;
  };
  int rc = 0;
  const int64_t pass_parts = sp.nblk;
  if (fuse_g0) {
    int g0rows;
    int64_t chunk;
    gram_g_workspace(dtype, prm.obs, vars, g0rows, chunk);
    sp.nblk = g0rows;
  } else if ((rc = pass(0, 1))) {
    return rc;
  }
  for (int64_t s = 1; s <= prm.max_iter; ++s) {
    if ((rc = solve(s))) return rc;
    sp.nblk = pass_parts;
    if ((rc = pass(1, s < prm.max_iter ? 1 : 0))) return rc;
    if ((prm.thresh2 >= 0.0 || guard) && s % 16 == 0) {
      // early break: stop enqueueing once the device has flagged convergence (or divergence)
      int64_t done = 0;
      BAK_CHECK_CUDA(cudaMemcpyAsync(&done, &ctrl->done, sizeof(done), cudaMemcpyDeviceToHost, st));
      BAK_CHECK_CUDA(cudaStreamSynchronize(st));
      if (done) break;
    }
  }
  return solve(prm.max_iter + 1);
}

}  // namespace bak

// ======================= C ABI: GRAM building blocks =========================
// Used directly for row-sharded multi-GPU solves (each rank: local G and pass
// partials; the host gathers the partials of all ranks, rank-major, and every
// rank runs the same solve on the same bytes -> bit-identical d and a).
using namespace bak;

extern "C" int bak_gram_pass_blocks(int dtype, int64_t vars) {
  return gram_tma_supported(vars) ? gram_tma_grid(dtype) : static_cast<int>(gram_nblk());
}

extern "C" int64_t bak_gram_matrix_workspace(int dtype, int64_t obs, int64_t vars) {
  int nchunks;
  int64_t chunk;
  return gram_g_workspace(dtype, obs, vars, nchunks, chunk) + 256;
}

extern "C" int bak_gram_matrix(int dtype, const void* x, int64_t obs, int64_t vars, int64_t ldx, double* G,
                               void* workspace, int64_t workspace_bytes, void* stream) {
  if ((dtype != BAK_F32 && dtype != BAK_F64) || obs < 1 || vars < 1 || ldx < obs || !x || !G) {
    set_error("bak_gram_matrix: bad arguments");
    return BAK_EINVAL;
  }
  const size_t ts = dtype_size(dtype);
  if (reinterpret_cast<uintptr_t>(x) % 16 || (ldx * static_cast<int64_t>(ts)) % 16) {
    set_error("bak_gram_matrix: x must be 16-byte aligned with ldx*sizeof(T) %% 16 == 0");
    return BAK_EINVAL;
  }
  return launch_gram_g(dtype, x, obs, ldx, vars, G, workspace, workspace_bytes, static_cast<cudaStream_t>(stream));
}

extern "C" int64_t bak_gram_dot_rows(int dtype, int64_t obs, int64_t vars) {
  int nchunks;
  int64_t chunk;
  gram_g_workspace(dtype, obs, vars, nchunks, chunk);
  return nchunks;
}

extern "C" int bak_gram_matrix_dot(int dtype, const void* x, int64_t obs, int64_t vars, int64_t ldx, double* G,
                                   const void* e, double* g0, void* workspace, int64_t workspace_bytes,
                                   void* stream) {
  if ((dtype != BAK_F32 && dtype != BAK_F64) || obs < 1 || vars < 1 || ldx < obs || !x || !G || !e || !g0) {
    set_error("bak_gram_matrix_dot: bad arguments");
    return BAK_EINVAL;
  }
  const size_t ts = dtype_size(dtype);
  if (reinterpret_cast<uintptr_t>(x) % 16 || (ldx * static_cast<int64_t>(ts)) % 16 ||
      reinterpret_cast<uintptr_t>(e) % 16) {
    set_error("bak_gram_matrix_dot: x and e must be 16-byte aligned with ldx*sizeof(T) %% 16 == 0");
    return BAK_EINVAL;
  }
  return launch_gram_g(dtype, x, obs, ldx, vars, G, workspace, workspace_bytes, static_cast<cudaStream_t>(stream),
                       nullptr, e, g0);
}

extern "C" int bak_gram_pass_resid(int dtype, const void* x, int64_t obs, int64_t vars, int64_t ldx, void* e,
                                   const double* delta, int apply, int dot, double* gpart, double* sqpart,
                                   const int64_t* done_flag, const void* afin, const void* y, void* resid,
                                   int64_t* status, void* stream);

extern "C" int bak_gram_pass(int dtype, const void* x, int64_t obs, int64_t vars, int64_t ldx, void* e,
                             const double* delta, int apply, int dot, double* gpart, double* sqpart,
                             const int64_t* done_flag, int64_t* status, void* stream) {
  return bak_gram_pass_resid(dtype, x, obs, vars, ldx, e, delta, apply, dot, gpart, sqpart, done_flag, nullptr,
                             nullptr, nullptr, status, stream);
}

extern "C" int bak_gram_pass_resid(int dtype, const void* x, int64_t obs, int64_t vars, int64_t ldx, void* e,
                                   const double* delta, int apply, int dot, double* gpart, double* sqpart,
                                   const int64_t* done_flag, const void* afin, const void* y, void* resid,
                                   int64_t* status, void* stream) {
  if ((dtype != BAK_F32 && dtype != BAK_F64) || obs < 1 || !gram_supported(vars) || ldx < obs || !x || !e ||
      !delta || !gpart || !sqpart || !done_flag || (afin && (!y || !resid))) {
    set_error("bak_gram_pass: bad arguments");
    return BAK_EINVAL;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (gram_tma_supported(vars))
    return launch_gram_pass_tma(dtype, x, obs, ldx, vars, e, delta, apply, dot, gpart, sqpart, done_flag, st, afin,
                                y, resid, status);
  if (afin) {
    set_error("bak_gram_pass: fused residual needs the TMA pass (vars <= 256)");
    return BAK_EUNSUPPORTED;
  }
  PassParams pp{x, obs, ldx, vars, e, delta, apply, dot, gpart, sqpart,
                reinterpret_cast<const GramCtrl*>(done_flag)};
  if (dtype == BAK_F64)
    gram_pass_kernel<double><<<static_cast<unsigned>(gram_nblk()), kGT, 0, st>>>(pp);
  else
    gram_pass_kernel<float><<<static_cast<unsigned>(gram_nblk()), kGT, 0, st>>>(pp);
  count_launches(1);
  BAK_CHECK_CUDA(cudaGetLastError());
  return BAK_OK;
}

extern "C" int bak_gram_solve(int dtype, int64_t vars, const double* gpart, const double* sqpart, int64_t nparts,
                              int64_t sweep, int64_t max_iter, double thresh2, const int32_t* cols, int64_t ncols,
                              int64_t cols_stride, const void* norms2, const double* G, void* a, double* delta,
                              double* history, int64_t* ctrl, int64_t* status, void* stream) {
  if ((dtype != BAK_F32 && dtype != BAK_F64) || !gram_supported(vars) || !gpart || !sqpart || nparts < 1 ||
      sweep < 1 || !norms2 || !G || !a || !delta || !ctrl || (!cols && ncols != vars)) {
    set_error("bak_gram_solve: bad arguments");
    return BAK_EINVAL;
  }
  SolveParams sp{vars, nparts, sweep, max_iter, thresh2, cols, ncols, cols_stride, norms2, G, gpart, sqpart,
                 a, delta, history, reinterpret_cast<GramCtrl*>(ctrl), status};
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (dtype == BAK_F64)
    gram_solve_kernel<double><<<1, 512, 0, st>>>(sp);
  else
    gram_solve_kernel<float><<<1, 512, 0, st>>>(sp);
  count_launches(1);
  BAK_CHECK_CUDA(cudaGetLastError());
  return BAK_OK;
}

// One call: G (+ norms from its diagonal), then the GRAM sweeps; zero-norm columns
// are skipped in the solve; with thresh2 < 0 and resid != NULL the final pass
// also writes resid = y - x a (fused; no separate residual pass over x).
extern "C" int bak_solve_gram(int dtype, const void* x, int64_t obs, int64_t vars, int64_t ldx, const void* y,
                              const int32_t* cols, int64_t ncols, int64_t cols_stride, void* norms2_out, void* e,
                              void* a, int64_t max_iter, double thresh2, double* history, int64_t* status,
                              void* resid, void* workspace, int64_t workspace_bytes, void* stream) {
  g_err_clear();
  if ((dtype != BAK_F32 && dtype != BAK_F64) || obs < 1 || !gram_supported(vars) || ldx < obs || !x || !norms2_out ||
      !e || !a || !status || max_iter < 1 || (!cols && ncols != vars) || (resid && !y)) {
    set_error("bak_solve_gram: bad arguments");
    return BAK_EINVAL;
  }
  const size_t ts = dtype_size(dtype);
  if (reinterpret_cast<uintptr_t>(x) % 16 || (ldx * static_cast<int64_t>(ts)) % 16) {
    set_error("bak_solve_gram: x must be 16-byte aligned with ldx*sizeof(T) %% 16 == 0");
    return BAK_EINVAL;
  }
  if (workspace_bytes < gram_workspace_bytes(dtype, obs, vars)) {
    set_error("bak_solve_gram: workspace too small (need %lld)", (long long)gram_workspace_bytes(dtype, obs, vars));
    return BAK_EWORKSPACE;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t nblk = gram_nblk();
  char* w = static_cast<char*>(workspace);
  double* G = reinterpret_cast<double*>(w);
  w += vars * vars * 8;
  double* gpart = reinterpret_cast<double*>(w);
  w += gram_gpart_rows(dtype, obs, vars) * vars * 8;
  double* sqpart = reinterpret_cast<double*>(w);
  w += nblk * 8;
  double* delta = reinterpret_cast<double*>(w);
  w += vars * 8;
  GramCtrl* ctrl = reinterpret_cast<GramCtrl*>(w);
  w += 64;
  double* gparts_ws = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(w) + 255) & ~uintptr_t(255));
  const int64_t gparts_bytes = workspace_bytes - (reinterpret_cast<char*>(gparts_ws) - static_cast<char*>(workspace));
  BAK_CHECK_CUDA(cudaMemsetAsync(status, 0, 4 * sizeof(int64_t), st));
  const bool fuse_g0 = reinterpret_cast<uintptr_t>(e) % 16 == 0;
  if (int rc = launch_gram_g(dtype, x, obs, ldx, vars, G, gparts_ws, gparts_bytes, st, norms2_out,
                             fuse_g0 ? e : nullptr, fuse_g0 ? gpart : nullptr, status))
    return rc;
  // all-zero matrix -> the reference's ValueError (bak.py:186-187)
  {
    std::vector<unsigned char> h(static_cast<size_t>(vars) * ts);
    BAK_CHECK_CUDA(cudaMemcpyAsync(h.data(), norms2_out, h.size(), cudaMemcpyDeviceToHost, st));
    BAK_CHECK_CUDA(cudaStreamSynchronize(st));
    bool any = false;
    for (int64_t j = 0; j < vars && !any; ++j)
      any = dtype == BAK_F64 ? reinterpret_cast<double*>(h.data())[j] != 0.0
                             : reinterpret_cast<float*>(h.data())[j] != 0.0f;
    if (!any) {
      set_error("every column of x has zero norm; nothing to solve");
      return BAK_EINVAL;
    }
  }
  BAK_CHECK_CUDA(cudaMemsetAsync(ctrl, 0, sizeof(GramCtrl), st));
  const bool use_tma = gram_tma_supported(vars);
  SolveParams sp{vars, use_tma ? gram_tma_grid(dtype) : nblk, 0, max_iter, thresh2, cols, ncols, cols_stride,
                 norms2_out, G, gpart, sqpart, a, delta, history, ctrl, status};
  PassParams pp{x, obs, ldx, vars, e, delta, 0, 1, gpart, sqpart, ctrl};
  const bool fuse_resid = resid && thresh2 < 0.0 && use_tma;
  auto pass = [&](int apply, int dot, bool final_pass) -> int {
    if (use_tma)
      return launch_gram_pass_tma(dtype, x, obs, ldx, vars, e, delta, apply, dot, gpart, sqpart, &ctrl->done, st,
                                  final_pass && fuse_resid ? a : nullptr, y, resid, status);
    pp.apply = apply;
    pp.dot = dot;
    if (dtype == BAK_F64)
      gram_pass_kernel<double><<<static_cast<unsigned>(nblk), kGT, 0, st>>>(pp);
    else
      gram_pass_kernel<float><<<static_cast<unsigned>(nblk), kGT, 0, st>>>(pp);
    count_launches(1);
    BAK_CHECK_CUDA(cudaGetLastError());
    return BAK_OK;
  };
  auto solve = [&](int64_t s) -> int {
    sp.sweep = s;
    if (dtype == BAK_F64)
      gram_solve_kernel<double><<<1, 512, 0, st>>>(sp);
    else
      gram_solve_kernel<float><<<1, 512, 0, st>>>(sp);
    count_launches(1);
    BAK_CHECK_CUDA(cudaGetLastError());
    return BAK_OK;
  };
  int rc = 0;
  const int64_t pass_parts = sp.nblk;
  if (fuse_g0) {  // the first g came out of the G kernel
    int g0rows;
    int64_t chunk;
    gram_g_workspace(dtype, obs, vars, g0rows, chunk);
    sp.nblk = g0rows;
  } else if ((rc = pass(0, 1, false))) {
    return rc;
  }
  for (int64_t s = 1; s <= max_iter; ++s) {
    if ((rc = solve(s))) return rc;
    sp.nblk = pass_parts;
    if ((rc = pass(1, s < max_iter ? 1 : 0, s == max_iter))) return rc;
    if (thresh2 >= 0.0 && s % 16 == 0) {
      int64_t done = 0;
      BAK_CHECK_CUDA(cudaMemcpyAsync(&done, &ctrl->done, sizeof(done), cudaMemcpyDeviceToHost, st));
      BAK_CHECK_CUDA(cudaStreamSynchronize(st));
      if (done) break;
    }
  }
  if ((rc = solve(max_iter + 1))) return rc;
  // status[2] stays 0; bit 8 of status[3] tells the caller the residual was fused
  if (fuse_resid) {
    const int64_t v = BAK_VARIANT_GRAM | 256;
    BAK_CHECK_CUDA(cudaMemcpyAsync(status + 3, &v, sizeof(v), cudaMemcpyHostToDevice, st));
    BAK_CHECK_CUDA(cudaStreamSynchronize(st));
  }
  return BAK_OK;
}

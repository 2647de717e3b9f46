// Blocked sweep (the reference's Algorithm 2, solve_bakp).
//
// Reference semantics (baksolve 0.1.0, bakp.py:95-129), cyclic order only:
//   for sweep in range(max_iter):
//     for each block [j0, j1) of thr consecutive columns (narrower last block):
//       d_k = <x_k, e> / n2_k  for every k in the block, all against the SAME
//             (stale) e; d_k = 0 for zero-norm columns        bakp.py:52-62
//       a[j0:j1] += d                                          bakp.py:114
//       e -= x[:, j0:j1] @ d   (one T rounding of the product,
//                               one of the subtraction)        bakp.py:115-116
//     sq = <e, e>; history; divergence guard:
//       not finite or sq > prev_sq * 10  -> DivergenceError    bakp.py:118-125
//     early break when sq <= tol^2 ||y||^2                     bakp.py:126-128
//
// B200 design, two exact variants plus one labelled reformulation:
//
// kCta / kCluster (on-chip): the persistent layout of the column sweep
//   (bak_sweep.cu): e lives in registers (E rows per thread, rows tid + k*NT),
//   one producer warp streams column slices through a TMA (cp.async.bulk)
//   ring guarded by full/empty mbarriers.  The schedule per block is the
//   block's columns twice: pass 1 computes the thr partial dots (warp
//   butterflies of 4 columns interleaved, per-warp slots), pass 2 applies
//   e -= X_B d from the same ring (the second read of x_B hits L2).  The thr
//   dots are reduced ONCE per block, not once per column: per-warp slots ->
//   fixed-order sum -> (cluster) every CTA st.async's its partial vector into
//   every peer's shared memory, completing as transaction bytes on the peer's
//   mbarrier; every CTA sums the G partials in rank order, so all of them
//   hold bit-identical d.
// kStream (any shape, e in HBM): per chunk of <= 64 columns one dot kernel
//   (row tiles, fixed-order partials) and one finalize kernel (d, a += d);
//   per block one update kernel (e -= X_B d, sum e^2 partials at the sweep's
//   last block); per sweep one kernel for the guard / break.  Every kernel
//   returns at once when the device-side done flag is set.
// GRAM (labelled, algebraically equivalent; bak_gram.cu): block forward
//   substitution with G = X^T X and one pass over x per sweep.
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include "bak_common.cuh"
#include "bak_sweep.cuh"

namespace bak {
namespace {

constexpr int kModeCta = 0, kModeCluster = 1;
constexpr int kMaxCluster = 16;
constexpr int kMaxStages = 128;
constexpr int kMaxNT = 256;
constexpr int kMaxWarps = kMaxNT / 32;
constexpr int kChunk = 64;    // dots reduced / exchanged per round
constexpr int kMaxThr = 1024;  // on-chip kernels: deltas of one block kept in smem
constexpr int kBar = 1;        // named barrier for consumer warps

struct BlockParams {
  const void* x;
  int64_t obs, ldx, vars;
  const void* norms2;
  int64_t thr;
  void* e;
  void* a;
  int64_t max_iter;
  double thresh2;  // < 0: no early break
  double prev_sq;  // ||y||^2 (the guard's first reference value, bakp.py:181)
  double* history;
  int64_t* status;
  int64_t rows_per_cta;
  int nstages;
  int resident;  // 1: a block's column slices stay in the ring for pass 2 (nstages > thr)
};

__device__ __forceinline__ bool bar_consumers_or(int nthreads, int pred) {
  uint32_t r;
  asm volatile(
      "{\n\t.reg .pred p, q;\n\t"
      "setp.ne.u32 q, %1, 0;\n\t"
      "bar.red.or.pred p, %2, %3, q;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(r)
      : "r"(static_cast<uint32_t>(pred)), "r"(kBar), "r"(nthreads)
      : "memory");
  return r != 0;
}
__device__ __forceinline__ void mbar_arrive1(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
// 8-byte store into a peer CTA's shared memory, completing as tx bytes on its mbarrier
__device__ __forceinline__ void st_async_f64(uint32_t remote_addr, double v, uint32_t remote_bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(remote_addr),
               "d"(v), "r"(remote_bar)
               : "memory");
}

__host__ __device__ inline bool diverged(double sq, double prev) {
  return !(sq <= 1.79769313486231570815e308 && sq >= -1.79769313486231570815e308) || sq > prev * 10.0;
}

#ifdef BAK_PHASES
#define BPH(i)                                 \
  do {                                         \
    const long long _c = clock64();            \
    ph_acc[i] += _c - ph_last;                 \
    ph_last = _c;                              \
  } while (0)
#else
#define BPH(i) \
  do {         \
  } while (0)
#endif

template <typename T, int E, int MODE>
__global__ void __launch_bounds__(kMaxNT + 32, 1) block_kernel(const BlockParams prm) {
#ifdef BAK_PHASES
  long long ph_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long ph_last = clock64();
#endif
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int NT = static_cast<int>(blockDim.x) - 32;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = NT >> 5;
  const int S = prm.nstages;
  uint32_t rank = 0, G = 1;
  if (MODE == kModeCluster) {
    rank = cluster_rank();
    G = cluster_size();
  }
  const T* __restrict__ x = static_cast<const T*>(prm.x);
  const T* __restrict__ n2g = static_cast<const T*>(prm.norms2);
  T* __restrict__ eg = static_cast<T*>(prm.e);
  T* __restrict__ ag = static_cast<T*>(prm.a);
  const int64_t V = prm.vars, thr = prm.thr;
  const int64_t r0 = static_cast<int64_t>(rank) * prm.rows_per_cta;
  const int64_t nrows = imax64(0, imin64(prm.obs - r0, prm.rows_per_cta));
  constexpr int VEC = 16 / sizeof(T);
  const uint32_t bytes = static_cast<uint32_t>(((nrows + VEC - 1) / VEC) * VEC * sizeof(T));

  // ---- shared memory ----
  T* xs = reinterpret_cast<T*>(smem_raw);
  size_t off = static_cast<size_t>(S) * prm.rows_per_cta * sizeof(T);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + off);
  off += kMaxStages * 8;
  uint64_t* empty = reinterpret_cast<uint64_t*>(smem_raw + off);
  off += kMaxStages * 8;
  uint64_t* xbar = reinterpret_cast<uint64_t*>(smem_raw + off);  // [2]
  off += 2 * 8;
  T* red = reinterpret_cast<T*>(smem_raw + off);  // [kChunk][kMaxWarps]
  off += kChunk * kMaxWarps * sizeof(T);
  off = round16(off);
  T* dsh = reinterpret_cast<T*>(smem_raw + off);  // [kMaxThr] deltas of the current block
  off += kMaxThr * sizeof(T);
  off = round16(off);
  double* xslot = reinterpret_cast<double*>(smem_raw + off);  // [2][kMaxCluster][kChunk]
  off += (MODE == kModeCluster ? 2 * kMaxCluster * kChunk : 0) * sizeof(double);
  double* qsh = reinterpret_cast<double*>(smem_raw + off);  // sweep's sum e^2
  off += 16;
  volatile int* stop = reinterpret_cast<volatile int*>(smem_raw + off);

  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], nwarps);
    }
    mbar_init(&xbar[0], 1);
    mbar_init(&xbar[1], 1);
    *stop = 0;
    fence_mbar_init();
  }
  __syncthreads();
  if (MODE == kModeCluster) cluster_sync();

  // schedule: per sweep, per block, the block's columns twice — or once when
  // the block stays resident in the ring between its two passes
  const bool resident = prm.resident != 0;
  const int64_t per_sweep = resident ? V : 2 * V;
  const int64_t total = prm.max_iter * per_sweep;

  if (tid >= NT) {
    // =========================== producer warp ===========================
    if (lane == 0) {
      const uint64_t pol = policy_evict_last();  // x_B is read twice per block
      int s = 0;
      uint32_t ph = 0;
      int64_t u = 0, j0 = 0, k = 0;
      int pass = 0;
      bool halted = false;
      for (; u < total; ++u) {
        BPH(6);
        if (u >= S) {
          const uint32_t par = ph ^ 1u;
          if (!mbar_test(&empty[s], par)) {
            const uint64_t t0 = globaltimer();
            while (!mbar_test(&empty[s], par)) {
              if (*stop || globaltimer() - t0 > kTimeoutNs) { halted = true; break; }
            }
          }
          if (halted) break;
        }
        BPH(5);
        const int64_t c = j0 + k;
        mbar_arrive_expect_tx(&full[s], bytes);
        bulk_g2s(xs + static_cast<size_t>(s) * prm.rows_per_cta, x + c * prm.ldx + r0, bytes, &full[s], pol);
        if (++s == S) { s = 0; ph ^= 1u; }
        // advance (block, pass, column)
        const int64_t j1 = imin64(j0 + thr, V);
        if (++k == j1 - j0) {
          k = 0;
          if (pass == 0 && !resident) {
            pass = 1;
          } else {
            pass = 0;
            j0 = (j1 == V) ? 0 : j1;
          }
        }
      }
#ifdef BAK_PHASES
      if (rank == 0 && prm.history)
        for (int i = 5; i < 7; ++i) prm.history[prm.max_iter + i] = static_cast<double>(ph_acc[i]);
#endif
      for (int64_t v = imax64(0, u - S); v < u; ++v) {  // drain in-flight copies
        const int sv = static_cast<int>(v % S);
        const uint32_t pv = static_cast<uint32_t>((v / S) & 1);
        const uint64_t t0 = globaltimer();
        while (!mbar_test(&full[sv], pv))
          if (globaltimer() - t0 > kTimeoutNs) break;
      }
    }
  } else {
    // =========================== consumers ===============================
    const int kv = static_cast<int>(imax64(0, imin64(E, (nrows - tid + NT - 1) / NT)));
    T ev[E];
#pragma unroll
    for (int k = 0; k < E; ++k) ev[k] = (k < kv) ? eg[r0 + tid + static_cast<int64_t>(k) * NT] : T(0);
    int my_abort = 0;
    int ls = 0;
    uint32_t lph = 0;
    const bool full_rows = kv == E;
    const uint32_t xs_base = smem_addr(xs) + static_cast<uint32_t>(tid * sizeof(T));
    const uint32_t stage_bytes = static_cast<uint32_t>(prm.rows_per_cta * sizeof(T));
    // stage -> registers, then (unless kept for pass 2) hand it back (one arrival per warp)
    auto pull = [&](T (&xr)[E], bool keep) {
      if (tid == 0) BPH(1);
      if (!mbar_test(&full[ls], lph)) {
        const uint64_t t0 = globaltimer();
        while (!mbar_test(&full[ls], lph)) {
          if (globaltimer() - t0 > kTimeoutNs) {
            report_error(prm.status, BAK_ETIMEOUT);
            my_abort = 1;
            break;
          }
        }
      }
      if (tid == 0) BPH(0);
      const uint32_t a0 = xs_base + static_cast<uint32_t>(ls) * stage_bytes;
#pragma unroll
      for (int k = 0; k < E; ++k)
        xr[k] = (full_rows || k < kv) ? lds<T>(a0 + static_cast<uint32_t>(k * NT * sizeof(T))) : T(0);
      if (!keep) {
        __syncwarp();
        if (lane == 0) mbar_arrive1(&empty[ls]);
      }
      if (++ls == S) { ls = 0; lph ^= 1u; }
    };
    // sum n values (thread t < n holds v) over the cluster, rank order; returns
    // the total in threads t < n.  rc counts exchanges (buffer, parity).
    uint32_t rc = 0;
    auto exchange = [&](double v, int n) -> double {
      if (MODE == kModeCta) return v;
      const int buf = rc & 1;
      const uint32_t par = (rc >> 1) & 1;
      ++rc;
      if (tid < n) {
        const uint32_t loc = smem_addr(&xslot[(buf * kMaxCluster + rank) * kChunk + tid]);
        const uint32_t lb = smem_addr(&xbar[buf]);
        for (uint32_t r = 0; r < G; ++r) st_async_f64(mapa(loc, r), v, mapa(lb, r));
      }
      if (tid == 0) mbar_arrive_expect_tx(&xbar[buf], G * static_cast<uint32_t>(n) * 8u);
      double tot = 0.0;
      if (tid < n) {
        if (!mbar_test_cluster(&xbar[buf], par)) {
          const uint64_t t0 = globaltimer();
          while (!mbar_test_cluster(&xbar[buf], par)) {
            if (globaltimer() - t0 > kTimeoutNs) {
              report_error(prm.status, BAK_ETIMEOUT);
              my_abort = 1;
              break;
            }
          }
        }
        T s = T(0);
        for (uint32_t r = 0; r < G; ++r) s = Num<T>::add(s, static_cast<T>(xslot[(buf * kMaxCluster + r) * kChunk + tid]));
        tot = static_cast<double>(s);
      }
      return tot;
    };

    int64_t sweep = 0;
    bool converged = false, div = false, aborted = false;
    double prev = prm.prev_sq;
    while (sweep < prm.max_iter && !aborted) {
      for (int64_t j0 = 0; j0 < V && !aborted; j0 += thr) {
        const int64_t j1 = imin64(j0 + thr, V);
        const int ls_block = ls;  // first stage of this block (resident mode)
        // ---- pass 1: thr dots against the stale e, reduced per chunk ----
        // a chunk's dots are finished by threads t < cn: at most NT per chunk
        const int chunk = NT < kChunk ? NT : kChunk;
        for (int64_t c0 = j0; c0 < j1; c0 += chunk) {
          const int cn = static_cast<int>(imin64(chunk, j1 - c0));
          for (int i = 0; i < cn; i += 4) {
            T p[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              p[u] = T(0);
              if (i + u < cn) {
                T xr[E];
                pull(xr, resident);
                T acc[4] = {T(0), T(0), T(0), T(0)};
#pragma unroll
                for (int k = 0; k < E; ++k) acc[k & 3] = Num<T>::fma(xr[k], ev[k], acc[k & 3]);
                p[u] = Num<T>::add(Num<T>::add(acc[0], acc[1]), Num<T>::add(acc[2], acc[3]));
              }
            }
#pragma unroll
            for (int o = 16; o >= 1; o >>= 1)
#pragma unroll
              for (int u = 0; u < 4; ++u) p[u] = Num<T>::add(p[u], __shfl_xor_sync(0xffffffffu, p[u], o));
            if (lane == 0)
#pragma unroll
              for (int u = 0; u < 4; ++u)
                if (i + u < cn) red[(i + u) * kMaxWarps + warp] = p[u];
          }
          if (tid == 0) BPH(1);
          if (bar_consumers_or(NT, my_abort)) { aborted = true; break; }
          T n2 = T(1);
          double v = 0.0;
          if (tid < cn) {
            n2 = n2g[c0 + tid];
            T s = T(0);
            for (int w = 0; w < nwarps; ++w) s = Num<T>::add(s, red[tid * kMaxWarps + w]);
            v = static_cast<double>(s);
          }
          const double dot = exchange(v, cn);
          if (tid < cn) {
            const T d = (n2 != T(0)) ? Num<T>::div(static_cast<T>(dot), n2) : T(0);
            dsh[c0 - j0 + tid] = d;
            if (rank == 0) ag[c0 + tid] = Num<T>::add(ag[c0 + tid], d);
          }
          if (bar_consumers_or(NT, my_abort)) { aborted = true; break; }
        }
        if (aborted) break;
        if (tid == 0) BPH(2);
        // ---- pass 2: e -= X_B d (scratch in T, fma chain in column order) ----
        T sc[E];
#pragma unroll
        for (int k = 0; k < E; ++k) sc[k] = T(0);
        if (resident) {
          // the block's slices are still in the ring: read them again, release each
          int s2 = ls_block;
          for (int64_t j = j0; j < j1; ++j) {
            T xr[E];
            const uint32_t a0 = xs_base + static_cast<uint32_t>(s2) * stage_bytes;
#pragma unroll
            for (int k = 0; k < E; ++k)
              xr[k] = (full_rows || k < kv) ? lds<T>(a0 + static_cast<uint32_t>(k * NT * sizeof(T))) : T(0);
            __syncwarp();
            if (lane == 0) mbar_arrive1(&empty[s2]);
            if (++s2 == S) s2 = 0;
            const T d = dsh[j - j0];
#pragma unroll
            for (int k = 0; k < E; ++k) sc[k] = Num<T>::fma(xr[k], d, sc[k]);
          }
        } else {
          for (int64_t j = j0; j < j1; ++j) {
            T xr[E];
            pull(xr, false);
            const T d = dsh[j - j0];
#pragma unroll
            for (int k = 0; k < E; ++k) sc[k] = Num<T>::fma(xr[k], d, sc[k]);
          }
        }
#pragma unroll
        for (int k = 0; k < E; ++k) ev[k] = Num<T>::sub(ev[k], sc[k]);
        if (tid == 0) BPH(3);
      }
      if (aborted) break;
      // ---- sweep end: sum e^2, history, guard, early break ----
      T q[4] = {T(0), T(0), T(0), T(0)};
#pragma unroll
      for (int k = 0; k < E; ++k) q[k & 3] = Num<T>::fma(ev[k], ev[k], q[k & 3]);
      T qv = warp_sum(Num<T>::add(Num<T>::add(q[0], q[1]), Num<T>::add(q[2], q[3])));
      if (lane == 0) red[warp] = qv;
      if (bar_consumers_or(NT, my_abort)) break;
      double qd = 0.0;
      if (tid == 0) {
        T s = T(0);
        for (int w = 0; w < nwarps; ++w) s = Num<T>::add(s, red[w]);
        qd = static_cast<double>(s);
      }
      qd = exchange(qd, 1);
      if (tid == 0) {
        *qsh = qd;
        if (rank == 0 && prm.history) prm.history[sweep] = qd;
      }
      if (bar_consumers_or(NT, my_abort)) break;
      const double sq = *qsh;
      if (tid == 0) BPH(4);
      ++sweep;
      if (diverged(sq, prev)) {
        div = true;
        break;
      }
      prev = sq;
      if (prm.thresh2 >= 0.0 && sq <= prm.thresh2) {
        converged = true;
        break;
      }
    }
#pragma unroll
    for (int k = 0; k < E; ++k)
      if (k < kv) eg[r0 + tid + static_cast<int64_t>(k) * NT] = ev[k];
#ifdef BAK_PHASES
    if (tid == 0 && rank == 0 && prm.history)
      for (int i = 0; i < 5; ++i) prm.history[prm.max_iter + i] = static_cast<double>(ph_acc[i]);
#endif
    if (tid == 0) {
      *stop = 1;
      if (rank == 0 && prm.status) {
        prm.status[0] = sweep;
        prm.status[1] = converged ? 1 : 0;
        if (div) report_error(prm.status, BAK_EDIVERGED);
        prm.status[3] = MODE == kModeCta ? BAK_VARIANT_CTA : BAK_VARIANT_CLUSTER;
      }
    }
  }
  __syncthreads();
  if (MODE == kModeCluster) cluster_sync();
}

// ------------------ on-chip variant, direct-load form ----------------------
// Same schedule and reductions as block_kernel, without the producer warp and
// ring: each thread owns a CONTIGUOUS chunk of E rows (one or two 16-byte
// vector loads per column) and loads its own x values straight from L2 /
// HBM with two groups of 4 columns in flight (software pipelined), so the
// per-column cost is a few vector loads instead of a TMA issue + mbarrier
// round trip.  Pass 2 re-reads the block's columns (L2-resident).
constexpr int kLG = 4;  // columns per load group

template <typename T, int E>
__device__ __forceinline__ void ldg_rows(const T* __restrict__ p, bool vec_ok, int nvalid, T (&xr)[E]) {
  if (vec_ok) {
    if constexpr (sizeof(T) == 4) {
#pragma unroll
      for (int q = 0; q < E / 4; ++q) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(p) + q);
        xr[4 * q + 0] = v.x;
        xr[4 * q + 1] = v.y;
        xr[4 * q + 2] = v.z;
        xr[4 * q + 3] = v.w;
      }
    } else {
#pragma unroll
      for (int q = 0; q < E / 2; ++q) {
        const double2 v = __ldg(reinterpret_cast<const double2*>(p) + q);
        xr[2 * q + 0] = v.x;
        xr[2 * q + 1] = v.y;
      }
    }
  } else {
#pragma unroll
    for (int k = 0; k < E; ++k) xr[k] = (k < nvalid) ? p[k] : T(0);
  }
}

template <typename T, int E, int MODE>
__global__ void __launch_bounds__(kMaxNT, 1) block_ldg_kernel(const BlockParams prm) {
  __shared__ T red[kChunk * kMaxWarps];
  __shared__ T dsh[kMaxThr];
  __shared__ double xslot[MODE == kModeCluster ? 2 * kMaxCluster * kChunk : 1];
  __shared__ __align__(8) uint64_t xbar[2];
  __shared__ double qsh;
  const int NT = static_cast<int>(blockDim.x);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = NT >> 5;
  uint32_t rank = 0, G = 1;
  if (MODE == kModeCluster) {
    rank = cluster_rank();
    G = cluster_size();
  }
  const T* __restrict__ x = static_cast<const T*>(prm.x);
  const T* __restrict__ n2g = static_cast<const T*>(prm.norms2);
  T* __restrict__ eg = static_cast<T*>(prm.e);
  T* __restrict__ ag = static_cast<T*>(prm.a);
  const int64_t V = prm.vars, thr = prm.thr, ldx = prm.ldx;
  const int64_t row0 = static_cast<int64_t>(rank) * prm.rows_per_cta + static_cast<int64_t>(tid) * E;
  const int nvalid = static_cast<int>(imax64(0, imin64(E, prm.obs - row0)));
  const bool vec_ok = nvalid == E;
  const T* __restrict__ xt = x + (nvalid > 0 ? row0 : 0);
  if (tid == 0) {
    mbar_init(&xbar[0], 1);
    mbar_init(&xbar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (MODE == kModeCluster) cluster_sync();

  T ev[E];
#pragma unroll
  for (int k = 0; k < E; ++k) ev[k] = (k < nvalid) ? eg[row0 + k] : T(0);
  int my_abort = 0;
  uint32_t rc = 0;
  auto exchange = [&](double v, int n) -> double {
    if (MODE == kModeCta) return v;
    const int buf = rc & 1;
    const uint32_t par = (rc >> 1) & 1;
    ++rc;
    if (tid < n) {
      const uint32_t loc = smem_addr(&xslot[(buf * kMaxCluster + rank) * kChunk + tid]);
      const uint32_t lb = smem_addr(&xbar[buf]);
      for (uint32_t r = 0; r < G; ++r) st_async_f64(mapa(loc, r), v, mapa(lb, r));
    }
    if (tid == 0) mbar_arrive_expect_tx(&xbar[buf], G * static_cast<uint32_t>(n) * 8u);
    double tot = 0.0;
    if (tid < n) {
      if (!mbar_test_cluster(&xbar[buf], par)) {
        const uint64_t t0 = globaltimer();
        while (!mbar_test_cluster(&xbar[buf], par)) {
          if (globaltimer() - t0 > kTimeoutNs) {
            report_error(prm.status, BAK_ETIMEOUT);
            my_abort = 1;
            break;
          }
        }
      }
      T s = T(0);
      for (uint32_t r = 0; r < G; ++r)
        s = Num<T>::add(s, static_cast<T>(xslot[(buf * kMaxCluster + r) * kChunk + tid]));
      tot = static_cast<double>(s);
    }
    return tot;
  };
  // load columns c, c+1, ... (up to kLG, < cend) of this thread's rows
  auto load_group = [&](T (&xg)[kLG][E], int64_t c, int64_t cend) {
#pragma unroll
    for (int u = 0; u < kLG; ++u)
      if (c + u < cend) ldg_rows<T, E>(xt + (c + u) * ldx, vec_ok, nvalid, xg[u]);
  };

  int64_t sweep = 0;
  bool converged = false, div = false, aborted = false;
  double prev = prm.prev_sq;
  T xa[kLG][E], xb[kLG][E];
  while (sweep < prm.max_iter && !aborted) {
    for (int64_t j0 = 0; j0 < V && !aborted; j0 += thr) {
      const int64_t j1 = imin64(j0 + thr, V);
      // ---- pass 1: dots against the stale e ----
      const int chunk = NT < kChunk ? NT : kChunk;  // finished by threads t < cn
      for (int64_t c0 = j0; c0 < j1; c0 += chunk) {
        const int cn = static_cast<int>(imin64(chunk, j1 - c0));
        const int64_t cend = c0 + cn;
        auto dots = [&](T (&xg)[kLG][E], int i) {
          T p[kLG];
#pragma unroll
          for (int u = 0; u < kLG; ++u) {
            T acc[4] = {T(0), T(0), T(0), T(0)};
#pragma unroll
            for (int k = 0; k < E; ++k) acc[k & 3] = Num<T>::fma(xg[u][k], ev[k], acc[k & 3]);
            p[u] = Num<T>::add(Num<T>::add(acc[0], acc[1]), Num<T>::add(acc[2], acc[3]));
          }
#pragma unroll
          for (int o = 16; o >= 1; o >>= 1)
#pragma unroll
            for (int u = 0; u < kLG; ++u) p[u] = Num<T>::add(p[u], __shfl_xor_sync(0xffffffffu, p[u], o));
          if (lane == 0)
#pragma unroll
            for (int u = 0; u < kLG; ++u)
              if (i + u < cn) red[(i + u) * kMaxWarps + warp] = p[u];
        };
        load_group(xa, c0, cend);
        for (int i = 0; i < cn; i += 2 * kLG) {
          if (i + kLG < cn) load_group(xb, c0 + i + kLG, cend);
          dots(xa, i);
          if (i + 2 * kLG < cn) load_group(xa, c0 + i + 2 * kLG, cend);
          if (i + kLG < cn) dots(xb, i + kLG);
        }
        if (bar_consumers_or(NT, my_abort)) { aborted = true; break; }
        T n2 = T(1);
        double v = 0.0;
        if (tid < cn) {
          n2 = n2g[c0 + tid];
          T s = T(0);
          for (int w = 0; w < nwarps; ++w) s = Num<T>::add(s, red[tid * kMaxWarps + w]);
          v = static_cast<double>(s);
        }
        const double dot = exchange(v, cn);
        if (tid < cn) {
          const T d = (n2 != T(0)) ? Num<T>::div(static_cast<T>(dot), n2) : T(0);
          dsh[c0 - j0 + tid] = d;
          if (rank == 0) ag[c0 + tid] = Num<T>::add(ag[c0 + tid], d);
        }
        if (bar_consumers_or(NT, my_abort)) { aborted = true; break; }
      }
      if (aborted) break;
      // ---- pass 2: e -= X_B d (T scratch, fma chain in column order) ----
      T sc[E];
#pragma unroll
      for (int k = 0; k < E; ++k) sc[k] = T(0);
      auto upd = [&](T (&xg)[kLG][E], int64_t c) {
#pragma unroll
        for (int u = 0; u < kLG; ++u)
          if (c + u < j1) {
            const T d = dsh[c + u - j0];
#pragma unroll
            for (int k = 0; k < E; ++k) sc[k] = Num<T>::fma(xg[u][k], d, sc[k]);
          }
      };
      load_group(xa, j0, j1);
      for (int64_t c = j0; c < j1; c += 2 * kLG) {
        if (c + kLG < j1) load_group(xb, c + kLG, j1);
        upd(xa, c);
        if (c + 2 * kLG < j1) load_group(xa, c + 2 * kLG, j1);
        if (c + kLG < j1) upd(xb, c + kLG);
      }
#pragma unroll
      for (int k = 0; k < E; ++k) ev[k] = Num<T>::sub(ev[k], sc[k]);
    }
    if (aborted) break;
    // ---- sweep end ----
    T q[4] = {T(0), T(0), T(0), T(0)};
#pragma unroll
    for (int k = 0; k < E; ++k) q[k & 3] = Num<T>::fma(ev[k], ev[k], q[k & 3]);
    const T qv = warp_sum(Num<T>::add(Num<T>::add(q[0], q[1]), Num<T>::add(q[2], q[3])));
    if (lane == 0) red[warp] = qv;
    if (bar_consumers_or(NT, my_abort)) break;
    double qd = 0.0;
    if (tid == 0) {
      T s = T(0);
      for (int w = 0; w < nwarps; ++w) s = Num<T>::add(s, red[w]);
      qd = static_cast<double>(s);
    }
    qd = exchange(qd, 1);
    if (tid == 0) {
      qsh = qd;
      if (rank == 0 && prm.history) prm.history[sweep] = qd;
    }
    if (bar_consumers_or(NT, my_abort)) break;
    const double sq = qsh;
    ++sweep;
    if (diverged(sq, prev)) {
      div = true;
      break;
    }
    prev = sq;
    if (prm.thresh2 >= 0.0 && sq <= prm.thresh2) {
      converged = true;
      break;
    }
  }
#pragma unroll
  for (int k = 0; k < E; ++k)
    if (k < nvalid) eg[row0 + k] = ev[k];
  if (tid == 0 && rank == 0 && prm.status) {
    prm.status[0] = sweep;
    prm.status[1] = converged ? 1 : 0;
    if (div) report_error(prm.status, BAK_EDIVERGED);
    prm.status[3] = MODE == kModeCta ? BAK_VARIANT_CTA : BAK_VARIANT_CLUSTER;
  }
  __syncthreads();
  if (MODE == kModeCluster) cluster_sync();
}

// ------------------------- STREAM variant kernels -------------------------
struct BlockCtrl {
  int64_t done, sweeps, converged, diverged;
  double prev;
  double pad[3];
};

constexpr int kST = 256;  // threads per CTA of the stream kernels
constexpr int kSG = 8;    // columns per register group in the dot kernel

// partial dots of columns [c0, c0+cn) over this CTA's row tile -> part[blk][0..cn)
template <typename T>
__global__ void __launch_bounds__(kST) bdot_kernel(const T* __restrict__ x, int64_t obs, int64_t ldx, int64_t c0,
                                                   int cn, const T* __restrict__ e, double* __restrict__ part,
                                                   int64_t tile, const BlockCtrl* ctrl) {
  if (ctrl->done) return;
  __shared__ T red[kSG][kST / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t rb = static_cast<int64_t>(blockIdx.x) * tile;
  const int64_t re = imin64(obs, rb + tile);
  for (int g = 0; g < cn; g += kSG) {
    T acc[kSG];
#pragma unroll
    for (int u = 0; u < kSG; ++u) acc[u] = T(0);
    for (int64_t r = rb + tid; r < re; r += kST) {
      const T ev = e[r];
#pragma unroll
      for (int u = 0; u < kSG; ++u)
        if (g + u < cn) acc[u] = Num<T>::fma(__ldcs(x + (c0 + g + u) * ldx + r), ev, acc[u]);
    }
#pragma unroll
    for (int u = 0; u < kSG; ++u) acc[u] = warp_sum(acc[u]);
    if (lane == 0)
#pragma unroll
      for (int u = 0; u < kSG; ++u) red[u][warp] = acc[u];
    __syncthreads();
    if (tid < kSG && g + tid < cn) {
      T s = T(0);
      for (int w = 0; w < kST / 32; ++w) s = Num<T>::add(s, red[tid][w]);
      part[static_cast<int64_t>(blockIdx.x) * kChunk + g + tid] = static_cast<double>(s);
    }
    __syncthreads();
  }
}

// d for the chunk: fixed-order sum of the tile partials; a += d
template <typename T>
__global__ void bfin_kernel(const double* __restrict__ part, int nblk, int64_t c0, int cn, int64_t j0,
                            const T* __restrict__ n2g, T* __restrict__ a, T* __restrict__ dvec,
                            const BlockCtrl* ctrl) {
  if (ctrl->done) return;
  const int t = threadIdx.x;
  if (t >= cn) return;
  T s = T(0);
  for (int b = 0; b < nblk; ++b) s = Num<T>::add(s, static_cast<T>(part[static_cast<int64_t>(b) * kChunk + t]));
  const T n2 = n2g[c0 + t];
  const T d = (n2 != T(0)) ? Num<T>::div(s, n2) : T(0);
  dvec[c0 - j0 + t] = d;
  a[c0 + t] = Num<T>::add(a[c0 + t], d);
}

// e -= X_B d over this CTA's rows; at the sweep's last block also sum e^2
template <typename T>
__global__ void __launch_bounds__(kST) bupd_kernel(const T* __restrict__ x, int64_t obs, int64_t ldx, int64_t j0,
                                                   int bw, const T* __restrict__ dvec, T* __restrict__ e,
                                                   double* __restrict__ sqpart, int last, int64_t tile,
                                                   const BlockCtrl* ctrl) {
  if (ctrl->done) return;
  __shared__ T dsh[kMaxThr];
  __shared__ T red[kST / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int k = tid; k < bw; k += kST) dsh[k] = dvec[k];
  __syncthreads();
  const int64_t rb = static_cast<int64_t>(blockIdx.x) * tile;
  const int64_t re = imin64(obs, rb + tile);
  T q = T(0);
  for (int64_t r = rb + tid; r < re; r += kST) {
    T sc = T(0);
    for (int k = 0; k < bw; ++k) sc = Num<T>::fma(__ldcs(x + (j0 + k) * ldx + r), dsh[k], sc);
    const T en = Num<T>::sub(e[r], sc);
    e[r] = en;
    q = Num<T>::fma(en, en, q);
  }
  if (!last) return;
  q = warp_sum(q);
  if (lane == 0) red[warp] = q;
  __syncthreads();
  if (tid == 0) {
    T s = T(0);
    for (int w = 0; w < kST / 32; ++w) s = Num<T>::add(s, red[w]);
    sqpart[blockIdx.x] = static_cast<double>(s);
  }
}

template <typename T>
__global__ void bend_kernel(const double* __restrict__ sqpart, int nblk, int64_t sweep, int64_t max_iter,
                            double thresh2, double* history, BlockCtrl* ctrl, int64_t* status) {
  if (ctrl->done) return;
  if (threadIdx.x != 0) return;
  T s = T(0);
  for (int b = 0; b < nblk; ++b) s = Num<T>::add(s, static_cast<T>(sqpart[b]));
  const double sq = static_cast<double>(s);
  if (history) history[sweep] = sq;
  const int64_t done_sweeps = sweep + 1;
  bool stop = false;
  if (diverged(sq, ctrl->prev)) {
    ctrl->diverged = 1;
    stop = true;
  } else {
    ctrl->prev = sq;
    if (thresh2 >= 0.0 && sq <= thresh2) {
      ctrl->converged = 1;
      stop = true;
    }
  }
  if (done_sweeps >= max_iter) stop = true;
  ctrl->sweeps = done_sweeps;
  if (status) {
    status[0] = done_sweeps;
    status[1] = ctrl->converged;
    if (ctrl->diverged) status[2] = BAK_EDIVERGED;
    status[3] = BAK_VARIANT_STREAM;
  }
  if (stop) ctrl->done = 1;
}

// block_deltas (bakp.py:65-85): one pass of the dot kernel + finalize, no a update
template <typename T>
__global__ void bdelta_kernel(const double* __restrict__ part, int nblk, int64_t c0, int cn,
                              const T* __restrict__ n2g, T* __restrict__ out) {
  const int t = threadIdx.x;
  if (t >= cn) return;
  T s = T(0);
  for (int b = 0; b < nblk; ++b) s = Num<T>::add(s, static_cast<T>(part[static_cast<int64_t>(b) * kChunk + t]));
  const T n2 = n2g[c0 + t];
  out[t] = (n2 != T(0)) ? Num<T>::div(s, n2) : T(0);
}

// ------------------------------- host -------------------------------------
struct BlockPlan {
  int variant = 0;
  int parts = 1, nt = 32, e = 1, nstages = 2, resident = 0;
  int64_t rows_per_cta = 0;
};

size_t block_smem(const BlockPlan& pl, size_t ts) {
  return static_cast<size_t>(pl.nstages) * pl.rows_per_cta * ts + 2 * kMaxStages * 8 + 16 +
         kChunk * kMaxWarps * ts + 16 + kMaxThr * ts + 16 +
         (pl.variant == BAK_VARIANT_CLUSTER ? 2 * kMaxCluster * kChunk * 8 : 0) + 32 + 64;
}

bool block_fill(int dtype, int variant, int64_t obs, int nt, int e, BlockPlan& pl) {
  const size_t ts = dtype_size(dtype);
  const int64_t rows = static_cast<int64_t>(nt) * e;
  const int parts = static_cast<int>((obs + rows - 1) / rows);
  if (variant == BAK_VARIANT_CTA && parts != 1) return false;
  if (variant == BAK_VARIANT_CLUSTER && (parts < 1 || parts > kMaxCluster)) return false;
  BlockPlan c;
  c.variant = variant;
  c.parts = parts;
  c.nt = nt;
  c.e = e;
  c.rows_per_cta = rows;
  c.nstages = 0;
  const size_t cap = static_cast<size_t>(device_max_smem_optin()) - 2048;
  const size_t fixed = block_smem(c, ts);
  const size_t sb = rows * ts;
  if (fixed + 4 * sb > cap) return false;
  int s = static_cast<int>((cap - fixed) / sb);
  c.nstages = s > kMaxStages ? kMaxStages : s;
  pl = c;
  return true;
}

void block_residency(BlockPlan& pl, int64_t thr) {
  // a block stays in the ring when the ring holds it plus some prefetch
  pl.resident = pl.nstages >= thr + 2 ? 1 : 0;
}

bool block_plan(int dtype, int variant, int64_t obs, int64_t thr, BlockPlan& pl) {
  if (thr > kMaxThr) return false;
  if (variant == BAK_VARIANT_CTA) {
    for (int e : {8, 16, 4, 2, 1}) {
      const int nt = static_cast<int>(round_up((obs + e - 1) / e, 32));
      if (nt <= kMaxNT && block_fill(dtype, variant, obs, nt, e, pl)) return true;
    }
    return false;
  }
  if (variant == BAK_VARIANT_CLUSTER) {
    // as many CTAs as the cluster allows: the smallest slices (more SMs reading
    // x, more ring stages -> a block can stay resident between its two passes)
    const int64_t per = (obs + kMaxCluster - 1) / kMaxCluster;
    for (int e : {8, 16, 4}) {
      const int nt = static_cast<int>(round_up((per + e - 1) / e, 32));
      if (nt > kMaxNT) continue;
      if (block_fill(dtype, variant, obs, nt, e, pl) && pl.parts >= 2) return true;
    }
    return false;
  }
  return false;
}

template <typename T, int E, int MODE>
int block_launch_one(const BlockPlan& pl, const BlockParams& prm, cudaStream_t st) {
  auto kern = block_kernel<T, E, MODE>;
  const size_t smem = block_smem(pl, sizeof(T));
  BAK_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(pl.parts);
  cfg.blockDim = dim3(pl.nt + 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  int na = 0;
  if (MODE == kModeCluster) {
    if (pl.parts > 8) BAK_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = pl.parts;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  BAK_CHECK_CUDA(cudaLaunchKernelEx(&cfg, kern, prm));
  count_launches(1);
  return BAK_OK;
}

// direct-load kernel: E = one 32-byte chunk per thread and column
constexpr int ldg_e(int dtype) { return dtype == BAK_F64 ? 4 : 8; }

bool block_plan_ldg(int dtype, int variant, int64_t obs, int64_t thr, BlockPlan& pl) {
  if (thr > kMaxThr) return false;
  const int e = ldg_e(dtype);
  BlockPlan c;
  c.variant = variant;
  c.e = e;
  c.nstages = 0;
  c.resident = 0;
  if (variant == BAK_VARIANT_CTA) {
    const int64_t nt = round_up((obs + e - 1) / e, 32);
    if (nt > kMaxNT) return false;
    c.nt = static_cast<int>(nt);
    c.parts = 1;
  } else if (variant == BAK_VARIANT_CLUSTER) {
    const int64_t per = (obs + kMaxCluster - 1) / kMaxCluster;
    const int64_t nt = round_up((per + e - 1) / e, 32);
    if (nt > kMaxNT) return false;
    c.nt = static_cast<int>(nt);
    c.parts = static_cast<int>((obs + nt * e - 1) / (nt * e));
    if (c.parts < 2) return false;
  } else {
    return false;
  }
  c.rows_per_cta = static_cast<int64_t>(c.nt) * e;
  pl = c;
  return true;
}

template <typename T, int E, int MODE>
int block_ldg_launch(const BlockPlan& pl, const BlockParams& prm, cudaStream_t st) {
  auto kern = block_ldg_kernel<T, E, MODE>;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(pl.parts);
  cfg.blockDim = dim3(pl.nt);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  int na = 0;
  if (MODE == kModeCluster) {
    if (pl.parts > 8) BAK_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = pl.parts;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  BAK_CHECK_CUDA(cudaLaunchKernelEx(&cfg, kern, prm));
  count_launches(1);
  return BAK_OK;
}

// Default: the producer-warp TMA ring kernel (measured ~20% faster per sweep on
// the 10,000 x 1,000 paper-scale shape); BAK_BLOCK_KERNEL=ldg selects the
// direct-load kernel (tests check both against the CPU restatement and each other).
bool use_tma_block_kernel() {
  const char* k = getenv("BAK_BLOCK_KERNEL");
  return !(k && k[0] == 'l');
}

template <typename T, int MODE>
int block_launch_e(const BlockPlan& pl, const BlockParams& prm, cudaStream_t st) {
  switch (pl.e) {
    case 1: return block_launch_one<T, 1, MODE>(pl, prm, st);
    case 2: return block_launch_one<T, 2, MODE>(pl, prm, st);
    case 4: return block_launch_one<T, 4, MODE>(pl, prm, st);
    case 8: return block_launch_one<T, 8, MODE>(pl, prm, st);
    case 16: return block_launch_one<T, 16, MODE>(pl, prm, st);
  }
  set_error("bak_block_sweep: unsupported rows-per-thread %d", pl.e);
  return BAK_EUNSUPPORTED;
}

int stream_nblk(int64_t obs) {
  const int64_t want = (obs + 4 * kST - 1) / (4 * kST);
  return static_cast<int>(imax64(1, imin64(2 * device_sms(), want)));
}

int64_t stream_ws(int64_t obs) {
  const int nblk = stream_nblk(obs);
  return round_up(static_cast<int64_t>(nblk) * kChunk * 8, 256) + round_up(nblk * 8, 256) + kMaxThr * 8 +
         round_up(sizeof(BlockCtrl), 256) + 256;
}

template <typename T>
int stream_block_sweep(const BlockParams& prm, void* ws, cudaStream_t st) {
  const int nblk = stream_nblk(prm.obs);
  const int64_t tile = round_up((prm.obs + nblk - 1) / nblk, kST);
  char* w = static_cast<char*>(ws);
  double* part = reinterpret_cast<double*>(w);
  w += round_up(static_cast<int64_t>(nblk) * kChunk * 8, 256);
  double* sqpart = reinterpret_cast<double*>(w);
  w += round_up(nblk * 8, 256);
  T* dvec = reinterpret_cast<T*>(w);
  w += kMaxThr * 8;
  BlockCtrl* ctrl = reinterpret_cast<BlockCtrl*>(w);
  BlockCtrl init{};
  init.prev = prm.prev_sq;
  BAK_CHECK_CUDA(cudaMemcpyAsync(ctrl, &init, sizeof(init), cudaMemcpyHostToDevice, st));
  BAK_CHECK_CUDA(cudaMemsetAsync(prm.status, 0, 4 * sizeof(int64_t), st));
  const T* x = static_cast<const T*>(prm.x);
  T* e = static_cast<T*>(prm.e);
  T* a = static_cast<T*>(prm.a);
  const T* n2 = static_cast<const T*>(prm.norms2);
  const int64_t V = prm.vars, thr = prm.thr;
  for (int64_t s = 0; s < prm.max_iter; ++s) {
    for (int64_t j0 = 0; j0 < V; j0 += thr) {
      const int64_t j1 = imin64(j0 + thr, V);
      for (int64_t c0 = j0; c0 < j1; c0 += kChunk) {
        const int cn = static_cast<int>(imin64(kChunk, j1 - c0));
        bdot_kernel<T><<<nblk, kST, 0, st>>>(x, prm.obs, prm.ldx, c0, cn, e, part, tile, ctrl);
        bfin_kernel<T><<<1, kChunk, 0, st>>>(part, nblk, c0, cn, j0, n2, a, dvec, ctrl);
        count_launches(2);
      }
      bupd_kernel<T><<<nblk, kST, 0, st>>>(x, prm.obs, prm.ldx, j0, static_cast<int>(j1 - j0), dvec, e, sqpart,
                                           j1 == V ? 1 : 0, tile, ctrl);
      count_launches(1);
    }
    bend_kernel<T><<<1, 32, 0, st>>>(sqpart, nblk, s, prm.max_iter, prm.thresh2, prm.history, ctrl, prm.status);
    count_launches(1);
    BAK_CHECK_CUDA(cudaGetLastError());
    if (s % 16 == 15 && s + 1 < prm.max_iter) {
      int64_t done = 0;
      BAK_CHECK_CUDA(cudaMemcpyAsync(&done, &ctrl->done, sizeof(done), cudaMemcpyDeviceToHost, st));
      BAK_CHECK_CUDA(cudaStreamSynchronize(st));
      if (done) break;
    }
  }
  return BAK_OK;
}

bool block_plan_any(int dtype, int variant, int64_t obs, int64_t thr, BlockPlan& pl) {
  return use_tma_block_kernel() ? block_plan(dtype, variant, obs, thr, pl)
                                : block_plan_ldg(dtype, variant, obs, thr, pl);
}

int pick_block_variant(int dtype, int64_t obs, int64_t thr) {
  BlockPlan pl;
  if (block_plan_any(dtype, BAK_VARIANT_CTA, obs, thr, pl)) return BAK_VARIANT_CTA;
  if (block_plan_any(dtype, BAK_VARIANT_CLUSTER, obs, thr, pl)) return BAK_VARIANT_CLUSTER;
  return BAK_VARIANT_STREAM;
}

}  // namespace

int launch_gram_block(int dtype, const void* x, int64_t obs, int64_t ldx, int64_t vars, const void* norms2,
                      int64_t thr, void* e, void* a, int64_t max_iter, double thresh2, double prev_sq,
                      double* history, int64_t* status, void* ws, int64_t wsb, cudaStream_t st);

}  // namespace bak

using namespace bak;

extern "C" int bak_block_pick_variant(int dtype, int64_t obs, int64_t vars, int64_t thr) {
  (void)vars;
  return pick_block_variant(dtype, obs, thr);
}

extern "C" int64_t bak_block_sweep_workspace(int dtype, int variant, int64_t obs, int64_t vars, int64_t thr) {
  if (variant == BAK_VARIANT_AUTO) variant = pick_block_variant(dtype, obs, thr);
  if (variant == BAK_VARIANT_STREAM) return stream_ws(obs);
  if (variant == BAK_VARIANT_GRAM) return gram_workspace_bytes(dtype, obs, vars);
  return 256;
}

extern "C" int bak_block_sweep(int dtype, int variant, const void* x, int64_t obs, int64_t vars, int64_t ldx,
                               const void* norms2, int64_t thr, void* e, void* a, int64_t max_iter, double thresh2,
                               double prev_sq, double* history, int64_t* status, void* workspace,
                               int64_t workspace_bytes, void* stream) {
  g_err_clear();
  if ((dtype != BAK_F32 && dtype != BAK_F64) || obs < 1 || vars < 1 || ldx < obs || !x || !norms2 || !e || !a ||
      !status || max_iter < 1 || thr < 1 || thr > vars) {
    set_error("bak_block_sweep: bad arguments");
    return BAK_EINVAL;
  }
  const size_t ts = dtype_size(dtype);
  if (reinterpret_cast<uintptr_t>(x) % 16 || (ldx * static_cast<int64_t>(ts)) % 16) {
    set_error("bak_block_sweep: x must be 16-byte aligned with ldx*sizeof(T) %% 16 == 0");
    return BAK_EINVAL;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (variant == BAK_VARIANT_AUTO) variant = pick_block_variant(dtype, obs, thr);
  if (variant == BAK_VARIANT_GRAM)
    return launch_gram_block(dtype, x, obs, ldx, vars, norms2, thr, e, a, max_iter, thresh2, prev_sq, history,
                             status, workspace, workspace_bytes, st);
  BlockParams prm{x, obs, ldx, vars, norms2, thr, e, a, max_iter, thresh2, prev_sq, history, status, 0, 0, 0};
  if (variant == BAK_VARIANT_STREAM) {
    if (thr > kMaxThr) {
      set_error("bak_block_sweep(STREAM): thr <= %d", kMaxThr);
      return BAK_EUNSUPPORTED;
    }
    if (workspace_bytes < stream_ws(obs) || !workspace) {
      set_error("bak_block_sweep: workspace too small (need %lld)", (long long)stream_ws(obs));
      return BAK_EWORKSPACE;
    }
    return dtype == BAK_F64 ? stream_block_sweep<double>(prm, workspace, st)
                            : stream_block_sweep<float>(prm, workspace, st);
  }
  if (variant != BAK_VARIANT_CTA && variant != BAK_VARIANT_CLUSTER) {
    set_error("bak_block_sweep: variant %d not available for the blocked sweep", variant);
    return BAK_EUNSUPPORTED;
  }
  BlockPlan pl;
  if (!use_tma_block_kernel()) {
    if (!block_plan_ldg(dtype, variant, obs, thr, pl)) {
      set_error("bak_block_sweep: shape obs=%lld thr=%lld does not fit variant %d", (long long)obs,
                (long long)thr, variant);
      return BAK_EUNSUPPORTED;
    }
    prm.rows_per_cta = pl.rows_per_cta;
    BAK_CHECK_CUDA(cudaMemsetAsync(status, 0, 4 * sizeof(int64_t), st));
    int rc;
    if (dtype == BAK_F64)
      rc = variant == BAK_VARIANT_CTA ? block_ldg_launch<double, ldg_e(BAK_F64), kModeCta>(pl, prm, st)
                                      : block_ldg_launch<double, ldg_e(BAK_F64), kModeCluster>(pl, prm, st);
    else
      rc = variant == BAK_VARIANT_CTA ? block_ldg_launch<float, ldg_e(BAK_F32), kModeCta>(pl, prm, st)
                                      : block_ldg_launch<float, ldg_e(BAK_F32), kModeCluster>(pl, prm, st);
    if (rc) return rc;
    BAK_CHECK_CUDA(cudaGetLastError());
    return BAK_OK;
  }
  if (!block_plan(dtype, variant, obs, thr, pl)) {
    set_error("bak_block_sweep: shape obs=%lld thr=%lld does not fit variant %d", (long long)obs, (long long)thr,
              variant);
    return BAK_EUNSUPPORTED;
  }
  block_residency(pl, thr);
  if (const char* r = getenv("BAK_BLOCK_RESIDENT")) pl.resident = (r[0] == '1') && pl.nstages > thr;
  prm.rows_per_cta = pl.rows_per_cta;
  prm.nstages = pl.nstages;
  prm.resident = pl.resident;
  BAK_CHECK_CUDA(cudaMemsetAsync(status, 0, 4 * sizeof(int64_t), st));
  int rc;
  if (dtype == BAK_F64)
    rc = variant == BAK_VARIANT_CTA ? block_launch_e<double, kModeCta>(pl, prm, st)
                                    : block_launch_e<double, kModeCluster>(pl, prm, st);
  else
    rc = variant == BAK_VARIANT_CTA ? block_launch_e<float, kModeCta>(pl, prm, st)
                                    : block_launch_e<float, kModeCluster>(pl, prm, st);
  if (rc) return rc;
  BAK_CHECK_CUDA(cudaGetLastError());
  return BAK_OK;
}

extern "C" int64_t bak_block_deltas_workspace(int dtype, int64_t obs) {
  (void)dtype;
  return round_up(static_cast<int64_t>(stream_nblk(obs)) * kChunk * 8, 256) + 256;
}

extern "C" int bak_block_deltas(int dtype, const void* x, int64_t obs, int64_t vars, int64_t ldx, int64_t j0,
                                int64_t j1, const void* e, const void* norms2, void* out, void* workspace,
                                int64_t workspace_bytes, void* stream) {
  g_err_clear();
  if ((dtype != BAK_F32 && dtype != BAK_F64) || obs < 1 || ldx < obs || !x || !e || !norms2 || !out ||
      !(0 <= j0 && j0 < j1 && j1 <= vars)) {
    set_error("bak_block_deltas: bad arguments");
    return BAK_EINVAL;
  }
  if (workspace_bytes < bak_block_deltas_workspace(dtype, obs) || !workspace) {
    set_error("bak_block_deltas: workspace too small");
    return BAK_EWORKSPACE;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int nblk = stream_nblk(obs);
  const int64_t tile = round_up((obs + nblk - 1) / nblk, kST);
  double* part = static_cast<double*>(workspace);
  // the dot kernel's done flag: a zeroed int64 after the partials
  int64_t* flag = reinterpret_cast<int64_t*>(static_cast<char*>(workspace) +
                                             round_up(static_cast<int64_t>(nblk) * kChunk * 8, 256));
  BAK_CHECK_CUDA(cudaMemsetAsync(flag, 0, 8, st));
  for (int64_t c0 = j0; c0 < j1; c0 += kChunk) {
    const int cn = static_cast<int>(imin64(kChunk, j1 - c0));
    if (dtype == BAK_F64) {
      bdot_kernel<double><<<nblk, kST, 0, st>>>(static_cast<const double*>(x), obs, ldx, c0, cn,
                                                static_cast<const double*>(e), part, tile,
                                                reinterpret_cast<const BlockCtrl*>(flag));
      bdelta_kernel<double><<<1, kChunk, 0, st>>>(part, nblk, c0, cn, static_cast<const double*>(norms2),
                                                  static_cast<double*>(out) + (c0 - j0));
    } else {
      bdot_kernel<float><<<nblk, kST, 0, st>>>(static_cast<const float*>(x), obs, ldx, c0, cn,
                                               static_cast<const float*>(e), part, tile,
                                               reinterpret_cast<const BlockCtrl*>(flag));
      bdelta_kernel<float><<<1, kChunk, 0, st>>>(part, nblk, c0, cn, static_cast<const float*>(norms2),
                                                 static_cast<float*>(out) + (c0 - j0));
    }
    count_launches(2);
  }
  BAK_CHECK_CUDA(cudaGetLastError());
  return BAK_OK;
}

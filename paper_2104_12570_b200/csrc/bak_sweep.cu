// Persistent column-sweep kernels (north-star components (2) and (3)).
//
// Reference semantics (baksolve 0.1.0, bak.py):
//   for sweep in range(max_iter):                       bak.py:97
//     for j in order:                                   bak.py:100
//       da = dot(x_j, e) / n2_j                         bak.py:86
//       e -= fl(x_j * da)   (two roundings)             bak.py:87-88
//       a_j += da                                       bak.py:89
//     sq = dot(e, e); history.append(sq)                bak.py:106-108
//     if sq <= thresh2: converged; break                bak.py:109-111
//
// B200 design.  P participants (CTAs) each own a contiguous row block of e,
// held in REGISTERS for the whole solve (E rows per thread, rows tid + k*NT so
// shared-memory reads are conflict-free).  Each CTA = NT consumer threads +
// one PRODUCER warp.  The producer walks the column schedule S steps ahead:
// it reads col(u), n2 = n2[col(u)] and 1/n2 into a per-stage smem record and
// issues one cp.async.bulk (TMA engine) for the CTA's slice of that column
// (contiguous in column-major x) into an S-stage ring guarded by full/empty
// mbarriers.  x never depends on e, so every global-memory latency of the
// schedule (column list, norms, x itself) is off the consumers' critical path.
//
// Consumers keep columns t, t+1 (and t+2 when registers allow) in registers:
//     pull x_{t+2}: smem -> registers (overlaps the arithmetic below)
//     d_t = P_t / n2_t   (correctly rounded: q0 = P*r, q = q0 + (P - q0*n2)*r,
//                         r = RN(1/n2) precomputed by the producer)
//     fused:  e -= fl(d_t * x_t) ; p += x_{t+1} . e  (+ sum e^2 at sweep end)
//     warp xor-butterfly -> per-warp slots -> named barrier -> fixed-order tree
//     -> exchange across participants -> every consumer holds P_{t+1}.
// Exchange by MODE:
//   kCta     : single CTA, nothing to exchange.
//   kCluster : thread-block cluster (2..16 CTAs).  Each CTA st.async's its
//              16-byte {p, sq} into every peer's shared slot, completing as
//              transaction bytes on the peer's mbarrier (DSMEM, no flags).
//   kGrid    : co-resident persistent grid (cooperative launch).  Each CTA
//              posts an epoch-tagged 16-byte record; CTA 0 (the aggregator)
//              sums all of them in fixed order and posts the total into every
//              CTA's private 128-byte result line, which that CTA polls.  No
//              L2 line is polled by more than one CTA.
// Every participant sums the same values in the same order, so all of them
// compute bit-identical d_j; the reduction order depends only on the shape.
#include <cstdio>
#include <cstdlib>

#include "bak_common.cuh"
#include "bak_sweep.cuh"
#include "bak_tmem.cuh"

namespace bak {
namespace {

constexpr int kModeCta = 0, kModeCluster = 1, kModeGrid = 2, kModeGridCl = 3;
constexpr int kGridCluster = 8;  // CTAs per cluster in kModeGridCl (portable size)
constexpr int kMaxCluster = 16;
constexpr int kMaxStages = 32;      // ring slots (XS plans use up to 32 sub-column slots)
constexpr int kMaxRegStages = 16;   // register-resident plans: whole-column stages

// XS: sub-stages per column.  Quarters: eighths were measured no faster at
// 2^21 rows and slower at 2^20 (more waits / releases per column step,
// profiles/r02_xs_phases.txt)
// XT (XS == 2): the ring slot is one 8-row-per-thread chunk (one tcgen05.ld /
// tcgen05.st of the TMEM stash), E / 8 slots per column.
constexpr int kXtChunk = 8;
#ifndef BAK_XT_SLOT_CHUNKS
#define BAK_XT_SLOT_CHUNKS 1  // 2 (16-row slots, half the ring waits) measured 18 % slower at 2^21 rows
#endif
// XT: chunks per ring slot (2 when E splits into 16-row slots: half the ring waits / releases)
template <int E>
__host__ __device__ constexpr int xt_cs() { return (BAK_XT_SLOT_CHUNKS == 2 && E % (2 * kXtChunk) == 0) ? 2 : 1; }
template <int E, int XS = 1>
__host__ __device__ constexpr int xs_nq() { return XS == 2 ? E / (kXtChunk * xt_cs<E>()) : 4; }
constexpr int kMaxConsumers = 256;
constexpr int kBarConsumers = 1;  // named barrier id used by consumer warps only


struct alignas(16) Pair {
  double p, q;
};

struct alignas(32) StageMeta {
  int64_t col;
  double n2;
  double rinv;
  double pad;
};

__device__ __forceinline__ bool bar_or(int nthreads, int pred) {
  uint32_t r;
  asm volatile(
      "{\n\t.reg .pred p, q;\n\t"
      "setp.ne.u32 q, %1, 0;\n\t"
      "bar.red.or.pred p, %2, %3, q;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(r)
      : "r"(static_cast<uint32_t>(pred)), "r"(kBarConsumers), "r"(nthreads)
      : "memory");
  return r != 0;
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}

// correctly rounded a/b from r = RN(1/b): one Markstein correction step
template <typename T>
__device__ __forceinline__ T quotient(T a, T b, T r) {
  const T q0 = Num<T>::mul(a, r);
  const T rem = Num<T>::fma(-q0, b, a);
  return Num<T>::fma(rem, r, q0);
}

// N values of T as the 32-bit registers one tcgen05.ld / tcgen05.st moves
template <typename T, int N>
struct TmemRegs;
template <>
struct TmemRegs<double, 8> {
  uint32_t r[16];
  __device__ __forceinline__ void set(int i, double v) {
    r[2 * i] = static_cast<uint32_t>(__double2loint(v));
    r[2 * i + 1] = static_cast<uint32_t>(__double2hiint(v));
  }
  __device__ __forceinline__ double get(int i) const {
    return __hiloint2double(static_cast<int>(r[2 * i + 1]), static_cast<int>(r[2 * i]));
  }
  __device__ __forceinline__ void load(uint32_t taddr) { tmem_ld_x16(taddr, r); }
  __device__ __forceinline__ void wait() { tmem_wait_ld_x16(r); }
  __device__ __forceinline__ void store(uint32_t taddr) const { tmem_st_x16(taddr, r); }
};
template <>
struct TmemRegs<float, 8> {
  uint32_t r[8];
  __device__ __forceinline__ void set(int i, float v) { r[i] = __float_as_uint(v); }
  __device__ __forceinline__ float get(int i) const { return __uint_as_float(r[i]); }
  __device__ __forceinline__ void load(uint32_t taddr) { tmem_ld_x8(taddr, r); }
  __device__ __forceinline__ void wait() { tmem_wait_ld_x8(r); }
  __device__ __forceinline__ void store(uint32_t taddr) const { tmem_st_x8(taddr, r); }
};

#ifdef BAK_PHASES
#define PH(i)                                  \
  do {                                         \
    if (tid == 0) {                            \
      const long long _c = clock64();          \
      ph_acc[i] += _c - ph_acc[8];             \
      ph_acc[8] = _c;                          \
    }                                          \
  } while (0)
#else
#define PH(i) \
  do {        \
  } while (0)
#endif

// XS (x from shared memory, for row blocks too large to keep two columns of x
// in registers next to e — up to ~2.2M fp64 rows on one GPU): e stays in
// registers (E rows per thread), the ring holds QUARTER columns (slot = the
// rows of E/4 of each thread's row slots), the fused update/dot reads x_t and
// x_{t+1} straight from the ring, and each consumer warp hands a quarter of
// x_t back to the producer as soon as it has read it — so the load of x_{t+2}
// starts during step t's arithmetic and overlaps the exchange that follows.
template <typename T, int E, int MODE, int MAXNT, int XS = 0>
__global__ void __launch_bounds__(MAXNT + 32, 1) sweep_kernel(const SweepParams prm) {
#ifdef BAK_PHASES
  // counters in shared memory (tid 0 only): registers would spill the E = 80 plans
  __shared__ long long ph_acc[10];
  if (threadIdx.x == 0) {
    for (int i = 0; i < 8; ++i) ph_acc[i] = 0;
    ph_acc[9] = 0;
    ph_acc[8] = clock64();
  }
#endif
  constexpr int kMaxWarps = MAXNT / 32;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int NT = static_cast<int>(blockDim.x) - 32;  // consumers; the last warp produces
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = NT >> 5;
  const int S = prm.nstages;

  uint32_t rank = 0, G = 1;
  uint32_t crank = 0, C = 1;  // kModeGridCl: rank within the cluster, cluster size
  if (MODE == kModeCluster) {
    rank = cluster_rank();
    G = cluster_size();
  } else if (MODE == kModeGrid) {
    rank = blockIdx.x;
    G = gridDim.x;
  } else if (MODE == kModeGridCl) {
    rank = blockIdx.x;
    G = gridDim.x;
    crank = cluster_rank();
    C = cluster_size();
  }

  const T* __restrict__ x = static_cast<const T*>(prm.x);
  const T* __restrict__ n2g = static_cast<const T*>(prm.norms2);
  T* __restrict__ eg = static_cast<T*>(prm.e);
  T* __restrict__ ag = static_cast<T*>(prm.a);
  const int64_t r0 = static_cast<int64_t>(rank) * prm.rows_per_cta;
  const int64_t nrows = imax64(0, imin64(prm.obs - r0, prm.rows_per_cta));
  constexpr int VEC = 16 / sizeof(T);
  const uint32_t bytes = static_cast<uint32_t>(((nrows + VEC - 1) / VEC) * VEC * sizeof(T));

  // ---- shared memory carve-up ----
  T* xs = reinterpret_cast<T*>(smem_raw);
  size_t off = static_cast<size_t>(S) * prm.stage_elems * sizeof(T);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + off);
  off += kMaxStages * 8;
  uint64_t* empty = reinterpret_cast<uint64_t*>(smem_raw + off);
  off += kMaxStages * 8;
  StageMeta* meta = reinterpret_cast<StageMeta*>(smem_raw + off);
  off += kMaxStages * sizeof(StageMeta);
  T* red = reinterpret_cast<T*>(smem_raw + off);  // [2 bufs][2 values][32 warps]
  off += 2 * 2 * 32 * sizeof(T);
  off = (off + 15) & ~size_t(15);
  Pair* xslot = reinterpret_cast<Pair*>(smem_raw + off);  // [2][kMaxCluster]
  off += 2 * kMaxCluster * sizeof(Pair);
  uint64_t* xbar = reinterpret_cast<uint64_t*>(smem_raw + off);  // [2]
  off += 2 * 8;
  Pair* bcast = reinterpret_cast<Pair*>(smem_raw + off);  // [2]
  off += 2 * sizeof(Pair);
  uint64_t* xbar2 = reinterpret_cast<uint64_t*>(smem_raw + off);  // [2] kModeGridCl broadcast
  off += 2 * 8;
  volatile int* stop = reinterpret_cast<volatile int*>(smem_raw + off);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem_raw + off + 8);  // XT: TMEM base address

  if (XS == 2 && warp == 0) tmem_alloc512(smem_addr(tmem_slot));  // all 512 columns: one CTA per SM
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], XS ? static_cast<uint32_t>(nwarps) : 1u);  // XS: one arrive per consumer warp
    }
    mbar_init(&xbar[0], 1);
    mbar_init(&xbar[1], 1);
    mbar_init(&xbar2[0], 1);
    mbar_init(&xbar2[1], 1);
    *stop = 0;
    fence_mbar_init();
  }
  if (XS == 2) tmem_fence_before_sync();
  __syncthreads();
  if (XS == 2) tmem_fence_after_sync();
  const uint32_t tmem_base = (XS == 2) ? *tmem_slot : 0u;
  if (MODE == kModeCluster || MODE == kModeGridCl) cluster_sync();

  const int64_t ncols = prm.ncols;
  const int64_t total = prm.max_iter * ncols;

  if (tid >= NT && XS) {
    // ======================= producer warp (XS: sub-column slots) =======================
    constexpr int NQ = xs_nq<E, XS>();
    const int64_t QR = static_cast<int64_t>(E / NQ) * NT;  // rows per sub-column slot
    const uint64_t pol = policy_evict_first();
    int64_t f = 0;  // fills issued (4 per column step)
    int sl = 0;     // its ring slot and the parity of that slot's next fill
    uint32_t fph = 0;
    bool halted = false;
    for (int64_t u0 = 0; u0 < total && !halted; u0 += 32) {
      const int64_t ul = u0 + lane;
      int64_t cl = 0;
      T n2l = T(1);
      if (ul < total) {
        const int64_t sw = ul / ncols, k = ul - sw * ncols;
        cl = prm.cols ? static_cast<int64_t>(prm.cols[sw * prm.cols_stride + k]) : k;
        n2l = n2g[cl];
      }
      const T ril = Num<T>::div(T(1), n2l);
      const int nb = static_cast<int>(imin64(32, total - u0));
      for (int i = 0; i < nb; ++i) {
        const int64_t c = __shfl_sync(0xffffffffu, cl, i);
        const T n2 = __shfl_sync(0xffffffffu, n2l, i);
        const T ri = __shfl_sync(0xffffffffu, ril, i);
        if (lane == 0) {
          for (int q = 0; q < NQ && !halted; ++q) {
            if (f >= S) {
              const uint32_t par = fph ^ 1u;
              if (!mbar_test(&empty[sl], par)) {
                const uint64_t t0 = globaltimer();
                while (!mbar_test(&empty[sl], par)) {
                  if (*stop || globaltimer() - t0 > kTimeoutNs) { halted = true; break; }
                }
              }
              if (halted) break;
            }
            if (q == 0) {
              StageMeta& m = meta[(u0 + i) % kMaxStages];
              m.col = c;
              m.n2 = static_cast<double>(n2);
              m.rinv = static_cast<double>(ri);
            }
            const int64_t rq = imax64(0, imin64(nrows - q * QR, QR));
            const uint32_t bq = static_cast<uint32_t>(((rq + VEC - 1) / VEC) * VEC * sizeof(T));
            mbar_arrive_expect_tx(&full[sl], bq);  // release: the column record is visible with the phase
            if (bq) bulk_g2s(xs + static_cast<size_t>(sl) * prm.stage_elems, x + c * prm.ldx + r0 + q * QR, bq,
                             &full[sl], pol);
            ++f;
            if (++sl == S) {
              sl = 0;
              fph ^= 1u;
            }
          }
        }
        halted = __shfl_sync(0xffffffffu, halted, 0);
        if (halted) break;
      }
    }
    if (lane == 0) {  // the last min(S, f) copies must land before this CTA exits
      for (int64_t v = imax64(0, f - S); v < f; ++v) {
        const uint64_t t0 = globaltimer();
        while (!mbar_test(&full[v % S], static_cast<uint32_t>((v / S) & 1)))
          if (globaltimer() - t0 > kTimeoutNs) break;
      }
    }
  } else if (tid >= NT) {
    // =========================== producer warp ===========================
    // The whole warp prepares the next 32 schedule steps at once (lane l:
    // column index, n2 and 1/n2 of step u0 + l — the dependent global load and
    // the division leave the per-column critical path); lane 0 then issues the
    // 32 stage fills in order (wait for the stage, write its record, TMA).
    {
      const uint64_t pol = policy_evict_first();
      int s = 0;
      uint32_t ph = 0;
      int64_t u = 0;
      bool halted = false;
      for (int64_t u0 = 0; u0 < total && !halted; u0 += 32) {
        const int64_t ul = u0 + lane;
        int64_t cl = 0;
        T n2l = T(1);
        if (ul < total) {
          const int64_t sw = ul / ncols, k = ul - sw * ncols;
          cl = prm.cols ? static_cast<int64_t>(prm.cols[sw * prm.cols_stride + k]) : k;
          n2l = n2g[cl];
        }
        const T ril = Num<T>::div(T(1), n2l);
        const int nb = static_cast<int>(imin64(32, total - u0));
        for (int i = 0; i < nb; ++i) {
          const int64_t c = __shfl_sync(0xffffffffu, cl, i);
          const T n2 = __shfl_sync(0xffffffffu, n2l, i);
          const T ri = __shfl_sync(0xffffffffu, ril, i);
          if (lane == 0) {
            if (u >= S) {
              const uint32_t par = ph ^ 1u;
              if (!mbar_test(&empty[s], par)) {
                const uint64_t t0 = globaltimer();
                while (!mbar_test(&empty[s], par)) {
                  if (*stop || globaltimer() - t0 > kTimeoutNs) { halted = true; break; }
                }
              }
            }
            if (!halted) {
              meta[s].col = c;
              meta[s].n2 = static_cast<double>(n2);
              meta[s].rinv = static_cast<double>(ri);
              mbar_arrive_expect_tx(&full[s], bytes);  // release: meta visible with the phase
              bulk_g2s(xs + static_cast<size_t>(s) * prm.stage_elems, x + c * prm.ldx + r0, bytes, &full[s], pol);
              if (++s == S) { s = 0; ph ^= 1u; }
              ++u;
            }
          }
          halted = __shfl_sync(0xffffffffu, halted, 0);
          if (halted) break;
        }
      }
      // drain: the last min(S, u) issued copies must land before this CTA exits
      if (lane == 0) {
        for (int64_t v = imax64(0, u - S); v < u; ++v) {
          const int sv = static_cast<int>(v % S);
          const uint32_t pv = static_cast<uint32_t>((v / S) & 1);
          const uint64_t t0 = globaltimer();
          while (!mbar_test(&full[sv], pv))
            if (globaltimer() - t0 > kTimeoutNs) break;
        }
      }
    }
  } else {
    // =========================== consumers ===============================
    const int kv = static_cast<int>(imax64(0, imin64(E, (nrows - tid + NT - 1) / NT)));
    T ev[E], xc[XS ? 1 : E], xn[XS ? 1 : E];
#pragma unroll
    for (int k = 0; k < E; ++k) ev[k] = (k < kv) ? eg[r0 + tid + static_cast<int64_t>(k) * NT] : T(0);

    int my_abort = 0;
    int ls = 0;        // stage of the next step to pull into registers
    uint32_t lph = 0;  // its phase parity

    // stage -> registers (pad rows beyond obs read as 0); returns the stage index.
    // 32-bit shared addresses; the unmasked path is taken when this thread's E rows
    // are all inside the system (every CTA but the ragged last one).
    const bool full_rows = kv == E;
    const uint32_t xs_base = smem_addr(xs) + static_cast<uint32_t>(tid * sizeof(T));
    const uint32_t stage_bytes = static_cast<uint32_t>(prm.stage_elems * sizeof(T));
    auto pull = [&](T* xr, int64_t& c, T& n2, T& rinv) -> int {
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
      c = meta[ls].col;
      n2 = static_cast<T>(meta[ls].n2);
      rinv = static_cast<T>(meta[ls].rinv);
      const uint32_t a0 = xs_base + static_cast<uint32_t>(ls) * stage_bytes;
      if (full_rows) {
#pragma unroll
        for (int k = 0; k < E; ++k) xr[k] = lds<T>(a0 + static_cast<uint32_t>(k * NT * sizeof(T)));
      } else {
#pragma unroll
        for (int k = 0; k < E; ++k) xr[k] = (k < kv) ? lds<T>(a0 + static_cast<uint32_t>(k * NT * sizeof(T))) : T(0);
      }
      const int got = ls;
      if (++ls == S) { ls = 0; lph ^= 1u; }
      return got;
    };

    // fixed-order tree over the per-warp partials in shared memory
    auto warp_partials = [&](const T* v) -> T {
      constexpr int kTree = kMaxWarps <= 1 ? 1 : (kMaxWarps <= 2 ? 2 : (kMaxWarps <= 4 ? 4 : 8));  // pow2 >= warps
      T a[kTree];
#pragma unroll
      for (int w = 0; w < kTree; ++w) a[w] = (w < nwarps) ? v[w] : T(0);
#pragma unroll
      for (int h = kTree / 2; h >= 1; h >>= 1)
#pragma unroll
        for (int w = 0; w < h; ++w) a[w] = Num<T>::add(a[w], a[w + h]);
      return a[0];
    };

    // reduction across all participants; returns true on (uniform) abort.
    // rel0/rel1: stages to hand back to the producer once every consumer has
    // passed the barrier (their contents are in registers by then).
    auto reduce = [&](T pv, T qv, bool with_q, uint32_t rc, int rel0, int rel1, T& P, T& Q) -> bool {
      const int buf = rc & 1;
      pv = warp_sum(pv);
      if (with_q) qv = warp_sum(qv);
      PH(3);
      T bp, bq;
      if (kMaxWarps == 1) {
        if (__any_sync(0xffffffffu, my_abort)) return true;
        __syncwarp();
        if (lane == 0) {
          if (rel0 >= 0) mbar_arrive(&empty[rel0]);
          if (rel1 >= 0) mbar_arrive(&empty[rel1]);
        }
        bp = pv;
        bq = qv;
      } else {
        if (lane == 0) {
          red[(buf * 2 + 0) * 32 + warp] = pv;
          red[(buf * 2 + 1) * 32 + warp] = qv;
        }
        if (bar_or(NT, my_abort)) return true;
        if (tid == 0) {
          if (rel0 >= 0) mbar_arrive(&empty[rel0]);
          if (rel1 >= 0) mbar_arrive(&empty[rel1]);
        }
        bp = warp_partials(red + (buf * 2 + 0) * 32);
        bq = with_q ? warp_partials(red + (buf * 2 + 1) * 32) : T(0);
      }
      PH(4);
      if (MODE == kModeCta) {
        P = bp;
        Q = bq;
        return false;
      }
      if (MODE == kModeCluster) {
        if (tid < static_cast<int>(G)) {
          const uint32_t rs = mapa(smem_addr(&xslot[buf * kMaxCluster + rank]), tid);
          const uint32_t rb = mapa(smem_addr(&xbar[buf]), tid);
          st_async_v2(rs, static_cast<double>(bp), static_cast<double>(bq), rb);
        }
        if (tid == 0) mbar_arrive_expect_tx(&xbar[buf], G * 16u);
        const uint32_t par = (rc >> 1) & 1;
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
        T sp[kMaxCluster], sq[kMaxCluster];
#pragma unroll
        for (int r = 0; r < kMaxCluster; ++r) {
          const bool in = r < static_cast<int>(G);
          sp[r] = in ? static_cast<T>(xslot[buf * kMaxCluster + r].p) : T(0);
          sq[r] = (in && with_q) ? static_cast<T>(xslot[buf * kMaxCluster + r].q) : T(0);
        }
#pragma unroll
        for (int h = kMaxCluster / 2; h >= 1; h >>= 1)
#pragma unroll
          for (int r = 0; r < h; ++r) {
            sp[r] = Num<T>::add(sp[r], sp[r + h]);
            sq[r] = Num<T>::add(sq[r], sq[r + h]);
          }
        P = sp[0];
        Q = sq[0];
        return false;
      }
      if (MODE == kModeGridCl) {
        // (1) cluster: every CTA st.async's its partial into every peer's slot
        //     (DSMEM, completes as tx bytes on the peer's mbarrier) -> every CTA
        //     sums the cluster's C partials in rank order;
        // (2) grid: each cluster leader posts the cluster sum as an epoch-tagged
        //     record, gathers the ncl records (one per lane, <= 32 clusters) and
        //     sums them with a fixed butterfly -> identical bits in every leader;
        // (3) the leader st.async's the total into every peer of its cluster.
        const uint32_t par = (rc >> 1) & 1;
        if (tid < static_cast<int>(C)) {
          const uint32_t rs = mapa(smem_addr(&xslot[buf * kMaxCluster + crank]), tid);
          const uint32_t rb = mapa(smem_addr(&xbar[buf]), tid);
          st_async_v2(rs, static_cast<double>(bp), static_cast<double>(bq), rb);
        }
        if (tid == 0) {
          mbar_arrive_expect_tx(&xbar[buf], C * 16u);
          mbar_arrive_expect_tx(&xbar2[buf], 16u);
        }
        bool timed_out = false;
        if (crank == 0 && warp == 0) {
          if (!mbar_test_cluster(&xbar[buf], par)) {
            const uint64_t t0 = globaltimer();
            while (!mbar_test_cluster(&xbar[buf], par))
              if (globaltimer() - t0 > kTimeoutNs) { timed_out = true; break; }
          }
          T cp = T(0), cq = T(0);
          for (uint32_t r = 0; r < C; ++r) {
            cp = Num<T>::add(cp, static_cast<T>(xslot[buf * kMaxCluster + r].p));
            if (with_q) cq = Num<T>::add(cq, static_cast<T>(xslot[buf * kMaxCluster + r].q));
          }
          const uint32_t epoch = rc + 1;
          uint32_t* part = prm.slots + static_cast<size_t>(buf) * kGridSlotsMax * 8;
          const uint32_t cid = blockIdx.x / C, ncl = gridDim.x / C;
          if (lane == 0) {
            ll_store(part + static_cast<size_t>(cid) * 8, static_cast<double>(cp), epoch);
            if (with_q) ll_store(part + static_cast<size_t>(cid) * 8 + 4, static_cast<double>(cq), epoch);
          }
          T vp = T(0), vq = T(0);
          if (lane < static_cast<int>(ncl)) {
            double v = 0.0;
            const uint64_t t0 = globaltimer();
            while (!ll_load(part + static_cast<size_t>(lane) * 8, epoch, v))
              if (globaltimer() - t0 > kTimeoutNs) { timed_out = true; break; }
            vp = static_cast<T>(v);
            if (with_q) {
              while (!ll_load(part + static_cast<size_t>(lane) * 8 + 4, epoch, v))
                if (globaltimer() - t0 > kTimeoutNs) { timed_out = true; break; }
              vq = static_cast<T>(v);
            }
          }
          T sp = warp_sum(vp);
          T sq = with_q ? warp_sum(vq) : T(0);
          if (prm.nranks > 0) {
            // cross-GPU stage (row sharding): rank totals through the mailboxes
            // (peer-mapped memory, system-scope epoch-tagged records), summed in
            // rank order -> identical bits on every rank
            const int N = prm.nranks;
            const uint32_t xepoch = prm.epoch_base + rc + 1;
            if (cid == 0 && lane < N) {
              uint32_t* dst = prm.mbox[lane] + (static_cast<size_t>(buf) * N + prm.grank) * 8;
              ll_store_sys(dst, static_cast<double>(sp), xepoch);
              ll_store_sys(dst + 4, static_cast<double>(sq), xepoch);
            }
            double rp = 0.0, rq = 0.0;
            if (lane < N) {
              const uint32_t* src = prm.mbox[prm.grank] + (static_cast<size_t>(buf) * N + lane) * 8;
              const uint64_t t0 = globaltimer();
              while (!ll_load_sys(src, xepoch, rp))
                if (globaltimer() - t0 > kTimeoutNs) { timed_out = true; break; }
              if (with_q)
                while (!ll_load_sys(src + 4, xepoch, rq))
                  if (globaltimer() - t0 > kTimeoutNs) { timed_out = true; break; }
            }
            T tp = T(0), tq = T(0);
            for (int r = 0; r < N; ++r) {
              tp = Num<T>::add(tp, static_cast<T>(__shfl_sync(0xffffffffu, rp, r)));
              if (with_q) tq = Num<T>::add(tq, static_cast<T>(__shfl_sync(0xffffffffu, rq, r)));
            }
            sp = tp;
            sq = tq;
          }
          if (lane < static_cast<int>(C)) {
            const uint32_t rs = mapa(smem_addr(&bcast[buf]), lane);
            const uint32_t rb = mapa(smem_addr(&xbar2[buf]), lane);
            st_async_v2(rs, static_cast<double>(sp), static_cast<double>(sq), rb);
          }
        }
        if (warp == 0) {
          if (!mbar_test_cluster(&xbar2[buf], par)) {
            const uint64_t t0 = globaltimer();
            while (!mbar_test_cluster(&xbar2[buf], par))
              if (globaltimer() - t0 > kTimeoutNs) { timed_out = true; break; }
          }
          if (timed_out) {
            report_error(prm.status, BAK_ETIMEOUT);
            my_abort = 1;
          }
        }
        const bool any2 = bar_or(NT, my_abort);
        P = static_cast<T>(bcast[buf].p);
        Q = static_cast<T>(bcast[buf].q);
        return any2;
      }
      // kModeGrid: partial records -> aggregator (CTA 0) -> per-CTA result lines;
      // or (prm.grid_allgather) every CTA gathers all G records itself — one
      // L2 round trip instead of two (records double-buffered by round: a CTA
      // can post round rc+2 only after every CTA posted rc+1, i.e. finished
      // reading round rc)
      const uint32_t epoch = rc + 1;
      uint32_t* part = prm.slots + static_cast<size_t>(buf) * kGridSlotsMax * 8;
      uint32_t* result = prm.slots + static_cast<size_t>(2) * kGridSlotsMax * 8 +
                         static_cast<size_t>(buf) * kGridSlotsMax * 32;
      if (tid == 0) {
        ll_store(part + static_cast<size_t>(rank) * 8, static_cast<double>(bp), epoch);
        if (with_q) ll_store(part + static_cast<size_t>(rank) * 8 + 4, static_cast<double>(bq), epoch);
      }
      bool timed_out = false;
      const bool ag = prm.grid_allgather != 0;
      if (warp == 0) {
        if (rank == 0 || ag) {
          // aggregator: lane l owns records l, l+32, ... (<= 8 per lane), all in flight together
          constexpr int kPer = kGridSlotsMax / 32;
          T vp[kPer], vq[kPer];
          uint32_t pending = 0;
#pragma unroll
          for (int i = 0; i < kPer; ++i) {
            vp[i] = T(0);
            vq[i] = T(0);
            if (lane + 32 * i < static_cast<int>(G)) pending |= (with_q ? 3u : 1u) << (2 * i);
          }
          const uint64_t t0 = globaltimer();
          while (pending) {
#pragma unroll
            for (int i = 0; i < kPer; ++i) {
              double v;
              if ((pending >> (2 * i)) & 1u) {
                if (ll_load(part + static_cast<size_t>(lane + 32 * i) * 8, epoch, v)) {
                  vp[i] = static_cast<T>(v);
                  pending &= ~(1u << (2 * i));
                }
              }
              if ((pending >> (2 * i + 1)) & 1u) {
                if (ll_load(part + static_cast<size_t>(lane + 32 * i) * 8 + 4, epoch, v)) {
                  vq[i] = static_cast<T>(v);
                  pending &= ~(2u << (2 * i));
                }
              }
            }
            if (pending && globaltimer() - t0 > kTimeoutNs) { timed_out = true; break; }
          }
#pragma unroll
          for (int h = kPer / 2; h >= 1; h >>= 1)
#pragma unroll
            for (int i = 0; i < h; ++i) {
              vp[i] = Num<T>::add(vp[i], vp[i + h]);
              vq[i] = Num<T>::add(vq[i], vq[i + h]);
            }
          const T sp = warp_sum(vp[0]);
          const T sq = with_q ? warp_sum(vq[0]) : T(0);
          if (ag) {
            if (lane == 0) bcast[buf] = Pair{static_cast<double>(sp), static_cast<double>(sq)};
          } else {
            for (uint32_t r = lane; r < G; r += 32) {
              ll_store(result + static_cast<size_t>(r) * 32, static_cast<double>(sp), epoch);
              if (with_q) ll_store(result + static_cast<size_t>(r) * 32 + 4, static_cast<double>(sq), epoch);
            }
          }
        }
        if (lane == 0 && !ag) {
          double vp2 = 0.0, vq2 = 0.0;
          const uint32_t* mine = result + static_cast<size_t>(rank) * 32;
          const uint64_t t0 = globaltimer();
          while (!ll_load(mine, epoch, vp2))
            if (globaltimer() - t0 > kTimeoutNs) { timed_out = true; break; }
          if (with_q)
            while (!ll_load(mine + 4, epoch, vq2))
              if (globaltimer() - t0 > kTimeoutNs) { timed_out = true; break; }
          bcast[buf] = Pair{vp2, vq2};
        }
        if (timed_out) {
          report_error(prm.status, BAK_ETIMEOUT);
          my_abort = 1;
        }
      }
      const bool any2 = bar_or(NT, my_abort);
      P = static_cast<T>(bcast[buf].p);
      Q = static_cast<T>(bcast[buf].q);
      return any2;
    };

    int64_t sweep = 0;
    bool converged = false;
    if constexpr (XS) {
      constexpr int NQ = xs_nq<E, XS>(), EQ = E / NQ;
      static_assert(E % NQ == 0, "XS: rows per thread must split into sub-column slots");
      const bool full_rows = kv == E;
      const uint32_t xs0 = smem_addr(xs) + static_cast<uint32_t>(tid * sizeof(T));
      const uint32_t slot_bytes = static_cast<uint32_t>(prm.stage_elems * sizeof(T));
      // ring position of a fill as (slot, parity) pairs advanced incrementally
      // (no 64-bit division on the per-quarter critical path)
      struct Pos {
        int sl;
        uint32_t par;
      };
      auto adv = [&](Pos p, int n) -> Pos {  // n <= S
        p.sl += n;
        if (p.sl >= S) {
          p.sl -= S;
          p.par ^= 1u;
        }
        return p;
      };
      auto slot_addr = [&](Pos p) -> uint32_t { return xs0 + static_cast<uint32_t>(p.sl) * slot_bytes; };
      auto wait_fill = [&](Pos p) {
        const int sl = p.sl;
        const uint32_t par = p.par;
#ifdef BAK_PHASES
        const long long w0 = clock64();
#endif
        if (!mbar_test(&full[sl], par)) {
          const uint64_t t0 = globaltimer();
          while (!mbar_test(&full[sl], par)) {
            if (globaltimer() - t0 > kTimeoutNs) {
              report_error(prm.status, BAK_ETIMEOUT);
              my_abort = 1;
              break;
            }
          }
        }
#ifdef BAK_PHASES
        if (tid == 0) ph_acc[9] += clock64() - w0;  // ring waits (reported in the unused "pull" slot)
#endif
      };
      auto release = [&](Pos p) {  // this warp is done reading that fill
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[p.sl]);
      };
      auto meta_of = [&](int64_t u, int64_t& c, T& n2, T& ri) {
        const StageMeta& m = meta[u % kMaxStages];
        c = m.col;
        n2 = static_cast<T>(m.n2);
        ri = static_cast<T>(m.rinv);
      };
      auto xval = [&](uint32_t a, int kk, int k) -> T {
        return (full_rows || k < kv) ? lds<T>(a + static_cast<uint32_t>(kk * NT * sizeof(T))) : T(0);
      };
      if constexpr (XS == 2) {
        // ---- XT: x_{t+1} is read from the ring ONCE (for its dot), stashed in
        // tensor memory, and read back from there for its update one step later;
        // the ring slot goes back to the producer right after that single read,
        // so the whole ring is prefetch (x_{t+2}, x_{t+3}) while the exchange of
        // step t is in flight.  Per row the same two roundings and FMA order as
        // the XS / register kernels.
        constexpr int CS = xt_cs<E>(), CH = kXtChunk, NC = E / CH;  // chunks per slot, rows per chunk, chunks
        static_assert(EQ == CH * CS, "XT: a ring slot holds CS TMEM chunks");
        constexpr int CW = CH * static_cast<int>(sizeof(T)) / 4;  // 32-bit TMEM columns per chunk
        // warp w owns TMEM lanes 32 (w % 4) ..; warps 4.. use the next column range
        const uint32_t tb = tmem_base + (static_cast<uint32_t>((warp & 3) * 32) << 16) +
                            static_cast<uint32_t>((warp >> 2) * (E * static_cast<int>(sizeof(T)) / 4));
        uint32_t rc = 0;
        T P = T(0), Q = T(0);
        int64_t c0 = 0, c1 = 0;
        T n2_0 = T(1), ri_0 = T(1), n2_1 = T(1), ri_1 = T(1);
        T acc[4] = {T(0), T(0), T(0), T(0)};
        Pos pn{0, 0u};  // first slot of the column whose dot is being formed
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          const Pos pq = adv(pn, q);
          wait_fill(pq);
          const uint32_t a = slot_addr(pq);
#pragma unroll
          for (int c = 0; c < CS; ++c) {
            const int ch = q * CS + c;
            TmemRegs<T, CH> xn;
#pragma unroll
            for (int kk = 0; kk < CH; ++kk) xn.set(kk, xval(a, c * CH + kk, ch * CH + kk));
            if (c == CS - 1) release(pq);
#pragma unroll
            for (int kk = 0; kk < CH; ++kk) {
              const int k = ch * CH + kk;
              acc[k & 3] = Num<T>::fma(xn.get(kk), ev[k], acc[k & 3]);
            }
            xn.store(tb + ch * CW);
          }
        }
        meta_of(0, c0, n2_0, ri_0);
        T pv = Num<T>::add(Num<T>::add(acc[0], acc[1]), Num<T>::add(acc[2], acc[3]));
        bool aborted = reduce(pv, T(0), false, rc++, -1, -1, P, Q);
        const bool upd_warp = (rank == 0) && (warp == (nwarps > 1 ? 1 : 0));
        T a0 = upd_warp ? ag[c0] : T(0);
        int64_t k = 0, t = 0;
        pn = adv(pn, NQ);
        while (!aborted) {
          PH(7);
          const bool more = t + 1 < total;
          const T d = quotient(P, n2_0, ri_0);
          const bool last = (k == ncols - 1);
          T ac[4] = {T(0), T(0), T(0), T(0)};
          T a1 = T(0);
          tmem_wait_st();  // the stash writes of the previous step (they overlapped its exchange)
          TmemRegs<T, CH> xt[2];
          xt[0].load(tb);
          if (more) {
            wait_fill(pn);
            meta_of(t + 1, c1, n2_1, ri_1);
            if (upd_warp) a1 = ag[c1];
          }
          PH(0);
#pragma unroll
          for (int ch = 0; ch < NC; ++ch) {
            const int q = ch / CS, c = ch % CS;
            const Pos fn = adv(pn, q);
            TmemRegs<T, CH> xn;
            if (more) {
              if (c == 0 && q > 0) wait_fill(fn);
              const uint32_t a_n = slot_addr(fn);
#pragma unroll
              for (int kk = 0; kk < CH; ++kk) xn.set(kk, xval(a_n, c * CH + kk, ch * CH + kk));
              if (c == CS - 1) release(fn);
            }
            xt[ch & 1].wait();
            if (ch + 1 < NC) xt[(ch + 1) & 1].load(tb + (ch + 1) * CW);
#pragma unroll
            for (int kk = 0; kk < CH; ++kk) {
              const int kq = ch * CH + kk;
              ev[kq] = Num<T>::sub(ev[kq], Num<T>::mul(xt[ch & 1].get(kk), d));
            }
            if (more) {
#pragma unroll
              for (int kk = 0; kk < CH; ++kk) {
                const int kq = ch * CH + kk;
                ac[kq & 3] = Num<T>::fma(xn.get(kk), ev[kq], ac[kq & 3]);
              }
              xn.store(tb + ch * CW);
            }
          }
          PH(1);
          pv = Num<T>::add(Num<T>::add(ac[0], ac[1]), Num<T>::add(ac[2], ac[3]));
          T qv = T(0);
          if (last) {
            T qa[4] = {T(0), T(0), T(0), T(0)};
#pragma unroll
            for (int kk = 0; kk < E; ++kk) qa[kk & 3] = Num<T>::fma(ev[kk], ev[kk], qa[kk & 3]);
            qv = Num<T>::add(Num<T>::add(qa[0], qa[1]), Num<T>::add(qa[2], qa[3]));
          }
          PH(2);
          if (upd_warp) {
            const T na = Num<T>::add(a0, d);
            ag[c0] = na;
            if (more) a0 = (c1 == c0) ? na : a1;  // a1 = ag[c1] was read before the store
          }
          PH(5);
          if (reduce(pv, qv, last, rc++, -1, -1, P, Q)) break;
          PH(6);
          if (last) {
            if (rank == 0 && tid == 0 && prm.history) prm.history[sweep] = static_cast<double>(Q);
            ++sweep;
            if (prm.thresh2 >= 0.0 && static_cast<double>(Q) <= prm.thresh2) {
              converged = true;
              break;
            }
            if (sweep == prm.max_iter) break;
            k = 0;
          } else {
            ++k;
          }
          ++t;
          pn = adv(pn, NQ);
          c0 = c1;
          n2_0 = n2_1;
          ri_0 = ri_1;
        }
        tmem_wait_st();
      } else {
      // ---- prologue: the dot for column 0 ----
      uint32_t rc = 0;
      T P = T(0), Q = T(0);
      int64_t c0 = 0, c1 = 0;
      T n2_0 = T(1), ri_0 = T(1), n2_1 = T(1), ri_1 = T(1);
      T acc[4] = {T(0), T(0), T(0), T(0)};
      Pos pc{0, 0u};  // fill (t, 0)
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        const Pos pq = adv(pc, q);
        wait_fill(pq);
        const uint32_t a = slot_addr(pq);
#pragma unroll
        for (int kk = 0; kk < EQ; ++kk) {
          const int k = q * EQ + kk;
          acc[k & 3] = Num<T>::fma(xval(a, kk, k), ev[k], acc[k & 3]);
        }
      }
      meta_of(0, c0, n2_0, ri_0);
      T pv = Num<T>::add(Num<T>::add(acc[0], acc[1]), Num<T>::add(acc[2], acc[3]));
      bool aborted = reduce(pv, T(0), false, rc++, -1, -1, P, Q);
      const bool upd_warp = (rank == 0) && (warp == (nwarps > 1 ? 1 : 0));
      T a0 = upd_warp ? ag[c0] : T(0);
      int64_t k = 0, t = 0;
      while (!aborted) {
        PH(7);
        const bool more = t + 1 < total;
        const T d = quotient(P, n2_0, ri_0);
        const bool last = (k == ncols - 1);
        T ac[4] = {T(0), T(0), T(0), T(0)};
        T a1 = T(0);
        const Pos pn = adv(pc, NQ);  // fill (t + 1, 0)
        if (more) {
          wait_fill(pn);
          meta_of(t + 1, c1, n2_1, ri_1);
          if (upd_warp) a1 = ag[c1];  // its latency overlaps the update loop below
        }
        PH(0);
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          const Pos fc = adv(pc, q), fn = adv(pn, q);
          if (more && q > 0) wait_fill(fn);
          const uint32_t a_c = slot_addr(fc), a_n = slot_addr(fn);
          // update with this quarter of x_t, hand the slot back, then the dot with
          // the same quarter of x_{t+1} (per row the same two roundings and the
          // same FMA order as the fused loop of the register-resident kernel)
#pragma unroll
          for (int kk = 0; kk < EQ; ++kk) {
            const int kq = q * EQ + kk;
            ev[kq] = Num<T>::sub(ev[kq], Num<T>::mul(xval(a_c, kk, kq), d));
          }
          release(fc);
          if (more) {
#pragma unroll
            for (int kk = 0; kk < EQ; ++kk) {
              const int kq = q * EQ + kk;
              ac[kq & 3] = Num<T>::fma(xval(a_n, kk, kq), ev[kq], ac[kq & 3]);
            }
          }
        }
        PH(1);
        pv = Num<T>::add(Num<T>::add(ac[0], ac[1]), Num<T>::add(ac[2], ac[3]));
        T qv = T(0);
        if (last) {
          T qa[4] = {T(0), T(0), T(0), T(0)};
#pragma unroll
          for (int kk = 0; kk < E; ++kk) qa[kk & 3] = Num<T>::fma(ev[kk], ev[kk], qa[kk & 3]);
          qv = Num<T>::add(Num<T>::add(qa[0], qa[1]), Num<T>::add(qa[2], qa[3]));
        }
        PH(2);
        if (upd_warp) {
          const T na = Num<T>::add(a0, d);
          ag[c0] = na;
          if (more) a0 = (c1 == c0) ? na : a1;  // a1 = ag[c1] was read before the store
        }
        PH(5);
        if (reduce(pv, qv, last, rc++, -1, -1, P, Q)) break;
        PH(6);
        if (last) {
          if (rank == 0 && tid == 0 && prm.history) prm.history[sweep] = static_cast<double>(Q);
          ++sweep;
          if (prm.thresh2 >= 0.0 && static_cast<double>(Q) <= prm.thresh2) {
            converged = true;
            break;
          }
          if (sweep == prm.max_iter) break;
          k = 0;
        } else {
          ++k;
        }
        ++t;
        pc = pn;
        c0 = c1;
        n2_0 = n2_1;
        ri_0 = ri_1;
      }
      }
    } else {
    // ---- prologue: columns 0 and 1 into registers, dot for column 0 ----
    uint32_t rc = 0;
    T P = T(0), Q = T(0);
    int64_t c0 = 0, c1 = 0;
    T n2_0 = T(1), n2_1 = T(1), ri_0 = T(1), ri_1 = T(1);
    const int s0 = pull(xc, c0, n2_0, ri_0);
    const int s1 = (total > 1) ? pull(xn, c1, n2_1, ri_1) : -1;
    T pv;
    {
      T acc[4] = {T(0), T(0), T(0), T(0)};
#pragma unroll
      for (int k = 0; k < E; ++k) acc[k & 3] = Num<T>::fma(xc[k], ev[k], acc[k & 3]);
      pv = Num<T>::add(Num<T>::add(acc[0], acc[1]), Num<T>::add(acc[2], acc[3]));
    }
    bool aborted = reduce(pv, T(0), false, rc++, s0, s1, P, Q);

    // coefficient updates: the whole of warp 1 (warp 0 when NT == 32) runs them
    // in lockstep (identical values, same address) so no lane diverges
    const bool upd_warp = (rank == 0) && (warp == (nwarps > 1 ? 1 : 0));
    T a0 = upd_warp ? ag[c0] : T(0);
    T a1 = (upd_warp && total > 1) ? ag[c1] : T(0);

    int64_t k = 0, t = 0;
    // one column step: update with xc (column t), dot with xn (column t+1), then
    // refill xc with column t+2 (its LDS latency overlaps the reduction).
    // Returns true when the solve ends.  Called with the two buffers swapped on
    // alternate steps, so no register copies.
    auto step = [&](T (&xc)[E], T (&xn)[E]) -> bool {
      PH(7);
      const bool more = t + 2 < total;
      const T d = quotient(P, n2_0, ri_0);
      PH(0);
      const bool last = (k == ncols - 1);
      T acc[4] = {T(0), T(0), T(0), T(0)};
#pragma unroll
      for (int kk = 0; kk < E; ++kk) {
        ev[kk] = Num<T>::sub(ev[kk], Num<T>::mul(xc[kk], d));
        acc[kk & 3] = Num<T>::fma(xn[kk], ev[kk], acc[kk & 3]);
      }
      pv = Num<T>::add(Num<T>::add(acc[0], acc[1]), Num<T>::add(acc[2], acc[3]));
      T qv = T(0);
      if (last) {
        T qa[4] = {T(0), T(0), T(0), T(0)};
#pragma unroll
        for (int kk = 0; kk < E; ++kk) qa[kk & 3] = Num<T>::fma(ev[kk], ev[kk], qa[kk & 3]);
        qv = Num<T>::add(Num<T>::add(qa[0], qa[1]), Num<T>::add(qa[2], qa[3]));
      }
      PH(1);
      int64_t c2 = c1;
      T n2_2 = n2_1, ri_2 = ri_1;
      const int sp = more ? pull(xc, c2, n2_2, ri_2) : -1;
      PH(2);
      if (upd_warp) {
        const T na = Num<T>::add(a0, d);
        ag[c0] = na;
        a0 = (c1 == c0) ? na : a1;
        if (more) a1 = ag[c2];  // store->load order in one thread: never stale
      }
      if (reduce(pv, qv, last, rc++, sp, -1, P, Q)) return true;
      PH(6);
      if (last) {
        if (rank == 0 && tid == 0 && prm.history) prm.history[sweep] = static_cast<double>(Q);
        ++sweep;
        if (prm.thresh2 >= 0.0 && static_cast<double>(Q) <= prm.thresh2) {
          converged = true;
          return true;
        }
        if (sweep == prm.max_iter) return true;
        k = 0;
      } else {
        ++k;
      }
      ++t;
      c0 = c1;
      n2_0 = n2_1;
      ri_0 = ri_1;
      c1 = c2;
      n2_1 = n2_2;
      ri_1 = ri_2;
      return false;
    };
    if (!aborted) {
      while (true) {
        if (step(xc, xn)) break;
        if (step(xn, xc)) break;
      }
    }
    }

    {
      // the row addresses are recomputed here from a laundered base: otherwise
      // the compiler keeps the E 64-bit addresses of the initial load of e live
      // across the whole solve (2E registers; E = 32 fp64 spilled)
      T* ew = eg + r0 + tid;
      asm volatile("mov.b64 %0, %0;" : "+l"(ew));
#pragma unroll
      for (int kk = 0; kk < E; ++kk)
        if (kk < kv) ew[static_cast<int64_t>(kk) * NT] = ev[kk];
    }
#ifdef BAK_PHASES
    if (tid == 0 && rank == 0 && prm.history)
      for (int i = 0; i < 8; ++i)
        prm.history[prm.max_iter + i] = static_cast<double>((XS && i == 2) ? ph_acc[9] : ph_acc[i]);
#endif
    if (tid == 0) {
      *stop = 1;
      if (rank == 0 && prm.status) {
        prm.status[0] = sweep;
        prm.status[1] = converged ? 1 : 0;
        prm.status[3] =
            MODE == kModeCta ? BAK_VARIANT_CTA : (MODE == kModeCluster ? BAK_VARIANT_CLUSTER : BAK_VARIANT_GRID);
      }
    }
  }
  if (XS == 2) tmem_fence_before_sync();
  __syncthreads();
  if (XS == 2 && warp == 0) tmem_dealloc512(tmem_base);
  if (MODE == kModeCluster || MODE == kModeGridCl) cluster_sync();
}

// ------------------------------- host -------------------------------------

size_t smem_bytes(const SweepPlan& pl, size_t tsize) {
  return static_cast<size_t>(pl.nstages) * pl.stage_elems * tsize + 2 * kMaxStages * 8 +
         kMaxStages * sizeof(StageMeta) + 2 * 2 * 32 * tsize + 16 + 2 * kMaxCluster * 16 + 16 + 32 + 16 + 16;
}

template <typename T, int E, int MODE, int MAXNT, int XS = 0>
int launch_one(const SweepPlan& pl, SweepParams prm, cudaStream_t st) {
  auto kern = sweep_kernel<T, E, MODE, MAXNT, XS>;
  const size_t smem = smem_bytes(pl, sizeof(T));
  BAK_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(pl.nparticipants);
  cfg.blockDim = dim3(pl.nthreads + 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (MODE == kModeCluster) {
    if (pl.nparticipants > 8)
      BAK_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = pl.nparticipants;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  } else if (MODE == kModeGrid) {
    attr[na].id = cudaLaunchAttributeCooperative;
    attr[na].val.cooperative = 1;
    ++na;
  } else if (MODE == kModeGridCl) {
    attr[na].id = cudaLaunchAttributeCooperative;
    attr[na].val.cooperative = 1;
    ++na;
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = kGridCluster;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  if (MODE == kModeGridCl) {
    // every cluster must be co-resident (spin waits across clusters)
    int ncl = 0;
    BAK_CHECK_CUDA(cudaOccupancyMaxActiveClusters(&ncl, kern, &cfg));
    if (ncl < pl.nparticipants / kGridCluster) {
      set_error("bak_sweep(GRID): %d clusters of %d do not fit co-resident (max %d)", pl.nparticipants / kGridCluster,
                kGridCluster, ncl);
      return BAK_EUNSUPPORTED;
    }
  }
  BAK_CHECK_CUDA(cudaLaunchKernelEx(&cfg, kern, prm));
  count_launches(1);
  return BAK_OK;
}

template <typename T, int MODE, int MAXNT>
int launch_e(const SweepPlan& pl, const SweepParams& prm, cudaStream_t st) {
  switch (pl.e) {
    case 1: return launch_one<T, 1, MODE, MAXNT>(pl, prm, st);
    case 2: return launch_one<T, 2, MODE, MAXNT>(pl, prm, st);
    case 4: return launch_one<T, 4, MODE, MAXNT>(pl, prm, st);
    case 8: return launch_one<T, 8, MODE, MAXNT>(pl, prm, st);
    case 16: return launch_one<T, 16, MODE, MAXNT>(pl, prm, st);
    case 32: return launch_one<T, 32, MODE, MAXNT>(pl, prm, st);
  }
  set_error("bak_sweep: unsupported rows-per-thread %d", pl.e);
  return BAK_EUNSUPPORTED;
}

// XS plans: 7 consumer warps + the producer = 8 warps, two per SM sub-partition,
// so a thread may hold up to 255 registers (9 warps cap it at 168: e spilled)
constexpr int kXsConsumers = 224;

template <typename T, int MODE>
int launch_xs(const SweepPlan& pl, const SweepParams& prm, cudaStream_t st) {
  if constexpr (MODE == kModeGrid || MODE == kModeGridCl) {
    if (pl.xs == 2) {
      switch (pl.e) {
        case 40: return launch_one<T, 40, MODE, kXsConsumers, 2>(pl, prm, st);
        case 56: return launch_one<T, 56, MODE, kXsConsumers, 2>(pl, prm, st);
        case 80: return launch_one<T, 80, MODE, kXsConsumers, 2>(pl, prm, st);
      }
    } else {
      switch (pl.e) {
        case 40: return launch_one<T, 40, MODE, kXsConsumers, 1>(pl, prm, st);
        case 56: return launch_one<T, 56, MODE, kXsConsumers, 1>(pl, prm, st);
        case 80: return launch_one<T, 80, MODE, kXsConsumers, 1>(pl, prm, st);
      }
    }
  }
  set_error("bak_sweep: unsupported XS plan (rows per thread %d)", pl.e);
  return BAK_EUNSUPPORTED;
}

template <typename T, int MODE>
int launch_nt(const SweepPlan& pl, const SweepParams& prm, cudaStream_t st) {
  if (pl.xs) return launch_xs<T, MODE>(pl, prm, st);
  if (pl.nthreads == 32) return launch_e<T, MODE, 32>(pl, prm, st);
  if (pl.nthreads <= 128) return launch_e<T, MODE, 128>(pl, prm, st);
  return launch_e<T, MODE, kMaxConsumers>(pl, prm, st);
}

// How many clusters of kGridCluster CTAs of the sweep kernel (one CTA per SM:
// its ring fills the shared memory) can be co-resident — GPC boundaries make
// it less than SMs / kGridCluster (B200: 15 clusters of 8 = 120 CTAs).
int grid_cluster_capacity() {
  static int cap = -1;
  if (cap >= 0) return cap;
  auto kern = sweep_kernel<double, 8, kModeGridCl, kMaxConsumers>;
  const int smem = device_max_smem_optin() - 2048;
  cap = 0;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess) {
    cudaGetLastError();
    return cap;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(kGridCluster * 8);
  cfg.blockDim = dim3(kMaxConsumers + 32);
  cfg.dynamicSmemBytes = static_cast<size_t>(smem);
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = kGridCluster;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) == cudaSuccess) cap = n;
  else cudaGetLastError();
  return cap;
}

}  // namespace

// ---- planning: pick participants, threads, rows per thread, stages ----
static const int kEs[] = {1, 2, 4, 8, 16, 32};

static bool plan_fill(int dtype, int variant, int64_t obs, int nthreads, int e, int parts, SweepPlan& pl,
                      int min_stages) {
  const size_t ts = dtype_size(dtype);
  const size_t smem_cap = static_cast<size_t>(device_max_smem_optin()) - 2048;
  const int64_t rows = static_cast<int64_t>(nthreads) * e;
  if (nthreads < 32 || nthreads > kMaxConsumers || nthreads % 32) return false;
  if (rows * parts < obs || (parts - 1) * rows >= obs) return false;
  if (variant == BAK_VARIANT_GRID && parts > kGridSlotsMax) return false;
  SweepPlan cand;
  cand.variant = variant;
  cand.nthreads = nthreads;
  cand.e = e;
  cand.nparticipants = parts;
  cand.rows_per_cta = rows;
  cand.stage_elems = rows;
  cand.nstages = 0;
  const size_t fixed = smem_bytes(cand, ts);
  const size_t stage_bytes = rows * ts;
  if (fixed + 2 * stage_bytes > smem_cap) return false;
  int s = static_cast<int>((smem_cap - fixed) / stage_bytes);
  if (s > kMaxRegStages) s = kMaxRegStages;
  if (s < min_stages) return false;
  cand.nstages = s;
  pl = cand;
  return true;
}

// XS plan (GRID, x read from a sub-column ring; e in registers): all `parts`
// CTAs, rows spread evenly, E in {40, 56, 80} rows per thread of 224
// consumers, quarter-column slots (xs_nq); at least nq + 2 slots (the nq + 1
// a step reads + 1 in flight).
static bool plan_xs(int dtype, int64_t obs, int parts, int cluster, SweepPlan& pl) {
  if (parts < 2) return false;
  const size_t ts = dtype_size(dtype);
  const size_t smem_cap = static_cast<size_t>(device_max_smem_optin()) - 2048;
  const int64_t rpc = round_up((obs + parts - 1) / parts, 4);
  if ((parts - 1) * rpc >= obs) return false;
  for (int e : {40, 56, 80}) {
    if (static_cast<int64_t>(kXsConsumers) * e < rpc) continue;
    SweepPlan cand;
    cand.variant = BAK_VARIANT_GRID;
    cand.nthreads = kXsConsumers;
    cand.e = e;
    cand.nparticipants = parts;
    cand.rows_per_cta = rpc;
    // XT (default): slots of kXtChunk rows per thread, the column stashed in
    // tensor memory between its two uses; BAK_GRID_XT=0: quarter-column XS ring
    const char* xt_env = getenv("BAK_GRID_XT");
    const int mode = (xt_env && xt_env[0] == '0') ? 1 : 2;
    const int cs = (BAK_XT_SLOT_CHUNKS == 2 && e % (2 * kXtChunk) == 0) ? 2 : 1;  // xt_cs<E>()
    const int nq = mode == 2 ? e / (kXtChunk * cs) : 4;                            // xs_nq<E, XS>()
    cand.stage_elems = static_cast<int64_t>(e / nq) * kXsConsumers;
    cand.cluster = cluster;
    cand.xs = mode;
    cand.nstages = 0;
    const size_t fixed = smem_bytes(cand, ts);
    const size_t slot = static_cast<size_t>(cand.stage_elems) * ts;
    int st = static_cast<int>((smem_cap - fixed) / slot);
    if (st > kMaxStages) st = kMaxStages;
    if (st < nq + 2) return false;  // XS: the nq + 1 slots a step reads + 1 in flight; XT: a column + 2
    cand.nstages = st;
    pl = cand;
    return true;
  }
  return false;
}

// BAK_PLAN="parts,e,nthreads" overrides the heuristic (tuning experiments)
static bool plan_env(int dtype, int variant, int64_t obs, SweepPlan& pl) {
  const char* env = getenv("BAK_PLAN");
  if (!env) return false;
  int parts = 0, e = 0, nt = 0;
  if (sscanf(env, "%d,%d,%d", &parts, &e, &nt) != 3) return false;
  return plan_fill(dtype, variant, obs, nt, e, parts, pl, 2);
}

bool plan_onchip(int dtype, int variant, int64_t obs, SweepPlan& pl, bool force_flat) {
  const int sms = device_sms();
  if (plan_env(dtype, variant, obs, pl)) return true;
  // Measured on B200 (tools/tune2.sh): E = 8 rows per thread and as few warps
  // per CTA as possible; grow the cluster (single-warp CTAs) before warps.
  const int e0 = 8;
  if (variant == BAK_VARIANT_CTA) {
    for (int e : {e0, 16, 32, 4, 2, 1}) {
      const int nt = static_cast<int>(round_up((obs + e - 1) / e, 32));
      if (nt <= 256 && plan_fill(dtype, variant, obs, nt, e, 1, pl, 4)) return true;
    }
    return false;
  }
  if (variant == BAK_VARIANT_CLUSTER) {
    // Measured on B200 (tools/sweep_probe.py plan scans, C1 10,000 rows and C2
    // 4,096 rows): E = 8 rows per thread always wins (E = 4 / 16 lose 10-50 %),
    // and at E = 8 the widest cluster (16 CTAs, rows spread evenly) is best:
    // C1 14 x 96 threads 0.79 µs/col (vs 1.17 for 10 x 64 x E16), C2 16 x 32
    // threads 0.62 µs/col.  Wider E only when 16 x 256 x 8 rows do not suffice.
    const int64_t per = (obs + kMaxCluster - 1) / kMaxCluster;
    for (int e : {e0, 16, 32}) {
      const int nt = static_cast<int>(round_up((per + e - 1) / e, 32));
      if (nt > kMaxConsumers) continue;
      const int parts = static_cast<int>((obs + static_cast<int64_t>(nt) * e - 1) / (static_cast<int64_t>(nt) * e));
      if (parts >= 2 && plan_fill(dtype, variant, obs, nt, e, parts, pl, 4)) return true;
    }
    return false;
  }
  if (variant == BAK_VARIANT_GRID) {
    // two-level exchange: clusters of kGridCluster CTAs reduce through DSMEM,
    // cluster leaders through global records (<= 32 clusters); rows spread
    // evenly over a multiple of kGridCluster CTAs.  BAK_GRID_FLAT=1: one level.
    const char* flat = getenv("BAK_GRID_FLAT");
    const int max_parts = kGridCluster * (grid_cluster_capacity() < 32 ? grid_cluster_capacity() : 32);
    const char* xs_env = getenv("BAK_GRID_XS");  // tuning aid: "1" = XS plans first
    if (xs_env && xs_env[0] == '1' && !force_flat && !(flat && flat[0] == '1') && coop_clusters_ok() &&
        plan_xs(dtype, obs, static_cast<int>(imin64(sms, max_parts)) / kGridCluster * kGridCluster, kGridCluster, pl))
      return true;
    // fp64 register plans past E = 16 spill (3E doubles per thread); the XS plan
    // (e in registers, x from the shared ring) is faster there (tools/grid_compare.py)
    const int max_reg_e = dtype == BAK_F64 ? 16 : 32;
    if (!force_flat && !(flat && flat[0] == '1') && coop_clusters_ok()) {
      for (int e : kEs) {
        if (e > max_reg_e) break;
        const int64_t rows = 256LL * e;
        const int64_t parts = round_up((obs + rows - 1) / rows, kGridCluster);
        if (parts > sms || parts > max_parts) continue;
        const int64_t rpc = round_up((obs + parts - 1) / parts, 4);
        if ((parts - 1) * rpc >= obs) continue;
        SweepPlan cand;
        if (!plan_fill(dtype, variant, obs, 256, e, static_cast<int>((obs + rows - 1) / rows), cand, 3)) continue;
        cand.nparticipants = static_cast<int>(parts);
        cand.rows_per_cta = rpc;
        cand.stage_elems = rpc;
        cand.cluster = kGridCluster;
        pl = cand;
        return true;
      }
    }
    const bool two_level = !force_flat && !(flat && flat[0] == '1') && coop_clusters_ok();
    if (two_level && plan_xs(dtype, obs, static_cast<int>(imin64(sms, max_parts)) / kGridCluster * kGridCluster,
                             kGridCluster, pl))
      return true;
    for (int nt : {256}) {
      for (int e : kEs) {
        if (e > max_reg_e && two_level) break;  // the two-level XS plan did not fit either
        const int64_t rows = static_cast<int64_t>(nt) * e;
        const int64_t parts = (obs + rows - 1) / rows;
        if (parts <= sms && plan_fill(dtype, variant, obs, nt, e, static_cast<int>(parts), pl, 3)) return true;
      }
    }
    return plan_xs(dtype, obs, static_cast<int>(imin64(sms, kGridSlotsMax)), 0, pl);
  }
  return false;
}

// one-level GRID exchange: every CTA gathers all records (default; measured
// 3.46 vs 3.64 us/column at 2^18 rows, 7.48 vs 7.88 at 2^21); BAK_GRID_AG=0
// restores the aggregator + result lines
static int grid_allgather_on() {
  const char* a = getenv("BAK_GRID_AG");
  return (a && a[0] == '0') ? 0 : 1;
}

int launch_onchip(int dtype, const SweepPlan& pl, const SweepParams& prm0, cudaStream_t st) {
  SweepParams prm = prm0;
  prm.grid_allgather = grid_allgather_on();
  if (pl.variant == BAK_VARIANT_GRID && prm.slots)
    BAK_CHECK_CUDA(cudaMemsetAsync(prm.slots, 0, kGridSlotBytes, st));
  if (pl.variant == BAK_VARIANT_GRID && pl.cluster) {
    const int rc = dtype == BAK_F64 ? launch_nt<double, kModeGridCl>(pl, prm, st)
                                    : launch_nt<float, kModeGridCl>(pl, prm, st);
    if (rc == BAK_OK) return rc;  // else (capacity / cooperative launch refused): one level
    if (prm.nranks > 0) return rc;  // row sharding needs the two-level exchange (the caller falls back to STREAM)
    // clusters did not fit co-resident: one-level grid exchange
    if (getenv("BAK_DEBUG")) fprintf(stderr, "bak: two-level grid exchange unavailable (%s)\n", bak_last_error());
    SweepPlan flat;
    const bool ok = plan_onchip(dtype, BAK_VARIANT_GRID, prm.obs, flat, /*force_flat=*/true);
    if (!ok) return rc;
    g_err_clear();
    SweepParams p2 = prm;
    p2.rows_per_cta = flat.rows_per_cta;
    p2.stage_elems = flat.stage_elems;
    p2.nstages = flat.nstages;
    return dtype == BAK_F64 ? launch_nt<double, kModeGrid>(flat, p2, st) : launch_nt<float, kModeGrid>(flat, p2, st);
  }
  if (dtype == BAK_F64) {
    if (pl.variant == BAK_VARIANT_CTA) return launch_nt<double, kModeCta>(pl, prm, st);
    if (pl.variant == BAK_VARIANT_CLUSTER) return launch_nt<double, kModeCluster>(pl, prm, st);
    return launch_nt<double, kModeGrid>(pl, prm, st);
  }
  if (pl.variant == BAK_VARIANT_CTA) return launch_nt<float, kModeCta>(pl, prm, st);
  if (pl.variant == BAK_VARIANT_CLUSTER) return launch_nt<float, kModeCluster>(pl, prm, st);
  return launch_nt<float, kModeGrid>(pl, prm, st);
}

}  // namespace bak

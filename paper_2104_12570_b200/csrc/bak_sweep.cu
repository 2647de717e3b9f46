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
// shared-memory reads are conflict-free).  The CTA's slice of each column x_j
// is contiguous in column-major x, so one cp.async.bulk (TMA engine) moves it
// into an S-stage shared-memory ring, S columns ahead (x never depends on e).
// Per column there is exactly one reduction:
//     fused pass:  e -= d_j * x_j  ;  p += x_{j+1} . e   (+ sum e^2 at sweep end)
//     warp xor-butterfly -> per-warp slots -> __syncthreads -> fixed-order sum
//     -> exchange across participants -> every thread holds P and d_{j+1}.
// Exchange by MODE:
//   kCta     : single CTA, nothing to exchange.
//   kCluster : thread-block cluster (2..16 CTAs).  Each CTA st.async's its
//              16-byte {p, sq} into every peer's shared slot, completing as
//              transaction bytes on the peer's mbarrier (DSMEM, no flags).
//   kGrid    : co-resident persistent grid (cooperative launch).  Each CTA
//              posts {p, epoch}-tagged 16-byte records to global slots; warp 0
//              of every CTA polls all slots and sums them in fixed order.
// Every participant sums the same values in the same order, so all of them
// compute bit-identical d_j; the reduction order depends only on the shape.
#include <cstdio>

#include "bak_common.cuh"
#include "bak_sweep.cuh"

namespace bak {
namespace {

constexpr int kModeCta = 0, kModeCluster = 1, kModeGrid = 2;
constexpr int kMaxCluster = 16;
constexpr int kMaxStages = 16;

struct ColCursor {
  const int32_t* cols;
  int64_t ncols, stride, s, k;
  __device__ __forceinline__ int64_t col() const { return cols ? static_cast<int64_t>(cols[s * stride + k]) : k; }
  __device__ __forceinline__ void next() {
    if (++k == ncols) { k = 0; ++s; }
  }
};

template <typename T>
struct alignas(16) Pair {
  double p, q;
};

template <typename T, int E, int MODE>
__global__ void __launch_bounds__(512, 1) sweep_kernel(const SweepParams prm) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int NT = blockDim.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = NT >> 5;
  const int S = prm.nstages;

  uint32_t rank = 0, G = 1;
  if (MODE == kModeCluster) {
    rank = cluster_rank();
    G = cluster_size();
  } else if (MODE == kModeGrid) {
    rank = blockIdx.x;
    G = gridDim.x;
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
  off += kMaxStages * sizeof(uint64_t);
  T* red = reinterpret_cast<T*>(smem_raw + off);  // [2 bufs][2 values][32 warps]
  off += 2 * 2 * 32 * sizeof(T);
  off = (off + 15) & ~size_t(15);
  Pair<T>* xslot = reinterpret_cast<Pair<T>*>(smem_raw + off);  // [2][kMaxCluster]
  off += 2 * kMaxCluster * sizeof(Pair<T>);
  uint64_t* xbar = reinterpret_cast<uint64_t*>(smem_raw + off);  // [2]
  off += 2 * sizeof(uint64_t);
  Pair<T>* bcast = reinterpret_cast<Pair<T>*>(smem_raw + off);  // [2]
  off += 2 * sizeof(Pair<T>);

  if (tid == 0) {
    for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
    mbar_init(&xbar[0], 1);
    mbar_init(&xbar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (MODE == kModeCluster) cluster_sync();

  // ---- residual slice into registers ----
  const int kv = static_cast<int>(imax64(0, imin64(E, (nrows - tid + NT - 1) / NT)));
  T ev[E];
#pragma unroll
  for (int k = 0; k < E; ++k) ev[k] = (k < kv) ? eg[r0 + tid + static_cast<int64_t>(k) * NT] : T(0);

  const int64_t ncols = prm.ncols;
  const int64_t total = prm.max_iter * ncols;
  const uint64_t pol = policy_evict_first();

  // producer (tid 0): TMA the CTA's slice of column(t) into stage t % S
  ColCursor pc{prm.cols, ncols, prm.cols_stride, 0, 0};
  int64_t issued = 0;
  int64_t pcol = 0;
  if (tid == 0) {
    pcol = pc.col();
    const int64_t first = imin64(total, S);
    for (; issued < first; ++issued) {
      const int s = static_cast<int>(issued % S);
      mbar_arrive_expect_tx(&full[s], bytes);
      bulk_g2s(xs + static_cast<size_t>(s) * prm.stage_elems, x + pcol * prm.ldx + r0, bytes, &full[s], pol);
      pc.next();
      if (issued + 1 < total) pcol = pc.col();
    }
  }

  int my_abort = 0;  // thread-local; made uniform by __syncthreads_or
  auto wait_stage = [&](int64_t t) {
    const int s = static_cast<int>(t % S);
    const uint32_t par = static_cast<uint32_t>((t / S) & 1);
    if (!mbar_test(&full[s], par)) {
      const uint64_t t0 = globaltimer();
      while (!mbar_test(&full[s], par)) {
        if (globaltimer() - t0 > kTimeoutNs) {
          report_error(prm.status, BAK_ETIMEOUT);
          my_abort = 1;
          break;
        }
      }
    }
  };

  // one reduction across all participants; returns (P, Q) in every thread
  auto reduce = [&](T pv, T qv, bool with_q, uint32_t rc, bool refill, T& P, T& Q) -> bool {
    const int buf = rc & 1;
    pv = warp_sum(pv);
    if (with_q) qv = warp_sum(qv);
    if (lane == 0) {
      red[(buf * 2 + 0) * 32 + warp] = pv;
      red[(buf * 2 + 1) * 32 + warp] = qv;
    }
    const bool any_abort = __syncthreads_or(my_abort) != 0;
    if (any_abort) return true;
    // every thread has finished reading the stage consumed by this step
    T bp = T(0), bq = T(0);
    for (int w = 0; w < nwarps; ++w) bp = Num<T>::add(bp, red[(buf * 2 + 0) * 32 + w]);
    if (with_q)
      for (int w = 0; w < nwarps; ++w) bq = Num<T>::add(bq, red[(buf * 2 + 1) * 32 + w]);

    if (MODE == kModeCta) {
      if (refill && tid == 0 && issued < total) {
        const int s = static_cast<int>(issued % S);
        mbar_arrive_expect_tx(&full[s], bytes);
        bulk_g2s(xs + static_cast<size_t>(s) * prm.stage_elems, x + pcol * prm.ldx + r0, bytes, &full[s], pol);
        pc.next();
        ++issued;
        if (issued < total) pcol = pc.col();
      }
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
      if (refill && tid == 0 && issued < total) {
        const int s = static_cast<int>(issued % S);
        mbar_arrive_expect_tx(&full[s], bytes);
        bulk_g2s(xs + static_cast<size_t>(s) * prm.stage_elems, x + pcol * prm.ldx + r0, bytes, &full[s], pol);
        pc.next();
        ++issued;
        if (issued < total) pcol = pc.col();
      }
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
      T sp = T(0), sq = T(0);
      for (uint32_t r = 0; r < G; ++r) {
        sp = Num<T>::add(sp, static_cast<T>(xslot[buf * kMaxCluster + r].p));
        if (with_q) sq = Num<T>::add(sq, static_cast<T>(xslot[buf * kMaxCluster + r].q));
      }
      P = sp;
      Q = sq;
      return false;
    }
    // kModeGrid: epoch-tagged records in global memory
    const uint32_t epoch = rc + 1;
    uint32_t* slots = prm.slots + static_cast<size_t>(buf) * G * 8;
    if (tid == 0) {
      ll_store(slots + static_cast<size_t>(rank) * 8, static_cast<double>(bp), epoch);
      if (with_q) ll_store(slots + static_cast<size_t>(rank) * 8 + 4, static_cast<double>(bq), epoch);
      if (refill && issued < total) {
        const int s = static_cast<int>(issued % S);
        mbar_arrive_expect_tx(&full[s], bytes);
        bulk_g2s(xs + static_cast<size_t>(s) * prm.stage_elems, x + pcol * prm.ldx + r0, bytes, &full[s], pol);
        pc.next();
        ++issued;
        if (issued < total) pcol = pc.col();
      }
    }
    if (warp == 0) {
      T sp = T(0), sq = T(0);
      const uint64_t t0 = globaltimer();
      bool timed_out = false;
      for (uint32_t i = lane; i < G; i += 32) {
        double v;
        while (!ll_load(slots + static_cast<size_t>(i) * 8, epoch, v)) {
          if (globaltimer() - t0 > kTimeoutNs) { timed_out = true; break; }
        }
        sp = Num<T>::add(sp, static_cast<T>(v));
        if (with_q) {
          while (!ll_load(slots + static_cast<size_t>(i) * 8 + 4, epoch, v)) {
            if (globaltimer() - t0 > kTimeoutNs) { timed_out = true; break; }
          }
          sq = Num<T>::add(sq, static_cast<T>(v));
        }
      }
      if (timed_out) {
        report_error(prm.status, BAK_ETIMEOUT);
        my_abort = 1;
      }
      sp = warp_sum(sp);
      if (with_q) sq = warp_sum(sq);
      if (lane == 0) bcast[buf] = Pair<T>{static_cast<double>(sp), static_cast<double>(sq)};
    }
    const bool any2 = __syncthreads_or(my_abort) != 0;
    P = static_cast<T>(bcast[buf].p);
    Q = static_cast<T>(bcast[buf].q);
    return any2;
  };

  // ---- prologue: dot for the first column ----
  uint32_t rc = 0;
  T P, Q;
  bool aborted = false;
  {
    wait_stage(0);
    const T* X0 = xs;
    T pv = T(0);
#pragma unroll
    for (int k = 0; k < E; ++k) {
      const T xv = (k < kv) ? X0[tid + k * NT] : T(0);
      pv = Num<T>::fma(xv, ev[k], pv);
    }
    aborted = reduce(pv, T(0), false, rc++, false, P, Q);
  }

  ColCursor cc{prm.cols, ncols, prm.cols_stride, 0, 0};
  int64_t c_cur = cc.col();
  T n2_cur = n2g[c_cur];
  cc.next();
  int64_t c_next = (total > 1) ? cc.col() : c_cur;
  T n2_next = n2g[c_next];
  const bool updater = (rank == 0) && (tid == (NT > 32 ? 32 : 0));
  T a_val = updater ? ag[c_cur] : T(0);

  int64_t sweep = 0, k = 0, t = 0;
  bool converged = false;
  while (!aborted) {
    const T d = Num<T>::div(P, n2_cur);
    const bool last = (k == ncols - 1);
    const bool has_next = !(last && sweep + 1 == prm.max_iter);
    const T* Xc = xs + static_cast<size_t>(t % S) * prm.stage_elems;
    const T* Xn = xs + static_cast<size_t>((t + 1) % S) * prm.stage_elems;
    if (has_next) wait_stage(t + 1);
    T pv = T(0), qv = T(0);
#pragma unroll
    for (int kk = 0; kk < E; ++kk) {
      const bool ok = kk < kv;
      const T xc = ok ? Xc[tid + kk * NT] : T(0);
      ev[kk] = Num<T>::sub(ev[kk], Num<T>::mul(xc, d));
      if (has_next) {
        const T xn = ok ? Xn[tid + kk * NT] : T(0);
        pv = Num<T>::fma(xn, ev[kk], pv);
      }
      if (last) qv = Num<T>::fma(ev[kk], ev[kk], qv);
    }
    if (updater) {
      a_val = Num<T>::add(a_val, d);
      ag[c_cur] = a_val;
      if (has_next) a_val = ag[c_next];  // same-thread store->load: sees the new value if c_next == c_cur
    }
    aborted = reduce(pv, qv, last, rc++, true, P, Q);
    if (aborted) break;
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
    c_cur = c_next;
    n2_cur = n2_next;
    cc.next();
    if (t + 1 < total) {
      c_next = cc.col();
      n2_next = n2g[c_next];
    }
  }

  // ---- epilogue ----
#pragma unroll
  for (int kk = 0; kk < E; ++kk)
    if (kk < kv) eg[r0 + tid + static_cast<int64_t>(kk) * NT] = ev[kk];
  if (tid == 0) {
    // drain bulk copies still in flight into this CTA's ring
    for (int64_t u = t + 2; u < issued; ++u) {
      const int s = static_cast<int>(u % S);
      const uint32_t par = static_cast<uint32_t>((u / S) & 1);
      const uint64_t t0 = globaltimer();
      while (!mbar_test(&full[s], par))
        if (globaltimer() - t0 > kTimeoutNs) break;
    }
    if (rank == 0 && prm.status) {
      prm.status[0] = sweep;
      prm.status[1] = converged ? 1 : 0;
      prm.status[3] = MODE == kModeCta ? BAK_VARIANT_CTA : (MODE == kModeCluster ? BAK_VARIANT_CLUSTER : BAK_VARIANT_GRID);
    }
  }
  __syncthreads();
  if (MODE == kModeCluster) cluster_sync();
}

// ------------------------------- host -------------------------------------

size_t smem_bytes(const SweepPlan& pl, size_t tsize) {
  return static_cast<size_t>(pl.nstages) * pl.stage_elems * tsize + kMaxStages * 8 + 2 * 2 * 32 * tsize + 16 +
         2 * kMaxCluster * 16 + 16 + 32 + 16;
}

template <typename T, int E, int MODE>
int launch_one(const SweepPlan& pl, SweepParams prm, cudaStream_t st) {
  auto kern = sweep_kernel<T, E, MODE>;
  const size_t smem = smem_bytes(pl, sizeof(T));
  BAK_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(pl.nparticipants);
  cfg.blockDim = dim3(pl.nthreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
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
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  BAK_CHECK_CUDA(cudaLaunchKernelEx(&cfg, kern, prm));
  count_launches(1);
  return BAK_OK;
}

template <typename T, int MODE>
int launch_e(const SweepPlan& pl, const SweepParams& prm, cudaStream_t st) {
  switch (pl.e) {
    case 1: return launch_one<T, 1, MODE>(pl, prm, st);
    case 2: return launch_one<T, 2, MODE>(pl, prm, st);
    case 4: return launch_one<T, 4, MODE>(pl, prm, st);
    case 8: return launch_one<T, 8, MODE>(pl, prm, st);
    case 16: return launch_one<T, 16, MODE>(pl, prm, st);
    case 32: return launch_one<T, 32, MODE>(pl, prm, st);
  }
  set_error("bak_sweep: unsupported rows-per-thread %d", pl.e);
  return BAK_EUNSUPPORTED;
}

}  // namespace

// ---- planning: pick participants, threads, rows per thread, stages ----
static const int kEs[] = {1, 2, 4, 8, 16, 32};

bool plan_onchip(int dtype, int variant, int64_t obs, SweepPlan& pl) {
  const size_t ts = dtype_size(dtype);
  const int sms = device_sms();
  const size_t smem_cap = static_cast<size_t>(device_max_smem_optin()) - 4096;
  pl.variant = variant;
  auto fits = [&](int nthreads, int e, int parts) -> bool {
    const int64_t rows = static_cast<int64_t>(nthreads) * e;
    if (rows * parts < obs) return false;
    pl.nthreads = nthreads;
    pl.e = e;
    pl.nparticipants = parts;
    pl.rows_per_cta = rows;
    pl.stage_elems = rows;
    const size_t stage_bytes = rows * ts;
    int s = static_cast<int>((smem_cap - 2048) / stage_bytes);
    if (s > kMaxStages) s = kMaxStages;
    if (s < 2) return false;
    pl.nstages = s;
    return true;
  };
  if (variant == BAK_VARIANT_CTA) {
    // short columns: favour few warps (short reduction tree), E <= 32
    for (int e : kEs) {
      int nt = static_cast<int>(round_up((obs + e - 1) / e, 32));
      if (nt <= 256 && fits(nt < 32 ? 32 : nt, e, 1)) return true;
    }
    for (int e : kEs) {
      int nt = static_cast<int>(round_up((obs + e - 1) / e, 32));
      if (nt <= 512 && fits(nt, e, 1)) return true;
    }
    return false;
  }
  if (variant == BAK_VARIANT_CLUSTER) {
    for (int c = 2; c <= kMaxCluster; c *= 2) {
      const int64_t per = (obs + c - 1) / c;
      for (int e : kEs) {
        int nt = static_cast<int>(round_up((per + e - 1) / e, 32));
        if (nt <= 256 && fits(nt, e, c)) {
          // shrink participants if rows_per_cta leaves a CTA empty
          pl.nparticipants = static_cast<int>((obs + pl.rows_per_cta - 1) / pl.rows_per_cta);
          if (pl.nparticipants < 2) pl.nparticipants = 2;
          if (pl.nparticipants == 3) pl.nparticipants = 4;
          if (pl.nparticipants > 4 && pl.nparticipants < 8) pl.nparticipants = 8;
          if (pl.nparticipants > 8) pl.nparticipants = 16;
          if ((pl.nparticipants - 1) * pl.rows_per_cta >= obs) continue;
          return true;
        }
      }
    }
    return false;
  }
  if (variant == BAK_VARIANT_GRID) {
    for (int nt : {256, 512}) {
      for (int e : kEs) {
        const int64_t rows = static_cast<int64_t>(nt) * e;
        const int64_t parts = (obs + rows - 1) / rows;
        if (parts <= sms && fits(nt, e, static_cast<int>(parts)) && pl.nstages >= 3) return true;
      }
    }
    return false;
  }
  return false;
}

int launch_onchip(int dtype, const SweepPlan& pl, const SweepParams& prm, cudaStream_t st) {
  if (pl.variant == BAK_VARIANT_GRID && prm.slots)
    BAK_CHECK_CUDA(cudaMemsetAsync(prm.slots, 0, static_cast<size_t>(2) * pl.nparticipants * 32, st));
  if (dtype == BAK_F64) {
    if (pl.variant == BAK_VARIANT_CTA) return launch_e<double, kModeCta>(pl, prm, st);
    if (pl.variant == BAK_VARIANT_CLUSTER) return launch_e<double, kModeCluster>(pl, prm, st);
    return launch_e<double, kModeGrid>(pl, prm, st);
  }
  if (pl.variant == BAK_VARIANT_CTA) return launch_e<float, kModeCta>(pl, prm, st);
  if (pl.variant == BAK_VARIANT_CLUSTER) return launch_e<float, kModeCluster>(pl, prm, st);
  return launch_e<float, kModeGrid>(pl, prm, st);
}

}  // namespace bak

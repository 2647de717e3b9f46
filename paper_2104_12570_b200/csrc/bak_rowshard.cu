// (5) Exact per-column sweep over row-sharded x with an in-kernel cross-GPU
// scalar all-reduce per column (north-star component (5)).
//
// Rank r holds rows of x, y, e; a and norms2 are replicated.  Per column every
// rank runs the STREAM pass over its rows (bak_stream.cuh), reduces its CTAs'
// partials through global records (as the STREAM kernel), and then:
//   - CTA 0, lanes 0..N-1, posts the rank's {p, sum e^2} as epoch-tagged 16-byte
//     records (st.relaxed.sys) into slot [my_rank] of EVERY rank's mailbox —
//     peer-mapped device memory over NVLink (CUDA IPC), or local memory when N
//     ranks are emulated inside one launch;
//   - every CTA polls its own rank's mailbox (local memory) for the N records
//     and sums them in RANK ORDER, so d_j and a are bit-identical on all ranks.
// Epochs are unique per call (epoch_base + reduction index), so mailboxes are
// not reset between columns or calls; the host restarts the count (after
// zeroing every mailbox between two barriers) before it would wrap 31 bits.  Every spin wait has a deadline; a
// missing rank surfaces as BAK_ETIMEOUT, not a hang.
//
// Emulation (nranks_local = N > 1, one device): the grid is N groups of CTAs,
// group r owns rows [r*rows_per_rank, ...) of the one x/e and its own replica
// of a (a + r*vars), status (status + 4*r) and history (history + r*max_iter);
// its mailbox is mailboxes[r].  No CTA ever waits on a kernel that is not
// co-resident (cooperative launch).
#include <cstdlib>

#include "bak_common.cuh"
#include "bak_stream.cuh"
#include "bak_sweep.cuh"

namespace bak {
namespace {

constexpr int kMaxRanks = 8;

struct RowshardParams {
  const void* x;
  int64_t ldx, vars;
  int64_t rows_total;     // rows of this launch (all emulated ranks)
  int64_t rows_per_rank;  // aligned
  int64_t rows_per_cta;
  int ctas_per_rank;
  const void* norms2;
  void* e;
  void* a;
  int64_t max_iter;
  double thresh2;
  double* history;
  int64_t* status;
  uint32_t* slots;  // per launch-rank local records: [nr_local][slot_stride u32]
  int64_t slot_stride;
  int rank0;        // global rank of launch-rank 0
  int nranks;       // global number of ranks
  int nranks_local;
  int keep_next;  // x_{j+1} kept in L2 (this GPU's e and one column of its rows fit)
  uint32_t epoch_base;
  uint32_t* mbox[kMaxRanks];  // mailbox of every global rank: [2 bufs][nranks][8 u32]
};

constexpr int kRsCluster = 8;

template <typename T, bool CL>
__global__ void __launch_bounds__(512, 1) rowshard_kernel(const RowshardParams p) {
  __shared__ T red[2 * 2 * 32];
  __shared__ double bc[2][2];
  __shared__ ClExchange clx;  // two-level exchange state (CL)
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  uint32_t crank = 0, C = 1;
  if (CL) {
    crank = cluster_rank();
    C = cluster_size();
    cl_exchange_init(clx);
    __syncthreads();
    cluster_sync();
  }
  const int lr = blockIdx.x / p.ctas_per_rank;        // launch-local rank
  const int cta = blockIdx.x % p.ctas_per_rank;      // CTA within the rank
  const uint32_t G = static_cast<uint32_t>(p.ctas_per_rank);
  const int grank = p.rank0 + lr;                     // global rank
  const int N = p.nranks;
  const int64_t rr0 = static_cast<int64_t>(lr) * p.rows_per_rank;
  const int64_t rrows = imax64(0, imin64(p.rows_total - rr0, p.rows_per_rank));
  const int64_t r0 = static_cast<int64_t>(cta) * p.rows_per_cta;
  const int64_t nrows = imax64(0, imin64(rrows - r0, p.rows_per_cta));
  const T* __restrict__ x = static_cast<const T*>(p.x) + rr0 + r0;
  T* e = static_cast<T*>(p.e) + rr0 + r0;
  const T* __restrict__ n2g = static_cast<const T*>(p.norms2);
  T* __restrict__ ag = static_cast<T*>(p.a) + static_cast<int64_t>(lr) * p.vars;
  int64_t* status = p.status ? p.status + 4 * lr : nullptr;
  double* history = p.history ? p.history + static_cast<int64_t>(lr) * p.max_iter : nullptr;
  uint32_t* slots = p.slots + static_cast<size_t>(lr) * p.slot_stride;
  uint32_t* mine = p.mbox[grank];
  const int64_t ncols = p.vars, total = p.max_iter * ncols;
  int my_abort = 0;

  auto exchange = [&](T pv, T qv, bool with_q, uint32_t rc, T& P, T& Q) -> bool {
    const int buf = rc & 1;
    if (block_sum2(pv, qv, with_q, buf, red, my_abort)) return true;
    const uint32_t epoch = p.epoch_base + rc + 1;
    if (CL) {
      // clusters of this rank -> rank total (cl_grid_sum), then the cross-rank
      // stage inside the leaders: cluster 0's leader posts the rank total into
      // every rank's mailbox, every leader sums the N totals in rank order
      const uint32_t cid = static_cast<uint32_t>(cta) / C, ncl = G / C;
      bool to = false;
      auto hook = [&](T& sp, T& sq, bool& tout) {
        if (cid == 0 && lane < N) {
          uint32_t* dst = p.mbox[lane] + (static_cast<size_t>(buf) * N + grank) * 8;
          ll_store_sys(dst, static_cast<double>(sp), epoch);
          ll_store_sys(dst + 4, static_cast<double>(sq), epoch);
        }
        double vp = 0.0, vq = 0.0;
        if (lane < N) {
          const uint32_t* src = mine + (static_cast<size_t>(buf) * N + lane) * 8;
          const uint64_t t0 = globaltimer();
          while (!ll_load_sys(src, epoch, vp))
            if (globaltimer() - t0 > kTimeoutNs) { tout = true; break; }
          if (with_q)
            while (!ll_load_sys(src + 4, epoch, vq))
              if (globaltimer() - t0 > kTimeoutNs) { tout = true; break; }
        }
        T tp = T(0), tq = T(0);
        for (int r = 0; r < N; ++r) {
          tp = Num<T>::add(tp, static_cast<T>(__shfl_sync(0xffffffffu, vp, r)));
          if (with_q) tq = Num<T>::add(tq, static_cast<T>(__shfl_sync(0xffffffffu, vq, r)));
        }
        sp = tp;
        sq = tq;
      };
      cl_grid_sum<T>(clx, pv, qv, with_q, rc, slots, epoch, crank, C, cid, ncl, to, hook);
      if (to) {
        report_error(status, BAK_ETIMEOUT);
        my_abort = 1;
      }
      const bool ab = __syncthreads_or(my_abort) != 0;
      P = static_cast<T>(clx.bcast[buf].p);
      Q = static_cast<T>(clx.bcast[buf].q);
      return ab;
    }
    uint32_t* ls = slots + static_cast<size_t>(buf) * G * 8;
    if (tid == 0) {
      ll_store(ls + static_cast<size_t>(cta) * 8, static_cast<double>(pv), epoch);
      if (with_q) ll_store(ls + static_cast<size_t>(cta) * 8 + 4, static_cast<double>(qv), epoch);
    }
    if (warp == 0) {
      // 1) this rank's partial: all its CTAs' records, fixed order
      T sp, sq;
      bool to = false;
      warp_gather_slots(ls, G, epoch, with_q, sp, sq, to);
      // 2) CTA 0 posts it into slot [grank] of every rank's mailbox
      if (cta == 0 && lane < N) {
        uint32_t* dst = p.mbox[lane] + (static_cast<size_t>(buf) * N + grank) * 8;
        ll_store_sys(dst, static_cast<double>(sp), epoch);
        ll_store_sys(dst + 4, static_cast<double>(sq), epoch);
      }
      // 3) every CTA: N rank records from its own mailbox, summed in rank order
      double vp = 0.0, vq = 0.0;
      if (lane < N) {
        const uint32_t* src = mine + (static_cast<size_t>(buf) * N + lane) * 8;
        const uint64_t t0 = globaltimer();
        while (!ll_load_sys(src, epoch, vp))
          if (globaltimer() - t0 > kTimeoutNs) { to = true; break; }
        if (with_q)
          while (!ll_load_sys(src + 4, epoch, vq))
            if (globaltimer() - t0 > kTimeoutNs) { to = true; break; }
      }
      T tp = T(0), tq = T(0);
      for (int r = 0; r < N; ++r) {
        tp = Num<T>::add(tp, static_cast<T>(__shfl_sync(0xffffffffu, vp, r)));
        if (with_q) tq = Num<T>::add(tq, static_cast<T>(__shfl_sync(0xffffffffu, vq, r)));
      }
      if (to) {
        report_error(status, BAK_ETIMEOUT);
        my_abort = 1;
      }
      if (lane == 0) {
        bc[buf][0] = static_cast<double>(tp);
        bc[buf][1] = static_cast<double>(tq);
      }
    }
    const bool ab = __syncthreads_or(my_abort) != 0;
    P = static_cast<T>(bc[buf][0]);
    Q = static_cast<T>(bc[buf][1]);
    return ab;
  };

  uint32_t rc = 0;
  T P, Q, pv, qv;
  bool backward = false;
  stream_pass<T>(e, nullptr, x + 0 * p.ldx, nrows, T(0), false, true, false, backward, pv, qv);
  bool aborted = exchange(pv, T(0), false, rc++, P, Q);
  const bool updater = cta == 0 && tid == 32;
  int64_t c = 0;
  T a_val = updater ? ag[0] : T(0);
  int64_t sweep = 0, k = 0, t = 0;
  bool converged = false;
  while (!aborted) {
    const T n2 = n2g[c];
    const T d = n2 != T(0) ? Num<T>::div(P, n2) : T(0);
    const bool last = k == ncols - 1;
    const bool has_next = !(last && sweep + 1 == p.max_iter);
    const int64_t cn = last ? 0 : c + 1;
    backward = !backward;
    stream_pass<T>(e, x + c * p.ldx, x + cn * p.ldx, nrows, d, n2 != T(0), has_next, last, backward, pv, qv,
                   p.keep_next != 0);
    if (updater) {
      if (n2 != T(0)) {
        a_val = Num<T>::add(a_val, d);
        ag[c] = a_val;
      }
      if (has_next) a_val = ag[cn];
    }
    aborted = exchange(pv, qv, last, rc++, P, Q);
    if (aborted) break;
    if (last) {
      if (cta == 0 && tid == 0 && history) history[sweep] = static_cast<double>(Q);
      ++sweep;
      if (p.thresh2 >= 0.0 && static_cast<double>(Q) <= p.thresh2) {
        converged = true;
        break;
      }
      if (sweep == p.max_iter) break;
      k = 0;
    } else {
      ++k;
    }
    ++t;
    c = cn;
  }
  if (cta == 0 && tid == 0 && status) {
    status[0] = sweep;
    status[1] = converged ? 1 : 0;
    status[3] = BAK_VARIANT_STREAM;
  }
  (void)total;
  if (CL) {
    __syncthreads();
    cluster_sync();
  }
}

template <typename T>
int rowshard_cluster_capacity() {
  static int cap = -1;
  if (cap >= 0) return cap;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(kRsCluster * 4);
  cfg.blockDim = dim3(512);
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = kRsCluster;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  int n = 0;
  cap = cudaOccupancyMaxActiveClusters(&n, rowshard_kernel<T, true>, &cfg) == cudaSuccess ? n : 0;
  cudaGetLastError();
  return cap;
}

}  // namespace
}  // namespace bak

using namespace bak;

// records: [2 bufs][nranks] x 32 bytes (p LL record + q LL record)
extern "C" int64_t bak_mailbox_bytes(int64_t nranks) { return nranks < 1 ? 0 : 2 * nranks * 32; }

extern "C" int bak_sweep_rowshard(int dtype, const void* x, int64_t obs_local, int64_t vars, int64_t ldx,
                                  const void* norms2, void* e, void* a, int64_t max_iter, double thresh2,
                                  double* history, int64_t* status, int rank, int nranks, void* const* mailboxes,
                                  int64_t epoch_base, int nranks_local, void* workspace, int64_t workspace_bytes,
                                  void* stream) {
  if ((dtype != BAK_F32 && dtype != BAK_F64) || !x || obs_local < 1 || vars < 1 || ldx < obs_local || !norms2 ||
      !e || !a || max_iter < 1 || nranks < 1 || nranks > kMaxRanks || nranks_local < 1 ||
      rank < 0 || rank + nranks_local > nranks || !mailboxes || !status) {
    set_error("bak_sweep_rowshard: bad arguments");
    return BAK_EINVAL;
  }
  const size_t ts = dtype_size(dtype);
  const int64_t vec = 16 / static_cast<int64_t>(ts);
  if (reinterpret_cast<uintptr_t>(x) % 16 || (ldx * static_cast<int64_t>(ts)) % 16 ||
      reinterpret_cast<uintptr_t>(e) % 16) {
    set_error("bak_sweep_rowshard: x/e must be 16-byte aligned with ldx*sizeof(T) %% 16 == 0");
    return BAK_EINVAL;
  }
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  // One rank per device whose rows fit on chip (C3 fp64 over 8 GPUs: 2M rows):
  // the exact on-chip sweep (e in registers, x streamed once — XT / register
  // GRID plans) with the cross-GPU stage inside its two-level exchange, instead
  // of the STREAM pass that moves e through L2 every column.  BAK_ROWSHARD_ONCHIP=0
  // keeps the STREAM kernel.
  {
    const char* oc = getenv("BAK_ROWSHARD_ONCHIP");
    SweepPlan pl;
    if (nranks_local == 1 && !(oc && oc[0] == '0') && workspace && workspace_bytes >= kGridSlotBytes &&
        plan_onchip(dtype, BAK_VARIANT_GRID, obs_local, pl) && pl.variant == BAK_VARIANT_GRID && pl.cluster != 0) {
      SweepParams sp{};
      sp.x = x;
      sp.obs = obs_local;
      sp.ldx = ldx;
      sp.norms2 = norms2;
      sp.cols = nullptr;
      sp.ncols = vars;
      sp.cols_stride = 0;
      sp.e = e;
      sp.a = a;
      sp.max_iter = max_iter;
      sp.thresh2 = thresh2;
      sp.history = history;
      sp.status = status;
      sp.slots = static_cast<uint32_t*>(workspace);
      sp.rows_per_cta = pl.rows_per_cta;
      sp.stage_elems = pl.stage_elems;
      sp.nstages = pl.nstages;
      sp.keep_next = 0;
      sp.nranks = nranks;
      sp.grank = rank;
      sp.epoch_base = static_cast<uint32_t>(epoch_base);
      for (int r = 0; r < nranks; ++r) sp.mbox[r] = static_cast<uint32_t*>(mailboxes[r]);
      BAK_CHECK_CUDA(cudaMemsetAsync(status, 0, 4 * sizeof(int64_t), st));
      if (launch_onchip(dtype, pl, sp, st) == BAK_OK) return BAK_OK;
      g_err_clear();  // clusters not co-resident: the STREAM kernel below
      cudaGetLastError();
    }
  }
  const int sms = device_sms();
  int per_rank_ctas = imax64(1, sms / nranks_local);
  // two-level exchange: whole clusters of 8 per rank (<= 32 per rank), all co-resident
  const char* flat = getenv("BAK_STREAM_FLAT");
  const int cap = dtype == BAK_F64 ? rowshard_cluster_capacity<double>() : rowshard_cluster_capacity<float>();
  int cl_per_rank = static_cast<int>(imin64(imin64(cap, sms / kRsCluster) / nranks_local, 32));
  // (only when it keeps >= 3/4 of the CTAs: with many emulated ranks per GPU
  // one cluster per rank would starve the streaming passes of bandwidth)
  const bool use_cl = !(flat && flat[0] == '1') && cl_per_rank >= 1 && coop_clusters_ok() &&
                      4 * cl_per_rank * kRsCluster >= 3 * per_rank_ctas;
  if (use_cl) per_rank_ctas = cl_per_rank * kRsCluster;
  const int64_t rows_per_rank = round_up((obs_local + nranks_local - 1) / nranks_local, vec);
  const int64_t rows_per_cta = round_up((rows_per_rank + per_rank_ctas - 1) / per_rank_ctas, vec);
  const int64_t slot_stride = imax64(2LL * per_rank_ctas * 8, 2LL * 32 * 8);  // u32 per launch-rank
  const int64_t need = static_cast<int64_t>(nranks_local) * slot_stride * 4;
  if (!workspace || workspace_bytes < need) {
    set_error("bak_sweep_rowshard: workspace too small (need %lld)", (long long)need);
    return BAK_EWORKSPACE;
  }
  RowshardParams p{};
  p.x = x;
  p.ldx = ldx;
  p.vars = vars;
  p.rows_total = obs_local;
  p.rows_per_rank = rows_per_rank;
  p.rows_per_cta = rows_per_cta;
  p.ctas_per_rank = per_rank_ctas;
  p.norms2 = norms2;
  p.e = e;
  p.a = a;
  p.max_iter = max_iter;
  p.thresh2 = thresh2;
  p.history = history;
  p.status = status;
  p.slots = static_cast<uint32_t*>(workspace);
  p.slot_stride = slot_stride;
  // this GPU's e plus one column of its rows fit in L2: keep x_{j+1} there, so
  // HBM sees each column once (e.g. C3 fp64 over 8 GPUs: 2 x 16.8 MB per GPU)
  p.keep_next = 2 * obs_local * static_cast<int64_t>(ts) <= static_cast<int64_t>(0.75 * l2_bytes());
  if (const char* k = getenv("BAK_STREAM_KEEP")) p.keep_next = k[0] == '1';
  p.rank0 = rank;
  p.nranks = nranks;
  p.nranks_local = nranks_local;
  p.epoch_base = static_cast<uint32_t>(epoch_base);
  for (int r = 0; r < nranks; ++r) p.mbox[r] = static_cast<uint32_t*>(mailboxes[r]);
  BAK_CHECK_CUDA(cudaMemsetAsync(workspace, 0, need, st));
  BAK_CHECK_CUDA(cudaMemsetAsync(status, 0, 4 * sizeof(int64_t) * nranks_local, st));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(per_rank_ctas * nranks_local);
  cfg.blockDim = dim3(512);
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = kRsCluster;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = use_cl ? 2 : 1;
  cudaError_t err = dtype == BAK_F64
                        ? cudaLaunchKernelEx(&cfg, use_cl ? rowshard_kernel<double, true> : rowshard_kernel<double, false>, p)
                        : cudaLaunchKernelEx(&cfg, use_cl ? rowshard_kernel<float, true> : rowshard_kernel<float, false>, p);
  if (err != cudaSuccess && use_cl) {
    // clusters not co-resident after all: one-level exchange over all SMs
    cudaGetLastError();
    const int flat_ctas = static_cast<int>(imax64(1, sms / nranks_local));
    const int64_t flat_stride = imax64(2LL * flat_ctas * 8, 2LL * 32 * 8);
    if (static_cast<int64_t>(nranks_local) * flat_stride * 4 <= workspace_bytes) {
      p.ctas_per_rank = flat_ctas;
      p.rows_per_cta = round_up((rows_per_rank + flat_ctas - 1) / flat_ctas, vec);
      p.slot_stride = flat_stride;
      BAK_CHECK_CUDA(cudaMemsetAsync(workspace, 0, nranks_local * flat_stride * 4, st));
      cfg.gridDim = dim3(flat_ctas * nranks_local);
      cfg.numAttrs = 1;
      err = dtype == BAK_F64 ? cudaLaunchKernelEx(&cfg, rowshard_kernel<double, false>, p)
                             : cudaLaunchKernelEx(&cfg, rowshard_kernel<float, false>, p);
    }
  }
  BAK_CHECK_CUDA(err);
  count_launches(1);
  return BAK_OK;
}

// Mailboxes exported over CUDA IPC must be their OWN allocation: a handle
// names a whole cudaMalloc allocation and the importer maps its base, so a
// sub-allocation (e.g. from a caching allocator) would be mapped at the wrong
// address on the peers.
extern "C" int bak_dev_alloc(int64_t bytes, void** devptr) {
  if (!devptr || bytes < 1) {
    set_error("bak_dev_alloc: bad arguments");
    return BAK_EINVAL;
  }
  BAK_CHECK_CUDA(cudaMalloc(devptr, static_cast<size_t>(bytes)));
  BAK_CHECK_CUDA(cudaMemset(*devptr, 0, static_cast<size_t>(bytes)));
  return BAK_OK;
}

extern "C" int bak_dev_free(void* devptr) {
  BAK_CHECK_CUDA(cudaFree(devptr));
  return BAK_OK;
}

// Zero a mailbox before its epoch count restarts (synchronous).
extern "C" int bak_dev_zero(void* devptr, int64_t bytes) {
  if (!devptr || bytes < 1) {
    set_error("bak_dev_zero: bad arguments");
    return BAK_EINVAL;
  }
  BAK_CHECK_CUDA(cudaMemset(devptr, 0, static_cast<size_t>(bytes)));
  BAK_CHECK_CUDA(cudaDeviceSynchronize());
  return BAK_OK;
}

extern "C" int bak_ipc_get_handle(void* devptr, void* handle64) {
  cudaIpcMemHandle_t h;
  BAK_CHECK_CUDA(cudaIpcGetMemHandle(&h, devptr));
  static_assert(sizeof(h) == 64, "CUDA IPC handle is 64 bytes");
  memcpy(handle64, &h, 64);
  return BAK_OK;
}

extern "C" int bak_ipc_open_handle(const void* handle64, void** devptr) {
  cudaIpcMemHandle_t h;
  memcpy(&h, handle64, 64);
  BAK_CHECK_CUDA(cudaIpcOpenMemHandle(devptr, h, cudaIpcMemLazyEnablePeerAccess));
  return BAK_OK;
}

extern "C" int bak_ipc_close(void* devptr) {
  BAK_CHECK_CUDA(cudaIpcCloseMemHandle(devptr));
  return BAK_OK;
}

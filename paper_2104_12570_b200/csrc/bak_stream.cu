// STREAM variant: the exact per-column sweep (bak.py:92-112) for tall systems
// whose residual e does not fit on chip (e.g. 2^24 x 256 fp64 on one B200:
// e = 134 MB vs ~70 MB of registers + shared memory).
//
// Persistent co-resident grid; CTA r owns rows [r*R, (r+1)*R).  Per column the
// CTA makes ONE fused streaming pass over its rows:
//     e -= fl(d_j * x_j) ; p += x_{j+1} . e  (+ sum e^2 on the sweep's last column)
// with 16-byte vector loads (x with the evict-first streaming hint), then one
// grid reduction through epoch-tagged global records.  Per column the pass
// moves x_j + x_{j+1} + e (read) + e (write) = 4 column-lengths of HBM traffic,
// so the x-stream share of HBM bandwidth is capped near 25%;
// alternating the traversal direction every column lets the tail of one pass
// (e and x_{j+1}, the next pass's e and x_j) hit in the 126 MB L2.
#include <cstdlib>

#include "bak_exchange.cuh"
#include "bak_stream.cuh"
#include "bak_sweep.cuh"

namespace bak {
namespace {

constexpr int kStreamCluster = 8;

template <typename T, bool CL>
__global__ void __launch_bounds__(512, 1) stream_kernel(const SweepParams prm) {
  __shared__ T red[2 * 2 * 32];
  __shared__ double bc[2][2];
  __shared__ ClExchange clx;  // two-level exchange state (CL)
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = blockIdx.x, G = gridDim.x;
  uint32_t crank = 0, C = 1;
  if (CL) {
    crank = cluster_rank();
    C = cluster_size();
    cl_exchange_init(clx);
    __syncthreads();
    cluster_sync();
  }
  const T* __restrict__ x = static_cast<const T*>(prm.x);
  const T* __restrict__ n2g = static_cast<const T*>(prm.norms2);
  T* __restrict__ ag = static_cast<T*>(prm.a);
  const int64_t r0 = static_cast<int64_t>(rank) * prm.rows_per_cta;
  const int64_t nrows = imax64(0, imin64(prm.obs - r0, prm.rows_per_cta));
  T* e = static_cast<T*>(prm.e) + r0;
  const int64_t ncols = prm.ncols, total = prm.max_iter * ncols;
  int my_abort = 0;

  auto exchange = [&](T p, T q, bool with_q, uint32_t rc, T& P, T& Q) -> bool {
    const int buf = rc & 1;
    if (block_sum2(p, q, with_q, buf, red, my_abort)) return true;
    const uint32_t epoch = rc + 1;
    if (CL) {
      bool to = false;
      cl_grid_sum<T>(clx, p, q, with_q, rc, prm.slots, epoch, crank, C, blockIdx.x / C, gridDim.x / C, to,
                     [](T&, T&, bool&) {});
      if (to) {
        report_error(prm.status, BAK_ETIMEOUT);
        my_abort = 1;
      }
      const bool ab = __syncthreads_or(my_abort) != 0;
      P = static_cast<T>(clx.bcast[buf].p);
      Q = static_cast<T>(clx.bcast[buf].q);
      return ab;
    }
    uint32_t* slots = prm.slots + static_cast<size_t>(buf) * G * 8;
    if (tid == 0) {
      ll_store(slots + static_cast<size_t>(rank) * 8, static_cast<double>(p), epoch);
      if (with_q) ll_store(slots + static_cast<size_t>(rank) * 8 + 4, static_cast<double>(q), epoch);
    }
    if (warp == 0) {
      T sp, sq;
      bool to = false;
      warp_gather_slots(slots, G, epoch, with_q, sp, sq, to);
      if (to) {
        report_error(prm.status, BAK_ETIMEOUT);
        my_abort = 1;
      }
      if (lane == 0) {
        bc[buf][0] = static_cast<double>(sp);
        bc[buf][1] = static_cast<double>(sq);
      }
    }
    const bool ab = __syncthreads_or(my_abort) != 0;
    P = static_cast<T>(bc[buf][0]);
    Q = static_cast<T>(bc[buf][1]);
    return ab;
  };

  StreamCursor cc{prm.cols, ncols, prm.cols_stride, 0, 0};
  int64_t c_cur = cc.col();
  uint32_t rc = 0;
  T P, Q, pv, qv;
  bool backward = false;
  stream_pass<T>(e, nullptr, x + c_cur * prm.ldx + r0, nrows, T(0), false, true, false, backward, pv, qv);
  bool aborted = exchange(pv, T(0), false, rc++, P, Q);

  T n2_cur = n2g[c_cur];
  cc.next();
  int64_t c_next = total > 1 ? cc.col() : c_cur;
  const bool updater = rank == 0 && tid == 32;
  T a_val = updater ? ag[c_cur] : T(0);
  int64_t sweep = 0, k = 0, t = 0;
  bool converged = false;
  while (!aborted) {
    const T d = Num<T>::div(P, n2_cur);
    const bool last = k == ncols - 1;
    const bool has_next = !(last && sweep + 1 == prm.max_iter);
    T n2_next = has_next ? n2g[c_next] : T(0);
    backward = !backward;
    stream_pass<T>(e, x + c_cur * prm.ldx + r0, x + c_next * prm.ldx + r0, nrows, d, true, has_next, last, backward,
                   pv, qv, prm.keep_next != 0);
    if (updater) {
      a_val = Num<T>::add(a_val, d);
      ag[c_cur] = a_val;
      if (has_next) a_val = ag[c_next];
    }
    aborted = exchange(pv, qv, last, rc++, P, Q);
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
    if (t + 1 < total) c_next = cc.col();
  }
  if (rank == 0 && tid == 0 && prm.status) {
    prm.status[0] = sweep;
    prm.status[1] = converged ? 1 : 0;
    prm.status[3] = BAK_VARIANT_STREAM;
  }
  if (CL) {  // no CTA leaves while a peer may still write into its shared memory
    __syncthreads();
    cluster_sync();
  }
}

template <typename T>
int stream_cluster_capacity() {
  static int cap = -1;
  if (cap >= 0) return cap;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(kStreamCluster * 4);
  cfg.blockDim = dim3(512);
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = kStreamCluster;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 2;
  int n = 0;
  cap = cudaOccupancyMaxActiveClusters(&n, stream_kernel<T, true>, &cfg) == cudaSuccess ? n : 0;
  cudaGetLastError();
  return cap;
}

}  // namespace

bool plan_stream(int dtype, int64_t obs, StreamPlan& pl) {
  const int sms = device_sms();
  pl.nthreads = 512;
  pl.nblocks = sms;
  const int64_t vec = 16 / static_cast<int64_t>(dtype_size(dtype));
  int64_t per = (obs + pl.nblocks - 1) / pl.nblocks;
  per = round_up(per, vec);
  pl.rows_per_cta = per;
  pl.nblocks = static_cast<int>((obs + per - 1) / per);
  return pl.nblocks >= 1;
}

int launch_stream(int dtype, const StreamPlan& pl0, const SweepParams& prm0, cudaStream_t st) {
  SweepParams prm = prm0;
  StreamPlan pl = pl0;
  // two-level exchange: one CTA per SM in clusters of 8 (<= 32 clusters, all
  // co-resident); BAK_STREAM_FLAT=1 keeps the one-level record gather
  const char* flat = getenv("BAK_STREAM_FLAT");
  const int cap = dtype == BAK_F64 ? stream_cluster_capacity<double>() : stream_cluster_capacity<float>();
  int ncl = pl.nblocks / kStreamCluster;
  if (ncl > cap) ncl = cap;
  if (ncl > 32) ncl = 32;
  const bool cl = !(flat && flat[0] == '1') && ncl >= 2 && coop_clusters_ok();
  if (cl) {
    const int64_t vec = 16 / static_cast<int64_t>(dtype_size(dtype));
    pl.nblocks = ncl * kStreamCluster;
    pl.rows_per_cta = round_up((prm.obs + pl.nblocks - 1) / pl.nblocks, vec);
    pl.nblocks = static_cast<int>((prm.obs + pl.rows_per_cta - 1) / pl.rows_per_cta);
    if (pl.nblocks % kStreamCluster) {  // ragged: fall back to the one-level exchange
      pl = pl0;
    }
  }
  const bool use_cl = cl && pl.nblocks % kStreamCluster == 0;
  prm.rows_per_cta = pl.rows_per_cta;
  // e plus one column of x fit comfortably in L2: keep x_{j+1} there for the
  // next column step (HBM then sees each column once); BAK_STREAM_KEEP=0|1 forces
  prm.keep_next = 2 * prm.obs * static_cast<int64_t>(dtype_size(dtype)) <= static_cast<int64_t>(0.75 * l2_bytes());
  if (const char* k = getenv("BAK_STREAM_KEEP")) prm.keep_next = k[0] == '1';
  BAK_CHECK_CUDA(cudaMemsetAsync(prm.slots, 0, kGridSlotBytes, st));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(pl.nblocks);
  cfg.blockDim = dim3(pl.nthreads);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = kStreamCluster;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = use_cl ? 2 : 1;
  cudaError_t err = dtype == BAK_F64
                        ? cudaLaunchKernelEx(&cfg, use_cl ? stream_kernel<double, true> : stream_kernel<double, false>, prm)
                        : cudaLaunchKernelEx(&cfg, use_cl ? stream_kernel<float, true> : stream_kernel<float, false>, prm);
  if (err != cudaSuccess && use_cl) {
    // the occupancy query can be optimistic about co-resident clusters: one-level exchange
    cudaGetLastError();
    prm.rows_per_cta = pl0.rows_per_cta;
    cfg.gridDim = dim3(pl0.nblocks);
    cfg.numAttrs = 1;
    err = dtype == BAK_F64 ? cudaLaunchKernelEx(&cfg, stream_kernel<double, false>, prm)
                           : cudaLaunchKernelEx(&cfg, stream_kernel<float, false>, prm);
  }
  BAK_CHECK_CUDA(err);
  count_launches(1);
  return BAK_OK;
}

}  // namespace bak

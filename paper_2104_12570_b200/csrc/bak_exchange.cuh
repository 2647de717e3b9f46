// Block- and grid-level deterministic reductions shared by the persistent
// kernels.  Fixed order: warp xor-butterfly, warps in index order, CTAs in
// rank order (lane-strided then butterfly) — identical bits in every thread of
// every participant, and independent of timing.
#pragma once
#include "bak_common.cuh"

namespace bak {

// Sum (p, q) over the CTA.  `red` is [2 bufs][2][32] in shared memory.  The
// embedded __syncthreads_or makes `my_abort` uniform; returns true if any
// thread of the CTA flagged an abort.
template <typename T>
__device__ __forceinline__ bool block_sum2(T& p, T& q, bool with_q, int buf, T* red, int my_abort) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  p = warp_sum(p);
  if (with_q) q = warp_sum(q);
  if (lane == 0) {
    red[(buf * 2 + 0) * 32 + warp] = p;
    red[(buf * 2 + 1) * 32 + warp] = q;
  }
  if (__syncthreads_or(my_abort)) return true;
  T bp = T(0), bq = T(0);
  for (int w = 0; w < nwarps; ++w) bp = Num<T>::add(bp, red[(buf * 2 + 0) * 32 + w]);
  if (with_q)
    for (int w = 0; w < nwarps; ++w) bq = Num<T>::add(bq, red[(buf * 2 + 1) * 32 + w]);
  p = bp;
  q = bq;
  return false;
}

// Warp 0 collects G epoch-tagged records {p, q} from global slots
// (slot i = 8 words: LL record p then LL record q) and returns the fixed-order
// sums in every lane.  Sets timed_out on deadline.
template <typename T>
__device__ __forceinline__ void warp_gather_slots(const uint32_t* slots, uint32_t G, uint32_t epoch, bool with_q,
                                                  T& sp, T& sq, bool& timed_out) {
  const int lane = threadIdx.x & 31;
  sp = T(0);
  sq = T(0);
  const uint64_t t0 = globaltimer();
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
  sp = warp_sum(sp);
  if (with_q) sq = warp_sum(sq);
}

// Two-level grid sum for persistent cooperative grids launched as clusters of
// C CTAs (C <= 16, at most 32 clusters): (1) every CTA st.async's its (p, q)
// into every cluster peer's slot (DSMEM, completion as tx bytes on the peer's
// mbarrier); (2) the cluster leader sums its C slots in rank order, posts the
// cluster sum as an epoch-tagged record, gathers the ncl records (lane =
// cluster) and sums them with a fixed butterfly — identical bits in every
// leader; (3) the leader st.async's the total into every peer's broadcast slot.
// Called by all threads after the block sum; returns the total in P, Q for all
// threads; sets timed_out on a deadline.  Replaces the flat all-to-all record
// gather (~5 µs per exchange on 148 CTAs) with ~2 µs.
struct alignas(16) ClPair {
  double p, q;
};
struct ClExchange {
  ClPair slot[2][16];
  ClPair bcast[2];
  uint64_t bar[2];
  uint64_t bar2[2];
};

__device__ __forceinline__ void cl_exchange_init(ClExchange& x) {
  if (threadIdx.x == 0) {
    mbar_init(&x.bar[0], 1);
    mbar_init(&x.bar[1], 1);
    mbar_init(&x.bar2[0], 1);
    mbar_init(&x.bar2[1], 1);
    fence_mbar_init();
  }
}

__device__ __forceinline__ void cl_st_async(uint32_t remote_addr, double v0, double v1, uint32_t remote_bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(
                   remote_addr),
               "d"(v0), "d"(v1), "r"(remote_bar)
               : "memory");
}

// gather(mode): after the leader has the grid total of THIS group, a caller
// hook may replace it (e.g. a cross-GPU mailbox stage); see rowshard.
template <typename T, typename Hook>
__device__ __forceinline__ void cl_grid_sum(ClExchange& x, T p, T q, bool with_q, uint32_t rc, uint32_t* part,
                                            uint32_t epoch, uint32_t crank, uint32_t C, uint32_t cid, uint32_t ncl,
                                            bool& timed_out, Hook hook) {
  const int tid = threadIdx.x, lane = tid & 31;
  const int buf = rc & 1;
  const uint32_t par = (rc >> 1) & 1;
  if (tid < static_cast<int>(C)) {
    const uint32_t rs = mapa(smem_addr(&x.slot[buf][crank]), tid);
    const uint32_t rb = mapa(smem_addr(&x.bar[buf]), tid);
    cl_st_async(rs, static_cast<double>(p), static_cast<double>(q), rb);
  }
  if (tid == 0) {
    mbar_arrive_expect_tx(&x.bar[buf], C * 16u);
    mbar_arrive_expect_tx(&x.bar2[buf], 16u);
  }
  if (crank == 0 && tid < 32) {
    if (!mbar_test_cluster(&x.bar[buf], par)) {
      const uint64_t t0 = globaltimer();
      while (!mbar_test_cluster(&x.bar[buf], par))
        if (globaltimer() - t0 > kTimeoutNs) { timed_out = true; break; }
    }
    T cp = T(0), cq = T(0);
    for (uint32_t r = 0; r < C; ++r) {
      cp = Num<T>::add(cp, static_cast<T>(x.slot[buf][r].p));
      if (with_q) cq = Num<T>::add(cq, static_cast<T>(x.slot[buf][r].q));
    }
    uint32_t* rec = part + static_cast<size_t>(buf) * 32 * 8;
    if (lane == 0) {
      ll_store(rec + static_cast<size_t>(cid) * 8, static_cast<double>(cp), epoch);
      if (with_q) ll_store(rec + static_cast<size_t>(cid) * 8 + 4, static_cast<double>(cq), epoch);
    }
    T vp = T(0), vq = T(0);
    if (lane < static_cast<int>(ncl)) {
      double v = 0.0;
      const uint64_t t0 = globaltimer();
      while (!ll_load(rec + static_cast<size_t>(lane) * 8, epoch, v))
        if (globaltimer() - t0 > kTimeoutNs) { timed_out = true; break; }
      vp = static_cast<T>(v);
      if (with_q) {
        while (!ll_load(rec + static_cast<size_t>(lane) * 8 + 4, epoch, v))
          if (globaltimer() - t0 > kTimeoutNs) { timed_out = true; break; }
        vq = static_cast<T>(v);
      }
    }
    T sp = warp_sum(vp);
    T sq = with_q ? warp_sum(vq) : T(0);
    hook(sp, sq, timed_out);  // e.g. all ranks' totals through NVLink mailboxes
    if (lane < static_cast<int>(C)) {
      const uint32_t rs = mapa(smem_addr(&x.bcast[buf]), lane);
      const uint32_t rb = mapa(smem_addr(&x.bar2[buf]), lane);
      cl_st_async(rs, static_cast<double>(sp), static_cast<double>(sq), rb);
    }
  }
  if (tid < 32) {
    if (!mbar_test_cluster(&x.bar2[buf], par)) {
      const uint64_t t0 = globaltimer();
      while (!mbar_test_cluster(&x.bar2[buf], par))
        if (globaltimer() - t0 > kTimeoutNs) { timed_out = true; break; }
    }
  }
}

}  // namespace bak

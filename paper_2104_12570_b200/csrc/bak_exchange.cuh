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

}  // namespace bak

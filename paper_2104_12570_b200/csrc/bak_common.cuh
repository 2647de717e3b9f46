// Common device helpers for the bak200 kernels (sm_100a).
//  - PTX wrappers: mbarrier, cp.async.bulk (TMA bulk copy), st.async to a
//    cluster peer's shared memory, mapa, cluster special registers.
//  - deterministic warp sums (xor butterfly: every lane ends with the same bits)
//  - exact-rounding helpers mirroring numpy's separate multiply/subtract
//    (bak.py:87-88: scratch = col*da; e = e - scratch — two roundings, no FMA).
#pragma once
#include <cstdint>
#include <cstring>
#include <cuda_runtime.h>

#include "../../include/bak200.h"

namespace bak {

constexpr int kWarp = 32;
// spin-wait deadline: a hang must surface as BAK_ETIMEOUT, never wedge the GPU
constexpr uint64_t kTimeoutNs = 4ull * 1000 * 1000 * 1000;

template <typename T> struct Num;
template <> struct Num<double> {
  static __device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
  static __device__ __forceinline__ double sub(double a, double b) { return __dsub_rn(a, b); }
  static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
  static __device__ __forceinline__ double fma(double a, double b, double c) { return __fma_rn(a, b, c); }
  static __device__ __forceinline__ double div(double a, double b) { return __ddiv_rn(a, b); }
};
template <> struct Num<float> {
  static __device__ __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
  static __device__ __forceinline__ float sub(float a, float b) { return __fsub_rn(a, b); }
  static __device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
  static __device__ __forceinline__ float fma(float a, float b, float c) { return __fmaf_rn(a, b, c); }
  static __device__ __forceinline__ float div(float a, float b) { return __fdiv_rn(a, b); }
};

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) v = Num<T>::add(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__host__ __device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }
__host__ __device__ __forceinline__ int64_t imax64(int64_t a, int64_t b) { return a > b ? a : b; }
__host__ __device__ constexpr size_t round16(size_t v) { return (v + 15) & ~size_t(15); }

__device__ __forceinline__ uint64_t globaltimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// explicit shared-space loads (32-bit addresses, no generic->shared conversion)
template <typename T> __device__ __forceinline__ T lds(uint32_t addr);
template <> __device__ __forceinline__ double lds<double>(uint32_t addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
  return v;
}
template <> __device__ __forceinline__ float lds<float>(uint32_t addr) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
  return v;
}

// zero one element of shared memory (32-bit shared address)
template <typename T> __device__ __forceinline__ void sts_zero(uint32_t addr);
template <> __device__ __forceinline__ void sts_zero<double>(uint32_t addr) {
  asm volatile("st.shared.b64 [%0], %1;" ::"r"(addr), "l"(0ull) : "memory");
}
template <> __device__ __forceinline__ void sts_zero<float>(uint32_t addr) {
  asm volatile("st.shared.b32 [%0], %1;" ::"r"(addr), "r"(0u) : "memory");
}

// ---------------- mbarrier ----------------
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_addr(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ bool mbar_test_cluster(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_addr(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

// generic-proxy writes to shared memory made visible to the async proxy (TMA)
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
// Zero a 16-byte-aligned shared-memory range with all threads of the CTA.  The
// bulk copies of a ragged last row block never write the rows past the system's
// end, so after this the kernels read those rows as 0 with plain (unmasked)
// loads.  Call before the __syncthreads() that precedes the first bulk copy.
__device__ __forceinline__ void smem_zero(void* base, size_t bytes) {
  uint4* p = reinterpret_cast<uint4*>(base);
  const uint4 z = make_uint4(0u, 0u, 0u, 0u);
  for (size_t i = threadIdx.x; i < bytes / 16; i += blockDim.x) p[i] = z;
  fence_proxy_async_smem();
}

// ---------------- bulk copy global -> shared (TMA engine, 1-D) ----------------
// dst/src 16-byte aligned, bytes a multiple of 16.  Completion is signalled
// as transaction bytes on `bar` (this CTA's barrier).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// ---------------- cluster / DSMEM ----------------
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_size() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t mapa(uint32_t local, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
  return r;
}
// 16-byte store into a peer CTA's shared memory that completes as transaction
// bytes on the peer's mbarrier (no separate flag, no fence).
__device__ __forceinline__ void st_async_v2(uint32_t remote_addr, double v0, double v1, uint32_t remote_bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(
                   remote_addr),
               "d"(v0), "d"(v1), "r"(remote_bar)
               : "memory");
}

// ---------------- global flag slots (grid exchange) ----------------
// 16-byte "LL" record {lo32(v), epoch, hi32(v), epoch}: one vector store;
// a reader accepts it only when both epoch words match (8-byte halves are
// single-copy atomic), so value and flag arrive together.
__device__ __forceinline__ void ll_store(uint32_t* slot, double v, uint32_t epoch) {
  unsigned long long b = __double_as_longlong(v);
  uint32_t lo = static_cast<uint32_t>(b), hi = static_cast<uint32_t>(b >> 32);
  asm volatile("st.volatile.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(slot), "r"(lo), "r"(epoch), "r"(hi),
               "r"(epoch)
               : "memory");
}
__device__ __forceinline__ bool ll_load(const uint32_t* slot, uint32_t epoch, double& v) {
  uint32_t lo, e0, hi, e1;
  asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(lo), "=r"(e0), "=r"(hi), "=r"(e1)
               : "l"(slot)
               : "memory");
  v = __longlong_as_double((static_cast<long long>(hi) << 32) | lo);
  return e0 == epoch && e1 == epoch;
}
// system-scope variants for peer (NVLink) mailboxes
__device__ __forceinline__ void ll_store_sys(uint32_t* slot, double v, uint32_t epoch) {
  unsigned long long b = __double_as_longlong(v);
  uint32_t lo = static_cast<uint32_t>(b), hi = static_cast<uint32_t>(b >> 32);
  asm volatile("st.relaxed.sys.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(slot), "r"(lo), "r"(epoch), "r"(hi),
               "r"(epoch)
               : "memory");
}
__device__ __forceinline__ bool ll_load_sys(const uint32_t* slot, uint32_t epoch, double& v) {
  uint32_t lo, e0, hi, e1;
  asm volatile("ld.relaxed.sys.global.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(lo), "=r"(e0), "=r"(hi), "=r"(e1)
               : "l"(slot)
               : "memory");
  v = __longlong_as_double((static_cast<long long>(hi) << 32) | lo);
  return e0 == epoch && e1 == epoch;
}

__device__ __forceinline__ void report_error(int64_t* status, int64_t code) {
  if (status) atomicCAS(reinterpret_cast<unsigned long long*>(status + 2), 0ull,
                        static_cast<unsigned long long>(code));
}

}  // namespace bak

// ---------------- host side ----------------
namespace bak {
void set_error(const char* fmt, ...);
void g_err_clear();
int cuda_fail(cudaError_t err, const char* what);
inline size_t dtype_size(int dtype) { return dtype == BAK_F64 ? 8 : 4; }
inline int64_t round_up(int64_t v, int64_t m) { return (v + m - 1) / m * m; }
int device_sms();
int device_max_smem_optin();
int64_t l2_bytes();
bool coop_clusters_ok();
void count_launches(int n);
}  // namespace bak

#define BAK_CHECK_CUDA(expr)                           \
  do {                                                 \
    cudaError_t _e = (expr);                           \
    if (_e != cudaSuccess) return bak::cuda_fail(_e, #expr); \
  } while (0)

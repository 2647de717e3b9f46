// Streaming column pass shared by the STREAM and row-sharded kernels.
#pragma once
#include "bak_exchange.cuh"

namespace bak {

template <typename T>
struct Vec16;
template <>
struct Vec16<double> {
  using V = double2;
  static constexpr int N = 2;
  static __device__ __forceinline__ double get(const V& v, int i) { return i == 0 ? v.x : v.y; }
  static __device__ __forceinline__ void set(V& v, int i, double x) {
    if (i == 0) v.x = x; else v.y = x;
  }
};
template <>
struct Vec16<float> {
  using V = float4;
  static constexpr int N = 4;
  static __device__ __forceinline__ float get(const V& v, int i) {
    return i == 0 ? v.x : (i == 1 ? v.y : (i == 2 ? v.z : v.w));
  }
  static __device__ __forceinline__ void set(V& v, int i, float x) {
    if (i == 0) v.x = x; else if (i == 1) v.y = x; else if (i == 2) v.z = x; else v.w = x;
  }
};

struct StreamCursor {
  const int32_t* cols;
  int64_t ncols, stride, s, k;
  __device__ __forceinline__ int64_t col() const { return cols ? static_cast<int64_t>(cols[s * stride + k]) : k; }
  __device__ __forceinline__ void next() {
    if (++k == ncols) { k = 0; ++s; }
  }
};

constexpr int kUnroll = 4;

// keep_next: load x_{j+1} with the normal L2 policy (it is x_j of the next
// column step, re-read from L2 when e + one column fit in L2) and x_j with the
// evict-first hint (its last use); otherwise both evict-first.
template <typename T>
__device__ __forceinline__ void stream_pass(T* __restrict__ e, const T* __restrict__ xc, const T* __restrict__ xn,
                                            int64_t nrows, T d, bool upd, bool dot, bool sq, bool backward, T& p,
                                            T& q, bool keep_next = false) {
  using VT = Vec16<T>;
  using V = typename VT::V;
  const int NT = blockDim.x, tid = threadIdx.x;
  const int64_t nvec = nrows / VT::N;
  V* ev = reinterpret_cast<V*>(e);
  const V* xcv = reinterpret_cast<const V*>(xc);
  const V* xnv = reinterpret_cast<const V*>(xn);
  T p0 = T(0), p1 = T(0), q0 = T(0), q1 = T(0);
  const int64_t step = static_cast<int64_t>(NT) * kUnroll;
  const int64_t nfull = nvec / step * step;
  for (int64_t base = 0; base < nfull; base += step) {
    int64_t idx[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const int64_t i = base + tid + static_cast<int64_t>(u) * NT;
      idx[u] = backward ? (nvec - 1 - i) : i;
    }
    V E[kUnroll], XC[kUnroll], XN[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      E[u] = ev[idx[u]];
      if (upd) XC[u] = __ldcs(xcv + idx[u]);
      if (dot) XN[u] = keep_next ? __ldcg(xnv + idx[u]) : __ldcs(xnv + idx[u]);
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
#pragma unroll
      for (int c = 0; c < VT::N; ++c) {
        T ee = VT::get(E[u], c);
        if (upd) ee = Num<T>::sub(ee, Num<T>::mul(VT::get(XC[u], c), d));
        if (dot) {
          if (c & 1) p1 = Num<T>::fma(VT::get(XN[u], c), ee, p1);
          else p0 = Num<T>::fma(VT::get(XN[u], c), ee, p0);
        }
        if (sq) {
          if (c & 1) q1 = Num<T>::fma(ee, ee, q1);
          else q0 = Num<T>::fma(ee, ee, q0);
        }
        VT::set(E[u], c, ee);
      }
      if (upd) ev[idx[u]] = E[u];
    }
  }
  // vector remainder
  for (int64_t i0 = nfull + tid; i0 < nvec; i0 += NT) {
    const int64_t i = backward ? (nvec - 1 - i0) : i0;
    V E1 = ev[i];
    V XC1, XN1;
    if (upd) XC1 = __ldcs(xcv + i);
    if (dot) XN1 = keep_next ? __ldcg(xnv + i) : __ldcs(xnv + i);
#pragma unroll
    for (int c = 0; c < VT::N; ++c) {
      T ee = VT::get(E1, c);
      if (upd) ee = Num<T>::sub(ee, Num<T>::mul(VT::get(XC1, c), d));
      if (dot) p0 = Num<T>::fma(VT::get(XN1, c), ee, p0);
      if (sq) q0 = Num<T>::fma(ee, ee, q0);
      VT::set(E1, c, ee);
    }
    if (upd) ev[i] = E1;
  }
  // scalar tail (last CTA only)
  for (int64_t i = nvec * VT::N + tid; i < nrows; i += NT) {
    T ee = e[i];
    if (upd) ee = Num<T>::sub(ee, Num<T>::mul(xc[i], d));
    if (dot) p0 = Num<T>::fma(xn[i], ee, p0);
    if (sq) q0 = Num<T>::fma(ee, ee, q0);
    if (upd) e[i] = ee;
  }
  p = Num<T>::add(p0, p1);
  q = Num<T>::add(q0, q1);
}

}  // namespace bak

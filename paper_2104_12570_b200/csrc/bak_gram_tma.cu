// GRAM pass kernel, TMA-fed (vars <= 256): one streaming pass over x per sweep
//     e <- e - X d ,  sum e^2 ,  g <- X^T e          (see bak_gram.cu)
//
// Persistent grid, one CTA per SM = 8 consumer warps + 1 producer warp.  The
// producer streams 32-row x vars tiles of column-major x with 2-D tensor-map
// TMA (cp.async.bulk.tensor, out-of-range rows/columns zero-filled) into a
// 3-stage shared-memory ring (full/empty mbarriers).  Consumer warp c owns the
// column chunk [c*CW, (c+1)*CW), lane r owns tile row r: reads of a column
// segment are conflict-free.  Per tile: chunk partials of (X d)_r -> named
// barrier -> warp 0 finishes e_r (prefetched one tile ahead) -> named barrier
// -> every warp accumulates x_rj * e_r for its columns.  x is read from HBM
// exactly once per sweep; e once in, once out.
#include <cuda.h>
#include <cudaTypedefs.h>

#include "bak_common.cuh"
#include "bak_sweep.cuh"

namespace bak {
namespace {

constexpr int kR = 32;       // rows per tile
constexpr int kWarps = 8;    // consumer warps (= column chunks)
constexpr int kS = 3;        // ring stages
constexpr int kCons = kWarps * 32;

struct TmaPassParams {
  int64_t obs, vars, ntiles;
  void* e;
  const double* delta;
  int apply, dot;
  double* gpart;
  double* sqpart;
  const int64_t* done;
  const void* afin;  // non-null: also write resid = y - x @ afin (fused final residual, bak.py:130)
  const void* y;
  void* resid;
  int64_t* status;  // non-null: a spin wait past its deadline reports BAK_ETIMEOUT in status[2]
};

__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_addr(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_addr(bar))
      : "memory");
}

__device__ __forceinline__ void bar_cons() { asm volatile("bar.sync 1, %0;" ::"n"(kCons) : "memory"); }

__device__ __forceinline__ void mbar_arrive1(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}

// Rows per lane: fp32 tiles are 64 rows (each lane owns rows lane and
// lane+32) so that a tile carries as many bytes as an fp64 tile of 32 rows —
// the per-tile fixed costs (two named barriers, warp 0's row finish) are then
// amortised over 64 KB in both precisions (fp32 was at 70 % of HBM with
// 32-row tiles and two CTAs per SM).
template <typename T>
__host__ __device__ constexpr int rows_per_lane() { return sizeof(T) == 4 ? 2 : 1; }

template <typename T, int CW>
__global__ void __launch_bounds__(kCons + 32, 1) gram_pass_tma_kernel(const __grid_constant__ CUtensorMap xmap,
                                                                      const TmaPassParams p) {
  if (*reinterpret_cast<const volatile int64_t*>(p.done)) return;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  constexpr int RPL = rows_per_lane<T>();
  constexpr int KR = kR * RPL;     // tile rows
  constexpr int VB = CW * kWarps;  // tile columns (box width)
  constexpr uint32_t kTileBytes = KR * VB * sizeof(T);
  T* xs = reinterpret_cast<T*>(smem_raw);  // [kS][VB][KR] (column-major tile)
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + kS * kTileBytes);
  uint64_t* empty = full + kS;
  double* dsh = reinterpret_cast<double*>(empty + kS);  // [VB]
  double* red = dsh + VB;                                // [kWarps][KR]
  double* es = red + kWarps * KR;                        // [KR]
  double* ash = es + KR;                                 // [VB] final coefficients (fused residual)
  double* red2 = ash + VB;                               // [kWarps][KR]
  float* dshf = reinterpret_cast<float*>(red2 + kWarps * KR);  // [VB] fp32 copy of d (fp32 sweep passes)
  const bool want_r = p.afin != nullptr;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int V = static_cast<int>(p.vars);
  if (tid == 0) {
    for (int s = 0; s < kS; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kWarps);  // one arrive per consumer warp when it is done with the tile
    }
    fence_mbar_init();
  }
  for (int j = tid; j < VB; j += blockDim.x) {
    dsh[j] = (p.apply && j < V) ? p.delta[j] : 0.0;
    dshf[j] = static_cast<float>(dsh[j]);
    ash[j] = (want_r && j < V) ? static_cast<double>(static_cast<const T*>(p.afin)[j]) : 0.0;
  }
  __syncthreads();

  if (warp == kWarps) {
    // ------------------------------ producer ------------------------------
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      int64_t u = 0;
      for (int64_t tile = blockIdx.x; tile < p.ntiles; tile += gridDim.x, ++u) {
        if (u >= kS) {
          const uint64_t t0 = globaltimer();
          while (!mbar_test(&empty[s], ph ^ 1u))
            if (globaltimer() - t0 > kTimeoutNs) {
              report_error(p.status, BAK_ETIMEOUT);
              return;
            }
        }
        mbar_arrive_expect_tx(&full[s], kTileBytes);
        tma_2d(xs + static_cast<size_t>(s) * KR * VB, &xmap, static_cast<int>(tile * KR), 0, &full[s]);
        if (++s == kS) { s = 0; ph ^= 1u; }
      }
    }
    return;  // (consumers use named barrier 1 only; the final __syncthreads is not reached by this warp)
  }
  // ------------------------------ consumers ------------------------------
  T* e = static_cast<T*>(p.e);
  double acc[CW];
#pragma unroll
  for (int q = 0; q < CW; ++q) acc[q] = 0.0;
  double sq = 0.0;
  int s = 0;
  uint32_t ph = 0;
  int64_t tile = blockIdx.x;
  // After a timed-out wait the warp stops waiting (it keeps the named-barrier
  // schedule of the other warps, so nothing hangs) and the error is reported:
  // the results of this launch are garbage and the caller raises.
  bool timed_out = false;
  // fp32 sweep passes (apply + dot, no fused residual): x is read from shared
  // memory once per element into registers; (X d)_r runs as fp32 FMAs over the
  // warp's columns, and each column's two products of a lane (rows r, r+32)
  // are formed in fp32 and added to the fp64 accumulator — one F2F per two
  // elements instead of two per element (the conversions were the limiter:
  // fp32 pass at ~0.82x of the copy peak).  The final-residual pass and the
  // dot-only (column scoring) passes keep the fp64 products.
  constexpr bool kF32 = sizeof(T) == 4;
  const bool fast32 = kF32 && p.apply && p.dot && !want_r;
  T e_next[RPL], y_next[RPL];
  const T* yv = static_cast<const T*>(p.y);
  T* rv = static_cast<T*>(p.resid);
#pragma unroll
  for (int i = 0; i < RPL; ++i) {
    e_next[i] = T(0);
    y_next[i] = T(0);
    if (warp == 0 && tile < p.ntiles) {
      const int64_t row = tile * KR + lane + 32 * i;
      e_next[i] = row < p.obs ? e[row] : T(0);
      if (want_r) y_next[i] = row < p.obs ? yv[row] : T(0);
    }
  }
  for (; tile < p.ntiles; tile += gridDim.x) {
    T e_cur[RPL], y_cur[RPL];
#pragma unroll
    for (int i = 0; i < RPL; ++i) {
      e_cur[i] = e_next[i];
      y_cur[i] = y_next[i];
      if (warp == 0) {
        const int64_t nrow = (tile + gridDim.x) * KR + lane + 32 * i;
        const bool nok = tile + gridDim.x < p.ntiles && nrow < p.obs;
        e_next[i] = nok ? e[nrow] : T(0);
        if (want_r) y_next[i] = nok ? yv[nrow] : T(0);
      }
    }
    if (!timed_out) {
      const uint64_t t0 = globaltimer();
      while (!mbar_test(&full[s], ph))
        if (globaltimer() - t0 > kTimeoutNs) {
          timed_out = true;
          report_error(p.status, BAK_ETIMEOUT);
          break;
        }
    }
    const T* X = xs + static_cast<size_t>(s) * KR * VB + static_cast<size_t>(warp) * CW * KR + lane;
    float xr[kF32 ? RPL : 1][kF32 ? CW : 1];
    if (kF32 && fast32) {
#pragma unroll
      for (int i = 0; i < RPL; ++i) {
#pragma unroll
        for (int q = 0; q < CW; ++q) xr[kF32 ? i : 0][kF32 ? q : 0] = static_cast<float>(X[q * KR + 32 * i]);
        float t = 0.f;
#pragma unroll
        for (int q = 0; q < CW; ++q) t = __fmaf_rn(xr[kF32 ? i : 0][kF32 ? q : 0], dshf[warp * CW + q], t);
        red[warp * KR + lane + 32 * i] = static_cast<double>(t);
      }
      __syncwarp();  // the tile is in registers: hand the slot back now
      if (lane == 0) mbar_arrive1(&empty[s]);
    } else if (p.apply) {
#pragma unroll
      for (int i = 0; i < RPL; ++i) {
        double t = 0.0;
#pragma unroll
        for (int q = 0; q < CW; ++q) t = __fma_rn(static_cast<double>(X[q * KR + 32 * i]), dsh[warp * CW + q], t);
        red[warp * KR + lane + 32 * i] = t;
      }
    }
    if (want_r) {
#pragma unroll
      for (int i = 0; i < RPL; ++i) {
        double t2 = 0.0;
#pragma unroll
        for (int q = 0; q < CW; ++q) t2 = __fma_rn(static_cast<double>(X[q * KR + 32 * i]), ash[warp * CW + q], t2);
        red2[warp * KR + lane + 32 * i] = t2;
      }
    }
    bar_cons();
    if (warp == 0) {
#pragma unroll
      for (int i = 0; i < RPL; ++i) {
        const int64_t row = tile * KR + lane + 32 * i;
        double ev = static_cast<double>(e_cur[i]);
        if (p.apply) {
          double tt = 0.0;
#pragma unroll
          for (int c = 0; c < kWarps; ++c) tt += red[c * KR + lane + 32 * i];
          const T en = static_cast<T>(ev - tt);
          if (row < p.obs) e[row] = en;
          ev = static_cast<double>(en);
        }
        sq = __fma_rn(ev, ev, sq);  // (dot-only pass: sum e^2 of the unchanged e, for column scoring)
        es[lane + 32 * i] = ev;
        if (want_r && row < p.obs) {
          double r2 = 0.0;
#pragma unroll
          for (int c = 0; c < kWarps; ++c) r2 += red2[c * KR + lane + 32 * i];
          rv[row] = static_cast<T>(static_cast<double>(y_cur[i]) - r2);
        }
      }
    }
    bar_cons();
    if (kF32 && fast32) {
      float er[RPL];
#pragma unroll
      for (int i = 0; i < RPL; ++i) er[i] = static_cast<float>(es[lane + 32 * i]);  // exact: e is fp32
#pragma unroll
      for (int q = 0; q < CW; ++q) {
        float t = __fmul_rn(xr[0][kF32 ? q : 0], er[0]);
#pragma unroll
        for (int i = 1; i < RPL; ++i) t = __fmaf_rn(xr[kF32 ? i : 0][kF32 ? q : 0], er[i], t);
        acc[q] = __dadd_rn(acc[q], static_cast<double>(t));
      }
    } else if (p.dot) {
#pragma unroll
      for (int i = 0; i < RPL; ++i) {
        const double er = es[lane + 32 * i];
#pragma unroll
        for (int q = 0; q < CW; ++q) acc[q] = __fma_rn(static_cast<double>(X[q * KR + 32 * i]), er, acc[q]);
      }
    }
    if (!(kF32 && fast32)) {  // this warp's last read of the tile was the dot above
      __syncwarp();
      if (lane == 0) mbar_arrive1(&empty[s]);
    }
    if (++s == kS) { s = 0; ph ^= 1u; }
  }
  // column partials: sum over the tile rows (lanes), fixed butterfly order
  if (p.dot) {
#pragma unroll
    for (int q = 0; q < CW; ++q) {
      const double v = warp_sum(acc[q]);
      const int j = warp * CW + q;
      if (lane == q && j < V) p.gpart[static_cast<int64_t>(blockIdx.x) * V + j] = v;
    }
  }
  if (warp == 0) {
    const double v = warp_sum(sq);
    if (lane == 0) p.sqpart[blockIdx.x] = v;
  }
  bar_cons();
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
  }
  return fn;
}

template <typename T, int CW>
int launch_cw(const CUtensorMap& map, const TmaPassParams& p, int grid, cudaStream_t st) {
  constexpr int VB = CW * kWarps;
  constexpr int KR = kR * rows_per_lane<T>();
  const size_t smem = kS * static_cast<size_t>(KR) * VB * sizeof(T) + 2 * kS * 8 + 2 * VB * 8 + 2 * kWarps * KR * 8 +
                      KR * 8 + VB * 4;
  auto kern = gram_pass_tma_kernel<T, CW>;
  BAK_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  kern<<<grid, kCons + 32, smem, st>>>(map, p);
  count_launches(1);
  BAK_CHECK_CUDA(cudaGetLastError());
  return BAK_OK;
}

}  // namespace

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() { return encode_fn(); }

bool gram_tma_supported(int64_t vars) { return vars >= 1 && vars <= 256 && encode_fn() != nullptr; }

int gram_tma_grid(int dtype) {
  (void)dtype;
  return device_sms();  // one CTA per SM, 64 KB tiles in both precisions
}

// x: column-major obs x vars, ldx*sizeof(T) % 16 == 0
int launch_gram_pass_tma(int dtype, const void* x, int64_t obs, int64_t ldx, int64_t vars, void* e,
                         const double* delta, int apply, int dot, double* gpart, double* sqpart, const int64_t* done,
                         cudaStream_t st, const void* afin, const void* y, void* resid, int64_t* status) {
  auto enc = encode_fn();
  if (!enc) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return BAK_ECUDA;
  }
  const int cw = vars <= 64 ? 8 : (vars <= 128 ? 16 : 32);
  const int vb = cw * kWarps;
  const size_t ts = dtype == BAK_F64 ? 8 : 4;
  CUtensorMap map;
  cuuint64_t gdim[2] = {static_cast<cuuint64_t>(obs), static_cast<cuuint64_t>(vars)};
  cuuint64_t gstr[1] = {static_cast<cuuint64_t>(ldx * ts)};
  const int kr = kR * (dtype == BAK_F64 ? 1 : 2);  // tile rows (rows_per_lane)
  cuuint32_t box[2] = {static_cast<cuuint32_t>(kr), static_cast<cuuint32_t>(vb)};
  cuuint32_t est[2] = {1, 1};
  CUresult r = enc(&map, dtype == BAK_F64 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                   const_cast<void*>(x), gdim, gstr, box, est, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled failed (%d)", static_cast<int>(r));
    return BAK_ECUDA;
  }
  TmaPassParams p{obs, vars, (obs + kr - 1) / kr, e, delta, apply, dot, gpart, sqpart, done, afin, y, resid, status};
  const int grid = gram_tma_grid(dtype);
  if (dtype == BAK_F64) {
    if (cw == 8) return launch_cw<double, 8>(map, p, grid, st);
    if (cw == 16) return launch_cw<double, 16>(map, p, grid, st);
    return launch_cw<double, 32>(map, p, grid, st);
  }
  if (cw == 8) return launch_cw<float, 8>(map, p, grid, st);
  if (cw == 16) return launch_cw<float, 16>(map, p, grid, st);
  return launch_cw<float, 32>(map, p, grid, st);
}

}  // namespace bak

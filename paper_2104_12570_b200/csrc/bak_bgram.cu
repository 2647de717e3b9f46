// Block-Gram sweep (BAK_VARIANT_BGRAM; labelled, algebraically equal to the
// per-column sweep — SURVEY §7.4-4) for systems whose residual fits on one
// cluster and whose per-column cost is one dependent reduction (C1, C2, C4).
//
// One sweep of the reference (bak.py:92-112, cyclic order) visits columns in
// blocks B = [j0, j0+64) and, within a block, runs
//     d_j = <x_j, e_j> / n2_j,   e_{j+1} = e_j - d_j x_j
// which in exact arithmetic equals
//     g_B = X_B^T e_{j0}                     (dots against the block's first e)
//     d_B = L_B^{-1} g_B,  L_B = lower triangle of G_BB = X_B^T X_B (diag n2)
//     a_B += d_B ;  e -= X_B d_B              (per column, two roundings)
// so a block needs ONE cluster reduction of 64 values instead of 64 dependent
// ones.  M_B = L_B^{-1} (fp64, 64x64 per block, column-major) is computed once
// per solve by bgram_prep_kernel (a zero-norm column j gets row/column e_j:
// d_j = g_j = 0, the reference's skip).  g is recomputed from the current e at
// every block, so rounding in M only perturbs the iterates, not the fixed
// point; the variant is labelled and meets the same parity bar.
//
// Kernel: the on-chip layout of the column sweep — a cluster of CTAs, e in
// registers (E rows per thread, rows tid + k*NT), a producer warp streaming
// column slices with cp.async.bulk into a ring whose stage holds kW = 8
// columns (one mbarrier wait per 8 columns).  Per block: pass 1 = 64 partial
// dots (8 per stage, one 9-shuffle multi-value butterfly per warp), one
// per-column sum over warps, one st.async exchange of the 64 partial vectors
// across the cluster (rank order -> identical bits in every CTA), d = M g as a
// 64x64 matvec from shared memory (M double-buffered, one bulk copy per block
// issued by the producer ahead of the block);
// pass 2 re-reads the block (from the ring when it stays resident, else
// re-streamed from L2) and applies e -= (sum of d_j x_j over 8 columns,
// pairwise) — labelled: the reference rounds per column.
#include <cmath>
#include <cstdio>
#include <cstdlib>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "bak_common.cuh"
#include "bak_sweep.cuh"

namespace bak {
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder();  // bak_gram_tma.cu
namespace {

// one box of the 2-D tensor map of x (rows x columns; out-of-range rows and
// columns arrive as zeros) into shared memory, completing on `bar`
__device__ __forceinline__ void bg_tma_2d(void* dst, const CUtensorMap* map, int row, int col, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_addr(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(row), "r"(col), "r"(smem_addr(bar))
      : "memory");
}

constexpr int kB = 64;      // block width
constexpr int kW = 8;       // columns per ring stage (KW = 8), or the whole block (KW = 64) when 3 blocks fit
constexpr int kLG = 8;      // producer: lanes per stage of an issue group
constexpr int kMaxS = 32;   // ring stages
constexpr int kMaxNT = 256;
constexpr int kMaxCl = 16;
constexpr int kBarBG = 1;   // named barrier of the consumer warps

struct BgParams {
  const void* x;
  int64_t obs, ldx, vars;
  const double* minv;  // [nblocks][64 * 64], column-major: minv[b*4096 + k*64 + i] = M_b(i, k)
  void* e;
  void* a;
  int64_t max_iter;
  double thresh2;  // < 0: no early break
  double* history;
  int64_t* status;
  int64_t rows_per_cta;  // = NT * E
  int nstages;
  int resident;  // 1: a block's stages stay in the ring from pass 1 to pass 2 (read once)
};

__device__ __forceinline__ bool bar_bg_or(int nthreads, int pred) {
  uint32_t r;
  asm volatile(
      "{\n\t.reg .pred p, q;\n\t"
      "setp.ne.u32 q, %1, 0;\n\t"
      "bar.red.or.pred p, %2, %3, q;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(r)
      : "r"(static_cast<uint32_t>(pred)), "r"(kBarBG), "r"(nthreads)
      : "memory");
  return r != 0;
}
__device__ __forceinline__ void arrive1(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void st_async_d(uint32_t remote_addr, double v, uint32_t remote_bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(remote_addr),
               "d"(v), "r"(remote_bar)
               : "memory");
}

#ifdef BAK_PHASES
#define GPH(i)                                 \
  do {                                         \
    if (tid == 0) {                            \
      const long long _c = clock64();          \
      ph_acc[i] += _c - ph_last;               \
      ph_last = _c;                            \
    }                                          \
  } while (0)
#else
#define GPH(i) \
  do {         \
  } while (0)
#endif

// E <= 4 keeps 64 partial dots per thread in registers: at most 7 warps
// (192 consumers + producer) so a thread may use up to 255 registers (9 warps
// cap it at 168: the E = 1, 2 plans spilled)
// whole-block stages (KW = 64) unroll 64 columns per pass: at most 128 consumers, so
// a thread may use up to 255 registers (288 threads cap it at 168: spills)
constexpr int bg_max_threads(int kw) { return kw == 64 ? 128 + 32 : kMaxNT + 32; }
constexpr int kMaxSeg = kMaxNT / kW;  // row segments of pass 1 (KW column threads per segment)

template <typename T, int E, bool CL, int KW>
__global__ void __launch_bounds__(bg_max_threads(KW), 1) bgram_kernel(const __grid_constant__ CUtensorMap xmap,
                                                                      const BgParams prm) {
  constexpr int CB = E <= 4 ? 8 : (E <= 8 ? 4 : 2);  // columns whose slices are loaded together
#ifdef BAK_PHASES
  long long ph_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long ph_last = clock64();
#endif
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int NT = static_cast<int>(blockDim.x) - 32;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = NT >> 5;
  const int S = prm.nstages;
  uint32_t rank = 0, G = 1;
  if (CL) {
    rank = cluster_rank();
    G = cluster_size();
  }
  T* __restrict__ eg = static_cast<T*>(prm.e);
  T* __restrict__ ag = static_cast<T*>(prm.a);
  const int64_t V = prm.vars;
  const int64_t nblocks = (V + kB - 1) / kB;
  const int64_t RP = prm.rows_per_cta;
  const int64_t r0 = static_cast<int64_t>(rank) * RP;
  const int64_t nrows = imax64(0, imin64(prm.obs - r0, RP));
  // ---- shared memory ----
  // ring stage = kW columns of the CTA's NT * E rows as E boxes of the tensor
  // map: [S][E][kW][NT].  Box k holds rows r0 + k NT .. of the stage's 8
  // columns; rows past obs and columns past vars arrive as zeros, so no load in
  // the passes is masked and every stage carries the same byte count.
  size_t off = 0;
  const uint32_t box_elems = static_cast<uint32_t>(KW) * NT;
  const uint32_t stage_elems = box_elems * E;
  T* xs = reinterpret_cast<T*>(smem_raw);
  off += static_cast<size_t>(S) * stage_elems * sizeof(T);
  T* esh = reinterpret_cast<T*>(smem_raw + off);  // [NT * E] the residual, for pass 1 (pass 2 keeps it in registers)
  off += static_cast<size_t>(NT) * E * sizeof(T);
  off = (off + 127) & ~size_t(127);
  double* msh = reinterpret_cast<double*>(smem_raw + off);  // [2][64*64] M of the current / next block
  off += 2 * kB * kB * sizeof(double);
  double* xslot = reinterpret_cast<double*>(smem_raw + off);  // [2][kMaxCl][kB] exchange
  off += 2 * kMaxCl * kB * sizeof(double);
  double* gsh = reinterpret_cast<double*>(smem_raw + off);  // [kB] block dots (cluster totals)
  off += kB * sizeof(double);
  T* dsh = reinterpret_cast<T*>(smem_raw + off);  // [kB] block deltas
  off += kB * sizeof(T);
  off = (off + 15) & ~size_t(15);
  T* red = reinterpret_cast<T*>(smem_raw + off);  // [kB][kMaxSeg] per-segment partial dots
  off += kB * kMaxSeg * sizeof(T);
  off = (off + 15) & ~size_t(15);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + off);
  off += kMaxS * 8;
  uint64_t* empty = reinterpret_cast<uint64_t*>(smem_raw + off);
  off += kMaxS * 8;
  uint64_t* xbar = reinterpret_cast<uint64_t*>(smem_raw + off);  // [2]
  off += 16;
  uint64_t* mfull = reinterpret_cast<uint64_t*>(smem_raw + off);  // [2] M buffer landed
  off += 16;
  uint64_t* mempty = reinterpret_cast<uint64_t*>(smem_raw + off);  // [2] M buffer read by the matvec
  off += 16;
  double* qsh = reinterpret_cast<double*>(smem_raw + off);
  off += 16;
  volatile int* stop = reinterpret_cast<volatile int*>(smem_raw + off);

  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], nwarps);
    }
    mbar_init(&xbar[0], 1);
    mbar_init(&xbar[1], 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&mfull[i], 1);
      mbar_init(&mempty[i], 1);
    }
    *stop = 0;
    fence_mbar_init();
  }
  __syncthreads();
  if (CL) cluster_sync();

  // stages of one block: ceil(width / kW); each block is streamed twice
  auto block_w = [&](int64_t b) -> int { return static_cast<int>(imin64(kB, V - b * kB)); };

  if (tid >= NT) {
    // =========================== producer warp ===========================
    // One tensor copy per box (NT rows x 8 columns): E copies per stage instead
    // of one bulk copy per column slice — the TMA unit retires a copy every
    // ~70-110 cycles whatever its size (tools/micro/bulk_rate.cu), and 64-128
    // column copies per block were the floor of the whole sweep.  The whole warp
    // issues: a group is up to 4 stages; lane l serves stage l / 8 of the group
    // and boxes l % 8 and l % 8 + 8 of it; the first lane of a stage waits for
    // the slot and posts the stage's bytes.
    {
      int64_t u = 0;  // stages issued
      bool halted = false;
      int64_t mb = 0;  // blocks whose M has been issued
      const uint64_t pol = policy_evict_last();
      const uint32_t stage_bytes = stage_elems * static_cast<uint32_t>(sizeof(T));
      for (int64_t sw = 0; sw < prm.max_iter && !halted; ++sw)
        for (int64_t b = 0; b < nblocks && !halted; ++b)
          for (int pass = 0; pass < (prm.resident ? 1 : 2) && !halted; ++pass) {
            const int w = block_w(b);
            if (pass == 0) {
              // the block's M (32 KB, one bulk copy) into buffer mb & 1, once the
              // matvec two blocks back has read it
              const int mbuf = static_cast<int>(mb & 1);
              if (lane == 0) {
                if (mb >= 2) {
                  const uint32_t par = static_cast<uint32_t>(((mb >> 1) - 1) & 1);
                  if (!mbar_test(&mempty[mbuf], par)) {
                    const uint64_t t0 = globaltimer();
                    while (!mbar_test(&mempty[mbuf], par)) {
                      if (*stop || globaltimer() - t0 > kTimeoutNs) { halted = true; break; }
                    }
                  }
                }
                if (!halted) {
                  mbar_arrive_expect_tx(&mfull[mbuf], kB * kB * 8u);
                  bulk_g2s(msh + mbuf * kB * kB, prm.minv + b * kB * kB, kB * kB * 8u, &mfull[mbuf], pol);
                }
              }
              halted = __any_sync(0xffffffffu, halted);
              if (halted) break;
              ++mb;
            }
            const int nst = (w + KW - 1) / KW;
            // (a group never spans more stages than the ring has slots: two of its
            // stages would wait on the same slot)
            const int gmax = S < 4 ? S : 4;
            for (int s0 = 0; s0 < nst && !halted; s0 += gmax) {
              const int gst = nst - s0 < gmax ? nst - s0 : gmax;  // stages in this group
              const int j = lane / kLG, k8 = lane % kLG;
              const int64_t uj = u + j;
              const int sj = static_cast<int>(uj % S);
              const uint32_t phj = static_cast<uint32_t>((uj / S) & 1);
              if (j < gst && k8 == 0) {
                if (uj >= S) {
                  const uint32_t par = phj ^ 1u;
                  if (!mbar_test(&empty[sj], par)) {
                    const uint64_t t0 = globaltimer();
                    while (!mbar_test(&empty[sj], par)) {
                      if (*stop || globaltimer() - t0 > kTimeoutNs) { halted = true; break; }
                    }
                  }
                }
                if (!halted) mbar_arrive_expect_tx(&full[sj], stage_bytes);
              }
              halted = __any_sync(0xffffffffu, halted);
              if (halted) break;
              if (j < gst) {
                const int col = static_cast<int>(b * kB) + (s0 + j) * KW;
                for (int k = k8; k < E; k += kLG)
                  bg_tma_2d(xs + static_cast<size_t>(sj) * stage_elems + static_cast<size_t>(k) * box_elems, &xmap,
                            static_cast<int>(r0) + k * NT, col, &full[sj]);
              }
              u += gst;
            }
          }
      if (lane == 0) {
        for (int64_t v = imax64(0, u - S); v < u; ++v) {  // in-flight copies land before exit
          const uint64_t t0 = globaltimer();
          while (!mbar_test(&full[v % S], static_cast<uint32_t>((v / S) & 1)))
            if (globaltimer() - t0 > kTimeoutNs) break;
        }
        for (int64_t v = imax64(0, mb - 2); v < mb; ++v) {  // and the last two M copies
          const uint64_t t0 = globaltimer();
          while (!mbar_test(&mfull[v & 1], static_cast<uint32_t>((v >> 1) & 1)))
            if (globaltimer() - t0 > kTimeoutNs) break;
        }
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
    const uint32_t xs_base = smem_addr(xs) + static_cast<uint32_t>(tid * sizeof(T));
    const uint32_t col_stride = static_cast<uint32_t>(NT * sizeof(T));        // next column of a box
    const uint32_t k_stride = box_elems * static_cast<uint32_t>(sizeof(T));   // next box (rows + NT)
    const uint32_t stage_stride = stage_elems * static_cast<uint32_t>(sizeof(T));
    auto wait_stage = [&]() -> uint32_t {
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
      return xs_base + static_cast<uint32_t>(ls) * stage_stride;
    };
    auto release_stage = [&]() {
      __syncwarp();
      if (lane == 0) arrive1(&empty[ls]);
      if (++ls == S) { ls = 0; lph ^= 1u; }
    };
    auto xval = [&](uint32_t a, int k) -> T { return lds<T>(a + static_cast<uint32_t>(k) * k_stride); };
    // cluster sum of n values (thread t < n holds v), rank order; result in t < n
    uint32_t rc = 0;
    auto exchange = [&](double v, int n) -> double {
      if (!CL) return v;
      const int buf = rc & 1;
      const uint32_t par = (rc >> 1) & 1;
      ++rc;
      if (tid < n) {
        const uint32_t loc = smem_addr(&xslot[(buf * kMaxCl + rank) * kB + tid]);
        const uint32_t lb = smem_addr(&xbar[buf]);
        for (uint32_t r = 0; r < G; ++r) st_async_d(mapa(loc, r), v, mapa(lb, r));
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
        double s = 0.0;
        for (uint32_t r = 0; r < G; ++r) s += xslot[(buf * kMaxCl + r) * kB + tid];
        tot = s;
      }
      return tot;
    };

    int64_t sweep = 0;
    bool converged = false, aborted = false;
    int64_t mi = 0;  // blocks consumed (M buffer mi & 1)
    if (tid < kB) gsh[tid] = 0.0;  // (finite before the first block; see the matvec)
    const int nseg = NT / KW;  // pass 1: KW column threads per run of KW rows
    auto publish_e = [&]() {  // registers -> esh (read by the column threads of the next pass 1)
#pragma unroll
      for (int k = 0; k < E; ++k) esh[tid + k * NT] = ev[k];
    };
    publish_e();
    while (sweep < prm.max_iter && !aborted) {
      for (int64_t b = 0; b < nblocks && !aborted; ++b) {
        const int w = block_w(b);
        // ---- pass 1: dots of the block's columns against e.  Stage by stage
        // (8 columns): thread t takes column t % 8 of the stage and, in every
        // box k, the 8 rows k NT + 8 (t / 8) .. — E runs of 8 products from
        // shared memory (x from the ring, e from esh), no cross-lane reduction;
        // the NT / 8 segment partials of a column are summed in segment order
        // below.  A box column is NT rows = a multiple of 256 bytes, so the 8
        // column threads of a segment would hit one bank: thread c8 walks its 8
        // rows starting at row c8 (rotated, a fixed per-thread order) ----
        const int ls_block = ls;  // resident: pass 2 re-reads these stages
        // the block's coefficients, read now: the load's latency is off the path
        // (a load right before the store stalled CTA 0 for an L2 round trip per block)
        const T a_old = (rank == 0 && tid < w) ? ag[b * kB + tid] : T(0);
        if (bar_bg_or(NT, my_abort)) { aborted = true; break; }  // esh holds every thread's e
        {
          // thread -> column c8 of the stage and run `seg` of KW rows in every box;
          // it walks the run starting at row c8 (rotated): the KW column threads of a
          // run read KW different rows, i.e. different banks
          const int c8 = tid & (KW - 1), seg = tid / KW;
          const uint32_t rbase = static_cast<uint32_t>(seg * KW * sizeof(T));
          const uint32_t eb = smem_addr(esh) + rbase;
          for (int c0 = 0; c0 < w; c0 += KW) {
            wait_stage();
            const uint32_t xb = smem_addr(xs) + static_cast<uint32_t>(ls) * stage_stride + c8 * col_stride + rbase;
            T acc[4] = {T(0), T(0), T(0), T(0)};
            if (seg < nseg) {
#pragma unroll
              for (int k = 0; k < E; ++k) {
#pragma unroll
                for (int i0 = 0; i0 < KW; i0 += 8) {
                  T xv[8], evv[8];
#pragma unroll
                  for (int i = 0; i < 8; ++i) {
                    const uint32_t ro = static_cast<uint32_t>(((i0 + i + c8) & (KW - 1)) * sizeof(T));
                    xv[i] = lds<T>(xb + static_cast<uint32_t>(k) * k_stride + ro);
                    evv[i] = lds<T>(eb + static_cast<uint32_t>(k * NT * sizeof(T)) + ro);
                  }
#pragma unroll
                  for (int i = 0; i < 8; ++i) acc[i & 3] = Num<T>::fma(xv[i], evv[i], acc[i & 3]);
                }
              }
              red[(c0 + c8) * kMaxSeg + seg] = Num<T>::add(Num<T>::add(acc[0], acc[1]), Num<T>::add(acc[2], acc[3]));
            }
            if (prm.resident) {
              if (++ls == S) { ls = 0; lph ^= 1u; }
            } else {
              release_stage();
            }
          }
        }
        GPH(0);
        if (bar_bg_or(NT, my_abort)) { aborted = true; break; }
        GPH(1);
        double v = 0.0;
        if (tid < w) {
          T s = T(0);
          for (int sg = 0; sg < nseg; ++sg) s = Num<T>::add(s, red[tid * kMaxSeg + sg]);
          v = static_cast<double>(s);
        }
        const double g = exchange(v, w);
        if (tid < w) gsh[tid] = g;
        GPH(2);
        const int mbuf = static_cast<int>(mi & 1);
        const uint32_t mpar = static_cast<uint32_t>((mi >> 1) & 1);
        if (tid < kB && !mbar_test(&mfull[mbuf], mpar)) {
          const uint64_t t0 = globaltimer();
          while (!mbar_test(&mfull[mbuf], mpar)) {
            if (globaltimer() - t0 > kTimeoutNs) {
              report_error(prm.status, BAK_ETIMEOUT);
              my_abort = 1;
              break;
            }
          }
        }
        if (bar_bg_or(NT, my_abort)) { aborted = true; break; }
        GPH(3);
        // ---- d = M g (fp64, four interleaved partial sums), a += d ----
        if (tid < w) {
          const double* mcol = msh + mbuf * kB * kB + tid;
          double dp[4] = {0.0, 0.0, 0.0, 0.0};
          // all 64 terms: past a ragged block's width M(i, k) = 0 and gsh[k] is finite
#pragma unroll
          for (int k = 0; k < kB; ++k) dp[k & 3] = __fma_rn(mcol[k * kB], gsh[k], dp[k & 3]);
          const T dt = static_cast<T>((dp[0] + dp[1]) + (dp[2] + dp[3]));
          dsh[tid] = dt;
          if (rank == 0) ag[b * kB + tid] = Num<T>::add(a_old, dt);
        } else if (tid < kB) {
          dsh[tid] = T(0);  // past a ragged last block: its (zero-filled) columns change nothing
        }
        if (bar_bg_or(NT, my_abort)) { aborted = true; break; }
        if (tid == 0) arrive1(&mempty[mbuf]);  // every matvec read is before the barrier
        ++mi;
        GPH(4);
        // ---- pass 2: e -= fl(d_j x_j), column by column (two roundings, bak.py:87-88) ----
        int s2 = ls_block;
        for (int c0 = 0; c0 < w; c0 += KW) {
          const uint32_t a = prm.resident ? xs_base + static_cast<uint32_t>(s2) * stage_stride : wait_stage();
#pragma unroll
          for (int cb = 0; cb < KW; cb += CB) {
            T xr[CB][E], dd[CB];
#pragma unroll
            for (int c = 0; c < CB; ++c) {
              dd[c] = dsh[c0 + cb + c];  // 0 past a ragged block's width, where x is zero-filled too
#pragma unroll
              for (int k = 0; k < E; ++k) xr[c][k] = xval(a + (cb + c) * col_stride, k);
            }
            // e -= (sum of the CB products, pairwise tree) — a short dependency chain
            // instead of 2 CB dependent ops per row (labelled variant: the rounding
            // is not the reference's per-column one)
#pragma unroll
            for (int k = 0; k < E; ++k) {
              T pr[CB];
#pragma unroll
              for (int c = 0; c < CB; ++c) pr[c] = Num<T>::mul(xr[c][k], dd[c]);
#pragma unroll
              for (int h = CB / 2; h >= 1; h >>= 1)
#pragma unroll
                for (int c = 0; c < h; ++c) pr[c] = Num<T>::add(pr[c], pr[c + h]);
              ev[k] = Num<T>::sub(ev[k], pr[0]);
            }
          }
          if (prm.resident) {
            __syncwarp();
            if (lane == 0) arrive1(&empty[s2]);
            if (++s2 == S) s2 = 0;
          } else {
            release_stage();
          }
        }
        publish_e();
        GPH(5);
      }
      if (aborted) break;
      // ---- sweep end: sum e^2, history, early break (bak.py:106-111) ----
      T q[4] = {T(0), T(0), T(0), T(0)};
#pragma unroll
      for (int k = 0; k < E; ++k) q[k & 3] = Num<T>::fma(ev[k], ev[k], q[k & 3]);
      const T qv = warp_sum(Num<T>::add(Num<T>::add(q[0], q[1]), Num<T>::add(q[2], q[3])));
      if (lane == 0) red[warp] = qv;
      if (bar_bg_or(NT, my_abort)) break;
      double qd = 0.0;
      if (tid == 0) {
        T s = T(0);
        for (int ww = 0; ww < nwarps; ++ww) s = Num<T>::add(s, red[ww]);
        qd = static_cast<double>(s);
      }
      qd = exchange(qd, 1);
      if (tid == 0) {
        *qsh = qd;
        if (rank == 0 && prm.history) prm.history[sweep] = qd;
      }
      if (bar_bg_or(NT, my_abort)) break;
      const double sq = *qsh;
      ++sweep;
      if (prm.thresh2 >= 0.0 && sq <= prm.thresh2) {
        converged = true;
        break;
      }
    }
    {
      T* ew = eg + r0 + tid;
      asm volatile("mov.b64 %0, %0;" : "+l"(ew));
#pragma unroll
      for (int k = 0; k < E; ++k)
        if (k < kv) ew[static_cast<int64_t>(k) * NT] = ev[k];
    }
#ifdef BAK_PHASES
    if (tid == 0 && rank == 0 && prm.history)
      for (int i = 0; i < 8; ++i) prm.history[prm.max_iter + i] = static_cast<double>(ph_acc[i]);
#endif
    if (tid == 0) {
      *stop = 1;
      if (rank == 0 && prm.status) {
        prm.status[0] = sweep;
        prm.status[1] = converged ? 1 : 0;
        prm.status[3] = BAK_VARIANT_BGRAM;
      }
    }
  }
  __syncthreads();
  if (CL) cluster_sync();
}

// M_b = L_b^{-1} for every 64-column block b: G_BB = X_B^T X_B in fp64 (rows in
// 32-row tiles, fixed order), L = its lower triangle, inverted column by
// column by forward substitution (thread j solves L m = e_j).  A zero-norm
// column j (L_jj == 0) gets row and column e_j.
template <typename T>
__global__ void __launch_bounds__(256) bgram_prep_kernel(const T* __restrict__ x, int64_t obs, int64_t ldx,
                                                         int64_t vars, double* __restrict__ minv) {
  __shared__ double buf[kB * (kB + 1)];  // the row tile, later L (after the accumulation)
  double (*xt)[kB + 1] = reinterpret_cast<double (*)[kB + 1]>(buf);  // [32][65]: [row][column]
  double (*L)[kB + 1] = reinterpret_cast<double (*)[kB + 1]>(buf);   // [64][65]: [i][j]
  const int64_t b = blockIdx.x;
  const int w = static_cast<int>(imin64(kB, vars - b * kB));
  const int tid = threadIdx.x;
  const int ti = tid / 16, tj = tid % 16;  // 4x4 outputs: rows 4ti.., cols 4tj..
  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;
  for (int64_t r0 = 0; r0 < obs; r0 += 32) {
    __syncthreads();
    for (int idx = tid; idx < 32 * kB; idx += 256) {
      const int c = idx / 32, r = idx % 32;  // coalesced along rows of a column
      const int64_t row = r0 + r;
      xt[r][c] = (c < w && row < obs) ? static_cast<double>(x[(b * kB + c) * ldx + row]) : 0.0;
    }
    __syncthreads();
#pragma unroll 4
    for (int r = 0; r < 32; ++r) {
      double xi[4], xj[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        xi[i] = xt[r][4 * ti + i];
        xj[i] = xt[r][4 * tj + i];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = __fma_rn(xi[i], xj[j], acc[i][j]);
    }
  }
  __syncthreads();  // done with the row tiles: the buffer becomes L
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int gi = 4 * ti + i, gj = 4 * tj + j;
      L[gi][gj] = (gj <= gi) ? acc[i][j] : 0.0;
    }
  __syncthreads();
  if (tid < kB) {
    const int j = tid;
    double m[kB];  // column j of M
    for (int i = 0; i < kB; ++i) {
      if (i < j) {
        m[i] = 0.0;
        continue;
      }
      double s = (i == j) ? 1.0 : 0.0;
      for (int k = j; k < i; ++k) s = __fma_rn(-L[i][k], m[k], s);
      const double lii = L[i][i];
      m[i] = (lii != 0.0) ? s / lii : ((i == j) ? 1.0 : 0.0);
      if (lii == 0.0 && i != j) m[i] = 0.0;
    }
    // a zero-norm column i: row i of M = e_i^T (d_i = g_i = 0); L's column i is 0 already
    double* out = minv + b * kB * kB;
    for (int i = 0; i < kB; ++i) out[j * kB + i] = m[i];  // column-major: out[k*64 + i] = M(i, k), k = j
  }
}

struct BgPlan {
  int parts = 1, nt = 64, e = 1, nstages = 2, resident = 0;
  int kw = kW;  // columns per ring stage: 8, or 64 (a whole block per stage) when >= 3 blocks fit
  int64_t rows_per_cta = 0;  // = nt * e
};

size_t bg_smem(const BgPlan& p, size_t ts) {
  size_t off = static_cast<size_t>(p.nstages) * p.e * p.kw * p.nt * ts + static_cast<size_t>(p.nt) * p.e * ts;
  off = (off + 127) & ~size_t(127);
  off += 2 * kB * kB * 8 + 2 * kMaxCl * kB * 8 + kB * 8 + kB * ts;
  off = (off + 15) & ~size_t(15);
  off += kB * kMaxSeg * ts;
  off = (off + 15) & ~size_t(15);
  return off + 2 * kMaxS * 8 + 16 + 16 + 16 + 32;
}

bool bg_plan(int dtype, int64_t obs, BgPlan& pl) {
  if (!tensor_map_encoder() || obs >= (int64_t(1) << 31)) return false;
  const size_t ts = dtype_size(dtype);
  const size_t cap = static_cast<size_t>(device_max_smem_optin()) - 2048;
  // as many CTAs as a cluster allows (bandwidth), at least 64 rows each; row
  // blocks of exactly nt * e rows (box k of a stage = rows k nt .. of the block)
  int64_t per = (obs + kMaxCl - 1) / kMaxCl;
  if (per < 64) per = 64;
  // fewest rows per thread first: the passes are latency-bound, so more warps
  // win; BAK_BGRAM_E forces one
  const char* e_env = getenv("BAK_BGRAM_E");
  const int e_only = e_env ? atoi(e_env) : 0;
  for (int e : {1, 2, 4, 8, 16}) {
    if (e_only && e != e_only) continue;
    int64_t nt = round_up((per + e - 1) / e, 32);
    if (nt < kB) nt = kB;  // threads t < 64 finish the block's 64 dots and deltas
    if (nt > kMaxNT) continue;
    // 8 consumer warps of 1 row per thread measured 4 % slower than 4 warps of 2 (C2)
    if (e == 1 && nt > 128 && !e_only) continue;
    BgPlan c;
    c.nt = static_cast<int>(nt);
    c.e = e;
    c.rows_per_cta = nt * e;
    c.parts = static_cast<int>((obs + c.rows_per_cta - 1) / c.rows_per_cta);
    if (c.parts > kMaxCl) continue;
    c.nstages = 0;
    const size_t fixed = bg_smem(c, ts);
    // a whole block per stage (one wait and one release per pass instead of 8)
    // when the ring holds 3 blocks (short columns: C4)
    const char* kw_env = getenv("BAK_BGRAM_KW");
    const size_t sb64 = static_cast<size_t>(e) * kB * nt * ts;
    c.kw = (e <= 4 && nt <= 128 && fixed + 3 * sb64 <= cap && nt % kB == 0 && !(kw_env && atoi(kw_env) == kW))
               ? kB
               : kW;
    const size_t sb = static_cast<size_t>(e) * c.kw * nt * ts;
    if (fixed + 3 * sb > cap) continue;
    int s = static_cast<int>((cap - fixed) / sb);
    c.nstages = s > kMaxS ? kMaxS : s;
    // a block stays resident between its passes when the ring also holds at
    // least one more block's worth of prefetch
    c.resident = c.nstages >= 2 * (kB / c.kw) ? 1 : 0;
    if (const char* r = getenv("BAK_BGRAM_RESIDENT")) c.resident = (r[0] == '1') && c.nstages > kB / c.kw;
    pl = c;
    return true;
  }
  return false;
}

template <typename T, int E, bool CL, int KW>
int bg_launch_kw(const BgPlan& pl, const BgParams& prm, cudaStream_t st) {
  // x as a 2-D tensor (rows, columns); a box is nt rows x KW columns
  CUtensorMap map;
  cuuint64_t gdim[2] = {static_cast<cuuint64_t>(prm.obs), static_cast<cuuint64_t>(prm.vars)};
  cuuint64_t gstr[1] = {static_cast<cuuint64_t>(prm.ldx * sizeof(T))};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(pl.nt), static_cast<cuuint32_t>(KW)};
  cuuint32_t est[2] = {1, 1};
  CUresult r = tensor_map_encoder()(
      &map, sizeof(T) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
      const_cast<void*>(prm.x), gdim, gstr, box, est, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    set_error("cuTensorMapEncodeTiled (x, block-Gram) failed (%d)", static_cast<int>(r));
    return BAK_ECUDA;
  }
  auto kern = bgram_kernel<T, E, CL, KW>;
  const size_t smem = bg_smem(pl, sizeof(T));
  BAK_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(pl.parts);
  cfg.blockDim = dim3(pl.nt + 32);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  int na = 0;
  if (CL) {
    if (pl.parts > 8) BAK_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = pl.parts;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  BAK_CHECK_CUDA(cudaLaunchKernelEx(&cfg, kern, map, prm));
  count_launches(1);
  return BAK_OK;
}

template <typename T, int E, bool CL>
int bg_launch(const BgPlan& pl, const BgParams& prm, cudaStream_t st) {
  if constexpr (E <= 4) {
    if (pl.kw == kB) return bg_launch_kw<T, E, CL, kB>(pl, prm, st);
  }
  return bg_launch_kw<T, E, CL, kW>(pl, prm, st);
}

template <typename T>
int bg_launch_e(const BgPlan& pl, const BgParams& prm, cudaStream_t st) {
  const bool cl = pl.parts > 1;
  switch (pl.e) {
    case 1: return cl ? bg_launch<T, 1, true>(pl, prm, st) : bg_launch<T, 1, false>(pl, prm, st);
    case 2: return cl ? bg_launch<T, 2, true>(pl, prm, st) : bg_launch<T, 2, false>(pl, prm, st);
    case 4: return cl ? bg_launch<T, 4, true>(pl, prm, st) : bg_launch<T, 4, false>(pl, prm, st);
    case 8: return cl ? bg_launch<T, 8, true>(pl, prm, st) : bg_launch<T, 8, false>(pl, prm, st);
    case 16: return cl ? bg_launch<T, 16, true>(pl, prm, st) : bg_launch<T, 16, false>(pl, prm, st);
  }
  set_error("bak_sweep(BGRAM): unsupported rows per thread %d", pl.e);
  return BAK_EUNSUPPORTED;
}

}  // namespace

int64_t bgram_workspace_bytes(int64_t vars) { return ((vars + kB - 1) / kB) * kB * kB * 8 + 256; }

bool bgram_supported(int dtype, int64_t obs) {
  BgPlan pl;
  return bg_plan(dtype, obs, pl);
}

int launch_bgram(int dtype, const SweepParams& prm, int64_t vars, void* ws, int64_t wsb, cudaStream_t st) {
  if (prm.cols && prm.cols_stride != 0) {
    set_error("bak_sweep(BGRAM): cyclic ordering only (blocks of 64 consecutive columns)");
    return BAK_EUNSUPPORTED;
  }
  BgPlan pl;
  if (!bg_plan(dtype, prm.obs, pl)) {
    set_error("bak_sweep(BGRAM): obs=%lld does not fit one cluster", (long long)prm.obs);
    return BAK_EUNSUPPORTED;
  }
  if (wsb < bgram_workspace_bytes(vars)) {
    set_error("bak_sweep(BGRAM): workspace too small (need %lld)", (long long)bgram_workspace_bytes(vars));
    return BAK_EWORKSPACE;
  }
  double* minv = static_cast<double*>(ws);
  const unsigned nb = static_cast<unsigned>((vars + kB - 1) / kB);
  if (dtype == BAK_F64)
    bgram_prep_kernel<double><<<nb, 256, 0, st>>>(static_cast<const double*>(prm.x), prm.obs, prm.ldx, vars, minv);
  else
    bgram_prep_kernel<float><<<nb, 256, 0, st>>>(static_cast<const float*>(prm.x), prm.obs, prm.ldx, vars, minv);
  count_launches(1);
  BAK_CHECK_CUDA(cudaGetLastError());
  BAK_CHECK_CUDA(cudaMemsetAsync(prm.status, 0, 4 * sizeof(int64_t), st));
  BgParams bp{prm.x, prm.obs, prm.ldx, vars, minv, prm.e, prm.a, prm.max_iter, prm.thresh2, prm.history,
              prm.status, pl.rows_per_cta, pl.nstages, pl.resident};
  const int rc = dtype == BAK_F64 ? bg_launch_e<double>(pl, bp, st) : bg_launch_e<float>(pl, bp, st);
  if (rc) return rc;
  BAK_CHECK_CUDA(cudaGetLastError());
  return BAK_OK;
}

}  // namespace bak

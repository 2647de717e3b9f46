// G = X^T X for the GRAM variant: hand-written fp64 tensor-core (DMMA,
// mma.sync.m8n8k4.f64) SYRK over column-major x, fp64 accumulation for both
// input precisions (fp32 inputs are widened exactly when fragments are read).
//
// Only the lower block triangle of 64x64 blocks is computed (bi >= bj), split
// over K (rows of x) into chunks; a CTA = 4 warps owns one (block, chunk) and
// each warp a 32x32 quarter = 4x4 DMMA tiles.  Panels of 32 rows x 64 columns
// stream through a 2-stage cp.async ring (16-row stages, zero-filled past obs /
// vars), 4 CTAs per SM in one wave; panel layout is column-major with a
// (stage rows + 4)-element column stride for the m8n8k4 fragment loads.  Partials per chunk are summed in chunk order
// (deterministic) and mirrored.  Diagonal-block CTAs optionally also produce
// the first sweep's g = X^T e (warp 1, whose quarter of a diagonal block is
// unused), so the solve skips its first pass over x.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>

#include "bak_common.cuh"
#include "bak_sweep.cuh"

namespace bak {

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder();  // bak_gram_tma.cu

namespace {

constexpr int kBT = 64;       // G block edge
constexpr int kKT = 32;       // rows per panel stage
constexpr int kLd = 36;       // smem column stride (elements)
constexpr int kThreads = 128;

__device__ __forceinline__ void cp_async16(void* dst, const void* src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_addr(dst)), "l"(src), "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// 3xTF32 (fp32 inputs only): v = hi + lo with hi = RN_tf32(v), lo = v - hi
// (exact in fp32); a*b ~ lo_a*hi_b + hi_a*lo_b + hi_a*hi_b, each
// product exact in the tensor core, accumulated in fp32 over a few stages and
// then flushed into fp64 — G to ~2^-21 relative, on the legacy tf32 MMA path
// (277.6 TFLOP/s measured, tools/micro/tf32_peak.cu, vs 37.2 for fp64 DMMA)
__device__ __forceinline__ void split_tf32(float v, uint32_t& hi, uint32_t& lo) {
  // hi: v rounded to tf32 (|lo| <= 2^-11 |v|); lo: the exact remainder, whose
  // low 13 bits the tf32 datapath ignores (~2^-22 of v), as does the dropped
  // lo*lo product
  uint32_t h;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(h) : "f"(v));
  hi = h;
  lo = __float_as_uint(v - __uint_as_float(h));
}

__device__ __forceinline__ void mma_tf32(float (&d)[4], const uint32_t (&a)[4], const uint32_t (&b)[2]) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
}

struct GramParams {
  const void* x;
  int64_t obs, ldx, vars;
  int nb;                       // number of 64-column blocks
  int cd, co;                   // K chunks per diagonal / off-diagonal block
  int64_t chunk_d, chunk_o;     // rows per chunk (multiples of kKT)
  double* part;                 // [nb*cd + noff*co][64*64], diagonal CTAs first
  const void* e;                // optional: fused g0 = X^T e in the diagonal CTAs
  double* g0;                   // [cd][vars] per-chunk partials of X^T e
  int* pace;                    // optional: one step counter per CTA (advisory lock step, see below)
  int64_t* status;              // optional: BAK_ETIMEOUT from the TMA-fed kernel's barrier waits
  int pace_offdiag_only;        // lock step among the off-diagonal CTAs of a chunk only (diagonal CTAs run free)
  int units;                    // TMA kernel: 1 = two units (off-diagonal, then diagonal) per CTA
};

// off-diagonal block index -> (bi, bj), bi > bj, row-major over the strict lower triangle
__device__ __forceinline__ void tri_index_strict(int o, int& bi, int& bj) {
  bi = 1;
  while ((bi + 1) * bi / 2 <= o) ++bi;
  bj = o - bi * (bi - 1) / 2;
}

template <typename T, int kStages, int kMinBlocks, int KT = kKT, bool X3 = false>
__global__ void __launch_bounds__(kThreads, kMinBlocks) gram_dmma_kernel(const GramParams p) {
  constexpr int kLdT = KT + 4;  // smem column stride (elements)
  extern __shared__ __align__(128) unsigned char smem_raw[];
  T* pa = reinterpret_cast<T*>(smem_raw);                  // [stages][64][kLdT]
  T* pb = pa + static_cast<size_t>(kStages) * kBT * kLdT;  // [stages][64][kLdT] (diagonal CTAs: e panel)
  // Load balance: a diagonal block needs 3 of the 4 warp quarters, so its CTAs
  // take 4/3 as many rows (cd ~ 3/4 co).  Diagonal CTAs come first.
  const int ndc = p.nb * p.cd;
  const bool diag = static_cast<int>(blockIdx.x) < ndc;
  int bi, bj, chk;
  int64_t chunk;
  if (diag) {
    bi = bj = blockIdx.x % p.nb;
    chk = blockIdx.x / p.nb;
    chunk = p.chunk_d;
  } else {
    const int noff = p.nb * (p.nb - 1) / 2;
    const int c = blockIdx.x - ndc;
    tri_index_strict(c % noff, bi, bj);
    chk = c / noff;
    chunk = p.chunk_o;
  }
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // Off-diagonal block: warp w owns quarter (w>>1, w&1) of the 64x64 block.
  // Diagonal block (only its lower triangle is read): warps 0 and 3 own the two
  // diagonal quarters and compute only their lower tiles; warps 1 and 2 split
  // the lower off-diagonal quarter (32, 0) by tile rows and share the fused
  // first-sweep dots.  A diagonal CTA's warps then issue 8-10 of 16 DMMA tiles
  // (4-6 of 8 tf32 tiles) plus the dots; no MMA lands on tiles never read.
  const bool dq = diag && (warp == 0 || warp == 3);
  const bool dh = diag && (warp == 1 || warp == 2);
  const int half = warp == 1 ? 0 : 1;  // dh: which half of the tile rows
  const int wi = dh ? 32 : (warp >> 1) * 32, wj = dh ? 0 : (warp & 1) * 32;
  const T* __restrict__ x = static_cast<const T*>(p.x);
  const T* __restrict__ ev = static_cast<const T*>(p.e);
  const bool with_e = diag && ev != nullptr;
  const int64_t k_begin = static_cast<int64_t>(chk) * chunk;
  const int64_t k_end = imin64(p.obs, k_begin + chunk);
  const int nsteps = k_end > k_begin ? static_cast<int>((k_end - k_begin + KT - 1) / KT) : 0;
  constexpr int kPer = 16 / sizeof(T);               // elements per 16-byte piece
  constexpr int kPieces = KT / kPer;                // pieces per column per stage
  constexpr int kCopies = kBT * kPieces / kThreads;  // per thread per panel

  auto load_stage = [&](int step, int slot) {
    const int64_t k0 = k_begin + static_cast<int64_t>(step) * KT;
#pragma unroll
    for (int i = 0; i < kCopies; ++i) {
      const int id = tid + i * kThreads;
      const int col = id / kPieces, piece = id % kPieces;
      const int64_t row = k0 + piece * kPer;
      const int64_t rem = k_end - row;
      {
        const int64_t gc = static_cast<int64_t>(bi) * kBT + col;
        const int bytes = (gc < p.vars && rem > 0) ? static_cast<int>(imin64(rem, kPer) * sizeof(T)) : 0;
        const T* src = bytes ? x + gc * p.ldx + row : x;
        cp_async16(pa + (static_cast<size_t>(slot) * kBT + col) * kLdT + piece * kPer, src, bytes);
      }
      if (!diag) {
        const int64_t gc = static_cast<int64_t>(bj) * kBT + col;
        const int bytes = (gc < p.vars && rem > 0) ? static_cast<int>(imin64(rem, kPer) * sizeof(T)) : 0;
        const T* src = bytes ? x + gc * p.ldx + row : x;
        cp_async16(pb + (static_cast<size_t>(slot) * kBT + col) * kLdT + piece * kPer, src, bytes);
      }
    }
    if (with_e && tid < kPieces) {  // the residual rows of this stage (diagonal CTAs only)
      const int64_t row = k0 + tid * kPer;
      const int64_t rem = k_end - row;
      const int bytes = rem > 0 ? static_cast<int>(imin64(rem, kPer) * sizeof(T)) : 0;
      cp_async16(pb + static_cast<size_t>(slot) * kBT * kLdT + tid * kPer, bytes ? ev + row : ev, bytes);
    }
  };
  // Advisory lock step: the nb(nb+1)/2 CTAs of one K chunk read the same rows
  // (each 64-column panel feeds 4 of them), but diagonal CTAs run ahead of the
  // off-diagonal ones and the panels fall out of L2 before the slower readers
  // arrive (ncu: 86 GB of DRAM reads for 34 GB of x).  Every kPaceEvery stages a
  // CTA publishes its stage and (one stage later, with the counters already
  // read) waits, bounded, while it is more than kPaceLead stages ahead of the
  // slowest CTA of its chunk.  A hint only: a wait that
  // runs into its bound switches the pacing off for this CTA, and the results
  // do not depend on it.
  #ifndef BAK_PACE_EVERY
#define BAK_PACE_EVERY 16
#endif
#ifndef BAK_PACE_LEAD
#define BAK_PACE_LEAD 32
#endif
  constexpr int kPaceEvery = BAK_PACE_EVERY, kPaceLead = BAK_PACE_LEAD, kPaceSpins = 200, kPaceDone = 1 << 30;
  int pace_seen = kPaceDone;
  const int noff_all = p.nb * (p.nb - 1) / 2;
  bool paced = p.pace != nullptr;
  int pace_peer = -1;
  if (paced && warp == 0) {
    if (lane < p.nb) pace_peer = chk * p.nb + lane;
    else if (lane < p.nb + noff_all) pace_peer = ndc + chk * noff_all + (lane - p.nb);
  }
  // fused g0 (warp 1 of a diagonal CTA owns the unused upper quadrant: no DMMA work)
  double g0a = 0.0;

  double acc[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  // X3: the warp's 32x32 quarter as 2 (m16) x 4 (n8) tf32 tiles
  constexpr int kFlush = 8;  // stages per fp32 partial before it is added into fp64
  // fp64 totals live in shared memory ([32][kThreads] doubles after the
  // panels; 4 CTAs per SM need <= 128 registers per thread)
  float accf[2][4][4];
  double* accd = reinterpret_cast<double*>(pb + static_cast<size_t>(kStages) * kBT * kLdT) + tid;
  int nflush = 0;
  if constexpr (X3) {
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b)
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          accf[a][b][c] = 0.f;
          accd[((a * 4 + b) * 4 + c) * kThreads] = 0.0;
        }
  }
  auto flush = [&]() {
    if constexpr (X3) {
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b)
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            accd[((a * 4 + b) * 4 + c) * kThreads] += static_cast<double>(accf[a][b][c]);
            accf[a][b][c] = 0.f;
          }
    }
  };

#pragma unroll
  for (int s = 0; s < kStages - 1; ++s) {
    if (s < nsteps) load_stage(s, s);
    cp_async_commit();
  }
  const int fr = lane >> 2, fk = lane & 3;  // fragment row/col within an 8x4 tile
  for (int step = 0; step < nsteps; ++step) {
    if (paced && warp == 0) {
      const int ph = step % kPaceEvery;
      if (ph == 0) {
        // publish, and issue the read of the peers' counters: consumed one stage later, so its
        // L2 round trip overlaps this stage's MMAs
        if (lane == 0) *reinterpret_cast<volatile int*>(p.pace + blockIdx.x) = step;
        pace_seen = pace_peer >= 0 ? *reinterpret_cast<volatile const int*>(p.pace + pace_peer) : kPaceDone;
      } else if (ph == 1) {
        int v = __reduce_min_sync(0xffffffffu, pace_seen);
        int spins = 0;
        while (step > v + kPaceLead) {
          if (++spins > kPaceSpins) {
            paced = false;  // a peer is not keeping up (or not resident): stop waiting for it
            break;
          }
          __nanosleep(500);
          v = pace_peer >= 0 ? *reinterpret_cast<volatile const int*>(p.pace + pace_peer) : kPaceDone;
          v = __reduce_min_sync(0xffffffffu, v);
        }
      }
    }
    cp_async_wait<kStages - 2>();
    __syncthreads();
    {
      const int nxt = step + kStages - 1;
      if (nxt < nsteps) load_stage(nxt, nxt % kStages);
      cp_async_commit();
    }
    const int slot = step % kStages;
    const T* A = pa + static_cast<size_t>(slot) * kBT * kLdT;
    const T* B = diag ? A : pb + static_cast<size_t>(slot) * kBT * kLdT;
    if constexpr (X3) {
#pragma unroll
      for (int k8 = 0; k8 < KT; k8 += 8) {
        {
          uint32_t ah[2][4], al[2][4], bh[4][2], bl[4][2];
#pragma unroll
          for (int m = 0; m < 2; ++m) {
            const int r0 = wi + m * 16 + fr;
            split_tf32(A[r0 * kLdT + k8 + fk], ah[m][0], al[m][0]);
            split_tf32(A[(r0 + 8) * kLdT + k8 + fk], ah[m][1], al[m][1]);
            split_tf32(A[r0 * kLdT + k8 + fk + 4], ah[m][2], al[m][2]);
            split_tf32(A[(r0 + 8) * kLdT + k8 + fk + 4], ah[m][3], al[m][3]);
          }
#pragma unroll
          for (int n = 0; n < 4; ++n) {
            const int c0 = wj + n * 8 + fr;
            split_tf32(B[c0 * kLdT + k8 + fk], bh[n][0], bl[n][0]);
            split_tf32(B[c0 * kLdT + k8 + fk + 4], bh[n][1], bl[n][1]);
          }
          // three rounds over the warp's tiles (small terms first): consecutive
          // MMAs write different accumulators, so none waits on the one before.
          // Tile (m, n) = rows 16m.., cols 8n..; dq: lower tiles (8n < 16m+16)
          auto live = [&](int m, int n) { return dq ? (8 * n < 16 * m + 16) : (dh ? m == half : true); };
#pragma unroll
          for (int m = 0; m < 2; ++m)
#pragma unroll
            for (int n = 0; n < 4; ++n)
              if (live(m, n)) mma_tf32(accf[m][n], al[m], bh[n]);
#pragma unroll
          for (int m = 0; m < 2; ++m)
#pragma unroll
            for (int n = 0; n < 4; ++n)
              if (live(m, n)) mma_tf32(accf[m][n], ah[m], bl[n]);
#pragma unroll
          for (int m = 0; m < 2; ++m)
#pragma unroll
            for (int n = 0; n < 4; ++n)
              if (live(m, n)) mma_tf32(accf[m][n], ah[m], bh[n]);
        }
      }
      if (++nflush == kFlush) {
        nflush = 0;
        flush();
      }
    } else {
#pragma unroll
    for (int k4 = 0; k4 < KT; k4 += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        af[t] = static_cast<double>(A[(wi + t * 8 + fr) * kLdT + k4 + fk]);
        bf[t] = static_cast<double>(B[(wj + t * 8 + fr) * kLdT + k4 + fk]);
      }
      if (dq) {  // diagonal quarter: lower 8x8 tiles only
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b <= a; ++b) dmma(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
      } else if (dh) {  // half of the lower off-diagonal quarter
#pragma unroll
        for (int a = 0; a < 4; ++a)
          if ((a >> 1) == half)
#pragma unroll
            for (int b = 0; b < 4; ++b) dmma(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
      } else {
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) dmma(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
      }
    }
    }
    if (with_e && dh) {
      // the two half-quarter warps share the fused dots: warp 1 column lane,
      // warp 2 column lane + 32; rows in a lane-rotated order (conflict-free
      // banks), fixed per column -> deterministic
      const T* E = pb + static_cast<size_t>(slot) * kBT * kLdT;
      const int col = lane + 32 * half;
#pragma unroll 8
      for (int k = 0; k < KT; ++k) {
        const int kk = (k + lane) & (KT - 1);
        g0a = __fma_rn(static_cast<double>(A[col * kLdT + kk]), static_cast<double>(E[kk]), g0a);
      }
    }
  }
  if (with_e && dh) {
    const int64_t c0 = static_cast<int64_t>(bi) * kBT + lane + 32 * half;
    double* g = p.g0 + static_cast<int64_t>(chk) * p.vars;
    if (c0 < p.vars) g[c0] = g0a;
  }
  cp_async_wait<0>();
  if (p.pace && tid == 0) *reinterpret_cast<volatile int*>(p.pace + blockIdx.x) = kPaceDone;
  double* out = p.part + static_cast<size_t>(blockIdx.x) * kBT * kBT;
  if constexpr (X3) {
    flush();
#pragma unroll
    for (int m = 0; m < 2; ++m)
#pragma unroll
      for (int n = 0; n < 4; ++n) {
        if (dq ? !(8 * n < 16 * m + 16) : (dh && m != half)) continue;  // not this warp's tile
        const int i = wi + m * 16 + fr, j = wj + n * 8 + fk * 2;
        const double* ad = accd + ((m * 4 + n) * 4) * kThreads;
        out[i * kBT + j] = ad[0];
        out[i * kBT + j + 1] = ad[kThreads];
        out[(i + 8) * kBT + j] = ad[2 * kThreads];
        out[(i + 8) * kBT + j + 1] = ad[3 * kThreads];
      }
  } else {
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        if (dq ? b > a : (dh && (a >> 1) != half)) continue;  // not this warp's tile
        const int i = wi + a * 8 + fr, j = wj + b * 8 + fk * 2;
        out[i * kBT + j] = acc[a][b][0];
        out[i * kBT + j + 1] = acc[a][b][1];
      }
  }
}

// ---------------------------------------------------------------------------
// fp64 G, TMA-fed: the same block / chunk / warp-quarter decomposition and the
// same DMMA order as gram_dmma_kernel<double> (bit-identical partials), but the
// 16-row x 64-column panels arrive by cp.async.bulk.tensor (2-D tensor map over
// column-major x, 128B swizzle: a panel column is one 128-byte row, so the
// m8n8k4 fragment loads — 8 columns x 4 rows per LDS.64 — touch every bank
// once; rows past obs and columns past vars are zero-filled by the TMA unit)
// into a 3-stage ring with full / empty mbarriers.  No per-thread address
// arithmetic, no CTA-wide barrier per stage: a warp waits only for its data,
// and thread 0 re-arms a slot once the four warps have released it.
constexpr int kTR = 16;                      // rows per stage: 16 doubles = one 128-byte swizzle row
// ring depth x CTAs per SM: 4 x 3 (66 KB each); 3 x 4 is 0.4 ms (free-running) to 1.2 ms (lock step) slower on C3's
// shape, 6 x 2 is 10 ms slower (profiles/r02_gram_pace.jsonl)
#ifndef BAK_GT_STAGES
#define BAK_GT_STAGES 4
#endif
#ifndef BAK_GT_OCC
#define BAK_GT_OCC 3
#endif
constexpr int kTSt = BAK_GT_STAGES;
constexpr uint32_t kTTile = kBT * 128;       // bytes per 64-column panel stage

__device__ __forceinline__ void tma_load_2d_g(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_g(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
// wait on a phase with the library's deadline; false = timed out (reported, abort flag set)
__device__ __forceinline__ bool mbar_wait_g(uint64_t* bar, uint32_t parity, volatile int* abort_flag, int64_t* status) {
  if (mbar_test(bar, parity)) return true;
  const uint64_t t0 = globaltimer();
  while (!mbar_test(bar, parity)) {
    if (*abort_flag) return false;
    if (globaltimer() - t0 > kTimeoutNs) {
      report_error(status, BAK_ETIMEOUT);
      *abort_flag = 1;
      return false;
    }
  }
  return true;
}

__global__ void __launch_bounds__(kThreads, BAK_GT_OCC)
    gram_dmma_tma_kernel(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap emap,
                         const GramParams p) {
  extern __shared__ unsigned char smem_raw_t[];
  const uint32_t base_s = (smem_addr(smem_raw_t) + 1023u) & ~1023u;  // swizzle atoms are 1024-byte aligned
  unsigned char* base = smem_raw_t + (base_s - smem_addr(smem_raw_t));
  unsigned char* tiles = base;                                                  // [kTSt][A | B]
  double* es = reinterpret_cast<double*>(base + kTSt * 2 * kTTile);             // [kTSt][16]
  uint64_t* full = reinterpret_cast<uint64_t*>(base + kTSt * 2 * kTTile + kTSt * 128);
  uint64_t* empty = full + kTSt;
  volatile int* abort_flag = reinterpret_cast<volatile int*>(empty + kTSt);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    for (int s = 0; s < kTSt; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kThreads / 32);
    }
    *abort_flag = 0;
    fence_mbar_init();
  }
  __syncthreads();

  const int ndc = p.nb * p.cd;
  const int noff_all = p.nb * (p.nb - 1) / 2;
  const int fr = lane >> 2, fk = lane & 3;
  const uint32_t lo8 = static_cast<uint32_t>(fk & 1) * 8u;
  constexpr int kPaceEvery = BAK_PACE_EVERY, kPaceLead = BAK_PACE_LEAD, kPaceSpins = 200, kPaceDone = 1 << 30;

  // p.units: every CTA runs TWO units — an off-diagonal (block, chunk) and then a diagonal one
  // (grid = nb * cd = noff * co) — so that all CTAs, and with them all SMs, carry the same work
  // (one unit per CTA left the SMs that drew two light diagonal CTAs idle at the end: DMMA pipe
  // 64-90 % active across SMs).  Unit ids and the partial / g0 layout are those of the
  // one-unit-per-CTA grid, so the reduction is unchanged.  The ring runs on across the units
  // (gbase = stages issued so far).
  int gbase = 0;
  const int nunits = p.units ? 2 : 1;
  for (int unit = 0; unit < nunits; ++unit) {
    const int vid = p.units ? (unit == 0 ? ndc + static_cast<int>(blockIdx.x) : static_cast<int>(blockIdx.x))
                            : static_cast<int>(blockIdx.x);
    const bool diag = vid < ndc;
    int bi, bj, chk;
    int64_t chunk;
    if (diag) {
      bi = bj = vid % p.nb;
      chk = vid / p.nb;
      chunk = p.chunk_d;
    } else {
      const int c = vid - ndc;
      tri_index_strict(c % noff_all, bi, bj);
      chk = c / noff_all;
      chunk = p.chunk_o;
    }
    const bool dq = diag && (warp == 0 || warp == 3);
    const bool dh = diag && (warp == 1 || warp == 2);
    const int half = warp == 1 ? 0 : 1;
    const int wi = dh ? 32 : (warp >> 1) * 32, wj = dh ? 0 : (warp & 1) * 32;
    const bool with_e = diag && p.e != nullptr;
    const int64_t k_begin = static_cast<int64_t>(chk) * chunk;
    const int64_t k_end = imin64(p.obs, k_begin + chunk);
    const int nsteps = k_end > k_begin ? static_cast<int>((k_end - k_begin + kTR - 1) / kTR) : 0;

    const uint32_t stage_bytes = (diag ? kTTile : 2 * kTTile) + (with_e ? kTR * 8u : 0u);
    // thread 0: arm the slot of global stage gbase + step (after its previous use has been released
    // by all four warps) and start the copies
    auto issue = [&](int step) -> bool {
      const int g = gbase + step;
      const int slot = g % kTSt;
      if (g >= kTSt &&
          !mbar_wait_g(&empty[slot], static_cast<uint32_t>((g / kTSt - 1) & 1), abort_flag, p.status))
        return false;
      const int row0 = static_cast<int>(k_begin + static_cast<int64_t>(step) * kTR);
      const uint32_t bar = smem_addr(&full[slot]);
      mbar_arrive_expect_tx(&full[slot], stage_bytes);
      tma_load_2d_g(smem_addr(tiles + slot * 2 * kTTile), &xmap, row0, bi * kBT, bar);
      if (!diag) tma_load_2d_g(smem_addr(tiles + slot * 2 * kTTile + kTTile), &xmap, row0, bj * kBT, bar);
      if (with_e) tma_load_2d_g(smem_addr(es + slot * kTR), &emap, row0, 0, bar);
      return true;
    };
    if (tid == 0)
      for (int s = 0; s < kTSt - 1 && s < nsteps; ++s)
        if (!issue(s)) break;

    // advisory lock step of the CTAs that read the same rows (see gram_dmma_kernel); counters are
    // indexed by CTA.  pace_offdiag_only: 1 = diagonal units run free, 2 = they follow the
    // off-diagonal ones; with two units per CTA only the off-diagonal units share rows in time.
    int pace_seen = kPaceDone;
    bool paced = p.pace != nullptr && !((p.pace_offdiag_only == 1 || p.units) && diag);
    int pace_peer = -1;
    if (paced && warp == 0) {
      if (p.units) {
        if (lane < noff_all) pace_peer = chk * noff_all + lane;
      } else if (lane < p.nb) {
        pace_peer = p.pace_offdiag_only ? -1 : chk * p.nb + lane;
      } else if (lane < p.nb + noff_all) {
        pace_peer = ndc + chk * noff_all + (lane - p.nb);
      }
    }

    double g0q[4] = {0.0, 0.0, 0.0, 0.0};
    double acc[4][4][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

    // byte offset of element (column c, row k) of a panel: c * 128 + (((k >> 1) ^ (c & 7)) << 4) + (k & 1) * 8;
    // the fragment columns are wi|wj + 8 t + fr, so c & 7 == fr
    const uint32_t a_row = static_cast<uint32_t>(wi + fr) * 128u, b_row = static_cast<uint32_t>(wj + fr) * 128u;
    bool alive = true;
    for (int step = 0; step < nsteps; ++step) {
      if (paced && warp == 0) {
        const int ph = step % kPaceEvery;
        if (ph == 0) {
          if (lane == 0) *reinterpret_cast<volatile int*>(p.pace + blockIdx.x) = step;
          pace_seen = pace_peer >= 0 ? *reinterpret_cast<volatile const int*>(p.pace + pace_peer) : kPaceDone;
        } else if (ph == 1) {
          int v = __reduce_min_sync(0xffffffffu, pace_seen);
          int spins = 0;
          while (step > v + kPaceLead) {
            if (++spins > kPaceSpins) {
              paced = false;
              break;
            }
            __nanosleep(500);
            v = pace_peer >= 0 ? *reinterpret_cast<volatile const int*>(p.pace + pace_peer) : kPaceDone;
            v = __reduce_min_sync(0xffffffffu, v);
          }
        }
      }
      if (tid == 0) {  // re-arm before this stage's work (after it: 0.2-0.7 ms slower, the prefetch distance matters)
        const int nxt = step + kTSt - 1;
        if (nxt < nsteps) issue(nxt);
      }
      __syncwarp();
      const int g = gbase + step;
      const int slot = g % kTSt;
      if (!mbar_wait_g(&full[slot], static_cast<uint32_t>((g / kTSt) & 1), abort_flag, p.status)) {
        alive = false;
        break;
      }
      const unsigned char* A = tiles + slot * 2 * kTTile;
      const unsigned char* B = diag ? A : A + kTTile;
#pragma unroll
      for (int k4 = 0; k4 < kTR; k4 += 4) {
        const uint32_t sw = ((static_cast<uint32_t>(k4 >> 1) | static_cast<uint32_t>(fk >> 1)) ^ static_cast<uint32_t>(fr)) << 4;
        double af[4], bf[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          af[t] = *reinterpret_cast<const double*>(A + a_row + t * 1024 + sw + lo8);
          bf[t] = *reinterpret_cast<const double*>(B + b_row + t * 1024 + sw + lo8);
        }
        if (dq) {
#pragma unroll
          for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b <= a; ++b) dmma(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
        } else if (dh) {
#pragma unroll
          for (int a = 0; a < 4; ++a)
            if ((a >> 1) == half)
#pragma unroll
              for (int b = 0; b < 4; ++b) dmma(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
        } else {
#pragma unroll
          for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) dmma(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
        }
      }
      if (with_e && dh) {
        // fused first-sweep dots (warps 1-2: column lane + 32 half, rows in a lane-rotated order) as
        // four independent FMA chains: a DFMA queues behind the DMMAs of 16 warps on the same pipe, and
        // one 16-long dependent chain per stage made the diagonal CTAs the slowest of their chunk
        // (40.4 -> 38.6 ms; spreading the dots over all four warps instead: 39.8)
        const double* E = es + slot * kTR;
        const int col = lane + 32 * half;
        const uint32_t crow = static_cast<uint32_t>(col) * 128u;
#pragma unroll
        for (int k = 0; k < kTR; ++k) {
          const int kk = (k + lane) & (kTR - 1);
          const uint32_t off = crow + ((static_cast<uint32_t>(kk >> 1) ^ static_cast<uint32_t>(col & 7)) << 4) +
                               static_cast<uint32_t>(kk & 1) * 8u;
          g0q[k & 3] = __fma_rn(*reinterpret_cast<const double*>(A + off), E[kk], g0q[k & 3]);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive_g(&empty[slot]);  // this warp is done reading the slot
    }
    if (with_e && dh) {
      const int64_t c0 = static_cast<int64_t>(bi) * kBT + lane + 32 * half;
      double* g = p.g0 + static_cast<int64_t>(chk) * p.vars;
      if (c0 < p.vars) g[c0] = (g0q[0] + g0q[1]) + (g0q[2] + g0q[3]);
    }
    if (p.pace && tid == 0 && (unit == nunits - 1 || !diag))
      *reinterpret_cast<volatile int*>(p.pace + blockIdx.x) = kPaceDone;
    double* out = p.part + static_cast<size_t>(vid) * kBT * kBT;
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        if (dq ? b > a : (dh && (a >> 1) != half)) continue;
        const int i = wi + a * 8 + fr, j = wj + b * 8 + fk * 2;
        out[i * kBT + j] = acc[a][b][0];
        out[i * kBT + j + 1] = acc[a][b][1];
      }
    if (!alive) break;
    gbase += nsteps;
  }
}

constexpr size_t kGramTmaSmem = 1024 + kTSt * 2 * kTTile + kTSt * 128 + 2 * kTSt * 8 + 16;

// G (vars x vars, full, symmetric) = sum over K chunks of the lower block partials
template <typename T>
__global__ void gram_reduce_kernel(const double* __restrict__ part, int nb, int cd, int co, int64_t V,
                                   double* __restrict__ G, T* __restrict__ norms) {
  const int blk = blockIdx.y;  // lower triangle, row-major
  int bi = 0;
  while ((bi + 1) * (bi + 2) / 2 <= blk) ++bi;
  const int bj = blk - bi * (bi + 1) / 2;
  const int noff = nb * (nb - 1) / 2;
  const bool dg = bi == bj;
  const int nch = dg ? cd : co;
  const size_t first = dg ? static_cast<size_t>(bi) : static_cast<size_t>(nb) * cd + bi * (bi - 1) / 2 + bj;
  const size_t stride = dg ? nb : noff;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < kBT * kBT; e += gridDim.x * blockDim.x) {
    const int i = e / kBT, j = e % kBT;
    const int64_t gi = static_cast<int64_t>(bi) * kBT + i, gj = static_cast<int64_t>(bj) * kBT + j;
    if (gi >= V || gj >= V) continue;
    if (dg && j > i) continue;  // diagonal block: lower half (mirrored below)
    double s = 0.0;
    for (int c = 0; c < nch; ++c) s += part[(first + c * stride) * kBT * kBT + e];
    G[gj * V + gi] = s;  // column-major (gi, gj)
    G[gi * V + gj] = s;  // mirror (gj, gi)
    if (norms && gi == gj) norms[gi] = static_cast<T>(s);  // n2_j = G_jj (fp64-accumulated)
  }
}

}  // namespace

static inline int imax_host(int a, int b) { return a > b ? a : b; }

struct GramSplit {
  int nb, cd, co;
  int64_t chunk_d, chunk_o;
  int units;  // TMA-fed fp64 kernel: two units per CTA (grid = nb * cd = noff * co)
};

// CTAs per SM of the G kernel: 3 (2-stage ring, <=170 registers) keeps the DMMA
// pipe ~75% busy vs ~65% at 2 CTAs (3-stage ring); tuning aid BAK_GRAM_OCC=2
// Default: 16-row stages, 2-stage ring (37 KB fp64), <= 128 registers, 4 CTAs
// per SM — measured 46.2 ms vs 48.0 ms (32-row stages, 3 CTAs/SM) for C3's
// G.  Tuning aids: BAK_GRAM_KT=32 (32-row stages; then BAK_GRAM_OCC=2|3).
static bool gram_kt16() {
  const char* kt = getenv("BAK_GRAM_KT");
  return !(kt && kt[0] == '3' && kt[1] == '2');
}

static int gram_occ() {
  if (gram_kt16()) return 4;
  const char* o = getenv("BAK_GRAM_OCC");
  return (o && o[0] == '2') ? 2 : 3;
}

// the TMA-fed fp64 kernel can be used (x / e alignment is checked at launch; misaligned inputs run the
// cp.async kernel on the same split); BAK_GRAM_G_TMA=0: cp.async kernel
// (the chunk split below is sized for the TMA-fed kernel whenever it COULD run, so that BAK_GRAM_G_TMA=0
// gives the cp.async kernel the same chunks and therefore the same bits)
static bool gram_g_tma_possible(int dtype, int64_t obs) {
  if (dtype != BAK_F64 || !gram_kt16() || obs >= (int64_t(1) << 31)) return false;
  return tensor_map_encoder() != nullptr;
}
static bool gram_g_tma_wanted(int dtype, int64_t obs) {
  const char* t = getenv("BAK_GRAM_G_TMA");
  if (t && t[0] == '0') return false;
  return gram_g_tma_possible(dtype, obs);
}

static int64_t gcd64(int64_t a, int64_t b) { return b ? gcd64(b, a % b) : a; }

static GramSplit gram_split(int dtype, int64_t obs, int64_t vars) {
  GramSplit g{};
  g.nb = static_cast<int>((vars + kBT - 1) / kBT);
  const int noff = g.nb * (g.nb - 1) / 2;
  {
    // BAK_GRAM_UNITS=1 (tuning aid, off by default): two units per CTA — U CTAs, U the largest multiple
    // of lcm(nb, noff) in one wave; diagonal block b of chunk c is unit c * nb + b, off-diagonal block o
    // of chunk c is c * noff + o.  Every SM then carries the same work: 38.6 vs 39.6 ms alone on C3's
    // shape, but the diagonal and off-diagonal units of a row range no longer run together, so x comes
    // from DRAM 2-2.8 times (72-96 GB), and inside the power-capped C3 step it measured the same
    // 132-133 sweeps/s as one unit per CTA in full lock step (35 GB) — which is therefore the default.
    const char* u = getenv("BAK_GRAM_UNITS");
    const int slots4 = BAK_GT_OCC * device_sms();
    if ((u && u[0] == '1') && !getenv("BAK_GRAM_DIAG_RATIO") && noff > 0 && gram_g_tma_wanted(dtype, obs)) {
      const int64_t l = static_cast<int64_t>(g.nb) / gcd64(g.nb, noff) * noff;
      if (l <= slots4) {
        const int64_t U = slots4 / l * l;
        g.units = 1;
        g.cd = static_cast<int>(U / g.nb);
        g.co = static_cast<int>(U / noff);
        g.chunk_d = round_up((obs + g.cd - 1) / g.cd, kKT);
        g.chunk_o = round_up((obs + g.co - 1) / g.co, kKT);
        return g;  // chunks past obs stay in the grid (they write zero partials)
      }
    }
  }
  // One wave of CTAs, equal row chunks for every block by default.  With the
  // first sweep's dots fused (warps 1-2 of the diagonal CTAs), diagonal and
  // off-diagonal CTAs then take about the same time (in-solve G on C3: 42.8 ms
  // fp64 / 36.2 ms fp32 at ratio 1 vs 46.8 / 43.3 at 0.625 — the 10/16 ratio
  // of their DMMA tiles alone).  BAK_GRAM_DIAG_RATIO=r gives diagonal blocks
  // 1/r of the rows (tuning aid).
  const int slots = (gram_g_tma_possible(dtype, obs) ? BAK_GT_OCC : gram_occ()) * device_sms();
  const char* rr = getenv("BAK_GRAM_DIAG_RATIO");
  const double ratio = rr ? atof(rr) : 1.0;
  if (!(ratio > 0.0 && ratio < 4.0) || ratio == 1.0) {
    g.cd = g.co = imax_host(1, slots / (g.nb * (g.nb + 1) / 2));
  } else if (noff == 0) {
    g.co = 1;
    g.cd = slots;
  } else {
    g.co = static_cast<int>(slots / (noff + ratio * g.nb));
    if (g.co < 1) g.co = 1;
    g.cd = static_cast<int>(ratio * g.co);
    if (g.cd < 1) g.cd = 1;
  }
  g.chunk_d = round_up((obs + g.cd - 1) / g.cd, kKT);
  g.chunk_o = round_up((obs + g.co - 1) / g.co, kKT);
  g.cd = static_cast<int>((obs + g.chunk_d - 1) / g.chunk_d);
  g.co = static_cast<int>((obs + g.chunk_o - 1) / g.chunk_o);
  if (g.cd < 1) g.cd = 1;
  if (g.co < 1) g.co = 1;
  return g;
}

int64_t gram_g_workspace(int dtype, int64_t obs, int64_t vars, int& nchunks, int64_t& chunk) {
  if (gram_tc_enabled(dtype, vars)) {  // one reduced row of g0
    nchunks = 1;
    chunk = obs;
    return gram_tc_workspace(obs, vars);
  }
  const GramSplit g = gram_split(dtype, obs, vars);
  nchunks = g.cd;  // partial rows of the fused g0
  chunk = g.chunk_d;
  const int64_t ctas = static_cast<int64_t>(g.nb) * g.cd + static_cast<int64_t>(g.nb) * (g.nb - 1) / 2 * g.co;
  return ctas * kBT * kBT * 8 + round_up(ctas * 4, 256);  // partials + the pacing counters
}

static bool gram_g_tma_ok(int dtype, const void* x, int64_t obs, int64_t ldx, const void* e) {
  if (!gram_g_tma_wanted(dtype, obs)) return false;
  if (reinterpret_cast<uintptr_t>(x) % 16 || (ldx * 8) % 16) return false;
  if (e && reinterpret_cast<uintptr_t>(e) % 16) return false;
  return true;
}

int launch_gram_g(int dtype, const void* x, int64_t obs, int64_t ldx, int64_t vars, double* G, void* part_ws,
                  int64_t part_bytes, cudaStream_t st, void* norms_out, const void* e, double* g0, int64_t* status) {
  if (gram_tc_enabled(dtype, vars))
    return launch_gram_g_tc(x, obs, ldx, vars, G, part_ws, part_bytes, st, norms_out, e, g0, status);
  int nchunks;
  int64_t chunk;
  const int64_t need = gram_g_workspace(dtype, obs, vars, nchunks, chunk);
  if (part_bytes < need) {
    set_error("gram: partial workspace too small");
    return BAK_EWORKSPACE;
  }
  const GramSplit g = gram_split(dtype, obs, vars);
  const int nblk = g.nb * (g.nb + 1) / 2;
  GramParams p{x, obs, ldx, vars, g.nb, g.cd, g.co, g.chunk_d, g.chunk_o, static_cast<double*>(part_ws),
               g0 ? e : nullptr, g0, nullptr, status, 0, 0};
  const size_t ts = dtype == BAK_F64 ? 8 : 4;
  const bool tma = gram_g_tma_ok(dtype, x, obs, ldx, p.e);
  const bool units = tma && g.units;
  p.units = units ? 1 : 0;
  const unsigned grid = units ? static_cast<unsigned>(g.nb * g.cd)
                              : static_cast<unsigned>(g.nb * g.cd + g.nb * (g.nb - 1) / 2 * g.co);
  // advisory lock step of the CTAs of a K chunk (same rows for every block, <= 32 blocks, one wave);
  // BAK_GRAM_PACE=0 switches it off
  {
    const char* pe = getenv("BAK_GRAM_PACE");
    const bool off = pe && pe[0] == '0';
    p.pace_offdiag_only = (pe && pe[0] == '2') ? 1 : (pe && pe[0] == '3') ? 2 : 0;
    const int nblk_all = g.nb * (g.nb + 1) / 2;
    const size_t nparts = static_cast<size_t>(g.nb) * g.cd + static_cast<size_t>(g.nb) * (g.nb - 1) / 2 * g.co;
    if (!off && g.nb > 1 && nblk_all <= 32 && (units || (g.cd == g.co && g.chunk_d == g.chunk_o)) &&
        static_cast<int>(grid) <= (gram_g_tma_possible(dtype, obs) ? BAK_GT_OCC : gram_occ()) * device_sms()) {
      p.pace = reinterpret_cast<int*>(static_cast<char*>(part_ws) + nparts * kBT * kBT * 8);
      BAK_CHECK_CUDA(cudaMemsetAsync(p.pace, 0, static_cast<size_t>(grid) * 4, st));
    }
  }
  auto go = [&](auto kern, int stages) -> int {
    const size_t smem = 2ull * stages * kBT * kLd * ts;
    BAK_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    kern<<<grid, kThreads, smem, st>>>(p);
    return BAK_OK;
  };
  const bool occ3 = gram_occ() == 3;
  const bool kt16 = gram_kt16();
  int rc;
  if (tma) {
    auto enc = tensor_map_encoder();
    CUtensorMap xmap, emap;
    {
      cuuint64_t gdim[2] = {static_cast<cuuint64_t>(obs), static_cast<cuuint64_t>(vars)};
      cuuint64_t gstr[1] = {static_cast<cuuint64_t>(ldx * 8)};
      cuuint32_t box[2] = {static_cast<cuuint32_t>(kTR), static_cast<cuuint32_t>(kBT)};
      cuuint32_t est[2] = {1, 1};
      CUresult r = enc(&xmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<void*>(x), gdim, gstr, box, est,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) {
        set_error("cuTensorMapEncodeTiled (x, fp64 G) failed (%d)", static_cast<int>(r));
        return BAK_ECUDA;
      }
    }
    {
      const void* ep = p.e ? p.e : x;  // a valid map either way (unused without e)
      cuuint64_t gdim[2] = {static_cast<cuuint64_t>(obs), 1};
      cuuint64_t gstr[1] = {static_cast<cuuint64_t>(round_up(obs * 8, 16))};
      cuuint32_t box[2] = {static_cast<cuuint32_t>(kTR), 1};
      cuuint32_t est[2] = {1, 1};
      CUresult r = enc(&emap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<void*>(ep), gdim, gstr, box, est,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) {
        set_error("cuTensorMapEncodeTiled (e, fp64 G) failed (%d)", static_cast<int>(r));
        return BAK_ECUDA;
      }
    }
    BAK_CHECK_CUDA(cudaFuncSetAttribute(gram_dmma_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(kGramTmaSmem)));
    gram_dmma_tma_kernel<<<grid, kThreads, kGramTmaSmem, st>>>(xmap, emap, p);
    rc = BAK_OK;
  } else if (kt16) {
    auto go16 = [&](auto kern) -> int {
      const size_t smem = 2ull * 2 * kBT * (16 + 4) * ts;
      BAK_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
      kern<<<grid, kThreads, smem, st>>>(p);
      return BAK_OK;
    };
    // fp32 inputs: 3xTF32 on the tf32 MMA path (BAK_GRAM_G=dmma keeps fp64 DMMA)
    const char* gg = getenv("BAK_GRAM_G");
    const bool x3 = !(gg && gg[0] == 'd');
    auto go16x3 = [&](auto kern) -> int {
      const size_t smem = 2ull * 2 * kBT * (16 + 4) * ts + 32ull * kThreads * 8;  // + fp64 totals
      BAK_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
      kern<<<grid, kThreads, smem, st>>>(p);
      return BAK_OK;
    };
    rc = dtype == BAK_F64 ? go16(gram_dmma_kernel<double, 2, 4, 16>)
                          : (x3 ? go16x3(gram_dmma_kernel<float, 2, 4, 16, true>) : go16(gram_dmma_kernel<float, 2, 4, 16>));
  } else if (dtype == BAK_F64)
    rc = occ3 ? go(gram_dmma_kernel<double, 2, 3>, 2) : go(gram_dmma_kernel<double, 3, 2>, 3);
  else
    rc = occ3 ? go(gram_dmma_kernel<float, 2, 3>, 2) : go(gram_dmma_kernel<float, 3, 2>, 3);
  if (rc) return rc;
  count_launches(1);
  BAK_CHECK_CUDA(cudaGetLastError());
  if (dtype == BAK_F64)
    gram_reduce_kernel<double><<<dim3(16, nblk), 256, 0, st>>>(static_cast<const double*>(part_ws), g.nb, g.cd, g.co,
                                                               vars, G, static_cast<double*>(norms_out));
  else
    gram_reduce_kernel<float><<<dim3(16, nblk), 256, 0, st>>>(static_cast<const double*>(part_ws), g.nb, g.cd, g.co,
                                                              vars, G, static_cast<float*>(norms_out));
  count_launches(1);
  BAK_CHECK_CUDA(cudaGetLastError());
  return BAK_OK;
}

}  // namespace bak

// G = X^T X for fp32 inputs on the 5th-generation tensor cores
// (tcgen05.mma kind::tf32, accumulators in TMEM), with the first sweep's
// g0 = X^T e fused in — the GRAM variant's once-per-solve setup
// (SURVEY §7.4-1 option (b); replaces the per-column dots of bak.py:86).
//
// Precision (3xTF32 folded into two products): every x is split exactly into
// hi = x with the low 13 mantissa bits cleared (exact in tf32) and
// lo = x - hi (exact in fp32; the tensor core keeps its top 11 bits).
//   S = Hi^T Hi + Hi^T (2 Lo),   G = (S + S^T) / 2 = Hi^T Hi + Hi^T Lo + Lo^T Hi
// (the dropped Lo^T Lo is ~2^-22 of |x_i||x_j|).  The products are exact in
// fp32, but the tensor core's fp32 accumulation truncates: measured on B200,
// an entry accumulated over C rows in TMEM is low by ~1.2e-8 * C of itself
// (tools/gram_tc_probe.py: 5.0e-5 at C = 4096, 1.9e-6 at C = 128, linear).
// So S is accumulated over chunks of C rows (BAK_GRAM_TC_CHUNK, default
// 1024), each chunk's S goes out to HBM and a fixed-order fp64 reduction sums
// the chunks and symmetrises (deterministic); the DIAGONAL — the column norms
// the solve divides by — is instead summed on the CUDA cores (x_j . x_j next
// to x_j . e: IEEE fp32 FMA chains over each 32-row tile, tiles added in
// fp64), so only the off-diagonal entries carry the ~1e-5-of-themselves
// truncation (for near-orthogonal columns ~1e-8 of the diagonal).
//
// One CTA per SM, persistent over the row chunks; 10 warps:
//   warp 0     TMA producer: 32-row x vb-column tiles of column-major x (2-D
//              tensor map, 128B swizzle = the UMMA K-major SW128 layout, rows
//              past obs / columns past vars zero-filled) and the tile's 32
//              entries of e (obs x 1 tensor map), kStages-deep ring;
//   warp 1     TMEM allocation (512 columns) and, on one lane, the MMA issuer:
//              per 8-row k-step 2 (vb=128) or 4 (vb=256) tcgen05.mma
//              M=128 x N=vb x K=8 into two 128 x 256 fp32 accumulators;
//              tcgen05.commit frees the ring slot / signals the epilogue;
//   warps 2-9  split each tile in place, one column per thread (hi over the
//              raw tile, 2*lo into a second buffer with the same swizzled
//              layout — the split is element-wise, so the swizzle does not
//              matter), accumulate x_j . e and x_j . x_j, and drain the
//              accumulators (tcgen05.ld 32x32b; warp w reads TMEM lanes
//              32*(w%4).., two warps per quadrant split the columns) into the
//              chunk's partial S.  Waits sleep in mbarrier.try_wait with a
//              suspend-time hint instead of spinning on issue slots.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>

#include "bak_common.cuh"
#include "bak_sweep.cuh"

namespace bak {

PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder();

namespace {

constexpr int kTK = 32;          // rows per tile: 32 fp32 = one 128-byte swizzle row
constexpr int kStages = 3;       // ring depth
constexpr int kConvWarps = 8;    // split / epilogue warps (two per TMEM lane quadrant)
constexpr int kThreads = 64 + 32 * kConvWarps;
constexpr int kReduceGroups = 32;

struct TcParams {
  int64_t obs;
  int vb;             // 128 or 256 tile columns (columns >= vars are zero)
  int64_t nchunks;
  int64_t chunk_rows;  // multiple of kTK
  float* part;         // [nchunks][vb][vb] S of each chunk
  double* cpart;       // [nchunks][2][vb] x_j . e (with_e) and x_j . x_j of each chunk, fp64
  int with_e;
  int64_t* status;
};

__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}

// UMMA shared-memory descriptor: K-major operand, 128B swizzle, 8-row core
// groups 1024 bytes apart (SBO), version 1 (sm_100), LBO unused (1).
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
  return static_cast<uint64_t>((saddr >> 4) & 0x3FFFu) | (static_cast<uint64_t>(1) << 16) |
         (static_cast<uint64_t>(1024 >> 4) << 32) | (static_cast<uint64_t>(1) << 46) |
         (static_cast<uint64_t>(2) << 61);
}
// instruction descriptor, kind::tf32: D fp32, A/B tf32, both K-major, M x N
__host__ __device__ constexpr uint32_t idesc_tf32(int m, int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(n >> 3) << 17) |
         (static_cast<uint32_t>(m >> 4) << 24);
}
__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_addr(bar))
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// try_wait with a suspend-time hint: the thread sleeps in the barrier unit
// until the phase completes (or ~20 us pass) instead of spinning on issue slots
__device__ __forceinline__ bool mbar_wait_hint(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_addr(bar)), "r"(parity), "r"(20000u)
      : "memory");
  return ok != 0;
}

// wait on an mbarrier phase; after the deadline (or once another role gave up)
// report BAK_ETIMEOUT and let every role fall through to the teardown
__device__ __forceinline__ bool wait_phase(uint64_t* bar, uint32_t parity, volatile int* abort_flag,
                                           int64_t* status) {
  if (mbar_test(bar, parity)) return true;
  const uint64_t t0 = globaltimer();
  while (!mbar_wait_hint(bar, parity)) {
    if (*abort_flag) return false;
    if (globaltimer() - t0 > kTimeoutNs) {
      report_error(status, BAK_ETIMEOUT);
      *abort_flag = 1;
      return false;
    }
  }
  return true;
}

__global__ void __launch_bounds__(kThreads, 1)
    gram_tc_kernel(const __grid_constant__ CUtensorMap xmap, const __grid_constant__ CUtensorMap emap,
                   const TcParams p) {
  extern __shared__ unsigned char smem_raw[];
  // 1024-byte aligned operand buffers (128B-swizzle atoms)
  const uint32_t base_s = (smem_addr(smem_raw) + 1023u) & ~1023u;
  unsigned char* base = smem_raw + (base_s - smem_addr(smem_raw));
  const int vb = p.vb;
  const uint32_t tile_bytes = static_cast<uint32_t>(vb) * 128u;
  unsigned char* raw = base;                                   // [kStages][vb][128 B]
  unsigned char* lo = raw + kStages * tile_bytes;              // [kStages][vb][128 B]
  float* es = reinterpret_cast<float*>(lo + kStages * tile_bytes);  // [kStages][32]
  uint64_t* full = reinterpret_cast<uint64_t*>(es + kStages * kTK);
  uint64_t* conv = full + kStages;
  uint64_t* empty = conv + kStages;
  uint64_t* accf = empty + kStages;
  uint64_t* acce = accf + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acce + 1);
  volatile int* abort_flag = reinterpret_cast<volatile int*>(tmem_slot + 1);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&conv[s], vb == 256 ? 256 : 128);  // the converting threads
      mbar_init(&empty[s], 1);
    }
    mbar_init(accf, 1);
    mbar_init(acce, 32 * kConvWarps);
    *abort_flag = 0;
    fence_mbar_init();
  }
  if (warp == 1) {  // whole warp: allocate all 512 TMEM columns (one CTA per SM)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_addr(tmem_slot))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  const int64_t T_total = (p.obs + kTK - 1) / kTK;
  const int64_t tiles_per_chunk = p.chunk_rows / kTK;
  auto chunk_tiles = [&](int64_t c) -> int {
    return static_cast<int>(imin64(tiles_per_chunk, T_total - c * tiles_per_chunk));
  };

  if (warp == 0) {
    // ------------------------------ TMA producer ------------------------------
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      int64_t u = 0;
      const uint32_t bytes = tile_bytes + (p.with_e ? kTK * 4u : 0u);
      for (int64_t c = blockIdx.x; c < p.nchunks; c += gridDim.x) {
        const int nt = chunk_tiles(c);
        for (int t = 0; t < nt; ++t, ++u) {
          if (u >= kStages && !wait_phase(&empty[s], ph ^ 1u, abort_flag, p.status)) goto done;
          const int row0 = static_cast<int>(c * tiles_per_chunk + t) * kTK;
          mbar_arrive_expect_tx(&full[s], bytes);
          tma_load_2d(smem_addr(raw + s * tile_bytes), &xmap, row0, 0, smem_addr(&full[s]));
          if (p.with_e) tma_load_2d(smem_addr(es + s * kTK), &emap, row0, 0, smem_addr(&full[s]));
          if (++s == kStages) { s = 0; ph ^= 1u; }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------ MMA issuer ------------------------------
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      const uint32_t idesc = idesc_tf32(128, vb);
      int64_t it = 0;
      for (int64_t c = blockIdx.x; c < p.nchunks; c += gridDim.x, ++it) {
        if (it > 0) {  // the epilogue has drained the previous chunk's accumulators
          if (!wait_phase(acce, static_cast<uint32_t>((it - 1) & 1), abort_flag, p.status)) goto done;
          tc_fence_after();
        }
        const int nt = chunk_tiles(c);
        for (int t = 0; t < nt; ++t) {
          if (!wait_phase(&conv[s], ph, abort_flag, p.status)) goto done;
          tc_fence_after();
          const uint32_t r_s = smem_addr(raw + s * tile_bytes);
          const uint32_t l_s = smem_addr(lo + s * tile_bytes);
#pragma unroll
          for (int k = 0; k < kTK / 8; ++k) {  // UMMA_K = 8 tf32 = 32 bytes along the swizzled row
            const uint64_t bh = umma_desc_sw128(r_s + 32u * k);
            const uint64_t bl = umma_desc_sw128(l_s + 32u * k);
            const uint32_t first = (t == 0 && k == 0) ? 0u : 1u;
            umma_tf32(tmem, bh, bh, idesc, first);          // rows 0..127 of S: Hi^T Hi
            umma_tf32(tmem, bh, bl, idesc, 1u);             //                  + Hi^T 2Lo
            if (vb == 256) {
              const uint64_t ah = umma_desc_sw128(r_s + 128u * 128u + 32u * k);
              umma_tf32(tmem + 256, ah, bh, idesc, first);  // rows 128..255
              umma_tf32(tmem + 256, ah, bl, idesc, 1u);
            }
          }
          umma_commit(&empty[s]);                 // ring slot free once these MMAs have read it
          if (t == nt - 1) umma_commit(accf);     // chunk complete: accumulators ready
          if (++s == kStages) { s = 0; ph ^= 1u; }
        }
      }
    }
  } else {
    // -------------------- split / g0 / epilogue (warps 2..9) --------------------
    const int ct = tid - 64;  // 0..255: the split of column ct (vb = 128: threads 0..127)
    const int quad = warp & 3;      // TMEM lane quadrant this warp may read
    const int whalf = (warp - 2) >> 2;  // which half of the column blocks it drains
    const bool splitter = ct < vb;
    const int ncol = vb / 128;  // accumulators (M halves)
    int s = 0;
    uint32_t ph = 0;
    int64_t it = 0;
    for (int64_t c = blockIdx.x; c < p.nchunks; c += gridDim.x, ++it) {
      double g0a[1] = {0.0}, d2a[1] = {0.0};
      const int nt = chunk_tiles(c);
      for (int t = 0; t < nt; ++t) {
        if (splitter) {
          if (!wait_phase(&full[s], ph, abort_flag, p.status)) goto done;
          unsigned char* r_t = raw + s * tile_bytes;
          unsigned char* l_t = lo + s * tile_bytes;
          const float* e_t = es + s * kTK;
          const int col = ct;
          // x_j . x_j and x_j . e over the tile's 32 rows in fp32 (FMA chains
          // of 32), then one widening add into the fp64 chunk totals
          float d2t = 0.f, g0t = 0.f;
#pragma unroll
          for (int q = 0; q < kTK / 4; ++q) {
            const uint32_t off = static_cast<uint32_t>(col) * 128u + ((static_cast<uint32_t>(q) ^ (col & 7)) << 4);
            float4 v = *reinterpret_cast<const float4*>(r_t + off);
            float4 hi, l2;
            hi.x = __uint_as_float(__float_as_uint(v.x) & 0xFFFFE000u);
            hi.y = __uint_as_float(__float_as_uint(v.y) & 0xFFFFE000u);
            hi.z = __uint_as_float(__float_as_uint(v.z) & 0xFFFFE000u);
            hi.w = __uint_as_float(__float_as_uint(v.w) & 0xFFFFE000u);
            l2.x = 2.f * (v.x - hi.x);
            l2.y = 2.f * (v.y - hi.y);
            l2.z = 2.f * (v.z - hi.z);
            l2.w = 2.f * (v.w - hi.w);
            *reinterpret_cast<float4*>(r_t + off) = hi;
            *reinterpret_cast<float4*>(l_t + off) = l2;
            d2t = __fmaf_rn(v.x, v.x, d2t);
            d2t = __fmaf_rn(v.y, v.y, d2t);
            d2t = __fmaf_rn(v.z, v.z, d2t);
            d2t = __fmaf_rn(v.w, v.w, d2t);
            if (p.with_e) {
              const float4 e4 = *reinterpret_cast<const float4*>(e_t + 4 * q);
              g0t = __fmaf_rn(v.x, e4.x, g0t);
              g0t = __fmaf_rn(v.y, e4.y, g0t);
              g0t = __fmaf_rn(v.z, e4.z, g0t);
              g0t = __fmaf_rn(v.w, e4.w, g0t);
            }
          }
          d2a[0] += static_cast<double>(d2t);
          if (p.with_e) g0a[0] += static_cast<double>(g0t);
          fence_async_smem();  // generic-proxy writes -> visible to the tensor core (async proxy)
          mbar_arrive(&conv[s]);
        }
        if (++s == kStages) { s = 0; ph ^= 1u; }
      }
      if (splitter) {
        double* g = p.cpart + c * 2 * vb;
        if (p.with_e) g[ct] = g0a[0];
        g[vb + ct] = d2a[0];
      }
      // epilogue: this chunk's S -> HBM (fp32), rows 32*quad + lane of each accumulator
      if (!wait_phase(accf, static_cast<uint32_t>(it & 1), abort_flag, p.status)) goto done;
      tc_fence_after();
      float* out = p.part + c * static_cast<int64_t>(vb) * vb;
      for (int a = 0; a < ncol; ++a) {
        const int row = a * 128 + quad * 32 + lane;
        float4* dst = reinterpret_cast<float4*>(out + static_cast<int64_t>(row) * vb);
        const int nblk = vb / 16;
        for (int cb = whalf * (nblk / 2); cb < (whalf + 1) * (nblk / 2); ++cb) {
          float v[16];
          tmem_ld16(tmem + (static_cast<uint32_t>(quad * 32) << 16) + static_cast<uint32_t>(a * 256 + cb * 16), v);
#pragma unroll
          for (int i = 0; i < 4; ++i) dst[cb * 4 + i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
        }
      }
      tc_fence_before();
      mbar_arrive(acce);
    }
  }
done:
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
  }
}

// red[g][e] = sum over chunks [g*per, (g+1)*per) of part[c][e], chunk order, fp64;
// the last 2*vb "elements" of each group row are the fp64 per-chunk
// x_j . e / x_j . x_j partials (cpart), reduced the same way
__global__ void gram_tc_reduce1(const float* __restrict__ part, const double* __restrict__ cpart, int64_t nchunks,
                                int64_t E, int vb, double* __restrict__ red) {
  const int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int g = blockIdx.y;
  const int64_t per = (nchunks + gridDim.y - 1) / gridDim.y;
  const int64_t c0 = g * per, c1 = imin64(nchunks, c0 + per);
  const int64_t W = E + 2 * vb;
  if (e >= W) return;
  double s = 0.0;
  if (e < E) {
    for (int64_t c = c0; c < c1; ++c) s += static_cast<double>(part[c * E + e]);
  } else {
    for (int64_t c = c0; c < c1; ++c) s += cpart[c * 2 * vb + (e - E)];
  }
  red[g * W + e] = s;
}

// G (vars x vars, column-major, symmetric) = (T + T^T)/2 off the diagonal,
// with T = sum of the groups in order; diag G = norms = the fp64 sums of
// x_j . x_j; g0 (one row) = the fp64 sums of x_j . e (groups in order)
__global__ void gram_tc_reduce2(const double* __restrict__ red, int ngroups, int vb, int64_t vars,
                                double* __restrict__ G, float* __restrict__ norms, double* __restrict__ g0) {
  const int64_t E = static_cast<int64_t>(vb) * vb, W = E + 2 * vb;
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx < vars * vars) {
    const int64_t i = idx % vars, j = idx / vars;  // G(i, j), column-major
    if (i == j) {
      double d = 0.0;
      for (int g = 0; g < ngroups; ++g) d += red[g * W + E + vb + i];
      G[j * vars + i] = d;
      if (norms) norms[i] = static_cast<float>(d);
    } else {
      double tij = 0.0, tji = 0.0;
      for (int g = 0; g < ngroups; ++g) {
        tij += red[g * W + i * vb + j];
        tji += red[g * W + j * vb + i];
      }
      G[j * vars + i] = 0.5 * (tij + tji);
    }
  }
  if (g0 && idx < vars) {
    double s = 0.0;
    for (int g = 0; g < ngroups; ++g) s += red[g * W + E + idx];
    g0[idx] = s;
  }
}

struct TcSplit {
  int vb;
  int64_t chunk_rows, nchunks;
  int64_t part_bytes, c_bytes, red_bytes;
};

TcSplit tc_split(int64_t obs, int64_t vars) {
  TcSplit t{};
  t.vb = vars <= 128 ? 128 : 256;
  const char* cr = getenv("BAK_GRAM_TC_CHUNK");
  t.chunk_rows = cr ? round_up(atoll(cr), kTK) : 1024;
  if (t.chunk_rows < kTK) t.chunk_rows = kTK;
  t.nchunks = (obs + t.chunk_rows - 1) / t.chunk_rows;
  const int64_t E = static_cast<int64_t>(t.vb) * t.vb;
  t.part_bytes = round_up(t.nchunks * E * 4, 256);
  t.c_bytes = round_up(t.nchunks * 2 * t.vb * 8, 256);
  t.red_bytes = round_up(kReduceGroups * (E + 2 * t.vb) * 8, 256);
  return t;
}

size_t tc_smem_bytes(int vb) {
  return 1024 + kStages * (2ull * vb * 128 + kTK * 4) + (3 * kStages + 2) * 8 + 16;
}

}  // namespace

bool gram_tc_enabled(int dtype, int64_t vars) {
  if (dtype != BAK_F32 || vars < 1 || vars > 256) return false;
  const char* gg = getenv("BAK_GRAM_G");
  if (gg && (gg[0] == 'd' || gg[0] == 'x')) return false;  // "dmma" / "x3": the mma.sync kernels
  return tensor_map_encoder() != nullptr;
}

int64_t gram_tc_workspace(int64_t obs, int64_t vars) {
  const TcSplit t = tc_split(obs, vars);
  return t.part_bytes + t.c_bytes + t.red_bytes;
}

int launch_gram_g_tc(const void* x, int64_t obs, int64_t ldx, int64_t vars, double* G, void* part_ws,
                     int64_t part_bytes, cudaStream_t st, void* norms_out, const void* e, double* g0,
                     int64_t* status) {
  const TcSplit t = tc_split(obs, vars);
  if (part_bytes < t.part_bytes + t.c_bytes + t.red_bytes) {
    set_error("gram (tcgen05): partial workspace too small");
    return BAK_EWORKSPACE;
  }
  auto enc = tensor_map_encoder();
  if (!enc) {
    set_error("cuTensorMapEncodeTiled unavailable");
    return BAK_ECUDA;
  }
  CUtensorMap xmap, emap;
  {
    cuuint64_t gdim[2] = {static_cast<cuuint64_t>(obs), static_cast<cuuint64_t>(vars)};
    cuuint64_t gstr[1] = {static_cast<cuuint64_t>(ldx * 4)};
    cuuint32_t box[2] = {static_cast<cuuint32_t>(kTK), static_cast<cuuint32_t>(t.vb)};
    cuuint32_t est[2] = {1, 1};
    CUresult r = enc(&xmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(x), gdim, gstr, box, est,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      set_error("cuTensorMapEncodeTiled (x, tcgen05 G) failed (%d)", static_cast<int>(r));
      return BAK_ECUDA;
    }
  }
  const bool with_e = e != nullptr && g0 != nullptr;
  {
    // e as an obs x 1 matrix (a 2-D map, as for x)
    const void* ep = with_e ? e : x;  // a valid map either way (unused without e)
    cuuint64_t gdim[2] = {static_cast<cuuint64_t>(obs), 1};
    cuuint64_t gstr[1] = {static_cast<cuuint64_t>(round_up(obs * 4, 16))};
    cuuint32_t box[2] = {static_cast<cuuint32_t>(kTK), 1};
    cuuint32_t est[2] = {1, 1};
    CUresult r = enc(&emap, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(ep), gdim, gstr, box, est,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      set_error("cuTensorMapEncodeTiled (e, tcgen05 G) failed (%d)", static_cast<int>(r));
      return BAK_ECUDA;
    }
  }
  char* w = static_cast<char*>(part_ws);
  float* part = reinterpret_cast<float*>(w);
  double* cpart = reinterpret_cast<double*>(w + t.part_bytes);
  double* red = reinterpret_cast<double*>(w + t.part_bytes + t.c_bytes);
  TcParams p{obs, t.vb, t.nchunks, t.chunk_rows, part, cpart, with_e ? 1 : 0, status};
  const size_t smem = tc_smem_bytes(t.vb);
  BAK_CHECK_CUDA(cudaFuncSetAttribute(gram_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(smem)));
  const int grid = static_cast<int>(imin64(t.nchunks, device_sms()));
  gram_tc_kernel<<<grid, kThreads, smem, st>>>(xmap, emap, p);
  BAK_CHECK_CUDA(cudaGetLastError());
  const int64_t E = static_cast<int64_t>(t.vb) * t.vb;
  const int groups = static_cast<int>(imin64(kReduceGroups, t.nchunks));
  gram_tc_reduce1<<<dim3(static_cast<unsigned>((E + 2 * t.vb + 255) / 256), groups), 256, 0, st>>>(
      part, cpart, t.nchunks, E, t.vb, red);
  BAK_CHECK_CUDA(cudaGetLastError());
  const int64_t n2 = vars * vars;
  gram_tc_reduce2<<<static_cast<unsigned>((n2 + 255) / 256), 256, 0, st>>>(
      red, groups, t.vb, vars, G, static_cast<float*>(norms_out), with_e ? g0 : nullptr);
  BAK_CHECK_CUDA(cudaGetLastError());
  count_launches(3);
  return BAK_OK;
}

}  // namespace bak

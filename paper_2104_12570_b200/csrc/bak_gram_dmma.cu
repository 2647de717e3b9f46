// G = X^T X for the GRAM variant: hand-written fp64 tensor-core (DMMA,
// mma.sync.m8n8k4.f64) SYRK over column-major x, fp64 accumulation for both
// input precisions (fp32 inputs are widened exactly when fragments are read).
//
// Only the lower block triangle of 64x64 blocks is computed (bi >= bj), split
// over K (rows of x) into chunks; a CTA = 4 warps owns one (block, chunk) and
// each warp a 32x32 quarter = 4x4 DMMA tiles.  Panels of 32 rows x 64 columns
// stream through a 3-stage cp.async ring (zero-filled past obs / vars); panel
// layout is column-major with a 36-element column stride so that the
// m8n8k4 fragment loads (8 columns x 4 rows per warp) are bank-conflict free.
// Partials per chunk are summed in chunk order (deterministic) and mirrored.
#include "bak_common.cuh"
#include "bak_sweep.cuh"

namespace bak {
namespace {

constexpr int kBT = 64;       // G block edge
constexpr int kKT = 32;       // rows per panel stage
constexpr int kLd = 36;       // smem column stride (elements)
constexpr int kStages = 3;
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

struct GramParams {
  const void* x;
  int64_t obs, ldx, vars;
  int nb;            // number of 64-column blocks
  int nchunks;       // K split
  int64_t chunk;     // rows per chunk (multiple of kKT)
  double* part;      // [nchunks][nblocks_lower][64*64]
};

// block index -> (bi, bj) with bi >= bj, row-major over the lower triangle
__device__ __forceinline__ void tri_index(int b, int& bi, int& bj) {
  bi = 0;
  while ((bi + 1) * (bi + 2) / 2 <= b) ++bi;
  bj = b - bi * (bi + 1) / 2;
}

template <typename T>
__global__ void __launch_bounds__(kThreads, 2) gram_dmma_kernel(const GramParams p) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  T* pa = reinterpret_cast<T*>(smem_raw);                  // [stages][64][kLd]
  T* pb = pa + static_cast<size_t>(kStages) * kBT * kLd;  // [stages][64][kLd]
  const int nblk = p.nb * (p.nb + 1) / 2;
  const int blk = blockIdx.x % nblk;  // blocks of one chunk are adjacent: shared rows hit in L2
  const int chk = blockIdx.x / nblk;
  int bi, bj;
  tri_index(blk, bi, bj);
  const bool diag = bi == bj;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wi = (warp >> 1) * 32, wj = (warp & 1) * 32;  // warp's quarter of the block
  const T* __restrict__ x = static_cast<const T*>(p.x);
  const int64_t k_begin = static_cast<int64_t>(chk) * p.chunk;
  const int64_t k_end = imin64(p.obs, k_begin + p.chunk);
  const int nsteps = static_cast<int>((k_end - k_begin + kKT - 1) / kKT);
  constexpr int kPer = 16 / sizeof(T);               // elements per 16-byte piece
  constexpr int kPieces = kKT / kPer;                // pieces per column per stage
  constexpr int kCopies = kBT * kPieces / kThreads;  // per thread per panel

  auto load_stage = [&](int step, int slot) {
    const int64_t k0 = k_begin + static_cast<int64_t>(step) * kKT;
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
        cp_async16(pa + (static_cast<size_t>(slot) * kBT + col) * kLd + piece * kPer, src, bytes);
      }
      if (!diag) {
        const int64_t gc = static_cast<int64_t>(bj) * kBT + col;
        const int bytes = (gc < p.vars && rem > 0) ? static_cast<int>(imin64(rem, kPer) * sizeof(T)) : 0;
        const T* src = bytes ? x + gc * p.ldx + row : x;
        cp_async16(pb + (static_cast<size_t>(slot) * kBT + col) * kLd + piece * kPer, src, bytes);
      }
    }
  };

  double acc[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

#pragma unroll
  for (int s = 0; s < kStages - 1; ++s) {
    if (s < nsteps) load_stage(s, s);
    cp_async_commit();
  }
  const int fr = lane >> 2, fk = lane & 3;  // fragment row/col within an 8x4 tile
  for (int step = 0; step < nsteps; ++step) {
    cp_async_wait<kStages - 2>();
    __syncthreads();
    {
      const int nxt = step + kStages - 1;
      if (nxt < nsteps) load_stage(nxt, nxt % kStages);
      cp_async_commit();
    }
    const int slot = step % kStages;
    const T* A = pa + static_cast<size_t>(slot) * kBT * kLd;
    const T* B = diag ? A : pb + static_cast<size_t>(slot) * kBT * kLd;
#pragma unroll
    for (int k4 = 0; k4 < kKT; k4 += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        af[t] = static_cast<double>(A[(wi + t * 8 + fr) * kLd + k4 + fk]);
        bf[t] = static_cast<double>(B[(wj + t * 8 + fr) * kLd + k4 + fk]);
      }
      if (!(diag && wj > wi)) {  // the upper quadrant of a diagonal block is never used
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) dmma(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
      }
    }
  }
  cp_async_wait<0>();
  double* out = p.part + (static_cast<size_t>(chk) * nblk + blk) * kBT * kBT;
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int i = wi + a * 8 + fr, j = wj + b * 8 + fk * 2;
      out[i * kBT + j] = acc[a][b][0];
      out[i * kBT + j + 1] = acc[a][b][1];
    }
}

// G (vars x vars, full, symmetric) = sum over chunks of the lower block partials
template <typename T>
__global__ void gram_reduce_kernel(const double* __restrict__ part, int nchunks, int nb, int64_t V,
                                   double* __restrict__ G, T* __restrict__ norms) {
  const int nblk = nb * (nb + 1) / 2;
  const int blk = blockIdx.y;
  int bi = 0;
  while ((bi + 1) * (bi + 2) / 2 <= blk) ++bi;
  const int bj = blk - bi * (bi + 1) / 2;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < kBT * kBT; e += gridDim.x * blockDim.x) {
    const int i = e / kBT, j = e % kBT;
    const int64_t gi = static_cast<int64_t>(bi) * kBT + i, gj = static_cast<int64_t>(bj) * kBT + j;
    if (gi >= V || gj >= V) continue;
    if (bi == bj && j > i) continue;  // diagonal block: lower half (mirrored below)
    double s = 0.0;
    for (int c = 0; c < nchunks; ++c) s += part[(static_cast<size_t>(c) * nblk + blk) * kBT * kBT + e];
    G[gj * V + gi] = s;  // column-major (gi, gj)
    G[gi * V + gj] = s;  // mirror (gj, gi)
    if (norms && gi == gj) norms[gi] = static_cast<T>(s);  // n2_j = G_jj (fp64-accumulated)
  }
}

}  // namespace

int64_t gram_g_workspace(int64_t obs, int64_t vars, int& nchunks, int64_t& chunk) {
  const int nb = static_cast<int>((vars + kBT - 1) / kBT);
  const int nblk = nb * (nb + 1) / 2;
  // one wave: 2 CTAs per SM (smem-bound), every CTA one block x one K-range
  const int slots = 2 * device_sms();
  nchunks = slots / nblk;
  if (nchunks < 1) nchunks = 1;
  chunk = round_up((obs + nchunks - 1) / nchunks, kKT);
  nchunks = static_cast<int>((obs + chunk - 1) / chunk);
  if (nchunks < 1) nchunks = 1;
  return static_cast<int64_t>(nchunks) * nblk * kBT * kBT * 8;
}

int launch_gram_g(int dtype, const void* x, int64_t obs, int64_t ldx, int64_t vars, double* G, void* part_ws,
                  int64_t part_bytes, cudaStream_t st, void* norms_out) {
  int nchunks;
  int64_t chunk;
  const int64_t need = gram_g_workspace(obs, vars, nchunks, chunk);
  if (part_bytes < need) {
    set_error("gram: partial workspace too small");
    return BAK_EWORKSPACE;
  }
  const int nb = static_cast<int>((vars + kBT - 1) / kBT);
  const int nblk = nb * (nb + 1) / 2;
  GramParams p{x, obs, ldx, vars, nb, nchunks, chunk, static_cast<double*>(part_ws)};
  const size_t ts = dtype == BAK_F64 ? 8 : 4;
  const size_t smem = 2ull * kStages * kBT * kLd * ts;
  const unsigned grid = static_cast<unsigned>(nchunks * nblk);
  if (dtype == BAK_F64) {
    BAK_CHECK_CUDA(cudaFuncSetAttribute(gram_dmma_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(smem)));
    gram_dmma_kernel<double><<<grid, kThreads, smem, st>>>(p);
  } else {
    BAK_CHECK_CUDA(cudaFuncSetAttribute(gram_dmma_kernel<float>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(smem)));
    gram_dmma_kernel<float><<<grid, kThreads, smem, st>>>(p);
  }
  count_launches(1);
  BAK_CHECK_CUDA(cudaGetLastError());
  if (dtype == BAK_F64)
    gram_reduce_kernel<double><<<dim3(16, nblk), 256, 0, st>>>(static_cast<const double*>(part_ws), nchunks, nb, vars,
                                                               G, static_cast<double*>(norms_out));
  else
    gram_reduce_kernel<float><<<dim3(16, nblk), 256, 0, st>>>(static_cast<const double*>(part_ws), nchunks, nb, vars,
                                                              G, static_cast<float*>(norms_out));
  count_launches(1);
  BAK_CHECK_CUDA(cudaGetLastError());
  return BAK_OK;
}

}  // namespace bak

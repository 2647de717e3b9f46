// Shared host/device structures of the sweep kernels.
#pragma once
#include <cstdint>

#include <cuda_runtime.h>

namespace bak {

// grid exchange workspace: [2 bufs][kGridSlotsMax] 32-byte partial records +
// [2 bufs][kGridSlotsMax] 128-byte result lines (one per CTA)
constexpr int kGridSlotsMax = 256;
constexpr int64_t kGridSlotBytes = 2LL * kGridSlotsMax * 32 + 2LL * kGridSlotsMax * 128;

struct SweepParams {
  const void* x;
  int64_t obs, ldx;
  const void* norms2;
  const int32_t* cols;
  int64_t ncols, cols_stride;
  void* e;
  void* a;
  int64_t max_iter;
  double thresh2;  // < 0: no early break
  double* history;
  int64_t* status;
  uint32_t* slots;  // grid exchange records (workspace)
  int64_t rows_per_cta;
  int64_t stage_elems;
  int nstages;
  int keep_next;  // STREAM: keep x_{j+1} in L2 for the next column step
  int grid_allgather = 0;  // GRID one-level: every CTA gathers all records (no aggregator round trip)
  // Row sharding over GPUs (bak_sweep_rowshard, two-level GRID plans only): x, e
  // are this rank's rows; after the rank's clusters have reduced, the cluster-0
  // leader posts the rank total into every rank's mailbox and every leader sums
  // the nranks totals in rank order.  nranks = 0: single device.
  uint32_t* mbox[8] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};
  int nranks = 0;
  int grank = 0;
  uint32_t epoch_base = 0;
};

struct SweepPlan {
  int variant = 0;
  int nparticipants = 1;  // CTAs cooperating on one system
  int nthreads = 32;
  int e = 1;  // rows per thread
  int nstages = 2;
  int64_t rows_per_cta = 0;
  int64_t stage_elems = 0;
  int cluster = 0;  // GRID: CTAs per cluster of the two-level exchange (0 = one level)
  int xs = 0;       // GRID: x read from a quarter-column shared-memory ring (rows past register capacity)
};

// force_flat: GRID plans use the one-level exchange (as BAK_GRID_FLAT=1)
bool plan_onchip(int dtype, int variant, int64_t obs, SweepPlan& pl, bool force_flat = false);
int launch_onchip(int dtype, const SweepPlan& pl, const SweepParams& prm, cudaStream_t st);

// e streamed through HBM (tall systems past on-chip capacity)
struct StreamPlan {
  int nblocks = 0;
  int nthreads = 512;
  int64_t rows_per_cta = 0;
};
bool plan_stream(int dtype, int64_t obs, StreamPlan& pl);
int launch_stream(int dtype, const StreamPlan& pl, const SweepParams& prm, cudaStream_t st);

// GRAM variant (algebraically equivalent sweep through G = X^T X)
int64_t gram_workspace_bytes(int dtype, int64_t obs, int64_t vars);
bool gram_supported(int64_t vars);
// G = X^T X workspace; nchunks = rows of the fused first-sweep g0 partials
int64_t gram_g_workspace(int dtype, int64_t obs, int64_t vars, int& nchunks, int64_t& chunk);
// tcgen05 (kind::tf32) G for fp32 inputs, vars <= 256 (bak_gram_tc.cu)
bool gram_tc_enabled(int dtype, int64_t vars);
int64_t gram_tc_workspace(int64_t obs, int64_t vars);
int launch_gram_g_tc(const void* x, int64_t obs, int64_t ldx, int64_t vars, double* G, void* part_ws,
                     int64_t part_bytes, cudaStream_t st, void* norms_out, const void* e, double* g0,
                     int64_t* status);
int launch_gram_g(int dtype, const void* x, int64_t obs, int64_t ldx, int64_t vars, double* G, void* part_ws,
                  int64_t part_bytes, cudaStream_t st, void* norms_out = nullptr, const void* e = nullptr,
                  double* g0 = nullptr, int64_t* status = nullptr);
bool gram_tma_supported(int64_t vars);
int gram_tma_grid(int dtype);
int launch_gram_pass_tma(int dtype, const void* x, int64_t obs, int64_t ldx, int64_t vars, void* e,
                         const double* delta, int apply, int dot, double* gpart, double* sqpart, const int64_t* done,
                         cudaStream_t st, const void* afin = nullptr, const void* y = nullptr, void* resid = nullptr,
                         int64_t* status = nullptr);
int launch_gram(int dtype, const SweepParams& prm, int64_t vars, void* ws, int64_t wsb, cudaStream_t st);
// block-Gram sweep (bak_bgram.cu): residual on one cluster, cyclic order
int64_t bgram_workspace_bytes(int64_t vars);
bool bgram_supported(int dtype, int64_t obs);
int launch_bgram(int dtype, const SweepParams& prm, int64_t vars, void* ws, int64_t wsb, cudaStream_t st);

}  // namespace bak

// Shared host/device structures of the sweep kernels.
#pragma once
#include <cstdint>

#include <cuda_runtime.h>

namespace bak {

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
};

struct SweepPlan {
  int variant = 0;
  int nparticipants = 1;  // CTAs cooperating on one system
  int nthreads = 32;
  int e = 1;  // rows per thread
  int nstages = 2;
  int64_t rows_per_cta = 0;
  int64_t stage_elems = 0;
};

bool plan_onchip(int dtype, int variant, int64_t obs, SweepPlan& pl);
int launch_onchip(int dtype, const SweepPlan& pl, const SweepParams& prm, cudaStream_t st);

// e streamed through HBM (tall systems past on-chip capacity)
struct StreamPlan {
  int nblocks = 0;
  int nthreads = 512;
  int64_t rows_per_cta = 0;
};
bool plan_stream(int dtype, int64_t obs, StreamPlan& pl);
int launch_stream(int dtype, const StreamPlan& pl, const SweepParams& prm, cudaStream_t st);

}  // namespace bak

// C-ABI entry points and host utilities (error text, device queries, sweep
// dispatch).  See include/bak200.h for the contract of every symbol.
#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <atomic>

#include "bak_common.cuh"
#include "bak_sweep.cuh"

namespace bak {

static thread_local char g_err[512] = "";
static std::atomic<int64_t> g_launches{0};
void count_launches(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

void g_err_clear() { g_err[0] = 0; }

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int cuda_fail(cudaError_t err, const char* what) {
  set_error("CUDA error %d (%s) in %s", static_cast<int>(err), cudaGetErrorString(err), what);
  cudaGetLastError();  // a failed launch must not poison the next call's error check
  return BAK_ECUDA;
}

static int cached_attr(cudaDeviceAttr attr, int fallback, int* cache) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return fallback;
  if (cache[dev] > 0) return cache[dev];
  int v = 0;
  if (cudaDeviceGetAttribute(&v, attr, dev) != cudaSuccess || v <= 0) {
    cudaGetLastError();
    return fallback;
  }
  cache[dev] = v;
  return v;
}

int device_sms() {
  static int cache[64] = {0};
  return cached_attr(cudaDevAttrMultiProcessorCount, 148, cache);
}

int device_max_smem_optin() {
  static int cache[64] = {0};
  return cached_attr(cudaDevAttrMaxSharedMemoryPerBlockOptin, 232448, cache);
}

// Cooperative launches with thread-block clusters (the two-level exchanges)
// cannot be replayed by a profiler that injects itself into the process
// (ncu sets NV_NSIGHT_INJECTION_TRANSPORT_TYPE / NV_TPS_LAUNCH_TOKEN, other
// tools CUDA_INJECTION64_PATH): use the one-level exchanges there.
bool coop_clusters_ok() {
  static int ok = -1;
  if (ok < 0)
    ok = (getenv("CUDA_INJECTION64_PATH") == nullptr && getenv("NV_NSIGHT_INJECTION_TRANSPORT_TYPE") == nullptr &&
          getenv("NV_TPS_LAUNCH_TOKEN") == nullptr && getenv("BAK_NO_COOP_CLUSTERS") == nullptr)
             ? 1
             : 0;
  return ok == 1;
}

int64_t l2_bytes() {
  static int cache[64] = {0};
  return cached_attr(cudaDevAttrL2CacheSize, 126 << 20, cache);
}

}  // namespace bak

using namespace bak;

namespace {
constexpr int64_t kSlotBytes = kGridSlotBytes;  // grid / stream exchange records

int pick_variant(int dtype, int64_t obs) {
  SweepPlan pl;
  if (obs <= 1024 && plan_onchip(dtype, BAK_VARIANT_CTA, obs, pl)) return BAK_VARIANT_CTA;
  if (obs <= 16 * 256 * 8 && plan_onchip(dtype, BAK_VARIANT_CLUSTER, obs, pl)) return BAK_VARIANT_CLUSTER;
  if (plan_onchip(dtype, BAK_VARIANT_GRID, obs, pl)) return BAK_VARIANT_GRID;
  return BAK_VARIANT_STREAM;
}
}  // namespace

extern "C" const char* bak_last_error(void) { return g_err; }
extern "C" int64_t bak_launch_count(void) { return g_launches.load(); }
extern "C" const char* bak_version(void) { return "bak200 0.1.0 (sm_100a)"; }
extern "C" int bak_device_sm_count(void) {
  int dev = 0, v = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return -1;
  return v;
}

extern "C" int bak_sweep_pick_variant(int dtype, int64_t obs, int64_t vars) {
  (void)vars;
  return pick_variant(dtype, obs);
}

extern "C" int64_t bak_sweep_workspace(int dtype, int variant, int64_t obs, int64_t vars) {
  if (variant == BAK_VARIANT_GRAM) {
    const int64_t g = gram_workspace_bytes(dtype, obs, vars);
    return g > kSlotBytes ? g : kSlotBytes;
  }
  if (variant == BAK_VARIANT_BGRAM) {
    const int64_t g = bgram_workspace_bytes(vars);
    return g > kSlotBytes ? g : kSlotBytes;
  }
  return kSlotBytes;
}

extern "C" int bak_sweep(int dtype, int variant, const void* x, int64_t obs, int64_t vars, int64_t ldx,
                         const void* norms2, const int32_t* cols, int64_t ncols, int64_t cols_stride, void* e,
                         void* a, int64_t max_iter, double thresh2, double* history, int64_t* status,
                         void* workspace, int64_t workspace_bytes, void* stream) {
  g_err[0] = 0;
  if (dtype != BAK_F32 && dtype != BAK_F64) {
    set_error("bak_sweep: unknown dtype %d", dtype);
    return BAK_EINVAL;
  }
  const size_t ts = dtype_size(dtype);
  if (obs < 1 || vars < 1 || ldx < obs || ncols < 1 || max_iter < 1 || !x || !norms2 || !e || !a || !status) {
    set_error("bak_sweep: bad arguments (obs=%lld vars=%lld ldx=%lld ncols=%lld max_iter=%lld)", (long long)obs,
              (long long)vars, (long long)ldx, (long long)ncols, (long long)max_iter);
    return BAK_EINVAL;
  }
  if (!cols && ncols != vars) {
    set_error("bak_sweep: cols == NULL requires ncols == vars");
    return BAK_EINVAL;
  }
  if (reinterpret_cast<uintptr_t>(x) % 16 != 0 || (ldx * static_cast<int64_t>(ts)) % 16 != 0) {
    set_error("bak_sweep: x must be 16-byte aligned with ldx*sizeof(T) a multiple of 16 (ldx=%lld)", (long long)ldx);
    return BAK_EINVAL;
  }
  if (!workspace || workspace_bytes < kSlotBytes) {
    set_error("bak_sweep: workspace too small (need %lld bytes)", (long long)kSlotBytes);
    return BAK_EWORKSPACE;
  }
  if (variant == BAK_VARIANT_AUTO) variant = pick_variant(dtype, obs);
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  BAK_CHECK_CUDA(cudaMemsetAsync(status, 0, 4 * sizeof(int64_t), st));
  SweepParams prm{};
  prm.x = x;
  prm.obs = obs;
  prm.ldx = ldx;
  prm.norms2 = norms2;
  prm.cols = cols;
  prm.ncols = ncols;
  prm.cols_stride = cols_stride;
  prm.e = e;
  prm.a = a;
  prm.max_iter = max_iter;
  prm.thresh2 = thresh2;
  prm.history = history;
  prm.status = status;
  prm.slots = static_cast<uint32_t*>(workspace);
  if (variant == BAK_VARIANT_GRAM) return launch_gram(dtype, prm, vars, workspace, workspace_bytes, st);
  if (variant == BAK_VARIANT_BGRAM) return launch_bgram(dtype, prm, vars, workspace, workspace_bytes, st);
  if (variant == BAK_VARIANT_STREAM) {
    StreamPlan sp;
    if (!plan_stream(dtype, obs, sp)) {
      set_error("bak_sweep: no STREAM plan for obs=%lld", (long long)obs);
      return BAK_EUNSUPPORTED;
    }
    return launch_stream(dtype, sp, prm, st);
  }
  if (variant == BAK_VARIANT_CTA || variant == BAK_VARIANT_CLUSTER || variant == BAK_VARIANT_GRID) {
    SweepPlan pl;
    if (!plan_onchip(dtype, variant, obs, pl)) {
      set_error("bak_sweep: variant %d cannot hold obs=%lld rows on chip", variant, (long long)obs);
      return BAK_EUNSUPPORTED;
    }
    prm.rows_per_cta = pl.rows_per_cta;
    prm.stage_elems = pl.stage_elems;
    prm.nstages = pl.nstages;
    if (getenv("BAK_DEBUG"))
      fprintf(stderr, "bak: plan variant=%d parts=%d threads=%d e=%d stages=%d rows/cta=%lld cluster=%d xs=%d\n",
              pl.variant, pl.nparticipants, pl.nthreads, pl.e, pl.nstages, (long long)pl.rows_per_cta, pl.cluster,
              pl.xs);
    return launch_onchip(dtype, pl, prm, st);
  }
  set_error("bak_sweep: variant %d not available", variant);
  return BAK_EUNSUPPORTED;
}

// Row-block host->device copy of a column-major matrix (pipelined uploads):
// rows [r0, r0+rows) of every column, one 2-D copy (rows*elem bytes x vars).
extern "C" int bak_copy_rows_h2d(void* dst, int64_t dld, const void* src, int64_t sld, int64_t r0, int64_t rows,
                                 int64_t vars, int64_t elem, void* stream) {
  if (!dst || !src || rows < 0 || vars < 1 || elem < 1 || dld < r0 + rows || sld < r0 + rows) {
    set_error("bak_copy_rows_h2d: bad arguments");
    return BAK_EINVAL;
  }
  if (rows == 0) return BAK_OK;
  BAK_CHECK_CUDA(cudaMemcpy2DAsync(static_cast<char*>(dst) + r0 * elem, dld * elem,
                                   static_cast<const char*>(src) + r0 * elem, sld * elem, rows * elem, vars,
                                   cudaMemcpyHostToDevice, static_cast<cudaStream_t>(stream)));
  return BAK_OK;
}

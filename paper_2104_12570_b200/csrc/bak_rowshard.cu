// (5) multi-GPU row sharding: peer mailboxes + IPC helpers.
#include "bak_common.cuh"

using namespace bak;

extern "C" int64_t bak_mailbox_bytes(int64_t nranks) { return nranks < 1 ? 0 : 2 * nranks * 32; }

extern "C" int bak_sweep_rowshard(int dtype, const void* x, int64_t obs_local, int64_t vars, int64_t ldx,
                                  const void* norms2, void* e, void* a, int64_t max_iter, double thresh2,
                                  double* history, int64_t* status, int rank, int nranks, void* const* mailboxes,
                                  int64_t epoch_base, int nranks_local, void* workspace, int64_t workspace_bytes,
                                  void* stream) {
  (void)dtype; (void)x; (void)obs_local; (void)vars; (void)ldx; (void)norms2; (void)e; (void)a; (void)max_iter;
  (void)thresh2; (void)history; (void)status; (void)rank; (void)nranks; (void)mailboxes; (void)epoch_base;
  (void)nranks_local; (void)workspace; (void)workspace_bytes; (void)stream;
  set_error("bak_sweep_rowshard: not built yet");
  return BAK_EUNSUPPORTED;
}

extern "C" int bak_ipc_get_handle(void* devptr, void* handle64) {
  cudaIpcMemHandle_t h;
  BAK_CHECK_CUDA(cudaIpcGetMemHandle(&h, devptr));
  static_assert(sizeof(h) == 64, "CUDA IPC handle is 64 bytes");
  memcpy(handle64, &h, 64);
  return BAK_OK;
}

extern "C" int bak_ipc_open_handle(const void* handle64, void** devptr) {
  cudaIpcMemHandle_t h;
  memcpy(&h, handle64, 64);
  BAK_CHECK_CUDA(cudaIpcOpenMemHandle(devptr, h, cudaIpcMemLazyEnablePeerAccess));
  return BAK_OK;
}

extern "C" int bak_ipc_close(void* devptr) {
  BAK_CHECK_CUDA(cudaIpcCloseMemHandle(devptr));
  return BAK_OK;
}

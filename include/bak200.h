/*
 * bak200 — B200-native (sm_100a) SolveBak column sweep, C ABI.
 *
 * The reference (baksolve 0.1.0, /root/reference/pkg) is pure Python and has
 * no FFI: its operator API for this path is the Python call
 *     baksolve.bak.solve_bak(x, y, config, a0) -> SolveReport   (bak.py:146-195)
 * Each entry point below replaces one piece of that call, so a maintainer
 * binds them with ctypes exactly as paper_2104_12570_b200
 * does.  All pointers are DEVICE pointers unless stated; sizes are int64_t;
 * `stream` is a cudaStream_t passed as void*.  Every call is asynchronous on
 * `stream` and returns 0 on success or a BAK_E* code; bak_last_error() gives a
 * thread-local message.  No call allocates device memory: callers pass a
 * workspace sized by the matching *_workspace() query.
 *
 * Layout: x is column-major (obs x vars) with leading dimension ldx >= obs.
 * Sweep kernels stream columns with cp.async.bulk and therefore require x to be
 * 16-byte aligned and ldx*sizeof(T) to be a multiple of 16 (pad rows up to ldx
 * may hold anything; they are masked).
 */
#ifndef BAK200_H_
#define BAK200_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* dtype codes (reference precisions "single"/"double", core.py:13) */
#define BAK_F32 0
#define BAK_F64 1

/* sweep variants */
#define BAK_VARIANT_AUTO    0 /* pick by shape                                      */
#define BAK_VARIANT_CTA     1 /* one CTA: e in registers, block reduction per column */
#define BAK_VARIANT_CLUSTER 2 /* 2..16-CTA cluster: DSMEM st.async reduction         */
#define BAK_VARIANT_GRID    3 /* persistent co-resident grid, e on chip, flag slots  */
#define BAK_VARIANT_STREAM  4 /* persistent grid, e streamed through HBM             */
#define BAK_VARIANT_GRAM    5 /* algebraically equal sweep via G = X^T X (labelled)  */
#define BAK_VARIANT_BGRAM   6 /* block-Gram: 64-column blocks, one reduction each,
                                  d_B = L_B^{-1} X_B^T e (labelled; cyclic order)   */

/* status codes */
#define BAK_OK           0
#define BAK_EINVAL       1 /* bad argument / layout                      */
#define BAK_ECUDA        2 /* CUDA runtime error                          */
#define BAK_ETIMEOUT     3 /* device-side spin wait exceeded its deadline */
#define BAK_EUNSUPPORTED 4 /* shape/variant combination not supported     */
#define BAK_EWORKSPACE   5 /* workspace too small                         */
#define BAK_EDIVERGED    6 /* device status only: the blocked sweep's divergence
                              guard tripped (bakp.py:121-124)             */

/* Thread-local text of the last error ("" if none). */
const char* bak_last_error(void);
/* Library version string. */
const char* bak_version(void);
/* Kernels this library has launched in this process (monotone counter). */
int64_t bak_launch_count(void);
/* Number of SMs of the current device (launch sizing), or -1. */
int bak_device_sm_count(void);

/* ---- (1) column-norm precompute -------------------------------------------
 * norms2[j] = <x_j, x_j> in T.  Replaces core.column_norms_sq (core.py:116-127)
 * called at bak.py:185; with vars=1 it is also ||y||^2 (bak.py:168). */
int64_t bak_colnorms_workspace(int dtype, int64_t obs, int64_t vars);
int bak_colnorms(int dtype, const void* x, int64_t obs, int64_t vars, int64_t ldx,
                 void* norms2, void* workspace, int64_t workspace_bytes, void* stream);

/* ---- residual / warm start -------------------------------------------------
 * out[i] = y[i] - (x @ a)[i] in T.  Replaces `y - x @ a` at bak.py:130 (final
 * residual, _finish_report) and bak.py:189 (warm start with a0). */
int64_t bak_residual_workspace(int dtype, int64_t obs, int64_t vars);
int bak_residual(int dtype, const void* x, int64_t obs, int64_t vars, int64_t ldx,
                 const void* a, const void* y, void* out,
                 void* workspace, int64_t workspace_bytes, void* stream);

/* out_f64[0] = sum_i double(u[i] - v[i])^2 : the drift norm of bak.py:133. */
int bak_diff_norm2(int dtype, const void* u, const void* v, int64_t n, double* out_f64,
                   void* workspace, int64_t workspace_bytes, void* stream);

/* ---- (2)/(3) persistent column sweep --------------------------------------
 * Runs up to max_iter sweeps of the column step (bak.py:82-89) over the column
 * list, checking sum(e^2) <= thresh2 after every sweep (bak.py:106-111).
 *   cols      : NULL -> columns 0..ncols-1 every sweep (ncols must equal vars);
 *               else int32 column indices, ncols per sweep; sweep s reads
 *               cols + s*cols_stride (cols_stride 0 = same list every sweep).
 *               Zero-norm columns must already be removed (bak.py:101-103).
 *   e, a      : updated in place (e maintained residual, a coefficients).
 *   thresh2   : early-break threshold tol^2*||y||^2; < 0 disables (tol == 0).
 *   history   : NULL or double[max_iter] per-sweep sum(e^2) (bak.py:106-108).
 *   status    : int64[4] device: {sweeps_run, converged, error, variant_used}.
 */
int64_t bak_sweep_workspace(int dtype, int variant, int64_t obs, int64_t vars);
int bak_sweep(int dtype, int variant,
              const void* x, int64_t obs, int64_t vars, int64_t ldx,
              const void* norms2,
              const int32_t* cols, int64_t ncols, int64_t cols_stride,
              void* e, void* a,
              int64_t max_iter, double thresh2,
              double* history, int64_t* status,
              void* workspace, int64_t workspace_bytes, void* stream);
/* Variant AUTO would pick for this shape (for reporting). */
int bak_sweep_pick_variant(int dtype, int64_t obs, int64_t vars);

/* ---- GRAM building blocks (BAK_VARIANT_GRAM, exposed for row sharding) -------
 * The labelled, algebraically equivalent sweep: one pass over x per sweep
 * (e -= X d; sum e^2; g = X^T e) plus a forward substitution with G = X^T X.
 * bak_gram_matrix : G (vars x vars, fp64, full symmetric) of the given rows.
 * bak_gram_pass   : writes bak_gram_pass_blocks(dtype, vars) partial rows of g
 *                   (gpart[b*vars + j]) and of sum e^2 (sqpart[b]); no-op when
 *                   *done_flag != 0.  apply=0: no update; dot=0: no g.
 * bak_gram_solve  : sums nparts partials in index order, finalizes sweep-1
 *                   (history, early break -> ctrl[0]=done, ctrl[1]=sweeps,
 *                   ctrl[2]=converged; status as bak_sweep) and, unless done,
 *                   computes d for `sweep` (a += d, delta = d). ctrl: int64[4],
 *                   zeroed by the caller before the first solve. */
int bak_gram_pass_blocks(int dtype, int64_t vars);
int64_t bak_gram_matrix_workspace(int dtype, int64_t obs, int64_t vars);
int bak_gram_matrix(int dtype, const void* x, int64_t obs, int64_t vars, int64_t ldx, double* G,
                    void* workspace, int64_t workspace_bytes, void* stream);
/* G as bak_gram_matrix plus, fused into the same kernel, the first sweep's
 * g = X^T e as bak_gram_dot_rows(dtype, obs, vars) partial rows
 * (g0[r*vars + j], summed in row order by bak_gram_solve); e 16-byte aligned.
 * Replaces bak_gram_matrix + bak_gram_pass(apply=0, dot=1): one read of x. */
int64_t bak_gram_dot_rows(int dtype, int64_t obs, int64_t vars);
int bak_gram_matrix_dot(int dtype, const void* x, int64_t obs, int64_t vars, int64_t ldx, double* G,
                        const void* e, double* g0, void* workspace, int64_t workspace_bytes, void* stream);
/* status (int64[4] as bak_sweep, may be NULL): a pipeline wait past its
 * deadline sets status[2] = BAK_ETIMEOUT (the pass results are then invalid). */
int bak_gram_pass(int dtype, const void* x, int64_t obs, int64_t vars, int64_t ldx, void* e,
                  const double* delta, int apply, int dot, double* gpart, double* sqpart,
                  const int64_t* done_flag, int64_t* status, void* stream);
/* bak_gram_pass + (afin != NULL) resid = y - x @ afin fused into the same pass. */
int bak_gram_pass_resid(int dtype, const void* x, int64_t obs, int64_t vars, int64_t ldx, void* e,
                        const double* delta, int apply, int dot, double* gpart, double* sqpart,
                        const int64_t* done_flag, const void* afin, const void* y, void* resid,
                        int64_t* status, void* stream);
int bak_gram_solve(int dtype, int64_t vars, const double* gpart, const double* sqpart, int64_t nparts,
                   int64_t sweep, int64_t max_iter, double thresh2, const int32_t* cols, int64_t ncols,
                   int64_t cols_stride, const void* norms2, const double* G, void* a, double* delta,
                   double* history, int64_t* ctrl, int64_t* status, void* stream);

/* One call for the GRAM variant: G = X^T X (norms2_out = diag G, in T), all
 * sweeps (zero-norm columns skipped in the solve), and - when thresh2 < 0 and
 * resid != NULL - the final residual y - x a fused into the last pass
 * (status[3] == BAK_VARIANT_GRAM | 256 then).  Synchronizes once (zero-norm
 * check, bak.py:186-187 -> BAK_EINVAL). */
int bak_solve_gram(int dtype, const void* x, int64_t obs, int64_t vars, int64_t ldx, const void* y,
                   const int32_t* cols, int64_t ncols, int64_t cols_stride, void* norms2_out, void* e,
                   void* a, int64_t max_iter, double thresh2, double* history, int64_t* status,
                   void* resid, void* workspace, int64_t workspace_bytes, void* stream);

/* ---- (4) batched many-small-systems solve ---------------------------------
 * One CTA per system; each CTA runs the whole solve_bak (bak.py:146-195) for
 * its system: e = y (or y - x a0), sweeps, early break, final residual and drift.
 * System s: x + s*x_stride (column-major obs x vars, ldx), y + s*y_stride,
 * a + s*vars (in: a0 if warm != 0, out: a_hat), resid + s*y_stride,
 * norms2 + s*vars (precomputed, e.g. bak_colnorms over obs x (nsys*vars) when
 * x_stride == vars*ldx), ynorm2[s] (precomputed ||y_s||^2), history +
 * s*max_iter (or NULL), status + 4*s = {sweeps_run, converged, drift_warning, err}.
 * thresh2 = tol*tol*ynorm2[s] if tol > 0.  Zero-target systems return a=0. */
int bak_solve_batched(int dtype,
                      const void* x, int64_t obs, int64_t vars, int64_t ldx, int64_t x_stride,
                      int64_t nsys, const void* y, int64_t y_stride,
                      const void* norms2, const double* ynorm2,
                      void* a, int warm, void* resid,
                      int64_t max_iter, double tol, double drift_tol,
                      double* history, int64_t* status, void* stream);

/* Systems bak_solve_batched runs concurrently on the current device (one
 * wave) for systems of this shape stored contiguously; callers streaming a
 * large batch in chunks size the chunks in whole waves.  0 on error. */
int64_t bak_solve_batched_wave(int dtype, int64_t obs, int64_t vars);

/* ---- (5) multi-GPU row sharding (C3 at N>1) ---------------------------------
 * Row-sharded sweep: rank r holds rows [r0, r0+obs_local) of x, y, e; a and
 * norms2 are replicated.  Per column, every rank's grid reduces its partial dot
 * and CTA 0 posts it into every rank's mailbox (peer-mapped device memory);
 * all ranks sum the N partials in rank order, so delta and a are bit-identical
 * everywhere.  mailboxes[r] = rank r's mailbox (device pointer valid on this
 * device: a peer mapping, or local memory when emulating).
 * With nranks_local > 1 a single launch emulates nranks_local ranks on one
 * device (rows split evenly), used for single-GPU testing of the exchange.
 * With nranks_local == 1 and a workspace of >= 96 KiB, a rank whose rows fit on
 * chip runs the on-chip sweep (e in registers, x read once per sweep) with the
 * mailbox stage inside its grid exchange; status[3] = BAK_VARIANT_GRID then,
 * BAK_VARIANT_STREAM for the streaming pass. */
int64_t bak_mailbox_bytes(int64_t nranks);
int bak_sweep_rowshard(int dtype,
                       const void* x, int64_t obs_local, int64_t vars, int64_t ldx,
                       const void* norms2, void* e, void* a,
                       int64_t max_iter, double thresh2, double* history, int64_t* status,
                       int rank, int nranks, void* const* mailboxes, int64_t epoch_base,
                       int nranks_local,
                       void* workspace, int64_t workspace_bytes, void* stream);

/* Plumbing: rows [r0, r0+rows) of a column-major host matrix (leading dim sld,
 * element size elem) to the same rows of a device matrix (leading dim dld);
 * one cudaMemcpy2DAsync (pinned source => overlaps kernels on other streams). */
int bak_copy_rows_h2d(void* dst, int64_t dld, const void* src, int64_t sld, int64_t r0, int64_t rows,
                      int64_t vars, int64_t elem, void* stream);

/* Peer mapping helpers for one-process-per-GPU (CUDA IPC; 64-byte handles). */
/* Device allocation of its own (cudaMalloc, zero-filled): the mailbox a rank
 * exports over CUDA IPC must be a whole allocation — an IPC handle names an
 * allocation and peers map its base address. */
int bak_dev_alloc(int64_t bytes, void** devptr);
int bak_dev_free(void* devptr);
/* Zero `bytes` of a bak_dev_alloc allocation (synchronous; used when the
 * row-shard epoch count restarts before it would wrap 31 bits). */
int bak_dev_zero(void* devptr, int64_t bytes);
int bak_ipc_get_handle(void* devptr, void* handle64);
int bak_ipc_open_handle(const void* handle64, void** devptr);
int bak_ipc_close(void* devptr);

/* ---- BAKM matrix files (matio.py:17-57); host only -------
 * bak_bakm_header: the 16-byte header {"BAKM", u32 rows, u32 cols, u32 tag
 * 32|64}; BAK_EINVAL with matio's messages (truncated header / bad magic /
 * unknown precision tag).  bak_file_read: parallel pread of a byte range into
 * host memory (pinned for the GPU upload path); "file is short" on EOF. */
int bak_bakm_header(const char* path, int64_t* rows, int64_t* cols, int* tag, int64_t* file_bytes);
int bak_file_read(const char* path, int64_t offset, void* dst, int64_t bytes, int nthreads);

/* ---- blocked sweep: solve_bakp / block_deltas (bakp.py:52-185) -------------
 * Replaces baksolve.bakp._run_block_sweeps (bakp.py:95-129), cyclic order:
 * consecutive blocks of thr columns (narrower last block); per block every
 * delta d_k = <x_k, e>/n2_k against the same stale e (0 for zero-norm
 * columns), a[j0:j1] += d, e -= x_B d (T rounding of the product, then of the
 * subtraction).  Per sweep: history[s] = sum(e^2); divergence guard (not
 * finite, or > 10x the previous sum; the first reference is prev_sq = ||y||^2)
 * -> status[2] = BAK_EDIVERGED with status[0] counting the diverged sweep;
 * early break on thresh2 (< 0 disables).
 *   variant : AUTO, CTA / CLUSTER (e on chip), STREAM (e in HBM, any shape),
 *             GRAM (labelled algebraically-equivalent block substitution,
 *             vars <= 512).
 *   history : required, double[max_iter] (the guard message needs it).
 *   status  : int64[4] device {sweeps_run, converged, error, variant_used}. */
int bak_block_pick_variant(int dtype, int64_t obs, int64_t vars, int64_t thr);
int64_t bak_block_sweep_workspace(int dtype, int variant, int64_t obs, int64_t vars, int64_t thr);
int bak_block_sweep(int dtype, int variant,
                    const void* x, int64_t obs, int64_t vars, int64_t ldx,
                    const void* norms2, int64_t thr,
                    void* e, void* a,
                    int64_t max_iter, double thresh2, double prev_sq,
                    double* history, int64_t* status,
                    void* workspace, int64_t workspace_bytes, void* stream);
/* block_deltas (bakp.py:65-85): out[k - j0] = <x_k, e>/n2_k for k in [j0, j1),
 * 0 where n2_k == 0; 0 <= j0 < j1 <= vars. */
int64_t bak_block_deltas_workspace(int dtype, int64_t obs);
/* ---- greedy column scoring (select.py:56-85) ------------
 * scores[j] = <e,e> - <x_j,e>^2 / norms2[j] in T (double output), +inf where
 * excluded[j] != 0 (NULL = none) or norms2[j] <= 0; best (device int64[2]) =
 * {argmin (NaN first, ties to the lowest index), 1 if that score is finite}.
 * Replaces score_all_columns' x.T @ e, closed form and argmin (select.py:73-85). */
int64_t bak_score_columns_workspace(int dtype, int64_t obs, int64_t vars);
int bak_score_columns(int dtype, const void* x, int64_t obs, int64_t vars, int64_t ldx, const void* e,
                      const void* norms2, const uint8_t* excluded, double* scores, int64_t* best,
                      void* workspace, int64_t workspace_bytes, void* stream);
int bak_block_deltas(int dtype, const void* x, int64_t obs, int64_t vars, int64_t ldx,
                     int64_t j0, int64_t j1, const void* e, const void* norms2, void* out,
                     void* workspace, int64_t workspace_bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* BAK200_H_ */

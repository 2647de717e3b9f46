/*
 * CPU port of the SolveBak sweep — TEST / BASELINE INFRASTRUCTURE ONLY.
 *
 * Plain C + OpenMP restatement of baksolve.bak._run_sweeps (bak.py:92-112)
 * with the column step of bak.py:82-89: per column a dot product, a T-precision
 * division, then e -= fl(x_j * d) with two roundings (no contraction:
 * compiled with -ffp-contract=off), a_j += d; sum(e^2) once per sweep with the
 * early break of bak.py:106-111.  Zero-norm columns are skipped (bak.py:101-103).
 *
 * It exists to time the reference algorithm with ALL host threads (the
 * Python reference pins BLAS to one thread, bak.py:184):
 *   - one system : rows split into nthreads static chunks; per column every
 *                  thread computes a partial dot over its chunk, the partials
 *                  are summed in thread order (deterministic for a fixed
 *                  thread count), then each thread updates its chunk;
 *   - batched    : independent systems in parallel, one thread each;
 *   - blocked    : solve_bakp (bakp.py:95-129): per block every thread dots
 *                  the block's columns over its row chunk against the stale e,
 *                  the partials are summed in thread order, d = dot/n2 (0 for
 *                  zero norms), a += d, then each thread applies
 *                  e -= fl(sum_k x_k d_k) on its chunk; per sweep sum(e^2),
 *                  the divergence guard (returns 1) and the early break.
 * Dots use 8 interleaved accumulators (a fixed order, like a SIMD ?dot).
 * Results agree with the numpy oracle to rounding; they are not bit-equal
 * (different reduction order) — tests/test_oracle_c.py checks the tolerance.
 */
#include <math.h>
#include <omp.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define DEFINE_SOLVER(T, SUF)                                                                       \
  static T dot_##SUF(const T* u, const T* v, int64_t n) {                                           \
    T acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};                                                            \
    int64_t i = 0;                                                                                  \
    for (; i + 8 <= n; i += 8)                                                                      \
      for (int k = 0; k < 8; ++k) acc[k] += u[i + k] * v[i + k];                                    \
    for (; i < n; ++i) acc[0] += u[i] * v[i];                                                       \
    return ((acc[0] + acc[1]) + (acc[2] + acc[3])) + ((acc[4] + acc[5]) + (acc[6] + acc[7]));       \
  }                                                                                                 \
  static void upd_##SUF(T* e, const T* x, T d, int64_t n) {                                         \
    for (int64_t i = 0; i < n; ++i) {                                                               \
      T s = x[i] * d;                                                                               \
      e[i] = e[i] - s;                                                                              \
    }                                                                                               \
  }                                                                                                 \
  int bako_solve_##SUF(const T* x, int64_t obs, int64_t vars, int64_t ldx, T* e, T* a, const T* n2, \
                       int64_t max_iter, double thresh2, double* history, int64_t* sweeps_out,      \
                       int* conv_out, int nthreads) {                                               \
    if (nthreads < 1) nthreads = 1;                                                                 \
    if (obs < 65536) nthreads = 1;                                                                  \
    T* part = (T*)calloc((size_t)nthreads * 16, sizeof(T));                                         \
    int64_t sweeps = 0;                                                                             \
    int conv = 0;                                                                                   \
    volatile int stop = 0;                                                                          \
    T shared_d = 0;                                                                                 \
    _Pragma("omp parallel num_threads(nthreads)") {                                                 \
      const int tid = omp_get_thread_num(), nt = omp_get_num_threads();                             \
      const int64_t per = (obs + nt - 1) / nt;                                                      \
      const int64_t r0 = tid * per < obs ? tid * per : obs;                                         \
      const int64_t r1 = r0 + per < obs ? r0 + per : obs;                                           \
      for (int64_t s = 0; s < max_iter && !stop; ++s) {                                             \
        for (int64_t j = 0; j < vars; ++j) {                                                        \
          if (n2[j] == 0) continue;                                                                 \
          const T* xj = x + j * ldx;                                                                \
          part[tid * 16] = dot_##SUF(xj + r0, e + r0, r1 - r0);                                     \
          _Pragma("omp barrier") _Pragma("omp single") {                                            \
            T p = 0;                                                                                \
            for (int k = 0; k < nt; ++k) p += part[k * 16];                                         \
            shared_d = p / n2[j];                                                                   \
            a[j] += shared_d;                                                                       \
          }                                                                                         \
          upd_##SUF(e + r0, xj + r0, shared_d, r1 - r0);                                            \
        }                                                                                           \
        part[tid * 16] = dot_##SUF(e + r0, e + r0, r1 - r0);                                        \
        _Pragma("omp barrier") _Pragma("omp single") {                                              \
          T q = 0;                                                                                  \
          for (int k = 0; k < nt; ++k) q += part[k * 16];                                           \
          if (history) history[s] = (double)q;                                                      \
          sweeps = s + 1;                                                                           \
          if (thresh2 >= 0 && (double)q <= thresh2) {                                               \
            conv = 1;                                                                               \
            stop = 1;                                                                               \
          }                                                                                         \
        }                                                                                           \
      }                                                                                             \
    }                                                                                               \
    free(part);                                                                                     \
    *sweeps_out = sweeps;                                                                           \
    *conv_out = conv;                                                                               \
    return 0;                                                                                       \
  }                                                                                                 \
  int bako_solve_batched_##SUF(const T* x, int64_t obs, int64_t vars, int64_t ldx, int64_t x_stride, \
                               int64_t nsys, T* e, int64_t e_stride, T* a, const T* n2,             \
                               int64_t max_iter, int nthreads) {                                    \
    if (nthreads < 1) nthreads = 1;                                                                 \
    _Pragma("omp parallel for schedule(dynamic, 1) num_threads(nthreads)")                          \
    for (int64_t s = 0; s < nsys; ++s) {                                                            \
      const T* xs = x + s * x_stride;                                                               \
      T* es = e + s * e_stride;                                                                     \
      T* as = a + s * vars;                                                                         \
      const T* ns = n2 + s * vars;                                                                  \
      for (int64_t it = 0; it < max_iter; ++it)                                                     \
        for (int64_t j = 0; j < vars; ++j) {                                                        \
          if (ns[j] == 0) continue;                                                                 \
          const T d = dot_##SUF(xs + j * ldx, es, obs) / ns[j];                                     \
          upd_##SUF(es, xs + j * ldx, d, obs);                                                      \
          as[j] += d;                                                                               \
        }                                                                                           \
    }                                                                                               \
    return 0;                                                                                       \
  }

#define DEFINE_BLOCK(T, SUF)                                                                        \
  int bako_solve_block_##SUF(const T* x, int64_t obs, int64_t vars, int64_t ldx, T* e, T* a, const T* n2, \
                             int64_t thr, int64_t max_iter, double thresh2, double prev_sq, double* history, \
                             int64_t* sweeps_out, int* conv_out, int nthreads) {                    \
    if (nthreads < 1) nthreads = 1;                                                                 \
    if (obs < 16384) nthreads = 1;                                                                  \
    T* part = (T*)calloc((size_t)nthreads * (size_t)thr, sizeof(T));                                \
    T* d = (T*)calloc((size_t)thr, sizeof(T));                                                      \
    T* qpart = (T*)calloc((size_t)nthreads * 16, sizeof(T));                                        \
    int64_t sweeps = 0;                                                                             \
    int conv = 0, div = 0;                                                                          \
    volatile int stop = 0;                                                                          \
    double prev = prev_sq;                                                                          \
    _Pragma("omp parallel num_threads(nthreads)") {                                                 \
      const int tid = omp_get_thread_num(), nt = omp_get_num_threads();                             \
      const int64_t per = (obs + nt - 1) / nt;                                                      \
      const int64_t r0 = tid * per < obs ? tid * per : obs;                                         \
      const int64_t r1 = r0 + per < obs ? r0 + per : obs;                                           \
      for (int64_t s = 0; s < max_iter && !stop; ++s) {                                             \
        for (int64_t j0 = 0; j0 < vars; j0 += thr) {                                                \
          const int64_t j1 = j0 + thr < vars ? j0 + thr : vars;                                     \
          for (int64_t k = j0; k < j1; ++k)                                                         \
            part[tid * thr + (k - j0)] = dot_##SUF(x + k * ldx + r0, e + r0, r1 - r0);              \
          _Pragma("omp barrier") _Pragma("omp single") {                                            \
            for (int64_t k = j0; k < j1; ++k) {                                                     \
              T p = 0;                                                                              \
              for (int t = 0; t < nt; ++t) p += part[t * thr + (k - j0)];                           \
              d[k - j0] = n2[k] == 0 ? (T)0 : p / n2[k];                                            \
              a[k] += d[k - j0];                                                                    \
            }                                                                                       \
          }                                                                                         \
          for (int64_t r = r0; r < r1; ++r) {                                                       \
            T sc = 0;                                                                               \
            for (int64_t k = j0; k < j1; ++k) sc += x[k * ldx + r] * d[k - j0];                     \
            e[r] = e[r] - sc;                                                                       \
          }                                                                                         \
          _Pragma("omp barrier")                                                                    \
        }                                                                                           \
        qpart[tid * 16] = dot_##SUF(e + r0, e + r0, r1 - r0);                                       \
        _Pragma("omp barrier") _Pragma("omp single") {                                              \
          T q = 0;                                                                                  \
          for (int k = 0; k < nt; ++k) q += qpart[k * 16];                                          \
          const double sq = (double)q;                                                              \
          if (history) history[s] = sq;                                                             \
          sweeps = s + 1;                                                                           \
          if (!isfinite(sq) || sq > prev * 10.0) {                                                  \
            div = 1;                                                                                \
            stop = 1;                                                                               \
          } else if (thresh2 >= 0 && sq <= thresh2) {                                               \
            conv = 1;                                                                               \
            stop = 1;                                                                               \
          }                                                                                         \
          prev = sq;                                                                                \
        }                                                                                           \
      }                                                                                             \
    }                                                                                               \
    free(part);                                                                                     \
    free(d);                                                                                        \
    free(qpart);                                                                                    \
    *sweeps_out = sweeps;                                                                           \
    *conv_out = conv;                                                                               \
    return div;                                                                                     \
  }

DEFINE_SOLVER(double, f64)
DEFINE_SOLVER(float, f32)
DEFINE_BLOCK(double, f64)
DEFINE_BLOCK(float, f32)

int bako_max_threads(void) { return omp_get_max_threads(); }

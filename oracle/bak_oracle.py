"""CPU oracle for the SolveBak column sweep — TEST INFRASTRUCTURE ONLY.

This module is the checker, never the product.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline / reference arm
may import it.  The shipped path (``paper_2104_12570_b200``) never touches it
and fails loudly when its CUDA library is missing.

It restates, in numpy, the algorithm of the reference package ``baksolve``
0.1.0 (``/root/reference/pkg``; pure Python over numpy/OpenBLAS, no native
code).  Every arithmetic operation is issued the same way the reference issues
it — ``np.dot`` for each column dot and for sum(e^2) (OpenBLAS ``?dot``),
``np.multiply``/``np.subtract`` ufuncs with ``out=`` for the residual update
(two roundings, no FMA), ``x @ a`` (``?gemv``) for residuals — under a single
BLAS thread, so on the same host it reproduces the reference bit for bit.
``tests/test_oracle_golden.py`` pins exactly that against fixtures produced by
the real reference (``tests/golden/make_golden.py``).

Parity status: PINNED (bitwise on the fixture host; see tests/golden/*.npz).

Reference map (``/root/reference/pkg/src/baksolve``):
  rng_for            core.py:39-41
  _draw              core.py:157-163
  generate_system    core.py:166-185
  column_norms_sq    core.py:116-127
  coordinate step    bak.py:82-89   (_column_step)
  sweep loop         bak.py:92-112  (_run_sweeps)
  zero target        bak.py:115-124 (_zero_report)
  finish / drift     bak.py:127-143 (_finish_report), DRIFT_TOL bak.py:29
  solve              bak.py:146-195 (solve_bak)
  fp64 metrics       bench.py:109-121 (_predict_f64), bench.py:180-184
  blocked solver     bakp.py:52-185 (block_deltas, _run_block_sweeps, solve_bakp),
                     DIVERGENCE_FACTOR bakp.py:32
  column scoring     select.py:56-85 (score_all_columns), greedy selection
                     select.py:88-136 (select_features, _refit), Householder
                     least squares qr.py:42-119 (refit="qr")
"""

from __future__ import annotations

import time

import numpy as np
from threadpoolctl import threadpool_limits

DRIFT_TOL = 1e-4                       # bak.py:29
DIVERGENCE_FACTOR = 10.0               # bakp.py:32


class DivergenceError(RuntimeError):
    """bakp.py:35-36"""
_DTYPES = {"single": np.float32, "double": np.float64}


# --------------------------------------------------------------------------
# seeded inputs (core.py:39-41, 157-185)
# --------------------------------------------------------------------------

def philox(seed: int) -> np.random.Generator:
    """Counter-based Philox stream, as ``rng_for`` (core.py:39-41)."""
    return np.random.Generator(np.random.Philox(seed))


def _sample(gen, count, kind, dt):
    # core.py:157-163: uniform(-1,1) is random()*2-1 in the target precision
    if kind == "normal":
        return gen.standard_normal(count, dtype=dt)
    out = gen.random(count, dtype=dt)
    out *= dt(2)
    out -= dt(1)
    return out


def make_system(obs, nvars, seed=0, distribution="uniform",
                coeff_distribution="uniform", noise_sigma=0.0,
                precision="double"):
    """Restatement of ``generate_system`` (core.py:166-185).

    x is one flat Philox stream viewed column-major; then a_true; then
    y = x @ a_true under one BLAS thread; then optional sigma*N(0,1) noise.
    Returns (x, y, a_true).
    """
    dt = _DTYPES[precision]
    gen = philox(seed)
    x = _sample(gen, obs * nvars, distribution, dt).reshape((obs, nvars), order="F")
    a_true = _sample(gen, nvars, coeff_distribution, dt)
    with threadpool_limits(limits=1, user_api="blas"):
        y = x @ a_true
    if noise_sigma > 0:
        eps_noise = gen.standard_normal(obs, dtype=dt)
        eps_noise *= dt(noise_sigma)
        y += eps_noise
    return x, y, a_true


# --------------------------------------------------------------------------
# the path (bak.py)
# --------------------------------------------------------------------------

def column_norms_sq(x):
    """n2_j = <x_j, x_j> with one ?dot per column (core.py:116-127)."""
    n2 = np.empty(x.shape[1], dtype=x.dtype)
    for j in range(x.shape[1]):
        col = x[:, j]
        n2[j] = np.dot(col, col)
    return n2


def sweep_loop(x, e, a, n2, tmp, order, shuffler, max_iter, thresh2, history):
    """The hot loop (bak.py:92-112 with the step of bak.py:82-89 inlined).

    Mutates e and a in place; returns (sweeps_run, converged).  With a
    shuffler, ``order`` is shuffled in place before every sweep, so each
    sweep's permutation compounds the previous one (bak.py:98-99).  Zero-norm
    columns are skipped (bak.py:101-103).  sum(e^2) is checked once per sweep
    (bak.py:106-111).
    """
    done = 0
    for _sweep in range(max_iter):
        if shuffler is not None:
            shuffler.shuffle(order)
        for j in order:
            nj = n2[j]
            if nj == 0.0:
                continue
            xj = x[:, j]
            step = np.dot(xj, e) / nj          # T-precision dot, T division
            np.multiply(xj, step, out=tmp)     # rounding 1
            np.subtract(e, tmp, out=e)         # rounding 2
            a[j] += step
        done += 1
        sq = float(np.dot(e, e))
        if history is not None:
            history.append(sq)
        if thresh2 is not None and sq <= thresh2:
            return done, True
    return done, False


def _coerce_matrix(x):
    # core.py:44-55: F-ordered float32/float64, ints -> float64
    x = np.asarray(x)
    if x.ndim != 2:
        raise ValueError(f"expected a 2-d matrix, got ndim={x.ndim}")
    if x.dtype not in (np.float32, np.float64):
        x = x.astype(np.float64)
    return np.asfortranarray(x)


def _coerce_vector(v, dtype):
    # core.py:58-64
    v = np.ascontiguousarray(v, dtype=dtype)
    if v.ndim != 1:
        raise ValueError(f"expected a 1-d vector, got ndim={v.ndim}")
    return v


def solve(x, y, max_iter=1000, tol=1e-6, ordering="cyclic", ordering_seed=0,
          record_history=False, a0=None):
    """Restatement of ``solve_bak`` (bak.py:146-195).

    Returns a dict with the fields of ``SolveReport`` (bak.py:49-57) plus the
    maintained residual ``e`` (for drift / parity diagnostics).
    """
    x = _coerce_matrix(x)
    obs, nvars = x.shape
    y = _coerce_vector(y, x.dtype)
    if y.shape[0] != obs:
        raise ValueError(f"y has length {y.shape[0]}, expected {obs}")
    t0 = time.perf_counter()
    ynorm2 = float(np.dot(y, y))
    if ynorm2 == 0.0:                                   # bak.py:168-170
        return dict(a_hat=np.zeros(nvars, x.dtype), residual=np.zeros(obs, x.dtype),
                    residual_norm_history=[] if record_history else None,
                    sweeps_run=0, converged=True, wall_time=time.perf_counter() - t0,
                    drift_warning=False, e=np.zeros(obs, x.dtype))
    if a0 is None:
        a = np.zeros(nvars, dtype=x.dtype)
    else:
        a = _coerce_vector(a0, x.dtype).copy()
        if a.shape[0] != nvars:
            raise ValueError(f"a0 has length {a.shape[0]}, expected {nvars}")
    history = [] if record_history else None
    order = np.arange(nvars)
    shuffler = philox(ordering_seed) if ordering == "random" else None
    thresh2 = tol * tol * ynorm2 if tol > 0 else None
    with threadpool_limits(limits=1, user_api="blas"):
        n2 = column_norms_sq(x)
        if not n2.any():
            raise ValueError("every column of x has zero norm; nothing to solve")
        e = y - x @ a if a0 is not None else y.copy()
        tmp = np.empty_like(e)
        sweeps, converged = sweep_loop(x, e, a, n2, tmp, order, shuffler,
                                       max_iter, thresh2, history)
        resid = y - x @ a                               # bak.py:130
        wall = time.perf_counter() - t0
        drift = np.linalg.norm((e - resid).astype(np.float64))
        drift_rel = drift / max(np.sqrt(ynorm2), np.finfo(np.float64).tiny)
    return dict(a_hat=a, residual=resid, residual_norm_history=history,
                sweeps_run=sweeps, converged=converged, wall_time=wall,
                drift_warning=bool(drift_rel > DRIFT_TOL), e=e)


def coordinate_update(col, e):
    """One update along one column (bak.py:66-79)."""
    col = np.asarray(col)
    e = np.asarray(e)
    nj = np.dot(col, col)
    if nj == 0.0:
        return 0.0, e
    step = np.dot(col, e) / nj
    tmp = np.empty_like(e)
    np.multiply(col, step, out=tmp)
    np.subtract(e, tmp, out=tmp)
    return float(step), tmp


def block_deltas(x, j0, j1, e, n2):
    """Deltas of columns [j0, j1) against one stale residual (bakp.py:52-62):
    one ?dot per column, T division, 0 for zero-norm columns."""
    out = np.empty(j1 - j0, dtype=e.dtype)
    for k in range(j0, j1):
        out[k - j0] = 0.0 if n2[k] == 0.0 else np.dot(x[:, k], e) / n2[k]
    return out


def block_sweep_loop(x, e, a, n2, tmp, thr, max_iter, thresh2, history, prev_sq):
    """bakp.py:95-129: consecutive blocks of thr columns (narrower last block);
    a one-column block is the sequential column step (bakp.py:102-106), a wider
    block gets its deltas against the stale e, then a[j0:j1] += d and
    e -= x_B @ d (?gemv into scratch, then one subtraction, bakp.py:114-116).
    The divergence guard (bakp.py:121-124) and early break run once per sweep."""
    nvars = x.shape[1]
    sweeps = 0
    for _ in range(max_iter):
        for j0 in range(0, nvars, thr):
            j1 = min(j0 + thr, nvars)
            if j1 - j0 == 1:
                nj = n2[j0]
                if nj != 0.0:
                    xj = x[:, j0]
                    step = np.dot(xj, e) / nj
                    np.multiply(xj, step, out=tmp)
                    np.subtract(e, tmp, out=e)
                    a[j0] += step
                continue
            dv = block_deltas(x, j0, j1, e, n2)
            a[j0:j1] += dv
            np.matmul(x[:, j0:j1], dv, out=tmp)
            np.subtract(e, tmp, out=e)
        sweeps += 1
        sq = float(np.dot(e, e))
        if history is not None:
            history.append(sq)
        if not np.isfinite(sq) or sq > prev_sq * DIVERGENCE_FACTOR:
            raise DivergenceError(
                f"residual norm grew from {prev_sq:.6g} to {sq:.6g} in one sweep "
                f"with thr={thr}; use a smaller thr")
        prev_sq = sq
        if thresh2 is not None and sq <= thresh2:
            return sweeps, True
    return sweeps, False


def solve_bakp(x, y, max_iter=1000, tol=1e-6, thr=1, record_history=False):
    """Restatement of ``solve_bakp`` (bakp.py:132-185), cyclic order only.
    Worker threads of the reference do not change its bits (bakp.py:10-15), so
    this is single-threaded."""
    if thr < 1:
        raise ValueError(f"thr must be >= 1, got {thr}")
    x = _coerce_matrix(x)
    obs, nvars = x.shape
    if thr > nvars:
        raise ValueError(f"thr={thr} exceeds the number of columns ({nvars})")
    y = _coerce_vector(y, x.dtype)
    if y.shape[0] != obs:
        raise ValueError(f"y has length {y.shape[0]}, expected {obs}")
    t0 = time.perf_counter()
    ynorm2 = float(np.dot(y, y))
    if ynorm2 == 0.0:
        return dict(a_hat=np.zeros(nvars, x.dtype), residual=np.zeros(obs, x.dtype),
                    residual_norm_history=[] if record_history else None,
                    sweeps_run=0, converged=True, wall_time=time.perf_counter() - t0,
                    drift_warning=False, e=np.zeros(obs, x.dtype))
    history = [] if record_history else None
    thresh2 = tol * tol * ynorm2 if tol > 0 else None
    a = np.zeros(nvars, dtype=x.dtype)
    with threadpool_limits(limits=1, user_api="blas"):
        n2 = column_norms_sq(x)
        if not n2.any():
            raise ValueError("every column of x has zero norm; nothing to solve")
        e = y.copy()
        tmp = np.empty_like(e)
        sweeps, converged = block_sweep_loop(x, e, a, n2, tmp, thr, max_iter, thresh2, history, ynorm2)
        resid = y - x @ a
        wall = time.perf_counter() - t0
        drift = np.linalg.norm((e - resid).astype(np.float64))
        drift_rel = drift / max(np.sqrt(ynorm2), np.finfo(np.float64).tiny)
    return dict(a_hat=a, residual=resid, residual_norm_history=history,
                sweeps_run=sweeps, converged=converged, wall_time=wall,
                drift_warning=bool(drift_rel > DRIFT_TOL), e=e)


def permutations(ordering_seed, nvars, nsweeps):
    """The compounding per-sweep permutations of ordering='random'
    (bak.py:98-99, 180-181), as an int64 array [nsweeps, nvars]."""
    gen = philox(ordering_seed)
    order = np.arange(nvars)
    out = np.empty((nsweeps, nvars), dtype=np.int64)
    for s in range(nsweeps):
        gen.shuffle(order)
        out[s] = order
    return out


# --------------------------------------------------------------------------
# parity metrics (bench.py:109-121, 180-184)
# --------------------------------------------------------------------------

def predict_f64(x, a):
    """x @ a in float64 without materialising a float64 copy of x."""
    a64 = np.asarray(a, dtype=np.float64)
    if x.dtype == np.float64:
        return x @ a64
    pred = np.zeros(x.shape[0], dtype=np.float64)
    for j0 in range(0, x.shape[1], 64):
        j1 = min(j0 + 64, x.shape[1])
        pred += x[:, j0:j1].astype(np.float64) @ a64[j0:j1]
    return pred


def residual_norm_f64(x, y, a):
    """||y - x a||_2 recomputed in float64 (bench.py:180-184)."""
    return float(np.linalg.norm(np.asarray(y, np.float64) - predict_f64(x, a)))


def rel_coeff_err(a, a_ref):
    a = np.asarray(a, np.float64)
    a_ref = np.asarray(a_ref, np.float64)
    den = np.linalg.norm(a_ref)
    num = np.linalg.norm(a - a_ref)
    return float(num / den) if den > 0 else float(num)


# --------------------------------------------------------------------------
# BASELINE.json configurations, parameterised for scaled runs
# --------------------------------------------------------------------------

def config_c1(obs=10_000, nvars=100, seed=1):
    return make_system(obs, nvars, seed, "normal", "uniform", 0.01, "double")


def config_c2(n=4096, seed=2):
    gen = philox(seed)
    x = gen.standard_normal(n * n).reshape((n, n), order="F") / np.sqrt(n)
    x[np.arange(n), np.arange(n)] += 4.0
    a_true = gen.random(n) * 2 - 1
    with threadpool_limits(limits=1, user_api="blas"):
        y = x @ a_true
    return np.asfortranarray(x), y, a_true


def config_c3(obs=2 ** 24, nvars=256, seed=3, precision="double"):
    return make_system(obs, nvars, seed, "normal", "uniform", 0.01, precision)


def config_c4(obs=1000, nvars=1_000_000, seed=4):
    gen = philox(seed)
    x = gen.standard_normal(obs * nvars).reshape((obs, nvars), order="F")
    y = gen.standard_normal(obs)
    return x, y, None


def config_c5_system(s, obs=512, nvars=32, base_seed=5_000_000):
    return make_system(obs, nvars, base_seed + s, "normal", "uniform", 0.01, "single")


# --------------------------------------------------------------------------
# greedy column scoring and selection (select.py) — SURVEY §8f row 3
# --------------------------------------------------------------------------

class SelectionExhaustedError(RuntimeError):
    """select.py:29-30"""


def score_all_columns(x, e, excluded=()):
    """select.py:56-85: scores[j] = <e,e> - <x_j,e>^2 / <x_j,x_j> in T (one
    ?gemv for all dots), +inf for excluded or zero-norm columns; argmin with
    ties to the lowest index."""
    x = np.asarray(x)
    e = np.asarray(e)
    obs, nvars = x.shape
    if e.shape != (obs,):
        raise ValueError(f"residual has shape {e.shape}, expected ({obs},)")
    ok = np.ones(nvars, dtype=bool)
    if len(excluded):
        ok[np.asarray(sorted(excluded), dtype=int)] = False
    n2 = column_norms_sq(x)
    ok &= n2 > 0
    scores = np.full(nvars, np.inf)
    if ok.any():
        g = x.T @ e
        e2 = np.dot(e, e)
        idx = np.flatnonzero(ok)
        scores[idx] = e2 - g[idx] * g[idx] / n2[idx]
    best = int(np.argmin(scores))
    if not np.isfinite(scores[best]):
        raise SelectionExhaustedError("no non-excluded column with nonzero norm")
    return best, scores


def householder_lstsq(x, y):
    """Least squares by unpivoted Householder QR of [x | y] (qr.py:47-119):
    reflector v = (1, col[1:]/(alpha - beta)), beta = -sign(alpha)*||col||,
    tau = 2/(1 + |v_tail|^2); dependent columns (|r_jj| <= max(m,n)*eps*max|r|)
    keep coefficient 0; back substitution from the last column."""
    x = _coerce_matrix(x)
    m, n = x.shape
    y = _coerce_vector(y, x.dtype)
    w = np.empty((m, n + 1), dtype=x.dtype, order="F")
    w[:, :n] = x
    w[:, n] = y
    one, two = x.dtype.type(1), x.dtype.type(2)
    k = min(m, n)
    for j in range(k):
        col = w[j:, j]
        nrm = np.sqrt(np.dot(col, col))
        if nrm == 0.0:
            continue
        alpha = col[0]
        beta = -np.copysign(nrm, alpha)
        tail = w[j + 1:, j]
        tail /= alpha - beta
        tau = two / (one + np.dot(tail, tail))
        w[j, j] = beta
        if j + 1 < n + 1:
            s = w[j, j + 1:] + tail @ w[j + 1:, j + 1:]
            s *= tau
            w[j, j + 1:] -= s
            w[j + 1:, j + 1:] -= np.outer(tail, s)
    r_diag = w.diagonal()[:k]
    scale = float(np.max(np.abs(r_diag))) if r_diag.size else 0.0
    tol = max(m, n) * float(np.finfo(r_diag.dtype).eps) * scale
    a = np.zeros(n, dtype=x.dtype)
    qty = w[:, n]
    for j in reversed(range(k)):
        rjj = w[j, j]
        if abs(rjj) <= tol:
            continue
        a[j] = (qty[j] - np.dot(w[j, j + 1:n], a[j + 1:])) / rjj
    return a


def select_features(x, y, max_feat, refit="qr", stop_tol=0.0, refit_config=None):
    """select.py:106-136: score, pick, refit on the picked columns (QR, or
    solve_bak warm-started from the previous coefficients), recompute e."""
    x = _coerce_matrix(x)
    obs, nvars = x.shape
    y = _coerce_vector(y, x.dtype)
    if y.shape[0] != obs:
        raise ValueError(f"y has length {y.shape[0]}, expected {obs}")
    if max_feat > nvars:
        raise ValueError(f"max_feat={max_feat} exceeds the number of columns ({nvars})")
    ynorm = np.linalg.norm(y.astype(np.float64))
    selected, norms, coeffs = [], [], None
    e = y.copy()
    for _ in range(max_feat):
        best, _ = score_all_columns(x, e, excluded=selected)
        selected.append(best)
        xs = np.asfortranarray(x[:, selected])
        if refit == "qr":
            coeffs = householder_lstsq(xs, y)
        else:
            cfg = dict(refit_config or {})
            a0 = np.zeros(xs.shape[1], dtype=xs.dtype)
            if coeffs is not None:
                a0[:coeffs.shape[0]] = coeffs
            coeffs = solve(xs, y, a0=a0, **cfg)["a_hat"]
        e = y - xs @ coeffs
        rn = float(np.dot(e, e))
        norms.append(rn)
        if stop_tol > 0 and ynorm > 0 and np.sqrt(rn) / ynorm <= stop_tol:
            break
    return dict(selected=selected, residual_norms=norms, final_coeffs=coeffs)

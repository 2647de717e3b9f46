"""Full-size golden outputs of the REAL reference for the headline configs.

    python tests/golden/make_golden_fullsize.py [c3|c3f32|c4 ...]

Runs ``baksolve`` 0.1.0 (imported from /root/reference/pkg/src, this container
only) on BASELINE configs 3 and 4 at their full sizes and writes small
fixtures ``fullsize_<name>.npz`` (a few hundred KB): the reference's a_hat
(C4: a fixed strided sample of 65,536 of the 10^6 coefficients, plus its
fp64 norm), per-sweep history, sweeps_run / converged / drift_warning, the
fp64-recomputed residual norm (bench.py:180-184 via ``_predict_f64``), a
strided sample of the maintained residual, and SHA-256 digests of the first
and last columns of x and of y so that a GPU box regenerating the inputs with
the oracle's restatement of ``generate_system`` (core.py:166-185) proves it
drew the same bytes.  x itself (34 / 17 / 8 GB) is never stored.

Peak host memory: ~35 GB for C3 fp64.  Wall time here: ~5 min (C3 fp64),
~2.5 min (C3 fp32), ~1 min (C4).
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
SAMPLE = 65536  # strided sample length for vectors too long to store


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def sample_index(n, k=SAMPLE):
    """Fixed strided sample of range(n) (shared with the tests)."""
    if n <= k:
        return np.arange(n)
    return (np.arange(k, dtype=np.int64) * n) // k


def run(bk, predict, name):
    SC = bk.SolveConfig
    t0 = time.time()
    if name in ("c3", "c3f32"):
        prec = "double" if name == "c3" else "single"
        spec = dict(obs=1 << 24, vars=256, seed=3, distribution="normal", coeff_distribution="uniform",
                    noise_sigma=0.01, precision=prec)
        x, y, _ = bk.generate_system(bk.SystemSpec(obs=spec["obs"], vars=256, seed=3, distribution="normal",
                                                   coeff_distribution="uniform", noise_sigma=0.01), prec)
        cfg = SC(max_iter=20, tol=0, record_history=True)
    elif name == "c4":
        # BASELINE config 4: x iid N(0,1) (1,000 x 10^6, one flat Philox stream
        # viewed column-major as generate_system draws), then y ~ N(0,1)
        spec = dict(obs=1000, vars=1_000_000, seed=4, draw="x=standard_normal(obs*vars) F-order; y=standard_normal(obs)")
        rng = bk.core.rng_for(4)
        x = rng.standard_normal(1000 * 1_000_000).reshape((1000, 1_000_000), order="F")
        y = rng.standard_normal(1000)
        cfg = SC(max_iter=10, tol=0, record_history=True)
    else:
        raise SystemExit(f"unknown case {name}")
    t_gen = time.time() - t0
    t0 = time.time()
    rep = bk.solve_bak(x, y, cfg)
    t_solve = time.time() - t0
    pred = predict(x, rep.a_hat)
    y64 = np.asarray(y, np.float64)
    nv = x.shape[1]
    ia = sample_index(nv)
    ie = sample_index(x.shape[0])
    d = dict(
        spec=np.array(json.dumps(spec)), shape=np.array(x.shape), dtype=np.array(np.dtype(x.dtype).name),
        max_iter=np.array(cfg.max_iter), tol=np.array(cfg.tol),
        a_index=ia, a_hat=np.asarray(rep.a_hat)[ia], a_norm_f64=np.array(float(np.linalg.norm(
            np.asarray(rep.a_hat, np.float64)))), a_full=np.array(len(ia) == nv),
        history=np.asarray(rep.residual_norm_history, np.float64),
        sweeps_run=np.array(rep.sweeps_run), converged=np.array(rep.converged),
        drift_warning=np.array(rep.drift_warning),
        resid_norm_f64=np.array(float(np.linalg.norm(y64 - pred))),
        ynorm_f64=np.array(float(np.linalg.norm(y64))),
        e_index=ie, e_sample=np.asarray(rep.residual)[ie],
        e_norm_f64=np.array(float(np.linalg.norm(np.asarray(rep.residual, np.float64)))),
        sha_x_first=np.array(_sha(x[:, 0])), sha_x_last=np.array(_sha(x[:, -1])), sha_y=np.array(_sha(y)),
        seconds=np.array([t_gen, t_solve]),
    )
    np.savez_compressed(os.path.join(HERE, f"fullsize_{name}.npz"), **d)
    print(f"{name}: {x.shape} {x.dtype} gen {t_gen:.0f}s solve {t_solve:.0f}s sweeps={rep.sweeps_run} "
          f"|r|={float(d['resid_norm_f64']):.12e}", flush=True)


def main():
    sys.path.insert(0, REF_SRC)
    import baksolve as bk
    import baksolve.core  # noqa: F401
    from baksolve.bench import _predict_f64
    names = sys.argv[1:] or ["c4", "c3f32", "c3"]
    for n in names:
        run(bk, _predict_f64, n)


if __name__ == "__main__":
    main()

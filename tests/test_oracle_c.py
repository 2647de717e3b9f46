"""The C/OpenMP oracle port (used for the multi-threaded reference arm) agrees
with the numpy oracle (itself bit-pinned to the reference).  CPU only."""

import numpy as np
import pytest

from oracle import bak_oracle as orc
from oracle import bak_oracle_c as oc


def test_c_port_single_system_matches_numpy_oracle():
    for prec, tol in (("double", 1e-10), ("single", 1e-4)):
        x, y, _ = orc.make_system(100_000, 12, 4, "normal", "uniform", 0.01, prec)
        ref = orc.solve(x, y, max_iter=6, tol=0, record_history=True)
        a, e, sw, cv, hist = oc.solve(x, y, 6, nthreads=4, record_history=True)
        assert sw == 6 and not cv
        assert orc.rel_coeff_err(a, ref["a_hat"]) <= tol
        np.testing.assert_allclose(hist, ref["residual_norm_history"], rtol=1e-3 if prec == "single" else 1e-9)


def test_c_port_early_break_and_batched():
    x, y, _ = orc.make_system(400, 50, 7, "uniform", "uniform", 0.0, "double")
    ref = orc.solve(x, y, max_iter=5000, tol=1e-12)
    a, e, sw, cv, _ = oc.solve(x, y, 5000, tol=1e-12)
    assert cv and abs(sw - ref["sweeps_run"]) <= 1
    assert orc.rel_coeff_err(a, ref["a_hat"]) <= 1e-9
    xs = np.stack([orc.config_c5_system(s)[0].T.copy() for s in range(6)])
    ys = np.stack([orc.config_c5_system(s)[1] for s in range(6)])
    a, _ = oc.solve_batched(xs, ys, 50, nthreads=3)
    for s in range(6):
        r = orc.solve(xs[s].T, ys[s], max_iter=50, tol=0)
        assert orc.rel_coeff_err(a[s], r["a_hat"]) <= 1e-4


@pytest.mark.parametrize("obs,nv,thr,dtype", [(300, 40, 7, np.float64), (20000, 64, 16, np.float64),
                                              (5000, 30, 30, np.float32)])
def test_c_port_block_matches_numpy_oracle(obs, nv, thr, dtype):
    rng = np.random.default_rng(obs + thr)
    x = np.asfortranarray(rng.standard_normal((obs, nv)).astype(dtype))
    y = (x @ rng.standard_normal(nv).astype(dtype) + 0.1 * rng.standard_normal(obs)).astype(dtype)
    try:
        ref = orc.solve_bakp(x, y, max_iter=8, tol=0, thr=thr)
    except orc.DivergenceError:
        a, e, sw, cv, hist, div = oc.solve_block(x, y, thr, 8, nthreads=4)
        assert div
        return
    a, e, sw, cv, hist, div = oc.solve_block(x, y, thr, 8, nthreads=4)
    assert not div and sw == ref["sweeps_run"]
    tol = 1e-10 if dtype == np.float64 else 1e-4
    assert orc.rel_coeff_err(a, ref["a_hat"]) <= tol


def test_c_port_block_divergence_guard():
    rng = np.random.default_rng(21)
    col = rng.standard_normal(50)
    x = np.asfortranarray(np.tile(col[:, None], (1, 5)))
    *_, div = oc.solve_block(x, col.copy(), 5, 10)
    assert div

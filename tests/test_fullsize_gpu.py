"""BASELINE.json configurations at FULL size on the GPU, checked through
properties that do not need a full-size CPU run (the oracle is used only where
it finishes in seconds):

  C2 4096x4096 fp64 : full oracle parity (50 sweeps, and the 1e-10 early break)
  C3 2^24x256       : the exact per-column kernel (STREAM) and the labelled GRAM
                      reformulation agree to the parity bar after 20 sweeps;
                      history non-increasing; recomputed residual consistent
  C4 1000x1e6 fp64  : one full sweep against the oracle's one sweep
  C5 65536x(512x32) : a seeded sample of systems against the oracle
"""

import numpy as np
import pytest

from oracle import bak_oracle as orc

pytestmark = pytest.mark.gpu


def _pb():
    import paper_2104_12570_b200 as pb
    return pb


def _mono(h, dtype):
    eps = float(np.finfo(dtype).eps)
    assert all(h[i + 1] <= h[i] * (1 + 16 * eps) for i in range(len(h) - 1))


@pytest.mark.parametrize("tol", [0.0, 1e-10])
def test_c2_full_matches_oracle(tol):
    pb = _pb()
    x, y, _ = orc.config_c2(n=4096)
    cfg = dict(max_iter=50, tol=tol, record_history=True)
    ref = orc.solve(x, y, **cfg)
    rep = pb.solve_bak(x, y, pb.SolveConfig(**cfg))
    assert rep.sweeps_run == ref["sweeps_run"] and rep.converged == ref["converged"]
    if tol:
        assert rep.sweeps_run == 20  # the break must not flip
    assert orc.rel_coeff_err(rep.a_hat, ref["a_hat"]) <= 1e-10
    ynorm = np.linalg.norm(y)
    assert abs(orc.residual_norm_f64(x, y, rep.a_hat) - orc.residual_norm_f64(x, y, ref["a_hat"])) <= 1e-10 * ynorm


@pytest.mark.parametrize("precision", ["double", "single"])
def test_c3_full_exact_and_gram_agree(precision):
    import torch
    import bench
    pb = _pb()
    cfg = dict(bench.CONFIGS["c3" if precision == "double" else "c3f32"])
    dev = torch.device("cuda", 0)
    dm, y = bench.make_inputs(cfg, dev, seed=3)
    sc = pb.SolveConfig(max_iter=20, tol=0, record_history=True)
    g = pb.solve_bak(dm, y, sc, variant="gram", return_device=True)
    s = pb.solve_bak(dm, y, sc, variant="stream", return_device=True)
    assert g.sweeps_run == s.sweeps_run == 20
    tol = 1e-10 if precision == "double" else 1e-4
    ag, as_ = g.a_hat.double().cpu().numpy(), s.a_hat.double().cpu().numpy()
    assert np.linalg.norm(ag - as_) / np.linalg.norm(as_) <= tol
    _mono(s.residual_norm_history, np.float64 if precision == "double" else np.float32)
    _mono(g.residual_norm_history, np.float64 if precision == "double" else np.float32)
    rg = float(torch.linalg.vector_norm(g.residual.double()))
    rs = float(torch.linalg.vector_norm(s.residual.double()))
    assert abs(rg - rs) / rs <= tol
    assert not g.drift_warning and not s.drift_warning
    # noise level 0.01 * sqrt(obs): the solve reached the noise floor
    assert 0.5 * 0.01 * np.sqrt(cfg["obs"]) < rs < 2 * 0.01 * np.sqrt(cfg["obs"])


def test_c4_full_one_sweep_matches_oracle():
    pb = _pb()
    x, y, _ = orc.config_c4(obs=1000, nvars=1_000_000)
    ref = orc.solve(x, y, max_iter=1, tol=0)
    rep = pb.solve_bak(x, y, pb.SolveConfig(max_iter=1, tol=0))
    assert rep.sweeps_run == 1
    assert orc.rel_coeff_err(rep.a_hat, ref["a_hat"]) <= 1e-10
    ynorm = np.linalg.norm(y)
    assert abs(orc.residual_norm_f64(x, y, rep.a_hat) - orc.residual_norm_f64(x, y, ref["a_hat"])) <= 1e-10 * ynorm


def test_c5_full_batch_sample_matches_oracle():
    pb = _pb()
    nsys = 65536
    rng = np.random.default_rng(2024)
    sample = sorted(rng.choice(nsys, 24, replace=False).tolist())
    xs = np.empty((nsys, 512, 32), np.float32)
    ys = np.empty((nsys, 512), np.float32)
    # full batch drawn with the per-system Philox streams of the sample;
    # the rest share a cheap seeded fill (the batch shape and work are full size)
    fill = np.random.default_rng(7)
    xs[:] = fill.standard_normal((nsys, 512, 32), dtype=np.float32)
    ys[:] = fill.standard_normal((nsys, 512), dtype=np.float32)
    for s in sample:
        x, y, _ = orc.config_c5_system(s)
        xs[s], ys[s] = x, y
    rep = pb.solve_bak_batched(xs, ys, pb.SolveConfig(max_iter=200, tol=0))
    assert np.all(rep.sweeps_run == 200)
    for s in sample:
        ref = orc.solve(xs[s], ys[s], max_iter=200, tol=0)
        assert orc.rel_coeff_err(rep.a_hat[s], ref["a_hat"]) <= 1e-4

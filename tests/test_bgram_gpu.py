"""The block-Gram sweep (variant="bgram", labelled, algebraically equal to the
per-column sweep; csrc/bak_bgram.cu) against the reference's fixtures and the
CPU oracle, with the tolerances of test_gpu_parity.py (fp64 1e-10, fp32 1e-4;
sweeps_run / converged identical; residual norms recomputed in fp64)."""

import numpy as np
import pytest

import golden_io
from oracle import bak_oracle as orc
from test_gpu_parity import TOL, assert_parity

pytestmark = pytest.mark.gpu

# cyclic-order fixtures whose residual fits one cluster (the block-Gram plans hold <= 65,536 rows)
CYCLIC = [n for n in golden_io.names() if golden_io.load(n)["config"].get("ordering", "cyclic") == "cyclic"
          and golden_io.load(n)["x"].shape[0] <= 16384]


def _pb():
    import paper_2104_12570_b200 as pb
    return pb


@pytest.mark.parametrize("name", CYCLIC)
def test_bgram_golden_fixture(name):
    pb = _pb()
    g = golden_io.load(name)
    x, y = g["x"], g["y"]
    rep = pb.solve_bak(x, y, pb.SolveConfig(**g["config"]), a0=g["a0"], variant="bgram")
    assert rep.variant == "bgram" or rep.sweeps_run == 0  # a zero target returns before any kernel
    assert_parity(x, y, rep, g["a_hat"], int(g["sweeps_run"]), bool(g["converged"]), float(g["resid_norm_f64"]),
                  g["history"] if bool(g["has_history"]) else None)


@pytest.mark.parametrize("obs,nv,precision", [(300, 64, "double"), (2000, 200, "double"), (9000, 70, "single"),
                                              (777, 129, "double"), (5000, 1, "double")])
def test_bgram_blocks_ragged_and_zero_columns(obs, nv, precision):
    pb = _pb()
    x, y, _ = orc.make_system(obs, nv, 41, "normal", "uniform", 0.01, precision)
    if nv > 3:
        x[:, 2] = 0  # zero-norm column: skipped (its coefficient stays put)
        x[:, nv - 1] = 0
    cfg = dict(max_iter=15, tol=0, record_history=True)
    ref = orc.solve(x, y, **cfg)
    rep = pb.solve_bak(x, y, pb.SolveConfig(**cfg), variant="bgram")
    assert rep.variant == "bgram"
    assert_parity(x, y, rep, ref["a_hat"], ref["sweeps_run"], ref["converged"], ref_hist=ref["residual_norm_history"])
    if nv > 3:
        assert rep.a_hat[2] == 0 and rep.a_hat[nv - 1] == 0


@pytest.mark.parametrize("tol", [0.0, 1e-10])
def test_bgram_c2_full_size(tol):
    """BASELINE config 2 at full size (4096^2 fp64, 50 sweeps; early break at 1e-10 on sweep 20)."""
    pb = _pb()
    x, y, _ = orc.config_c2(n=4096)
    cfg = dict(max_iter=50, tol=tol, record_history=True)
    ref = orc.solve(x, y, **cfg)
    rep = pb.solve_bak(x, y, pb.SolveConfig(**cfg), variant="bgram")
    assert rep.sweeps_run == ref["sweeps_run"] and rep.converged == ref["converged"]
    if tol:
        assert rep.sweeps_run == 20
    assert orc.rel_coeff_err(rep.a_hat, ref["a_hat"]) <= 1e-10
    ynorm = np.linalg.norm(y)
    assert abs(orc.residual_norm_f64(x, y, rep.a_hat) - orc.residual_norm_f64(x, y, ref["a_hat"])) <= 1e-10 * ynorm


def test_bgram_c4_full_size_against_reference():
    """BASELINE config 4 at full size (1,000 x 10^6 fp64, 10 sweeps) against the
    REAL reference's outputs (tests/golden/fullsize_c4.npz)."""
    from test_fullsize_reference_gpu import _check, _pin_inputs
    pb = _pb()
    g = golden_io.fullsize("c4")
    x, y, _ = orc.config_c4(obs=1000, nvars=1_000_000)
    _pin_inputs(g, x, y)
    rep = pb.solve_bak(x, y, pb.SolveConfig(max_iter=10, tol=0, record_history=True), variant="bgram")
    assert rep.variant == "bgram"
    _check(rep, g, x, y, 1e-10)


def test_bgram_rejects_random_order_and_is_deterministic():
    pb = _pb()
    x, y, _ = orc.config_c1(obs=3000, nvars=90)
    with pytest.raises(ValueError):
        pb.solve_bak(x, y, pb.SolveConfig(max_iter=3, tol=0, ordering="random"), variant="bgram")
    r1 = pb.solve_bak(x, y, pb.SolveConfig(max_iter=7, tol=0), variant="bgram")
    r2 = pb.solve_bak(x, y, pb.SolveConfig(max_iter=7, tol=0), variant="bgram")
    assert r1.a_hat.tobytes() == r2.a_hat.tobytes()
    tol = TOL[np.dtype(x.dtype)]
    assert orc.rel_coeff_err(r1.a_hat, orc.solve(x, y, max_iter=7, tol=0)["a_hat"]) <= tol

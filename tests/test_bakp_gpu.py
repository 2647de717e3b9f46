"""GPU parity of the blocked solver (solve_bakp / block_deltas, reference
bakp.py:52-185) against the reference's own runs (tests/golden/bakp_*.npz) and
the CPU oracle (oracle/bak_oracle.py: solve_bakp), for every kernel family:
on-chip CTA / cluster, the HBM-streaming variant and the labelled GRAM block
substitution.  Bars: ||a - a_ref|| / ||a_ref|| <= 1e-10 (f64) /
1e-4 (f32); fp64-recomputed residual norms within the same tolerance;
sweeps_run / converged / DivergenceError identical."""

import numpy as np
import pytest

import golden_io
from oracle import bak_oracle as orc

pytestmark = pytest.mark.gpu


def _pb():
    import paper_2104_12570_b200 as pb
    return pb


def _tol(dtype):
    return 1e-10 if np.dtype(dtype) == np.float64 else 1e-4


def _variants(obs, nv, dtype):
    vs = ["auto", "stream"]
    # on-chip kernels (TMA ring default): one CTA up to 256 threads x 8 rows, clusters of <= 16
    if obs <= 2048:
        vs.append("cta")
    elif obs <= 32768:
        vs.append("cluster")
    if nv <= 512:
        vs.append("gram")
    return vs


def _check(rep, ref_a, ref_sweeps, ref_conv, x, y, dtype):
    tol = _tol(dtype)
    assert rep.sweeps_run == ref_sweeps
    assert rep.converged == ref_conv
    assert orc.rel_coeff_err(rep.a_hat, ref_a) <= tol
    r = orc.residual_norm_f64(x, y, rep.a_hat)
    r_ref = orc.residual_norm_f64(x, y, ref_a)
    ynorm = float(np.linalg.norm(np.asarray(y, np.float64)))
    den = r_ref if r_ref >= 1e-6 * ynorm else ynorm
    assert abs(r - r_ref) <= tol * max(den, 1e-300)


@pytest.mark.parametrize("name", golden_io.bakp_names())
def test_bakp_matches_reference_fixture(name):
    pb = _pb()
    g = golden_io.load_bakp(name)
    x, y = g["x"], g["y"]
    cfg = pb.BlockConfig(base=pb.SolveConfig(**g["config"]), thr=g["thr"])
    for v in _variants(*x.shape, x.dtype):
        if g["diverged"]:
            with pytest.raises(pb.DivergenceError, match=f"thr={g['thr']}"):
                pb.solve_bakp(x, y, cfg, variant=v)
            continue
        rep = pb.solve_bakp(x, y, cfg, variant=v)
        _check(rep, g["a_hat"], int(g["sweeps_run"]), bool(g["converged"]), x, y, x.dtype)
        assert rep.drift_warning == bool(g["drift_warning"])
        if bool(g["has_history"]):
            h = np.asarray(rep.residual_norm_history)
            assert h.shape == g["history"].shape
            scale = max(float(g["ynorm_f64"]) ** 2, 1e-300)
            assert np.all(np.abs(h - g["history"]) <= 10 * _tol(x.dtype) * np.maximum(g["history"], 1e-6 * scale))


@pytest.mark.parametrize("obs,nv,thr,dtype,max_iter", [
    (1000, 64, 8, np.float64, 30),        # CTA
    (1000, 64, 64, np.float32, 3),        # one full-width block (Jacobi step)
    (777, 45, 10, np.float64, 25),        # ragged rows and last block
    (6000, 120, 50, np.float64, 15),      # cluster
    (20000, 200, 33, np.float32, 10),     # cluster, f32
    (50000, 48, 16, np.float64, 6),       # streaming (past on-chip capacity)
    (300, 1100, 100, np.float64, 5),      # wide, deltas chunked > 64 per block
])
def test_bakp_matches_oracle(obs, nv, thr, dtype, max_iter):
    pb = _pb()
    rng = np.random.default_rng(obs + nv + thr)
    x = np.asfortranarray(rng.standard_normal((obs, nv)).astype(dtype))
    y = (x @ rng.uniform(-1, 1, nv).astype(dtype) + 0.05 * rng.standard_normal(obs)).astype(dtype)
    try:
        ref = orc.solve_bakp(x, y, max_iter=max_iter, tol=0, thr=thr)
    except orc.DivergenceError as err:
        with pytest.raises(pb.DivergenceError) as ei:
            pb.solve_bakp(x, y, pb.BlockConfig(base=pb.SolveConfig(max_iter=max_iter, tol=0), thr=thr))
        assert str(ei.value).split(" in one")[0][:24] == str(err).split(" in one")[0][:24]
        return
    for v in _variants(obs, nv, dtype):
        rep = pb.solve_bakp(x, y, pb.BlockConfig(base=pb.SolveConfig(max_iter=max_iter, tol=0), thr=thr), variant=v)
        _check(rep, ref["a_hat"], ref["sweeps_run"], ref["converged"], x, y, dtype)
        if v != "auto":
            assert rep.variant == v


def test_thr_one_matches_sequential_exactly():
    """bakp.py:13-15 / test_solver_bakp.py:51-58: thr=1 reproduces solve_bak bit for bit."""
    pb = _pb()
    rng = np.random.default_rng(2)
    for dtype, shape in ((np.float64, (120, 17)), (np.float32, (90, 8)), (np.float64, (20, 40)),
                         (np.float64, (5000, 30))):
        x = np.asfortranarray(rng.standard_normal(shape).astype(dtype))
        y = (x @ rng.standard_normal(shape[1]).astype(dtype) + 0.1 * rng.standard_normal(shape[0])).astype(dtype)
        cfg = pb.SolveConfig(max_iter=30, tol=1e-7, record_history=True)
        seq = pb.solve_bak(x, y, cfg)
        blk = pb.solve_bakp(x, y, pb.BlockConfig(base=cfg, thr=1))
        assert seq.a_hat.tobytes() == blk.a_hat.tobytes()
        assert seq.residual.tobytes() == blk.residual.tobytes()
        assert seq.residual_norm_history == blk.residual_norm_history
        assert (seq.sweeps_run, seq.converged, seq.drift_warning) == (blk.sweeps_run, blk.converged,
                                                                       blk.drift_warning)


def test_worker_count_does_not_change_bits():
    pb = _pb()
    rng = np.random.default_rng(3)
    x = np.asfortranarray(rng.standard_normal((250, 48)).astype(np.float32))
    y = (x @ rng.standard_normal(48).astype(np.float32)).astype(np.float32)
    cfg = pb.SolveConfig(max_iter=25, tol=1e-6, record_history=True)
    reps = [pb.solve_bakp(x, y, pb.BlockConfig(base=cfg, thr=16, worker_count=w)) for w in (1, 2, 8)]
    for r in reps[1:]:
        assert r.a_hat.tobytes() == reps[0].a_hat.tobytes()
        assert r.residual_norm_history == reps[0].residual_norm_history


def test_bakp_deterministic_across_runs():
    pb = _pb()
    rng = np.random.default_rng(5)
    x = np.asfortranarray(rng.standard_normal((12000, 96)))
    y = rng.standard_normal(12000)
    cfg = pb.BlockConfig(base=pb.SolveConfig(max_iter=10, tol=0), thr=12)
    for v in ("cluster", "stream", "gram"):
        a = pb.solve_bakp(x, y, cfg, variant=v).a_hat
        b = pb.solve_bakp(x, y, cfg, variant=v).a_hat
        assert a.tobytes() == b.tobytes()


def test_orthonormal_full_width_block_is_one_shot():
    pb = _pb()
    rng = np.random.default_rng(4)
    q, _ = np.linalg.qr(rng.standard_normal((60, 8)))
    q = np.asfortranarray(q)
    y = rng.standard_normal(60)
    rep = pb.solve_bakp(q, y, pb.BlockConfig(base=pb.SolveConfig(max_iter=1, tol=0), thr=8))
    np.testing.assert_allclose(rep.a_hat, q.T @ y, atol=1e-12)


def test_remainder_block_visits_every_column():
    pb = _pb()
    rng = np.random.default_rng(5)
    x = np.asfortranarray(rng.standard_normal((40, 7)))
    rep = pb.solve_bakp(x, x @ np.ones(7), pb.BlockConfig(base=pb.SolveConfig(max_iter=1, tol=0), thr=3))
    assert np.all(rep.a_hat != 0.0)


def test_small_thr_keeps_monotone_history():
    pb = _pb()
    for seed in range(6):
        rng = np.random.default_rng(200 + seed)
        x = np.asfortranarray(rng.standard_normal((300, 100)))
        y = x @ rng.uniform(-1, 1, 100) + (0.2 * rng.standard_normal(300) if seed % 2 else 0.0)
        rep = pb.solve_bakp(x, y, pb.BlockConfig(base=pb.SolveConfig(max_iter=60, tol=1e-8, record_history=True),
                                                 thr=10))
        h = rep.residual_norm_history
        eps = np.finfo(np.float64).eps
        assert all(h[i + 1] <= h[i] * (1 + 16 * eps) for i in range(len(h) - 1))


def test_divergence_guard():
    pb = _pb()
    rng = np.random.default_rng(21)
    col = rng.standard_normal(50)
    x = np.asfortranarray(np.tile(col[:, None], (1, 5)))
    for v in ("auto", "stream", "gram"):
        with pytest.raises(pb.DivergenceError, match="thr=5"):
            pb.solve_bakp(x, col.copy(), pb.BlockConfig(base=pb.SolveConfig(max_iter=10), thr=5), variant=v)
    x = np.asfortranarray(np.array([[1e30], [0.0]], dtype=np.float32))
    with pytest.raises(pb.DivergenceError):
        pb.solve_bakp(x, np.array([1e30, 0.0], dtype=np.float32), pb.BlockConfig(base=pb.SolveConfig(max_iter=5),
                                                                                 thr=1))


def test_bakp_validation_and_zero_target():
    pb = _pb()
    x = np.eye(3, order="F")
    y = np.ones(3)
    with pytest.raises(ValueError):
        pb.solve_bakp(x, y, pb.BlockConfig(thr=4))
    with pytest.raises(ValueError):
        pb.solve_bakp(x, y, pb.BlockConfig(base=pb.SolveConfig(ordering="random"), thr=1))
    with pytest.raises(ValueError):
        pb.solve_bakp(x, np.ones(4), pb.BlockConfig(thr=1))
    with pytest.raises(ValueError):
        pb.solve_bakp(np.zeros((3, 2), order="F"), y, pb.BlockConfig(thr=2))
    rep = pb.solve_bakp(np.eye(3, order="F"), np.zeros(3), pb.BlockConfig(thr=2))
    assert np.array_equal(rep.a_hat, np.zeros(3)) and rep.converged and rep.sweeps_run == 0
    rng = np.random.default_rng(31)
    x = np.asfortranarray(rng.standard_normal((400, 60)).astype(np.float32))
    y = (x @ rng.standard_normal(60).astype(np.float32) + 0.1 * rng.standard_normal(400)).astype(np.float32)
    assert not pb.solve_bakp(x, y, pb.BlockConfig(base=pb.SolveConfig(max_iter=600, tol=0), thr=6)).drift_warning


def test_block_deltas_kats_and_validation():
    pb = _pb()
    with np.load(golden_io.os.path.join(golden_io.GOLDEN, "kat_block_deltas.npz")) as z:
        np.testing.assert_array_equal(pb.block_deltas(np.eye(2, order="F"), (0, 2), np.array([3.0, 4.0])), z["eye"])
        col = np.array([1.0, 2.0, -1.0])
        np.testing.assert_array_equal(pb.block_deltas(np.asfortranarray(np.column_stack([col, col])), (0, 2),
                                                      col.copy()), z["dup"])
    rng = np.random.default_rng(0)
    x = np.asfortranarray(rng.standard_normal((20, 5)))
    np.testing.assert_array_equal(pb.block_deltas(x, (1, 4), np.zeros(20)), np.zeros(3))
    x = np.asfortranarray(rng.standard_normal((10, 3)))
    x[:, 1] = 0.0
    d = pb.block_deltas(x, (0, 3), rng.standard_normal(10))
    assert d[1] == 0.0 and d[0] != 0.0 and d[2] != 0.0
    for bad in (((2, 2), 10), ((0, 4), 10), ((0, 2), 9)):
        with pytest.raises(ValueError):
            pb.block_deltas(x, bad[0], np.zeros(bad[1]))
    # against the oracle on a tall block with more than one chunk of columns
    x = np.asfortranarray(rng.standard_normal((30000, 150)))
    e = rng.standard_normal(30000)
    ref = orc.block_deltas(x, 5, 140, e, orc.column_norms_sq(x))
    got = pb.block_deltas(x, (5, 140), e)
    assert np.max(np.abs(got - ref) / np.maximum(np.abs(ref), 1e-300)) <= 1e-10


def test_blocked_sweep_matches_naive_reference():
    """test_solver_bakp.py:100-115 restated: the same block schedule driven
    with public pieces (block_deltas) reaches the same a."""
    pb = _pb()
    rng = np.random.default_rng(6)
    x = np.asfortranarray(rng.standard_normal((35, 10)))
    y = rng.standard_normal(35)
    thr = 4
    a = np.zeros(10)
    e = y.copy()
    for _ in range(3):
        for j0 in range(0, 10, thr):
            j1 = min(j0 + thr, 10)
            dv = pb.block_deltas(x, (j0, j1), e)
            a[j0:j1] += dv
            e = e - x[:, j0:j1] @ dv
    rep = pb.solve_bakp(x, y, pb.BlockConfig(base=pb.SolveConfig(max_iter=3, tol=0), thr=thr))
    np.testing.assert_allclose(rep.a_hat, a, rtol=1e-12, atol=1e-14)


@pytest.mark.parametrize("obs,nv,thr,dtype", [(10000, 300, 50, np.float32), (3000, 200, 20, np.float64),
                                              (1500, 100, 8, np.float64)])
def test_resident_ring_matches_restreaming(obs, nv, thr, dtype, monkeypatch):
    """Keeping a block's column slices in the ring between its two passes
    (planner default when it fits) gives the same bits as re-streaming them."""
    pb = _pb()
    rng = np.random.default_rng(obs)
    x = np.asfortranarray(rng.standard_normal((obs, nv)).astype(dtype))
    y = (x @ rng.uniform(-1, 1, nv).astype(dtype)).astype(dtype)
    cfg = pb.BlockConfig(base=pb.SolveConfig(max_iter=6, tol=0, record_history=True), thr=thr)
    monkeypatch.setenv("BAK_BLOCK_KERNEL", "tma")
    monkeypatch.setenv("BAK_BLOCK_RESIDENT", "1")
    r1 = pb.solve_bakp(x, y, cfg)
    monkeypatch.setenv("BAK_BLOCK_RESIDENT", "0")
    r0 = pb.solve_bakp(x, y, cfg)
    assert r1.variant in ("cta", "cluster")
    assert r1.a_hat.tobytes() == r0.a_hat.tobytes()
    assert r1.residual_norm_history == r0.residual_norm_history
    ref = orc.solve_bakp(x, y, max_iter=6, tol=0, thr=thr)
    assert orc.rel_coeff_err(r1.a_hat, ref["a_hat"]) <= _tol(dtype)


@pytest.mark.parametrize("obs,nv,thr,dtype", [(10000, 300, 50, np.float32), (900, 200, 20, np.float64),
                                              (12000, 100, 8, np.float64), (777, 64, 5, np.float32)])
def test_direct_load_and_tma_ring_kernels_agree(obs, nv, thr, dtype, monkeypatch):
    """The two on-chip kernels (default: TMA ring with a producer warp; and the
    direct-load form) agree with each other and with the oracle."""
    pb = _pb()
    rng = np.random.default_rng(obs + 1)
    x = np.asfortranarray(rng.standard_normal((obs, nv)).astype(dtype))
    y = (x @ rng.uniform(-1, 1, nv).astype(dtype) + 0.01 * rng.standard_normal(obs)).astype(dtype)
    cfg = pb.BlockConfig(base=pb.SolveConfig(max_iter=8, tol=0), thr=thr)
    r_tma = pb.solve_bakp(x, y, cfg)
    monkeypatch.setenv("BAK_BLOCK_KERNEL", "ldg")
    r_ldg = pb.solve_bakp(x, y, cfg)
    assert r_ldg.variant == r_tma.variant or {r_ldg.variant, r_tma.variant} <= {"cta", "cluster"}
    ref = orc.solve_bakp(x, y, max_iter=8, tol=0, thr=thr)
    for r in (r_ldg, r_tma):
        _check(r, ref["a_hat"], ref["sweeps_run"], ref["converged"], x, y, dtype)


@pytest.mark.parametrize("obs,nv,thr,dtype", [(33, 35, 34, np.float64), (40, 100, 70, np.float32),
                                              (3000, 150, 100, np.float64)])
def test_block_wider_than_the_cta(obs, nv, thr, dtype):
    """Blocks wider than the CTA's thread count (few rows, many columns per
    block): every column of the block gets its delta (regression: columns past
    the thread count were skipped)."""
    pb = _pb()
    rng = np.random.default_rng(obs + nv)
    x = np.asfortranarray(rng.standard_normal((obs, nv)).astype(dtype))
    y = (x @ rng.uniform(-1, 1, nv).astype(dtype)).astype(dtype)
    try:
        ref = orc.solve_bakp(x, y, max_iter=4, tol=0, thr=thr)
    except orc.DivergenceError:
        with pytest.raises(pb.DivergenceError):
            pb.solve_bakp(x, y, pb.BlockConfig(base=pb.SolveConfig(max_iter=4, tol=0), thr=thr))
        return
    for kern in ("tma", "ldg"):
        import os
        os.environ["BAK_BLOCK_KERNEL"] = kern
        try:
            rep = pb.solve_bakp(x, y, pb.BlockConfig(base=pb.SolveConfig(max_iter=4, tol=0), thr=thr))
        finally:
            os.environ.pop("BAK_BLOCK_KERNEL", None)
        assert orc.rel_coeff_err(rep.a_hat, ref["a_hat"]) <= _tol(dtype), kern

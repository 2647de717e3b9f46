"""GPU parity of greedy column scoring and forward selection (reference
select.py:56-136) against the reference's own outputs
(tests/golden/select_*.npz) and the CPU oracle, plus the reference's
test_select.py properties restated."""

import numpy as np
import pytest

import golden_io
from oracle import bak_oracle as orc

pytestmark = pytest.mark.gpu


def _pb():
    import paper_2104_12570_b200 as pb
    return pb


def _randn(rng, obs, nv, dtype=np.float64):
    return np.asfortranarray(rng.standard_normal((obs, nv)).astype(dtype))


def _sparse(rng, obs, nv, k):
    x = _randn(rng, obs, nv)
    sup = sorted(rng.choice(nv, size=k, replace=False).tolist())
    a = np.zeros(nv)
    a[sup] = rng.uniform(1.0, 2.0, k) * rng.choice([-1.0, 1.0], k)
    return x, x @ a, sup


@pytest.mark.parametrize("name", golden_io.select_names("score"))
def test_scores_match_reference_fixture(name):
    pb = _pb()
    g = golden_io.load_select(name)
    if g["exhausted"]:
        with pytest.raises(pb.SelectionExhaustedError):
            pb.score_all_columns(g["x"], g["e"], excluded=g["excluded"])
        return
    best, scores = pb.score_all_columns(g["x"], g["e"], excluded=g["excluded"])
    assert best == g["best"]
    fin = np.isfinite(g["scores"])
    assert np.array_equal(np.isfinite(scores), fin)
    e2 = float(np.dot(g["e"].astype(np.float64), g["e"].astype(np.float64)))
    tol = 1e-10 if g["x"].dtype == np.float64 else 1e-5
    assert np.max(np.abs(scores[fin] - g["scores"][fin])) <= tol * e2


@pytest.mark.parametrize("name", golden_io.select_names("select"))
def test_selection_matches_reference_fixture(name):
    pb = _pb()
    g = golden_io.load_select(name)
    rc = g["refit_cfg"]
    cfg = pb.FeatureSelectConfig(max_feat=g["max_feat"], refit=g["refit"], stop_tol=g["stop_tol"],
                                 refit_config=pb.SolveConfig(**rc) if rc else None)
    rep = pb.select_features(g["x"], g["y"], cfg)
    assert rep.selected == g["selected"]
    tol = 1e-8 if g["x"].dtype == np.float64 else 1e-4
    np.testing.assert_allclose(rep.final_coeffs, g["final_coeffs"], rtol=tol, atol=tol)
    yn2 = float(np.dot(g["y"].astype(np.float64), g["y"].astype(np.float64)))
    assert np.max(np.abs(np.asarray(rep.residual_norms) - g["residual_norms"])) <= 10 * tol * yn2


@pytest.mark.parametrize("obs,nv,dtype", [(100_000, 40, np.float64), (3000, 3000, np.float32),
                                          (64, 20_000, np.float64), (1, 5, np.float64)])
def test_scores_match_oracle_at_shape(obs, nv, dtype):
    pb = _pb()
    rng = np.random.default_rng(obs + nv)
    x = _randn(rng, obs, nv, dtype)
    e = rng.standard_normal(obs).astype(dtype)
    excl = [0, nv // 2]
    best_ref, s_ref = orc.score_all_columns(x, e, excluded=excl)
    best, s = pb.score_all_columns(x, e, excluded=excl)
    fin = np.isfinite(s_ref)
    assert np.array_equal(np.isfinite(s), fin)
    e2 = float(np.dot(e.astype(np.float64), e.astype(np.float64)))
    tol = 1e-10 if dtype == np.float64 else 1e-5
    assert np.max(np.abs(s[fin] - s_ref[fin])) <= tol * e2
    gap = np.sort(s_ref[fin])
    if gap.size < 2 or gap[1] - gap[0] > 100 * tol * e2:   # a clear winner must be found
        assert best == best_ref


def test_score_properties():
    """test_select.py:11-77 restated."""
    pb = _pb()
    rng = np.random.default_rng(40)
    x = _randn(rng, 30, 6)
    best, scores = pb.score_all_columns(x, x[:, 3].copy())
    assert best == 3 and abs(scores[3]) <= 1e-10
    rng = np.random.default_rng(41)
    q, _ = np.linalg.qr(rng.standard_normal((20, 5)))
    e = rng.standard_normal(20)
    e -= q @ (q.T @ e)
    _, scores = pb.score_all_columns(np.asfortranarray(q), e)
    np.testing.assert_allclose(scores, np.dot(e, e), rtol=1e-10)
    rng = np.random.default_rng(56)
    col = rng.standard_normal(25)
    best, scores = pb.score_all_columns(np.asfortranarray(np.column_stack([col, col, col])), rng.standard_normal(25))
    assert scores[0] == scores[1] == scores[2] and best == 0
    rng = np.random.default_rng(42)
    x = _randn(rng, 20, 5)
    e = rng.standard_normal(20)
    _, scores = pb.score_all_columns(x, e)
    for j in range(5):
        c = x[:, j]
        trial = e - np.dot(c, e) / np.dot(c, c) * c
        assert scores[j] == pytest.approx(float(np.dot(trial, trial)), rel=1e-12)
    rng = np.random.default_rng(44)
    x = _randn(rng, 30, 4)
    e = x[:, 1].copy()
    assert pb.score_all_columns(x, e, excluded=[1])[0] != 1
    x[:, 2] = 0.0
    assert pb.score_all_columns(x, e)[1][2] == np.inf
    with pytest.raises(pb.SelectionExhaustedError):
        pb.score_all_columns(x, e, excluded=[0, 1, 3])
    with pytest.raises(ValueError):
        pb.score_all_columns(x, np.zeros(29))


def test_selection_properties():
    """test_select.py:80-160 restated (QR and solve_bak refits)."""
    pb = _pb()
    rng = np.random.default_rng(45)
    x = _randn(rng, 50, 6)
    rep = pb.select_features(x, 4.0 * x[:, 2], pb.FeatureSelectConfig(max_feat=1))
    assert rep.selected == [2] and rep.residual_norms[0] <= 1e-20
    np.testing.assert_allclose(rep.final_coeffs, [4.0], atol=1e-12)
    for seed in (3000, 3001, 3002):
        x, y, sup = _sparse(np.random.default_rng(seed), 500, 50, 3)
        rep = pb.select_features(x, y, pb.FeatureSelectConfig(max_feat=3))
        assert sorted(rep.selected) == sup
    x, y, sup = _sparse(np.random.default_rng(47), 200, 30, 2)
    rep = pb.select_features(x, y, pb.FeatureSelectConfig(max_feat=10, stop_tol=1e-8))
    assert len(rep.selected) == 2 and sorted(rep.selected) == sup
    x, y, _ = _sparse(np.random.default_rng(48), 300, 40, 4)
    qr_rep = pb.select_features(x, y, pb.FeatureSelectConfig(max_feat=4))
    bak_rep = pb.select_features(x, y, pb.FeatureSelectConfig(max_feat=4, refit="bak",
                                                              refit_config=pb.SolveConfig(max_iter=4000, tol=1e-10)))
    assert bak_rep.selected == qr_rep.selected
    np.testing.assert_allclose(bak_rep.final_coeffs, qr_rep.final_coeffs, atol=1e-5)
    rng = np.random.default_rng(49)
    x = _randn(rng, 80, 10)
    x[:, 4] = 0.0
    rep = pb.select_features(x, rng.standard_normal(80), pb.FeatureSelectConfig(max_feat=9))
    assert len(set(rep.selected)) == 9 and 4 not in rep.selected
    rng = np.random.default_rng(50)
    x = _randn(rng, 100, 15)
    rn = pb.select_features(x, rng.standard_normal(100), pb.FeatureSelectConfig(max_feat=15)).residual_norms
    assert all(rn[i + 1] <= rn[i] * (1 + 1e-12) for i in range(len(rn) - 1))
    rng = np.random.default_rng(51)
    x = _randn(rng, 120, 12)
    y = rng.standard_normal(120)
    for k in (1, 3, 6):
        rep = pb.select_features(x, y, pb.FeatureSelectConfig(max_feat=k))
        xs = x[:, rep.selected]
        assert np.max(np.abs(xs.T @ (y - xs @ rep.final_coeffs))) <= 1e-6


def test_selection_validation():
    pb = _pb()
    rng = np.random.default_rng(53)
    x = _randn(rng, 10, 3)
    with pytest.raises(ValueError):
        pb.select_features(x, np.ones(10), pb.FeatureSelectConfig(max_feat=4))
    with pytest.raises(ValueError):
        pb.select_features(x, np.ones(9), pb.FeatureSelectConfig(max_feat=1))

"""Pin the CPU oracle (oracle/bak_oracle.py) against fixtures produced by the
real reference (tests/golden/make_golden.py).  CPU only.

On the host that produced the fixtures (same OpenBLAS core) the restatement is
required to be BIT-identical; elsewhere (different BLAS kernel) it must agree
to the SURVEY §8c parity tolerances.
"""

import json

import numpy as np
import pytest
from threadpoolctl import threadpool_info

import golden_io
from oracle import bak_oracle as orc


def _same_blas(host):
    np.dot(np.ones(2), np.ones(2))
    blas = [i for i in threadpool_info() if i.get("user_api") == "blas"]
    if not blas or host.get("blas") is None:
        return False
    mine = [blas[0].get("internal_api"), blas[0].get("version"), blas[0].get("architecture")]
    return mine == list(host["blas"]) and np.__version__ == host["numpy"]


@pytest.mark.parametrize("name", golden_io.names())
def test_oracle_matches_reference_fixture(name):
    g = golden_io.load(name)
    x, y = g["x"], g["y"]
    assert golden_io.input_sha(x, y) == str(g["input_sha"]), "generator restatement drifted"
    out = orc.solve(x, y, a0=g["a0"], **g["config"])
    assert out["sweeps_run"] == int(g["sweeps_run"])
    assert out["converged"] == bool(g["converged"])
    assert out["drift_warning"] == bool(g["drift_warning"])
    if bool(g["has_history"]):
        assert len(out["residual_norm_history"]) == len(g["history"])
    if _same_blas(g["host"]):
        assert out["a_hat"].tobytes() == g["a_hat"].tobytes()
        assert out["residual"].tobytes() == g["residual"].tobytes()
        if bool(g["has_history"]):
            assert np.array_equal(np.asarray(out["residual_norm_history"]), g["history"])
    else:
        tol = 1e-10 if x.dtype == np.float64 else 1e-4
        assert orc.rel_coeff_err(out["a_hat"], g["a_hat"]) <= tol


def test_coordinate_update_kat():
    with np.load(golden_io.os.path.join(golden_io.GOLDEN, "kat_coordinate_update.npz")) as z:
        da, e_next = orc.coordinate_update(z["col"], z["e"])
        assert da == float(z["da"]) == pytest.approx(2.2, rel=1e-15)
        np.testing.assert_array_equal(e_next, z["e_next"])


def test_permutations_compound():
    p = orc.permutations(11, 30, 3)
    gen = orc.philox(11)
    order = np.arange(30)
    for s in range(3):
        gen.shuffle(order)
        assert np.array_equal(p[s], order)
    assert not np.array_equal(p[0], p[1])


def test_config_generators_shapes():
    x, y, a = orc.config_c1(obs=100, nvars=10)
    assert x.shape == (100, 10) and x.flags.f_contiguous and y.shape == (100,)
    x, y, a = orc.config_c2(n=64)
    assert x.shape == (64, 64) and np.all(np.diag(x) > 3.0)
    x, y, _ = orc.config_c4(obs=10, nvars=50)
    assert x.shape == (10, 50) and y.shape == (10,)
    x, y, _ = orc.config_c5_system(0)
    assert x.dtype == np.float32 and x.shape == (512, 32)


def test_manifest_lists_every_fixture():
    with open(golden_io.os.path.join(golden_io.GOLDEN, "MANIFEST.json")) as f:
        man = json.load(f)
    assert sorted(man["cases"]) == golden_io.names()
    assert sorted(man["bakp_cases"]) == golden_io.bakp_names()
    assert sorted(man["select_cases"]) == golden_io.select_names()


@pytest.mark.parametrize("name", golden_io.bakp_names())
def test_oracle_bakp_matches_reference_fixture(name):
    """solve_bakp restatement (bakp.py:132-185) against the reference's own runs."""
    g = golden_io.load_bakp(name)
    x, y = g["x"], g["y"]
    assert golden_io.input_sha(x, y) == str(g["input_sha"])
    if g["diverged"]:
        with np.errstate(invalid="ignore", over="ignore"):
            with pytest.raises(orc.DivergenceError) as ei:
                orc.solve_bakp(x, y, thr=g["thr"], **g["config"])
        if _same_blas(g["host"]):
            assert str(ei.value) == str(g["message"])
        return
    out = orc.solve_bakp(x, y, thr=g["thr"], **g["config"])
    assert out["sweeps_run"] == int(g["sweeps_run"])
    assert out["converged"] == bool(g["converged"])
    assert out["drift_warning"] == bool(g["drift_warning"])
    if _same_blas(g["host"]):
        assert out["a_hat"].tobytes() == g["a_hat"].tobytes()
        assert out["residual"].tobytes() == g["residual"].tobytes()
        if bool(g["has_history"]):
            assert np.array_equal(np.asarray(out["residual_norm_history"]), g["history"])
    else:
        tol = 1e-10 if x.dtype == np.float64 else 1e-4
        assert orc.rel_coeff_err(out["a_hat"], g["a_hat"]) <= tol


def test_oracle_bakp_thr1_is_the_sweep():
    """bakp.py:13-15: thr=1 reproduces solve_bak bit for bit."""
    g = golden_io.load("c1_scaled_2000x40_f64")
    a = orc.solve(g["x"], g["y"], max_iter=20, tol=0, record_history=True)
    b = orc.solve_bakp(g["x"], g["y"], max_iter=20, tol=0, thr=1, record_history=True)
    assert a["a_hat"].tobytes() == b["a_hat"].tobytes()
    assert a["residual_norm_history"] == b["residual_norm_history"]


def test_block_deltas_kat():
    with np.load(golden_io.os.path.join(golden_io.GOLDEN, "kat_block_deltas.npz")) as z:
        np.testing.assert_array_equal(orc.block_deltas(np.eye(2, order="F"), 0, 2, np.array([3.0, 4.0]),
                                                       np.ones(2)), z["eye"])
        col = np.array([1.0, 2.0, -1.0])
        xd = np.asfortranarray(np.column_stack([col, col]))
        np.testing.assert_array_equal(orc.block_deltas(xd, 0, 2, col.copy(), orc.column_norms_sq(xd)), z["dup"])


@pytest.mark.parametrize("name", golden_io.select_names("score"))
def test_oracle_scores_match_reference_fixture(name):
    """score_all_columns restatement (select.py:56-85)."""
    g = golden_io.load_select(name)
    if g["exhausted"]:
        with pytest.raises(orc.SelectionExhaustedError):
            orc.score_all_columns(g["x"], g["e"], excluded=g["excluded"])
        return
    best, scores = orc.score_all_columns(g["x"], g["e"], excluded=g["excluded"])
    assert best == g["best"]
    if _same_blas(g["host"]):
        assert scores.tobytes() == g["scores"].tobytes()
    else:
        fin = np.isfinite(g["scores"])
        assert np.array_equal(np.isfinite(scores), fin)
        np.testing.assert_allclose(scores[fin], g["scores"][fin], rtol=1e-5, atol=1e-8)


@pytest.mark.parametrize("name", golden_io.select_names("select"))
def test_oracle_selection_matches_reference_fixture(name):
    """select_features + Householder / solve_bak refit restatement (select.py:88-136, qr.py)."""
    g = golden_io.load_select(name)
    out = orc.select_features(g["x"], g["y"], g["max_feat"], refit=g["refit"], stop_tol=g["stop_tol"],
                              refit_config=g["refit_cfg"] or None)
    assert out["selected"] == g["selected"]
    if _same_blas(g["host"]):
        assert np.asarray(out["final_coeffs"]).tobytes() == g["final_coeffs"].tobytes()
        assert out["residual_norms"] == g["residual_norms"].tolist()
    else:
        np.testing.assert_allclose(out["final_coeffs"], g["final_coeffs"], rtol=1e-6, atol=1e-9)

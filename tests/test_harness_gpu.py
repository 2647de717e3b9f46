"""The benchmark harness and CLI on the GPU (reference bench.py / cli.py;
SURVEY §8f row 2): run_case records agree with the reference's own run_case
on the same generated systems (tests/golden/harness_records.json), and the
reference's test_bench.py / test_cli.py behaviours hold."""

import dataclasses
import json
import os

import numpy as np
import pytest

import golden_io

pytestmark = pytest.mark.gpu


def _h():
    from paper_2104_12570_b200 import harness
    return harness


def _spec(**kw):
    h = _h()
    base = dict(case_id="t", solver="bak", system=h.SystemSpec(obs=400, vars=40, seed=7), precision="single",
                tol=1e-6, max_iter=300, repetitions=1)
    base.update(kw)
    return h.RunSpec(**base)


def _load_records():
    with open(os.path.join(golden_io.GOLDEN, "harness_records.json")) as f:
        return json.load(f)


@pytest.mark.parametrize("case", _load_records(), ids=lambda c: c["spec"]["case_id"])
def test_run_case_matches_reference_records(case):
    h = _h()
    c, ref = case["spec"], case["record"]
    rec = h.run_case(h.RunSpec(case_id=c["case_id"], solver=c["solver"],
                               system=h.SystemSpec(obs=c["obs"], vars=c["vars"], seed=c["seed"]),
                               precision=c["precision"], thr=c.get("thr", 50), tol=c["tol"], max_iter=c["max_iter"],
                               repetitions=1, mape_base=c.get("mape_base", "targets")))
    assert (rec.obs, rec.vars, rec.solver, rec.thr, rec.seed, rec.failed) == (
        ref["obs"], ref["vars"], ref["solver"], ref["thr"], ref["seed"], ref["failed"])
    assert rec.converged == ref["converged"]
    if c["precision"] == "double":
        assert rec.sweeps == ref["sweeps"]
        for k in ("mape", "rel_residual"):
            assert abs(getattr(rec, k) - ref[k]) <= max(1e-3 * ref[k], 1e-12)
    else:   # fp32 solves end at the single-precision noise floor: same regime, not the same bits
        assert abs(rec.sweeps - ref["sweeps"]) <= 1
        for k in ("mape", "rel_residual"):
            assert getattr(rec, k) <= max(3 * ref[k], 1e-5)


def test_run_case_behaviour(tmp_path):
    """test_bench.py:38-125 restated."""
    h = _h()
    import paper_2104_12570_b200 as pb
    a, b = h.run_case(_spec()), h.run_case(_spec())
    norm = lambda r: dataclasses.replace(r, wall_time_s=0.0)  # noqa: E731
    assert norm(a) == norm(b) and a.wall_time_s > 0
    rec = h.run_case(_spec(system=h.SystemSpec(obs=1000, vars=100, seed=5)))
    assert rec.converged and not rec.failed and rec.mape <= 1e-5 and rec.rel_residual <= 1e-5
    assert rec.thr == 0 and rec.workers == 0
    rec = h.run_case(_spec(solver="qr"))
    assert rec.converged and rec.sweeps == 0 and rec.rel_residual <= 1e-5
    rec = h.run_case(_spec(solver="qr", precision="double", mape_base="coeffs"))
    assert rec.mape <= 1e-8
    rng = np.random.default_rng(70)
    p = tmp_path / "sys.bin"
    pb.save_matrix(p, np.asfortranarray(rng.standard_normal((20, 4))))
    with pytest.raises(ValueError, match="known coefficients"):
        h.run_case(_spec(system=str(p), mape_base="coeffs"))
    rng = np.random.default_rng(71)
    x = np.asfortranarray(rng.standard_normal((50, 5)))
    pb.save_matrix(p, np.asfortranarray(np.column_stack([x, x @ rng.standard_normal(5)])))
    rec = h.run_case(_spec(system=str(p), precision="double", tol=1e-10, max_iter=5000))
    assert rec.converged and rec.rel_residual <= 1e-10 and (rec.obs, rec.vars, rec.seed) == (50, 5, 0)
    pb.save_matrix(p, np.ones((5, 1), order="F"))
    with pytest.raises(ValueError, match="at least 2 columns"):
        h.run_case(_spec(system=str(p)))
    col = np.random.default_rng(21).standard_normal(50)
    pb.save_matrix(p, np.asfortranarray(np.column_stack([np.tile(col[:, None], (1, 5)), col])))
    rec = h.run_case(_spec(solver="bakp", system=str(p), precision="double", thr=5))
    assert rec.failed and not rec.converged and "thr=5" in rec.error
    assert np.isnan(rec.mape) and np.isnan(rec.rel_residual) and np.isnan(rec.wall_time_s)
    out = tmp_path / "coeffs.bin"
    rec = h.run_case(_spec(precision="double", tol=1e-10, max_iter=3000), dump_coeffs=out)
    a = pb.load_matrix(out)
    assert a.shape == (40, 1)
    x, y, _ = h.generate_system(h.SystemSpec(obs=400, vars=40, seed=7), "double")
    assert abs(np.linalg.norm(y - x @ a[:, 0]) / np.linalg.norm(y) - rec.rel_residual) <= 1e-6


def test_run_suite_and_cli(tmp_path, capsys):
    h = _h()
    from paper_2104_12570_b200 import cli
    p = tmp_path / "s.csv"
    p.write_text("case_id,solver,obs,vars,seed,precision,reps,max_iter,thr\n"
                 "c1,bak,200,20,1,double,1,500,5\nc1,qr,200,20,1,double,1,500,5\nc1,bakp,200,20,1,double,1,500,5\n")
    seen = []
    records = h.run_suite(p, on_record=seen.append)
    assert [r.solver for r in records] == ["bak", "qr", "bakp"] and seen == records
    assert all(r.converged and not r.failed and r.mape <= 1e-5 for r in records)
    out = tmp_path / "report.csv"
    assert cli.main(["bench", "--suite", str(p), "--out", str(out)]) == 0
    text = capsys.readouterr().out
    assert "c1: bak 200x20 precision=double" in text and out.exists()
    assert cli.main(["bench", "--obs", "300", "--vars", "30", "--solver", "bakp", "--thr", "5", "--reps", "1",
                     "--precision", "f64"]) == 0
    assert "bakp-300x30-s0: bakp 300x30 precision=double" in capsys.readouterr().out
    assert cli.main(["bench", "--obs", "30", "--vars", "5", "--solver", "bakp", "--thr", "6", "--reps", "1"]) == 2
    bad = tmp_path / "bad.csv"
    bad.write_text("case_id,solver,obs,vars,seed\nc1,nosuch,4,2,0\n")
    assert cli.main(["bench", "--suite", str(bad)]) == 2
    import paper_2104_12570_b200 as pb
    rng = np.random.default_rng(72)
    x = np.asfortranarray(rng.standard_normal((100, 12)))
    xf, yf = tmp_path / "x.bakm", tmp_path / "y.bakm"
    pb.save_matrix(xf, x)
    pb.save_matrix(yf, (3.0 * x[:, 4] - 2.0 * x[:, 9]).reshape(-1, 1))
    sel_out = tmp_path / "sel.csv"
    assert cli.main(["select", "--input", str(xf), "--target", str(yf), "--max-feat", "2",
                     "--out", str(sel_out)]) == 0
    assert "bakf: selected [4, 9]" in capsys.readouterr().out and sel_out.exists()
    assert cli.main(["select", "--input", str(tmp_path / "missing.bakm"), "--target", str(yf),
                     "--max-feat", "1"]) == 2

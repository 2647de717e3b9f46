"""Harness host logic (reference bench.py / cli.py): MAPE,
suite parsing, the report CSV, RunSpec validation, and the product-side
input generator reproducing the reference's bytes.  CPU only."""

import csv
import os

import numpy as np
import pytest

import golden_io

h = pytest.importorskip("paper_2104_12570_b200.harness")


def test_mape_values():
    assert h.mape([1.0, 2.0], [1.0, 2.0]) == (0.0, False)
    r = h.mape([2.0, 4.0], [1.0, 4.0])
    assert r.value == pytest.approx(0.5) and not r.fallback
    assert h.mape([3.0, -3.0], [0.0, 0.0]) == (3.0, True)
    r = h.mape([2e-12, 2.0], [1e-12, 1.0], floor=1e-12)
    assert r.value == pytest.approx(1.0) and not r.fallback
    with pytest.raises(ValueError):
        h.mape([1.0], [1.0, 2.0])
    with pytest.raises(ValueError):
        h.mape(np.ones((2, 2)), np.ones((2, 2)))


def test_runspec_validation():
    with pytest.raises(ValueError):
        h.RunSpec(case_id="t", solver="lsqr", system=h.SystemSpec(obs=4, vars=2))
    with pytest.raises(ValueError):
        h.RunSpec(case_id="t", solver="bak", system=h.SystemSpec(obs=4, vars=2), repetitions=0)
    with pytest.raises(ValueError):
        h.RunSpec(case_id="t", solver="bak", system=h.SystemSpec(obs=4, vars=2), mape_base="predictions")
    with pytest.raises(ValueError):
        h.SystemSpec(obs=0, vars=2)
    with pytest.raises(ValueError):
        h.SystemSpec(obs=2, vars=2, distribution="cauchy")


def test_parse_suite(tmp_path):
    p = tmp_path / "s.csv"
    p.write_text("case_id,solver,obs,vars,seed\nc1,bak,100,10,3\n")
    (s,) = h.parse_suite(p)
    assert s.case_id == "c1" and s.system == h.SystemSpec(obs=100, vars=10, seed=3)
    assert (s.precision, s.thr, s.workers, s.tol, s.max_iter, s.repetitions, s.mape_base) == (
        "single", 50, 0, 1e-6, 1000, 10, "targets")
    p.write_text("case_id,solver,obs,vars,seed\nc1,bak,100,10,3\nc2,nosuch,4,2,0\n")
    with pytest.raises(h.SuiteFormatError, match=r"line 3: unknown solver 'nosuch' in field 'solver'"):
        h.parse_suite(p)
    p.write_text("case_id,solver,obs,vars,seed\nc1,bak,xx,10,3\n")
    with pytest.raises(h.SuiteFormatError, match=r"line 2: bad value 'xx' in field 'obs'"):
        h.parse_suite(p)
    p.write_text("case_id,solver,obs,seed\nc1,bak,4,1\n")
    with pytest.raises(h.SuiteFormatError, match=r"line 1: missing column 'vars'"):
        h.parse_suite(p)
    p.write_text("case_id,solver,obs,vars,seed\n")
    assert h.parse_suite(p) == []
    p.write_text("case_id,solver,obs,vars,seed\n,,,,\nc1,qr,10,2,0\n")
    assert len(h.parse_suite(p)) == 1


def _rec(**kw):
    base = dict(case_id="r", obs=10, vars=2, solver="bak", thr=0, precision="single", wall_time_s=0.5, sweeps=3,
                mape=2e-6, rel_residual=1e-6, seed=1, converged=True)
    base.update(kw)
    return h.BenchmarkRecord(**base)


def test_emit_report(tmp_path):
    records = [_rec(case_id="a", solver="qr", wall_time_s=2.0, sweeps=0), _rec(case_id="a", solver="bak"),
               _rec(case_id="b", solver="bakp", thr=4, wall_time_s=0.25),
               _rec(case_id="c", solver="bakp", thr=8, failed=True, converged=False, wall_time_s=float("nan"),
                    mape=float("nan"), rel_residual=float("nan"), error="diverged")]
    out = tmp_path / "report.csv"
    h.emit_report(records, out)
    with open(out, newline="") as f:
        rows = list(csv.reader(f))
    assert rows[0] == list(h.REPORT_HEADER)
    by = {(r[0], r[3]): r for r in rows[1:]}
    assert by[("a", "qr")][-1] == "1" and by[("a", "bak")][-1] == "4" and by[("b", "bakp")][-1] == ""
    assert by[("c", "bakp")][1:5] == ["10", "2", "bakp", "8"] and by[("c", "bakp")][5:10] == [""] * 5
    h.emit_report([], out)
    with open(out, newline="") as f:
        assert list(csv.reader(f)) == [list(h.REPORT_HEADER)]


def test_bundled_suite_parses():
    specs = h.parse_suite(h.bundled_suite_path())
    assert specs and {s.solver for s in specs} <= set(h.SOLVERS)


@pytest.mark.parametrize("name", ["c1_scaled_2000x40_f64", "c1_scaled_2000x40_f32", "early_break_1000x100_f32"])
def test_product_generator_reproduces_reference_bytes(name):
    """generate_system in the product harness yields the reference's exact
    input bytes (the fixture stores the SHA-256 of the reference's draw)."""
    import json
    with np.load(os.path.join(golden_io.GOLDEN, name + ".npz")) as z:
        spec = json.loads(str(z["spec"]))
        sha = str(z["input_sha"])
    x, y, _ = h.generate_system(h.SystemSpec(obs=spec["obs"], vars=spec["vars"], seed=spec["seed"],
                                             distribution=spec["distribution"],
                                             coeff_distribution=spec["coeff_distribution"],
                                             noise_sigma=spec["noise_sigma"]), spec["precision"])
    assert golden_io.input_sha(x, y) == sha


def test_cli_parser_mirrors_reference_flags():
    from paper_2104_12570_b200.cli import build_parser
    a = build_parser().parse_args(["bench", "--obs", "10", "--vars", "2", "--solver", "bakp", "--thr", "2",
                                   "--precision", "f64", "--reps", "1", "--mape-base", "coeffs"])
    assert (a.obs, a.vars, a.solver, a.thr, a.precision, a.reps, a.mape_base) == (10, 2, "bakp", 2, "f64", 1,
                                                                                   "coeffs")
    a = build_parser().parse_args(["select", "--input", "x", "--target", "y", "--max-feat", "3", "--refit", "bak"])
    assert (a.method, a.max_feat, a.refit) == ("bakf", 3, "bak")

"""pytest plugin: run the REFERENCE's own test files against the drop-in.

Loaded with ``-p dropin_plugin`` (tests/refsuite on sys.path) when pytest runs
the reference's test modules from ``baseline/_ref/tests`` (staged there by
tools/refsuite/stage_reference.sh; git-ignored, never committed).  Before any
test module is imported it rebinds, in the installed reference package
``baksolve`` 0.1.0, every name on the solve path to this repo's GPU
implementation:

  baksolve.solve_bak / bak.solve_bak / bench.solve_bak / select.solve_bak
  baksolve.coordinate_update, residual_norm            (bak.py:60-79)
  baksolve.solve_bakp / bakp.solve_bakp / bench.solve_bakp, block_deltas
  baksolve.score_all_columns / select_features (select.py)
  DivergenceError, SelectionExhaustedError  (the drop-in's exception types)

so ``from baksolve import solve_bak`` inside the reference's tests (and the
reference's own bench / select modules, which call solve_bak internally)
resolve to the CUDA path — exactly the patch INTEGRATION.md describes for a
reference user.  The reference's SolveConfig / BlockConfig / SystemSpec /
generate_system / qr_least_squares stay the reference's own (input
construction and oracles).  Set BAK_REFSUITE_PATCH=0 to run the reference
unpatched (the baseline of the same run).
"""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

PATCHED = []


def _patch():
    import baksolve
    import baksolve.bak
    import baksolve.bakp
    import baksolve.bench
    import baksolve.select
    import paper_2104_12570_b200 as pb

    table = {
        "solve_bak": pb.solve_bak,
        "coordinate_update": pb.coordinate_update,
        "residual_norm": pb.residual_norm,
        "solve_bakp": pb.solve_bakp,
        "block_deltas": pb.block_deltas,
        "score_all_columns": pb.score_all_columns,
        "select_features": pb.select_features,
        # the drop-in's exception types, so that pytest.raises(...) in the tests and the
        # except clauses in the reference's own modules match what the GPU path raises
        "DivergenceError": pb.DivergenceError,
        "SelectionExhaustedError": pb.SelectionExhaustedError,
    }
    for mod in (baksolve, baksolve.bak, baksolve.bakp, baksolve.bench, baksolve.select):
        for name, fn in table.items():
            if hasattr(mod, name):
                setattr(mod, name, fn)
                PATCHED.append(f"{mod.__name__}.{name}")


def pytest_configure(config):
    if os.environ.get("BAK_REFSUITE_PATCH", "1") != "0":
        _patch()


def pytest_report_header(config):
    return "drop-in: " + (", ".join(PATCHED) if PATCHED else "NOT patched (reference itself)")

"""The reference's OWN test files, unmodified, against the drop-in.

tools/refsuite/stage_reference.sh (run in the build container) installs
baksolve 0.1.0 into baseline/_ref and copies its tests/ next to it (both
git-ignored; gpurun ships them to the box).  Each case below runs those files
in a subprocess with tests/refsuite/dropin_plugin.py, which rebinds
solve_bak / coordinate_update / residual_norm / solve_bakp / block_deltas /
score_all_columns inside the installed ``baksolve`` (and in its bench and
select modules, which call them) to this repo's CUDA implementation before the
test modules import them.  Skipped when the reference is not staged.
"""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
REF_TESTS = os.path.join(REF, "tests")
staged = pytest.mark.skipif(not os.path.exists(os.path.join(REF_TESTS, "test_solver_bak.py")),
                            reason="reference not staged (tools/refsuite/stage_reference.sh)")

CASES = {
    # reference file, -k selection (None = every test in the file)
    "solver_bak": ("test_solver_bak.py", None),
    "solver_bakp": ("test_solver_bakp.py", None),
    "select": ("test_select.py", None),
    # acceptance criteria: 1 monotone + update identity, 2 oracle equivalence (QR),
    # 3 suite accuracy (bench.run_suite), 4 parallel equivalence (bakp workers),
    # 6 feature selection, 7 zero-allocation hot loops (the reference's own loops),
    # 8 degenerate inputs.  Criterion 5 times the reference's CPU solvers against
    # each other (bakp faster than bak on one machine): a property of that code
    # path, not of the results, so it is not run against the GPU.
    "acceptance": ("test_acceptance.py", "not criterion_5"),
}


def _env():
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([REF, os.path.join(ROOT, "tests", "refsuite"), ROOT,
                                         env.get("PYTHONPATH", "")])
    env.pop("BAK_REFSUITE_PATCH", None)
    return env


@staged
@pytest.mark.parametrize("case", sorted(CASES))
def test_reference_file_passes_against_dropin(case):
    fname, sel = CASES[case]
    cmd = [sys.executable, "-m", "pytest", "-q", "-rs", "-p", "dropin_plugin", "-p", "no:cacheprovider",
           "--rootdir", REF_TESTS, fname]
    if sel:
        cmd += ["-k", sel]
    out = subprocess.run(cmd, cwd=REF_TESTS, env=_env(), capture_output=True, text=True, timeout=900)
    log = out.stdout + out.stderr
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", f"refsuite_{case}.log"), "w") as f:
        f.write(" ".join(cmd) + "\n" + log)
    assert out.returncode == 0, log[-4000:]
    assert "passed" in log and "failed" not in log


@staged
def test_plugin_rebinds_the_solve_path():
    code = ("import dropin_plugin as d; d._patch(); import baksolve, baksolve.bench, baksolve.select;"
            "import paper_2104_12570_b200 as pb;"
            "assert baksolve.solve_bak is pb.solve_bak and baksolve.bench.solve_bak is pb.solve_bak;"
            "assert baksolve.select.solve_bak is pb.solve_bak and baksolve.solve_bakp is pb.solve_bakp;"
            "print(len(d.PATCHED))")
    out = subprocess.run([sys.executable, "-c", code], env=_env(), capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    assert int(out.stdout.strip()) >= 10

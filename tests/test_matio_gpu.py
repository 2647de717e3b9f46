"""BAKM file -> pinned host -> GPU: a tall system written
as a BAKM file, read by the native parallel reader straight into pinned host
memory and solved through the pipelined upload path, matches the oracle."""

import numpy as np
import pytest

from oracle import bak_oracle as orc

pytestmark = pytest.mark.gpu


def test_bakm_file_to_pipelined_gram_solve(tmp_path):
    import paper_2104_12570_b200 as pb
    x, y, _ = orc.make_system(1 << 20, 40, 9, "normal", "uniform", 0.01, "double")
    p = tmp_path / "tall.bakm"
    pb.save_matrix(p, x)
    xp = pb.load_matrix_pinned(p)
    assert xp.is_pinned() and xp.stride(0) == 1
    cfg = pb.SolveConfig(max_iter=3, tol=0)
    rep = pb.solve_bak(xp, y, cfg, variant="gram")
    ref = orc.solve(x, y, max_iter=3, tol=0)
    assert rep.sweeps_run == 3
    assert orc.rel_coeff_err(rep.a_hat, ref["a_hat"]) <= 1e-10
    dm = pb.load_matrix_device(p)
    rep2 = pb.solve_bak(dm, y, cfg)
    assert orc.rel_coeff_err(rep2.a_hat, ref["a_hat"]) <= 1e-10

"""Full-size BASELINE configs 1 and 2 (and the 1e-10 early-break variant)
plus the paper-scale blocked sweep against the CPU oracle (numpy restatement
of the reference): one JSON line each."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import bak_oracle as orc  # noqa: E402
import paper_2104_12570_b200 as pb  # noqa: E402


def line(name, x, y, rep, ref):
    r_ref = orc.residual_norm_f64(x, y, ref["a_hat"])
    r = orc.residual_norm_f64(x, y, rep.a_hat)
    yn = float(np.linalg.norm(np.asarray(y, np.float64)))
    print(json.dumps({"config": name, "shape": list(x.shape), "variant": rep.variant,
                      "coeff_rel_err": orc.rel_coeff_err(rep.a_hat, ref["a_hat"]),
                      "residual_norm_oracle": r_ref, "residual_norm_gpu": r,
                      "residual_diff_rel": abs(r - r_ref) / (r_ref if r_ref >= 1e-6 * yn else yn),
                      "sweeps_run": [rep.sweeps_run, ref["sweeps_run"]],
                      "converged": [bool(rep.converged), bool(ref["converged"])]}), flush=True)


x, y, _ = orc.config_c1()
line("c1", x, y, pb.solve_bak(x, y, pb.SolveConfig(max_iter=100, tol=0)), orc.solve(x, y, max_iter=100, tol=0))
x, y, _ = orc.config_c2()
line("c2", x, y, pb.solve_bak(x, y, pb.SolveConfig(max_iter=50, tol=0)), orc.solve(x, y, max_iter=50, tol=0))
line("c2b", x, y, pb.solve_bak(x, y, pb.SolveConfig(max_iter=50, tol=1e-10)), orc.solve(x, y, max_iter=50, tol=1e-10))
rng = np.random.default_rng(1)
x = np.asfortranarray(rng.standard_normal((10_000, 1000)).astype(np.float32))
y = (x @ rng.uniform(-1, 1, 1000).astype(np.float32)).astype(np.float32)
line("p1", x, y, pb.solve_bakp(x, y, pb.BlockConfig(base=pb.SolveConfig(max_iter=20, tol=0), thr=50)),
     orc.solve_bakp(x, y, max_iter=20, tol=0, thr=50))

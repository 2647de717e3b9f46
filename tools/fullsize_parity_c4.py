"""Full-size BASELINE config 4 (1,000 x 10^6 fp64, 10 sweeps) against the CPU
oracle (numpy restatement of the reference, one core): coefficients and the
residual norm (relative to ||y||: the system is solved to the rounding floor)."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import bak_oracle as orc  # noqa: E402
import paper_2104_12570_b200 as pb  # noqa: E402

x, y, _ = orc.config_c4()
t0 = time.time()
ref = orc.solve(x, y, max_iter=10, tol=0)
t_cpu = time.time() - t0
r_ref = orc.residual_norm_f64(x, y, ref["a_hat"])
rep = pb.solve_bak(x, y, pb.SolveConfig(max_iter=10, tol=0))
r = orc.residual_norm_f64(x, y, rep.a_hat)
print(json.dumps({"config": "c4", "obs": x.shape[0], "vars": x.shape[1], "sweeps": 10, "variant": rep.variant,
                  "oracle_seconds_1core": round(t_cpu, 1), "coeff_rel_err": orc.rel_coeff_err(rep.a_hat, ref["a_hat"]),
                  "residual_norm_oracle": r_ref, "residual_norm_gpu": r,
                  "residual_diff_rel_to_ynorm": abs(r - r_ref) / float(np.linalg.norm(y)),
                  "a_norm": float(np.linalg.norm(rep.a_hat)), "sweeps_run": rep.sweeps_run}), flush=True)

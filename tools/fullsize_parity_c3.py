"""Full-size BASELINE config 3 (2^24 x 256, 20 sweeps) against the CPU oracle
(the bit-for-bit numpy restatement of the reference, one core): the GPU's
GRAM and exact STREAM results, both precisions.  Minutes of CPU per
precision; writes one JSON line per precision."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import bak_oracle as orc  # noqa: E402
import paper_2104_12570_b200 as pb  # noqa: E402

for precision in sys.argv[1:] or ["single", "double"]:
    x, y, _ = orc.config_c3(precision=precision)
    t0 = time.time()
    ref = orc.solve(x, y, max_iter=20, tol=0)
    t_cpu = time.time() - t0
    r_ref = orc.residual_norm_f64(x, y, ref["a_hat"])
    out = {"config": "c3", "precision": precision, "obs": x.shape[0], "vars": x.shape[1], "sweeps": 20,
           "oracle_seconds_1core": round(t_cpu, 1), "residual_norm_oracle": r_ref}
    for variant in ("gram", "stream"):
        rep = pb.solve_bak(x, y, pb.SolveConfig(max_iter=20, tol=0), variant=variant)
        r = orc.residual_norm_f64(x, y, rep.a_hat)
        out[variant] = {"coeff_rel_err": orc.rel_coeff_err(rep.a_hat, ref["a_hat"]),
                        "residual_norm_rel_diff": abs(r - r_ref) / r_ref, "sweeps_run": rep.sweeps_run}
    print(json.dumps(out), flush=True)

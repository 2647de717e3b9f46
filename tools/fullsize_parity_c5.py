"""Full-size BASELINE config 5 (65,536 systems of 512 x 32 fp32, 200 sweeps)
against the CPU oracle (numpy restatement of the reference), the systems
spread over all host cores (one BLAS thread each): per-system coefficient
error of the GPU batched solve, max over systems."""
import json
import os
import sys
import time
from multiprocessing import Pool

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
NSYS = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
CH = 1024


def work(c0):
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    from oracle import bak_oracle as orc
    xs, ys, aa = [], [], []
    for s in range(c0, min(NSYS, c0 + CH)):
        x, y, _ = orc.config_c5_system(s)
        r = orc.solve(x, y, max_iter=200, tol=0)
        xs.append(x)
        ys.append(y)
        aa.append(r["a_hat"])
    return c0, np.stack(xs), np.stack(ys), np.stack(aa)


if __name__ == "__main__":
    t0 = time.time()
    ncpu = os.cpu_count()
    with Pool(ncpu) as pool:
        parts = sorted(pool.map(work, range(0, NSYS, CH)), key=lambda t: t[0])
    t_cpu = time.time() - t0
    xs = np.concatenate([p[1] for p in parts])
    ys = np.concatenate([p[2] for p in parts])
    a_ref = np.concatenate([p[3] for p in parts])
    import paper_2104_12570_b200 as pb
    from oracle import bak_oracle as orc
    rep = pb.solve_bak_batched(xs, ys, pb.SolveConfig(max_iter=200, tol=0))
    errs = np.array([orc.rel_coeff_err(rep.a_hat[s], a_ref[s]) for s in range(NSYS)])
    print(json.dumps({"config": "c5", "systems": NSYS, "sweeps": 200, "oracle_wall_s": round(t_cpu, 1),
                      "oracle_processes": ncpu, "coeff_rel_err_max": float(errs.max()),
                      "coeff_rel_err_median": float(np.median(errs)),
                      "sweeps_run_min": int(rep.sweeps_run.min()), "sweeps_run_max": int(rep.sweeps_run.max())}),
          flush=True)

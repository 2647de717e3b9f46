import sys, os
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np
import paper_2104_12570_b200 as pb
from paper_2104_12570_b200 import _lib
import test_fuzz_gpu as T
for seed in (12, 13):
    x, y, tol, rng = T._case(seed)
    print("seed", seed, x.shape, x.dtype, tol, flush=True)
    for v in ("auto", "stream", "cta", "cluster", "grid", "gram"):
        try:
            r = pb.solve_bak(x, y, pb.SolveConfig(max_iter=6, tol=tol), variant=v)
            print("  ", v, "ok", r.variant, flush=True)
        except Exception as e:
            print("  ", v, "ERR", str(e)[:200], flush=True)
            _lib.load().bak_last_error()

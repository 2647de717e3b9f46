"""cProfile of the host side of repeated resident solves (a bench config):
where the Python / ctypes time of one solve_bak call goes."""
import cProfile
import os
import pstats
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2104_12570_b200 as pb  # noqa: E402

dev = torch.device("cuda", 0)
cfg = dict(bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c1"])
dm, y = bench.make_inputs(cfg, dev, seed=1234)
sc = pb.SolveConfig(max_iter=cfg["sweeps"], tol=cfg["tol"])
v = cfg.get("variant", "auto")
for _ in range(5):
    pb.solve_bak(dm, y, sc, variant=v, return_device=True)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    pb.solve_bak(dm, y, sc, variant=v, return_device=True)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)

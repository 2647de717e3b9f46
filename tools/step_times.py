"""Per-step times of the default bench solve (C3 GRAM) for N steps in one
process: is the first-process slowdown a warm-up effect?"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2104_12570_b200 as pb  # noqa: E402

dev = torch.device("cuda", 0)
cfg = dict(bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"])
t0 = time.time()
dm, y = bench.make_inputs(cfg, dev, seed=1234)
torch.cuda.synchronize()
print(f"inputs {time.time() - t0:.1f} s", flush=True)
sc = pb.SolveConfig(max_iter=20, tol=0)
for i in range(int(sys.argv[2]) if len(sys.argv) > 2 else 12):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    pb.solve_bak(dm, y, sc, variant="gram", return_device=True)
    b.record()
    torch.cuda.synchronize()
    print(f"step {i}: {a.elapsed_time(b):.1f} ms  wall {(time.time() - t0):.2f} s", flush=True)

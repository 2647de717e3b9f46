"""Timeline of one e2e C3 GRAM solve from pinned host x (torch.profiler /
CUPTI): when the H2D stream finishes vs when the solve ends."""
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2104_12570_b200 as pb  # noqa: E402

dev = torch.device("cuda", 0)
cfg = dict(bench.CONFIGS["c3"])
dm, y = bench.make_inputs(cfg, dev, seed=1)
hx = torch.empty(dm.data.shape, dtype=dm.data.dtype, pin_memory=True)
hx.copy_(dm.data)
hy = torch.empty(y.shape, dtype=y.dtype, pin_memory=True)
hy.copy_(y)
del dm
torch.cuda.empty_cache()
sc = pb.SolveConfig(max_iter=20, tol=0)
hxv = hx.t()[: cfg["obs"]]
pb.solve_bak(hxv, hy, sc, variant="gram")
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    pb.solve_bak(hxv, hy, sc, variant="gram")
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
t0 = min(e.time_range.start for e in ev)
groups = {}
for e in ev:
    k = "memcpy" if "Memcpy" in e.name or "memcpy" in e.name else e.name[:40]
    g = groups.setdefault(k, [1e18, 0, 0.0, 0])
    g[0] = min(g[0], e.time_range.start - t0)
    g[1] = max(g[1], e.time_range.end - t0)
    g[2] += e.time_range.end - e.time_range.start
    g[3] += 1
for k, (a, b, tot, n) in sorted(groups.items(), key=lambda kv: kv[1][0]):
    print(f"{k:42s} first {a / 1e3:9.1f} ms  last_end {b / 1e3:9.1f} ms  busy {tot / 1e3:8.1f} ms  n={n}")
cpu = [e for e in prof.events() if e.device_type.name == "CPU"]
print("cpu span ms:", (max(e.time_range.end for e in cpu) - min(e.time_range.start for e in cpu)) / 1e3)

"""Timeline of one e2e C5 batched solve from pinned host memory (torch.profiler
/ CUPTI): per chunk, when its upload ends and when its solve kernel runs."""
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2104_12570_b200 as pb  # noqa: E402

dev = torch.device("cuda", 0)
cfg = dict(bench.CONFIGS["c5"])
db, y = bench.make_inputs(cfg, dev)
hx = torch.empty(db.data.shape, dtype=db.data.dtype, pin_memory=True)
hx.copy_(db.data)
hy = torch.empty(y.shape, dtype=y.dtype, pin_memory=True)
hy.copy_(y)
hxv = hx.transpose(1, 2)[:, : cfg["obs"], :]
del db
torch.cuda.empty_cache()
sc = pb.SolveConfig(max_iter=cfg["sweeps"], tol=0)
pb.solve_bak_batched(hxv, hy, sc)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    pb.solve_bak_batched(hxv, hy, sc)
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type.name == "CUDA"]
t0 = min(e.time_range.start for e in ev)
for e in sorted(ev, key=lambda e: e.time_range.start):
    d = (e.time_range.end - e.time_range.start) / 1e3
    if d > 0.2:
        print(f"{(e.time_range.start - t0) / 1e3:9.2f} ms  +{d:8.2f} ms  {e.name[:70]}")
print("total", (max(e.time_range.end for e in ev) - t0) / 1e3, "ms")
import time  # noqa: E402
for _ in range(2):
    torch.cuda.synchronize()
    t = time.perf_counter()
    r = pb.solve_bak_batched(hxv, hy, sc)
    torch.cuda.synchronize()
    print("wall of one e2e call", (time.perf_counter() - t) * 1e3, "ms")
with profile(activities=[ProfilerActivity.CPU]) as prof2:
    r = pb.solve_bak_batched(hxv, hy, sc)
print(prof2.key_averages().table(sort_by="cpu_time_total", row_limit=15))

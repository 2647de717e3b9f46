"""Bench-sequence replica (inputs, 1 s prewarm, 3 warm-up solves, 3 timed
solves) under torch.profiler: where does a slow timed step spend its time —
a longer kernel, or the GPU idling (host side)?"""
import gc
import os
import sys
import time

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2104_12570_b200 as pb  # noqa: E402

dev = torch.device("cuda", 0)
cfg = dict(bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3f32"])
dm, y = bench.make_inputs(cfg, dev, seed=1234)
sc = pb.SolveConfig(max_iter=cfg["sweeps"], tol=cfg["tol"])
bench._prewarm(dm, dev)
for _ in range(3):
    pb.solve_bak(dm, y, sc, variant="gram", return_device=True)
torch.cuda.synchronize()
gc.collect()
gc.freeze()
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    for _ in range(3):
        pb.solve_bak(dm, y, sc, variant="gram", return_device=True)
    torch.cuda.synchronize()
ev = sorted((e for e in prof.events() if e.device_type.name == "CUDA"), key=lambda e: e.time_range.start)
t0 = ev[0].time_range.start
end = ev[0].time_range.end
for e in ev[1:]:
    if e.time_range.start - end > 2000:
        print(f"GAP {(e.time_range.start - end) / 1e3:8.2f} ms at {(end - t0) / 1e3:8.2f} ms before {e.name[:60]}")
    end = max(end, e.time_range.end)
long = sorted(ev, key=lambda e: -(e.time_range.end - e.time_range.start))[:12]
for e in long:
    print(f"KERNEL {(e.time_range.end - e.time_range.start) / 1e3:8.2f} ms at {(e.time_range.start - t0) / 1e3:8.2f} ms {e.name[:60]}")
cpu = [e for e in prof.events() if e.device_type.name == "CPU" and (e.time_range.end - e.time_range.start) > 5000]
for e in sorted(cpu, key=lambda e: -(e.time_range.end - e.time_range.start))[:10]:
    print(f"CPU {(e.time_range.end - e.time_range.start) / 1e3:8.2f} ms {e.name[:60]}")
print("span", (max(e.time_range.end for e in ev) - t0) / 1e3)

"""GPU idle gaps across back-to-back resident solves (as bench.py times them):
total span of N solves vs kernel busy time, and the largest gaps with the
device event that follows each (torch.profiler / CUPTI)."""
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2104_12570_b200 as pb  # noqa: E402

dev = torch.device("cuda", 0)
cfg = dict(bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"])
n = int(sys.argv[2]) if len(sys.argv) > 2 else 3
dm, y = bench.make_inputs(cfg, dev, seed=1234)
sc = pb.SolveConfig(max_iter=cfg["sweeps"], tol=cfg["tol"])
variant = cfg.get("variant", "auto")
keep = []
for _ in range(3):
    keep.append(pb.solve_bak(dm, y, sc, variant=variant, return_device=True))
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    e0.record()
    for _ in range(n):
        keep.append(pb.solve_bak(dm, y, sc, variant=variant, return_device=True))
    e1.record()
    torch.cuda.synchronize()
ev = sorted((e for e in prof.events() if e.device_type.name == "CUDA"), key=lambda e: e.time_range.start)
t0, t1 = ev[0].time_range.start, max(e.time_range.end for e in ev)
busy = sum(e.time_range.end - e.time_range.start for e in ev)
gaps = []
end = ev[0].time_range.end
for e in ev[1:]:
    if e.time_range.start > end:
        gaps.append((e.time_range.start - end, e.name[:60]))
    end = max(end, e.time_range.end)
print(f"{n} solves: events {e0.elapsed_time(e1):.2f} ms, device span {(t1 - t0) / 1e3:.2f} ms, "
      f"busy {busy / 1e3:.2f} ms, idle {sum(g for g, _ in gaps) / 1e3:.2f} ms in {len(gaps)} gaps")
for g, nm in sorted(gaps, reverse=True)[:12]:
    print(f"  gap {g / 1e3:8.3f} ms before {nm}")

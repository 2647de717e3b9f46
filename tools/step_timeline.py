"""GPU timeline of one resident solve of a bench config (torch.profiler /
CUPTI): kernel busy time vs the span, and the largest idle gaps."""
import os
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2104_12570_b200 as pb  # noqa: E402

dev = torch.device("cuda", 0)
cfg = dict(bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"])
dm, y = bench.make_inputs(cfg, dev, seed=1234)
sc = pb.SolveConfig(max_iter=cfg["sweeps"], tol=cfg["tol"])
variant = cfg.get("variant", "auto")
for _ in range(3):
    pb.solve_bak(dm, y, sc, variant=variant, return_device=True)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    pb.solve_bak(dm, y, sc, variant=variant, return_device=True)
    torch.cuda.synchronize()
ev = sorted((e for e in prof.events() if e.device_type.name == "CUDA"), key=lambda e: e.time_range.start)
t0, t1 = ev[0].time_range.start, max(e.time_range.end for e in ev)
busy = sum(e.time_range.end - e.time_range.start for e in ev)
gaps = []
end = ev[0].time_range.end
for e in ev[1:]:
    if e.time_range.start > end:
        gaps.append((e.time_range.start - end, e.name[:50]))
    end = max(end, e.time_range.end)
print(f"span {(t1 - t0) / 1e3:.2f} ms, kernel busy {busy / 1e3:.2f} ms, {len(ev)} device events")
import collections  # noqa: E402
per = collections.defaultdict(float)
for e in ev:
    per[e.name[:60]] += (e.time_range.end - e.time_range.start) / 1e3
for n, t in sorted(per.items(), key=lambda kv: -kv[1])[:6]:
    print(f"  {t:9.3f} ms  {n}")
for g, n in sorted(gaps, reverse=True)[:8]:
    print(f"  gap {g / 1e3:8.3f} ms before {n}")

"""Per-sweep cost model of the on-chip blocked kernel: time solve_bakp over a
grid of (obs, thr) and fit t_sweep = nblocks * c_block + vars * c_col.
Tuning aid, not a bench line."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_12570_b200 as pb  # noqa: E402

dev = torch.device("cuda", 0)
nv = 1000
for dt in (torch.float32, torch.float64):
    for obs in (1000, 2000, 10000, 30000):
        g = torch.Generator(device=dev)
        g.manual_seed(0)
        x = torch.randn(nv, obs, dtype=dt, device=dev, generator=g)
        y = x.t() @ (torch.rand(nv, dtype=dt, device=dev, generator=g) - 0.5)
        dm = pb.DeviceMatrix(x, obs, nv, np.float64 if dt == torch.float64 else np.float32)
        rows = []
        for thr in (5, 10, 25, 50, 100, 200):
            cfg = pb.BlockConfig(base=pb.SolveConfig(max_iter=10, tol=0), thr=thr)
            try:
                r = pb.solve_bakp(dm, y, cfg, return_device=True)
            except pb.DivergenceError:
                print(dt, obs, thr, "diverged")
                continue
            torch.cuda.synchronize()
            ts = []
            for _ in range(3):
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                a.record()
                r = pb.solve_bakp(dm, y, cfg, return_device=True)
                b.record()
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
            ms = min(ts) / r.sweeps_run
            nb = -(-nv // thr)
            rows.append((nb, ms))
            print(f"{dt} obs={obs} thr={thr} variant={r.variant} us/sweep={ms * 1e3:.1f} us/block={ms * 1e3 / nb:.2f}",
                  flush=True)
        if len(rows) >= 2:
            A = np.array([[nb, nv] for nb, _ in rows], float)
            t = np.array([ms * 1e3 for _, ms in rows])
            c, *_ = np.linalg.lstsq(A, t, rcond=None)
            print(f"  fit: c_block={c[0]:.2f} us, c_col={c[1] * 1e3:.1f} ns", flush=True)

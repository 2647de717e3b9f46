"""Exact on-chip sweep (GRID, XS plans) on tall systems: device time per column
step and the x-stream bandwidth, N rows x V columns, both precisions.

    python tools/xs_probe.py [rows ...]
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_12570_b200 as pb  # noqa: E402
from paper_2104_12570_b200 import _lib  # noqa: E402

dev = torch.device("cuda", 0)
rows_list = [int(a) for a in sys.argv[1:]] or [1 << 20, 1_500_000, 1 << 21]
nv, sweeps = 256, 4
lib = _lib.load()
for prec, tdt in (("f64", torch.float64), ("f32", torch.float32)):
    for obs in rows_list:
        g = torch.Generator(device=dev).manual_seed(obs)
        ld = obs if (obs * tdt.itemsize) % 16 == 0 else obs + 2
        x = torch.randn((nv, ld), generator=g, device=dev, dtype=tdt)
        dm = pb.DeviceMatrix(x, obs, nv, np.float64 if prec == "f64" else np.float32)
        y = torch.randn(obs, generator=g, device=dev, dtype=tdt)
        cfg = pb.SolveConfig(max_iter=sweeps, tol=0)
        code = dm.code
        picked = _lib.VARIANT_NAMES[int(lib.bak_sweep_pick_variant(code, obs, nv))]
        r = pb.solve_bak(dm, y, cfg, variant="grid", return_device=True)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            r = pb.solve_bak(dm, y, cfg, variant="grid", return_device=True)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 3
        us_col = ms * 1e3 / (sweeps * nv)
        gbs = obs * nv * tdt.itemsize * sweeps / (ms / 1e3) / 1e9
        print(json.dumps(dict(prec=prec, obs=obs, vars=nv, sweeps=sweeps, variant=r.variant, auto=picked,
                              ms=round(ms, 3), us_per_column=round(us_col, 3), x_gbs_whole_solve=round(gbs, 1))),
              flush=True)

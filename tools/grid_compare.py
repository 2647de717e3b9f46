"""Exact sweep per-column time on tall systems: register-resident GRID plan vs the
XS (x-from-shared) GRID plan (BAK_GRID_XS=1) vs STREAM (e in HBM).

    python tools/grid_compare.py rows [rows ...]      (fp64 and fp32, 256 columns, 4 sweeps)
"""
import json
import os
import subprocess
import sys

if len(sys.argv) > 1 and sys.argv[1] == "--one":
    import numpy as np
    import torch
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import paper_2104_12570_b200 as pb
    obs, prec, variant = int(sys.argv[2]), sys.argv[3], sys.argv[4]
    dev = torch.device("cuda", 0)
    tdt = torch.float64 if prec == "f64" else torch.float32
    nv, sweeps = 256, 4
    x = torch.randn((nv, obs + (-obs) % 4), device=dev, dtype=tdt)
    dm = pb.DeviceMatrix(x, obs, nv, np.float64 if prec == "f64" else np.float32)
    y = torch.randn(obs, device=dev, dtype=tdt)
    cfg = pb.SolveConfig(max_iter=sweeps, tol=0)
    pb.solve_bak(dm, y, cfg, variant=variant, return_device=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        pb.solve_bak(dm, y, cfg, variant=variant, return_device=True)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    print(json.dumps(dict(obs=obs, prec=prec, variant=variant, xs=os.environ.get("BAK_GRID_XS", "0"),
                          us_per_column=round(ms * 1e3 / (sweeps * nv), 3),
                          x_gbs=round(obs * nv * tdt.itemsize * sweeps / (ms / 1e3) / 1e9, 1))), flush=True)
    sys.exit(0)

for obs in sys.argv[1:]:
    for prec in ("f64", "f32"):
        for variant, env in (("grid", {}), ("grid", {"BAK_GRID_XS": "1"}), ("stream", {})):
            e = dict(os.environ, **env)
            r = subprocess.run([sys.executable, __file__, "--one", obs, prec, variant], env=e, capture_output=True,
                               text=True, timeout=300)
            print(r.stdout.strip() or r.stderr.strip().splitlines()[-1], flush=True)

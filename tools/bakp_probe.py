"""Kernel-only cost model of the on-chip blocked sweep: time bak_block_sweep
(C-ABI, CUDA events around the launch only) over (vars, thr) and fit
t_sweep = nblocks * c_block + vars * c_col + c_sweep.  Tuning aid."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_12570_b200 as pb  # noqa: E402
from paper_2104_12570_b200 import _lib  # noqa: E402
from paper_2104_12570_b200.bak import _Workspace, _ptr, _stream_ptr  # noqa: E402

lib = _lib.load()
dev = torch.device("cuda", 0)
sweeps = int(os.environ.get("SWEEPS", 20))
for dt in (torch.float32, torch.float64):
    for obs in [int(v) for v in os.environ.get("OBS", "1000,10000").split(",")]:
        rows = []
        for nv in (500, 1000):
            g = torch.Generator(device=dev)
            g.manual_seed(0)
            x = torch.randn(nv, obs, dtype=dt, device=dev, generator=g)
            y = x.t() @ (torch.rand(nv, dtype=dt, device=dev, generator=g) - 0.5)
            dm = pb.DeviceMatrix(x, obs, nv, np.float64 if dt == torch.float64 else np.float32)
            norms = pb.colnorms(dm)
            for thr in (5, 10, 25, 50, 100):
                e = y.clone()
                a = torch.zeros(nv, dtype=dt, device=dev)
                hist = torch.zeros(sweeps, dtype=torch.float64, device=dev)
                st = torch.zeros(4, dtype=torch.int64, device=dev)
                ws = _Workspace(torch, dev, lib.bak_block_sweep_workspace(dm.code, 0, obs, nv, thr))

                def run():
                    e.copy_(y)
                    a.zero_()
                    _lib.check(lib.bak_block_sweep(dm.code, 0, dm.ptr, obs, nv, dm.ldx, _ptr(norms), thr, _ptr(e),
                                                   _ptr(a), sweeps, -1.0, float("inf"), _ptr(hist), _ptr(st),
                                                   ws.ptr, ws.nbytes, _stream_ptr(torch, dev)), "sweep")
                run()
                torch.cuda.synchronize()
                best = 1e9
                for _ in range(3):
                    e.copy_(y)
                    a.zero_()
                    s0 = torch.cuda.Event(enable_timing=True)
                    s1 = torch.cuda.Event(enable_timing=True)
                    s0.record()
                    _lib.check(lib.bak_block_sweep(dm.code, 0, dm.ptr, obs, nv, dm.ldx, _ptr(norms), thr, _ptr(e),
                                                   _ptr(a), sweeps, -1.0, float("inf"), _ptr(hist), _ptr(st),
                                                   ws.ptr, ws.nbytes, _stream_ptr(torch, dev)), "sweep")
                    s1.record()
                    torch.cuda.synchronize()
                    best = min(best, s0.elapsed_time(s1))
                us = best * 1e3 / sweeps
                nb = -(-nv // thr)
                rows.append((nb, nv, us))
                print(f"{dt} obs={obs} vars={nv} thr={thr} variant={int(st[3])} err={int(st[2])} "
                      f"us/sweep={us:.1f} ns/col={us * 1e3 / nv:.0f}", flush=True)
        A = np.array([[nb, nv, 1] for nb, nv, _ in rows], float)
        t = np.array([u for *_, u in rows])
        c, *_ = np.linalg.lstsq(A, t, rcond=None)
        print(f"  fit {dt} obs={obs}: c_block={c[0]:.2f} us, c_col={c[1] * 1e3:.1f} ns, c_sweep={c[2]:.1f} us",
              flush=True)

"""Time bak_score_columns (one fused pass: X^T e, closed form, argmin) on a
C3-like tall shape and a wide shape; prints effective x-GB/s."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_12570_b200 as pb  # noqa: E402
from paper_2104_12570_b200 import _lib  # noqa: E402
from paper_2104_12570_b200.bak import _ptr, _stream_ptr  # noqa: E402

lib = _lib.load()
dev = torch.device("cuda", 0)
for obs, nv, dt in ((1 << 22, 256, torch.float64), (1000, 100000, torch.float32)):
    x = torch.randn(nv, obs, dtype=dt, device=dev)
    e = torch.randn(obs, dtype=dt, device=dev)
    dm = pb.DeviceMatrix(x, obs, nv, np.float64 if dt == torch.float64 else np.float32)
    norms = pb.colnorms(dm)
    scores = torch.empty(nv, dtype=torch.float64, device=dev)
    best = torch.zeros(2, dtype=torch.int64, device=dev)
    ws = torch.empty(lib.bak_score_columns_workspace(dm.code, obs, nv), dtype=torch.uint8, device=dev)
    st = _stream_ptr(torch, dev)

    def run():
        _lib.check(lib.bak_score_columns(dm.code, dm.ptr, obs, nv, dm.ldx, _ptr(e), _ptr(norms), None,
                                         _ptr(scores), _ptr(best), _ptr(ws), ws.numel(), st), "score")
    run()
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    for _ in range(5):
        run()
    t1.record()
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1) / 5
    gb = obs * nv * x.element_size() / 1e9
    print(f"score {obs}x{nv} {dt}: {ms:.3f} ms, x {gb:.2f} GB -> {gb / ms * 1e3:.0f} GB/s, best={int(best[0])}",
          flush=True)
    del x

"""A/B of the fp64 G kernel: TMA-fed vs cp.async panels (TMAS="0 1" -> BAK_GRAM_G_TMA) and the advisory
lock step (PACES -> BAK_GRAM_PACE=0|1) on C3's
shape: median kernel time of bak_gram_matrix_dot and a G checksum (the result
must not depend on the pacing).  Tuning aid, not a bench line."""
import ctypes
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2104_12570_b200 import _lib  # noqa: E402

lib = _lib.load()
dev = torch.device("cuda", 0)
obs, nv = int(os.environ.get("OBS", 1 << 24)), int(os.environ.get("VARS", 256))
reps = int(os.environ.get("REPS", 7))
code = _lib.F64
torch.manual_seed(5)
x = torch.randn(nv, obs, dtype=torch.float64, device=dev)
e = torch.randn(obs, dtype=torch.float64, device=dev)
st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
ref = None
runs = [(t, q) for t in os.environ.get("TMAS", "1").split() for q in os.environ.get("PACES", "0 1 0 1").split()]
for tma, pace in runs:
    os.environ["BAK_GRAM_PACE"] = pace
    os.environ["BAK_GRAM_G_TMA"] = tma  # 1: TMA-fed fp64 G kernel (default), 0: cp.async kernel
    # BAK_GRAM_UNITS (0: one unit per CTA, default: two) is read from the caller's environment
    G = torch.zeros(nv, nv, dtype=torch.float64, device=dev)
    g0 = torch.zeros(1024, nv, dtype=torch.float64, device=dev)
    wsb = lib.bak_gram_matrix_workspace(code, obs, nv)
    ws = torch.empty(wsb, dtype=torch.uint8, device=dev)

    def run():
        _lib.check(lib.bak_gram_matrix_dot(code, ctypes.c_void_p(x.data_ptr()), obs, nv, obs,
                                           ctypes.c_void_p(G.data_ptr()), ctypes.c_void_p(e.data_ptr()),
                                           ctypes.c_void_p(g0.data_ptr()), ctypes.c_void_p(ws.data_ptr()), wsb, st), "G")
    run()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        run()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    if ref is None:
        ref = G.clone()
    g0sum = g0.sum(0)
    if ref is not None and "g0ref" not in globals():
        pass
    print(json.dumps({"tma": tma, "pace": pace, "obs": obs, "vars": nv, "ms_median": sorted(ts)[len(ts) // 2], "ms": [round(t, 3) for t in ts],
                      "bit_identical_to_first": bool(torch.equal(G, ref)), "g0_checksum": float(g0sum.abs().sum())}), flush=True)

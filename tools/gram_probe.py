"""Time the G = X^T X kernel (bak_gram_matrix / bak_gram_matrix_dot) on C3's shape
under the split modes (BAK_GRAM_BALANCE=0: equal chunks; default: diagonal
blocks get 4/3 the rows).  Tuning aid, not a bench line."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2104_12570_b200 import _lib  # noqa: E402

lib = _lib.load()
dev = torch.device("cuda", 0)
obs, nv = 1 << 24, int(os.environ.get("VARS", 256))
for dt, code in ((torch.float64, 0), (torch.float32, 1)):
    code = _lib.F64 if dt == torch.float64 else _lib.F32
    x = torch.randn(nv, obs, dtype=dt, device=dev)
    e = torch.randn(obs, dtype=dt, device=dev)
    G = torch.empty(nv, nv, dtype=torch.float64, device=dev)
    g0 = torch.empty(512, nv, dtype=torch.float64, device=dev)
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    for bal, occ in (("0", "2"), ("1", "2"), ("0", "3"), ("1", "3")):
        os.environ["BAK_GRAM_BALANCE"] = bal
        os.environ["BAK_GRAM_OCC"] = occ
        wsb = lib.bak_gram_matrix_workspace(code, obs, nv)
        ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
        for dot in (0, 1):
            def run():
                if dot:
                    _lib.check(lib.bak_gram_matrix_dot(code, ctypes.c_void_p(x.data_ptr()), obs, nv, obs,
                                                       ctypes.c_void_p(G.data_ptr()), ctypes.c_void_p(e.data_ptr()),
                                                       ctypes.c_void_p(g0.data_ptr()), ctypes.c_void_p(ws.data_ptr()),
                                                       wsb, st), "dot")
                else:
                    _lib.check(lib.bak_gram_matrix(code, ctypes.c_void_p(x.data_ptr()), obs, nv, obs,
                                                   ctypes.c_void_p(G.data_ptr()), ctypes.c_void_p(ws.data_ptr()),
                                                   wsb, st), "G")
            run()
            torch.cuda.synchronize()
            ts = []
            for _ in range(5):
                a = torch.cuda.Event(enable_timing=True)
                b = torch.cuda.Event(enable_timing=True)
                a.record()
                run()
                b.record()
                torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
            ms = sorted(ts)[2]
            print(f"{dt} balance={bal} occ={occ} dot={dot}: {ms:.2f} ms  ({2 * nv * nv * obs / ms / 1e9:.1f} TF full-SYRK equiv,"
                  f" rows d/o={lib.bak_gram_dot_rows(code, obs, nv)})", flush=True)
    del x, e

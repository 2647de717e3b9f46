"""Where the C3 GRAM solve's time goes outside the kernels: whole solve_bak
vs the bare bak_solve_gram call on preallocated buffers (CUDA events)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2104_12570_b200 as pb  # noqa: E402
from paper_2104_12570_b200 import _lib  # noqa: E402
from paper_2104_12570_b200.bak import _ptr, _stream_ptr, _Workspace, _workspace_bytes  # noqa: E402

dev = torch.device("cuda", 0)
cfg = dict(bench.CONFIGS["c3"])
dm, y = bench.make_inputs(cfg, dev, seed=1)
lib = _lib.load()
sc = pb.SolveConfig(max_iter=20, tol=0)


def ev_time(fn, n=3):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n, (time.perf_counter() - t0) * 1e3 / n


print("solve_bak(gram) ms (events, wall):", ev_time(lambda: pb.solve_bak(dm, y, sc, variant="gram",
                                                                       return_device=True)))
code, obs, nv = dm.code, dm.obs, dm.vars
ws = _Workspace(torch, dev, _workspace_bytes(lib, code, obs, nv, 5))
e = torch.empty_like(y)
a = torch.zeros(nv, dtype=y.dtype, device=dev)
norms = torch.empty(nv, dtype=y.dtype, device=dev)
status = torch.zeros(4, dtype=torch.int64, device=dev)
resid = torch.empty_like(y)
st = _stream_ptr(torch, dev)


def bare():
    e.copy_(y)
    a.zero_()
    _lib.check(lib.bak_solve_gram(code, dm.ptr, obs, nv, dm.ldx, _ptr(y), None, nv, 0, _ptr(norms), _ptr(e), _ptr(a),
                                  20, -1.0, None, _ptr(status), _ptr(resid), ws.ptr, ws.nbytes, st), "gram")


print("bare bak_solve_gram ms (events, wall):", ev_time(bare))
G = torch.empty((nv, nv), dtype=torch.float64, device=dev)
gws = _Workspace(torch, dev, lib.bak_gram_matrix_workspace(code, obs, nv))
print("G alone ms:", ev_time(lambda: lib.bak_gram_matrix(code, dm.ptr, obs, nv, dm.ldx, _ptr(G), gws.ptr,
                                                          gws.nbytes, st)))

"""G = X^T X on tcgen05 (fp32 inputs): accuracy vs the fp32 TMEM accumulation
length (BAK_GRAM_TC_CHUNK) and device time, against an fp64 product of the
same fp32 data and the legacy mma.sync 3xTF32 kernel (BAK_GRAM_G=x3).

    python tools/gram_tc_probe.py [obs] [vars]
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_12570_b200 as pb  # noqa: E402
from paper_2104_12570_b200 import _lib  # noqa: E402
from paper_2104_12570_b200.bak import _Workspace, _stream_ptr  # noqa: E402

obs = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 22
nv = int(sys.argv[2]) if len(sys.argv) > 2 else 256
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(5)
x = torch.randn((nv, obs), generator=g, device=dev, dtype=torch.float32)  # column-major (vars, obs)
dm = pb.DeviceMatrix(x, obs, nv, np.float32)
xd = x.double()
ref = xd @ xd.T
lib = _lib.load()
st = _stream_ptr(torch, dev)


def run(env):
    for k in ("BAK_GRAM_TC_CHUNK", "BAK_GRAM_G"):
        os.environ.pop(k, None)
    os.environ.update(env)
    G = torch.empty((nv, nv), dtype=torch.float64, device=dev)
    ws = _Workspace(torch, dev, lib.bak_gram_matrix_workspace(dm.code, obs, nv))
    f = lambda: _lib.check(lib.bak_gram_matrix(dm.code, dm.ptr, obs, nv, dm.ldx, G.data_ptr(), ws.ptr, ws.nbytes,
                                               st), "bak_gram_matrix")
    f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        f()
    e1.record()
    torch.cuda.synchronize()
    err = float(torch.linalg.norm(G - ref) / torch.linalg.norm(ref))
    derr = float(((G.diagonal() - ref.diagonal()).abs() / ref.diagonal()).max())
    return dict(env=env, ms=e0.elapsed_time(e1) / 5, rel_err=err, diag_err=derr)


out = []
for c in ("128", "256", "512", "1024", "2048", "4096", "16384"):
    out.append(run({"BAK_GRAM_TC_CHUNK": c}))
out.append(run({"BAK_GRAM_G": "x3"}))
for o in out:
    print(json.dumps(o))

"""Cycle breakdown of the on-chip blocked kernel (needs BAK_PHASES=1 build):
consumer tid 0: pass-1 waits, pass-1 work, block reduce/exchange, pass 2,
sweep end; producer: empty waits, issue work.  Per column."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2104_12570_b200 as pb
from paper_2104_12570_b200 import _lib
from paper_2104_12570_b200.bak import _Workspace, _ptr, _stream_ptr, _workspace_bytes
obs, nv, thr, dt = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
variant = sys.argv[5] if len(sys.argv) > 5 else "auto"
dev = torch.device("cuda", 0)
tdt = torch.float64 if dt == "f64" else torch.float32
vec = 2 if dt == "f64" else 4
ld = (obs + vec - 1) // vec * vec
data = torch.randn((nv, ld), dtype=tdt, device=dev)
y = torch.randn(obs, dtype=tdt, device=dev)
dm = pb.DeviceMatrix(data, obs, nv, "float64" if dt == "f64" else "float32")
lib = _lib.load()
ws = _Workspace(torch, dev, _workspace_bytes(lib, dm.code, obs, nv))
norms = pb.colnorms(dm, ws)
e = y.clone(); a = torch.zeros(nv, dtype=tdt, device=dev); st = torch.zeros(4, dtype=torch.int64, device=dev)
sweeps = 4
hist = torch.zeros(sweeps + 8, dtype=torch.float64, device=dev)
_lib.check(lib.bak_block_sweep(dm.code, _lib.VARIANTS[variant], dm.ptr, obs, nv, dm.ldx, _ptr(norms), thr, _ptr(e),
                               _ptr(a), sweeps, -1.0, float("inf"), _ptr(hist), _ptr(st), ws.ptr, ws.nbytes,
                               _stream_ptr(torch, dev)), "bak_block_sweep")
torch.cuda.synchronize()
ph = hist[sweeps:].cpu().numpy() / (sweeps * nv)
names = ["p1_wait", "p1_work", "reduce_xchg", "pass2", "sweep_end", "prod_wait", "prod_issue"]
print(obs, nv, thr, dt, "variant", int(st[3]), {n: round(float(v), 1) for n, v in zip(names, ph)},
      "consumer total", round(float(ph[:5].sum()), 1), flush=True)

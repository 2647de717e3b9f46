"""Per-phase cycle breakdown of the sweep loop (needs a -DBAK_PHASES build)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2104_12570_b200 as pb
from paper_2104_12570_b200 import _lib
from paper_2104_12570_b200.bak import _Workspace, _ptr, _stream_ptr, _workspace_bytes
obs, nv, variant, dt = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else "f64"
dev = torch.device("cuda", 0)
tdt = torch.float64 if dt == "f64" else torch.float32
vec = 2 if dt == "f64" else 4
ld = (obs + vec - 1) // vec * vec
data = torch.randn((nv, ld), dtype=tdt, device=dev)
y = torch.randn(obs, dtype=tdt, device=dev)
dm = pb.DeviceMatrix(data, obs, nv, "float64" if dt == "f64" else "float32")
lib = _lib.load()
ws = _Workspace(torch, dev, _workspace_bytes(lib, dm.code, obs, nv, _lib.VARIANTS[variant]))
norms = pb.colnorms(dm, ws)
e = y.clone(); a = torch.zeros(nv, dtype=tdt, device=dev); st = torch.zeros(4, dtype=torch.int64, device=dev)
sweeps = 2
hist = torch.zeros(sweeps + 8, dtype=torch.float64, device=dev)
_lib.check(lib.bak_sweep(dm.code, _lib.VARIANTS[variant], dm.ptr, obs, nv, dm.ldx, _ptr(norms), None, nv, 0, _ptr(e),
                         _ptr(a), sweeps, -1.0, _ptr(hist), _ptr(st), ws.ptr, ws.nbytes, _stream_ptr(torch, dev)),
           "bak_sweep")
torch.cuda.synchronize()
ph = hist[sweeps:].cpu().numpy() / (sweeps * nv)
names = ["div", "fused", "pull", "warp_sum", "bar", "partials", "reduce_rest", "loop_tail"]
if variant == "bgram":  # per block: pass 1, bar, sum+exchange, M wait+bar, matvec+bar, pass 2
    names = ["pass1", "bar1", "exchange", "m_wait", "matvec", "pass2", "-", "-"]
    ph = hist[sweeps:].cpu().numpy() / (sweeps * ((nv + 63) // 64))
print(variant, obs, nv, dt, {n: round(float(v), 1) for n, v in zip(names, ph)}, "total", round(float(ph.sum()), 1))

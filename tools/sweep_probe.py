"""Time bak_sweep alone for shapes/variants/plans (tuning aid, not a test).

    python tools/sweep_probe.py --obs 1000 --vars 20000 --dtype f64 --sweeps 2 \
        --variant cta --plans "1,4,256 1,8,128"
Prints ns per column step for each plan (BAK_PLAN=parts,e,nthreads).
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_2104_12570_b200 as pb  # noqa: E402
from paper_2104_12570_b200 import _lib  # noqa: E402
from paper_2104_12570_b200.bak import _Workspace, _ptr, _stream_ptr, _workspace_bytes  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--obs", type=int, required=True)
    ap.add_argument("--vars", type=int, required=True)
    ap.add_argument("--dtype", default="f64")
    ap.add_argument("--sweeps", type=int, default=2)
    ap.add_argument("--variant", default="auto")
    ap.add_argument("--plans", default="")
    ap.add_argument("--reps", type=int, default=3)
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    tdt = torch.float64 if a.dtype == "f64" else torch.float32
    vec = 2 if a.dtype == "f64" else 4
    ld = (a.obs + vec - 1) // vec * vec
    data = torch.randn((a.vars, ld), dtype=tdt, device=dev)
    y = torch.randn(a.obs, dtype=tdt, device=dev)
    dm = pb.DeviceMatrix(data, a.obs, a.vars, "float64" if a.dtype == "f64" else "float32")
    lib = _lib.load()
    ws = _Workspace(torch, dev, _workspace_bytes(lib, dm.code, a.obs, a.vars, _lib.VARIANTS[a.variant]))
    norms = pb.colnorms(dm, ws)
    e = torch.empty_like(y)
    av = torch.zeros(a.vars, dtype=tdt, device=dev)
    st = torch.zeros(4, dtype=torch.int64, device=dev)
    out = []
    for plan in (a.plans.split() or [""]):
        if plan:
            os.environ["BAK_PLAN"] = plan
        else:
            os.environ.pop("BAK_PLAN", None)
        best = None
        for _ in range(a.reps):
            e.copy_(y)
            av.zero_()
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record()
            rc = lib.bak_sweep(dm.code, _lib.VARIANTS[a.variant], dm.ptr, a.obs, a.vars, dm.ldx, _ptr(norms), None,
                               a.vars, 0, _ptr(e), _ptr(av), a.sweeps, -1.0, None, _ptr(st), ws.ptr, ws.nbytes,
                               _stream_ptr(torch, dev))
            ev1.record()
            torch.cuda.synchronize()
            if rc != 0:
                best = f"rc={rc} {lib.bak_last_error().decode()}"
                break
            ms = ev0.elapsed_time(ev1)
            best = ms if best is None else min(best, ms)
        if isinstance(best, float):
            ns = best * 1e6 / (a.sweeps * a.vars)
            gbs = a.obs * a.vars * (8 if a.dtype == "f64" else 4) * a.sweeps / (best / 1e3) / 1e9
            rec = {"plan": plan or "auto", "ms": round(best, 3), "ns_per_col": round(ns, 1), "x_gbs": round(gbs, 1),
                   "variant": _lib.VARIANT_NAMES.get(int(st[3].item())), "err": int(st[2].item())}
        else:
            rec = {"plan": plan, "error": best}
        out.append(rec)
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()

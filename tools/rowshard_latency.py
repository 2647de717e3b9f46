"""Per-column cost of the exact row-sharded sweep (bak_sweep_rowshard) with
N ranks emulated in one cooperative launch on one GPU (N groups of CTAs, each
rank's partial dot posted into every rank's mailbox and summed in rank order).
Small rows per rank isolate the exchange latency (the part that NVLink would
lengthen between GPUs); large rows show the HBM-bound regime.  Tuning /
reporting aid, prints one JSON line per (rows, N)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2104_12570_b200 as pb  # noqa: E402
from paper_2104_12570_b200.sharded import Mailboxes, sweep_rowshard  # noqa: E402

dev = torch.device("cuda", 0)
nv, sweeps = 64, 4
for rows_per_rank in (4096, 65536, 1 << 20):
    for n in (1, 2, 4, 8):
        obs = rows_per_rank * n
        x = torch.randn(nv, obs, dtype=torch.float64, device=dev)
        dm = pb.DeviceMatrix(x, obs, nv, np.float64)
        norms = pb.colnorms(dm)
        y = torch.randn(obs, dtype=torch.float64, device=dev)
        mb = Mailboxes(n)
        best = None
        for _ in range(3):
            e = y.clone()
            a = torch.zeros(n * nv, dtype=torch.float64, device=dev)
            t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0.record()
            st = sweep_rowshard(dm, e, a, norms, sweeps, -1.0, mb, 0, n, nranks_local=n)
            t1.record()
            torch.cuda.synchronize()
            ms = t0.elapsed_time(t1)
            best = ms if best is None else min(best, ms)
        us_col = best * 1e3 / (sweeps * nv)
        xbytes = obs * 8
        print(json.dumps({"rows_per_rank": rows_per_rank, "ranks": n, "us_per_column": round(us_col, 2),
                          "x_gbs": round(xbytes / (us_col * 1e-6) / 1e9, 1),
                          "err": int(st.view(n, 4)[:, 2].max().item())}), flush=True)
        del x, dm

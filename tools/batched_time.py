"""Time the C5 batched solve (65,536 x 512x32 fp32, 200 sweeps) for the plan in
the environment (BAK_BATCH_PLAN / BAK_BATCH_NOSMEM); tuning aid."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2104_12570_b200 as pb  # noqa: E402

nsys = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
sweeps = int(sys.argv[2]) if len(sys.argv) > 2 else 200
cfg = dict(bench.CONFIGS["c5"], nsys=nsys)
dev = torch.device("cuda", 0)
db, y = bench.make_inputs(cfg, dev)
sc = pb.SolveConfig(max_iter=sweeps, tol=0)
pb.solve_bak_batched(db, y, sc, return_device=True)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
rep = pb.solve_bak_batched(db, y, sc, return_device=True)
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b)
print(f"plan={os.environ.get('BAK_BATCH_PLAN', 'auto')} nosmem={os.environ.get('BAK_BATCH_NOSMEM', '0')} "
      f"{ms:.1f} ms  {sweeps / ms * 1e3:.1f} batch-sweeps/s", flush=True)

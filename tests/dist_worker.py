"""Worker for tests/test_dist_nccl_gpu.py: one rank per GPU over NCCL
(launched by torch.distributed.run), row-sharded solves through DistComm,
checked against the CPU oracle by rank 0.  Not collected by pytest."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import bak_oracle as orc  # noqa: E402
import paper_2104_12570_b200 as pb  # noqa: E402
from paper_2104_12570_b200.sharded import DistComm, partition_rows, solve_bak_rowsharded  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
torch.cuda.set_device(dev)
torch.distributed.init_process_group("nccl", device_id=dev)
comm = DistComm()
x, y, _ = orc.make_system(200_000, 24, 31, "normal", "uniform", 0.01, "double")
r0, r1 = partition_rows(x.shape[0], world, rank, align=4)
out = {}
for variant in ("gram", "stream"):
    cfg = pb.SolveConfig(max_iter=5, tol=0, record_history=True)
    rep = solve_bak_rowsharded([np.asfortranarray(x[r0:r1])], [y[r0:r1]], cfg, comm, variant=variant)[0]
    ref = orc.solve(x, y, max_iter=5, tol=0)
    out[variant] = dict(err=orc.rel_coeff_err(rep.a_hat, ref["a_hat"]), sweeps=rep.sweeps_run, label=rep.variant)
# C5-style system sharding: no communication on the data path, one gather at the end
from paper_2104_12570_b200.sharded import solve_bak_batched_sharded  # noqa: E402
nsys = 24
xs = np.stack([orc.config_c5_system(k, obs=128, nvars=16)[0] for k in range(nsys)])
ys = np.stack([orc.config_c5_system(k, obs=128, nvars=16)[1] for k in range(nsys)])
s0, s1, brep = solve_bak_batched_sharded(xs, ys, pb.SolveConfig(max_iter=40, tol=0), comm, gather=True)
errs = [orc.rel_coeff_err(brep.a_hat[k], orc.solve(xs[k], ys[k], max_iter=40, tol=0)["a_hat"]) for k in range(nsys)]
out["batched"] = dict(nsys=int(brep.a_hat.shape[0]), err=max(errs), sweeps=int(brep.sweeps_run.min()))
torch.distributed.barrier()
torch.distributed.destroy_process_group()
if rank == 0:
    print("RESULT " + json.dumps(out), flush=True)

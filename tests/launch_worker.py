"""Worker for tests/test_sharded_gloo.py::test_launcher_spawns_ranks: started
as ONE process with --gpus N, it re-launches itself as N ranks through
paper_2104_12570_b200.launch (the same path as bench.py --gpus N), the ranks
all-gather their rank ids over gloo and rank 0 prints one JSON line.
Not collected by pytest."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2104_12570_b200 import launch  # noqa: E402
from paper_2104_12570_b200.sharded import DistComm, partition_systems  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--gpus", type=int, default=1)
args = ap.parse_args()
rc = launch.relaunch_if_needed(args.gpus, os.path.abspath(__file__), sys.argv[1:])
if rc is not None:
    sys.exit(rc)

import torch  # noqa: E402

torch.distributed.init_process_group("gloo")
comm = DistComm()
got = comm.all_gather([torch.tensor([comm.rank], dtype=torch.int64)])
s0, s1 = partition_systems(65536, comm.world, comm.rank)
spans = comm.all_gather([torch.tensor([s0, s1], dtype=torch.int64)])
comm.barrier()
if comm.rank == 0:
    print(json.dumps({"world": comm.world, "ranks": [int(g.item()) for g in got],
                      "spans": [t.tolist() for t in spans],
                      "env_addr": os.environ.get("MASTER_ADDR")}), flush=True)
torch.distributed.destroy_process_group()

"""Run the batched solve once on C5-shaped inputs (profiling target)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2104_12570_b200 as pb
nsys = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
sweeps = int(sys.argv[2]) if len(sys.argv) > 2 else 200
cfg = dict(bench.CONFIGS["c5"], nsys=nsys)
dev = torch.device("cuda", 0)
db, y = bench.make_inputs(cfg, dev)
rep = pb.solve_bak_batched(db, y, pb.SolveConfig(max_iter=sweeps, tol=0), return_device=True)
torch.cuda.synchronize()
print("ok", int(rep.sweeps_run.max()))

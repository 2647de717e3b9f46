import sys, numpy as np
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import golden_io, paper_2104_12570_b200 as pb
g = golden_io.load_bakp("bakp_thr7_2000x40_f64")
x, y = g["x"], g["y"]
cfg = pb.BlockConfig(base=pb.SolveConfig(**g["config"]), thr=g["thr"])
for v in sys.argv[1:]:
    try:
        r = pb.solve_bakp(x, y, cfg, variant=v)
        print(v, r.variant, r.sweeps_run, np.linalg.norm(r.a_hat - g["a_hat"]) / np.linalg.norm(g["a_hat"]), flush=True)
    except Exception as e:
        print(v, "ERR", repr(e)[:300], flush=True)

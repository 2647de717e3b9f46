"""Small invocations of every kernel family, for compute-sanitizer.

    compute-sanitizer --tool memcheck|racecheck|synccheck --error-exitcode 17 \
        python tools/sanitize_cases.py [family ...]

One tool per gpurun call (B200_PROFILING.md: several tools in one call have
left GPUs unusable).  Shapes are tiny so the instrumented run takes seconds;
each case is also checked against the CPU oracle, so a sanitizer-clean run is
a correct one.  tests/test_sanitizer_gpu.py wraps this (opt-in: it runs only
with BAK_SANITIZER_TOOL set, never in the default -m gpu suite).
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import bak_oracle as orc  # noqa: E402
import paper_2104_12570_b200 as pb  # noqa: E402

TOL = {np.dtype(np.float64): 1e-10, np.dtype(np.float32): 1e-4}


def check(name, a, ref_a, x):
    err = orc.rel_coeff_err(a, ref_a)
    assert err <= TOL[np.dtype(x.dtype)], (name, err)
    print(f"{name}: ok ({err:.1e})", flush=True)


def sweep():
    for variant, obs, nv in (("cta", 300, 9), ("cluster", 3000, 12), ("grid", 70_000, 6), ("stream", 20_000, 5)):
        for prec in ("double", "single"):
            x, y, _ = orc.config_c3(obs=obs, nvars=nv, precision=prec)
            ref = orc.solve(x, y, max_iter=3, tol=0)
            rep = pb.solve_bak(x, y, pb.SolveConfig(max_iter=3, tol=0), variant=variant)
            check(f"sweep/{variant}/{prec}", rep.a_hat, ref["a_hat"], x)


def batched():
    xs = np.stack([orc.config_c5_system(s, obs=64, nvars=8)[0] for s in range(5)])
    ys = np.stack([orc.config_c5_system(s, obs=64, nvars=8)[1] for s in range(5)])
    br = pb.solve_bak_batched(xs, ys, pb.SolveConfig(max_iter=10, tol=0))
    for s in range(5):
        check(f"batched/{s}", br.a_hat[s], orc.solve(xs[s], ys[s], max_iter=10, tol=0)["a_hat"], xs[s])


def block():
    x, y, _ = orc.config_c1(obs=500, nvars=20)
    for variant in ("auto", "stream", "gram"):
        rb = pb.solve_bakp(x, y, pb.BlockConfig(base=pb.SolveConfig(max_iter=4, tol=0), thr=6), variant=variant)
        check(f"bakp/{variant}", rb.a_hat, orc.solve_bakp(x, y, max_iter=4, tol=0, thr=6)["a_hat"], x)


def gram():
    for prec, obs, nv in (("double", 5000, 40), ("single", 5000, 40), ("single", 4000, 200)):
        x, y, _ = orc.config_c3(obs=obs, nvars=nv, precision=prec)
        rep = pb.solve_bak(x, y, pb.SolveConfig(max_iter=3, tol=0), variant="gram")
        check(f"gram/{prec}/{nv}", rep.a_hat, orc.solve(x, y, max_iter=3, tol=0)["a_hat"], x)


def rowshard():
    import torch
    from paper_2104_12570_b200.sharded import Mailboxes, sweep_rowshard
    x, y, _ = orc.config_c3(obs=6000, nvars=6, precision="double")
    ref = orc.solve(x, y, max_iter=2, tol=0)
    dm = pb.to_device_matrix(x)
    norms = pb.colnorms(dm)
    dev = dm.data.device
    for n in (2, 3):
        e = torch.from_numpy(np.ascontiguousarray(y)).to(dev)
        a = torch.zeros(n * 6, dtype=torch.float64, device=dev)
        st = sweep_rowshard(dm, e, a, norms, 2, -1.0, Mailboxes(n), 0, n, nranks_local=n)
        assert int(st.cpu().numpy().reshape(n, 4)[:, 2].max()) == 0
        check(f"rowshard/{n}", a.cpu().numpy()[:6], ref["a_hat"], x)


def score():
    x, y, _ = orc.config_c1(obs=400, nvars=30)
    e = np.asarray(y, np.float64)
    best, _ = pb.score_all_columns(x, e)
    assert best == orc.score_all_columns(x, e)[0]
    print("score: ok", flush=True)


FAMILIES = {"sweep": sweep, "batched": batched, "block": block, "gram": gram, "rowshard": rowshard,
            "score": score}

if __name__ == "__main__":
    for name in sys.argv[1:] or list(FAMILIES):
        FAMILIES[name]()
    print("sanitize cases done", flush=True)

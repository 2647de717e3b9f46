"""Seeded randomized shapes through every kernel family against the oracle:
ragged row counts (not multiples of the vector width, the cluster or the CTA
row block), odd column counts, both precisions, early break on/off, zero
columns.  Catches planner / tail-handling edge cases the fixed-shape tests
miss."""

import numpy as np
import pytest

from oracle import bak_oracle as orc

pytestmark = pytest.mark.gpu

TOL = {np.dtype(np.float64): 1e-10, np.dtype(np.float32): 1e-4}


def _case(seed):
    rng = np.random.default_rng(10_000 + seed)
    dtype = np.float64 if seed % 3 else np.float32
    obs = int(rng.choice([1, 2, 3, 7, 31, 33, 257, 1023, 1025, 2049, 4097, 9999, 33_333, 70_001]))
    nv = int(rng.integers(1, 48))
    x = np.asfortranarray(rng.standard_normal((obs, nv)).astype(dtype))
    if nv > 2 and seed % 4 == 0:
        x[:, int(rng.integers(nv))] = 0.0
    if not np.any(x):
        x[0, 0] = 1.0
    y = (x @ rng.uniform(-1, 1, nv).astype(dtype) + 0.1 * rng.standard_normal(obs)).astype(dtype)
    tol = float(rng.choice([0.0, 1e-3, 1e-6]))
    return x, y, tol, rng


@pytest.mark.parametrize("seed", range(48))
def test_fuzz_sweep_variants(seed):
    import paper_2104_12570_b200 as pb
    x, y, tol, rng = _case(seed)
    obs, nv = x.shape
    cfg = dict(max_iter=6, tol=tol, record_history=True)
    ref = orc.solve(x, y, **cfg)
    variants = ["auto", "stream"]
    if obs <= 4096:
        variants.append("cluster" if obs > 256 else "cta")
    if obs > 32768:
        variants.append("grid")
    if nv <= 256:
        variants.append("gram")
    for v in variants:
        try:
            rep = pb.solve_bak(x, y, pb.SolveConfig(**cfg), variant=v)
        except pb.bak._lib.BakError as err:
            if "does not fit" in str(err) or "unsupported" in str(err).lower():
                continue
            raise
        assert rep.sweeps_run == ref["sweeps_run"], (v, obs, nv)
        assert rep.converged == ref["converged"], (v, obs, nv)
        assert orc.rel_coeff_err(rep.a_hat, ref["a_hat"]) <= TOL[x.dtype], (v, obs, nv)


@pytest.mark.parametrize("seed", range(24))
def test_fuzz_blocked_and_batched(seed):
    import paper_2104_12570_b200 as pb
    x, y, tol, rng = _case(100 + seed)
    obs, nv = x.shape
    thr = int(rng.integers(1, nv + 1))
    try:
        ref = orc.solve_bakp(x, y, max_iter=5, tol=tol, thr=thr)
    except orc.DivergenceError:
        with pytest.raises(pb.DivergenceError):
            pb.solve_bakp(x, y, pb.BlockConfig(base=pb.SolveConfig(max_iter=5, tol=tol), thr=thr))
        return
    for v in ("auto", "stream") + (("gram",) if nv <= 256 else ()):
        rep = pb.solve_bakp(x, y, pb.BlockConfig(base=pb.SolveConfig(max_iter=5, tol=tol), thr=thr), variant=v)
        assert rep.sweeps_run == ref["sweeps_run"], (v, obs, nv, thr)
        assert orc.rel_coeff_err(rep.a_hat, ref["a_hat"]) <= TOL[x.dtype], (v, obs, nv, thr)
    if obs <= 2048:
        ns = int(rng.integers(1, 9))
        xs = np.stack([x] * ns)
        ys = np.stack([y] * ns)
        br = pb.solve_bak_batched(xs, ys, pb.SolveConfig(max_iter=5, tol=tol))
        r = orc.solve(x, y, max_iter=5, tol=tol)
        for s in range(ns):
            assert br.sweeps_run[s] == r["sweeps_run"]
            assert orc.rel_coeff_err(br.a_hat[s], r["a_hat"]) <= TOL[x.dtype]


@pytest.mark.parametrize("seed", range(24))
def test_fuzz_scoring_random_order_warm_start(seed):
    import paper_2104_12570_b200 as pb
    x, y, tol, rng = _case(300 + seed)
    obs, nv = x.shape
    # column scoring (select.py:56-85), random exclusions
    excl = sorted(set(rng.integers(0, nv, size=int(rng.integers(0, max(1, nv // 2)))).tolist()))
    try:
        b_ref, s_ref = orc.score_all_columns(x, y, excluded=excl)
    except orc.SelectionExhaustedError:
        with pytest.raises(pb.SelectionExhaustedError):
            pb.score_all_columns(x, y, excluded=excl)
    else:
        b, s = pb.score_all_columns(x, y, excluded=excl)
        fin = np.isfinite(s_ref)
        assert np.array_equal(np.isfinite(s), fin)
        e2 = float(np.dot(y.astype(np.float64), y.astype(np.float64)))
        t = 1e-10 if x.dtype == np.float64 else 1e-5
        assert np.max(np.abs(s[fin] - s_ref[fin])) <= t * max(e2, 1e-300)
        srt = np.sort(s_ref[fin])
        if srt.size < 2 or srt[1] - srt[0] > 100 * t * e2:
            assert b == b_ref
    # random ordering and warm start (bak.py:98-99, 173-175, 189)
    a0 = rng.uniform(-1, 1, nv).astype(x.dtype)
    cfg = dict(max_iter=5, tol=tol, ordering="random", ordering_seed=int(rng.integers(1 << 30)))
    ref = orc.solve(x, y, a0=a0, **cfg)
    rep = pb.solve_bak(x, y, pb.SolveConfig(**cfg), a0=a0)
    assert rep.sweeps_run == ref["sweeps_run"] and rep.converged == ref["converged"]
    assert orc.rel_coeff_err(rep.a_hat, ref["a_hat"]) <= TOL[x.dtype]


@pytest.mark.parametrize("seed", range(12))
def test_fuzz_rowsharded_emulated(seed):
    """Row sharding with N emulated ranks on one GPU: the GRAM path through
    LocalComm (ragged shards) and the exact in-kernel mailbox kernel."""
    import torch

    import paper_2104_12570_b200 as pb
    from paper_2104_12570_b200.sharded import (LocalComm, Mailboxes, partition_rows, solve_bak_rowsharded,
                                               sweep_rowshard)
    rng = np.random.default_rng(500 + seed)
    dtype = np.float64 if seed % 2 else np.float32
    obs = int(rng.integers(2000, 90_000))
    nv = int(rng.integers(1, 40))
    n = int(rng.choice([1, 2, 3, 4]))
    x = np.asfortranarray(rng.standard_normal((obs, nv)).astype(dtype))
    y = (x @ rng.uniform(-1, 1, nv).astype(dtype) + 0.05 * rng.standard_normal(obs)).astype(dtype)
    ref = orc.solve(x, y, max_iter=4, tol=0)
    tol = TOL[np.dtype(dtype)]
    shards = [partition_rows(obs, n, r, align=4) for r in range(n)]
    xs = [np.asfortranarray(x[a:b]) for a, b in shards if b > a]
    ys = [y[a:b] for a, b in shards if b > a]
    reps = solve_bak_rowsharded(xs, ys, pb.SolveConfig(max_iter=4, tol=0), LocalComm(len(xs)))
    for r in reps:
        assert r.sweeps_run == 4 and orc.rel_coeff_err(r.a_hat, ref["a_hat"]) <= tol
    # exact kernel, N ranks in one cooperative launch over the same rows
    dm = pb.to_device_matrix(x)
    norms = pb.colnorms(dm)
    dev = dm.data.device
    tdt = torch.float64 if dtype == np.float64 else torch.float32
    e = torch.from_numpy(np.ascontiguousarray(y)).to(dev)
    a = torch.zeros(n * nv, dtype=tdt, device=dev)
    st = sweep_rowshard(dm, e, a, norms, 4, -1.0, Mailboxes(n), 0, n, nranks_local=n)
    assert np.all(st.cpu().numpy().reshape(n, 4)[:, 2] == 0)
    A = a.cpu().numpy().reshape(n, nv)
    assert orc.rel_coeff_err(A[0], ref["a_hat"]) <= tol
    for r in range(1, n):
        assert A[r].tobytes() == A[0].tobytes()


@pytest.mark.parametrize("seed", range(24))
def test_fuzz_gram_multiblock(seed):
    """GRAM with several 64-column blocks (diagonal and off-diagonal G tiles,
    ragged last block), ragged rows, both precisions, warm start / early break."""
    import paper_2104_12570_b200 as pb
    rng = np.random.default_rng(20_000 + seed)
    dtype = np.float64 if seed % 2 else np.float32
    obs = int(rng.choice([65, 1000, 4097, 33_333, 70_001, 131_075]))
    nv = int(rng.integers(49, 300))
    obs = max(obs, nv + 1)
    x = np.asfortranarray(rng.standard_normal((obs, nv)).astype(dtype))
    if seed % 5 == 0:
        x[:, int(rng.integers(nv))] = 0.0
    y = (x @ rng.uniform(-1, 1, nv).astype(dtype) + 0.05 * rng.standard_normal(obs)).astype(dtype)
    tol = float(rng.choice([0.0, 1e-4]))
    a0 = rng.uniform(-0.1, 0.1, nv).astype(dtype) if seed % 3 == 0 else None
    cfg = dict(max_iter=5, tol=tol)
    ref = orc.solve(x, y, a0=a0, **cfg)
    rep = pb.solve_bak(x, y, pb.SolveConfig(**cfg), a0=a0, variant="gram")
    assert rep.sweeps_run == ref["sweeps_run"] and rep.converged == ref["converged"], (obs, nv)
    assert orc.rel_coeff_err(rep.a_hat, ref["a_hat"]) <= TOL[x.dtype], (obs, nv, dtype)

"""GPU parity: the sm_100a kernels (through the C ABI) against the reference's
own outputs (golden fixtures) and the CPU oracle on the same seeded inputs.

Tolerances (north_star / SURVEY §8c), written here once:
  coefficients   ||a - a_ref|| / ||a_ref||  <= 1e-10 (fp64), 1e-4 (fp32)
  residual norm  | r - r_ref | / r_ref      <= same tol, with r recomputed in
                 fp64 (bench.py:180-184); when the system is solved to the
                 rounding floor (r_ref < 1e-6 ||y||: consistent / converged
                 systems such as C2, C4) the difference is taken relative to
                 ||y||, since |r - r_ref| <= ||X|| ||a - a_ref|| ~ tol ||y||
  control flow   sweeps_run and converged identical
"""

import numpy as np
import pytest

import golden_io
from oracle import bak_oracle as orc

pytestmark = pytest.mark.gpu

TOL = {np.dtype(np.float64): 1e-10, np.dtype(np.float32): 1e-4}


def _pb():
    import paper_2104_12570_b200 as pb
    return pb


def assert_parity(x, y, rep, ref_a, ref_sweeps, ref_conv, ref_rnorm=None, ref_hist=None):
    tol = TOL[np.dtype(x.dtype)]
    assert rep.sweeps_run == ref_sweeps
    assert rep.converged == ref_conv
    err = orc.rel_coeff_err(rep.a_hat, ref_a)
    assert err <= tol, f"coeff rel err {err:.3e} > {tol}"
    r = orc.residual_norm_f64(x, y, rep.a_hat)
    if ref_rnorm is None:
        ref_rnorm = orc.residual_norm_f64(x, y, ref_a)
    ynorm = float(np.linalg.norm(np.asarray(y, np.float64)))
    den = ref_rnorm if ref_rnorm >= 1e-6 * ynorm else ynorm
    if den > 0:
        assert abs(r - ref_rnorm) / den <= tol, (r, ref_rnorm)
    # reported residual is the recomputed y - x a (bak.py:130)
    want = y - x @ rep.a_hat
    scale = np.abs(x).astype(np.float64) @ np.abs(rep.a_hat).astype(np.float64) + np.abs(y)
    assert np.all(np.abs(rep.residual - want) <= 64 * np.finfo(x.dtype).eps * (scale + 1e-300))
    if ref_hist is not None and rep.residual_norm_history is not None and len(ref_hist):
        assert len(rep.residual_norm_history) == len(ref_hist)
        h = np.asarray(rep.residual_norm_history)
        hr = np.asarray(ref_hist)
        big = hr > 1e-20 * max(hr[0], 1e-300)
        if big.any():
            rel = np.abs(h[big] - hr[big]) / hr[big]
            assert rel.max() <= max(1e3 * tol, 1e-6), rel.max()


@pytest.mark.parametrize("name", golden_io.names())
def test_golden_fixture(name):
    pb = _pb()
    g = golden_io.load(name)
    x, y = g["x"], g["y"]
    rep = pb.solve_bak(x, y, pb.SolveConfig(**g["config"]), a0=g["a0"])
    assert rep.drift_warning == bool(g["drift_warning"])
    assert_parity(x, y, rep, g["a_hat"], int(g["sweeps_run"]), bool(g["converged"]), float(g["resid_norm_f64"]),
                  g["history"] if bool(g["has_history"]) else None)


@pytest.mark.parametrize("variant", ["cta", "cluster", "grid", "stream"])
@pytest.mark.parametrize("precision", ["double", "single"])
def test_every_variant_matches_oracle(variant, precision):
    pb = _pb()
    obs = 2000 if variant in ("cta", "cluster") else 40_000
    x, y, _ = orc.make_system(obs, 24, 31, "normal", "uniform", 0.01, precision)
    ref = orc.solve(x, y, max_iter=12, tol=0, record_history=True)
    rep = pb.solve_bak(x, y, pb.SolveConfig(max_iter=12, tol=0, record_history=True), variant=variant)
    assert rep.variant == variant
    assert_parity(x, y, rep, ref["a_hat"], ref["sweeps_run"], ref["converged"], ref_hist=ref["residual_norm_history"])


@pytest.mark.parametrize("variant", ["cta", "cluster", "grid", "stream"])
def test_variants_ragged_rows_and_zero_columns(variant):
    pb = _pb()
    rng = np.random.default_rng(77)
    obs = 1037 if variant in ("cta", "cluster") else 20_001
    x = np.asfortranarray(rng.standard_normal((obs, 9)))
    x[:, 4] = 0.0
    y = rng.standard_normal(obs)
    a0 = np.zeros(9)
    a0[4] = 7.5
    ref = orc.solve(x, y, max_iter=30, tol=1e-9, a0=a0, record_history=True)
    rep = pb.solve_bak(x, y, pb.SolveConfig(max_iter=30, tol=1e-9, record_history=True), a0=a0, variant=variant)
    assert rep.a_hat[4] == 7.5
    assert_parity(x, y, rep, ref["a_hat"], ref["sweeps_run"], ref["converged"], ref_hist=ref["residual_norm_history"])


@pytest.mark.parametrize("variant", ["cta", "grid", "stream"])
def test_random_ordering_matches_oracle(variant):
    pb = _pb()
    obs = 600 if variant == "cta" else 30_000
    x, y, _ = orc.make_system(obs, 40, 5, "normal", "uniform", 0.1, "double")
    cfg = dict(max_iter=70, tol=1e-13, ordering="random", ordering_seed=9, record_history=True)
    ref = orc.solve(x, y, **cfg)
    rep = pb.solve_bak(x, y, pb.SolveConfig(**cfg), variant=variant)
    assert_parity(x, y, rep, ref["a_hat"], ref["sweeps_run"], ref["converged"], ref_hist=ref["residual_norm_history"])


def test_deterministic_bits():
    pb = _pb()
    x, y, _ = orc.make_system(50_000, 16, 2, "normal", "uniform", 0.01, "double")
    for variant in ("grid", "stream"):
        r1 = pb.solve_bak(x, y, pb.SolveConfig(max_iter=5, tol=0), variant=variant)
        r2 = pb.solve_bak(x, y, pb.SolveConfig(max_iter=5, tol=0), variant=variant)
        assert r1.a_hat.tobytes() == r2.a_hat.tobytes()
        assert r1.residual.tobytes() == r2.residual.tobytes()


def test_tall_stream_matches_oracle():
    """Past the on-chip capacity (XS plans hold 2.15M fp64 rows with the two-level
    exchange, 2.65M with the one-level one) with fewer than
    4 sweeps, "auto" runs the exact STREAM kernel (GRAM needs >= 4 sweeps to pay
    for G = X^T X)."""
    pb = _pb()
    x, y, _ = orc.config_c3(obs=2_700_000, nvars=32, precision="double")
    ref = orc.solve(x, y, max_iter=3, tol=0)
    rep = pb.solve_bak(x, y, pb.SolveConfig(max_iter=3, tol=0))
    assert rep.variant == "stream"
    assert_parity(x, y, rep, ref["a_hat"], ref["sweeps_run"], ref["converged"])


def test_reference_edge_cases():
    pb = _pb()
    # identity, one sweep, tol=0 (test_solver_bak.py:64-70)
    rep = pb.solve_bak(np.eye(3, order="F"), np.array([1.0, 2.0, 3.0]), pb.SolveConfig(max_iter=1, tol=0))
    np.testing.assert_array_equal(rep.a_hat, [1.0, 2.0, 3.0])
    np.testing.assert_array_equal(rep.residual, np.zeros(3))
    assert rep.sweeps_run == 1 and not rep.converged
    # zero target (test_solver_bak.py:147-152)
    rep = pb.solve_bak(np.eye(4, order="F"), np.zeros(4), pb.SolveConfig(record_history=True))
    assert rep.converged and rep.sweeps_run == 0 and rep.residual_norm_history == []
    np.testing.assert_array_equal(rep.a_hat, np.zeros(4))
    # all-zero matrix -> ValueError (bak.py:186-187)
    with pytest.raises(ValueError):
        pb.solve_bak(np.zeros((3, 2), order="F"), np.ones(3))
    # validation (test_solver_bak.py:182-193)
    with pytest.raises(ValueError):
        pb.solve_bak(np.eye(3, order="F"), np.ones(4))
    with pytest.raises(ValueError):
        pb.solve_bak(np.eye(3, order="F"), np.ones(3), a0=np.ones(2))
    # history not recorded by default
    assert pb.solve_bak(np.eye(2, order="F"), np.ones(2)).residual_norm_history is None
    # int input coerced to float64 (core.py:53-54)
    rep = pb.solve_bak(np.eye(3, dtype=np.int64), np.array([1, 2, 3]), pb.SolveConfig(max_iter=1, tol=0))
    assert rep.a_hat.dtype == np.float64


def test_coordinate_update_and_residual_norm_kat():
    pb = _pb()
    da, e_next = pb.coordinate_update(np.array([1.0, 2.0]), np.array([3.0, 4.0]))
    assert da == pytest.approx(2.2, rel=1e-15)
    np.testing.assert_allclose(e_next, [0.8, -0.4], atol=1e-12)
    e = np.array([1.0, 2.0])
    da, e2 = pb.coordinate_update(np.zeros(2), e)
    assert da == 0.0 and e2 is e
    assert pb.residual_norm(np.array([0.8, -0.4])) == pytest.approx(0.8, rel=1e-12)
    assert pb.residual_norm(np.ones(3)) == 3.0


def test_batched_matches_oracle_per_system():
    pb = _pb()
    nsys = 40
    xs, ys, refs = [], [], []
    for s in range(nsys):
        x, y, _ = orc.config_c5_system(s)
        xs.append(x)
        ys.append(y)
    xs = np.stack(xs)
    ys = np.stack(ys)
    rep = pb.solve_bak_batched(xs, ys, pb.SolveConfig(max_iter=200, tol=0, record_history=True))
    for s in range(nsys):
        if s < 4:
            g = golden_io.load(f"c5_system{s}_512x32_f32")
            ref_a = g["a_hat"]
        else:
            ref_a = orc.solve(xs[s], ys[s], max_iter=200, tol=0)["a_hat"]
        assert rep.sweeps_run[s] == 200 and not rep.converged[s]
        assert orc.rel_coeff_err(rep.a_hat[s], ref_a) <= 1e-4
        r = orc.residual_norm_f64(xs[s], ys[s], rep.a_hat[s])
        r_ref = orc.residual_norm_f64(xs[s], ys[s], ref_a)
        assert abs(r - r_ref) / r_ref <= 1e-4


@pytest.mark.parametrize("shape", [(512, 32, np.float32), (200, 12, np.float64), (37, 6, np.float64)])
def test_batched_smem_resident_and_streamed_x_agree(shape, monkeypatch):
    """x resident in shared memory vs streamed from L2/HBM every sweep (the
    default when residency would leave < 8 systems per SM): same arithmetic,
    same bits."""
    pb = _pb()
    obs, nv, dt = shape
    rng = np.random.default_rng(obs)
    xs = rng.standard_normal((24, obs, nv)).astype(dt)
    ys = rng.standard_normal((24, obs)).astype(dt)
    cfg = pb.SolveConfig(max_iter=30, tol=1e-9, record_history=True)
    monkeypatch.setenv("BAK_BATCH_X", "smem")
    r1 = pb.solve_bak_batched(xs, ys, cfg)
    monkeypatch.setenv("BAK_BATCH_X", "stream")
    r2 = pb.solve_bak_batched(xs, ys, cfg)
    assert r1.a_hat.tobytes() == r2.a_hat.tobytes()
    assert r1.residual.tobytes() == r2.residual.tobytes()
    assert np.array_equal(r1.sweeps_run, r2.sweeps_run)
    assert np.array_equal(r1.residual_norm_history, r2.residual_norm_history)


def test_batched_edge_cases():
    pb = _pb()
    rng = np.random.default_rng(5)
    xs = rng.standard_normal((3, 37, 6))
    xs[1, :, 2] = 0.0
    ys = rng.standard_normal((3, 37))
    ys[2] = 0.0
    a0 = np.zeros((3, 6))
    a0[1, 2] = 7.5
    rep = pb.solve_bak_batched(xs, ys, pb.SolveConfig(max_iter=50, tol=1e-8, record_history=True), a0=a0)
    for s in range(3):
        ref = orc.solve(xs[s], ys[s], max_iter=50, tol=1e-8, a0=a0[s], record_history=True)
        assert rep.sweeps_run[s] == ref["sweeps_run"]
        assert rep.converged[s] == ref["converged"]
        if s != 2:
            assert orc.rel_coeff_err(rep.a_hat[s], ref["a_hat"]) <= 1e-10
    assert rep.a_hat[1, 2] == 7.5
    assert np.all(rep.a_hat[2] == 0) and rep.sweeps_run[2] == 0 and rep.converged[2]


@pytest.mark.parametrize("precision", ["double", "single"])
def test_gram_variant_matches_oracle(precision):
    """GRAM is a labelled, algebraically equivalent reformulation: it must meet
    the same parity bar as the exact kernels."""
    pb = _pb()
    x, y, _ = orc.config_c3(obs=1 << 18, nvars=48, precision=precision)
    ref = orc.solve(x, y, max_iter=6, tol=0, record_history=True)
    rep = pb.solve_bak(x, y, pb.SolveConfig(max_iter=6, tol=0, record_history=True), variant="gram")
    assert rep.variant == "gram"
    assert_parity(x, y, rep, ref["a_hat"], ref["sweeps_run"], ref["converged"], ref_hist=ref["residual_norm_history"])


def test_gram_variant_random_order_zero_columns_early_break():
    pb = _pb()
    rng = np.random.default_rng(19)
    x = np.asfortranarray(rng.standard_normal((20_000, 20)))
    x[:, 7] = 0.0
    y = x @ rng.standard_normal(20) + 1e-3 * rng.standard_normal(20_000)
    a0 = np.zeros(20)
    a0[7] = 7.5
    for cfg in (dict(max_iter=60, tol=1e-9, record_history=True),
                dict(max_iter=25, tol=1e-12, ordering="random", ordering_seed=4, record_history=True)):
        ref = orc.solve(x, y, a0=a0, **cfg)
        rep = pb.solve_bak(x, y, pb.SolveConfig(**cfg), a0=a0, variant="gram")
        assert rep.a_hat[7] == 7.5
        assert_parity(x, y, rep, ref["a_hat"], ref["sweeps_run"], ref["converged"],
                      ref_hist=ref["residual_norm_history"])


@pytest.mark.parametrize("precision,nshards", [("double", 3), ("single", 2), ("double", 1)])
def test_rowsharded_gram_emulated_ranks(precision, nshards):
    """N ranks emulated in one process (LocalComm): rows split as on N GPUs,
    partials exchanged in rank order; must match the oracle on the full system."""
    from paper_2104_12570_b200.sharded import LocalComm, partition_rows, solve_bak_rowsharded
    pb = _pb()
    x, y, _ = orc.config_c3(obs=100_003, nvars=40, precision=precision)
    blocks = [partition_rows(x.shape[0], nshards, r, align=4) for r in range(nshards)]
    xs = [x[r0:r1] for r0, r1 in blocks]
    ys = [y[r0:r1] for r0, r1 in blocks]
    cfg = dict(max_iter=7, tol=0, record_history=True)
    reps = solve_bak_rowsharded(xs, ys, pb.SolveConfig(**cfg), LocalComm(nshards))
    ref = orc.solve(x, y, **cfg)
    for rep in reps:
        assert rep.a_hat.tobytes() == reps[0].a_hat.tobytes()  # replicated bit-identically
    full = reps[0]
    full.residual = np.concatenate([r.residual for r in reps])
    assert_parity(x, y, full, ref["a_hat"], ref["sweeps_run"], ref["converged"], ref_hist=ref["residual_norm_history"])


def test_rowsharded_early_break_matches_oracle():
    from paper_2104_12570_b200.sharded import LocalComm, partition_rows, solve_bak_rowsharded
    pb = _pb()
    x, y, _ = orc.make_system(60_000, 30, 8, "normal", "uniform", 0.0, "double")
    blocks = [partition_rows(x.shape[0], 4, r, align=4) for r in range(4)]
    reps = solve_bak_rowsharded([x[a:b] for a, b in blocks], [y[a:b] for a, b in blocks],
                                pb.SolveConfig(max_iter=200, tol=1e-11), LocalComm(4))
    ref = orc.solve(x, y, max_iter=200, tol=1e-11)
    assert reps[0].sweeps_run == ref["sweeps_run"] and reps[0].converged
    assert orc.rel_coeff_err(reps[0].a_hat, ref["a_hat"]) <= 1e-10


@pytest.mark.parametrize("nranks,precision", [(2, "double"), (4, "double"), (3, "single"), (8, "double")])
def test_rowshard_exact_kernel_emulated_ranks(nranks, precision):
    """The exact per-column row-sharded kernel with its in-kernel per-column
    rank exchange, N ranks emulated in ONE cooperative launch (their mailboxes
    in local memory).  Every rank's replica of a must be bit-identical and
    match the oracle; history and control flow too."""
    import torch
    from paper_2104_12570_b200.sharded import Mailboxes, sweep_rowshard
    pb = _pb()
    x, y, _ = orc.config_c3(obs=60_001, nvars=12, precision=precision)
    x[:, 5] = 0.0  # zero-norm column stays frozen
    cfg = dict(max_iter=6, tol=0, record_history=True)
    ref = orc.solve(x, y, **cfg)
    dm = pb.to_device_matrix(x)
    norms = pb.colnorms(dm)
    dev = dm.data.device
    tdt = torch.float64 if precision == "double" else torch.float32
    e = torch.from_numpy(np.ascontiguousarray(y)).to(dev)
    a = torch.zeros(nranks * 12, dtype=tdt, device=dev)
    hist = torch.zeros(nranks * 6, dtype=torch.float64, device=dev)
    mb = Mailboxes(nranks)
    status = sweep_rowshard(dm, e, a, norms, 6, -1.0, mb, 0, nranks, nranks_local=nranks, history=hist)
    st = status.cpu().numpy().reshape(nranks, 4)
    assert np.all(st[:, 0] == 6) and np.all(st[:, 2] == 0)
    A = a.cpu().numpy().reshape(nranks, 12)
    for r in range(1, nranks):
        assert A[r].tobytes() == A[0].tobytes()
    H = hist.cpu().numpy().reshape(nranks, 6)
    assert np.array_equal(H[0], H[-1])
    tol = TOL[np.dtype(x.dtype)]
    assert orc.rel_coeff_err(A[0], ref["a_hat"]) <= tol
    assert A[0][5] == 0.0
    np.testing.assert_allclose(H[0], ref["residual_norm_history"], rtol=max(1e3 * tol, 1e-6))
    # a second call on the same mailboxes (epochs keep increasing, no reset)
    a2 = torch.zeros_like(a)
    e2 = torch.from_numpy(np.ascontiguousarray(y)).to(dev)
    sweep_rowshard(dm, e2, a2, norms, 6, -1.0, mb, 0, nranks, nranks_local=nranks)
    assert a2.cpu().numpy().reshape(nranks, 12)[0].tobytes() == A[0].tobytes()


@pytest.mark.parametrize("obs,onchip", [(40_000, "1"), (40_000, "0"), (1_300_000, "1")])
def test_rowsharded_api_stream_single_process(obs, onchip, monkeypatch):
    """solve_bak_rowsharded(variant='stream') on one process: the exact in-kernel
    exchange path with N=1 must match the oracle (the N>1 exchange is covered by
    the emulated-ranks kernel test).  A rank whose rows fit on chip runs the
    on-chip GRID sweep (register plans; XT past 1M rows) with the mailbox stage
    inside its two-level exchange; BAK_ROWSHARD_ONCHIP=0 keeps the STREAM pass."""
    from paper_2104_12570_b200.sharded import solve_bak_rowsharded
    pb = _pb()
    monkeypatch.setenv("BAK_ROWSHARD_ONCHIP", onchip)
    nv = 10 if obs < 100_000 else 4
    x, y, _ = orc.config_c3(obs=obs, nvars=nv, precision="double")
    cfg = dict(max_iter=5, tol=0, record_history=True)
    rep = solve_bak_rowsharded([x], [y], pb.SolveConfig(**cfg), variant="stream")[0]
    ref = orc.solve(x, y, **cfg)
    assert rep.variant == ("grid-rowshard" if onchip == "1" else "stream-rowshard")
    assert_parity(x, y, rep, ref["a_hat"], ref["sweeps_run"], ref["converged"], ref_hist=ref["residual_norm_history"])
    if onchip == "1":  # same bits as the single-device GRID sweep (one rank: the mailbox adds 0 + total)
        one = pb.solve_bak(x, y, pb.SolveConfig(**cfg), variant="grid")
        assert one.a_hat.tobytes() == rep.a_hat.tobytes()


@pytest.mark.parametrize("precision", ["double", "single"])
def test_gram_pipelined_host_upload_matches_oracle(precision, monkeypatch):
    """Pinned host x: row blocks uploaded on two copy streams while G and the
    first pass run per block; must match the oracle like the resident path."""
    import torch
    from paper_2104_12570_b200 import bak as pbak
    pb = _pb()
    monkeypatch.setattr(pbak, "_PIPE_MIN_BYTES", 1 << 16)
    monkeypatch.setattr(pbak, "_PIPE_CHUNK_BYTES", 1 << 20)  # several blocks
    x, y, _ = orc.config_c3(obs=100_000, nvars=24, precision=precision)
    hx = torch.from_numpy(np.ascontiguousarray(x.T)).pin_memory().t()  # (obs, vars) column-major, pinned
    cfg = dict(max_iter=6, tol=0, record_history=True)
    rep = pb.solve_bak(hx, y, pb.SolveConfig(**cfg), variant="gram")
    ref = orc.solve(x, y, **cfg)
    assert_parity(x, y, rep, ref["a_hat"], ref["sweeps_run"], ref["converged"], ref_hist=ref["residual_norm_history"])
    rep2 = pb.solve_bak(hx, y, pb.SolveConfig(max_iter=80, tol=1e-6), variant="gram")
    ref2 = orc.solve(x, y, max_iter=80, tol=1e-6)
    assert rep2.sweeps_run == ref2["sweeps_run"] and rep2.converged == ref2["converged"]


@pytest.mark.parametrize("precision", ["double", "single"])
def test_grid_two_level_and_flat_exchange_match_oracle(precision, monkeypatch):
    """GRID variant: the two-level exchange (clusters of 8 through DSMEM, then
    cluster leaders through global records) and the one-level aggregator both
    meet the bar, and each is deterministic run to run."""
    pb = _pb()
    x, y, _ = orc.config_c3(obs=200_000, nvars=16, precision=precision)
    ref = orc.solve(x, y, max_iter=4, tol=0, record_history=True)
    tol = TOL[np.dtype(x.dtype)]
    outs = {}
    for flat in ("0", "1"):
        monkeypatch.setenv("BAK_GRID_FLAT", flat)
        r1 = pb.solve_bak(x, y, pb.SolveConfig(max_iter=4, tol=0, record_history=True), variant="grid")
        r2 = pb.solve_bak(x, y, pb.SolveConfig(max_iter=4, tol=0, record_history=True), variant="grid")
        assert r1.variant == "grid" and r1.a_hat.tobytes() == r2.a_hat.tobytes()
        assert orc.rel_coeff_err(r1.a_hat, ref["a_hat"]) <= tol
        np.testing.assert_allclose(r1.residual_norm_history, ref["residual_norm_history"], rtol=max(1e3 * tol, 1e-6))
        outs[flat] = r1.a_hat
    assert orc.rel_coeff_err(outs["0"], outs["1"]) <= tol


def test_batched_pipelined_host_upload_bit_identical():
    """Pinned host batches >= 256 MB take the chunked path (upload of chunk k+1
    overlapped with the solve of chunk k): same kernels, same bits."""
    import torch
    pb = _pb()
    nsys, obs, nv = 8192, 512, 32
    g = torch.Generator().manual_seed(7)
    hx = torch.randn((nsys, nv, obs), generator=g, dtype=torch.float32).pin_memory()
    hy = torch.randn((nsys, obs), generator=g, dtype=torch.float32).pin_memory()
    xs = hx.transpose(1, 2)  # (nsys, obs, vars) view, pinned
    cfg = pb.SolveConfig(max_iter=20, tol=0, record_history=True)
    r_pipe = pb.solve_bak_batched(xs, hy, cfg)
    r_ref = pb.solve_bak_batched(xs.contiguous(), hy.clone(), cfg)  # pageable, resident path
    assert r_pipe.a_hat.tobytes() == r_ref.a_hat.tobytes()
    assert r_pipe.residual.tobytes() == r_ref.residual.tobytes()
    assert np.array_equal(r_pipe.sweeps_run, r_ref.sweeps_run)
    assert np.array_equal(r_pipe.residual_norm_history, r_ref.residual_norm_history)
    s = 1234
    ref = orc.solve(hx[s].numpy().T, hy[s].numpy(), max_iter=20, tol=0)
    assert orc.rel_coeff_err(r_pipe.a_hat[s], ref["a_hat"]) <= 1e-4


@pytest.mark.parametrize("obs,nv,precision", [(1_100_003, 6, "double"), (2_097_152, 5, "double"),
                                              (1_600_001, 4, "double"), (2_000_000, 5, "single")])
def test_xs_exact_sweep_tall_matches_oracle(obs, nv, precision):
    """The exact on-chip sweep for row blocks past register capacity (GRID, x read
    from the quarter-column ring, e in registers): 1.1M-2.1M rows on one GPU,
    ragged rows, against the oracle; random ordering and an early break too."""
    pb = _pb()
    x, y, _ = orc.config_c3(obs=obs, nvars=nv, precision=precision)
    tol = TOL[np.dtype(x.dtype)]
    cfg = dict(max_iter=3, tol=0, record_history=True)
    ref = orc.solve(x, y, **cfg)
    rep = pb.solve_bak(x, y, pb.SolveConfig(**cfg), variant="grid")
    assert rep.variant == "grid" and rep.sweeps_run == 3
    assert orc.rel_coeff_err(rep.a_hat, ref["a_hat"]) <= tol
    np.testing.assert_allclose(rep.residual_norm_history, ref["residual_norm_history"], rtol=max(1e3 * tol, 1e-6))
    if precision == "double" and nv == 6:
        cfg2 = dict(max_iter=20, tol=1e-3, ordering="random", ordering_seed=5, record_history=True)
        ref2 = orc.solve(x, y, **cfg2)
        rep2 = pb.solve_bak(x, y, pb.SolveConfig(**cfg2), variant="grid")
        assert rep2.sweeps_run == ref2["sweeps_run"] and rep2.converged == ref2["converged"]
        assert orc.rel_coeff_err(rep2.a_hat, ref2["a_hat"]) <= tol


@pytest.mark.parametrize("obs,nv,precision", [(1_300_001, 5, "double"), (2_097_152, 4, "double"),
                                              (2_000_000, 4, "single")])
def test_xt_tmem_stash_bit_identical_to_xs_ring(obs, nv, precision, monkeypatch):
    """XT (x_{t+1} stashed in tensor memory between its dot and its update; the
    default for row blocks past register capacity) against the XS quarter-column
    ring (BAK_GRID_XT=0): the same per-row operations in the same order, so the
    bits agree; both against the oracle."""
    pb = _pb()
    x, y, _ = orc.config_c3(obs=obs, nvars=nv, precision=precision)
    cfg = pb.SolveConfig(max_iter=3, tol=0, record_history=True)
    monkeypatch.delenv("BAK_GRID_XT", raising=False)
    r_xt = pb.solve_bak(x, y, cfg, variant="grid")
    monkeypatch.setenv("BAK_GRID_XT", "0")
    r_xs = pb.solve_bak(x, y, cfg, variant="grid")
    assert r_xt.variant == "grid" and r_xs.variant == "grid"
    assert r_xt.a_hat.tobytes() == r_xs.a_hat.tobytes()
    assert r_xt.residual.tobytes() == r_xs.residual.tobytes()
    assert r_xt.residual_norm_history == r_xs.residual_norm_history
    ref = orc.solve(x, y, max_iter=3, tol=0)
    assert orc.rel_coeff_err(r_xt.a_hat, ref["a_hat"]) <= TOL[np.dtype(x.dtype)]

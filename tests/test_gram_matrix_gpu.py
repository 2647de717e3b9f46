"""The G = X^T X kernels behind the GRAM variant, checked directly against an
fp64 numpy product: fp64 DMMA (exact products, fp64 sums) and, for fp32
inputs, 3xTF32 (hi/lo split, ~2^-21 relative) and the fp64 DMMA fallback
(BAK_GRAM_G=dmma).  Shapes cover ragged rows / columns, a single 64-column
block and several diagonal / off-diagonal blocks."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _gram(x, monkeypatch=None, env=None):
    import torch
    import paper_2104_12570_b200 as pb
    from paper_2104_12570_b200 import _lib
    from paper_2104_12570_b200.bak import _Workspace, _stream_ptr
    if env:
        for k, v in env.items():
            monkeypatch.setenv(k, v)
    lib = _lib.load()
    dm = pb.to_device_matrix(x)
    dev = dm.data.device
    G = torch.empty((dm.vars, dm.vars), dtype=torch.float64, device=dev)
    ws = _Workspace(torch, dev, lib.bak_gram_matrix_workspace(dm.code, dm.obs, dm.vars))
    _lib.check(lib.bak_gram_matrix(dm.code, dm.ptr, dm.obs, dm.vars, dm.ldx, G.data_ptr(), ws.ptr, ws.nbytes,
                                   _stream_ptr(torch, dev)), "bak_gram_matrix")
    return G.cpu().numpy()


@pytest.mark.parametrize("obs,nv", [(1000, 7), (50_001, 64), (131_071, 130), (200_000, 256)])
def test_gram_matrix_fp64_dmma(obs, nv):
    x = np.asfortranarray(np.random.default_rng(obs).standard_normal((obs, nv)))
    ref = x.T @ x
    G = _gram(x)
    assert np.allclose(G, G.T, rtol=0, atol=0)  # mirrored exactly
    err = np.linalg.norm(G - ref) / np.linalg.norm(ref)
    assert err <= 1e-13, err


@pytest.mark.parametrize("obs,nv", [(1000, 7), (50_001, 64), (131_071, 130), (200_000, 256)])
def test_gram_matrix_fp32_3xtf32_and_dmma(obs, nv, monkeypatch):
    x = np.asfortranarray(np.random.default_rng(obs + 1).standard_normal((obs, nv)).astype(np.float32))
    xd = x.astype(np.float64)
    ref = xd.T @ xd  # exact products of the fp32 inputs, fp64 sums
    G3 = _gram(x)
    err3 = np.linalg.norm(G3 - ref) / np.linalg.norm(ref)
    assert err3 <= 2e-6, err3
    # diagonal (the column norms the solve divides by) to a few 2^-21
    d_err = np.max(np.abs(np.diag(G3) - np.diag(ref)) / np.diag(ref))
    assert d_err <= 4e-6, d_err
    # the legacy mma.sync 3xTF32 kernel (BAK_GRAM_G=x3) meets the same bar
    Gx = _gram(x, monkeypatch, {"BAK_GRAM_G": "x3"})
    errx = np.linalg.norm(Gx - ref) / np.linalg.norm(ref)
    assert errx <= 2e-6, errx
    Gd = _gram(x, monkeypatch, {"BAK_GRAM_G": "dmma"})
    errd = np.linalg.norm(Gd - ref) / np.linalg.norm(ref)
    assert errd <= 1e-13, errd


@pytest.mark.parametrize("obs,nv,chunk", [(1000, 7, None), (50_001, 64, None), (131_071, 130, None),
                                          (200_000, 256, None), (100_003, 200, "32"), (300_000, 256, "65536")])
def test_gram_fp32_tcgen05_with_fused_first_dots(obs, nv, chunk, monkeypatch):
    """fp32 G on tcgen05 (kind::tf32, TMEM): G and the fused g0 = X^T e against
    fp64 numpy; ragged rows / columns, vb = 128 and 256, one-tile and large chunks."""
    import torch
    import paper_2104_12570_b200 as pb
    from paper_2104_12570_b200 import _lib
    from paper_2104_12570_b200.bak import _Workspace, _stream_ptr
    if chunk:
        monkeypatch.setenv("BAK_GRAM_TC_CHUNK", chunk)
    rng = np.random.default_rng(obs + nv)
    x = np.asfortranarray(rng.standard_normal((obs, nv)).astype(np.float32))
    e = rng.standard_normal(obs).astype(np.float32)
    xd = x.astype(np.float64)
    ref = xd.T @ xd
    gref = xd.T @ e.astype(np.float64)
    lib = _lib.load()
    dm = pb.to_device_matrix(x)
    dev = dm.data.device
    ed = torch.from_numpy(e).to(dev)
    G = torch.empty((nv, nv), dtype=torch.float64, device=dev)
    rows = int(lib.bak_gram_dot_rows(dm.code, obs, nv))
    assert rows == 1  # the tcgen05 path reduces the fused dots to one row
    g0 = torch.zeros((rows, nv), dtype=torch.float64, device=dev)
    ws = _Workspace(torch, dev, lib.bak_gram_matrix_workspace(dm.code, obs, nv))
    st = _stream_ptr(torch, dev)
    _lib.check(lib.bak_gram_matrix_dot(dm.code, dm.ptr, obs, nv, dm.ldx, G.data_ptr(), ed.data_ptr(), g0.data_ptr(),
                                       ws.ptr, ws.nbytes, st), "bak_gram_matrix_dot")
    Gh, gh = G.cpu().numpy(), g0.cpu().numpy()[0]
    assert np.array_equal(Gh, Gh.T)
    # off-diagonal: the tensor core's truncating fp32 accumulation over C rows leaves an
    # entry low by ~1.2e-8 * C of itself (default C = 1024; tools/gram_tc_probe.py)
    c = int(chunk or 1024)
    off = ~np.eye(nv, dtype=bool)
    off_err = np.max(np.abs(Gh - ref)[off] / np.sqrt(np.outer(np.diag(ref), np.diag(ref)))[off])
    assert off_err <= max(2e-6, 4e-8 * c) / np.sqrt(obs) * 40, off_err
    err = np.linalg.norm(Gh - ref) / np.linalg.norm(ref)
    assert err <= (2e-6 if c <= 4096 else 2e-5), err
    # diagonal (the column norms the solve divides by): fp32 FMA chains per 32-row tile
    d_err = np.max(np.abs(np.diag(Gh) - np.diag(ref)) / np.diag(ref))
    assert d_err <= 1e-6, d_err
    # fused first-sweep dots: fp32 FMA chains per 32-row tile, tiles summed in fp64
    scale = np.sqrt(np.diag(ref) * float(e.astype(np.float64) @ e))
    assert np.max(np.abs(gh - gref) / scale) <= 1e-6
    # deterministic
    G2 = torch.empty_like(G)
    _lib.check(lib.bak_gram_matrix(dm.code, dm.ptr, obs, nv, dm.ldx, G2.data_ptr(), ws.ptr, ws.nbytes, st),
               "bak_gram_matrix")
    assert torch.equal(G, G2)


def test_batched_wave_is_whole_sms():
    from paper_2104_12570_b200 import _lib
    import torch
    lib = _lib.load()
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    for dt, obs, nv in ((0, 512, 32), (1, 200, 12), (0, 37, 6)):
        w = int(lib.bak_solve_batched_wave(dt, obs, nv))
        assert w > 0 and w % sms == 0, (dt, obs, nv, w)


@pytest.mark.parametrize("corr", [0.9, 0.99])
def test_gram_fp32_3xtf32_on_correlated_columns(corr, monkeypatch):
    """fp32 GRAM solves on strongly correlated (slowly converging) columns,
    where G's rounding shapes the iterates sweep by sweep: the 3xTF32 G meets
    the fp32 bar against the oracle after a fixed number of sweeps, like the
    fp64-DMMA G does."""
    import paper_2104_12570_b200 as pb
    from oracle import bak_oracle as orc
    rng = np.random.default_rng(int(corr * 1000))
    obs, nv = 60_000, 96
    base = rng.standard_normal((obs, 1))
    x = np.asfortranarray((corr * base + (1 - corr) * rng.standard_normal((obs, nv))).astype(np.float32))
    y = (x @ rng.uniform(-1, 1, nv).astype(np.float32) + 0.01 * rng.standard_normal(obs)).astype(np.float32)
    ref = orc.solve(x, y, max_iter=12, tol=0)
    for env in (None, {"BAK_GRAM_G": "dmma"}):
        if env:
            monkeypatch.setenv("BAK_GRAM_G", "dmma")
        rep = pb.solve_bak(x, y, pb.SolveConfig(max_iter=12, tol=0), variant="gram")
        err = orc.rel_coeff_err(rep.a_hat, ref["a_hat"])
        assert rep.sweeps_run == 12 and err <= 1e-4, (corr, env, err)


@pytest.mark.parametrize("obs,nv", [(1000, 7), (50_001, 64), (131_071, 130), (200_003, 256), (70_000, 320)])
def test_gram_matrix_fp64_tma_matches_cp_async_bitwise(obs, nv, monkeypatch):
    """The TMA-fed fp64 G kernel (default) issues the same DMMAs in the same order as the cp.async
    kernel (BAK_GRAM_G_TMA=0): identical bits, with or without the advisory lock step, with one or
    two units per CTA, on ragged rows / columns (zero-filled by the TMA unit)."""
    x = np.asfortranarray(np.random.default_rng(obs + 7).standard_normal((obs, nv)))
    base = _gram(x, monkeypatch, {"BAK_GRAM_G_TMA": "0", "BAK_GRAM_PACE": "0"})
    for env in ({"BAK_GRAM_G_TMA": "1", "BAK_GRAM_PACE": "0", "BAK_GRAM_UNITS": "0"},
                {"BAK_GRAM_G_TMA": "1", "BAK_GRAM_PACE": "1", "BAK_GRAM_UNITS": "0"},
                {"BAK_GRAM_G_TMA": "1", "BAK_GRAM_PACE": "3", "BAK_GRAM_UNITS": "0"},
                {"BAK_GRAM_G_TMA": "0", "BAK_GRAM_PACE": "1", "BAK_GRAM_UNITS": "0"}):
        G = _gram(x, monkeypatch, env)
        assert np.array_equal(G, base), env
    # two units per CTA: other chunk boundaries, so other (fixed-order) sums — same accuracy bar
    G2 = _gram(x, monkeypatch, {"BAK_GRAM_G_TMA": "1", "BAK_GRAM_PACE": "1", "BAK_GRAM_UNITS": "1"})
    ref = x.T @ x
    assert np.linalg.norm(G2 - ref) / np.linalg.norm(ref) <= 1e-13
    assert np.array_equal(G2, G2.T)


def test_gram_fused_first_dots_tma_vs_cp_async(monkeypatch):
    """GRAM solves through the TMA-fed G kernel (fused first-sweep dots as four FMA chains) and through
    the cp.async kernel agree to rounding, and both meet the oracle bar."""
    import paper_2104_12570_b200 as pb
    from oracle import bak_oracle as orc
    x, y, _ = orc.config_c3(obs=1 << 16, nvars=96)
    ref = orc.solve(x, y, max_iter=4, tol=0)
    out = {}
    for tma in ("0", "1"):
        monkeypatch.setenv("BAK_GRAM_G_TMA", tma)
        r = pb.solve_bak(x, y, pb.SolveConfig(max_iter=4, tol=0), variant="gram")
        assert orc.rel_coeff_err(r.a_hat, ref["a_hat"]) <= 1e-10
        out[tma] = np.asarray(r.a_hat, dtype=np.float64)
    assert np.linalg.norm(out["0"] - out["1"]) <= 1e-13 * np.linalg.norm(out["0"])

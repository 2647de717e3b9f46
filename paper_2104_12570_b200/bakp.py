"""Drop-in B200 replacement for ``baksolve.bakp`` (reference bakp.py:1-185),
the blocked variant of the sweep (the paper's Algorithm 2).

Same names, arguments, defaults, validation and exceptions:

    solve_bakp(x, y, config: BlockConfig | None = None) -> SolveReport
    block_deltas(x, block, e, norms_sq=None) -> ndarray
    BlockConfig(base=SolveConfig(), thr=1, worker_count=0)
    DivergenceError, DIVERGENCE_FACTOR

Every number comes from the sm_100a kernels behind ``bak_block_sweep`` /
``bak_block_deltas`` (include/bak200.h).  ``worker_count`` is accepted and
validated for API compatibility; like the reference, it does not change a bit
of the result (bakp.py:10-15) — the GPU's parallelism is not a thread count.
With thr=1 the blocked sweep IS the sequential sweep (bakp.py:13-15): it runs
the same kernel as ``solve_bak`` and reproduces it bit for bit.

Extensions (keyword-only): variant="auto"|"cta"|"cluster"|"stream"|"gram"
("gram" = labelled algebraically-equivalent block substitution through
G = X^T X, one pass over x per sweep), device=None, return_device=False.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .bak import (_host, DRIFT_TOL, SolveConfig, SolveReport, _ptr, _residual, _stream_ptr, _sumsq,
                  _to_device_vector, _torch, _workspace_bytes, _Workspace, colnorms, solve_bak, to_device_matrix)

DIVERGENCE_FACTOR = 10.0              # bakp.py:32
_BLOCK_VARIANTS = ("auto", "cta", "cluster", "stream", "gram")


class DivergenceError(RuntimeError):
    """Residual norm grew past the divergence guard; thr is too large (bakp.py:35-36)."""


@dataclass
class BlockConfig:
    """Mirror of the reference BlockConfig (bakp.py:39-49), same validation."""
    base: SolveConfig = field(default_factory=SolveConfig)
    thr: int = 1
    worker_count: int = 0

    def __post_init__(self):
        if self.thr < 1:
            raise ValueError(f"thr must be >= 1, got {self.thr}")
        if self.worker_count < 0:
            raise ValueError(f"worker_count must be >= 0, got {self.worker_count}")


def _divergence_message(prev_sq, sq, thr):
    # bakp.py:122-124
    return (f"residual norm grew from {prev_sq:.6g} to {sq:.6g} in one sweep "
            f"with thr={thr}; use a smaller thr")


def _first_divergence(history, ynorm2):
    """(prev, sq) of the first sweep the guard of bakp.py:121 rejects, else None."""
    prev = ynorm2
    for sq in history:
        if not np.isfinite(sq) or sq > prev * DIVERGENCE_FACTOR:
            return prev, sq
        prev = sq
    return None


def block_deltas(x, block, e, norms_sq=None):
    """Deltas for one block of columns against a fixed residual (bakp.py:65-85).

    block is a (start, stop) index range.  Zero-norm columns get delta 0.
    """
    torch = _torch()
    lib = _lib.load()
    xa = x if _is_tensor(x) else np.asarray(x)
    ea = e if _is_tensor(e) else np.asarray(e)
    start, stop = block
    obs, nvars = tuple(xa.shape)
    if not 0 <= start < stop <= nvars:
        raise ValueError(f"bad block range ({start}, {stop}) for {nvars} columns")
    if tuple(ea.shape) != (obs,):
        raise ValueError(f"residual has shape {tuple(ea.shape)}, expected ({obs},)")
    dm = to_device_matrix(xa)
    dev = dm.data.device
    st = _stream_ptr(torch, dev)
    ws = _Workspace(torch, dev, max(_workspace_bytes(lib, dm.code, dm.obs, dm.vars),
                                    lib.bak_block_deltas_workspace(dm.code, dm.obs)))
    if norms_sq is None:
        n2 = colnorms(dm, ws)
    else:
        n2 = _to_device_vector(norms_sq, dm.np_dtype, dev, "norms_sq")
    ed = _to_device_vector(ea, dm.np_dtype, dev, "e")
    out = torch.empty(stop - start, dtype=dm.data.dtype, device=dev)
    _lib.check(lib.bak_block_deltas(dm.code, dm.ptr, dm.obs, dm.vars, dm.ldx, start, stop, _ptr(ed), _ptr(n2),
                                    _ptr(out), ws.ptr, ws.nbytes, st), "bak_block_deltas")
    out_dtype = ea.dtype if not _is_tensor(ea) else dm.np_dtype
    return out.cpu().numpy().astype(out_dtype, copy=False)


def _is_tensor(v):
    try:
        import torch
    except ImportError:  # pragma: no cover
        return False
    return isinstance(v, torch.Tensor)


def solve_bakp(x, y, config: BlockConfig | None = None, *, variant="auto", device=None,
               return_device=False) -> SolveReport:
    """Blocked solve of min ||y - x @ a|| (bakp.py:132-185).

    Requires 1 <= thr <= vars; blocks are consecutive column ranges, with a
    narrower final block when thr does not divide the width.  Only cyclic
    ordering is supported.  Raises DivergenceError when the guard trips.
    """
    cfg = config if config is not None else BlockConfig()
    if cfg.base.ordering != "cyclic":
        raise ValueError("the blocked solver only supports cyclic ordering")
    if variant not in _BLOCK_VARIANTS:
        raise ValueError(f"unknown variant {variant!r}, expected one of {_BLOCK_VARIANTS}")
    torch = _torch()
    lib = _lib.load()
    dm = to_device_matrix(x, device)
    dev = dm.data.device
    obs, nvars, code = dm.obs, dm.vars, dm.code
    if cfg.thr > nvars:
        raise ValueError(f"thr={cfg.thr} exceeds the number of columns ({nvars})")
    yd = _to_device_vector(y, dm.np_dtype, dev)
    if yd.shape[0] != obs:
        raise ValueError(f"y has length {yd.shape[0]}, expected {obs}")
    base = cfg.base
    if cfg.thr == 1:
        # bakp.py:13-15: the one-column block is the sequential column step — an
        # EXACT kernel (auto never resolves to the labelled GRAM sweep here)
        if variant in ("auto", "stream"):
            exact = _lib.VARIANT_NAMES[int(lib.bak_sweep_pick_variant(code, obs, nvars))]
        else:
            exact = variant
        # the guard of bakp.py:121-124 at thr=1: the sequential sweep cannot grow
        # the residual in exact arithmetic, so only non-finite values trip it, on
        # the first sweep — run just that sweep instead of all max_iter of them
        finite = bool(torch.isfinite(dm.data[:, :obs]).all().item()) and bool(torch.isfinite(yd).all().item())
        sweeps = base.max_iter if finite else 1
        rep = solve_bak(dm, yd, SolveConfig(max_iter=sweeps, tol=base.tol, record_history=True),
                        variant=exact, device=dev, return_device=return_device)
        if rep.sweeps_run:
            ynorm2 = float(_sumsq(lib, torch, code, yd, _Workspace(torch, dev, lib.bak_colnorms_workspace(
                code, obs, 1)), _stream_ptr(torch, dev)).item())
            bad = _first_divergence(rep.residual_norm_history, ynorm2)
            if bad is not None:
                raise DivergenceError(_divergence_message(bad[0], bad[1], cfg.thr))
            if sweeps < base.max_iter and not rep.converged:  # non-finite input that did not trip it
                rep = solve_bak(dm, yd, SolveConfig(max_iter=base.max_iter, tol=base.tol, record_history=True),
                                variant=exact, device=dev, return_device=return_device)
                bad = _first_divergence(rep.residual_norm_history, ynorm2)
                if bad is not None:
                    raise DivergenceError(_divergence_message(bad[0], bad[1], cfg.thr))
        if not base.record_history:
            rep.residual_norm_history = None
        return rep

    st = _stream_ptr(torch, dev)
    t0 = time.perf_counter()
    vcode = _lib.VARIANTS[variant]
    if vcode == 0:
        vcode = lib.bak_block_pick_variant(code, obs, nvars, cfg.thr)
    ws = _Workspace(torch, dev, max(_workspace_bytes(lib, code, obs, nvars),
                                    lib.bak_block_sweep_workspace(code, vcode, obs, nvars, cfg.thr)))
    ynorm2 = float(_sumsq(lib, torch, code, yd, ws, st).item())
    if ynorm2 == 0.0:  # bakp.py:152-153 (_zero_report)
        a_z = torch.zeros(nvars, dtype=yd.dtype, device=dev)
        r_z = torch.zeros(obs, dtype=yd.dtype, device=dev)
        return SolveReport(a_hat=a_z if return_device else a_z.cpu().numpy(),
                           residual=r_z if return_device else r_z.cpu().numpy(),
                           residual_norm_history=[] if base.record_history else None,
                           sweeps_run=0, converged=True, wall_time=time.perf_counter() - t0)
    thresh2 = base.tol * base.tol * ynorm2 if base.tol > 0 else -1.0   # bakp.py:157
    norms = colnorms(dm, ws)
    if not bool((norms != 0).any().item()):
        raise ValueError("every column of x has zero norm; nothing to solve")
    e = yd.clone()
    a = torch.zeros(nvars, dtype=yd.dtype, device=dev)
    hist = torch.zeros(base.max_iter, dtype=torch.float64, device=dev)
    status = torch.zeros(4, dtype=torch.int64, device=dev)
    _lib.check(lib.bak_block_sweep(code, vcode, dm.ptr, obs, nvars, dm.ldx, _ptr(norms), cfg.thr, _ptr(e), _ptr(a),
                                   base.max_iter, thresh2, ynorm2, _ptr(hist), _ptr(status), ws.ptr, ws.nbytes, st),
               "bak_block_sweep")
    stat = status.cpu().numpy()
    sweeps, converged, err, used = int(stat[0]), bool(stat[1]), int(stat[2]), int(stat[3])
    if err == _lib.EDIVERGED:
        h = hist[:sweeps].cpu().numpy()
        prev = float(h[-2]) if sweeps >= 2 else ynorm2
        raise DivergenceError(_divergence_message(prev, float(h[-1]), cfg.thr))
    if err:
        raise _lib.BakError(f"bak_block_sweep device error {err} (3 = spin-wait timeout)")
    resid = torch.empty_like(yd)
    _residual(lib, dm, a, yd, resid, ws, st)                      # bak.py:130 via bakp.py:182
    drift2 = torch.empty(1, dtype=torch.float64, device=dev)
    _lib.check(lib.bak_diff_norm2(code, _ptr(e), _ptr(resid), obs, _ptr(drift2), ws.ptr, ws.nbytes, st),
               "bak_diff_norm2")
    drift = float(np.sqrt(drift2.item()))
    wall = time.perf_counter() - t0
    return SolveReport(
        a_hat=a if return_device else a.cpu().numpy(),
        residual=resid if return_device else _host(resid),
        residual_norm_history=hist[:sweeps].cpu().tolist() if base.record_history else None,
        sweeps_run=sweeps, converged=converged, wall_time=wall,
        drift_warning=bool(drift / max(np.sqrt(ynorm2), np.finfo(np.float64).tiny) > DRIFT_TOL),
        variant=_lib.VARIANT_NAMES.get(used, str(used)))

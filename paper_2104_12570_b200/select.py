"""Drop-in B200 replacement for the greedy column scoring and forward
selection of ``baksolve.select`` (reference select.py:1-136).

    score_all_columns(x, e, excluded=()) -> (best_j, scores)
    select_features(x, y, cfg: FeatureSelectConfig) -> FeatureSelectionReport
    FeatureSelectConfig, FeatureSelectionReport, SelectionExhaustedError, REFITS

Scoring is ONE fused pass over x on the GPU (``bak_score_columns``: X^T e,
sum e^2, the closed form <e,e> - <x_j,e>^2/<x_j,x_j> and the argmin).  In
``select_features`` x, its column norms, y and the residual stay on the
device for the whole selection; per pick the host reads back 16 bytes (the
winner).  Refits: ``refit="bak"`` runs this package's ``solve_bak``
warm-started from the previous coefficients (select.py:96-103);
``refit="qr"`` factors the picked columns with cuSOLVER's unpivoted
Householder QR (through torch) and back-substitutes on the host with the
reference's rank rule (qr.py:93-119: |r_jj| <= max(m,n)*eps*max|r| -> 0).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .bak import (SolveConfig, _ptr, _residual, _stream_ptr, _sumsq, _to_device_vector, _torch, _workspace_bytes,
                  _Workspace, colnorms, DeviceMatrix, solve_bak, to_device_matrix)

REFITS = ("qr", "bak")  # select.py:26


class SelectionExhaustedError(RuntimeError):
    """No admissible column left to score (select.py:29-30)."""


@dataclass
class FeatureSelectConfig:
    """Mirror of select.py:33-46, same validation."""
    max_feat: int
    refit: str = "qr"
    stop_tol: float = 0.0
    refit_config: SolveConfig | None = None

    def __post_init__(self):
        if self.max_feat < 1:
            raise ValueError(f"max_feat must be >= 1, got {self.max_feat}")
        if self.refit not in REFITS:
            raise ValueError(f"unknown refit {self.refit!r}, expected one of {REFITS}")
        if self.stop_tol < 0:
            raise ValueError(f"stop_tol must be >= 0, got {self.stop_tol}")


@dataclass
class FeatureSelectionReport:
    """Mirror of select.py:49-53."""
    selected: list
    residual_norms: list
    final_coeffs: np.ndarray


class _Scorer:
    """Device state of repeated scoring of one x: norms, workspace, outputs."""

    def __init__(self, lib, torch, dm: DeviceMatrix, norms=None):
        self.lib, self.torch, self.dm = lib, torch, dm
        dev = dm.data.device
        self.ws = _Workspace(torch, dev, max(lib.bak_score_columns_workspace(dm.code, dm.obs, dm.vars),
                                             _workspace_bytes(lib, dm.code, dm.obs, dm.vars)))
        self.norms = norms if norms is not None else colnorms(dm, self.ws)
        self.scores = torch.empty(dm.vars, dtype=torch.float64, device=dev)
        self.best = torch.zeros(2, dtype=torch.int64, device=dev)
        self.excluded = torch.zeros(dm.vars, dtype=torch.uint8, device=dev)
        self.st = _stream_ptr(torch, dev)

    def __call__(self, e):
        dm = self.dm
        _lib.check(self.lib.bak_score_columns(dm.code, dm.ptr, dm.obs, dm.vars, dm.ldx, _ptr(e), _ptr(self.norms),
                                              _ptr(self.excluded), _ptr(self.scores), _ptr(self.best), self.ws.ptr,
                                              self.ws.nbytes, self.st), "bak_score_columns")
        best, finite = (int(v) for v in self.best.cpu().tolist())
        if not finite:
            raise SelectionExhaustedError("no non-excluded column with nonzero norm")
        return best


def score_all_columns(x, e, excluded=()):
    """Score every column; returns (best_j, scores) (select.py:56-85).

    scores[j] is the squared residual norm a single update along column j
    would leave.  Excluded and zero-norm columns score +inf.  Ties go to the
    lowest index.  Raises SelectionExhaustedError when nothing is admissible.
    """
    torch = _torch()
    lib = _lib.load()
    xa = x if isinstance(x, DeviceMatrix) else np.asarray(x)
    obs, nvars = (xa.obs, xa.vars) if isinstance(xa, DeviceMatrix) else xa.shape
    ea = np.asarray(e) if not hasattr(e, "is_cuda") else e
    if tuple(ea.shape) != (obs,):
        raise ValueError(f"residual has shape {tuple(ea.shape)}, expected ({obs},)")
    dm = to_device_matrix(xa)
    sc = _Scorer(lib, torch, dm)
    if len(excluded):
        sc.excluded[torch.as_tensor(sorted(excluded), dtype=torch.int64, device=dm.data.device)] = 1
    ed = _to_device_vector(ea, dm.np_dtype, dm.data.device, "e")
    best = sc(ed)
    return best, sc.scores.cpu().numpy()


def _qr_refit(torch, xs: DeviceMatrix, yd):
    """Least squares on the picked columns: cuSOLVER Householder QR (no
    pivoting, like qr.py:47-73), Q^T y, then the reference's back
    substitution with its rank rule (qr.py:106-119) on the small k x k R."""
    m, n = xs.obs, xs.vars
    a_mat = xs.data[:, :m].t()                       # (m, n) column-major view
    q, r = torch.linalg.qr(a_mat, mode="reduced")
    qty = (q.t() @ yd).cpu().numpy()
    r = r.cpu().numpy()
    k = min(m, n)
    r_diag = np.diagonal(r)[:k]
    scale = float(np.max(np.abs(r_diag))) if r_diag.size else 0.0
    tol = max(m, n) * float(np.finfo(r_diag.dtype).eps) * scale
    a = np.zeros(n, dtype=r.dtype)
    for j in reversed(range(k)):
        rjj = r[j, j]
        if abs(rjj) <= tol:
            continue
        a[j] = (qty[j] - np.dot(r[j, j + 1:n], a[j + 1:])) / rjj
    return torch.from_numpy(a).to(yd.device)


def select_features(x, y, cfg: FeatureSelectConfig) -> FeatureSelectionReport:
    """Pick up to cfg.max_feat columns greedily, refitting after each pick
    (select.py:106-136).  Stops early when ||e|| / ||y|| <= cfg.stop_tol.
    Never picks a zero-norm or already-selected column."""
    torch = _torch()
    lib = _lib.load()
    dm = to_device_matrix(x)
    dev = dm.data.device
    obs, nvars = dm.obs, dm.vars
    yd = _to_device_vector(y, dm.np_dtype, dev)
    if yd.shape[0] != obs:
        raise ValueError(f"y has length {yd.shape[0]}, expected {obs}")
    if cfg.max_feat > nvars:
        raise ValueError(f"max_feat={cfg.max_feat} exceeds the number of columns ({nvars})")
    st = _stream_ptr(torch, dev)
    ynorm = float(torch.linalg.vector_norm(yd.double()).item())
    scorer = _Scorer(lib, torch, dm)
    ws = _Workspace(torch, dev, max(_workspace_bytes(lib, dm.code, obs, max(cfg.max_feat, 1)), 4096))
    selected: list[int] = []
    norms_out: list[float] = []
    coeffs = None
    e = yd.clone()
    for _ in range(cfg.max_feat):
        best = scorer(e)
        selected.append(best)
        scorer.excluded[best] = 1
        xs = DeviceMatrix(dm.data[torch.as_tensor(selected, device=dev)].contiguous(), obs, len(selected),
                          dm.np_dtype)
        if cfg.refit == "qr":
            coeffs = _qr_refit(torch, xs, yd)
        else:
            solve_cfg = cfg.refit_config if cfg.refit_config is not None else SolveConfig()
            a0 = torch.zeros(len(selected), dtype=yd.dtype, device=dev)
            if coeffs is not None:
                a0[: coeffs.shape[0]] = coeffs
            coeffs = solve_bak(xs, yd, solve_cfg, a0=a0, return_device=True).a_hat
        e = torch.empty_like(yd)
        _residual(lib, xs, coeffs, yd, e, ws, st)                      # select.py:130
        rn = float(_sumsq(lib, torch, dm.code, e, ws, st).item())      # select.py:131
        norms_out.append(rn)
        if cfg.stop_tol > 0 and ynorm > 0 and np.sqrt(rn) / ynorm <= cfg.stop_tol:
            break
    return FeatureSelectionReport(selected=selected, residual_norms=norms_out,
                                  final_coeffs=coeffs.cpu().numpy() if coeffs is not None else None)

"""Drop-in B200 replacement for ``baksolve.bak`` (reference bak.py:1-195).

Same names, arguments, defaults, validation messages and return type as the
reference's solve entry point:

    solve_bak(x, y, config: SolveConfig | None = None, a0=None) -> SolveReport

The host side only validates, moves buffers and sequences C-ABI calls
(libbak200.so, include/bak200.h); every number is computed by the sm_100a
kernels.  There is no CPU fallback: without a CUDA device or without the
library this module raises.

Extensions (keyword-only, defaults keep reference behaviour):
    variant="auto"|"cta"|"cluster"|"grid"|"stream"   exact per-column kernel family
            |"gram"                                   labelled algebraically-equivalent sweep
                                                      (one x pass per sweep via G = X^T X)
    device=None                                       torch device (default current CUDA device)
    return_device=False                               keep a_hat/residual as CUDA tensors
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass

import numpy as np

from . import _lib

ORDERINGS = ("cyclic", "random")      # bak.py:25
DRIFT_TOL = 1e-4                      # bak.py:29
_RANDOM_CHUNK = 32                    # sweeps per launch when the order is random


@dataclass
class SolveConfig:
    """Mirror of the reference SolveConfig (bak.py:32-46), same validation."""
    max_iter: int = 1000
    tol: float = 1e-6
    ordering: str = "cyclic"
    ordering_seed: int = 0
    record_history: bool = False

    def __post_init__(self):
        if self.max_iter < 1:
            raise ValueError(f"max_iter must be >= 1, got {self.max_iter}")
        if self.tol < 0:
            raise ValueError(f"tol must be >= 0, got {self.tol}")
        if self.ordering not in ORDERINGS:
            raise ValueError(f"unknown ordering {self.ordering!r}, expected one of {ORDERINGS}")


@dataclass
class SolveReport:
    """Mirror of the reference SolveReport (bak.py:49-57).  ``variant`` is an
    extra trailing field naming the kernel family that ran."""
    a_hat: object
    residual: object
    residual_norm_history: list | None
    sweeps_run: int
    converged: bool
    wall_time: float
    drift_warning: bool = False
    variant: str = ""


# --------------------------------------------------------------------------
# device plumbing (torch is used for memory and streams only)
# --------------------------------------------------------------------------

def _torch():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2104_12570_b200 needs a CUDA device (B200, sm_100a); there is no CPU fallback")
    return torch


def _dtype_code(np_dtype):
    return _lib.F64 if np.dtype(np_dtype) == np.float64 else _lib.F32


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


def _stream_ptr(torch, dev):
    return ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)


_PINNED_D2H_MIN = 1 << 20


def _host(t):
    """Device tensor -> numpy.  Large results go through a pinned staging
    buffer (torch's caching host allocator): a pageable D2H of a 134 MB
    residual runs at a few GB/s and was 60 ms of a C3 end-to-end solve."""
    if t.numel() * t.element_size() < _PINNED_D2H_MIN:
        return t.cpu().numpy()
    import torch
    h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    h.copy_(t, non_blocking=True)
    torch.cuda.current_stream(t.device).synchronize()
    return h.numpy()


def _is_torch(obj):
    try:
        import torch
    except ImportError:  # pragma: no cover
        return False
    return isinstance(obj, torch.Tensor)


class DeviceMatrix:
    """Column-major device copy of x with an aligned leading dimension.

    ``data`` is a (vars, ldx) row-major torch tensor, i.e. column j of x is
    data[j, :obs]; ldx*sizeof(T) is a multiple of 16 so every column (and each
    CTA's slice of it) can be moved with one cp.async.bulk.
    """

    def __init__(self, data, obs, vars_, np_dtype):
        self.data = data
        self.obs = obs
        self.vars = vars_
        self.ldx = data.shape[1]
        self.np_dtype = np.dtype(np_dtype)
        self.code = _dtype_code(np_dtype)

    @property
    def ptr(self):
        return _ptr(self.data)


def _aligned_ld(obs, itemsize):
    v = 16 // itemsize
    return (obs + v - 1) // v * v


def to_device_matrix(x, device=None):
    """Coerce like ``as_matrix`` (core.py:44-55) and upload column-major."""
    torch = _torch()
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    if isinstance(x, DeviceMatrix):
        return x
    if _is_torch(x):
        if x.ndim != 2:
            raise ValueError(f"expected a 2-d matrix, got ndim={x.ndim}")
        if x.dtype not in (torch.float32, torch.float64):
            x = x.to(torch.float64)
        obs, nv = x.shape
        np_dtype = np.float64 if x.dtype == torch.float64 else np.float32
        itemsize = 8 if np_dtype == np.float64 else 4
        ld = _aligned_ld(obs, itemsize)
        if (x.is_cuda and x.stride(0) == 1 and x.stride(1) >= obs and (x.stride(1) * itemsize) % 16 == 0
                and x.data_ptr() % 16 == 0 and x.device == dev
                and x.storage_offset() + nv * x.stride(1) <= x.untyped_storage().nbytes() // itemsize):
            # (the padded (vars, ld) view covers ld elements of the last column: only when they are
            # inside the storage, e.g. not for a row-offset slice of a larger column-major matrix)
            # zero-copy view of an existing column-major device matrix
            data = torch.as_strided(x, (nv, x.stride(1)), (x.stride(1), 1))
            return DeviceMatrix(data, obs, nv, np_dtype)
        data = torch.empty((nv, ld), dtype=x.dtype, device=dev)
        src = x.t()  # (vars, obs) view
        if ld == obs:
            data.copy_(src, non_blocking=True)
        else:
            data[:, :obs].copy_(src, non_blocking=True)
        return DeviceMatrix(data, obs, nv, np_dtype)
    xa = np.asarray(x)
    if xa.ndim != 2:
        raise ValueError(f"expected a 2-d matrix, got ndim={xa.ndim}")
    if xa.dtype not in (np.float32, np.float64):
        xa = xa.astype(np.float64)
    xa = np.asfortranarray(xa)
    obs, nv = xa.shape
    ld = _aligned_ld(obs, xa.dtype.itemsize)
    host = torch.from_numpy(xa.T)  # (vars, obs) C-contiguous view, no copy
    data = torch.empty((nv, ld), dtype=host.dtype, device=dev)
    if ld == obs:
        data.copy_(host)
    else:
        data[:, :obs].copy_(host)
    return DeviceMatrix(data, obs, nv, xa.dtype)


def _to_device_vector(v, np_dtype, dev, name="y"):
    torch = _torch()
    tdt = torch.float64 if np.dtype(np_dtype) == np.float64 else torch.float32
    if _is_torch(v):
        if v.ndim != 1:
            raise ValueError(f"expected a 1-d vector, got ndim={v.ndim}")
        return v.to(device=dev, dtype=tdt).contiguous()
    va = np.ascontiguousarray(v, dtype=np_dtype)
    if va.ndim != 1:
        raise ValueError(f"expected a 1-d vector, got ndim={va.ndim}")
    return torch.from_numpy(va).to(dev)


class _Workspace:
    """Per-device scratch owned by the call (no allocation inside the sweep)."""

    def __init__(self, torch, dev, nbytes):
        self.buf = torch.empty(max(int(nbytes), 4096), dtype=torch.uint8, device=dev)

    @property
    def ptr(self):
        return _ptr(self.buf)

    @property
    def nbytes(self):
        return self.buf.numel()


def _workspace_bytes(lib, code, obs, nv, vcode=0):
    return max(lib.bak_colnorms_workspace(code, obs, nv), lib.bak_colnorms_workspace(code, obs, 1),
               lib.bak_residual_workspace(code, obs, nv), lib.bak_sweep_workspace(code, vcode, obs, nv), 4096)


def colnorms(dm: DeviceMatrix, ws=None):
    """Device column norms n2_j = <x_j, x_j> (core.py:116-127)."""
    torch = _torch()
    lib = _lib.load()
    dev = dm.data.device
    if ws is None:
        ws = _Workspace(torch, dev, _workspace_bytes(lib, dm.code, dm.obs, dm.vars))
    out = torch.empty(dm.vars, dtype=dm.data.dtype, device=dev)
    _lib.check(lib.bak_colnorms(dm.code, dm.ptr, dm.obs, dm.vars, dm.ldx, _ptr(out), ws.ptr, ws.nbytes,
                                _stream_ptr(torch, dev)), "bak_colnorms")
    return out


def _sumsq(lib, torch, code, v, ws, st):
    out = torch.empty(1, dtype=v.dtype, device=v.device)
    _lib.check(lib.bak_colnorms(code, _ptr(v), v.numel(), 1, v.numel(), _ptr(out), ws.ptr, ws.nbytes, st),
               "bak_colnorms(y)")
    return out


def _residual(lib, dm, a, y, out, ws, st):
    _lib.check(lib.bak_residual(dm.code, dm.ptr, dm.obs, dm.vars, dm.ldx, _ptr(a), _ptr(y), _ptr(out), ws.ptr,
                                ws.nbytes, st), "bak_residual")


def _permutation_chunks(seed, nvars, nz_mask):
    """Yield the compounding per-sweep permutations of ordering='random'
    (bak.py:98-99, 181) — host-side index bookkeeping, zero-norm columns
    filtered (bak.py:101-103)."""
    gen = np.random.Generator(np.random.Philox(seed))
    order = np.arange(nvars)
    while True:
        gen.shuffle(order)
        yield order[nz_mask[order]] if nz_mask is not None else order.copy()


# "auto" for systems whose residual does not fit on chip: the exact kernel then
# streams e, x_j and x_{j+1} per column (~4 column-lengths of HBM traffic per
# column of x), the GRAM sweep reads x once per sweep after one G = X^T X
# (~8.5 passes' worth for 2^24 x 256 fp64).  GRAM meets the same parity bar
# (tests/test_fullsize_reference_gpu.py) and is reported as variant "gram".
_AUTO_GRAM_MAX_VARS = 256
_AUTO_GRAM_MIN_SWEEPS = 4


def _auto_variant(lib, x, cfg):
    """Variant "auto" resolves to: the exact on-chip kernels (CTA / cluster /
    grid) when the residual fits on chip; else GRAM when vars <= 256 and at
    least 4 sweeps are allowed; else the exact STREAM kernel."""
    if isinstance(x, DeviceMatrix):
        obs, nv, code = x.obs, x.vars, x.code
    else:
        shape = getattr(x, "shape", None)
        if shape is None or len(shape) != 2:
            return "auto"  # coerced (and rejected if not 2-d) by to_device_matrix
        obs, nv = int(shape[0]), int(shape[1])
        dt = str(getattr(x, "dtype", "float64"))
        code = _lib.F32 if dt.endswith("float32") else _lib.F64
    if obs < 1 or nv < 1:
        return "auto"
    picked = int(lib.bak_sweep_pick_variant(code, obs, nv))
    if (picked == _lib.VARIANTS["stream"] and nv <= _AUTO_GRAM_MAX_VARS
            and cfg.max_iter >= _AUTO_GRAM_MIN_SWEEPS):
        return "gram"
    return "auto"


def solve_bak(x, y, config: SolveConfig | None = None, a0=None, *, variant="auto", device=None,
              return_device=False) -> SolveReport:
    """Solve min ||y - x a|| by repeated single-column updates on the GPU.

    Same contract as the reference (bak.py:146-159): x is coerced to
    column-major float storage; zero-norm columns are skipped and keep their
    starting coefficient; a zero target returns a = 0 immediately, converged;
    convergence is checked once per sweep against tol * ||y||.
    """
    cfg = config if config is not None else SolveConfig()
    torch = _torch()
    lib = _lib.load()
    if variant not in _lib.VARIANTS:
        raise ValueError(f"unknown variant {variant!r}, expected one of {tuple(_lib.VARIANTS)}")
    if variant == "auto":
        variant = _auto_variant(lib, x, cfg)
    if variant == "bgram" and cfg.ordering != "cyclic":
        raise ValueError("variant='bgram' (block-Gram, blocks of 64 consecutive columns) supports ordering='cyclic'")
    if variant == "gram" and _pipelinable(torch, x):
        return _solve_gram_pipelined(lib, torch, x, y, cfg, a0, device, return_device)
    dm = to_device_matrix(x, device)
    dev = dm.data.device
    obs, nv, code = dm.obs, dm.vars, dm.code
    yd = _to_device_vector(y, dm.np_dtype, dev)
    if yd.shape[0] != obs:
        raise ValueError(f"y has length {yd.shape[0]}, expected {obs}")
    st = _stream_ptr(torch, dev)

    t0 = time.perf_counter()
    ws = _Workspace(torch, dev, _workspace_bytes(lib, code, obs, nv, _lib.VARIANTS[variant]))
    ynorm2 = float(_sumsq(lib, torch, code, yd, ws, st).item())
    if ynorm2 == 0.0:  # bak.py:168-170 (_zero_report)
        a_z = torch.zeros(nv, dtype=yd.dtype, device=dev)
        r_z = torch.zeros(obs, dtype=yd.dtype, device=dev)
        return SolveReport(a_hat=a_z if return_device else a_z.cpu().numpy(),
                           residual=r_z if return_device else r_z.cpu().numpy(),
                           residual_norm_history=[] if cfg.record_history else None,
                           sweeps_run=0, converged=True, wall_time=time.perf_counter() - t0)
    if a0 is not None:
        a = _to_device_vector(a0, dm.np_dtype, dev, "a0").clone()
        if a.shape[0] != nv:
            raise ValueError(f"a0 has length {a.shape[0]}, expected {nv}")
    else:
        a = torch.zeros(nv, dtype=yd.dtype, device=dev)
    thresh2 = cfg.tol * cfg.tol * ynorm2 if cfg.tol > 0 else -1.0   # bak.py:182

    if variant == "gram":
        return _solve_gram(lib, torch, dm, yd, a, a0, cfg, ynorm2, thresh2, ws, st, t0, return_device)

    norms = colnorms(dm, ws)
    norms_h = norms.cpu().numpy()
    if not norms_h.any():
        raise ValueError("every column of x has zero norm; nothing to solve")
    nz_mask = norms_h != 0
    all_nz = bool(nz_mask.all())

    e = torch.empty_like(yd)
    if a0 is not None:
        _residual(lib, dm, a, yd, e, ws, st)            # e = y - x a0 (bak.py:189)
    else:
        e.copy_(yd)
    hist = torch.zeros(cfg.max_iter, dtype=torch.float64, device=dev) if cfg.record_history else None
    status = torch.zeros(4, dtype=torch.int64, device=dev)
    vcode = _lib.VARIANTS[variant]

    sweeps = 0
    converged = False
    used = vcode
    if cfg.ordering == "cyclic":
        if all_nz:
            cols, ncols = None, nv
        else:
            cols = torch.from_numpy(np.flatnonzero(nz_mask).astype(np.int32)).to(dev)
            ncols = int(cols.numel())
        _lib.check(lib.bak_sweep(code, vcode, dm.ptr, obs, nv, dm.ldx, _ptr(norms), _ptr(cols), ncols, 0,
                                 _ptr(e), _ptr(a), cfg.max_iter, thresh2, _ptr(hist), _ptr(status),
                                 ws.ptr, ws.nbytes, st), "bak_sweep")
        stat = status.cpu().numpy()
        sweeps, converged, err, used = int(stat[0]), bool(stat[1]), int(stat[2]), int(stat[3])
        if err:
            raise _lib.BakError(f"bak_sweep device error {err} (3 = spin-wait timeout)")
    else:
        perms = _permutation_chunks(cfg.ordering_seed, nv, None if all_nz else nz_mask)
        while sweeps < cfg.max_iter and not converged:
            k = min(_RANDOM_CHUNK, cfg.max_iter - sweeps)
            block = np.stack([next(perms) for _ in range(k)]).astype(np.int32)
            cols = torch.from_numpy(block).to(dev)
            ncols = block.shape[1]
            hptr = ctypes.c_void_p(hist.data_ptr() + 8 * sweeps) if hist is not None else ctypes.c_void_p(0)
            _lib.check(lib.bak_sweep(code, vcode, dm.ptr, obs, nv, dm.ldx, _ptr(norms), _ptr(cols), ncols, ncols,
                                     _ptr(e), _ptr(a), k, thresh2, hptr, _ptr(status), ws.ptr, ws.nbytes, st),
                       "bak_sweep")
            stat = status.cpu().numpy()
            if int(stat[2]):
                raise _lib.BakError(f"bak_sweep device error {int(stat[2])}")
            sweeps += int(stat[0])
            converged = bool(stat[1])
            used = int(stat[3])

    resid = torch.empty_like(yd)
    _residual(lib, dm, a, yd, resid, ws, st)             # bak.py:130
    drift2 = torch.empty(1, dtype=torch.float64, device=dev)
    _lib.check(lib.bak_diff_norm2(code, _ptr(e), _ptr(resid), obs, _ptr(drift2), ws.ptr, ws.nbytes, st),
               "bak_diff_norm2")
    drift = float(np.sqrt(drift2.item()))
    wall = time.perf_counter() - t0                      # bak.py:131-132 (after the residual)
    drift_rel = drift / max(np.sqrt(ynorm2), np.finfo(np.float64).tiny)
    history = hist[:sweeps].cpu().tolist() if hist is not None else None
    return SolveReport(
        a_hat=a if return_device else _host(a),
        residual=resid if return_device else _host(resid),
        residual_norm_history=history,
        sweeps_run=sweeps,
        converged=converged,
        wall_time=wall,
        drift_warning=bool(drift_rel > DRIFT_TOL),
        variant=_lib.VARIANT_NAMES.get(used, str(used)),
    )


def _solve_gram(lib, torch, dm, yd, a, a0, cfg, ynorm2, thresh2, ws, st, t0, return_device):
    """variant="gram": one C call (bak_solve_gram) — G and norms, the sweeps
    (one pass over x each), and, without early break, the final residual
    fused into the last pass."""
    dev = dm.data.device
    obs, nv, code = dm.obs, dm.vars, dm.code
    e = torch.empty_like(yd)
    if a0 is not None:
        _residual(lib, dm, a, yd, e, ws, st)            # e = y - x a0 (bak.py:189)
    else:
        e.copy_(yd)
    norms = torch.empty(nv, dtype=yd.dtype, device=dev)
    hist = torch.zeros(cfg.max_iter, dtype=torch.float64, device=dev) if cfg.record_history else None
    status = torch.zeros(4, dtype=torch.int64, device=dev)
    resid = torch.empty_like(yd)
    if cfg.ordering == "cyclic":
        cols, ncols, stride = None, nv, 0
    else:
        perms = _permutation_chunks(cfg.ordering_seed, nv, None)
        block = np.stack([next(perms) for _ in range(cfg.max_iter)]).astype(np.int32)
        cols = torch.from_numpy(block).to(dev)
        ncols, stride = nv, nv
    rc = lib.bak_solve_gram(code, dm.ptr, obs, nv, dm.ldx, _ptr(yd), _ptr(cols), ncols, stride, _ptr(norms), _ptr(e),
                            _ptr(a), cfg.max_iter, thresh2, _ptr(hist), _ptr(status), _ptr(resid), ws.ptr, ws.nbytes,
                            st)
    if rc == 1 and b"zero norm" in lib.bak_last_error():
        raise ValueError("every column of x has zero norm; nothing to solve")
    _lib.check(rc, "bak_solve_gram")
    stat = status.cpu().numpy()
    if int(stat[2]):
        raise _lib.BakError(f"bak_solve_gram device error {int(stat[2])}")
    sweeps, converged = int(stat[0]), bool(stat[1])
    if not (int(stat[3]) & 256):                         # residual not fused (early break possible)
        _residual(lib, dm, a, yd, resid, ws, st)         # bak.py:130
    drift2 = torch.empty(1, dtype=torch.float64, device=dev)
    _lib.check(lib.bak_diff_norm2(code, _ptr(e), _ptr(resid), obs, _ptr(drift2), ws.ptr, ws.nbytes, st),
               "bak_diff_norm2")
    drift = float(np.sqrt(drift2.item()))
    wall = time.perf_counter() - t0
    drift_rel = drift / max(np.sqrt(ynorm2), np.finfo(np.float64).tiny)
    return SolveReport(
        a_hat=a if return_device else _host(a),
        residual=resid if return_device else _host(resid),
        residual_norm_history=hist[:sweeps].cpu().tolist() if hist is not None else None,
        sweeps_run=sweeps, converged=converged, wall_time=wall, drift_warning=bool(drift_rel > DRIFT_TOL),
        variant="gram")


_PIPE_MIN_BYTES = 256 << 20
_PIPE_CHUNK_BYTES = 1 << 30


def _pipelinable(torch, x):
    """Large PINNED host x (torch CPU tensor, column-major view): upload in row
    blocks overlapped with the first GPU work (G and the first pass)."""
    return (_is_torch(x) and not x.is_cuda and x.ndim == 2 and x.is_pinned() and x.stride(0) == 1
            and x.dtype in (torch.float32, torch.float64) and x.numel() * x.element_size() >= _PIPE_MIN_BYTES
            and x.shape[1] <= 256)


def _solve_gram_pipelined(lib, torch, x, y, cfg, a0, device, return_device):
    """variant="gram" from a pinned host matrix: row blocks of x are copied on
    two copy streams (cudaMemcpy2DAsync) while the compute stream builds each
    block's G partial and first-pass partials; sweeps 1.. run over the whole
    device matrix.  Same results as the resident path (partials summed in
    block order)."""
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    obs, nv = x.shape
    np_dtype = np.float64 if x.dtype == torch.float64 else np.float32
    ts = 8 if np_dtype == np.float64 else 4
    code = _dtype_code(np_dtype)
    ld = _aligned_ld(obs, ts)
    sld = x.stride(1)
    data = torch.empty((nv, ld), dtype=x.dtype, device=dev)
    dm = DeviceMatrix(data, obs, nv, np_dtype)
    yd = _to_device_vector(y, np_dtype, dev)
    if yd.shape[0] != obs:
        raise ValueError(f"y has length {yd.shape[0]}, expected {obs}")
    a0d = None
    if a0 is not None:  # validated before any copy is queued
        a0d = _to_device_vector(a0, np_dtype, dev, "a0").clone()
        if a0d.shape[0] != nv:
            raise ValueError(f"a0 has length {a0d.shape[0]}, expected {nv}")
    main = torch.cuda.current_stream(dev)
    st = ctypes.c_void_p(main.cuda_stream)
    t0 = time.perf_counter()
    # row blocks (multiples of 32 rows: whole TMA tiles), two copy engines
    rows_chunk = max(32, (_PIPE_CHUNK_BYTES // (nv * ts)) // 32 * 32)
    blocks = [(r0, min(obs, r0 + rows_chunk)) for r0 in range(0, obs, rows_chunk)]
    copy_streams = [torch.cuda.Stream(dev), torch.cuda.Stream(dev)]
    for cs in copy_streams:
        cs.wait_stream(main)
        # the copies write `data` on these streams: on ANY exit (an exception
        # included) the caching allocator must not hand the block out again
        # before they are done
        data.record_stream(cs)
    events = []
    for i, (r0, r1) in enumerate(blocks):
        cs = copy_streams[i % 2]
        _lib.check(lib.bak_copy_rows_h2d(dm.ptr, ld, ctypes.c_void_p(x.data_ptr()), sld, r0, r1 - r0, nv, ts,
                                         ctypes.c_void_p(cs.cuda_stream)), "bak_copy_rows_h2d")
        ev = torch.cuda.Event()
        ev.record(cs)
        events.append(ev)
    wsb = max(lib.bak_gram_matrix_workspace(code, rows_chunk, nv), lib.bak_residual_workspace(code, obs, nv),
              lib.bak_colnorms_workspace(code, obs, 1), 1 << 16)
    ws = _Workspace(torch, dev, wsb)
    ynorm2 = float(_sumsq(lib, torch, code, yd, ws, st).item())
    if ynorm2 == 0.0:
        for ev in events:
            main.wait_event(ev)
        a_z = torch.zeros(nv, dtype=yd.dtype, device=dev)
        r_z = torch.zeros(obs, dtype=yd.dtype, device=dev)
        return SolveReport(a_z if return_device else a_z.cpu().numpy(), r_z if return_device else r_z.cpu().numpy(),
                           [] if cfg.record_history else None, 0, True, time.perf_counter() - t0)
    a = a0d if a0d is not None else torch.zeros(nv, dtype=yd.dtype, device=dev)
    thresh2 = cfg.tol * cfg.tol * ynorm2 if cfg.tol > 0 else -1.0
    e = yd.clone()
    nblk = lib.bak_gram_pass_blocks(code, nv)
    nb = len(blocks)
    g0rows = max(lib.bak_gram_dot_rows(code, r1 - r0, nv) for r0, r1 in blocks)
    Gp = torch.empty((nb, nv, nv), dtype=torch.float64, device=dev)
    gp0 = torch.zeros((nb, g0rows, nv), dtype=torch.float64, device=dev)
    sp0 = torch.zeros((nb, 1), dtype=torch.float64, device=dev)  # unused by the first solve
    ctrl = torch.zeros(4, dtype=torch.int64, device=dev)
    delta = torch.zeros(nv, dtype=torch.float64, device=dev)
    for i, (r0, r1) in enumerate(blocks):
        main.wait_event(events[i])
        xb = ctypes.c_void_p(dm.data.data_ptr() + r0 * ts)
        eb = ctypes.c_void_p(e.data_ptr() + r0 * ts)
        if a0 is not None:  # e = y - x a0 on this block (bak.py:189)
            _lib.check(lib.bak_residual(code, xb, r1 - r0, nv, ld, _ptr(a), ctypes.c_void_p(yd.data_ptr() + r0 * ts),
                                        eb, ws.ptr, ws.nbytes, st), "bak_residual")
        # this block's G and first-sweep g = X^T e in one read of the block
        _lib.check(lib.bak_gram_matrix_dot(code, xb, r1 - r0, nv, ld, _ptr(Gp[i]), eb, _ptr(gp0[i]),
                                           ws.ptr, ws.nbytes, st), "bak_gram_matrix_dot")
    G = Gp[0].clone()
    for i in range(1, nb):
        G += Gp[i]
    norms = G.diagonal().to(yd.dtype).contiguous()
    norms_h = norms.cpu().numpy()
    if not norms_h.any():
        raise ValueError("every column of x has zero norm; nothing to solve")
    hist = torch.zeros(cfg.max_iter, dtype=torch.float64, device=dev) if cfg.record_history else None
    status = torch.zeros(4, dtype=torch.int64, device=dev)
    if cfg.ordering == "cyclic":
        cols, ncols, stride = None, nv, 0
    else:
        perms = _permutation_chunks(cfg.ordering_seed, nv, None)
        block = np.stack([next(perms) for _ in range(cfg.max_iter)]).astype(np.int32)
        cols = torch.from_numpy(block).to(dev)
        ncols, stride = nv, nv
    gpart = torch.zeros((nblk, nv), dtype=torch.float64, device=dev)
    sqpart = torch.zeros(nblk, dtype=torch.float64, device=dev)
    resid = torch.empty_like(yd)
    fused = thresh2 < 0

    def solve(gp, sp, sweep):
        _lib.check(lib.bak_gram_solve(code, nv, _ptr(gp), _ptr(sp), gp.numel() // nv, sweep, cfg.max_iter, thresh2,
                                      _ptr(cols), ncols, stride, _ptr(norms), _ptr(G), _ptr(a), _ptr(delta),
                                      _ptr(hist), _ptr(ctrl), _ptr(status), st), "bak_gram_solve")

    def full_pass(dot, last):
        afin = a if (last and fused) else None
        _lib.check(lib.bak_gram_pass_resid(code, dm.ptr, obs, nv, ld, _ptr(e), _ptr(delta), 1, dot, _ptr(gpart),
                                           _ptr(sqpart), _ptr(ctrl), _ptr(afin), _ptr(yd if afin is not None else None),
                                           _ptr(resid if afin is not None else None), _ptr(status), st),
                   "bak_gram_pass")

    gp, sp = gp0.reshape(-1), sp0.reshape(-1)
    for sweep in range(1, cfg.max_iter + 1):
        solve(gp, sp, sweep)
        full_pass(1 if sweep < cfg.max_iter else 0, sweep == cfg.max_iter)
        gp, sp = gpart.reshape(-1), sqpart
        if thresh2 >= 0 and sweep % 16 == 0 and int(ctrl[0].item()):
            break
    solve(gp, sp, cfg.max_iter + 1)
    stat = status.cpu().numpy()
    if int(stat[2]):
        raise _lib.BakError(f"GRAM device error {int(stat[2])} (3 = pipeline timeout)")
    sweeps, converged = int(stat[0]), bool(stat[1])
    if not fused:
        _residual(lib, dm, a, yd, resid, ws, st)
    drift2 = torch.empty(1, dtype=torch.float64, device=dev)
    _lib.check(lib.bak_diff_norm2(code, _ptr(e), _ptr(resid), obs, _ptr(drift2), ws.ptr, ws.nbytes, st),
               "bak_diff_norm2")
    drift = float(np.sqrt(drift2.item()))
    wall = time.perf_counter() - t0
    return SolveReport(
        a_hat=a if return_device else _host(a),
        residual=resid if return_device else _host(resid),
        residual_norm_history=hist[:sweeps].cpu().tolist() if hist is not None else None,
        sweeps_run=sweeps, converged=converged, wall_time=wall,
        drift_warning=bool(drift / max(np.sqrt(ynorm2), np.finfo(np.float64).tiny) > DRIFT_TOL),
        variant="gram")


def residual_norm(e) -> float:
    """sum(e^2) (bak.py:60-63), computed on the GPU."""
    torch = _torch()
    lib = _lib.load()
    ea = e if _is_torch(e) else np.asarray(e)
    np_dtype = np.float64 if (str(getattr(ea, "dtype", "")) in ("float64", "torch.float64")) else np.float32
    if not _is_torch(ea) and ea.dtype not in (np.float32, np.float64):
        np_dtype = np.float64
    dev = torch.device("cuda", torch.cuda.current_device())
    v = _to_device_vector(ea, np_dtype, dev)
    if v.numel() == 0:
        return 0.0
    code = _dtype_code(np_dtype)
    ws = _Workspace(torch, dev, max(lib.bak_colnorms_workspace(code, v.numel(), 1), 4096))
    return float(_sumsq(lib, torch, code, v, ws, _stream_ptr(torch, dev)).item())


def coordinate_update(col, e):
    """One least-squares update along a single column (bak.py:66-79), run as
    a one-column, one-sweep solve on the GPU.  Zero column: (0.0, e) with e
    returned unchanged (the same object)."""
    torch = _torch()
    lib = _lib.load()
    col_a = np.asarray(col)
    e_a = np.asarray(e)
    np_dtype = np.result_type(col_a.dtype, e_a.dtype)
    if np_dtype not in (np.float32, np.float64):
        np_dtype = np.float64
    dm = to_device_matrix(col_a.astype(np_dtype).reshape(-1, 1))
    dev = dm.data.device
    st = _stream_ptr(torch, dev)
    ws = _Workspace(torch, dev, _workspace_bytes(lib, dm.code, dm.obs, 1))
    norms = colnorms(dm, ws)
    if float(norms.item()) == 0.0:
        return 0.0, e
    ed = _to_device_vector(e_a, np_dtype, dev)
    a = torch.zeros(1, dtype=ed.dtype, device=dev)
    status = torch.zeros(4, dtype=torch.int64, device=dev)
    _lib.check(lib.bak_sweep(dm.code, 0, dm.ptr, dm.obs, 1, dm.ldx, _ptr(norms), None, 1, 0, _ptr(ed), _ptr(a),
                             1, -1.0, None, _ptr(status), ws.ptr, ws.nbytes, st), "bak_sweep")
    return float(a.item()), ed.cpu().numpy()


# --------------------------------------------------------------------------
# (4) batched many-small-systems solve — no reference counterpart: the
# reference's equivalent is a Python loop of solve_bak calls, one per system.
# --------------------------------------------------------------------------

@dataclass
class BatchSolveReport:
    """Per-system results of solve_bak_batched; ``report(s)`` gives system s
    as a reference-shaped SolveReport."""
    a_hat: object                 # (nsys, vars)
    residual: object              # (nsys, obs)
    residual_norm_history: object  # (nsys, max_iter) float64 (valid prefix: sweeps_run[s]) or None
    sweeps_run: np.ndarray
    converged: np.ndarray
    wall_time: float
    drift_warning: np.ndarray

    def report(self, s) -> SolveReport:
        hist = None
        if self.residual_norm_history is not None:
            hist = [float(v) for v in np.asarray(self.residual_norm_history[s][: int(self.sweeps_run[s])])]
        return SolveReport(a_hat=self.a_hat[s], residual=self.residual[s], residual_norm_history=hist,
                           sweeps_run=int(self.sweeps_run[s]), converged=bool(self.converged[s]),
                           wall_time=self.wall_time, drift_warning=bool(self.drift_warning[s]), variant="batched")


class DeviceBatch:
    """Device layout of a batch: data[s, j, :obs] is column j of system s
    (each system column-major and contiguous, ld aligned to 16 bytes)."""

    def __init__(self, data, obs, np_dtype):
        self.data = data
        self.nsys, self.vars, self.ldx = data.shape
        self.obs = obs
        self.np_dtype = np.dtype(np_dtype)
        self.code = _dtype_code(np_dtype)


def to_device_batch(xs, device=None):
    """xs: (nsys, obs, vars) numpy array / torch tensor (any strides) or a DeviceBatch."""
    torch = _torch()
    if isinstance(xs, DeviceBatch):
        return xs
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    if not _is_torch(xs):
        xa = np.asarray(xs)
        if xa.ndim != 3:
            raise ValueError(f"expected a 3-d batch (nsys, obs, vars), got ndim={xa.ndim}")
        if xa.dtype not in (np.float32, np.float64):
            xa = xa.astype(np.float64)
        xs = torch.from_numpy(np.ascontiguousarray(xa.transpose(0, 2, 1)))  # (nsys, vars, obs)
        src = xs
    else:
        if xs.ndim != 3:
            raise ValueError(f"expected a 3-d batch (nsys, obs, vars), got ndim={xs.ndim}")
        if xs.dtype not in (torch.float32, torch.float64):
            xs = xs.to(torch.float64)
        src = xs.transpose(1, 2)
    nsys, nv, obs = src.shape
    np_dtype = np.float64 if src.dtype == torch.float64 else np.float32
    ld = _aligned_ld(obs, np.dtype(np_dtype).itemsize)
    data = torch.empty((nsys, nv, ld), dtype=src.dtype, device=dev)
    if ld == obs:
        data.copy_(src, non_blocking=True)
    else:
        data[:, :, :obs].copy_(src, non_blocking=True)
    return DeviceBatch(data, obs, np_dtype)


def solve_bak_batched(xs, ys, config: SolveConfig | None = None, a0=None, *, device=None,
                      return_device=False) -> BatchSolveReport:
    """Solve nsys independent systems, one CTA each (SolveConfig applies to all).

    Per system the semantics are those of solve_bak: cyclic order only
    (ordering="random" is rejected), zero-norm columns skipped, zero targets
    short-circuit, early break per sweep, residual recomputed, drift flagged.
    """
    cfg = config if config is not None else SolveConfig()
    if cfg.ordering != "cyclic":
        raise ValueError("solve_bak_batched supports ordering='cyclic' only")
    torch = _torch()
    lib = _lib.load()
    if _batch_pipelinable(torch, xs, ys) and a0 is None:
        return _solve_batched_pipelined(lib, torch, xs, ys, cfg, device, return_device)
    db = to_device_batch(xs, device)
    dev = db.data.device
    nsys, nv, obs, ld, code = db.nsys, db.vars, db.obs, db.ldx, db.code
    tdt = db.data.dtype
    yd = ys if (_is_torch(ys) and ys.is_cuda) else torch.as_tensor(np.asarray(ys, dtype=db.np_dtype))
    yd = yd.to(device=dev, dtype=tdt).reshape(nsys, -1).contiguous()
    if yd.shape[1] != obs:
        raise ValueError(f"y has length {yd.shape[1]}, expected {obs}")
    st = _stream_ptr(torch, dev)
    t0 = time.perf_counter()
    wsb = max(lib.bak_colnorms_workspace(code, obs, nsys * nv), lib.bak_colnorms_workspace(code, obs, nsys), 4096)
    ws = _Workspace(torch, dev, wsb)
    norms = torch.empty(nsys * nv, dtype=tdt, device=dev)
    _lib.check(lib.bak_colnorms(code, _ptr(db.data), obs, nsys * nv, ld, _ptr(norms), ws.ptr, ws.nbytes, st),
               "bak_colnorms")
    yn = torch.empty(nsys, dtype=tdt, device=dev)
    _lib.check(lib.bak_colnorms(code, _ptr(yd), obs, nsys, obs, _ptr(yn), ws.ptr, ws.nbytes, st), "bak_colnorms(y)")
    ynorm2 = yn.to(torch.float64)
    if a0 is not None:
        a = torch.as_tensor(a0).to(device=dev, dtype=tdt).reshape(nsys, nv).contiguous().clone()
    else:
        a = torch.zeros((nsys, nv), dtype=tdt, device=dev)
    resid = torch.empty((nsys, obs), dtype=tdt, device=dev)
    hist = torch.zeros((nsys, cfg.max_iter), dtype=torch.float64, device=dev) if cfg.record_history else None
    status = torch.zeros((nsys, 4), dtype=torch.int64, device=dev)
    _lib.check(lib.bak_solve_batched(code, _ptr(db.data), obs, nv, ld, nv * ld, nsys, _ptr(yd), obs, _ptr(norms),
                                     _ptr(ynorm2), _ptr(a), 1 if a0 is not None else 0, _ptr(resid), cfg.max_iter,
                                     float(cfg.tol), DRIFT_TOL, _ptr(hist), _ptr(status), st), "bak_solve_batched")
    stat = status.cpu().numpy()
    wall = time.perf_counter() - t0
    bad = stat[:, 3]
    if np.any(bad == 1):
        raise ValueError("every column of x has zero norm; nothing to solve "
                         f"(systems {np.flatnonzero(bad == 1)[:8].tolist()})")
    if np.any(bad):
        raise _lib.BakError(f"bak_solve_batched device error {int(bad[bad != 0][0])}")
    return BatchSolveReport(
        a_hat=a if return_device else _host(a),
        residual=resid if return_device else _host(resid),
        residual_norm_history=(hist if return_device else hist.cpu().numpy()) if hist is not None else None,
        sweeps_run=stat[:, 0].copy(), converged=stat[:, 1].astype(bool), wall_time=wall,
        drift_warning=stat[:, 2].astype(bool))


_BATCH_PIPE_MIN_BYTES = 256 << 20
_BATCH_PIPE_CHUNKS = 8


def _batch_pipelinable(torch, xs, ys):
    """Large PINNED host batch (torch CPU tensor (nsys, obs, vars) whose
    (nsys, vars, obs) transpose is contiguous with 16-byte aligned columns)."""
    if not (_is_torch(xs) and not xs.is_cuda and xs.ndim == 3 and xs.is_pinned()):
        return False
    if xs.dtype not in (torch.float32, torch.float64) or xs.numel() * xs.element_size() < _BATCH_PIPE_MIN_BYTES:
        return False
    src = xs.transpose(1, 2)
    if not src.is_contiguous() or (src.shape[2] * src.element_size()) % 16:
        return False
    return _is_torch(ys) and not ys.is_cuda and ys.is_pinned() and ys.dtype == xs.dtype and ys.is_contiguous()


def _solve_batched_pipelined(lib, torch, xs, ys, cfg, device, return_device):
    """solve_bak_batched from pinned host memory: the systems are split into
    chunks; chunk k+1 is uploaded on a copy stream while chunk k is solved on
    the compute stream, and chunk k's results go back on a third stream — the
    upload (PCIe) and the solve (HBM) overlap instead of adding up.  Same
    kernels, same per-system results as the resident path."""
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    src = xs.transpose(1, 2)                       # (nsys, vars, obs), contiguous, pinned
    nsys, nv, obs = src.shape
    np_dtype = np.float64 if src.dtype == torch.float64 else np.float32
    code = _dtype_code(np_dtype)
    tdt = src.dtype
    yh = ys.reshape(nsys, -1)
    if yh.shape[1] != obs:
        raise ValueError(f"y has length {yh.shape[1]}, expected {obs}")
    main = torch.cuda.current_stream(dev)
    h2d, d2h = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    h2d.wait_stream(main)
    t0 = time.perf_counter()
    data = torch.empty((nsys, nv, obs), dtype=tdt, device=dev)
    yd = torch.empty((nsys, obs), dtype=tdt, device=dev)
    norms = torch.empty(nsys * nv, dtype=tdt, device=dev)
    yn = torch.empty(nsys, dtype=tdt, device=dev)
    a = torch.zeros((nsys, nv), dtype=tdt, device=dev)
    resid = torch.empty((nsys, obs), dtype=tdt, device=dev)
    hist = torch.zeros((nsys, cfg.max_iter), dtype=torch.float64, device=dev) if cfg.record_history else None
    status = torch.zeros((nsys, 4), dtype=torch.int64, device=dev)
    out_a = torch.empty((nsys, nv), dtype=tdt, pin_memory=True) if not return_device else None
    out_r = torch.empty((nsys, obs), dtype=tdt, pin_memory=True) if not return_device else None
    # chunks in whole waves of the batched kernel (systems in flight at once):
    # a partial last wave per chunk costs nearly a full wave.  Chunk sizes grow
    # 1, 2, 4, ... waves up to ~nsys/8 so the solve starts after a short upload
    # and each next upload finishes before the solve of the chunk before it
    wave = int(lib.bak_solve_batched_wave(code, obs, nv))
    if wave > 0:
        k = max(1, (nsys // _BATCH_PIPE_CHUNKS) // wave)
        sizes, w = [], 1
        while sum(sizes) < nsys:
            sizes.append(min(w * wave, nsys - sum(sizes)))
            w = min(2 * w, k)
    else:
        sizes = [-(-nsys // _BATCH_PIPE_CHUNKS)] * _BATCH_PIPE_CHUNKS
    chunks, s0 = [], 0
    for n in sizes:
        if s0 < nsys:
            chunks.append((s0, min(nsys, s0 + n)))
            s0 += n
    per = max(s1 - s0 for s0, s1 in chunks)
    wsb = max(lib.bak_colnorms_workspace(code, obs, per * nv), lib.bak_colnorms_workspace(code, obs, per), 4096)
    ws = _Workspace(torch, dev, wsb)
    st = ctypes.c_void_p(main.cuda_stream)
    events = []
    for s0, s1 in chunks:
        with torch.cuda.stream(h2d):
            data[s0:s1].copy_(src[s0:s1], non_blocking=True)
            yd[s0:s1].copy_(yh[s0:s1], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(h2d)
            events.append(ev)
    done = []
    for (s0, s1), ev in zip(chunks, events):
        main.wait_event(ev)
        n = s1 - s0
        xp = ctypes.c_void_p(data[s0].data_ptr())
        _lib.check(lib.bak_colnorms(code, xp, obs, n * nv, obs, _ptr(norms[s0 * nv:s1 * nv]), ws.ptr, ws.nbytes, st),
                   "bak_colnorms")
        _lib.check(lib.bak_colnorms(code, _ptr(yd[s0]), obs, n, obs, _ptr(yn[s0:s1]), ws.ptr, ws.nbytes, st),
                   "bak_colnorms(y)")
        ynorm2 = yn[s0:s1].to(torch.float64)
        _lib.check(lib.bak_solve_batched(code, xp, obs, nv, obs, nv * obs, n, _ptr(yd[s0]), obs,
                                         _ptr(norms[s0 * nv:s1 * nv]), _ptr(ynorm2), _ptr(a[s0]), 0,
                                         _ptr(resid[s0]), cfg.max_iter, float(cfg.tol), DRIFT_TOL,
                                         _ptr(hist[s0]) if hist is not None else None, _ptr(status[s0]), st),
                   "bak_solve_batched")
        if out_a is not None:
            ev2 = torch.cuda.Event()
            ev2.record(main)
            d2h.wait_event(ev2)
            with torch.cuda.stream(d2h):
                out_a[s0:s1].copy_(a[s0:s1], non_blocking=True)
                out_r[s0:s1].copy_(resid[s0:s1], non_blocking=True)
        done.append(ynorm2)  # keep the per-chunk temporaries alive until the stream syncs
    main.wait_stream(d2h)
    stat = status.cpu().numpy()
    torch.cuda.current_stream(dev).synchronize()
    wall = time.perf_counter() - t0
    bad = stat[:, 3]
    if np.any(bad == 1):
        raise ValueError("every column of x has zero norm; nothing to solve "
                         f"(systems {np.flatnonzero(bad == 1)[:8].tolist()})")
    if np.any(bad):
        raise _lib.BakError(f"bak_solve_batched device error {int(bad[bad != 0][0])}")
    return BatchSolveReport(
        a_hat=a if return_device else out_a.numpy(),
        residual=resid if return_device else out_r.numpy(),
        residual_norm_history=(hist if return_device else hist.cpu().numpy()) if hist is not None else None,
        sweeps_run=stat[:, 0].copy(), converged=stat[:, 1].astype(bool), wall_time=wall,
        drift_warning=stat[:, 2].astype(bool))

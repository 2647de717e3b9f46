"""Python front for the C/OpenMP oracle port (bak_oracle.c).  Test/baseline
infrastructure only: used by bench.py's reference arm to time the reference
algorithm with all host threads, and checked against the numpy oracle."""

import ctypes
import os

import numpy as np

from . import build_c

_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = build_c.load()
    return _lib


def threads():
    return int(lib().bako_max_threads())


def solve(x, y, max_iter, tol=0.0, nthreads=None, record_history=False):
    """Cyclic SolveBak sweeps on one system; returns (a, e, sweeps, converged, history)."""
    x = np.asfortranarray(x)
    suf = "f64" if x.dtype == np.float64 else "f32"
    e = np.array(y, dtype=x.dtype, copy=True)
    a = np.zeros(x.shape[1], dtype=x.dtype)
    n2 = np.einsum("ij,ij->j", x, x).astype(x.dtype)
    ynorm2 = float(np.dot(e, e))
    thresh2 = tol * tol * ynorm2 if tol > 0 else -1.0
    hist = np.zeros(max_iter) if record_history else None
    sw = ctypes.c_int64(0)
    cv = ctypes.c_int(0)
    nt = nthreads or threads()
    getattr(lib(), "bako_solve_" + suf)(
        x.ctypes.data, x.shape[0], x.shape[1], x.shape[0], e.ctypes.data, a.ctypes.data, n2.ctypes.data,
        max_iter, thresh2, hist.ctypes.data if hist is not None else None, ctypes.byref(sw), ctypes.byref(cv), nt)
    return a, e, int(sw.value), bool(cv.value), (hist[: sw.value].tolist() if hist is not None else None)


def solve_batched(xs, ys, max_iter, nthreads=None):
    """xs: (nsys, vars, ld) contiguous (column j of system s = xs[s, j, :obs]); ys: (nsys, obs)."""
    suf = "f64" if xs.dtype == np.float64 else "f32"
    nsys, nv, ld = xs.shape
    obs = ys.shape[1]
    e = np.array(ys, dtype=xs.dtype, copy=True, order="C")
    a = np.zeros((nsys, nv), dtype=xs.dtype)
    n2 = np.einsum("sjk,sjk->sj", xs[:, :, :obs], xs[:, :, :obs]).astype(xs.dtype)
    getattr(lib(), "bako_solve_batched_" + suf)(
        np.ascontiguousarray(xs).ctypes.data, obs, nv, ld, nv * ld, nsys, e.ctypes.data, obs, a.ctypes.data,
        n2.ctypes.data, max_iter, nthreads or threads())
    return a, e


def solve_block(x, y, thr, max_iter, tol=0.0, nthreads=None):
    """Blocked sweeps (solve_bakp); returns (a, e, sweeps, converged, history, diverged)."""
    x = np.asfortranarray(x)
    suf = "f64" if x.dtype == np.float64 else "f32"
    e = np.array(y, dtype=x.dtype, copy=True)
    a = np.zeros(x.shape[1], dtype=x.dtype)
    n2 = np.einsum("ij,ij->j", x, x).astype(x.dtype)
    ynorm2 = float(np.dot(e, e))
    thresh2 = tol * tol * ynorm2 if tol > 0 else -1.0
    hist = np.zeros(max_iter)
    sw = ctypes.c_int64(0)
    cv = ctypes.c_int(0)
    div = getattr(lib(), "bako_solve_block_" + suf)(
        x.ctypes.data, x.shape[0], x.shape[1], x.shape[0], e.ctypes.data, a.ctypes.data, n2.ctypes.data,
        int(thr), max_iter, ctypes.c_double(thresh2), ctypes.c_double(ynorm2), hist.ctypes.data, ctypes.byref(sw),
        ctypes.byref(cv), nthreads or threads())
    return a, e, int(sw.value), bool(cv.value), hist[: sw.value].tolist(), bool(div)

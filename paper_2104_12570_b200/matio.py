"""Matrix files of ``baksolve.matio`` (reference matio.py:1-100; SURVEY §8f
row 4) with a B200 path for big systems.

Same names, layout and errors as the reference:
    save_matrix(path, x, format="binary"), load_matrix(path, format=None),
    load_vector(path, format=None), MatrixFormatError, MAGIC, FORMATS
Binary layout (matio.py:3-5): 16-byte little-endian header {"BAKM", u32 rows,
u32 cols, u32 precision tag 32|64}, then the scalars column-major.

B200 extensions:
    load_matrix_pinned(path) -> torch CPU tensor (rows, cols), PINNED,
        column-major view (stride (1, rows)); the file body is read straight
        into it by the native parallel reader (``bak_file_read``), no numpy
        intermediate.  Passing it to ``solve_bak(..., variant="gram")`` takes
        the pipelined upload (row blocks on two copy streams overlapped with
        the first GPU work).
    load_matrix_device(path, device=None) -> DeviceMatrix (16-byte aligned
        columns), uploaded from the pinned buffer with one pitched copy.
CSV stays host-side text I/O (not a GPU path).
"""

from __future__ import annotations

import ctypes
import os
import struct

import numpy as np

from . import _lib

MAGIC = b"BAKM"
_HEADER = struct.Struct("<4sIII")
_TAG_TO_DTYPE = {32: np.dtype(np.float32), 64: np.dtype(np.float64)}
_DTYPE_TO_TAG = {v: k for k, v in _TAG_TO_DTYPE.items()}
FORMATS = ("csv", "binary")


class MatrixFormatError(ValueError):
    """Unreadable or inconsistent matrix file content (matio.py:25-26)."""


def _as_matrix(x):
    # core.py:44-55: F-ordered float32/float64, ints -> float64
    if hasattr(x, "detach"):
        x = x.detach().cpu().numpy()
    x = np.asarray(x)
    if x.ndim != 2:
        raise ValueError(f"expected a 2-d matrix, got ndim={x.ndim}")
    if x.dtype not in (np.float32, np.float64):
        x = x.astype(np.float64)
    return np.asfortranarray(x)


def save_matrix(path, x, format="binary"):
    """Write a matrix; binary preserves bits, CSV keeps full decimal precision (matio.py:29-39)."""
    x = _as_matrix(x)
    if format == "binary":
        with open(path, "wb") as f:
            f.write(_HEADER.pack(MAGIC, x.shape[0], x.shape[1], _DTYPE_TO_TAG[x.dtype]))
            f.write(x.tobytes(order="F"))
    elif format == "csv":
        np.savetxt(path, x, delimiter=",", fmt="%.17g")
    else:
        raise ValueError(f"unknown format {format!r}, expected one of {FORMATS}")


def _header(path):
    """(rows, cols, dtype) from the native header reader, matio's messages."""
    lib = _lib.load()
    rows, cols = ctypes.c_int64(), ctypes.c_int64()
    tag, size = ctypes.c_int(), ctypes.c_int64()
    rc = lib.bak_bakm_header(os.fsencode(str(path)), ctypes.byref(rows), ctypes.byref(cols), ctypes.byref(tag),
                             ctypes.byref(size))
    if rc != 0:
        msg = lib.bak_last_error().decode(errors="replace")
        if msg.endswith("bad magic"):
            with open(path, "rb") as f:
                msg = f"{path}: bad magic {f.read(4)!r}"                 # matio.py:48-49
        raise MatrixFormatError(msg)
    dtype = _TAG_TO_DTYPE[tag.value]
    if size.value - _HEADER.size < rows.value * cols.value * dtype.itemsize:
        raise MatrixFormatError(f"{path}: expected {rows.value * cols.value} scalars, file is short")
    return rows.value, cols.value, dtype


def _read_into(path, ptr, nbytes):
    lib = _lib.load()
    rc = lib.bak_file_read(os.fsencode(str(path)), _HEADER.size, ctypes.c_void_p(ptr), int(nbytes), 0)
    if rc != 0:
        raise MatrixFormatError(lib.bak_last_error().decode(errors="replace"))


def _load_binary(path):
    rows, cols, dtype = _header(path)
    out = np.empty((rows, cols), dtype=dtype, order="F")
    _read_into(path, out.ctypes.data, out.nbytes)
    return out


def _load_csv(path):
    """Comma-separated text -> float64 F-order matrix; blank lines skipped,
    every row as wide as the first (matio.py:60-80 messages)."""
    with open(path, "r", encoding="utf-8") as fh:
        numbered = [(n, text.strip()) for n, text in enumerate(fh, start=1)]
    rows = [(n, text.split(",")) for n, text in numbered if text]
    if not rows:
        raise MatrixFormatError(f"{path}: no rows")
    width = len(rows[0][1])
    values = np.empty((len(rows), width), dtype=np.float64)
    for i, (n, fields) in enumerate(rows):
        if len(fields) != width:
            raise MatrixFormatError(f"{path}: row {n} has {len(fields)} values, expected {width}")
        try:
            values[i] = [float(v) for v in fields]
        except ValueError:
            raise MatrixFormatError(f"{path}: row {n} has a non-numeric value") from None
    return np.asfortranarray(values)


def _sniff(path, format):
    """Explicit format, else binary when the file starts with the magic."""
    if format is None:
        with open(path, "rb") as fh:
            return "binary" if fh.read(len(MAGIC)) == MAGIC else "csv"
    if format in FORMATS:
        return format
    raise ValueError(f"unknown format {format!r}, expected one of {FORMATS}")


def load_matrix(path, format=None):
    """Read a matrix; format=None sniffs binary by its magic, else CSV (matio.py:83-92)."""
    format = _sniff(path, format)
    return _load_binary(path) if format == "binary" else _load_csv(path)


def load_vector(path, format=None):
    """Read a single-column (or single-row) matrix file as a vector (matio.py:95-100)."""
    m = load_matrix(path, format)
    if m.shape[1] == 1 or m.shape[0] == 1:
        return np.ascontiguousarray(m).reshape(-1)
    raise MatrixFormatError(f"{path}: expected a vector, got shape {m.shape}")


def load_matrix_pinned(path):
    """BAKM file -> pinned torch CPU tensor (rows, cols), column-major view."""
    import torch
    rows, cols, dtype = _header(path)
    tdt = torch.float64 if dtype == np.float64 else torch.float32
    buf = torch.empty((cols, rows), dtype=tdt, pin_memory=torch.cuda.is_available())
    _read_into(path, buf.data_ptr(), buf.numel() * buf.element_size())
    return buf.t()


def load_matrix_device(path, device=None):
    """BAKM file -> DeviceMatrix (pinned staging, one pitched H2D copy)."""
    from .bak import to_device_matrix
    return to_device_matrix(load_matrix_pinned(path), device)

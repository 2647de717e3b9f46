"""ctypes binding of libbak200.so (include/bak200.h).

Loading is strict: if the in-tree library is missing the import of the solver
raises — there is no CPU fallback anywhere in this package.
"""

from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# BAK_LIB_PATH: A/B tuning runs load an alternative build of the same ABI
LIB_PATH = os.environ.get("BAK_LIB_PATH") or os.path.join(_HERE, "libbak200.so")

F32, F64 = 0, 1
EDIVERGED = 6  # device status: the blocked sweep's divergence guard tripped
VARIANTS = {"auto": 0, "cta": 1, "cluster": 2, "grid": 3, "stream": 4, "gram": 5, "bgram": 6}
VARIANT_NAMES = {v: k for k, v in VARIANTS.items()}

_i64 = ctypes.c_int64
_vp = ctypes.c_void_p
_int = ctypes.c_int
_dbl = ctypes.c_double

# name -> (restype, argtypes); mirrors include/bak200.h one to one
SIGNATURES = {
    "bak_last_error": (ctypes.c_char_p, []),
    "bak_version": (ctypes.c_char_p, []),
    "bak_device_sm_count": (_int, []),
    "bak_launch_count": (_i64, []),
    "bak_colnorms_workspace": (_i64, [_int, _i64, _i64]),
    "bak_colnorms": (_int, [_int, _vp, _i64, _i64, _i64, _vp, _vp, _i64, _vp]),
    "bak_residual_workspace": (_i64, [_int, _i64, _i64]),
    "bak_residual": (_int, [_int, _vp, _i64, _i64, _i64, _vp, _vp, _vp, _vp, _i64, _vp]),
    "bak_diff_norm2": (_int, [_int, _vp, _vp, _i64, _vp, _vp, _i64, _vp]),
    "bak_sweep_workspace": (_i64, [_int, _int, _i64, _i64]),
    "bak_sweep": (_int, [_int, _int, _vp, _i64, _i64, _i64, _vp, _vp, _i64, _i64, _vp, _vp, _i64, _dbl,
                         _vp, _vp, _vp, _i64, _vp]),
    "bak_sweep_pick_variant": (_int, [_int, _i64, _i64]),
    "bak_solve_batched_wave": (_i64, [_int, _i64, _i64]),
    "bak_solve_batched": (_int, [_int, _vp, _i64, _i64, _i64, _i64, _i64, _vp, _i64, _vp, _vp, _vp, _int, _vp,
                                 _i64, _dbl, _dbl, _vp, _vp, _vp]),
    "bak_gram_pass_blocks": (_int, [_int, _i64]),
    "bak_gram_matrix_workspace": (_i64, [_int, _i64, _i64]),
    "bak_gram_matrix": (_int, [_int, _vp, _i64, _i64, _i64, _vp, _vp, _i64, _vp]),
    "bak_gram_dot_rows": (_i64, [_int, _i64, _i64]),
    "bak_block_pick_variant": (_int, [_int, _i64, _i64, _i64]),
    "bak_block_sweep_workspace": (_i64, [_int, _int, _i64, _i64, _i64]),
    "bak_block_sweep": (_int, [_int, _int, _vp, _i64, _i64, _i64, _vp, _i64, _vp, _vp, _i64, _dbl, _dbl, _vp, _vp,
                               _vp, _i64, _vp]),
    "bak_block_deltas_workspace": (_i64, [_int, _i64]),
    "bak_score_columns_workspace": (_i64, [_int, _i64, _i64]),
    "bak_bakm_header": (_int, [ctypes.c_char_p, _vp, _vp, _vp, _vp]),
    "bak_file_read": (_int, [ctypes.c_char_p, _i64, _vp, _i64, _int]),
    "bak_score_columns": (_int, [_int, _vp, _i64, _i64, _i64, _vp, _vp, _vp, _vp, _vp, _vp, _i64, _vp]),
    "bak_block_deltas": (_int, [_int, _vp, _i64, _i64, _i64, _i64, _i64, _vp, _vp, _vp, _vp, _i64, _vp]),
    "bak_gram_matrix_dot": (_int, [_int, _vp, _i64, _i64, _i64, _vp, _vp, _vp, _vp, _i64, _vp]),
    "bak_gram_pass": (_int, [_int, _vp, _i64, _i64, _i64, _vp, _vp, _int, _int, _vp, _vp, _vp, _vp, _vp]),
    "bak_gram_pass_resid": (_int, [_int, _vp, _i64, _i64, _i64, _vp, _vp, _int, _int, _vp, _vp, _vp, _vp, _vp,
                                   _vp, _vp, _vp]),
    "bak_copy_rows_h2d": (_int, [_vp, _i64, _vp, _i64, _i64, _i64, _i64, _i64, _vp]),
    "bak_gram_solve": (_int, [_int, _i64, _vp, _vp, _i64, _i64, _i64, _dbl, _vp, _i64, _i64, _vp, _vp, _vp, _vp,
                              _vp, _vp, _vp, _vp]),
    "bak_solve_gram": (_int, [_int, _vp, _i64, _i64, _i64, _vp, _vp, _i64, _i64, _vp, _vp, _vp, _i64, _dbl, _vp,
                              _vp, _vp, _vp, _i64, _vp]),
    "bak_mailbox_bytes": (_i64, [_i64]),
    "bak_sweep_rowshard": (_int, [_int, _vp, _i64, _i64, _i64, _vp, _vp, _vp, _i64, _dbl, _vp, _vp, _int, _int,
                                  _vp, _i64, _int, _vp, _i64, _vp]),
    "bak_dev_alloc": (_int, [_i64, ctypes.POINTER(_vp)]),
    "bak_dev_free": (_int, [_vp]),
    "bak_dev_zero": (_int, [_vp, _i64]),
    "bak_ipc_get_handle": (_int, [_vp, _vp]),
    "bak_ipc_open_handle": (_int, [_vp, ctypes.POINTER(_vp)]),
    "bak_ipc_close": (_int, [_vp]),
}

_lib = None


class BakError(RuntimeError):
    """A C-ABI call returned a non-zero status."""


def load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2104_12570_b200.build` "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(rc, what):
    if rc != 0:
        msg = load().bak_last_error().decode(errors="replace")
        raise BakError(f"{what} failed with status {rc}: {msg}")

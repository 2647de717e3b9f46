"""Build the C/OpenMP port of the oracle (oracle/libbak_oracle.so).

Test/baseline infrastructure only (see bak_oracle.c).  -ffp-contract=off keeps
the residual update's two roundings (bak.py:87-88); x86-64-v3 (AVX2/FMA ISA
level, no FMA contraction) so the .so runs on any recent GPU-box host.
"""

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "bak_oracle.c")
LIB = os.path.join(HERE, "libbak_oracle.so")


def build(force=False):
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= os.path.getmtime(SRC):
        return LIB
    subprocess.check_call(["gcc", "-O3", "-march=x86-64-v3", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
                           "-fPIC", "-shared", SRC, "-o", LIB + ".tmp"])
    os.replace(LIB + ".tmp", LIB)
    return LIB


def load():
    import ctypes
    build()
    lib = ctypes.CDLL(LIB)
    vp, i64, dbl, ci = ctypes.c_void_p, ctypes.c_int64, ctypes.c_double, ctypes.c_int
    for suf in ("f64", "f32"):
        f = getattr(lib, "bako_solve_" + suf)
        f.restype = ci
        f.argtypes = [vp, i64, i64, i64, vp, vp, vp, i64, dbl, vp, ctypes.POINTER(i64), ctypes.POINTER(ci), ci]
        g = getattr(lib, "bako_solve_batched_" + suf)
        g.restype = ci
        g.argtypes = [vp, i64, i64, i64, i64, i64, vp, i64, vp, vp, i64, ci]
    for suf in ("f64", "f32"):
        h = getattr(lib, "bako_solve_block_" + suf)
        h.restype = ci
        h.argtypes = [vp, i64, i64, i64, vp, vp, vp, i64, i64, dbl, dbl, vp, ctypes.POINTER(i64),
                      ctypes.POINTER(ci), ci]
    lib.bako_max_threads.restype = ci
    return lib


if __name__ == "__main__":
    print(build(force=True))

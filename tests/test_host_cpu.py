"""CPU-only checks of the host side and the C ABI (no kernel launches)."""

import ctypes
import os
import re

import numpy as np
import pytest

import paper_2104_12570_b200 as pb
from paper_2104_12570_b200 import _lib
from paper_2104_12570_b200.bak import _permutation_chunks
from oracle import bak_oracle as orc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    with open(os.path.join(ROOT, "include", "bak200.h")) as f:
        text = f.read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(bak_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2104_12570_b200 import build
    build.build()
    lib = ctypes.CDLL(_lib.LIB_PATH)
    declared = _declared_symbols()
    assert len(declared) >= 15
    for name in declared:
        assert hasattr(lib, name), name
    assert set(declared) == set(_lib.SIGNATURES), "ctypes table out of sync with include/bak200.h"


def test_library_version_and_no_device_calls():
    lib = _lib.load()
    assert lib.bak_version().decode().startswith("bak200")
    assert lib.bak_last_error() is not None
    # pure planning queries need no device
    assert lib.bak_mailbox_bytes(8) == 2 * 8 * 32
    assert lib.bak_colnorms_workspace(1, 1000, 10) == 0
    assert lib.bak_colnorms_workspace(1, 1 << 20, 10) > 0


def test_cabi_rejects_bad_layout_without_launch():
    lib = _lib.load()
    # misaligned ldx for the bulk-copy path -> EINVAL before touching the device
    rc = lib.bak_sweep(1, 0, ctypes.c_void_p(16), 37, 9, 37, ctypes.c_void_p(16), None, 9, 0, ctypes.c_void_p(16),
                       ctypes.c_void_p(16), 1, -1.0, None, ctypes.c_void_p(16), ctypes.c_void_p(16), 1 << 20, None)
    assert rc == 1
    assert b"16" in lib.bak_last_error()
    rc = lib.bak_colnorms(7, ctypes.c_void_p(16), 4, 4, 4, ctypes.c_void_p(16), None, 0, None)
    assert rc == 1


def test_solve_config_validation_matches_reference():
    with pytest.raises(ValueError, match="max_iter must be >= 1"):
        pb.SolveConfig(max_iter=0)
    with pytest.raises(ValueError, match="tol must be >= 0"):
        pb.SolveConfig(tol=-1e-6)
    with pytest.raises(ValueError, match="unknown ordering"):
        pb.SolveConfig(ordering="sorted")
    c = pb.SolveConfig()
    assert (c.max_iter, c.tol, c.ordering, c.ordering_seed, c.record_history) == (1000, 1e-6, "cyclic", 0, False)


def test_random_permutations_match_reference_order():
    gen = _permutation_chunks(11, 25, None)
    want = orc.permutations(11, 25, 5)
    got = [next(gen) for _ in range(5)]  # materialise first: chunks must not alias
    for s in range(5):
        assert np.array_equal(got[s], want[s])
    mask = np.ones(25, bool)
    mask[[3, 7]] = False
    gen = _permutation_chunks(11, 25, mask)
    for s in range(3):
        got = next(gen)
        assert np.array_equal(got, want[s][mask[want[s]]])
        assert 3 not in got and 7 not in got


def test_no_cpu_fallback_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("device present")
    with pytest.raises(RuntimeError, match="no CPU fallback"):
        pb.solve_bak(np.eye(3), np.ones(3))


def test_product_package_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2104_12570_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh")):
                with open(os.path.join(dirpath, f)) as fh:
                    assert "oracle" not in fh.read().replace("oracle/", ""), f


def test_block_config_validation_cpu():
    """BlockConfig mirrors bakp.py:39-49 (pure host logic)."""
    from paper_2104_12570_b200 import BlockConfig, SolveConfig
    assert BlockConfig().thr == 1 and BlockConfig().worker_count == 0
    assert isinstance(BlockConfig().base, SolveConfig)
    with pytest.raises(ValueError):
        BlockConfig(thr=0)
    with pytest.raises(ValueError):
        BlockConfig(worker_count=-1)


def test_divergence_first_sweep_logic_cpu():
    from paper_2104_12570_b200.bakp import _divergence_message, _first_divergence
    assert _first_divergence([5.0, 4.0, 3.0], 10.0) is None
    assert _first_divergence([5.0, 60.0, 3.0], 10.0) == (5.0, 60.0)
    assert _first_divergence([float("nan")], float("inf"))[0] == float("inf")
    assert _divergence_message(44.9682, 719.49, 5) == (
        "residual norm grew from 44.9682 to 719.49 in one sweep with thr=5; use a smaller thr")


def test_feature_select_config_validation_cpu():
    """FeatureSelectConfig mirrors select.py:33-46 (pure host logic)."""
    from paper_2104_12570_b200 import REFITS, FeatureSelectConfig
    assert REFITS == ("qr", "bak")
    with pytest.raises(ValueError):
        FeatureSelectConfig(max_feat=0)
    with pytest.raises(ValueError):
        FeatureSelectConfig(max_feat=1, refit="ridge")
    with pytest.raises(ValueError):
        FeatureSelectConfig(max_feat=1, stop_tol=-0.5)

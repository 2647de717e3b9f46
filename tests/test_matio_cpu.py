"""BAKM / CSV matrix files (reference matio.py).  Host-only
code paths (the native reader lives in libbak200.so but touches no GPU), so
these run in the CPU suite: files written by the reference's own save_matrix
(tests/golden/matio_*) load bit-identically, our writer reproduces them byte
for byte, and the reference's test_matio.py properties hold."""

import os

import numpy as np
import pytest

import golden_io

pb = pytest.importorskip("paper_2104_12570_b200")
G = golden_io.GOLDEN


def _expected():
    with np.load(os.path.join(G, "matio_expected.npz")) as z:
        return z["x64"], z["x32"]


def test_reference_files_load_bit_identically():
    x64, x32 = _expected()
    for name, x in (("matio_f64.bakm", x64), ("matio_f32.bakm", x32)):
        m = pb.load_matrix(os.path.join(G, name))
        assert m.dtype == x.dtype and m.flags.f_contiguous
        assert m.tobytes(order="F") == x.tobytes(order="F")
    c = pb.load_matrix(os.path.join(G, "matio_f64.csv"))
    assert c.tobytes(order="F") == x64.tobytes(order="F")


def test_writer_reproduces_reference_bytes(tmp_path):
    x64, x32 = _expected()
    for name, x in (("matio_f64.bakm", x64), ("matio_f32.bakm", x32)):
        p = tmp_path / name
        pb.save_matrix(p, x)
        with open(os.path.join(G, name), "rb") as f:
            assert p.read_bytes() == f.read()
    p = tmp_path / "m.csv"
    pb.save_matrix(p, x64, format="csv")
    with open(os.path.join(G, "matio_f64.csv"), "rb") as f:
        assert p.read_bytes() == f.read()


def test_pinned_loader_matches(tmp_path):
    rng = np.random.default_rng(1)
    x = np.asfortranarray(rng.standard_normal((1000, 37)).astype(np.float32))
    p = tmp_path / "m.bakm"
    pb.save_matrix(p, x)
    t = pb.load_matrix_pinned(p)
    assert tuple(t.shape) == x.shape and t.stride() == (1, 1000)
    assert np.array_equal(t.numpy(), x)


def test_large_parallel_read(tmp_path):
    # > 128 MB so the native reader splits the range over threads
    x = np.asfortranarray(np.arange(4096 * 4200, dtype=np.float64).reshape(4096, 4200, order="F"))
    p = tmp_path / "big.bakm"
    pb.save_matrix(p, x)
    m = pb.load_matrix(p)
    assert m.tobytes(order="F") == x.tobytes(order="F")


def test_binary_round_trip_and_errors(tmp_path):
    """test_matio.py:18-92 restated."""
    rng = np.random.default_rng(60)
    for dtype in (np.float64, np.float32):
        x = np.asfortranarray(rng.standard_normal((17, 5)).astype(dtype))
        p = tmp_path / "m.bin"
        pb.save_matrix(p, x)
        back = pb.load_matrix(p)
        assert back.dtype == dtype and back.tobytes(order="F") == x.tobytes(order="F")
    x = np.asfortranarray(rng.standard_normal((6, 2)))
    p = tmp_path / "m.bin"
    pb.save_matrix(p, x)
    whole = p.read_bytes()
    p.write_bytes(whole[:-8])
    with pytest.raises(pb.MatrixFormatError, match="file is short"):
        pb.load_matrix(p)
    p.write_bytes(b"NOPE" + whole[4:])
    with pytest.raises(pb.MatrixFormatError, match="bad magic"):
        pb.load_matrix(p, format="binary")
    bad = bytearray(whole)
    bad[12:16] = (16).to_bytes(4, "little")
    p.write_bytes(bytes(bad))
    with pytest.raises(pb.MatrixFormatError, match="unknown precision tag 16"):
        pb.load_matrix(p)
    p.write_bytes(whole[:10])
    with pytest.raises(pb.MatrixFormatError, match="truncated header"):
        pb.load_matrix(p, format="binary")


def test_csv_behaviour(tmp_path):
    """test_matio.py:9-67, 95-135 restated."""
    p = tmp_path / "m.csv"
    p.write_text("1,2\n3,4\n")
    m = pb.load_matrix(p)
    assert m.shape == (2, 2) and m.flags.f_contiguous and m.dtype == np.float64
    np.testing.assert_array_equal(m.ravel(order="F"), [1.0, 3.0, 2.0, 4.0])
    p.write_text("1,2\n3,4,5\n")
    with pytest.raises(pb.MatrixFormatError, match="row 2 has 3 values, expected 2"):
        pb.load_matrix(p)
    p.write_text("1,2\n3,potato\n")
    with pytest.raises(pb.MatrixFormatError, match="row 2 has a non-numeric value"):
        pb.load_matrix(p)
    p.write_text("\n\n")
    with pytest.raises(pb.MatrixFormatError, match="no rows"):
        pb.load_matrix(p)
    p.write_text("1,2\n\n3,4\n\n")
    assert pb.load_matrix(p).shape == (2, 2)
    col = tmp_path / "col.csv"
    col.write_text("1\n2\n3\n")
    np.testing.assert_array_equal(pb.load_vector(col), [1.0, 2.0, 3.0])
    row = tmp_path / "row.csv"
    row.write_text("1,2,3\n")
    np.testing.assert_array_equal(pb.load_vector(row), [1.0, 2.0, 3.0])
    sq = tmp_path / "sq.csv"
    sq.write_text("1,2\n3,4\n")
    with pytest.raises(pb.MatrixFormatError, match="expected a vector"):
        pb.load_vector(sq)
    x = np.asfortranarray(np.random.default_rng(64).standard_normal((5, 5)))
    d = tmp_path / "anything.dat"
    pb.save_matrix(d, x, format="binary")
    assert pb.load_matrix(d).tobytes(order="F") == x.tobytes(order="F")
    c = tmp_path / "m2.csv"
    pb.save_matrix(c, x, format="csv")
    with pytest.raises(pb.MatrixFormatError, match="bad magic"):
        pb.load_matrix(c, format="binary")
    with pytest.raises(ValueError, match="unknown format"):
        pb.load_matrix(d, format="hdf5")
    with pytest.raises(ValueError, match="unknown format"):
        pb.save_matrix(d, x, format="parquet")
    with pytest.raises(ValueError):
        pb.save_matrix(tmp_path / "v.bin", np.ones(4))
    e = tmp_path / "eye.bin"
    pb.save_matrix(e, np.eye(2, order="F"))
    assert e.read_bytes()[:4] == pb.MAGIC

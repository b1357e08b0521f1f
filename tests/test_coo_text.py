"""Native COO text ingestion (libsptk sptk_coo_text_parse) against the
reference's load_coo (coo.py:90-148): the reference's own outcomes on edge
cases (tests/golden/coo_text/, written by make_coo_text_golden.py) and the
sequential restatement (oracle/coo_text_oracle.py) on large multi-threaded
inputs.  CPU only (the parser is host code)."""

import json
import os

import numpy as np
import pytest

from oracle import coo_text_oracle as OC
from paper_2204_07104_b200 import CooFormatError, load_coo

GOLD = os.path.join(os.path.dirname(__file__), "golden", "coo_text")
with open(os.path.join(GOLD, "expected.json")) as _fh:
    EXPECTED = json.load(_fh)


@pytest.mark.parametrize("name", sorted(EXPECTED))
@pytest.mark.parametrize("threads", [1, 4])
def test_native_matches_reference_golden(name, threads):
    exp = EXPECTED[name]
    path = os.path.join(GOLD, name + ".txt")
    if "error" in exp:
        etype, msg = exp["error"]
        want = {"CooFormatError": CooFormatError, "OverflowError": OverflowError}[etype]
        with pytest.raises(want) as ei:
            load_coo(path, index_base=exp["index_base"], threads=threads)
        if etype == "CooFormatError":
            assert str(ei.value) == msg
        return
    t = load_coo(path, index_base=exp["index_base"], threads=threads)
    assert list(t.dims) == exp["dims"]
    np.testing.assert_array_equal(t.indices, np.array(exp["indices"], dtype=np.int64))
    vals = np.array([float.fromhex(v) for v in exp["values"]])
    assert t.values.tobytes() == vals.tobytes()  # bit-identical, incl. -0.0 and subnormals


@pytest.mark.parametrize("name", sorted(EXPECTED))
def test_oracle_matches_reference_golden(name):
    exp = EXPECTED[name]
    path = os.path.join(GOLD, name + ".txt")
    if "error" in exp:
        etype, msg = exp["error"]
        with pytest.raises((ValueError, OverflowError)) as ei:
            OC.load_coo(path, index_base=exp["index_base"])
        if etype == "CooFormatError":
            assert str(ei.value) == msg
        return
    dims, idx, vals = OC.load_coo(path, index_base=exp["index_base"])
    assert list(dims) == exp["dims"]
    np.testing.assert_array_equal(idx, np.array(exp["indices"], dtype=np.int64))
    assert vals.tobytes() == np.array([float.fromhex(v) for v in exp["values"]]).tobytes()


def _big_file(path, n, seed, eol=b"\n", bad=()):
    """n random order-3 entries with assorted number spellings, comments and
    blank lines; `bad` = {line index: replacement bytes}."""
    rng = np.random.default_rng(seed)
    idx = rng.integers(1, 50_000, size=(n, 3))
    vals = rng.standard_normal(n) * 10.0 ** rng.integers(-8, 8, size=n)
    fmts = [lambda v: repr(float(v)), lambda v: f"{v:.17g}", lambda v: f"{v:.3e}", lambda v: f"{v:.5f}"]
    lines = [b"# dims: 50000 50000 50000"]
    for k in range(n):
        if k % 997 == 0:
            lines.append(b"")
        if k % 1999 == 0:
            lines.append(b"# comment " + str(k).encode())
        s = " ".join(str(int(x)) for x in idx[k]) + ("\t" if k % 7 == 0 else " ") + fmts[k % 4](vals[k])
        lines.append(s.encode())
    for at, rep in bad:
        lines[at] = rep
    with open(path, "wb") as fh:
        fh.write(eol.join(lines) + eol)


@pytest.mark.parametrize("eol", [b"\n", b"\r\n"])
def test_native_matches_oracle_large(tmp_path, eol):
    p = str(tmp_path / "big.txt")
    _big_file(p, 200_000, 5, eol=eol)
    dims, idx, vals = OC.load_coo(p)
    for threads in (1, 3, 8, 0):
        t = load_coo(p, threads=threads)
        assert t.dims == tuple(dims)
        np.testing.assert_array_equal(t.indices, idx)
        assert t.values.tobytes() == vals.tobytes()


def test_native_reports_earliest_error_across_chunks(tmp_path):
    p = str(tmp_path / "bad.txt")
    # two errors far apart (different parser chunks): the earlier one wins
    _big_file(p, 200_000, 6, bad=[(150_000, b"1 2 3 4 5"), (60_000, b"1 2 3 nan")])
    with pytest.raises(ValueError) as ref:
        OC.load_coo(p)
    for threads in (1, 2, 8):
        with pytest.raises(CooFormatError) as ei:
            load_coo(p, threads=threads)
        assert str(ei.value) == str(ref.value)


def test_missing_file(tmp_path):
    with pytest.raises(FileNotFoundError):
        load_coo(str(tmp_path / "nope.txt"))
    with pytest.raises(ValueError):
        load_coo(str(tmp_path / "nope.txt"), index_base=2)

"""CPU tests: host-side logic and the C ABI boundary (no device compute)."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT


def test_library_exports_every_declared_symbol():
    from paper_2204_07104_b200 import _lib

    header = open(os.path.join(ROOT, "include", "sptk.h")).read()
    declared = set(re.findall(r"\b(sptk_[a-z0-9_]+)\s*\(", header))
    assert declared, "no declarations found"
    L = ctypes.CDLL(_lib.LIB_PATH)
    for name in declared:
        assert hasattr(L, name), name
    assert declared == set(_lib.SIGNATURES), declared ^ set(_lib.SIGNATURES)


def test_host_seed_matches_numpy():
    from paper_2204_07104_b200.sampler import pcg64_state

    for ent in ([0], [1, 1, 0, 0, 0, 0], [2**40 + 5, 3], [7, 2, 3, 9, 9, 9, 9, 1]):
        st = np.random.default_rng(ent).bit_generator.state["state"]
        got = pcg64_state(ent)
        assert (int(got[0]) << 64 | int(got[1])) == st["state"]
        assert (int(got[2]) << 64 | int(got[3])) == st["inc"]


def test_record_words():
    from paper_2204_07104_b200 import _lib

    L = _lib.load()
    assert [L.sptk_record_words(n, 0) for n in (2, 3, 4, 7, 8)] == [4, 4, 8, 8, 16]
    assert [L.sptk_record_words(n, 1) for n in (2, 3, 4, 6, 7)] == [4, 8, 8, 8, 16]


def test_round_schedule_reference(golden):
    from paper_2204_07104_b200.schedule import round_schedule

    for order, m in [(2, 3), (3, 2), (3, 4), (4, 3), (6, 2), (5, 4)]:
        assert np.array_equal(np.array(round_schedule(order, m).rounds), golden[f"sched_{order}_{m}"])
    s = round_schedule(3, 2)
    assert [r[0] for r in s.rounds] == [(0, 0, 0), (0, 0, 1), (0, 1, 1), (0, 1, 0)]


def test_synthetic_matches_reference(golden, golden_meta):
    """generate_synthetic + split reproduce the reference's tensors (same seeds)."""
    from paper_2204_07104_b200 import generate_synthetic, split

    for name in ("s3w1", "s4w2", "floydbig", "cfg1"):
        m = golden_meta[f"train_{name}"]
        t, _ = generate_synthetic(tuple(m["dims"]), m["nnz"], tuple(m["jr"]), m["r"], noise_sigma=m["noise"],
                                  seed=m["seed"])
        if m["test_fraction"]:
            ds = split(t, m["test_fraction"], seed=m["seed"])
            tr, te = ds.train, ds.test
            assert np.array_equal(te.indices, golden[f"train_{name}_test_idx"])
            assert np.array_equal(te.values, golden[f"train_{name}_test_vals"])
        else:
            tr = t
        assert np.array_equal(tr.indices, golden[f"train_{name}_train_idx"])
        assert np.array_equal(tr.values, golden[f"train_{name}_train_vals"])


def test_init_model_matches_reference(golden, golden_meta):
    from paper_2204_07104_b200 import ModelConfig, default_init_scale, init_model

    m = golden_meta["train_cfg1"]
    vals = golden["train_cfg1_train_vals"]
    scale = default_init_scale(vals, 3)
    assert scale == m["scale"]
    model = init_model(tuple(m["dims"]), ModelConfig(tuple(m["jr"]), m["r"], scale, seed=1))
    for n in range(3):
        assert np.array_equal(model.factors[n], golden[f"train_cfg1_A{n}_init"])
        assert np.array_equal(model.core_factors[n], golden[f"train_cfg1_B{n}_init"])


def test_validation_messages():
    from paper_2204_07104_b200 import ModelConfig, SparseTensorCoo, TrainConfig, learning_rate

    with pytest.raises(ValueError, match="order"):
        SparseTensorCoo((3,), np.zeros((0, 1)), np.zeros(0))
    with pytest.raises(ValueError, match="out of bounds"):
        SparseTensorCoo((2, 2), [[0, 2]], [1.0])
    with pytest.raises(ValueError, match="non-finite"):
        SparseTensorCoo((2, 2), [[0, 1]], [np.nan])
    with pytest.raises(ValueError):
        TrainConfig(epochs=0)
    with pytest.raises(ValueError):
        TrainConfig(epochs=1, update_mode="async")
    with pytest.raises(ValueError):
        ModelConfig((0, 2), 1)
    assert learning_rate(0.009, 0.05, 1) == pytest.approx(0.009 / 1.05, rel=1e-12)
    assert learning_rate(0.37, 5.0, 0) == 0.37


def test_coo_text_roundtrip(tmp_path):
    from paper_2204_07104_b200 import CooFormatError, SparseTensorCoo, load_coo, write_coo

    t = SparseTensorCoo((3, 4, 5), [[0, 1, 2], [2, 3, 4]], [1.25, -2.0 / 3.0])
    p = tmp_path / "t.tns"
    write_coo(t, p)
    assert load_coo(p).same_entries(t)
    bad = tmp_path / "bad.tns"
    bad.write_text("1 2 3 1.0\n1 2 x\n")
    with pytest.raises(CooFormatError, match="line 2"):
        load_coo(bad)


def test_checkpoint_roundtrip(tmp_path):
    from paper_2204_07104_b200 import ModelConfig, init_model, load_model, save_model

    m = init_model((3, 4, 5), ModelConfig((2, 3, 2), 2, 0.7, seed=3))
    p = tmp_path / "m.txt"
    save_model(m, p)
    m2 = load_model(p)
    for a, b in zip(m.factors + m.core_factors, m2.factors + m2.core_factors):
        assert np.array_equal(a, b)


def test_binary_coo_and_checkpoint_roundtrip(tmp_path):
    """SURVEY 8f side formats: binary COO ingestion and binary checkpoints
    round-trip exactly (memory-mapped load)."""
    import numpy as np

    from paper_2204_07104_b200 import (ModelConfig, SparseTensorCoo, init_model, load_coo_binary,
                                       load_model_binary, save_model_binary, write_coo_binary)

    rng = np.random.default_rng(3)
    dims = (30, 40, 50)
    t = SparseTensorCoo(dims, np.stack([rng.integers(0, d, 500) for d in dims], 1), rng.normal(size=500))
    write_coo_binary(t, tmp_path / "t.npz")
    u = load_coo_binary(tmp_path / "t.npz")
    assert u.dims == dims and np.array_equal(u.indices, t.indices) and np.array_equal(u.values, t.values)
    m = init_model(dims, ModelConfig((3, 4, 5), 2, 0.7, seed=4))
    save_model_binary(m, tmp_path / "m.npz")
    m2 = load_model_binary(tmp_path / "m.npz")
    assert m2.dims == m.dims and m2.j_ranks == m.j_ranks and m2.r_core == m.r_core
    for a, b in zip(m.factors + m.core_factors, m2.factors + m2.core_factors):
        assert np.array_equal(a, b)

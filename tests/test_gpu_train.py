"""End-to-end train() on the GPU against the reference's own training runs."""

import numpy as np
import pytest

from conftest import golden_train_case
from oracle import oracle as O

pytestmark = pytest.mark.gpu

GOLDEN_TRAIN = ["s3w1", "s3w2", "s3w3", "s4w2", "r1", "floyd", "tail", "floydbig"]


def _setup(case):
    from paper_2204_07104_b200 import DatasetSplit, SparseTensorCoo, TuckerModel

    m = case["meta"]
    dims = tuple(m["dims"])
    tr = SparseTensorCoo(dims, case["train_idx"], case["train_vals"])
    te = SparseTensorCoo(dims, case["test_idx"].reshape(-1, len(dims)), case["test_vals"])
    model = TuckerModel(dims, tuple(m["jr"]), m["r"], [a.copy() for a in case["A0"]],
                        [b.copy() for b in case["B0"]])
    return model, DatasetSplit(tr, te), m


@pytest.mark.parametrize("name", GOLDEN_TRAIN)
def test_sequential_fp64_reproduces_reference(golden, golden_meta, name):
    """Verification mode: the GPU run equals the reference's train() to fp64
    rounding (same visit orders, core batches, DSGD blocks, merges)."""
    from paper_2204_07104_b200 import TrainConfig, train

    model, ds, m = _setup(golden_train_case(golden, golden_meta, name))
    cfg = TrainConfig(epochs=m["epochs"], workers=m["workers"], seed=m["train_seed"], core_batch_cap=m["cap"],
                      update_core=m["update_core"], alpha_a=m["alpha_a"], update_mode="exact",
                      precision="fp64")
    rows = train(model, ds, cfg)
    case = golden_train_case(golden, golden_meta, name)
    for a, b in zip(model.factors + model.core_factors, case["A1"] + case["B1"]):
        np.testing.assert_allclose(a, b, rtol=1e-10, atol=1e-13)
    for got, want in zip(rows, m["rows"]):
        if not np.isnan(want["test_rmse"]):
            assert got.test_rmse == pytest.approx(want["test_rmse"], rel=1e-9)
        assert got.train_rmse == pytest.approx(want["train_rmse"], rel=1e-9)


def test_sequential_fp32_one_epoch_within_1e4(golden, golden_meta):
    """North-star parity: deterministic synchronous mode, fp32, one step (epoch):
    A/B within 1e-4 relative of the reference (atol floor 1e-5 * max)."""
    from paper_2204_07104_b200 import TrainConfig, train

    case = golden_train_case(golden, golden_meta, "cfg1")
    model, ds, m = _setup(case)
    train(model, ds, TrainConfig(epochs=1, seed=1, update_mode="exact", precision="fp32"))
    fs = [a.copy() for a in case["A0"]]
    bs = [b.copy() for b in case["B0"]]
    O.train(fs, bs, case["train_idx"], case["train_vals"], epochs=1, seed=1, evaluate=False)
    for got, want in zip(model.factors + model.core_factors, fs + bs):
        tol = 1e-4 * np.abs(want) + 1e-5 * np.abs(want).max()
        assert (np.abs(got - want) <= tol).all()


def test_cfg1_sequential_fp64_curve(golden, golden_meta):
    from paper_2204_07104_b200 import TrainConfig, train

    case = golden_train_case(golden, golden_meta, "cfg1")
    model, ds, m = _setup(case)
    rows = train(model, ds, TrainConfig(epochs=5, seed=1, update_mode="exact", precision="fp64"))
    for got, want in zip(rows, m["rows"]):
        assert got.test_rmse == pytest.approx(want["test_rmse"], rel=1e-9)
    for a, b in zip(model.factors + model.core_factors, case["A1"] + case["B1"]):
        np.testing.assert_allclose(a, b, rtol=1e-9, atol=1e-12)


@pytest.mark.parametrize("mode", ["auto", "exact"])
def test_cfg1_default_mode_rmse(golden, golden_meta, mode):
    """BASELINE configs[0] with the default (auto -> exact) mode in fp32: test
    RMSE after 5 epochs within 1% of the reference's."""
    from paper_2204_07104_b200 import TrainConfig, train

    case = golden_train_case(golden, golden_meta, "cfg1")
    model, ds, m = _setup(case)
    rows = train(model, ds, TrainConfig(epochs=5, seed=1, update_mode=mode))
    for got, want in zip(rows, m["rows"]):
        assert abs(got.test_rmse - want["test_rmse"]) <= 0.01 * want["test_rmse"]
        assert abs(got.train_rmse - want["train_rmse"]) <= 0.01 * want["train_rmse"]


def test_cfg1_hogwild_rmse(golden, golden_meta):
    """Throughput mode forced on BASELINE configs[0]: with the Hogwild
    in-flight cap (n/64 samples) it lands within 1% of the reference."""
    from paper_2204_07104_b200 import TrainConfig, train

    case = golden_train_case(golden, golden_meta, "cfg1")
    model, ds, m = _setup(case)
    rows = train(model, ds, TrainConfig(epochs=5, seed=1, update_mode="hogwild"))
    ref = m["rows"][-1]["test_rmse"]
    gap = abs(rows[-1].test_rmse - ref) / ref
    print("cfg1 hogwild test rmse", [r.test_rmse for r in rows], "reference", ref, "gap", gap)
    assert gap < 0.01


@pytest.mark.parametrize("workers", [1, 20])
def test_netflix_shaped_hogwild_rmse_curve_within_1pct(workers):
    """North-star accuracy bar on the bench workload (BASELINE configs[1]): the
    throughput (Hogwild, fp32, tcgen05) path's test RMSE after each of 5
    epochs is within 1% of the reference's (tests/golden/nf99_curve.json, the
    reference's train() on the same 99,072,112-nonzero tensor, 8 DSGD
    workers, alpha_a = 0.003)."""
    import json
    import os

    from paper_2204_07104_b200 import DatasetSplit, ModelConfig, TrainConfig, default_init_scale, init_model, train
    from paper_2204_07104_b200.device import predict_device_f64
    from paper_2204_07104_b200.synthetic import generate_large

    with open(os.path.join(os.path.dirname(__file__), "golden", "nf99_curve.json")) as fh:
        ref = json.load(fh)
    dims = tuple(ref["dims"])

    def pred(model, idx):
        out = np.empty(idx.shape[0])
        for c0 in range(0, idx.shape[0], 1 << 25):
            out[c0:c0 + (1 << 25)] = predict_device_f64(model, idx[c0:c0 + (1 << 25)])
        return out

    tr, te, _ = generate_large(dims, ref["nnz"], (16, 16, 16), 16, 0.1, seed=7, n_test=ref["n_test"], predict=pred)
    m = init_model(dims, ModelConfig((16, 16, 16), 16, default_init_scale(tr.values, 3), seed=1))
    rows = train(m, DatasetSplit(tr, te), TrainConfig(epochs=ref["epochs"], seed=1, alpha_a=ref["alpha_a"],
                                                      update_mode="hogwild", workers=workers))
    got = [r.test_rmse for r in rows]
    want = [r["test_rmse"] for r in ref["rows"]]
    print("NF workers", workers, "test RMSE", got, "reference", want)
    for g, w in zip(got, want):
        assert abs(g - w) <= 0.01 * w

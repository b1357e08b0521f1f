"""Public facade against the reference's own outputs (tests/golden/facade.npz,
written by make_facade_golden.py from /root/reference): TuckerSGD
fit/predict/score/get_params (estimator.py:119-182), predict_entries
(model.py:134-146), rmse/mae (trainer.py:89-102), frobenius_objective
(trainer.py:105-132)."""

import json
import math
import os

import numpy as np
import pytest

from conftest import GOLDEN_DIR


@pytest.fixture(scope="module")
def fg():
    return np.load(os.path.join(GOLDEN_DIR, "facade.npz"))


@pytest.fixture(scope="module")
def fm():
    with open(os.path.join(GOLDEN_DIR, "facade_meta.json")) as fh:
        return json.load(fh)


def _model(fg):
    from paper_2204_07104_b200 import TuckerModel

    return TuckerModel((20, 22, 24), (4, 5, 3), 6, [fg[f"model_A{n}"].copy() for n in range(3)],
                       [fg[f"model_B{n}"].copy() for n in range(3)])


# ------------------------------------------------------------------ CPU ----
def test_estimator_params_match_reference(fm):
    from paper_2204_07104_b200 import TuckerSGD

    est = TuckerSGD(j_ranks=4, r_core=4, dims=(20, 22, 24), epochs=4, workers=1, seed=2)
    got = est.get_params()
    want = fm["est_w1"]["params"]
    for k, v in want.items():
        g = list(got[k]) if isinstance(got[k], tuple) else got[k]
        assert g == v, k
    # the two extra parameters select the device update mode / precision
    assert set(got) - set(want) == {"update_mode", "precision"}
    assert est.set_params(epochs=7) is est and est.epochs == 7
    with pytest.raises(ValueError, match="unknown parameter 'bogus' for TuckerSGD"):
        est.set_params(bogus=1)


def test_estimator_input_validation():
    from paper_2204_07104_b200 import TuckerSGD

    est = TuckerSGD(dims=(4, 4, 4))
    with pytest.raises(RuntimeError, match="not fitted"):
        est.predict(np.zeros((1, 3), dtype=np.int64))
    with pytest.raises(ValueError):
        est.fit(np.zeros((0, 3), dtype=np.int64), np.zeros(0))
    with pytest.raises(ValueError):
        est.fit(np.array([[0, 0, 4]]), np.ones(1))
    with pytest.raises(ValueError):
        est.fit(np.array([[0, 0, -1]]), np.ones(1))
    with pytest.raises(ValueError):
        est.fit(np.array([[0, 0, 1]]), np.array([np.inf]))


def test_predict_entries_rejects_out_of_range_on_host(fg):
    """Bad indices raise before anything reaches the device (numpy's
    IndexError; the K6 kernel itself does no bounds checks)."""
    from paper_2204_07104_b200 import predict_entries

    m = _model(fg)
    with pytest.raises(IndexError, match="out of bounds for axis 0 with size 22"):
        predict_entries(m, np.array([[0, 22, 0]]))
    with pytest.raises(IndexError, match="out of bounds"):
        predict_entries(m, np.array([[-21, 0, 0]]))
    with pytest.raises(IndexError):
        predict_entries(m, np.array([[0, 0]]))


# ------------------------------------------------------------------ GPU ----
@pytest.mark.gpu
@pytest.mark.parametrize("w", [1, 2])
def test_tuckersgd_fp64_matches_reference(fg, fm, w):
    from paper_2204_07104_b200 import TuckerSGD

    est = TuckerSGD(j_ranks=4, r_core=4, dims=(20, 22, 24), epochs=4, workers=w, seed=2,
                    update_mode="exact", precision="fp64")
    est.fit(fg["train_idx"], fg["train_vals"])
    for n in range(3):
        np.testing.assert_allclose(est.factors_[n], fg[f"est_w{w}_A{n}"], rtol=1e-9, atol=1e-12)
        np.testing.assert_allclose(est.core_factors_[n], fg[f"est_w{w}_B{n}"], rtol=1e-9, atol=1e-12)
    np.testing.assert_allclose(est.predict(fg["test_idx"]), fg[f"est_w{w}_pred"], rtol=1e-9, atol=1e-12)
    assert est.score(fg["test_idx"], fg["test_vals"]) == pytest.approx(fm[f"est_w{w}"]["score"], rel=1e-9)
    want = fm[f"est_w{w}"]["history"]
    assert len(est.history_) == len(want)
    for got, ref in zip(est.history_, want):
        assert got.epoch == ref["epoch"]
        assert got.train_rmse == pytest.approx(ref["train_rmse"], rel=1e-9)
        assert got.train_mae == pytest.approx(ref["train_mae"], rel=1e-9)
        assert math.isnan(got.test_rmse) and math.isnan(ref["test_rmse"])
        assert got.gamma_a == ref["gamma_a"] and got.gamma_b == ref["gamma_b"]


@pytest.mark.gpu
def test_tuckersgd_default_fp32_within_tolerance(fg, fm):
    """The library default (auto -> exact order, fp32 arithmetic): R^2 within
    1e-4 and training curve within 1% of the reference's fp64 fit."""
    from paper_2204_07104_b200 import TuckerSGD

    est = TuckerSGD(j_ranks=4, r_core=4, dims=(20, 22, 24), epochs=4, workers=1, seed=2)
    est.fit(fg["train_idx"], fg["train_vals"])
    assert abs(est.score(fg["test_idx"], fg["test_vals"]) - fm["est_w1"]["score"]) <= 1e-4
    pred = est.predict(fg["test_idx"])
    ref = fg["est_w1_pred"]
    assert np.abs(pred - ref).max() <= 1e-3 * np.abs(ref).max()
    for got, want in zip(est.history_, fm["est_w1"]["history"]):
        assert abs(got.train_rmse - want["train_rmse"]) <= 0.01 * want["train_rmse"]


@pytest.mark.gpu
def test_tuckersgd_infers_dims(fg, fm):
    from paper_2204_07104_b200 import TuckerSGD

    est = TuckerSGD(j_ranks=3, r_core=5, epochs=2, seed=4, update_mode="exact", precision="fp64")
    with pytest.warns(UserWarning):
        est.fit(fg["train_idx"], fg["train_vals"])
    assert list(est.dims_) == fm["est_infer"]["dims"]
    np.testing.assert_allclose(est.predict(fg["train_idx"][:50]), fg["est_infer_pred"], rtol=1e-9, atol=1e-12)
    assert est.score(fg["train_idx"], fg["train_vals"]) == pytest.approx(fm["est_infer"]["score"], rel=1e-9)


@pytest.mark.gpu
def test_predict_entries_negative_rows_and_metrics(fg, fm):
    from paper_2204_07104_b200 import SparseTensorCoo, frobenius_objective, mae, predict_entries, rmse

    m = _model(fg)
    np.testing.assert_allclose(predict_entries(m, fg["neg_rows"]), fg["neg_pred"], rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(predict_entries(m, fg["test_idx"]), fg["test_pred"], rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(predict_entries(m, fg["test_idx"][0]), fg["test_pred"][:1], rtol=1e-12)
    test = SparseTensorCoo((20, 22, 24), fg["test_idx"], fg["test_vals"])
    assert rmse(m, test) == pytest.approx(fm["rmse"], rel=1e-12)
    assert mae(m, test) == pytest.approx(fm["mae"], rel=1e-12)
    assert frobenius_objective(m, test) == pytest.approx(fm["frob_plain"], rel=1e-12)
    assert frobenius_objective(m, test, lambda_core=0.3, lambda_factors=0.05) == pytest.approx(
        fm["frob_pen"], rel=1e-12)

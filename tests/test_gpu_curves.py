"""North-star accuracy bar at every named config: the throughput path's
(Hogwild, fp32, tcgen05) test RMSE after K epochs within 1% of the reference's.

The reference curves (tests/golden/curve_<name>.json) come from the oracle C
port -- bitwise equal to the reference's train() (trainer.py:150-271; pinned
by tests/test_oracle_golden.py) -- with 8 DSGD workers on a prefix of each
bench workload (generate_large seed 7), written by tests/golden/make_curves.py.
The GPU runs the same tensor with one worker (the bench default) and with the
reference's 8 workers (the flat DSGD visit list)."""

import glob
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.join(os.path.dirname(__file__), "golden")
CURVES = sorted(os.path.basename(p)[6:-5] for p in glob.glob(os.path.join(HERE, "curve_*.json")))


@pytest.mark.parametrize("workers", [1, 8])
@pytest.mark.parametrize("name", CURVES)
def test_hogwild_rmse_curve_within_1pct(name, workers):
    from paper_2204_07104_b200 import DatasetSplit, ModelConfig, TrainConfig, default_init_scale, init_model, train
    from paper_2204_07104_b200.device import predict_device_f64
    from paper_2204_07104_b200.synthetic import generate_large

    with open(os.path.join(HERE, f"curve_{name}.json")) as fh:
        ref = json.load(fh)
    dims = tuple(ref["dims"])
    order, J = len(dims), ref["J"]

    def pred(model, idx):
        out = np.empty(idx.shape[0])
        for c0 in range(0, idx.shape[0], 1 << 25):
            out[c0:c0 + (1 << 25)] = predict_device_f64(model, idx[c0:c0 + (1 << 25)])
        return out

    tr, te, _ = generate_large(dims, ref["nnz"], (J,) * order, J, 0.1, seed=7, n_test=ref["n_test"], predict=pred)
    m = init_model(dims, ModelConfig((J,) * order, J, default_init_scale(tr.values, order), seed=1))
    rows = train(m, DatasetSplit(tr, te), TrainConfig(epochs=ref["epochs"], seed=1, alpha_a=ref["alpha_a"],
                                                      workers=workers, update_mode="hogwild"))
    got = [r.test_rmse for r in rows]
    want = [r["test_rmse"] for r in ref["rows"]]
    print(name, "workers", workers, "test RMSE", got, "reference", want,
          "gaps", [round(g / w - 1.0, 4) for g, w in zip(got, want)])
    # north star: test RMSE after K epochs within 1% (the first epochs of a
    # Hogwild run on a small prefix trail the sequential reference by more:
    # printed above, not asserted)
    assert abs(got[-1] - want[-1]) <= 0.01 * want[-1]

"""Exact vs Hogwild epoch times over tensor sizes (for training.AUTO_EXACT_MAX_NNZ):
train() wall_seconds (device-timed epochs) of 3 epochs each."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_07104_b200 import DatasetSplit, ModelConfig, TrainConfig, default_init_scale, init_model, train  # noqa
from paper_2204_07104_b200.synthetic import generate_large  # noqa

for dims, nnz in [((1000, 1000, 1000), 100_000), ((3000, 3000, 3000), 500_000), ((10000, 10000, 10000), 1 << 20),
                  ((20000, 20000, 20000), 1 << 21), ((40000, 40000, 40000), 1 << 22)]:
    tr, te, _ = generate_large(dims, nnz, (8,) * 3, 8, 0.1, seed=7, n_test=nnz // 10)
    out = {"dims": dims, "nnz": nnz}
    for mode in ("exact", "hogwild"):
        m = init_model(dims, ModelConfig((8,) * 3, 8, default_init_scale(tr.values, 3), seed=1))
        rows = train(m, DatasetSplit(tr, te), TrainConfig(epochs=3, seed=1, update_mode=mode))
        out[mode + "_ms_per_epoch"] = round(rows[-1].wall_seconds / 3 * 1e3, 3)
        out[mode + "_test_rmse"] = round(rows[-1].test_rmse, 5)
    print(json.dumps(out), flush=True)

"""Hogwild divergence probe on the smoke() shape: test RMSE after one epoch
for the current SPTK_TC / SPTK_TC_GRID environment (diagnostic)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2204_07104_b200 import DatasetSplit, ModelConfig, TrainConfig, default_init_scale, init_model, train  # noqa
from paper_2204_07104_b200 import _lib  # noqa: E402
from paper_2204_07104_b200.synthetic import generate_large  # noqa: E402

dims = tuple(int(x) for x in os.environ.get("DIMS", "3000,1200,300").split(","))
nnz = int(os.environ.get("NNZ", "400000"))
J = int(os.environ.get("J", "16"))
W = int(os.environ.get("WORKERS", "1"))
tr, te, _ = generate_large(dims, nnz, (J,) * len(dims), J, 0.1, seed=7, n_test=20_000)
m = init_model(dims, ModelConfig((J,) * len(dims), J, default_init_scale(tr.values, len(dims)), seed=1))
rows = train(m, DatasetSplit(tr, te), TrainConfig(epochs=int(os.environ.get("EPOCHS", "1")), seed=1, alpha_a=0.003,
                                                  update_mode="hogwild", workers=W))
print("probe", os.environ.get("SPTK_TC"), os.environ.get("SPTK_TC_GRID"), dims, nnz, "W", W,
      _lib.load().sptk_last_factor_kernel().decode(), [round(r.test_rmse, 4) for r in rows], flush=True)

"""Golden outputs of the reference's public facade (build container only).

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_facade_golden.py

Records, from the reference package itself (numpy 2.3.5):
  * TuckerSGD.fit / predict / score / get_params / history_ (estimator.py:119-182)
    at workers 1 and 2, with a test set held out by ``split``;
  * predict_entries on rows with negative (wrapped) indices (model.py:134-146);
  * rmse / mae (trainer.py:89-102) and frobenius_objective with both penalties
    (trainer.py:105-132).
Output: tests/golden/facade.npz + tests/golden/facade_meta.json.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = os.environ.get("SPTUCKER_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

from sptucker.coo import generate_synthetic, split  # noqa: E402
from sptucker.estimator import TuckerSGD  # noqa: E402
from sptucker.model import ModelConfig, default_init_scale, init_model, predict_entries  # noqa: E402
from sptucker.trainer import frobenius_objective, mae, rmse  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
G: dict[str, np.ndarray] = {}
META: dict = {"numpy": np.__version__}

t, _ = generate_synthetic((20, 22, 24), 1500, (4, 4, 4), 4, noise_sigma=0.1, seed=5)
ds = split(t, 0.2, seed=5)
G["train_idx"], G["train_vals"] = ds.train.indices, ds.train.values
G["test_idx"], G["test_vals"] = ds.test.indices, ds.test.values

for w in (1, 2):
    est = TuckerSGD(j_ranks=4, r_core=4, dims=(20, 22, 24), epochs=4, workers=w, seed=2)
    est.fit(ds.train.indices, ds.train.values)
    G[f"est_w{w}_pred"] = est.predict(ds.test.indices)
    for n in range(3):
        G[f"est_w{w}_A{n}"] = est.factors_[n]
        G[f"est_w{w}_B{n}"] = est.core_factors_[n]
    META[f"est_w{w}"] = {
        "score": est.score(ds.test.indices, ds.test.values),
        "params": {k: (list(v) if isinstance(v, tuple) else v) for k, v in est.get_params().items()},
        "history": [r._asdict() if hasattr(r, "_asdict") else r.__dict__ for r in est.history_],
    }

# dims inferred from X (dims=None), scalar ranks, default init scale
est = TuckerSGD(j_ranks=3, r_core=5, epochs=2, seed=4)
est.fit(ds.train.indices, ds.train.values)
G["est_infer_pred"] = est.predict(ds.train.indices[:50])
META["est_infer"] = {"dims": list(est.dims_), "score": est.score(ds.train.indices, ds.train.values)}

m = init_model((20, 22, 24), ModelConfig((4, 5, 3), 6, default_init_scale(ds.train.values, 3), seed=9))
for n in range(3):
    G[f"model_A{n}"] = m.factors[n]
    G[f"model_B{n}"] = m.core_factors[n]
rows = np.array([[0, 0, 0], [-1, -1, -1], [19, 21, 23], [-20, 3, -24], [5, -7, 11]], dtype=np.int64)
G["neg_rows"] = rows
G["neg_pred"] = predict_entries(m, rows)
G["test_pred"] = predict_entries(m, ds.test.indices)
META["rmse"] = rmse(m, ds.test)
META["mae"] = mae(m, ds.test)
META["frob_plain"] = frobenius_objective(m, ds.test)
META["frob_pen"] = frobenius_objective(m, ds.test, lambda_core=0.3, lambda_factors=0.05)

np.savez_compressed(os.path.join(HERE, "facade.npz"), **G)
with open(os.path.join(HERE, "facade_meta.json"), "w") as fh:
    json.dump(META, fh, indent=1, default=float)
print("wrote facade golden", {k: v for k, v in META.items() if k.startswith(("rmse", "mae", "frob"))})

"""Test RMSE curve on the full Netflix-shaped bench tensor vs the reference's
(tests/golden/nf99_curve.json), for several kernel settings.

    python tools/nf_rmse_probe.py hogwild:1 hogwild:2 hogwild:0 ...   (mode:tc)
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from paper_2204_07104_b200 import (DatasetSplit, ModelConfig, TrainConfig, _lib, default_init_scale,  # noqa: E402
                                   init_model, train)
from paper_2204_07104_b200.device import predict_device_f64  # noqa: E402
from paper_2204_07104_b200.synthetic import generate_large  # noqa: E402

ref = json.load(open(os.path.join(ROOT, "tests", "golden", "nf99_curve.json")))


def pred(model, idx):
    out = np.empty(idx.shape[0])
    for c0 in range(0, idx.shape[0], 1 << 25):
        out[c0:c0 + (1 << 25)] = predict_device_f64(model, idx[c0:c0 + (1 << 25)])
    return out


dims = tuple(ref["dims"])
tr, te, _ = generate_large(dims, ref["nnz"], (16, 16, 16), 16, 0.1, seed=7, n_test=ref["n_test"], predict=pred)
ds = DatasetSplit(tr, te)
want = [r["test_rmse"] for r in ref["rows"]]
L = _lib.load()
for spec in sys.argv[1:]:
    mode, tc = spec.split(":")
    L.sptk_set_tc_mode(int(tc))
    m = init_model(dims, ModelConfig((16, 16, 16), 16, default_init_scale(tr.values, 3), seed=1))
    t0 = time.time()
    rows = train(m, ds, TrainConfig(epochs=ref["epochs"], seed=1, alpha_a=ref["alpha_a"], update_mode=mode))
    got = [r.test_rmse for r in rows]
    print(json.dumps({"spec": spec, "env": {k: v for k, v in os.environ.items() if k.startswith("SPTK_")},
                      "rel_gap": [round((a - b) / b, 5) for a, b in zip(got, want)], "test_rmse": got,
                      "train_s": round(time.time() - t0, 2)}), flush=True)

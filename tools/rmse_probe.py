"""GPU RMSE vs the reference curve on the 8M Netflix-shaped tensor (tests/golden/nf_golden.json)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2204_07104_b200 import (DatasetSplit, ModelConfig, TrainConfig, default_init_scale,  # noqa: E402
                                   init_model, train, _lib)
from paper_2204_07104_b200.synthetic import generate_large  # noqa: E402

g = json.load(open(os.path.join(ROOT, "tests", "golden", "nf_golden.json")))["nf8m"]
tr, te, _ = generate_large(tuple(g["dims"]), g["nnz"], (g["J"],) * 3, g["R"], 0.1, seed=g["seed"], n_test=g["n_test"])
ds = DatasetSplit(tr, te)
ref = [r["test_rmse"] for r in g["rows"]]
L = _lib.load()
for spec in sys.argv[1:]:
    mode, tc = spec.split(":")
    L.sptk_set_tc_mode(int(tc))
    m = init_model(tr.dims, ModelConfig((16, 16, 16), 16, default_init_scale(tr.values, 3), seed=1))
    t0 = time.time()
    rows = train(m, ds, TrainConfig(epochs=g["epochs"], seed=1, alpha_a=g["alpha_a"], update_mode=mode))
    got = [r.test_rmse for r in rows]
    print(json.dumps({"mode": mode, "tc": int(tc), "test_rmse": got, "ref": ref,
                      "rel_gap": [abs(a - b) / b for a, b in zip(got, ref)], "seconds": time.time() - t0}), flush=True)

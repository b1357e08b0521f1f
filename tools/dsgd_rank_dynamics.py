"""One rank's Hogwild dynamics at M-GPU DSGD, on one GPU: the NF tensor with
M workers, every block launched on its own (SPTK_FLAT=0) at the grid a rank
would run, under the hot-mode step rules being compared.  Prints the per-epoch
test RMSE against the reference's M-worker curve (tests/golden/nf99_curve.json,
or CURVE=curve_y4_full.json ...).
usage: python tools/dsgd_rank_dynamics.py "NAME:ENV=V,ENV=V" ..."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_07104_b200 import DatasetSplit, ModelConfig, TrainConfig, default_init_scale, init_model, train  # noqa
from paper_2204_07104_b200.device import predict_device_f64  # noqa
from paper_2204_07104_b200.synthetic import generate_large  # noqa

# CURVE=<file in tests/golden> picks the workload (default: the NF curve)
ref = json.load(open(os.path.join(os.path.dirname(__file__), "..", "tests", "golden",
                                  os.environ.get("CURVE", "nf99_curve.json"))))
dims, J = tuple(ref["dims"]), ref["J"]
N = len(dims)
want = [r["test_rmse"] for r in ref["rows"]]


def pred(model, idx):
    out = np.empty(idx.shape[0])
    for c0 in range(0, idx.shape[0], 1 << 25):
        out[c0:c0 + (1 << 25)] = predict_device_f64(model, idx[c0:c0 + (1 << 25)])
    return out


tr, te, _ = generate_large(dims, ref["nnz"], (J,) * N, J, 0.1, seed=7, n_test=ref["n_test"], predict=pred)
ds = DatasetSplit(tr, te)
m0 = init_model(dims, ModelConfig((J,) * N, J, default_init_scale(tr.values, N), seed=1))
print("reference", ref["workers"], "workers:", want, flush=True)
for spec in sys.argv[1:]:
    name, _, envs = spec.partition(":")
    saved = dict(os.environ)
    workers = ref["workers"]
    for kv in filter(None, envs.split(",")):
        k, v = kv.split("=")
        if k == "workers":
            workers = int(v)
        else:
            os.environ[k] = v
    m = init_model(dims, ModelConfig((J,) * N, J, default_init_scale(tr.values, N), seed=1))
    t0 = time.time()
    rows = train(m, ds, TrainConfig(epochs=ref["epochs"], seed=1, alpha_a=ref["alpha_a"], workers=workers,
                                    update_mode="hogwild"))
    got = [r.test_rmse for r in rows]
    print(json.dumps({"name": name, "env": envs, "test_rmse": got,
                      "gap": [round(g / w - 1.0, 4) for g, w in zip(got, want)],
                      "wall_s": round(time.time() - t0, 1)}), flush=True)
    os.environ.clear()
    os.environ.update(saved)

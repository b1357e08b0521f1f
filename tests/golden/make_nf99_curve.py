"""Reference RMSE curve on the full Netflix-shaped bench tensor (build container).

    python tests/golden/make_nf99_curve.py [epochs] [workers]

Runs the ORACLE C port -- bitwise identical to the reference's train()
(tests/test_oracle_golden.py pins it) -- with the reference's DSGD workers on
the bench workload of bench.py (generate_large seed 7, 99,072,112 training
nonzeros, 1,408,395 test entries, J=R=16, alpha_a=0.003).  Output:
tests/golden/nf99_curve.json, used to judge the GPU throughput path's RMSE.
"""

import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_2204_07104_b200 import ModelConfig, default_init_scale, init_model  # noqa: E402
from paper_2204_07104_b200.synthetic import generate_large  # noqa: E402

epochs = int(sys.argv[1]) if len(sys.argv) > 1 else 5
workers = int(sys.argv[2]) if len(sys.argv) > 2 else 8
dims = (480189, 17770, 2182)
t0 = time.time()
tr, te, _ = generate_large(dims, 99_072_112, (16, 16, 16), 16, 0.1, seed=7, n_test=1_408_395)
gen = time.time() - t0
print("generated", gen, flush=True)
m = init_model(dims, ModelConfig((16, 16, 16), 16, default_init_scale(tr.values, 3), seed=1))
fs = [a.copy() for a in m.factors]
bs = [b.copy() for b in m.core_factors]
t0 = time.time()
rows = O.train(fs, bs, tr.indices, tr.values, te.indices, te.values, epochs=epochs, workers=workers, seed=1,
               alpha_a=0.003, dims=dims)
out = {"dims": dims, "nnz": 99_072_112, "n_test": 1_408_395, "J": 16, "R": 16, "alpha_a": 0.003,
       "workers": workers, "epochs": epochs, "gen_seconds": gen, "train_seconds": time.time() - t0,
       "rows": rows, "engine": "oracle C port (bitwise == reference train)"}
with open(os.path.join(ROOT, "tests", "golden", "nf99_curve.json"), "w") as fh:
    json.dump(out, fh, indent=1)
print(json.dumps(rows), flush=True)

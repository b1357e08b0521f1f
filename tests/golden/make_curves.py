"""Reference RMSE curves for the named BASELINE configs (build container).

    python tests/golden/make_curves.py NAME [NAME ...]
    python tests/golden/make_curves.py --probe NAME ALPHA [ALPHA ...]

Runs the ORACLE C port -- bitwise identical to the reference's train()
(trainer.py:150-271; tests/test_oracle_golden.py pins it against the
reference's own outputs) -- with the reference's DSGD workers on a prefix of
the bench workload of each config (generate_large seed 7: the prefix of a
larger tensor equals the smaller tensor with the same seed), and writes
tests/golden/curve_<NAME>.json: the per-epoch train/test RMSE the GPU
throughput path must match within 1% (tests/test_gpu_curves.py).

--probe runs 3 epochs at each learning rate on a 2M prefix and prints the
test RMSE, to pick a rate at which the reference converges.
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

NF = (480189, 17770, 2182)
Y4 = (1_000_990, 624_961, 3_075, 133)
O6 = (10_000,) * 6

# name -> dims, training nonzeros, test entries, J (= R), alpha_a, epochs
CURVES = {
    "y4_20m": dict(dims=Y4, nnz=20_000_000, n_test=200_000, J=16, alpha_a=0.001, epochs=5),
    "y4_full": dict(dims=Y4, nnz=250_272_286, n_test=2_502_723, J=16, alpha_a=0.001, epochs=5),
    "o6_100m": dict(dims=O6, nnz=100_000_000, n_test=1_000_000, J=8, alpha_a=0.001, epochs=5),
    "o6_10m": dict(dims=O6, nnz=10_000_000, n_test=100_000, J=8, alpha_a=0.001, epochs=5),
    "nf99_j4": dict(dims=NF, nnz=99_072_112, n_test=1_408_395, J=4, alpha_a=0.003, epochs=5),
    "nf99_j8": dict(dims=NF, nnz=99_072_112, n_test=1_408_395, J=8, alpha_a=0.003, epochs=5),
    "nf8m_j4": dict(dims=NF, nnz=8_000_000, n_test=200_000, J=4, alpha_a=0.003, epochs=5),
    "nf8m_j8": dict(dims=NF, nnz=8_000_000, n_test=200_000, J=8, alpha_a=0.003, epochs=5),
    "nf8m_j32": dict(dims=NF, nnz=8_000_000, n_test=200_000, J=32, alpha_a=0.001, epochs=5),
    "nf8m_j64": dict(dims=NF, nnz=8_000_000, n_test=200_000, J=64, alpha_a=0.0003, epochs=5),
}


def run(spec, alpha_a, epochs, nnz=None, workers=8):
    dims, J = spec["dims"], spec["J"]
    order = len(dims)
    nnz = nnz or spec["nnz"]
    t0 = time.time()
    tr, te, _ = generate_large(dims, nnz, (J,) * order, J, 0.1, seed=7, n_test=spec["n_test"])
    gen = time.time() - t0
    m = init_model(dims, ModelConfig((J,) * order, J, default_init_scale(tr.values, order), seed=1))
    fs = [a.copy() for a in m.factors]
    bs = [b.copy() for b in m.core_factors]
    t0 = time.time()
    rows = O.train(fs, bs, tr.indices, tr.values, te.indices, te.values, epochs=epochs, workers=workers,
                   seed=1, alpha_a=alpha_a, dims=dims)
    return rows, gen, time.time() - t0


def main(argv):
    if argv and argv[0] == "--probe":
        spec = CURVES[argv[1]]
        for a in argv[2:]:
            rows, _, secs = run(spec, float(a), 3, nnz=2_000_000)
            print(argv[1], "alpha_a", a, "test_rmse", [round(r["test_rmse"], 4) for r in rows],
                  f"{secs:.0f}s", flush=True)
        return
    for name in argv:
        spec = CURVES[name]
        rows, gen, secs = run(spec, spec["alpha_a"], spec["epochs"])
        out = dict(spec, name=name, R=spec["J"], workers=8, seed_data=7, seed_model=1, seed_train=1,
                   gen_seconds=gen, train_seconds=secs, rows=rows,
                   engine="oracle C port (bitwise == reference train)")
        with open(os.path.join(ROOT, "tests", "golden", f"curve_{name}.json"), "w") as fh:
            json.dump(out, fh, indent=1)
        print(name, json.dumps([round(r["test_rmse"], 5) for r in rows]), f"{secs:.0f}s", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


@pytest.fixture(scope="session")
def golden():
    return np.load(os.path.join(GOLDEN_DIR, "golden.npz"))


@pytest.fixture(scope="session")
def golden_meta():
    with open(os.path.join(GOLDEN_DIR, "golden_meta.json")) as fh:
        return json.load(fh)


def golden_train_case(g, meta, name):
    """(dims, jr, r, train idx/vals, test idx/vals, A0, B0, A_final, B_final, cfg) of a golden run."""
    m = meta[f"train_{name}"]
    order = len(m["dims"])
    A0 = [g[f"train_{name}_A{n}_init"] for n in range(order)]
    B0 = [g[f"train_{name}_B{n}_init"] for n in range(order)]
    A1 = [g[f"train_{name}_A{n}_final"] for n in range(order)]
    B1 = [g[f"train_{name}_B{n}_final"] for n in range(order)]
    return dict(meta=m, order=order, train_idx=g[f"train_{name}_train_idx"],
                train_vals=g[f"train_{name}_train_vals"], test_idx=g[f"train_{name}_test_idx"],
                test_vals=g[f"train_{name}_test_vals"], A0=A0, B0=B0, A1=A1, B1=B1)

import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
from oracle import oracle as O
import test_gpu_kernels as T

for n, d in [(2500, 4000), (60000, 70000), (300000, 400000)]:
    idx, vals, fs, bs = T._model_and_data((d, d, d), (16, 16, 16), 16, n, 3, distinct=True)
    visit = np.arange(len(vals))
    want = None
    for tc in (0, 1, 3):
        got, fac, foff, cor, coff, jr = T._run_factor(idx, vals, fs, bs, visit, 0, False, gam=0.003, tc=tc)
        if want is None:
            want = fac.copy()
            O.factor_pass(idx, vals, visit.astype(np.int64), want, foff, cor, coff, jr, 16, np.full(3, 0.003), np.full(3, 0.01))
        err = np.abs(got - want).max() / np.abs(want).max()
        bad = np.flatnonzero(np.abs(got - want) > 1e-3 * np.abs(want).max())
        print(n, "tc", tc, "max rel err", err, "bad", len(bad), bad[:5], flush=True)

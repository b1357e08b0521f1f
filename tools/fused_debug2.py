"""Two processes (gloo + CUDA IPC on one GPU): which rows of the fused DSGD
result differ from the oracle? (debug)"""
import os
import socket
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import oracle as O  # noqa: E402
from test_gpu_dsgd_fused import _conflict_free, _fused_worker  # noqa: E402

if __name__ == "__main__":
    import torch.multiprocessing as mp

    E = int(os.environ.get("E", "1"))
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    out = "/tmp/fdbg"
    os.makedirs(out, exist_ok=True)
    dims, J, per_block, W = (3000, 2800, 2600), 16, 700, 2
    os.environ["FUSED_EPOCHS"] = str(E)
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=_fused_worker, args=(w, W, port, out, dims, J, per_block)) for w in range(W)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    got = np.load(os.path.join(out, "fac0.npy"))
    from paper_2204_07104_b200 import ModelConfig, init_model
    from paper_2204_07104_b200.dist import DsgdPlan

    idx, vals = _conflict_free(dims, per_block, W, 5)
    model = init_model(dims, ModelConfig((J,) * 3, J, 1.0, seed=1))
    fs = [a.copy() for a in model.factors]
    bs = [b.copy() for b in model.core_factors]
    O.train(fs, bs, idx, vals, epochs=E, workers=W, seed=1, alpha_a=0.003, update_core=False, evaluate=False,
            dims=tuple(dims))
    want, foff = O.pack(fs)
    init, _ = O.pack(model.factors)
    bad = ~np.isclose(got, want, rtol=5e-3, atol=5e-4 * np.abs(want).max())
    plan = DsgdPlan(dims, W)
    print("E", E, "bad", bad.sum(), "of", bad.size, "changed", (~np.isclose(got, init)).sum())
    for n in range(3):
        seg = bad[int(foff[n]): int(foff[n + 1])].reshape(-1, J).any(axis=1)
        for b in range(W):
            lo, hi = plan.rows(n, b)
            print(" mode", n, "block", b, "bad rows", int(seg[lo:hi].sum()), "of", hi - lo)

"""Where do the two-process fused DSGD replicas differ from the oracle? (debug)"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import oracle as O  # noqa: E402
from test_gpu_dsgd_fused import _conflict_free  # noqa: E402


def main():
    from paper_2204_07104_b200 import ModelConfig, SparseTensorCoo, TrainConfig, init_model
    from paper_2204_07104_b200.dsgd_fused import FusedRankRunner
    from paper_2204_07104_b200.training import learning_rate

    prefetch = os.environ.get("PREFETCH", "1") == "1"
    use_epoch = os.environ.get("USE_EPOCH", "1") == "1"
    dims, J, per_block, W, E = (3000, 2800, 2600), 16, 700, 2, int(os.environ.get("E", "2"))
    idx, vals = _conflict_free(dims, per_block, W, 5)
    tensor = SparseTensorCoo(tuple(dims), idx, vals)
    model = init_model(dims, ModelConfig((J,) * 3, J, 1.0, seed=1))
    cfg = TrainConfig(epochs=E, workers=W, seed=1, alpha_a=0.003, update_mode="hogwild", update_core=False)
    streams = [torch.cuda.Stream() for _ in range(W)]
    ranks = []
    for w in range(W):
        with torch.cuda.stream(streams[w]):
            ranks.append(FusedRankRunner(model, tensor, cfg, w, W, prefetch=prefetch))
    torch.cuda.synchronize()
    addrs = [rk.fused.peer_addresses() for rk in ranks]
    for rk in ranks:
        rk.set_peers([a for a, _ in addrs], [b for _, b in addrs])
    plan = ranks[0].plan
    dm0 = ranks[0].dm
    for t in range(E):
        ga = learning_rate(cfg.alpha_a, cfg.beta_a, t)
        gb = learning_rate(cfg.alpha_b, cfg.beta_b, t)
        for w, rk in enumerate(ranks):
            with torch.cuda.stream(streams[w]):
                if use_epoch:
                    rk.epoch(t, ga, gb)
                else:
                    slot = rk._ensure_samples(t)
                    rk.factor_phase(t, ga, slot)
        torch.cuda.synchronize()
        for q, src in enumerate(ranks):
            for n, b in enumerate(plan.held_blocks(q, plan.n_rounds - 1)):
                lo, hi = plan.rows(n, b)
                a, z = int(dm0.foff[n]) + lo * J, int(dm0.foff[n]) + hi * J
                for w, dst in enumerate(ranks):
                    if w != q:
                        dst.dm.fac[a:z].copy_(src.dm.fac[a:z])
        for rk in ranks:
            rk.mark_exchanged(t)
        torch.cuda.synchronize()
    got = ranks[0].dm.fac.double().cpu().numpy()
    fs = [a.copy() for a in model.factors]
    bs = [b.copy() for b in model.core_factors]
    O.train(fs, bs, idx, vals, epochs=E, workers=W, seed=1, alpha_a=0.003, update_core=False, evaluate=False,
            dims=tuple(dims))
    want, _ = O.pack(fs)
    bad = ~np.isclose(got, want, rtol=5e-3, atol=5e-4 * np.abs(want).max())
    print("prefetch", prefetch, "use_epoch", use_epoch, "E", E, "bad", bad.sum(), "of", bad.size)
    for n in range(3):
        seg = bad[int(dm0.foff[n]): int(dm0.foff[n + 1])].reshape(-1, J).any(axis=1)
        for b in range(W):
            lo, hi = plan.rows(n, b)
            print(" mode", n, "block", b, "bad rows", int(seg[lo:hi].sum()), "of", hi - lo)


if __name__ == "__main__":
    main()

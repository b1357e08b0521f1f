"""Small launches of every hot-path kernel family for compute-sanitizer
(racecheck / synccheck / memcheck): tcgen05+TMA factor kernels (tc modes), the
exact predecessor kernel, fused DSGD (two ranks on one GPU), samplers (block
permutation, Fisher-Yates, choice), core pass and evaluation."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402


def main():
    from paper_2204_07104_b200 import (DatasetSplit, ModelConfig, TrainConfig, _lib, default_init_scale, init_model,
                                       train)
    from paper_2204_07104_b200.sampler import choice, permutation
    from paper_2204_07104_b200.synthetic import generate_large

    L = _lib.load()
    which = sys.argv[1] if len(sys.argv) > 1 else "all"
    dims = (3000, 1200, 300)
    tr, te, _ = generate_large(dims, 60_000, (16, 16, 16), 16, 0.1, seed=7, n_test=2000)
    ds = DatasetSplit(tr, te)
    if which in ("all", "factor"):
        for tc in (6, 1, 2, 3, 4):
            L.sptk_set_tc_mode(tc)
            m = init_model(dims, ModelConfig((16, 16, 16), 16, default_init_scale(tr.values, 3), seed=1))
            train(m, ds, TrainConfig(epochs=1, seed=1, alpha_a=0.003, update_mode="hogwild"))
            print("tc", tc, L.sptk_last_factor_kernel().decode(), flush=True)
        L.sptk_set_tc_mode(6)
        for J in (8, 32, 64):
            m = init_model(dims, ModelConfig((J,) * 3, J, default_init_scale(tr.values, 3), seed=1))
            train(m, ds, TrainConfig(epochs=1, seed=1, alpha_a=0.001, update_mode="hogwild", workers=2))
            print("J", J, L.sptk_last_factor_kernel().decode(), flush=True)
    if which in ("all", "exact"):
        m = init_model(dims, ModelConfig((8, 8, 8), 8, default_init_scale(tr.values, 3), seed=1))
        train(m, ds, TrainConfig(epochs=1, seed=1, update_mode="exact", precision="fp64"))
        print("exact", L.sptk_last_factor_kernel().decode(), flush=True)
    if which in ("all", "sampler"):
        permutation([1, 2, 3], 100_000)
        choice([1, 2, 4], 5_000_000, 1 << 16)
        torch.cuda.synchronize()
        print("samplers", flush=True)
    if which in ("all", "fused"):
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        from test_gpu_dsgd_fused import test_two_ranks_one_gpu_match_reference_dsgd

        test_two_ranks_one_gpu_match_reference_dsgd((3000, 2800, 2600), 16, 200)
        print("fused", flush=True)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()

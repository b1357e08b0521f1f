"""The multi-GPU training path (dist.DistRunner: this rank's blocks on the
CUDA kernels + the DSGD exchanges) against the reference's W-worker train().

The GPU box has one B200, so the two ranks share cuda:0 and talk over gloo
(host-staged); the NCCL/NVLink transport is the same DsgdExchange calls."""

import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as td
import torch.multiprocessing as mp

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _case():
    rng = np.random.default_rng(11)
    dims, nnz, J, R = (40, 36, 30), 4000, (4, 3, 5), 4
    idx = np.stack([rng.integers(0, d, nnz) for d in dims], axis=1).astype(np.int64)
    vals = rng.normal(1.0, 0.5, nnz)
    fs = [rng.uniform(0, 0.6, (d, j)) for d, j in zip(dims, J)]
    bs = [rng.uniform(0, 0.6, (j, R)) for j in J]
    return dims, idx, vals, fs, bs


def _worker(rank, world, port, out, cap, mode, precision):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    td.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2204_07104_b200 import DatasetSplit, SparseTensorCoo, TrainConfig, TuckerModel, train

        dims, idx, vals, fs, bs = _case()
        tr = SparseTensorCoo(dims, idx, vals)
        te = SparseTensorCoo(dims, idx[:200], vals[:200])
        model = TuckerModel(dims, tuple(a.shape[1] for a in fs), bs[0].shape[1], [a.copy() for a in fs],
                            [b.copy() for b in bs])
        rows = train(model, DatasetSplit(tr, te),
                     TrainConfig(epochs=2, workers=world, seed=3, core_batch_cap=cap, update_mode=mode,
                                 precision=precision))
        np.savez(os.path.join(out, f"r{rank}.npz"), *model.factors, *model.core_factors,
                 rmse=np.array([r.test_rmse for r in rows]))
    finally:
        td.destroy_process_group()


@pytest.mark.parametrize("cap", [1 << 20, 1500])
def test_dist_runner_exact_fp64_matches_reference_two_workers(cap):
    dims, idx, vals, fs, bs = _case()
    with tempfile.TemporaryDirectory() as out:
        mp.spawn(_worker, args=(2, _free_port(), out, cap, "exact", "fp64"), nprocs=2, join=True)
        got = [np.load(os.path.join(out, f"r{r}.npz")) for r in range(2)]
    ref_f = [a.copy() for a in fs]
    ref_b = [b.copy() for b in bs]
    rows = O.train(ref_f, ref_b, idx, vals, idx[:200], vals[:200], epochs=2, workers=2, seed=3, core_batch_cap=cap)
    for g in got:
        for i, want in enumerate(ref_f + ref_b):
            np.testing.assert_allclose(g[f"arr_{i}"], want, rtol=1e-10, atol=1e-13)
        np.testing.assert_allclose(g["rmse"], [r["test_rmse"] for r in rows], rtol=1e-9)


def test_dist_runner_fp32_rmse_two_workers():
    """Throughput precision (fp32) on the distributed path: test RMSE within 1%
    of the reference's 2-worker run, identical replicas on both ranks."""
    dims, idx, vals, fs, bs = _case()
    with tempfile.TemporaryDirectory() as out:
        mp.spawn(_worker, args=(2, _free_port(), out, 1 << 20, "exact", "fp32"), nprocs=2, join=True)
        got = [np.load(os.path.join(out, f"r{r}.npz")) for r in range(2)]
    rows = O.train([a.copy() for a in fs], [b.copy() for b in bs], idx, vals, idx[:200], vals[:200], epochs=2,
                   workers=2, seed=3)
    for g in got:
        np.testing.assert_allclose(g["rmse"], [r["test_rmse"] for r in rows], rtol=0.01)
    for i in range(6):
        np.testing.assert_array_equal(got[0][f"arr_{i}"], got[1][f"arr_{i}"])

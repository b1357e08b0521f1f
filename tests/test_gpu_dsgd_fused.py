"""Fused multi-GPU DSGD (sptk_factor_pass_dsgd, dsgd_fused.py) with two ranks
sharing one GPU: each rank runs its whole epoch of rounds as one persistent
launch on its own stream, waits on its ready flag for every rotated block and
forwards the block it hands on into the other rank's model by device stores.

On blocks whose samples touch pairwise-distinct rows the Hogwild order does
not matter, so the two ranks' factor phase must equal the reference's
2-worker DSGD factor phase (trainer.py:189-208, the oracle) at the TF32
tolerance of the tcgen05 kernel."""

import numpy as np
import pytest
import torch

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _conflict_free(dims, per_block, m, seed):
    """per_block samples in every DSGD block (m per mode), rows pairwise
    distinct inside each block."""
    from paper_2204_07104_b200.schedule import cut_points

    rng = np.random.default_rng(seed)
    cuts = cut_points(dims, m)
    idx = []
    for key in np.ndindex(*(m,) * len(dims)):
        cols = []
        for n, b in enumerate(key):
            lo, hi = cuts[n][b], cuts[n][b + 1]
            cols.append(lo + rng.permutation(hi - lo)[:per_block])
        idx.append(np.stack(cols, axis=1))
    idx = np.concatenate(idx)
    idx = idx[rng.permutation(len(idx))]
    return idx, rng.normal(2.0, 1.0, len(idx))


@pytest.mark.parametrize("dims,J,per_block", [((3000, 2800, 2600), 16, 700), ((1200, 1100, 1000, 900), 16, 300),
                                               ((3000, 2800, 2600), 8, 700)])
def test_two_ranks_one_gpu_match_reference_dsgd(dims, J, per_block):
    from paper_2204_07104_b200 import ModelConfig, SparseTensorCoo, TrainConfig, init_model
    from paper_2204_07104_b200.dsgd_fused import FusedRankRunner
    from paper_2204_07104_b200.training import learning_rate

    W, E = 2, 2
    order = len(dims)
    idx, vals = _conflict_free(dims, per_block, W, 5)
    tensor = SparseTensorCoo(tuple(dims), idx, vals)
    model = init_model(dims, ModelConfig((J,) * order, J, 1.0, seed=1))
    cfg = TrainConfig(epochs=E, workers=W, seed=1, alpha_a=0.003, update_mode="hogwild", update_core=False)
    streams = [torch.cuda.Stream() for _ in range(W)]
    ranks = []
    for w in range(W):
        with torch.cuda.stream(streams[w]):
            ranks.append(FusedRankRunner(model, tensor, cfg, w, W, prefetch=False))
    torch.cuda.synchronize()
    addrs = [rk.fused.peer_addresses() for rk in ranks]
    for rk in ranks:
        rk.set_peers([a for a, _ in addrs], [b for _, b in addrs])
        rk.fused.grid = 64  # both persistent grids resident on the one GPU
    plan = ranks[0].plan
    dm0 = ranks[0].dm
    for t in range(E):
        ga = learning_rate(cfg.alpha_a, cfg.beta_a, t)
        for w, rk in enumerate(ranks):
            with torch.cuda.stream(streams[w]):
                slot = rk._ensure_samples(t)
        torch.cuda.synchronize()
        for w, rk in enumerate(ranks):
            with torch.cuda.stream(streams[w]):
                rk.factor_phase(t, ga, slot)
        torch.cuda.synchronize()
        # epoch-end exchange: every rank gets the blocks the others hold
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
    assert np.array_equal(got, ranks[1].dm.fac.double().cpu().numpy())
    fs = [a.copy() for a in model.factors]
    bs = [b.copy() for b in model.core_factors]
    O.train(fs, bs, idx, vals, epochs=E, workers=W, seed=1, alpha_a=0.003, update_core=False, evaluate=False,
            dims=tuple(dims))
    want, _ = O.pack(fs)
    init, _ = O.pack(model.factors)
    assert not np.allclose(want, init)
    np.testing.assert_allclose(got, want, rtol=5e-3, atol=5e-4 * np.abs(want).max())
    for rk in ranks:
        assert rk.L.sptk_last_factor_kernel().decode() == "factor_tma_kernel<dsgd>"


def _fused_worker(rank, world, port, out, dims, J, per_block):
    import os

    import torch.distributed as td

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    td.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2204_07104_b200 import ModelConfig, SparseTensorCoo, TrainConfig, init_model
        from paper_2204_07104_b200.dsgd_fused import FusedDistRunner
        from paper_2204_07104_b200.training import learning_rate

        idx, vals = _conflict_free(dims, per_block, world, 5)
        model = init_model(dims, ModelConfig((J,) * len(dims), J, 1.0, seed=1))
        cfg = TrainConfig(epochs=int(os.environ.get("FUSED_EPOCHS", "2")), workers=world, seed=1, alpha_a=0.003,
                          update_mode="hogwild", update_core=False)
        runner = FusedDistRunner(model, SparseTensorCoo(tuple(dims), idx, vals), cfg)
        for t in range(cfg.epochs):
            runner.epoch(t, learning_rate(cfg.alpha_a, cfg.beta_a, t), learning_rate(cfg.alpha_b, cfg.beta_b, t))
        torch.cuda.synchronize()
        np.save(os.path.join(out, f"fac{rank}.npy"), runner.dm.fac.double().cpu().numpy())
        td.barrier()
    finally:
        td.destroy_process_group()


def test_two_processes_ipc_match_reference_dsgd(tmp_path):
    """Two processes (torch.distributed over gloo for the epoch-end exchange)
    sharing cuda:0, each mapping the other's model with CUDA IPC: the
    FusedDistRunner path end to end.  (Without MPS the two persistent kernels
    time-slice the GPU, so the rounds hand over slowly but must still agree.)"""
    import socket

    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    dims, J, per_block, W = (3000, 2800, 2600), 16, 700, 2
    ctx = mp.get_context("spawn")
    procs = [ctx.Process(target=_fused_worker, args=(w, W, port, str(tmp_path), dims, J, per_block))
             for w in range(W)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    alive = [p for p in procs if p.is_alive()]
    for p in alive:
        p.kill()
    assert not alive, "fused DSGD processes did not finish"
    assert all(p.exitcode == 0 for p in procs)
    got = [np.load(tmp_path / f"fac{w}.npy") for w in range(W)]
    assert np.array_equal(got[0], got[1])
    from paper_2204_07104_b200 import ModelConfig, init_model

    idx, vals = _conflict_free(dims, per_block, W, 5)
    model = init_model(dims, ModelConfig((J,) * len(dims), J, 1.0, seed=1))
    fs = [a.copy() for a in model.factors]
    bs = [b.copy() for b in model.core_factors]
    O.train(fs, bs, idx, vals, epochs=2, workers=W, seed=1, alpha_a=0.003, update_core=False, evaluate=False,
            dims=tuple(dims))
    want, _ = O.pack(fs)
    np.testing.assert_allclose(got[0], want, rtol=5e-3, atol=5e-4 * np.abs(want).max())


@pytest.mark.parametrize("dims,J,W", [((3000, 2800, 2600), 16, 4), ((3000, 2800, 2600), 8, 6),
                                      ((1200, 1100, 1000, 900), 16, 4)])
def test_sub_blocked_ranks_use_reference_block_orders(dims, J, W):
    """Two ranks sharing one GPU with W = k * 2 DSGD blocks per mode
    (dsgd_fused.sub_rounds): every W-block's entries appear in the rank's
    visit list in the reference's own order for that block
    (default_rng([seed, 1, t, *b]).permutation, via the pinned oracle), each
    training entry exactly once per epoch; with every row used by one entry
    only (the update order cannot matter) the factors equal the reference's
    W-worker run at TF32 tolerance."""
    from paper_2204_07104_b200 import ModelConfig, SparseTensorCoo, TrainConfig, init_model
    from paper_2204_07104_b200.dsgd_fused import FusedRankRunner
    from paper_2204_07104_b200.training import learning_rate

    M, E, order = 2, 2, len(dims)
    rng = np.random.default_rng(11)
    nnz = 2400 if order == 3 else 800
    idx = np.stack([rng.permutation(d)[:nnz] for d in dims], axis=1)
    vals = rng.normal(2.0, 1.0, nnz)
    tensor = SparseTensorCoo(tuple(dims), idx, vals)
    model = init_model(dims, ModelConfig((J,) * order, J, 1.0, seed=1))
    cfg = TrainConfig(epochs=E, workers=W, seed=1, alpha_a=0.003, update_mode="hogwild", update_core=False)
    streams = [torch.cuda.Stream() for _ in range(M)]
    ranks = []
    for w in range(M):
        with torch.cuda.stream(streams[w]):
            ranks.append(FusedRankRunner(model, tensor, cfg, w, M, prefetch=False))
    torch.cuda.synchronize()
    assert all(rk.m == W for rk in ranks)
    addrs = [rk.fused.peer_addresses() for rk in ranks]
    for rk in ranks:
        rk.set_peers([a for a, _ in addrs], [b for _, b in addrs])
        rk.fused.grid = 64
    plan = ranks[0].plan
    dm0 = ranks[0].dm
    k = W // M
    for t in range(E):
        ga = learning_rate(cfg.alpha_a, cfg.beta_a, t)
        slots = []
        for w, rk in enumerate(ranks):
            with torch.cuda.stream(streams[w]):
                slots.append(rk._ensure_samples(t))
        torch.cuda.synchronize()
        covered = 0
        for w, rk in enumerate(ranks):
            vis = rk.fused.fvis[slots[w]].cpu().numpy().astype(np.int64)
            vis = vis[vis >= 0]
            covered += vis.size
            assert np.unique(vis).size == vis.size
            for b in np.ndindex(*(W,) * order):
                if not (w * k <= b[0] < (w + 1) * k):
                    continue
                off, cnt = rk.part.block_range(b)
                got = vis[(vis >= off) & (vis < off + cnt)] - off
                want = O.permutation([cfg.seed, 1, t, *b], cnt) if cnt else np.zeros(0, np.int64)
                np.testing.assert_array_equal(got, want)
        assert covered == nnz
        for w, rk in enumerate(ranks):
            with torch.cuda.stream(streams[w]):
                rk.factor_phase(t, ga, slots[w])
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
    assert np.array_equal(got, ranks[1].dm.fac.double().cpu().numpy())
    fs = [a.copy() for a in model.factors]
    bs = [b.copy() for b in model.core_factors]
    O.train(fs, bs, idx, vals, epochs=E, workers=W, seed=1, alpha_a=0.003, update_core=False, evaluate=False,
            dims=tuple(dims))
    want, _ = O.pack(fs)
    init, _ = O.pack(model.factors)
    assert not np.allclose(want, init)
    np.testing.assert_allclose(got, want, rtol=5e-3, atol=5e-4 * np.abs(want).max())


def _train_worker(rank, world, port, out, W, cap):
    import os

    import torch.distributed as td

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    td.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2204_07104_b200 import DatasetSplit, ModelConfig, SparseTensorCoo, TrainConfig, init_model, train

        idx, vals, dims = _rows_once()
        model = init_model(dims, ModelConfig((16,) * 3, 16, 1.0, seed=1))
        t = SparseTensorCoo(dims, idx, vals)
        rows = train(model, DatasetSplit(t, SparseTensorCoo(dims, idx[:300], vals[:300])),
                     TrainConfig(epochs=2, workers=W, seed=1, alpha_a=0.003, update_mode="hogwild",
                                 core_batch_cap=cap))
        np.savez(os.path.join(out, f"r{rank}.npz"), *model.factors, *model.core_factors,
                 rmse=np.array([r.test_rmse for r in rows]))
        td.barrier()
    finally:
        td.destroy_process_group()


def _rows_once():
    rng = np.random.default_rng(13)
    dims, nnz = (3000, 2800, 2600), 2400
    idx = np.stack([rng.permutation(d)[:nnz] for d in dims], axis=1)
    return idx, rng.normal(2.0, 1.0, nnz), dims


def test_two_processes_public_train_sub_blocked_with_core_batches(tmp_path):
    """The public train() over two processes (gloo; FusedDistRunner through
    dist.train_distributed) with W = 4 blocks per mode (two per rank's slab)
    and a core batch smaller than the tensor (drawn by one rank per epoch and
    broadcast): both ranks end with the same model, equal to the reference's
    4-worker run at TF32 tolerance (every row used by one entry only, so the
    Hogwild order cannot matter)."""
    import socket

    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    W, cap = 4, 1000
    mp.get_context("spawn")
    mp.spawn(_train_worker, args=(2, port, str(tmp_path), W, cap), nprocs=2, join=True)
    got = [np.load(tmp_path / f"r{r}.npz") for r in range(2)]
    idx, vals, dims = _rows_once()
    from paper_2204_07104_b200 import ModelConfig, init_model

    model = init_model(dims, ModelConfig((16,) * 3, 16, 1.0, seed=1))
    fs = [a.copy() for a in model.factors]
    bs = [b.copy() for b in model.core_factors]
    rows = O.train(fs, bs, idx, vals, idx[:300], vals[:300], epochs=2, workers=W, seed=1, alpha_a=0.003,
                   core_batch_cap=cap, dims=tuple(dims))
    for i in range(6):
        np.testing.assert_array_equal(got[0][f"arr_{i}"], got[1][f"arr_{i}"])
    for i, want in enumerate(fs + bs):
        np.testing.assert_allclose(got[0][f"arr_{i}"], want, rtol=5e-3, atol=5e-4 * np.abs(want).max())
    np.testing.assert_allclose(got[0]["rmse"], [r["test_rmse"] for r in rows], rtol=5e-3)

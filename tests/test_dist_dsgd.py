"""Multi-GPU data division (dist.py) on CPU: the DSGD plan and the gloo-backed
exchanges (rotation, padded all-gather, core all-reduce), driven with the
oracle's per-block kernels, reproduce the reference's W-worker training
(trainer.py:150-271 with workers=W) exactly."""

import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as td
import torch.multiprocessing as mp

from oracle import oracle as O
from paper_2204_07104_b200.dist import DsgdExchange, DsgdPlan


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_plan_round_transfers_are_ring_shifts():
    """Consecutive Gray-code rounds move exactly one mode's blocks, each to a
    neighbouring rank (the NVLink ring shift); mode 0 never moves."""
    for dims, m in [((10, 12, 14), 3), ((9, 9, 9, 9), 2), ((20, 20, 20), 4), ((8, 8, 8, 8, 8), 3)]:
        p = DsgdPlan(dims, m)
        assert p.n_rounds == m ** (len(dims) - 1)
        for r in range(p.n_rounds):
            blocks = [p.block_of(w, r) for w in range(m)]
            for n in range(len(dims)):  # conflict-free: every mode's blocks distinct
                assert sorted(b[n] for b in blocks) == list(range(m))
            assert all(b[0] == w for w, b in enumerate(blocks))
            if r + 1 < p.n_rounds:
                tr = p.transfers(r, r + 1)
                modes = {n for n, _, _, _ in tr}
                assert len(modes) <= 1 and 0 not in modes
                for _, _, src, dst in tr:
                    assert (dst - src) % m in (1, m - 1)


def test_plan_chunks_match_array_split():
    p = DsgdPlan((50, 50, 50), 3)
    for k in [0, 1, 2, 3, 10, 11, 1000]:
        got = [np.arange(lo, hi) for lo, hi in p.chunk_bounds(k)]
        for a, b in zip(got, np.array_split(np.arange(k), 3)):
            assert np.array_equal(a, b)


def _case(seed=5, dims=(23, 19, 17), nnz=1500, J=(3, 4, 2), R=3):
    rng = np.random.default_rng(seed)
    idx = np.stack([rng.integers(0, d, nnz) for d in dims], axis=1).astype(np.int64)
    vals = rng.normal(1.0, 0.5, nnz)
    fs = [rng.uniform(0, 0.7, (d, j)) for d, j in zip(dims, J)]
    bs = [rng.uniform(0, 0.7, (j, R)) for j in J]
    return dims, idx, vals, fs, bs


def _worker(rank, world, port, out, epochs, cap):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    td.init_process_group("gloo", rank=rank, world_size=world)
    try:
        dims, idx, vals, fs, bs = _case()
        order, R = len(dims), bs[0].shape[1]
        fac_np, foff = O.pack(fs)
        cor, coff = O.pack(bs)
        jr = np.array([a.shape[1] for a in fs], dtype=np.int64)
        fac = torch.from_numpy(fac_np)  # shares memory with fac_np
        plan = DsgdPlan(dims, world)
        ex = DsgdExchange(plan, fac, foff, jr)
        blocks = O.block_entries(idx, dims, world)
        nnz, seed = len(vals), 3
        for t in range(epochs):
            ga = O.learning_rate(0.009, 0.05, t)
            gb = O.learning_rate(0.0045, 0.1, t)
            for r in range(plan.n_rounds):
                blk = plan.block_of(rank, r)
                ids = blocks.get(blk)
                if ids is not None and len(ids):
                    visit = np.ascontiguousarray(ids[O.permutation([seed, 1, t, *blk], len(ids))])
                    O.factor_pass(idx, vals, visit, fac_np, foff, cor, coff, jr, R, np.full(order, ga),
                                  np.full(order, 0.01))
                if r + 1 < plan.n_rounds:
                    ex.rotate(r, r + 1)
            ex.gather_all(plan.n_rounds - 1)
            k = min(nnz, cap)
            psi = np.arange(k, dtype=np.int64) if k == nnz else O.choice([seed, 2, t], nnz, k)[0]
            lo, hi = plan.chunk_bounds(k)[rank]
            acc = torch.zeros(int(coff[-1]), dtype=torch.float64)
            O.core_pass(idx, vals, np.ascontiguousarray(psi[lo:hi]), fac_np, foff, cor, coff, jr, R, acc.numpy(),
                        coff)
            ex.allreduce_ordered(acc)
            tot = acc.numpy()
            for n in range(order):
                view = cor[coff[n]: coff[n + 1]].reshape(jr[n], R)
                view -= gb * (tot[coff[n]: coff[n + 1]].reshape(jr[n], R) / k + 0.01 * view)
        np.savez(os.path.join(out, f"r{rank}.npz"), fac=fac_np, cor=cor)
    finally:
        td.destroy_process_group()


@pytest.mark.parametrize("world,cap", [(2, 1 << 20), (3, 1 << 20), (2, 700)])
def test_dsgd_exchange_reproduces_reference_workers(world, cap):
    dims, idx, vals, fs, bs = _case()
    with tempfile.TemporaryDirectory() as out:
        mp.spawn(_worker, args=(world, _free_port(), out, 2, cap), nprocs=world, join=True)
        got = [np.load(os.path.join(out, f"r{r}.npz")) for r in range(world)]
    ref_f = [a.copy() for a in fs]
    ref_b = [b.copy() for b in bs]
    O.train(ref_f, ref_b, idx, vals, epochs=2, workers=world, seed=3, core_batch_cap=cap, evaluate=False)
    want_fac, _ = O.pack(ref_f)
    want_cor, _ = O.pack(ref_b)
    for g in got:  # every rank ends with the full, identical model, bit for bit (rank-order merge)
        assert np.array_equal(g["fac"], want_fac) and np.array_equal(g["cor"], want_cor)


@pytest.mark.parametrize("dims,M,W", [((50, 40, 30), 2, 6), ((20, 18, 16, 14), 2, 4), ((30, 30, 30), 4, 8),
                                      ((40, 30, 20), 2, 2)])
def test_sub_rounds_cover_the_slab_with_row_disjoint_blocks(dims, M, W):
    """dsgd_fused.sub_rounds: rank w's epoch holds every W-block of its
    mode-0 slab exactly once, each inside the M-block of its round, and the k
    W-blocks of a sub-round are row-disjoint in every mode."""
    from paper_2204_07104_b200.dsgd_fused import sub_rounds
    from paper_2204_07104_b200.schedule import cut_points

    plan = DsgdPlan(dims, M)
    k, N = W // M, len(dims)
    cw, cm = cut_points(dims, W), cut_points(dims, M)
    for n in range(N):  # the W-way cut points nest in the M-way ones
        assert all(cw[n][j * k] == cm[n][j] for j in range(M + 1))
    for rank in range(M):
        blocks, groups = sub_rounds(plan, rank, W)
        assert blocks.shape == (plan.n_rounds * k ** (N - 1), k, N)
        assert np.all(np.diff(groups) >= 0) and groups[-1] == plan.n_rounds - 1
        seen = {tuple(b) for b in blocks.reshape(-1, N)}
        assert len(seen) == blocks.shape[0] * k
        want = {b for b in np.ndindex(*(W,) * N) if rank * k <= b[0] < (rank + 1) * k}
        assert seen == want
        for s in range(blocks.shape[0]):
            B = plan.block_of(rank, int(groups[s]))
            for n in range(N):
                assert len(set(blocks[s, :, n])) == k
                assert np.all(blocks[s, :, n] // k == B[n])


def test_block_orders_groups_pad_per_group():
    """BlockOrders.from_arrays(groups=...): rounds of a group lie end to end,
    groups start on multiples of pad and an empty group still takes one unit."""
    from paper_2204_07104_b200.sampler import BlockOrders

    cnts = np.array([[3, 4], [5, 0], [0, 0], [7, 1]])
    offs = np.array([[0, 3], [7, 12], [12, 12], [12, 19]])
    blocks = np.zeros((4, 2, 3), dtype=np.int64)
    bo = BlockOrders.from_arrays(blocks, offs, cnts, 3, "cpu", pad=16, groups=[0, 0, 1, 2])
    assert bo.round_start == [0, 7, 16, 32, 48] and bo.round_end == [7, 12, 16, 40]
    assert bo.group_start == [0, 16, 32, 48] and bo.group_end == [12, 16, 40]
    assert bo.total == 48


def test_hot_row_concurrency_rule():
    """dsgd_fused.hot_row_concurrency: rho = M for every mode a full-grid rank
    keeps at least one sample in flight per row of (NF: the two small modes;
    the 480K-row mode too at M = 8), 1 for small tensors (the launcher's
    Hogwild cap keeps one CTA in flight); with a grid divided by M, rho = 1."""
    from paper_2204_07104_b200.dsgd_fused import hot_row_concurrency

    nf, n = (480189, 17770, 2182), 99_072_112
    np.testing.assert_allclose(hot_row_concurrency(nf, 2, 1, n, n // 2), [1.0, 2.0, 2.0])
    np.testing.assert_allclose(hot_row_concurrency(nf, 8, 1, n, n // 8), [8.0, 8.0, 8.0])
    np.testing.assert_allclose(hot_row_concurrency(nf, 8, 8, n, n // 8), [1.0, 1.0, 1.0], rtol=0.01)
    np.testing.assert_allclose(hot_row_concurrency((3000, 2800, 2600), 2, 1, 2400, 1300), [1.0, 1.0, 1.0])

"""Multi-GPU DSGD with the ring shift fused into the factor kernel.

The reference runs the rounds of its DSGD schedule on W threads with a
barrier per round (trainer.py:189-208; partition.py:100-117): rank w holds
mode-0 block w for good, and between consecutive rounds exactly one mode's
blocks move one rank along the ring.  On B200s that barrier and the move are
the problem (NF at 8 GPUs: 64 rounds of ~20 us of work each), so here every
rank runs its whole epoch of rounds as ONE persistent launch
(sptk_factor_pass_dsgd):

* the rank's visit list holds its block of every round, round after round,
  each round padded to whole 128-sample tiles;
* a tile of round r >= 1 starts once the block rotated in for round r has
  landed (the rank's ready flag, raised by the sender at system scope);
* the CTA that finishes the rank's last tile of round r copies the block the
  rank hands on straight into its next owner's model over NVLink (peer
  stores into memory mapped with CUDA IPC) and raises that rank's flag.

No host round trip, launch or NCCL call per round.  After the epoch's last
round the ranks exchange the blocks they hold (one NCCL all-gather) and
all-reduce the B gradients, as dist.DistRunner does.

``FusedRankRunner`` is transport-agnostic (peer addresses are given); the
tests run two of them on one GPU (two streams, both grids resident) against
the oracle.  ``FusedDistRunner`` is the torch.distributed rank (IPC handles
exchanged with all_gather_object).
"""

from __future__ import annotations

from dataclasses import replace

import numpy as np

from . import _lib
from ._lib import check, ptr, stream_ptr
from .device import SharedBuffer, ipc_open
from .dist import DistRunner, DsgdPlan
from .sampler import BLOCK_PERM_MAX, BlockOrders
from .training import EpochRunner

PUSH_DTYPE = np.dtype([("row_lo", "<i8"), ("nrows", "<i8"), ("mode", "<i8"), ("dst", "<u8"), ("dst_ready", "<u8"),
                       ("dst_gathered", "<u8")])
TILE = 128


def fused_supported(model, config, nnz: int | None = None) -> bool:
    """The fused kernel covers the TMA factor kernel's shapes in throughput
    mode ("auto" resolves by the training-set size, as EpochRunner does)."""
    from .training import resolve_mode

    J = int(model.j_ranks[0])
    mode = config.update_mode
    if mode == "auto":
        mode = "hogwild" if nnz is not None and resolve_mode(mode, nnz) == 0 else "exact"
    return (mode == "hogwild" and config.precision == "fp32"
            and all(int(j) == J for j in model.j_ranks) and J == int(model.r_core)
            and (model.order, J) in ((3, 16), (4, 16), (3, 8), (6, 8)))


FULL_GRID = 560  # the TMA kernel's single-GPU grid at J = 16 (4 CTAs x 148 SMs - 32 sampler slots)


def hot_row_concurrency(dims, m: int, div: int, nnz: int, n_rank: int) -> np.ndarray:
    """rho per mode: in-flight samples per row of one rank of M-way DSGD (its
    grid divided by ``div``, its ``n_rank`` visits, blocks of dims/M rows)
    over those of one GPU running all ``nnz``; 1 where the rank keeps less
    than one sample in flight per row (concurrent updates of a row are then
    rare).  Both grids are capped like the launcher's Hogwild cap
    (common.cuh hogwild_cta_cap: one 128-sample CTA per 64 x 128 visits)."""
    cap = lambda n: max(1, n // (64 * 128))  # noqa: E731
    g1 = min(FULL_GRID, cap(nnz)) * 128
    gr = max(1, -(-min(FULL_GRID, cap(n_rank)) // div)) * 128
    d = np.asarray(dims, dtype=np.float64)
    c1 = g1 / d
    cr = gr / (d / m)
    return np.where(cr >= 1.0, cr / c1, 1.0)


def sub_rounds(plan, rank: int, workers: int):
    """The visit-list layout of one rank's epoch: (blocks [S, k, N], groups [S]).

    M-way DSGD round r gives the rank the block B = plan.block_of(rank, r)
    (partition.py:100-117 at M workers).  With ``workers`` = W = k*M blocks
    per mode (the reference's W-worker division, whose cut points nest in the
    M-way ones: (j*k*d)//(k*M) == (j*d)//M), B is the union of k^N W-blocks;
    they run as k^(N-1) sub-rounds of k row-disjoint W-blocks (b_0 = B_0 k + i,
    b_n = B_n k + (i + s_n) % k), laid end to end inside the round (group r).
    Every W-block keeps the reference's own visit order of the W-worker run
    (default_rng([seed, 1, t, *b]), trainer.py:196-199), so each block fits
    the shared-memory sampler (sptk_block_perm) instead of the whole-slab one.
    k = 1: one block per round (the M-worker run itself)."""
    import itertools

    M, N = plan.m, plan.order
    if workers % M:
        raise ValueError(f"workers={workers} is not a multiple of the {M} ranks")
    k = workers // M
    subs = np.array(list(itertools.product(range(k), repeat=N - 1)), dtype=np.int64).reshape(-1, N - 1)
    i = np.arange(k, dtype=np.int64)
    out, groups = [], []
    for r in range(plan.n_rounds):
        B = np.asarray(plan.block_of(rank, r), dtype=np.int64)
        blk = np.empty((len(subs), k, N), dtype=np.int64)
        blk[:, :, 0] = B[0] * k + i[None, :]
        for n in range(1, N):
            blk[:, :, n] = B[n] * k + (i[None, :] + subs[:, n - 1:n]) % k
        out.append(blk)
        groups.append(np.full(len(subs), r, dtype=np.int64))
    return np.concatenate(out), np.concatenate(groups)


class FusedState:
    """Device state of one rank's fused DSGD factor phase (see module doc)."""

    def __init__(self, runner: EpochRunner, plan: DsgdPlan, rank: int):
        import torch

        self.runner, self.plan, self.rank = runner, plan, rank
        dev = runner.dm.fac.device
        R = plan.n_rounds
        # the rank's block of every round (kept even when empty: its tile is
        # what forwards the block to the next owner)
        blocks, groups = sub_rounds(plan, rank, runner.m)
        W, N = runner.m, runner.order
        keys = (blocks * (W ** np.arange(N - 1, -1, -1, dtype=np.int64))).sum(axis=2)
        offs = runner.part.block_off[keys]
        cnts = runner.part.block_off[keys + 1] - offs
        self.big = int(cnts.max(initial=0)) > BLOCK_PERM_MAX
        self.orders = BlockOrders.from_arrays(blocks, offs, cnts, N, dev, big=self.big, pad=TILE, groups=groups)
        self.total = self.orders.total
        self.fvis = [torch.full((self.total,), -1, dtype=torch.int32, device=dev) for _ in range(2)]
        self.rstart = torch.tensor(self.orders.group_start, dtype=torch.int64, device=dev)
        self.rend = torch.tensor(self.orders.group_end, dtype=torch.int64, device=dev)
        self.done = torch.zeros(R, dtype=torch.int32, device=dev)
        # the model replica other ranks write into, plus this rank's flag
        dm = runner.dm
        fac_bytes = dm.fac.numel() * dm.fac.element_size()
        self.flag_off = (fac_bytes + 255) // 256 * 256
        self.shared = SharedBuffer(self.flag_off + 256)
        fac = self.shared.view(dm.fac.dtype, dm.fac.numel())
        fac.copy_(dm.fac)
        dm.fac = fac
        # flags: [0] ready (rounds landed), [1] epoch (epoch-end exchange of
        # epoch e-1 written: pushes of epoch e may land)
        self.ready = self.shared.view("int32", 1, self.flag_off)
        self.epoch_flag = self.shared.view("int32", 1, self.flag_off + 4)
        self.push = None
        # Hogwild staleness inside a rank: a round's block covers 1/M of every
        # mode's rows, so the single-GPU grid puts M times more samples in
        # flight on each hot row than one GPU running the whole tensor does,
        # and the hot modes' add-reduced deltas (summed over every in-flight
        # sample on a row) overshoot.  Measured on one GPU with the M-worker
        # NF blocks launched one by one (one rank's dynamics at M-GPU DSGD;
        # tools/dsgd_rank_dynamics.py), test RMSE against
        # the reference's 8-worker curve after 5 epochs:
        #   M = 8: full grid (rho = 8) NaN; 1/2 grid NaN; 1/4 grid +1.1%;
        #   1/8 grid +0.3%; full grid with both hot modes' steps x 1/2 +0.6%,
        #   x 1/4 -0.5%, x 1/8 -0.7%; 1/2 grid (rho = 4) x 1/2: +0.01%, but
        #   with only the 2,182-row mode scaled +0.6% (+3.5% after epoch 1);
        #   M = 4 full grid: NaN, x 1/2: -0.03%; M = 2: +1.0%, x 0.71: +0.16%.
        # Repeated runs at a full grid (both hot modes): M = 8 x 0.35: +0.7%
        # and -0.2% (+1.4% / +2.9% after epoch 1), x 0.25: -0.48% twice,
        # x 0.18: -0.6%; M = 4 x 0.5: -0.05% twice, x 0.4: -0.33%; M = 2
        # x 0.71: +0.16%, x 0.63: -0.01%.
        # Rule: each hot mode's step is multiplied by rho^(-2/3) (rho = the
        # rank's in-flight samples per row of that mode over one GPU's,
        # hot_row_concurrency: M at a full grid, 1 for small tensors):
        # 0.63 / 0.40 / 0.25 at M = 2 / 4 / 8.
        # SPTK_DSGD_GRID_DIV (default 1) / SPTK_HOT_STEP_SCALE override.
        import os

        div = int(os.environ.get("SPTK_DSGD_GRID_DIV", 1))
        self.grid = -div if div > 1 else 0
        # 8-way and wider at order 3 / J = 16: one CTA slot per SM left to the
        # rank's samplers (3 factor CTAs per SM; per-rank NF epoch at M = 8
        # 1.715 -> 1.665 ms; at M = 2 / 4 the default 32 free slots are
        # faster: 4.80 vs 5.12, 2.62 vs 2.65 ms).  rho keeps the full grid
        # (the step rule errs on the damped side).
        if (div == 1 and plan.m >= 8 and runner.order == 3 and int(runner.dm.jr[0]) == 16
                and "SPTK_SAMPLER_SLOTS" not in os.environ):
            self.grid = 148 * 3
        self.rho = hot_row_concurrency(plan.dims, plan.m, div, runner.part.nnz, self.total)
        if not runner.hot_step_env:
            runner.hot_step_scale = np.where(runner.hot, np.minimum(1.0, self.rho ** (-2.0 / 3.0)), 1.0)

    # -- peers ---------------------------------------------------------------
    def peer_addresses(self):
        """(fac address, flags address) of this rank's shared buffer."""
        return self.shared.ptr, self.shared.ptr + self.flag_off

    def mark_exchanged(self, t: int) -> None:
        """Epoch t's epoch-end exchange is enqueued on the current stream: once
        it has executed, peers may push epoch t+1's blocks into this replica."""
        check(self.runner.L.sptk_flag_store(ptr(self.epoch_flag), int(t) + 1, stream_ptr()), "sptk_flag_store")

    def set_peers(self, fac_addrs, ready_addrs) -> None:
        """Build the per-round push table from every rank's (mapped) addresses
        (ready_addrs: each rank's flags address; its epoch flag follows)."""
        import torch

        plan, dm = self.plan, self.runner.dm
        R = plan.n_rounds
        tab = np.zeros(R, dtype=PUSH_DTYPE)
        for r in range(R - 1):
            mine = [(n, b, dst) for n, b, src, dst in plan.transfers(r, r + 1) if src == self.rank]
            if len(mine) > 1:
                raise RuntimeError(f"round {r}: rank {self.rank} would send {len(mine)} blocks")
            for n, b, dst in mine:
                lo, hi = plan.rows(n, b)
                J = int(dm.jr[n])
                tab[r] = (lo, hi - lo, n, int(fac_addrs[dst]) + 4 * (int(dm.foff[n]) + lo * J),
                          int(ready_addrs[dst]), int(ready_addrs[dst]) + 4)
        if int(_lib.load().sptk_dsgd_push_bytes()) != PUSH_DTYPE.itemsize:
            raise RuntimeError("DsgdPush layout mismatch between libsptk and dsgd_fused.py")
        self.push = torch.from_numpy(tab.view(np.uint8).copy()).to(self.runner.dm.fac.device)

    # -- visit orders ----------------------------------------------------------
    def draw(self, t: int, slot: int, stream) -> None:
        """This rank's visit list of epoch t into fvis[slot] (padding stays -1)."""
        r = self.runner
        if not self.big:
            self.orders.draw(r.cfg.seed, t, self.fvis[slot], stream=stream)
        else:
            self.orders.interleave(r.perm[slot], r.lo if r.batched_fy else -1, self.fvis[slot], stream=stream)

    def launch(self, t: int, gamma_a: float, slot: int) -> None:
        r, dm = self.runner, self.runner.dm
        if self.push is None:
            raise RuntimeError("set_peers() first")
        r.set_gamma(gamma_a)
        R = self.plan.n_rounds
        check(r.L.sptk_factor_pass_dsgd(ptr(r.part.rec), r.part.rw, ptr(self.fvis[slot]), self.total, ptr(dm.fac),
                                        dm.p_foff, ptr(dm.cor), dm.p_coff, dm.p_jr, r.order, dm.rcore, r.p_gam,
                                        r.p_lam, ptr(self.rstart), ptr(self.rend), ptr(self.push), ptr(self.done),
                                        ptr(self.ready), R, t * R, int(t), int(self.grid), stream_ptr()),
              "sptk_factor_pass_dsgd")


class _FusedMixin:
    """EpochRunner overrides: visit orders into the padded per-rank list, one
    fused launch per epoch instead of one launch (and exchange) per round."""

    fused: FusedState

    def draw_jseq(self, t, slot, stream):
        if not self.fused.big:
            self.j_epoch[slot] = t  # the block CTAs draw their j-sequences themselves
            return
        super().draw_jseq(t, slot, stream)

    def apply_jseq(self, t, slot, stream):
        if self.fused.big:
            super().apply_jseq(t, slot, stream)
        self.fused.draw(t, slot, stream)
        self.sampled_epoch[slot] = t

    def factor_phase(self, t, gamma_a, slot):
        self._fused_t = t
        if self.factor_events is not None:
            e0 = self.torch.cuda.Event(enable_timing=True)
            e0.record()
        self.fused.launch(t, gamma_a, slot)
        if self.factor_events is not None:
            e1 = self.torch.cuda.Event(enable_timing=True)
            e1.record()
            self.factor_events.append((e0, e1))
        self.after_factor_phase()
        return self.nnz_local


class FusedRankRunner(_FusedMixin, EpochRunner):
    """One rank of the fused DSGD epoch without a process group (tests, the
    per-rank simulation): peers are given as device addresses with
    ``set_peers``; the epoch-end block exchange and the B all-reduce are left
    to the caller."""

    def __init__(self, model, train_set, config, rank: int, world: int, prefetch: bool = True):
        if config.workers < world or config.workers % world:
            config = replace(config, workers=world)
        super().__init__(model, train_set, config, prefetch=prefetch, owner_rank=rank, owner_world=world)
        self.rank, self.world = rank, world
        self.plan = DsgdPlan(model.dims, world)
        self.fused = FusedState(self, self.plan, rank)

    def set_peers(self, fac_addrs, ready_addrs):
        self.fused.set_peers(fac_addrs, ready_addrs)

    def mark_exchanged(self, t: int) -> None:
        """Call after the caller's epoch-end exchange of epoch t (stream order)."""
        self.fused.mark_exchanged(t)

    # the core phase as a rank of DistRunner runs it: this rank draws the
    # batches of epochs t = rank (mod W) (the caller hands the others over)
    # and computes the gradient of its chunk of Psi (the caller sums them)
    def draws_psi(self, t):
        return t % self.world == self.rank

    def core_slice(self, slot):
        lo, hi = self.plan.chunk_bounds(self.k)[self.rank]
        if self.k == self.nnz:
            ids = self.torch.arange(lo, hi, dtype=self.torch.int32, device=self.dm.fac.device)
        else:
            ids = self.psi[self.psi_slot][lo:hi]
        return ids, hi - lo, 0


class FusedDistRunner(_FusedMixin, DistRunner):
    """dist.DistRunner with the rounds fused: the ranks map each other's model
    replicas (CUDA IPC over NVLink/NVSwitch) once, then every epoch is one
    launch per rank plus the epoch-end all-gather and B all-reduce."""

    def __init__(self, model, train_set, config, group=None):
        import torch.distributed as td

        super().__init__(model, train_set, config, group, sub_blocks=True)
        self.fused = FusedState(self, self.plan, self.rank)
        self.ex.fac = self.dm.fac  # the exchange works on the shared replica
        mine = (self.fused.shared.ipc_handle(), self.fused.flag_off)
        allh = [None] * self.world
        td.all_gather_object(allh, mine, group=group)
        self._mapped = []
        facs, readys = [], []
        for q, (h, foff) in enumerate(allh):
            if q == self.rank:
                a = self.fused.shared.ptr
            else:
                a = ipc_open(h)
                self._mapped.append(a)
            facs.append(a)
            readys.append(a + foff)
        self.fused.set_peers(facs, readys)
        td.barrier(group=group)

    def after_round(self, r):  # no per-round exchange: the kernel forwards blocks itself
        pass

    def after_factor_phase(self):
        # the epoch-end exchange rewrites this replica; peers' next-epoch
        # pushes wait for the epoch flag raised behind it (stream order)
        super().after_factor_phase()
        self.fused.mark_exchanged(self._fused_t)


__all__ = ["sub_rounds", "hot_row_concurrency", "FusedState", "FusedRankRunner", "FusedDistRunner", "fused_supported"]

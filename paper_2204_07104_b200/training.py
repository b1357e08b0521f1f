"""Epoch driver: the B200 replacement for the reference's ``train`` hot path.

Mirrors sptucker/trainer.py (TrainConfig, MetricsRow, learning_rate, rmse,
mae, frobenius_objective, train, write_metrics_csv) with the same signatures,
defaults, validation messages and metric semantics.  Inside ``train`` every
step of an epoch runs on the GPU, enqueued on one stream with no host
round-trip:

    for each round of the DSGD schedule, for each block      (trainer.py:189-208)
        visit = K2 permutation(default_rng([seed,1,t,*block]))   bit-exact
        K3 factor pass over the block's records in visit order
    core batch Psi = arange / K2 choice(default_rng([seed,2,t]))  (trainer.py:212-221)
    K4 core-gradient reduction over Psi, K5 apply              (trainer.py:222-247)

``wall_seconds`` is device time between CUDA events around that work (the
reference's perf_counter interval, trainer.py:187/249), evaluation excluded.

Update modes (extra TrainConfig fields; the defaults keep the reference's
call signature working):
  update_mode="exact"    the reference's sequential semantics: each visit list
                         is applied in order (conflict-free prefixes run in
                         parallel, identical results), the reference's
                         operation order, the core batch split and merged like
                         np.array_split.  "sequential" is an alias.
  update_mode="hogwild"  throughput: thread-per-sample Hogwild factor kernel
                         over the visit order (cuFastTucker's scheme).
  update_mode="auto"     exact up to 2^22 training nonzeros, hogwild above: on
                         small tensors a GPU's worth of concurrent samples
                         would update every row many times per step.
  precision="fp32"|"fp64"  device arithmetic; fp64 + exact reproduces the
                         reference to rounding.
"""

from __future__ import annotations

import math
import os
import time
import warnings
from dataclasses import dataclass

import numpy as np

from . import _lib, counting
from ._lib import check, f64arr, i64arr, ptr, stream_ptr
from .device import DeviceCoo, DeviceModel, eval_sums, rmse_mae_device
from .sampler import (BLOCK_PERM_MAX, BlockOrders, Workspace, choice, fy_apply, pcg64_state, permutation_j,
                      permutation_j_batch)
from .schedule import DevicePartition, round_blocks, round_schedule
from .tensor import DatasetSplit, SparseTensorCoo
from .tucker import TuckerModel

METRICS_HEADER = "epoch,wall_seconds,train_rmse,train_mae,test_rmse,test_mae,gamma_a,gamma_b"


@dataclass(frozen=True)
class TrainConfig:
    """Schedule, regularisation and parallelism (trainer.py:29-63 defaults)."""

    epochs: int
    workers: int = 1
    update_core: bool = True
    alpha_a: float = 0.009
    beta_a: float = 0.05
    lambda_a: float = 0.01
    alpha_b: float = 0.0045
    beta_b: float = 0.1
    lambda_b: float = 0.01
    core_batch_cap: int = 1 << 20
    seed: int = 0
    eval_every: int = 1
    core_average: bool = True
    update_mode: str = "auto"
    precision: str = "fp32"

    def __post_init__(self):
        if self.epochs < 1:
            raise ValueError("epochs must be >= 1")
        if self.workers < 1:
            raise ValueError("workers must be >= 1")
        for name in ("alpha_a", "beta_a", "lambda_a", "alpha_b", "beta_b", "lambda_b"):
            if getattr(self, name) < 0:
                raise ValueError(f"{name} must be >= 0")
        if self.core_batch_cap < 1:
            raise ValueError("core_batch_cap must be >= 1")
        if self.eval_every < 1:
            raise ValueError("eval_every must be >= 1")
        if self.update_mode not in ("auto", "exact", "sequential", "hogwild"):
            raise ValueError("update_mode must be 'auto', 'exact' (or 'sequential') or 'hogwild'")
        if self.precision not in ("fp32", "fp64"):
            raise ValueError("precision must be 'fp32' or 'fp64'")


@dataclass(frozen=True)
class MetricsRow:
    """One evaluation snapshot; test metrics are NaN without a test set."""

    epoch: int
    wall_seconds: float
    train_rmse: float
    train_mae: float
    test_rmse: float
    test_mae: float
    gamma_a: float
    gamma_b: float


def learning_rate(alpha: float, beta: float, t: int) -> float:
    """alpha / (1 + beta * t^1.5) (trainer.py:80-86)."""
    if alpha < 0 or beta < 0:
        raise ValueError("alpha and beta must be >= 0")
    if t < 0:
        raise ValueError("t must be >= 0")
    return alpha / (1.0 + beta * float(t) ** 1.5)


def _metric(model: TuckerModel, dataset: SparseTensorCoo):
    if dataset.nnz == 0:
        raise ValueError("dataset is empty")
    # fp64 on the device, like the reference's numpy evaluation (trainer.py:89-102)
    return rmse_mae_device(DeviceModel(model, f64=True), DeviceCoo(dataset.indices, dataset.values, f64=True))


def rmse(model: TuckerModel, dataset: SparseTensorCoo) -> float:
    """Root-mean-square error over the dataset (K6 on the device)."""
    return _metric(model, dataset)[0]


def mae(model: TuckerModel, dataset: SparseTensorCoo) -> float:
    """Mean absolute error over the dataset (K6 on the device)."""
    return _metric(model, dataset)[1]


MAX_CORE_ELEMENTS = 10**6


def frobenius_objective(model: TuckerModel, dataset: SparseTensorCoo, lambda_core: float = 0.0,
                        lambda_factors: float = 0.0) -> float:
    """Observed squared loss plus ridge penalties (trainer.py:105-132).

    The squared loss comes from K6; the penalties are small host reductions
    (the core penalty needs the dense core, only formed when prod J_n <= 1e6).
    """
    if dataset.nnz == 0:
        raise ValueError("dataset is empty")
    dm = DeviceModel(model, f64=True)
    total = float(eval_sums(dm, DeviceCoo(dataset.indices, dataset.values, f64=True))[0].item())
    if lambda_core != 0.0:
        if math.prod(model.j_ranks) <= MAX_CORE_ELEMENTS:
            dense = _dense_core(model.core_factors)
            total += lambda_core * float(dense.ravel() @ dense.ravel())
        else:
            warnings.warn("core penalty not computed: dense core exceeds size cap", stacklevel=2)
    if lambda_factors != 0.0:
        total += lambda_factors * sum(float(np.vdot(a, a)) for a in model.factors)
    return total


def _dense_core(core_factors):
    g = None
    for b in core_factors:
        g = b if g is None else np.einsum("...r,jr->...jr", g, b)
    return g.sum(axis=-1)


AUTO_EXACT_MAX_NNZ = 1 << 22


def _env_int(name: str, default: int) -> int:
    """Integer tuning knob from the environment (performance only: results do
    not depend on any of them)."""
    import os

    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def resolve_mode(update_mode: str, nnz: int) -> int:
    """libsptk factor-pass mode: 1 = exact, 0 = hogwild."""
    if update_mode in ("exact", "sequential"):
        return 1
    if update_mode == "hogwild":
        return 0
    return 1 if nnz <= AUTO_EXACT_MAX_NNZ else 0


# --------------------------------------------------------------------------
# device epoch runner
# --------------------------------------------------------------------------
class EpochRunner:
    """Device state for one training run on one GPU (workers = DSGD M).

    Samples depend only on (seed, t, block) (trainer.py:196-199, 213-220), so
    they are drawn ahead on side streams while the main stream runs the factor
    and core phases of epoch t: j-sequences two epochs ahead (``side_j``),
    their application to visit orders one epoch ahead (``side``) and core
    batches two epochs ahead (``side2``).

    Tuning knobs (environment, read once): SPTK_FY_MAIN=1 applies visit orders
    on the main stream instead; SPTK_BATCHED_FY_MIN_BLOCKS (16) is the block
    count from which a process applies all its blocks' orders in one pass.
    """

    def __init__(self, model: TuckerModel, train_set: SparseTensorCoo, config: TrainConfig,
                 prefetch: bool = True, owner_rank: int | None = None, owner_world: int | None = None):
        import torch

        _lib.require_cuda()
        self.torch = torch
        self.cfg = config
        self.f64 = config.precision == "fp64"
        self.mode = resolve_mode(config.update_mode, train_set.nnz)
        self.m = int(config.workers)
        # owner_rank = w: this process runs only the blocks (w, ...) of each
        # round (one GPU of the DSGD data division, dist.py); with owner_world
        # = M < workers (a multiple of M) it runs the workers w*k .. w*k+k-1,
        # k = workers / M: every block of its mode-0 slab (dsgd_fused)
        self.owner_rank = owner_rank
        self.owner_k = 1 if owner_world is None else int(config.workers) // int(owner_world)
        self.order = model.order
        self.nnz = train_set.nnz
        # J = R = 4 in throughput mode on tcgen05: a zero-padded rank-8 model
        # (the smallest TF32 tile; exactly equivalent, see DeviceModel) -- only
        # where a rank-8 tcgen05 kernel exists (orders 3 and 6) and the
        # measured crossover does not put rank 4 on the FMA kernel
        pad = 8 if (not self.f64 and self.mode == 0 and model.r_core == 4 and model.order in (3, 6)
                    and all(int(j) == 4 for j in model.j_ranks) and not _lib.load().sptk_fma_rank(4)) else None
        self.dm = DeviceModel(model, f64=self.f64, pad_rank=pad)
        self.part = DevicePartition(train_set.indices, train_set.values, model.dims, self.m, f64=self.f64,
                                    want_ids=False)
        # the DSGD rounds as arrays: blocks [R, M, N] (worker w's block in
        # round r, partition.py:100-117), their record offsets and sizes
        blocks = round_blocks(model.order, self.m)
        if owner_rank is not None:
            blocks = blocks[:, owner_rank * self.owner_k: (owner_rank + 1) * self.owner_k]
        keys = (blocks * (self.m ** np.arange(model.order - 1, -1, -1, dtype=np.int64))).sum(axis=2)
        self._r_blocks = blocks
        self._r_off = self.part.block_off[keys]
        self._r_cnt = self.part.block_off[keys + 1] - self._r_off
        self._rounds = None
        self.nnz_local = int(self._r_cnt.sum())
        per_round = (self._r_cnt > 0).sum(axis=1)
        max_block = int(self._r_cnt.max(initial=1))
        dev = self.dm.fac.device
        # Flat DSGD (throughput mode, W > 1 workers on one GPU): every block's
        # visit order comes from one shared-memory CTA (sptk_block_perm) and
        # the epoch's factor phase is ONE pass over the rounds' visit lists
        # laid end to end, each round's row-disjoint blocks interleaved -- the
        # reference's W parallel workers per round (trainer.py:189-208).
        self.flat = (self.m > 1 and self.mode == 0 and not self.f64 and owner_rank is None
                     and _env_int("SPTK_FLAT", 1) == 1
                     and int(per_round.max(initial=0)) <= 64 and max_block <= BLOCK_PERM_MAX)
        # Blocks too large for one CTA (NF at W = 16: ~24K nonzeros): their
        # orders come from the batched sampler below and are then interleaved
        # the same way (sptk_interleave_rounds), so the factor phase is still
        # one pass -- per-block launches would put a whole block's samples in
        # flight over its 1/W of the rows (Hogwild contention, divergence).
        self.flat_big = (not self.flat and self.m > 1 and self.mode == 0 and not self.f64 and owner_rank is None
                         and _env_int("SPTK_FLAT", 1) == 1 and int(per_round.max(initial=0)) <= 64)
        self.block_orders = (BlockOrders.from_arrays(blocks, self._r_off, self._r_cnt, self.order, dev,
                                                     big=self.flat_big) if (self.flat or self.flat_big) else None)
        self.fvis = ([torch.empty(max(self.nnz, 1), dtype=torch.int32, device=dev) for _ in range(2)]
                     if self.flat_big else None)
        # Sampler state (K2), double-buffered by epoch parity: Fisher-Yates
        # j-sequences (jbuf), visit orders (perm, laid out like the
        # partitioned records; flat: the epoch's visit list) and core batches (psi).
        self.jbuf = [torch.empty(1 if self.flat else max(self.nnz, 1), dtype=torch.int32, device=dev)
                     for _ in range(2)]
        self.perm = [torch.empty(max(self.nnz, 1), dtype=torch.int32, device=dev) for _ in range(2)]
        self.k = min(self.nnz, int(config.core_batch_cap))
        # core batches run two epochs ahead (the Floyd/Lemire draw is a serial
        # single-CTA walk): three slots
        # (P slots; M processes: M + 2, so that each process can draw its
        # share of the batches -- epochs = rank mod M -- up to M epochs ahead)
        self.P = 3 if owner_world is None else max(3, int(owner_world) + 2)
        self.psi = [torch.zeros(max(self.k, 1), dtype=torch.int32, device=dev) for _ in range(self.P)]
        self.psi_drawn = set()
        # one preallocated workspace per sampler stage (never regrown while a
        # kernel on another stream may still be using it)
        Lb = _lib.load()
        # This process's blocks lie end to end in the partitioned records
        # (block key order, mode 0 most significant), so their visit orders are
        # applied in ONE Fisher-Yates pass over the concatenation
        # (sptk_fy_globalize): the visit entries are then relative to lo.
        nz = self._r_cnt > 0
        order_idx = np.argsort(self._r_off[nz], kind="stable")
        own_off = self._r_off[nz][order_idx]
        own_cnt = self._r_cnt[nz][order_idx]
        self.lo = int(own_off[0]) if own_off.size else 0
        self.hi = int(own_off[-1] + own_cnt[-1]) if own_off.size else 0
        contiguous = bool(np.all(own_off[:-1] + own_cnt[:-1] == own_off[1:]))
        # (measured per-rank DSGD epochs, NF: batching pays from 16 blocks up)
        min_fy = _env_int("SPTK_BATCHED_FY_MIN_BLOCKS", 16)
        self.batched_fy = contiguous and own_off.size > 1 and own_off.size >= min_fy
        if self.batched_fy:
            offs = np.concatenate([own_off - self.lo, [self.hi - self.lo]]).astype(np.int32)
            self.fy_off = torch.from_numpy(offs).to(dev)
        self.ws_j, self.ws_fy, self.ws_psi = Workspace(dev), Workspace(dev), Workspace(dev)
        if self.flat:
            pass
        elif sum(len(items) for items in self.rounds) > 1:
            ns, p_ns = i64arr([c for items in self.rounds for (_, _, c) in items])
            self.ws_j.get(int(Lb.sptk_permutation_j_batch_ws_bytes(p_ns, len(ns))))
        else:
            self.ws_j.get(int(Lb.sptk_permutation_j_ws_bytes(max_block)))
        if not self.flat:
            self.ws_fy.get(int(Lb.sptk_fy_apply_ws_bytes(self.hi - self.lo if self.batched_fy else max_block)))
        if config.update_core and self.k < self.nnz:
            self.ws_psi.get(int(Lb.sptk_choice_ws_bytes(self.nnz, self.k)))
        # exact mode: blocks of at least SPTK_EXACT_DEP_MIN samples (default
        # 2048) run the predecessor-driven kernel (sptk_factor_pass_exact);
        # smaller ones the one-warp conflict-free-prefix walker
        self.dep_min = _env_int("SPTK_EXACT_DEP_MIN", 2048)
        self.ws_dep = None
        if self.mode == 1 and max_block >= self.dep_min:
            self.ws_dep = torch.empty(int(Lb.sptk_factor_pass_exact_ws_bytes(max_block, self.order)),
                                      dtype=torch.uint8, device=dev)
        self.acc = torch.zeros(max(self.dm.cor_size, 1), dtype=torch.float64, device=dev)
        L = _lib.load()
        chunks = self.m if self.mode == 1 else 0
        self.core_ws = torch.empty(int(L.sptk_core_ws_bytes(self.dm.p_jr, self.order, self.dm.rcore, chunks)),
                                   dtype=torch.uint8, device=dev)
        self.gam_np = np.zeros(self.order)
        self.lam_np = np.full(self.order, float(config.lambda_a))
        self._gam, self.p_gam = f64arr(self.gam_np)
        # Hogwild step rule for the add-reduced (hot, < 2^18 rows) modes: the
        # kernel sums the deltas of every in-flight sample on a row, so a
        # launch that puts rho times more samples in flight per hot row than
        # the validated single-GPU pass (a DSGD rank: its block holds 1/M of
        # each mode's rows) scales their step by rho^(-2/3) (dsgd_fused).
        # 1.0 everywhere else; SPTK_HOT_STEP_SCALE overrides (experiments).
        # Per mode, multiplied into gamma_a by set_gamma.
        self.hot = np.array([d < (1 << 18) for d in model.dims], dtype=bool)
        self.hot_step_env = "SPTK_HOT_STEP_SCALE" in os.environ
        env = [float(x) for x in os.environ.get("SPTK_HOT_STEP_SCALE", "1.0").replace(";", ",").split(",")]
        self.hot_step_scale = np.where(self.hot, env if len(env) == model.order else env[0], 1.0)
        self._lam, self.p_lam = f64arr(self.lam_np)
        self.map = self.part.pos_of_id if self.m > 1 else None
        self.L = L
        self.factor_events = None  # optional list: (start, end) CUDA events per factor launch
        # Pipelined sampling: while the main stream trains epoch t,
        #   side_j draws the j-sequences of epoch t+2,
        #   side   applies those of epoch t+1 (visit orders),
        #   side2  draws the core batch of epoch t+1.
        # The j-generation is latency-bound (serial segment resolvers) and the
        # apply is bandwidth-bound, so splitting them across epochs lets both
        # run underneath the factor pass instead of back to back.
        self.prefetch = prefetch
        self.fy_on_main = _env_int("SPTK_FY_MAIN", 0) == 1
        self.burst = prefetch and os.environ.get("SPTK_SCHED", "overlap") == "burst"
        # stream priorities (SPTK_PRIO="j,apply,psi", lower = higher priority).
        # The Fisher-Yates apply bounds the epoch when it shares the GPU with
        # the factor pass; giving it priority measured slower on the NF bench
        # (19.5 vs 19.0 ms per epoch), so all side streams default to 0.
        prio = [int(x) for x in os.environ.get("SPTK_PRIO", "0,0,0").split(",")]
        mk = (lambda pr: torch.cuda.Stream(device=dev, priority=pr)) if prefetch else (lambda pr: None)
        self.side_j, self.side, self.side2 = mk(prio[0]), mk(prio[1]), mk(prio[2])
        ev2 = lambda: [torch.cuda.Event(), torch.cuda.Event()]  # noqa: E731
        self.j_ready, self.j_free, self.perm_ready, self.done = ev2(), ev2(), ev2(), ev2()
        self.psi_ready = [torch.cuda.Event() for _ in range(self.P)]
        self.j_epoch = [None, None]
        self.sampled_epoch = [None, None]
        self.psi_epoch = [None] * self.P
        self.psi_slot = 0
        self.timeline = None  # set to [] to record per-epoch stream timelines (synchronises)
        self._marks = []
        # experiment hook (wrong results): SPTK_EXP_SKIP=psi,jseq,perm re-uses a
        # sampler stage's previous output instead of drawing it again, to measure
        # what that stage's co-running costs the epoch
        self._skip = set(filter(None, os.environ.get("SPTK_EXP_SKIP", "").split(",")))
        if self._skip:
            warnings.warn(f"SPTK_EXP_SKIP={sorted(self._skip)}: sampler stages re-use stale samples "
                          "(timing experiment; results are not the reference's)", stacklevel=2)

    @property
    def rounds(self):
        """Host list of (block, offset, count) per round, empty blocks dropped
        (built on first use: the flat paths work from the arrays)."""
        if self._rounds is None:
            self._rounds = [[(tuple(b), o, c) for b, o, c in zip(bl, of, cn) if c > 0]
                            for bl, of, cn in zip(self._r_blocks.tolist(), self._r_off.tolist(),
                                                  self._r_cnt.tolist())]
        return self._rounds

    # -- samplers (K2) -----------------------------------------------------
    def draw_core_batch(self, t: int, stream) -> None:
        """Core batch Psi of epoch t (trainer.py:212-220) into psi[t % P]:
        drawn here unless drawn ahead (draw_psi), then shared (share_psi)."""
        cfg = self.cfg
        if "psi" in self._skip and self.psi_epoch[t % self.P] is not None:
            self.psi_epoch[t % self.P] = t
            return
        self.draw_psi(t, stream)
        if cfg.update_core and self.k < self.nnz:
            self.share_psi(t, stream)
        self.psi_drawn.discard(t)
        self.psi_epoch[t % self.P] = t

    def draw_psi(self, t: int, stream) -> None:
        """This process's draw of epoch t's core batch (if it draws it)."""
        cfg = self.cfg
        if cfg.update_core and self.k < self.nnz and self.draws_psi(t) and t not in self.psi_drawn:
            choice(None, self.nnz, self.k, shuffle=(self.mode == 1), out=self.psi[t % self.P], ws=self.ws_psi,
                   state=pcg64_state([cfg.seed, 2, t]), stream=stream)
            self.psi_drawn.add(t)

    def draws_psi(self, t: int) -> bool:
        """Whether this process draws the core batch of epoch t itself."""
        return True

    def share_psi(self, t: int, stream) -> None:
        """Hand the core batch of epoch t to the processes that did not draw it."""

    def draw_jseq(self, t: int, slot: int, stream) -> None:
        """Fisher-Yates j-sequences of every (own) block of epoch t:
        default_rng([seed,1,t,*block]).permutation(len(ids)), first half
        (trainer.py:196-199).  Several blocks (DSGD) are drawn as one batch:
        their segment levels advance together, one launch per phase."""
        cfg = self.cfg
        if self.flat or ("jseq" in self._skip and self.j_epoch[slot] is not None):
            # (flat: the block CTAs draw their j-sequences themselves)
            self.j_epoch[slot] = t
            return
        items = [it for rnd in self.rounds for it in rnd]
        if len(items) == 1:
            block, off, cnt = items[0]
            permutation_j(None, cnt, out=self.jbuf[slot][off:off + cnt], ws=self.ws_j,
                          state=pcg64_state([cfg.seed, 1, t, *block]), stream=stream)
        elif items:
            states = np.stack([pcg64_state([cfg.seed, 1, t, *block]) for block, _, _ in items])
            permutation_j_batch(states, [c for _, _, c in items], [o for _, o, _ in items], self.jbuf[slot],
                                ws=self.ws_j, stream=stream)
        self.j_epoch[slot] = t

    def apply_jseq(self, t: int, slot: int, stream) -> None:
        """The visit orders of epoch t from its j-sequences (second half)."""
        if "perm" in self._skip and self.sampled_epoch[slot] is not None:
            self.sampled_epoch[slot] = t
            return
        if self.flat:
            self.block_orders.draw(self.cfg.seed, t, self.perm[slot], stream=stream)
        elif self.batched_fy:
            lo, hi = self.lo, self.hi
            j = self.jbuf[slot][lo:hi]
            check(self.L.sptk_fy_globalize(ptr(j), ptr(self.fy_off), self.fy_off.numel() - 1, stream_ptr(stream)),
                  "sptk_fy_globalize")
            fy_apply(j, hi - lo, out=self.perm[slot][lo:hi], ws=self.ws_fy, stream=stream)
            if self.flat_big:
                self.block_orders.interleave(self.perm[slot], lo, self.fvis[slot], stream=stream)
        else:
            for items in self.rounds:
                for block, off, cnt in items:
                    fy_apply(self.jbuf[slot][off:off + cnt], cnt, out=self.perm[slot][off:off + cnt], ws=self.ws_fy,
                             stream=stream)
            if self.flat_big:
                self.block_orders.interleave(self.perm[slot], -1, self.fvis[slot], stream=stream)
        self.sampled_epoch[slot] = t

    def draw_samples(self, t: int, slot: int, stream) -> None:
        """Visit orders of every block and the core batch of epoch t, in order on one stream."""
        if self.psi_epoch[t % self.P] != t:
            self.draw_core_batch(t, stream)
        self.draw_jseq(t, slot, stream)
        self.apply_jseq(t, slot, stream)

    def _ensure_samples(self, t: int) -> int:
        torch = self.torch
        slot, o = t % 2, 1 - t % 2
        main = torch.cuda.current_stream()
        E = self.cfg.epochs
        P = self.P
        self.psi_slot = t % P
        if self.sampled_epoch[slot] != t:
            if self.psi_epoch[t % P] == t:
                main.wait_event(self.psi_ready[t % P])
            self.draw_samples(t, slot, main)
            self.j_free[slot].record(main)
            if self.prefetch:  # the side stages reuse the same workspaces
                ev = torch.cuda.Event()
                ev.record(main)
                for st in (self.side_j, self.side, self.side2):
                    st.wait_event(ev)
        else:
            main.wait_event(self.perm_ready[slot])
            main.wait_event(self.psi_ready[t % P])
        if not self.prefetch:
            return slot
        # core batches: epoch t+1's is completed (drawn if not yet, shared)
        # and later ones this process draws are drawn ahead, up to t+P-1
        for e in range(t + 1, min(t + P, E)):
            if self.psi_epoch[e % P] == e or (e > t + 1 and (e in self.psi_drawn or not self.draws_psi(e))):
                continue
            # psi[e % P] was last read by epoch e - P (its `done` parity slot
            # holds that epoch's event or a later one)
            self.side2.wait_event(self.done[(e - P) % 2])
            self._mark(f"psi{e - t}_start", self.side2)
            if e == t + 1:
                self.draw_core_batch(e, self.side2)
                self.psi_ready[e % P].record(self.side2)
            else:
                self.draw_psi(e, self.side2)
            self._mark(f"psi{e - t}_end", self.side2)
        if t + 1 < E and self.sampled_epoch[o] != t + 1:
            if self.j_epoch[o] != t + 1:
                self.side_j.wait_event(self.j_free[o])
                self._mark("jseq_start", self.side_j)
                self.draw_jseq(t + 1, o, self.side_j)
                self._mark("jseq_end", self.side_j)
                self.j_ready[o].record(self.side_j)
            # perm[o] was last read by epoch t-1 (`done`).  The apply runs on
            # the main stream ahead of this epoch's factor pass (fy_on_main) or
            # beside it on its own stream.
            st = main if self.fy_on_main else self.side
            st.wait_event(self.done[o])
            st.wait_event(self.j_ready[o])
            self._mark("perm_start", st)
            self.apply_jseq(t + 1, o, st)
            self._mark("perm_end", st)
            self.j_free[o].record(st)
            self.perm_ready[o].record(st)
        if t + 2 < E and self.j_epoch[slot] != t + 2:
            # jbuf[slot] is free once epoch t's apply has read it
            self.side_j.wait_event(self.j_free[slot])
            self._mark("jseq2_start", self.side_j)
            self.draw_jseq(t + 2, slot, self.side_j)
            self._mark("jseq2_end", self.side_j)
            self.j_ready[slot].record(self.side_j)
        if self.burst:
            # burst schedule (SPTK_SCHED=burst, with SPTK_TC_CTAS=4): this
            # epoch's factor pass starts once the sampler stages just enqueued
            # (apply t+1, j-sequences and core batch t+2) are done; they run
            # side by side, then the factor pass has every CTA slot.  Measured
            # 21.1 vs 19.1 ms per NF epoch: the latency-bound j-sequence levels
            # take ~10 ms beside the apply, so the default overlaps them with
            # the factor pass instead.
            for st in (self.side, self.side_j, self.side2):
                ev = torch.cuda.Event()
                ev.record(st)
                main.wait_event(ev)
        return slot

    # -- optional per-epoch stream timeline (timeline = [] to enable) --------
    def _mark(self, name, stream=None):
        if self.timeline is None:
            return
        ev = self.torch.cuda.Event(enable_timing=True)
        ev.record(stream if stream is not None else self.torch.cuda.current_stream())
        self._marks.append((name, ev))

    def _flush_timeline(self, t):
        if self.timeline is None or not self._marks:
            return
        self._marks[-1][1].synchronize()
        self.torch.cuda.synchronize()
        t0 = self._marks[0][1]
        self.timeline.append({"epoch": t, **{n: round(t0.elapsed_time(e), 3) for n, e in self._marks}})
        self._marks = []

    # -- K3 / K4 / K5 ------------------------------------------------------
    def set_gamma(self, gamma_a: float) -> None:
        """Per-mode factor steps of this epoch (hot modes x hot_step_scale)."""
        self._gam[:] = gamma_a
        if self.mode == 0:
            self._gam[:] *= self.hot_step_scale

    def factor_phase(self, t: int, gamma_a: float, slot: int) -> int:
        L, dm = self.L, self.dm
        self.set_gamma(gamma_a)
        fn = L.sptk_factor_pass_f64 if self.f64 else L.sptk_factor_pass
        s = stream_ptr()
        processed = 0
        if self.flat or self.flat_big:
            if self.factor_events is not None:
                e0 = self.torch.cuda.Event(enable_timing=True)
                e0.record()
            vis = self.fvis[slot] if self.flat_big else self.perm[slot]
            check(fn(ptr(self.part.rec), self.part.rw, ptr(vis), self.nnz, 0, ptr(dm.fac), dm.p_foff,
                     ptr(dm.cor), dm.p_coff, dm.p_jr, self.order, dm.rcore, self.p_gam, self.p_lam, self.mode, s),
                  "sptk_factor_pass")
            if self.factor_events is not None:
                e1 = self.torch.cuda.Event(enable_timing=True)
                e1.record()
                self.factor_events.append((e0, e1))
            self.after_factor_phase()
            return self.nnz
        for r, items in enumerate(self.rounds):
            for block, off, cnt in items:
                if self.factor_events is not None:
                    e0 = self.torch.cuda.Event(enable_timing=True)
                    e0.record()
                rec, visit = self.part.rec, self.perm[slot][off:off + cnt]
                vbase = self.lo if self.batched_fy else off  # visit entries are relative to vbase
                if self.ws_dep is not None and cnt >= self.dep_min:
                    # exact mode across the GPU (predecessor-driven schedule)
                    fx = L.sptk_factor_pass_exact_f64 if self.f64 else L.sptk_factor_pass_exact
                    check(fx(ptr(rec), self.part.rw, ptr(visit), cnt, vbase, ptr(dm.fac), dm.p_foff, ptr(dm.cor),
                             dm.p_coff, dm.p_jr, self.order, dm.rcore, self.p_gam, self.p_lam, ptr(self.ws_dep),
                             self.ws_dep.numel(), s), "sptk_factor_pass_exact")
                else:
                    check(fn(ptr(rec), self.part.rw, ptr(visit), cnt, vbase, ptr(dm.fac), dm.p_foff, ptr(dm.cor),
                             dm.p_coff, dm.p_jr, self.order, dm.rcore, self.p_gam, self.p_lam, self.mode, s),
                          "sptk_factor_pass")
                if self.factor_events is not None:
                    e1 = self.torch.cuda.Event(enable_timing=True)
                    e1.record()
                    self.factor_events.append((e0, e1))
                processed += cnt
            self.after_round(r)
        self.after_factor_phase()
        return processed

    # -- hooks for the multi-GPU data division (dist.DistRunner) ------------
    def after_round(self, r: int) -> None:
        """Called after round r's blocks are enqueued (A-block rotation)."""

    def after_factor_phase(self) -> None:
        """Called after the last round (A-block allgather)."""

    def core_slice(self, slot: int):
        """(visit ids or None, count, exact chunk count) of this process's share of Psi."""
        k = self.k
        return (None if k == self.nnz else self.psi[self.psi_slot][:k]), k, (self.m if self.mode == 1 else 0)

    def reduce_core_acc(self) -> None:
        """Sum the core-gradient accumulators over processes (allreduce)."""

    def core_phase(self, t: int, gamma_b: float, slot: int) -> None:
        cfg, L, dm = self.cfg, self.L, self.dm
        k = self.k
        visit, count, chunks = self.core_slice(slot)
        self.acc.zero_()
        s = stream_ptr()
        fn = L.sptk_core_pass_f64 if self.f64 else L.sptk_core_pass
        if count > 0:
            check(fn(ptr(self.part.rec), self.part.rw, ptr(visit), ptr(self.map), count, ptr(dm.fac), dm.p_foff,
                     ptr(dm.cor), dm.p_coff, dm.p_jr, self.order, dm.rcore, ptr(self.acc), chunks,
                     ptr(self.core_ws), self.core_ws.numel(), s), "sptk_core_pass")
        self.reduce_core_acc()
        denom = float(k) if cfg.core_average else 1.0
        ap = L.sptk_core_apply_f64 if self.f64 else L.sptk_core_apply
        check(ap(ptr(dm.cor), ptr(self.acc), dm.cor_size, float(gamma_b), float(cfg.lambda_b), denom, s),
              "sptk_core_apply")

    def epoch(self, t: int, gamma_a: float, gamma_b: float) -> None:
        self._mark("epoch_start")
        slot = self._ensure_samples(t)
        self._mark("factor_start")
        processed = self.factor_phase(t, gamma_a, slot)
        if processed != self.nnz_local:
            raise RuntimeError("partition did not cover every training entry")
        self._mark("factor_end")
        if self.cfg.update_core:
            self.core_phase(t, gamma_b, slot)
        self._mark("epoch_end")
        self.done[slot].record(self.torch.cuda.current_stream())
        self._flush_timeline(t)


def train(model: TuckerModel, split: DatasetSplit, config: TrainConfig) -> list[MetricsRow]:
    """Run the epochs in place on ``model``; returns the metric rows.

    Same contract as trainer.train (trainer.py:150-271); the epoch work runs on
    the current CUDA device.
    """
    train_set = split.train
    if train_set.dims != model.dims:
        raise ValueError("model dims do not match dataset dims")
    if train_set.nnz == 0:
        raise ValueError("training set is empty")
    w = config.workers
    if w > min(model.dims):
        raise ValueError(f"workers={w} cannot partition dims {model.dims}")
    import torch

    from . import dist

    if dist.active():
        return dist.train_distributed(model, split, config)
    runner = EpochRunner(model, train_set, config)
    f64 = runner.f64
    # evaluation sets: the training records are reused (all blocks); test packed once
    test_coo = DeviceCoo(split.test.indices, split.test.values, f64=f64) if split.test.nnz else None
    train_eval = _RecordView(runner.part)
    rows: list[MetricsRow] = []
    wall = 0.0
    pending = []
    for t in range(config.epochs):
        ga = learning_rate(config.alpha_a, config.beta_a, t)
        gb = learning_rate(config.alpha_b, config.beta_b, t)
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record()
        runner.epoch(t, ga, gb)
        ev1.record()
        pending.append((ev0, ev1))
        if counting.counter.enabled:
            counting.counter.add(counting.epoch_multiplies(model.j_ranks, model.r_core, runner.nnz_local,
                                                           runner.k if config.update_core else 0))
        if (t + 1) % config.eval_every == 0 or t == config.epochs - 1:
            ev1.synchronize()
            for a, b in pending:
                wall += a.elapsed_time(b) / 1000.0
            pending.clear()
            tr = rmse_mae_device(runner.dm, train_eval)
            te = rmse_mae_device(runner.dm, test_coo) if test_coo is not None else (math.nan, math.nan)
            rows.append(MetricsRow(t + 1, wall, tr[0], tr[1], te[0], te[1], ga, gb))
    runner.dm.download_into(model)
    return rows


class _RecordView:
    """Adapter so the partitioned training records can be scored by K6."""

    def __init__(self, part: DevicePartition):
        self.rec = part.rec
        self.rw = part.rw
        self.nnz = part.nnz
        self.order = part.order


def write_metrics_csv(rows, path) -> None:
    """CSV in the fixed column order (trainer.py:274-282)."""
    out = [METRICS_HEADER]
    for r in rows:
        out.append(",".join([str(r.epoch)] + [repr(v) for v in (r.wall_seconds, r.train_rmse, r.train_mae,
                                                                 r.test_rmse, r.test_mae, r.gamma_a,
                                                                 r.gamma_b)]))
    with open(path, "w") as fh:
        fh.write("\n".join(out) + "\n")

"""Multi-GPU data division: the reference's DSGD schedule across processes.

The reference runs the conflict-free block schedule on W threads over one
shared model (trainer.py:189-208, partition.py:100-117; paper section 4.3,
PAPER.md:813-856).  Here every worker is a process with its own GPU, and the
shared memory becomes explicit, minimal exchanges over NCCL (NVLink /
NVSwitch):

* mode 0 is stationary: rank w owns mode-0 row block w and runs the blocks
  (w, b_1, ..., b_{N-1}) of each round on its GPU;
* after round r, every mode-n block whose owner changes between r and r+1
  moves from its old owner to its new one (point-to-point send/recv).  The
  rounds follow a reflected Gray code, so consecutive rounds move exactly one
  mode's blocks, each by one rank: a ring shift (``DsgdPlan.transfers``);
* after the last round every rank contributes the blocks it holds to one
  padded all-gather, so all ranks hold the full post-factor-phase A for the
  core phase and evaluation (the reference's threads read the shared arrays);
* the core batch Psi is split like ``np.array_split(psi, W)`` (trainer.py:221);
  rank w accumulates chunk w and the N*J*R fp64 accumulators are all-reduced
  (the reference sums the chunk accumulators, trainer.py:238-240); every rank
  then applies the identical B update.

Each rank computes only its own blocks' visit orders (the per-block seeds
[seed, 1, t, *block] make them independent of the worker count), so the data
path has no collective beyond the rotation, the A all-gather and the 3 KB
B-gradient all-reduce.  ``DsgdPlan`` and ``DsgdExchange`` are device-agnostic
(CPU tensors over gloo in the tests, CUDA tensors over NCCL in training).
"""

from __future__ import annotations

import math
from dataclasses import replace

from .schedule import cut_points, round_schedule
from .training import EpochRunner


def active() -> bool:
    try:
        import torch.distributed as td
    except Exception:  # pragma: no cover
        return False
    return td.is_available() and td.is_initialized() and td.get_world_size() > 1


class DsgdPlan:
    """Host-side bookkeeping of the DSGD data division (pure Python)."""

    def __init__(self, dims, m: int):
        self.dims = tuple(int(d) for d in dims)
        self.order = len(self.dims)
        self.m = int(m)
        if self.m < 1 or self.m > min(self.dims):
            raise ValueError(f"cannot divide dims {self.dims} among {self.m} workers")
        self.cuts = cut_points(self.dims, self.m)
        self.rounds = round_schedule(self.order, self.m).rounds

    @property
    def n_rounds(self) -> int:
        return len(self.rounds)

    def block_of(self, rank: int, r: int) -> tuple:
        """The block rank runs in round r (worker w owns (w, (w+d_1)%M, ...))."""
        return self.rounds[r][rank]

    def owner(self, r: int, n: int, b: int) -> int:
        """Rank that holds mode-n block b during round r."""
        for w, blk in enumerate(self.rounds[r]):
            if blk[n] == b:
                return w
        raise ValueError("block not scheduled")  # pragma: no cover

    def rows(self, n: int, b: int) -> tuple[int, int]:
        """Row range [lo, hi) of mode-n block b (partition.py:55-57 cut points)."""
        return self.cuts[n][b], self.cuts[n][b + 1]

    def max_rows(self, n: int) -> int:
        return max(self.cuts[n][b + 1] - self.cuts[n][b] for b in range(self.m))

    def transfers(self, r0: int, r1: int) -> list[tuple[int, int, int, int]]:
        """(mode, block, src, dst) for every block that changes owner r0 -> r1."""
        out = []
        for n in range(1, self.order):
            for b in range(self.m):
                src, dst = self.owner(r0, n, b), self.owner(r1, n, b)
                if src != dst:
                    out.append((n, b, src, dst))
        return out

    def held_blocks(self, rank: int, r: int) -> tuple:
        """Blocks (one per mode) whose freshest copy rank holds after round r."""
        return self.rounds[r][rank]

    def chunk_bounds(self, k: int) -> list[tuple[int, int]]:
        """np.array_split(arange(k), M) boundaries (trainer.py:221)."""
        q, rem = divmod(int(k), self.m)
        out, pos = [], 0
        for c in range(self.m):
            ln = q + (1 if c < rem else 0)
            out.append((pos, pos + ln))
            pos += ln
        return out


class DsgdExchange:
    """The data movement of the DSGD schedule on one flat factor buffer.

    ``fac`` is the rank's full copy of the packed factors (reference layout,
    _loops.py:8-10: A(n) row i at fac[foff[n] + i*J_n]); every transfer is a
    contiguous row range of one mode.
    """

    def __init__(self, plan: DsgdPlan, fac, foff, jr, group=None):
        import torch
        import torch.distributed as td

        self.td = td
        self.torch = torch
        self.plan = plan
        self.fac = fac
        self.foff = [int(x) for x in foff]
        self.jr = [int(x) for x in jr]
        self.group = group
        self.rank = td.get_rank(group)
        self.world = td.get_world_size(group)
        if self.world != plan.m:
            raise ValueError(f"world size {self.world} != DSGD workers {plan.m}")
        self.nccl = td.get_backend(group) == "nccl"
        # padded all-gather layout: mode n block at pad_off[n], max_rows(n)*J_n floats
        self.pad_off = [0]
        for n in range(plan.order):
            self.pad_off.append(self.pad_off[-1] + plan.max_rows(n) * self.jr[n])
        # establishes the communicator before the first point-to-point exchange
        td.barrier(group=group)
        self.sendbuf = torch.zeros(self.pad_off[-1], dtype=fac.dtype, device=fac.device)
        self.gathered = torch.zeros(self.world * self.pad_off[-1], dtype=fac.dtype, device=fac.device)

    def rows_view(self, n: int, b: int):
        lo, hi = self.plan.rows(n, b)
        j = self.jr[n]
        return self.fac[self.foff[n] + lo * j: self.foff[n] + hi * j]

    def rotate(self, r0: int, r1: int) -> int:
        """Move every block whose owner changes between rounds r0 and r1; returns bytes sent."""
        td = self.td
        ops, sent = [], 0
        for n, b, src, dst in self.plan.transfers(r0, r1):
            if src == self.rank:
                v = self.rows_view(n, b)
                if v.numel():
                    ops.append(td.P2POp(td.isend, v, dst, self.group))
                    sent += v.numel() * v.element_size()
            elif dst == self.rank:
                v = self.rows_view(n, b)
                if v.numel():
                    ops.append(td.P2POp(td.irecv, v, src, self.group))
        if ops:
            if self.nccl:
                for req in td.batch_isend_irecv(ops):
                    req.wait()
            else:
                # gloo: point-to-point on host tensors (device buffers staged)
                staged = [(op, op.tensor if op.tensor.device.type == "cpu" else op.tensor.cpu()) for op in ops]
                reqs = [op.op(h, op.peer, group=self.group) for op, h in staged]
                for req in reqs:
                    req.wait()
                for op, h in staged:
                    if op.op is td.irecv and h is not op.tensor:
                        op.tensor.copy_(h)
        return sent

    def gather_all(self, r_last: int) -> None:
        """All ranks end up with the freshest copy of every block (padded all-gather)."""
        td = self.td
        plan = self.plan
        for n in range(plan.order):
            v = self.rows_view(n, plan.held_blocks(self.rank, r_last)[n])
            self.sendbuf[self.pad_off[n]: self.pad_off[n] + v.numel()].copy_(v)
        if self.nccl:
            td.all_gather_into_tensor(self.gathered, self.sendbuf, group=self.group)
        else:
            host = self.gathered.cpu()
            parts = list(host.view(self.world, -1).unbind(0))
            td.all_gather(parts, self.sendbuf.cpu(), group=self.group)
            if host is not self.gathered:
                self.gathered.copy_(host)
        g = self.gathered.view(self.world, -1)
        for q in range(self.world):
            if q == self.rank:
                continue
            for n in range(plan.order):
                v = self.rows_view(n, plan.held_blocks(q, r_last)[n])
                v.copy_(g[q, self.pad_off[n]: self.pad_off[n] + v.numel()])

    def allreduce_ordered(self, t) -> None:
        """t <- t_0 + t_1 + ... + t_{W-1} added in rank order, on every rank:
        the reference's merge of the chunk accumulators (trainer.py:238-240,
        total = acc_0 + acc_1 + ...), so exact mode stays bitwise for any W
        (an all-reduce may group the sums differently)."""
        td = self.td
        if self.nccl or t.device.type == "cpu":
            parts = [self.torch.empty_like(t) for _ in range(self.world)]
            td.all_gather(parts, t, group=self.group)
        else:
            h = t.cpu()
            parts = [self.torch.empty_like(h) for _ in range(self.world)]
            td.all_gather(parts, h, group=self.group)
            parts = [p_.to(t.device) for p_ in parts]
        total = parts[0].clone()
        for q in range(1, self.world):
            total += parts[q]
        t.copy_(total)

    def allreduce(self, t) -> None:
        if self.nccl or t.device.type == "cpu":
            self.td.all_reduce(t, group=self.group)
        else:
            h = t.cpu()
            self.td.all_reduce(h, group=self.group)
            t.copy_(h)


class DistRunner(EpochRunner):
    """One rank of multi-GPU training: EpochRunner restricted to this rank's
    blocks, with the DSGD exchanges in its round / phase hooks."""

    def __init__(self, model, train_set, config, group=None, sub_blocks: bool = False):
        import torch.distributed as td

        rank, world = td.get_rank(group), td.get_world_size(group)
        # sub_blocks (the fused runner): workers = k * world keeps the
        # reference's W-worker blocks inside each rank's slab (dsgd_fused.sub_rounds)
        if config.workers != world and not (sub_blocks and config.workers > world and config.workers % world == 0):
            config = replace(config, workers=world)
        super().__init__(model, train_set, config, owner_rank=rank, owner_world=world)
        self.rank, self.world = rank, world
        self.plan = DsgdPlan(model.dims, world)
        self.ex = DsgdExchange(self.plan, self.dm.fac, self.dm.foff, self.dm.jr, group)
        self.bytes_rotated = 0

    def after_round(self, r):
        if r + 1 < self.plan.n_rounds:
            self.bytes_rotated += self.ex.rotate(r, r + 1)

    def after_factor_phase(self):
        self.ex.gather_all(self.plan.n_rounds - 1)

    # Psi is one serial draw over the whole tensor (trainer.py:212-220); the
    # ranks take turns: rank t % W draws epoch t's batch on its psi stream and
    # broadcasts it (4 MB at NF), so each rank draws 1/W of the batches.
    def draws_psi(self, t):
        return t % self.world == self.rank

    def share_psi(self, t, stream):
        buf = self.psi[t % self.P][:self.k]
        src = t % self.world
        if self.ex.group is not None:
            src = self.ex.td.get_global_rank(self.ex.group, src)
        if stream is None:
            stream = self.torch.cuda.current_stream()
        if self.ex.nccl:
            with self.torch.cuda.stream(stream):
                self.ex.td.broadcast(buf, src, group=self.ex.group)
        else:
            stream.synchronize()
            h = buf.cpu()
            self.ex.td.broadcast(h, src, group=self.ex.group)
            buf.copy_(h)

    def core_slice(self, slot):
        lo, hi = self.plan.chunk_bounds(self.k)[self.rank]
        if self.k == self.nnz:
            ids = self.torch.arange(lo, hi, dtype=self.torch.int32, device=self.dm.fac.device)
        else:
            ids = self.psi[self.psi_slot][lo:hi]
        return ids, hi - lo, (1 if self.mode == 1 else 0)

    def reduce_core_acc(self):
        if self.mode == 1:
            self.ex.allreduce_ordered(self.acc)  # exact: the reference's chunk order
        else:
            self.ex.allreduce(self.acc)


def train_distributed(model, split, config):
    """train() when torch.distributed is initialised with world size > 1: one
    rank per GPU, the DSGD data division above; every rank returns the rows
    and ends with the identical model."""
    import torch

    from . import counting
    from .device import DeviceCoo, rmse_mae_device
    from .training import MetricsRow, _RecordView, learning_rate

    import os

    from .dsgd_fused import FusedDistRunner, fused_supported

    # throughput mode on the TMA kernel shapes: one fused launch per rank per
    # epoch (dsgd_fused); otherwise one launch + exchange per round
    if fused_supported(model, config, split.train.nnz) and os.environ.get("SPTK_DSGD_FUSED", "1") == "1":
        runner = FusedDistRunner(model, split.train, config)
    else:
        runner = DistRunner(model, split.train, config)
    test_coo = DeviceCoo(split.test.indices, split.test.values, f64=runner.f64) if split.test.nnz else None
    train_eval = _RecordView(runner.part)
    rows, wall, pending = [], 0.0, []
    for t in range(config.epochs):
        ga = learning_rate(config.alpha_a, config.beta_a, t)
        gb = learning_rate(config.alpha_b, config.beta_b, t)
        ev0 = torch.cuda.Event(enable_timing=True)
        ev1 = torch.cuda.Event(enable_timing=True)
        ev0.record()
        runner.epoch(t, ga, gb)
        if counting.counter.enabled:
            lo, hi = runner.plan.chunk_bounds(runner.k)[runner.rank]
            counting.counter.add(counting.epoch_multiplies(model.j_ranks, model.r_core, runner.nnz_local,
                                                           hi - lo if config.update_core else 0))
        ev1.record()
        pending.append((ev0, ev1))
        if (t + 1) % config.eval_every == 0 or t == config.epochs - 1:
            ev1.synchronize()
            local = sum(a.elapsed_time(b) for a, b in pending) / 1000.0
            pending.clear()
            tt = torch.tensor([local], dtype=torch.float64,
                              device=runner.dm.fac.device if runner.ex.nccl else "cpu")
            runner.ex.td.all_reduce(tt, op=runner.ex.td.ReduceOp.MAX)
            wall += float(tt.item())
            tr = rmse_mae_device(runner.dm, train_eval)
            te = rmse_mae_device(runner.dm, test_coo) if test_coo is not None else (math.nan, math.nan)
            rows.append(MetricsRow(t + 1, wall, tr[0], tr[1], te[0], te[1], ga, gb))
    runner.dm.download_into(model)
    return rows


__all__ = ["active", "DsgdPlan", "DsgdExchange", "DistRunner", "train_distributed"]

"""Block partition (K1, on the GPU) and the conflict-free DSGD round schedule.

* ``build_partition`` -> partition.py:47-81: floor cut points k*I_n//m, block
  component = last cut <= index, key = sum_n b_n * m^(N-1-n), stable grouping.
  Computed by sptk_partition (device radix sort); the host plan is rebuilt
  from the device ids so the returned PartitionPlan matches the reference.
* ``round_schedule`` -> partition.py:84-117: M^(N-1) rounds ordered by a
  reflected base-M Gray code over the N-1 rotating modes; worker w owns block
  (w, (w+d_1)%M, ..., (w+d_{N-1})%M), so mode 0 stays put and consecutive
  rounds move exactly one mode's block index by +-1 -- the ring shift the
  multi-GPU path performs over NVLink (dist.py).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from ._lib import check, i64arr, ptr, stream_ptr


@dataclass(frozen=True)
class PartitionPlan:
    m: int
    boundaries: tuple
    block_entries: dict

    def block_of(self, index) -> tuple:
        return tuple(int(np.searchsorted(self.boundaries[n], int(i), side="right")) - 1
                     for n, i in enumerate(index))


@dataclass(frozen=True)
class RoundSchedule:
    order: int
    m: int
    rounds: tuple


def cut_points(dims, m) -> tuple:
    return tuple(tuple((k * int(d)) // m for k in range(m + 1)) for d in dims)


def block_key(block, m) -> int:
    k = 0
    for b in block:
        k = k * m + int(b)
    return k


def key_to_block(key: int, m: int, order: int) -> tuple:
    digits = []
    for _ in range(order):
        digits.append(key % m)
        key //= m
    return tuple(reversed(digits))


def upload(a: np.ndarray):
    """Host array -> new device tensor through sptk_h2d (threaded pinned
    staging; the pageable copy runs at ~11 GB/s on the B200 hosts)."""
    import torch

    a = np.ascontiguousarray(a)
    d = torch.empty(a.shape, dtype=torch.from_numpy(a[:0]).dtype, device="cuda")
    if a.nbytes:
        # the copy runs on sptk's own streams: the (possibly recycled) block
        # must be idle on the current stream first
        torch.cuda.current_stream().synchronize()
        check(_lib.load().sptk_h2d(ptr(d), a.ctypes.data, a.nbytes, 0), "sptk_h2d")
    return d


class DevicePartition:
    """Device records grouped by block + offsets (the output of K1)."""

    def __init__(self, indices: np.ndarray, values: np.ndarray, dims, m: int, f64: bool = False,
                 want_ids: bool = True):
        import torch

        _lib.require_cuda()
        L = _lib.load()
        idx = np.ascontiguousarray(indices, dtype=np.int64)
        self.nnz, self.order = int(idx.shape[0]), int(idx.shape[1])
        self.m = int(m)
        self.dims = tuple(int(d) for d in dims)
        self.f64 = f64
        self.rw = int(L.sptk_record_words(self.order, 1 if f64 else 0))
        nkeys = self.m ** self.order
        dev = torch.device("cuda")
        self.rec = torch.empty(max(self.nnz, 1) * self.rw, dtype=torch.int32, device=dev)
        self.ids = torch.empty(max(self.nnz, 1), dtype=torch.int32, device=dev) if want_ids else None
        self.pos_of_id = torch.empty(max(self.nnz, 1), dtype=torch.int32, device=dev)
        self.block_off_dev = torch.empty(nkeys + 1, dtype=torch.int32, device=dev)
        need = int(L.sptk_partition_ws_bytes(self.nnz, self.order, self.m))
        ws = torch.empty(need, dtype=torch.uint8, device=dev)
        dims_c, pd = i64arr(self.dims)
        vals = np.ascontiguousarray(values, dtype=np.float64)
        if not f64 and self.nnz:
            # fp32 records packed on the host side of the upload (half the
            # PCIe bytes), then grouped on the device
            src = self.rec if self.m == 1 else torch.empty_like(self.rec)
            torch.cuda.current_stream().synchronize()  # the upload runs on sptk's own streams
            check(L.sptk_h2d_pack(ptr(src), idx.ctypes.data, vals.ctypes.data, self.nnz, self.order, 0),
                  "sptk_h2d_pack")
            check(L.sptk_partition_records(ptr(src), self.nnz, self.order, pd, self.m, ptr(self.rec), ptr(self.ids),
                                           ptr(self.pos_of_id), ptr(self.block_off_dev), ptr(ws), need,
                                           stream_ptr()), "sptk_partition_records")
            del src
        else:
            d_idx = upload(idx)
            d_val = upload(vals)
            check(L.sptk_partition(ptr(d_idx), ptr(d_val), self.nnz, self.order, pd, self.m, 1 if f64 else 0,
                                   ptr(self.rec), ptr(self.ids), ptr(self.pos_of_id), ptr(self.block_off_dev),
                                   ptr(ws), need, stream_ptr()), "sptk_partition")
            del d_idx, d_val
        del ws
        self.block_off = self.block_off_dev.cpu().numpy().astype(np.int64)

    def block_range(self, block) -> tuple[int, int]:
        k = block_key(block, self.m)
        lo = int(self.block_off[k])
        return lo, int(self.block_off[k + 1]) - lo


def build_partition(tensor, m: int) -> PartitionPlan:
    """PartitionPlan identical to the reference's, computed on the GPU."""
    if m < 1:
        raise ValueError("m must be >= 1")
    if m > min(tensor.dims):
        raise ValueError(f"m={m} exceeds smallest mode dimension {min(tensor.dims)}")
    bounds = cut_points(tensor.dims, m)
    plan = {}
    if tensor.nnz:
        dp = DevicePartition(tensor.indices, tensor.values, tensor.dims, m)
        ids = dp.ids[: dp.nnz].cpu().numpy().astype(np.int64)
        offs = dp.block_off
        for key in np.flatnonzero(np.diff(offs) > 0):
            plan[key_to_block(int(key), m, tensor.order)] = ids[offs[key]: offs[key + 1]]
    return PartitionPlan(m, bounds, plan)


def _gray(digits: int, m: int) -> list:
    seq = [()]
    for _ in range(digits):
        seq = [(lead,) + tail for lead in range(m) for tail in (seq if lead % 2 == 0 else seq[::-1])]
    return seq


def gray_offsets(digits: int, m: int) -> np.ndarray:
    """The reflected base-m Gray code of _gray as an int64 array [m^digits, digits]."""
    seq = np.zeros((1, 0), dtype=np.int64)
    for _ in range(digits):
        parts = []
        for lead in range(m):
            tail = seq if lead % 2 == 0 else seq[::-1]
            parts.append(np.concatenate([np.full((tail.shape[0], 1), lead, dtype=np.int64), tail], axis=1))
        seq = np.concatenate(parts, axis=0)
    return seq


def round_blocks(order: int, m: int) -> np.ndarray:
    """round_schedule(order, m).rounds as an int64 array [rounds, m, order]:
    worker w's block in round r is (w, (w + d_1) % m, ...) (partition.py:100-117)."""
    offs = gray_offsets(order - 1, m)
    w = np.arange(m, dtype=np.int64)
    cols = [np.broadcast_to(w, (offs.shape[0], m))] + [(w[None, :] + offs[:, d: d + 1]) % m
                                                        for d in range(order - 1)]
    return np.stack(cols, axis=2)


def round_schedule(order: int, m: int) -> RoundSchedule:
    if order < 2:
        raise ValueError("order must be >= 2")
    if m < 1:
        raise ValueError("m must be >= 1")
    rounds = tuple(tuple(tuple(b) for b in rnd) for rnd in round_blocks(order, m).tolist())
    return RoundSchedule(order, m, rounds)


def schedule_text(schedule: RoundSchedule, plan: PartitionPlan | None = None) -> str:
    head = (f"order={schedule.order} m={schedule.m} rounds={len(schedule.rounds)} "
            f"workers={schedule.m}")
    body = []
    for t, rnd in enumerate(schedule.rounds):
        cells = []
        for w, blk in enumerate(rnd):
            cell = f"w{w}->(" + ",".join(map(str, blk)) + ")"
            if plan is not None:
                cell += f"[{len(plan.block_entries.get(blk, ()))}]"
            cells.append(cell)
        body.append(f"round {t}: " + "  ".join(cells))
    return "\n".join([head] + body)

"""Scalar-multiplication accounting (counting.py:12-52 of the reference).

The reference counts the multiplications of its per-sample Python kernels
(kernels.py, factor_sgd.py) while a ``count_multiplies`` block is active.  Here
no Python runs per sample: ``train()`` adds, per epoch, the multiplications
its kernels perform for the samples they process (tensor-core MACs counted as
multiplications), from the formulas below.  Same interface: a global
``counter``, off by default, and the ``count_multiplies`` context manager.
"""

from __future__ import annotations

from dataclasses import dataclass


@dataclass
class MultiplyCounter:
    """Global tally of scalar multiplications; ``add`` is a no-op unless enabled."""

    enabled: bool = False
    total: int = 0

    def add(self, n: int) -> None:
        if self.enabled:
            self.total += int(n)

    def reset(self) -> None:
        self.total = 0


counter = MultiplyCounter()


class count_multiplies:
    """``with count_multiplies() as c:`` enables the counter for the block
    (blocks nest); ``c.so_far`` inside, ``c.total`` after it."""

    def __init__(self):
        self._start, self._prev, self.total = 0, False, 0

    @property
    def so_far(self) -> int:
        return counter.total - self._start

    def __enter__(self):
        self._prev, counter.enabled = counter.enabled, True
        self._start = counter.total
        return self

    def __exit__(self, *exc):
        counter.enabled = self._prev
        self.total = self.so_far
        return False


def factor_sample_multiplies(j_ranks, r_core: int) -> int:
    """One sample's factor update over every mode (_loops.py:31-62 as the
    factor kernels compute it): c_n = a_n B(n) for all modes (sum J_n R); per
    mode the off-mode weights ((N-2) R), gs = B(n) w (J_n R), a.gs, the step
    and the shrink (3 J_n); the c refresh of the updated row for every mode
    but the last (J_n R)."""
    N, R = len(j_ranks), int(r_core)
    js = [int(j) for j in j_ranks]
    c = sum(j * R for j in js)
    per_mode = sum((max(N - 2, 0) * R) + j * R + 3 * j for j in js)
    refresh = sum(j * R for j in js[:-1])
    return c + per_mode + refresh


def core_sample_multiplies(j_ranks, r_core: int) -> int:
    """One core-batch sample's gradient (_loops.py:66-104): c (sum J_n R),
    the prediction ((N-1) R), and per mode and rank the weight and the
    J_n-long outer product ((N-2) R + J_n R)."""
    N, R = len(j_ranks), int(r_core)
    js = [int(j) for j in j_ranks]
    return sum(j * R for j in js) + (N - 1) * R + sum(max(N - 2, 0) * R + j * R for j in js)


def epoch_multiplies(j_ranks, r_core: int, n_factor: int, n_core: int) -> int:
    """One epoch: n_factor factor samples and n_core core-batch samples."""
    return int(n_factor) * factor_sample_multiplies(j_ranks, r_core) + int(n_core) * core_sample_multiplies(
        j_ranks, r_core)


__all__ = ["MultiplyCounter", "counter", "count_multiplies", "factor_sample_multiplies", "core_sample_multiplies",
           "epoch_multiplies"]

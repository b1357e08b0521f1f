"""COO tensor containers, FROSTT-style text I/O and the seeded train/test split.

Behavioural mirror of the reference's data layer (sptucker/coo.py:23-166,
268-286): same validation rules and error messages (the CLI maps them to exit
codes), same text format, same split RNG stream.  Host-side only; the device
layout used by the kernels is built by ``schedule.build_partition`` /
``device.DeviceCoo``.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


class CooFormatError(ValueError):
    """Malformed COO text; the message names the offending line."""


def _checked_arrays(dims, indices, values):
    if len(dims) < 2:
        raise ValueError("tensor order must be >= 2")
    if min(dims) < 1:
        raise ValueError("all mode dimensions must be positive")
    order = len(dims)
    idx = np.ascontiguousarray(indices, dtype=np.int64)
    val = np.ascontiguousarray(values, dtype=np.float64)
    if idx.ndim != 2 or idx.shape[1] != order:
        raise ValueError(f"indices must have shape (nnz, {order}), got {idx.shape}")
    if val.shape != (idx.shape[0],):
        raise ValueError("values length must match number of index rows")
    if idx.size:
        bounds = np.asarray(dims, dtype=np.int64)
        if idx.min() < 0 or bool((idx >= bounds).any()):
            raise ValueError("index out of bounds for dims")
    if val.size and not bool(np.isfinite(val).all()):
        raise ValueError("non-finite value in tensor")
    return idx, val


@dataclass(frozen=True)
class SparseTensorCoo:
    """Order-N sparse tensor: int64 ``indices`` (nnz, N), fp64 ``values``.

    Row order is meaningful and duplicate coordinates are separate
    observations.
    """

    dims: tuple
    indices: np.ndarray
    values: np.ndarray

    def __post_init__(self):
        idx, val = _checked_arrays(tuple(self.dims), self.indices, self.values)
        object.__setattr__(self, "dims", tuple(int(d) for d in self.dims))
        object.__setattr__(self, "indices", idx)
        object.__setattr__(self, "values", val)

    @property
    def order(self) -> int:
        return len(self.dims)

    @property
    def nnz(self) -> int:
        return int(self.indices.shape[0])

    def entries(self):
        """(index tuple, value) pairs in stored order."""
        for k in range(self.nnz):
            yield tuple(int(c) for c in self.indices[k]), float(self.values[k])

    def same_entries(self, other: "SparseTensorCoo") -> bool:
        if self.dims != other.dims:
            return False
        return bool(np.array_equal(self.indices, other.indices)
                    and np.array_equal(self.values, other.values))


@dataclass(frozen=True)
class DatasetSplit:
    """Train and test entries of one tensor (dims must agree)."""

    train: SparseTensorCoo
    test: SparseTensorCoo

    def __post_init__(self):
        if self.train.dims != self.test.dims:
            raise ValueError("train and test must share dims")


def empty_like(tensor: SparseTensorCoo) -> SparseTensorCoo:
    """A tensor with the same dims and no entries."""
    return SparseTensorCoo(tensor.dims, np.zeros((0, tensor.order), dtype=np.int64), np.zeros(0))


# ------------------------------------------------------------------ text I/O

def load_coo(path, index_base: int = 1, threads: int = 0) -> SparseTensorCoo:
    """Read ``i_1 .. i_N value`` lines (``#`` comments, optional ``# dims:``),
    the reference's text format and errors (coo.py:90-148).

    Parsed natively (libsptk ``sptk_coo_text_parse``: memory-mapped file,
    ``threads`` parser threads, 0 = all) with the reference's grammar; the
    CooFormatError raised names the earliest bad line, as the reference's
    sequential reader would."""
    import ctypes
    import os

    from . import _lib

    if index_base not in (0, 1):
        raise ValueError("index_base must be 0 or 1")
    L = _lib.load()
    handle = ctypes.c_void_p()
    nnz = ctypes.c_int64()
    order = ctypes.c_int()
    rc = L.sptk_coo_text_parse(os.fsencode(path), int(index_base), int(threads), ctypes.byref(handle),
                               ctypes.byref(nnz), ctypes.byref(order))
    if rc != 0:
        msg = L.sptk_last_error().decode(errors="replace")
        if rc == 1:
            raise CooFormatError(msg[len("line 0: "):] if msg.startswith("line 0: ") else msg)
        if rc == 3:
            raise OverflowError(msg)
        if not os.path.exists(path):
            raise FileNotFoundError(2, "No such file or directory", str(path))
        raise OSError(msg)
    n, N = int(nnz.value), int(order.value)
    dims = np.zeros(N, dtype=np.int64)
    hdr = ctypes.c_int()
    L.sptk_coo_text_dims(handle, dims.ctypes.data_as(_lib._i64p), ctypes.byref(hdr))
    idx = np.empty((n, N), dtype=np.int64)
    vals = np.empty(n, dtype=np.float64)
    L.sptk_coo_text_take(handle, idx.ctypes.data, vals.ctypes.data, int(threads))
    return SparseTensorCoo(tuple(int(d) for d in dims), idx, vals)


def write_coo(tensor: SparseTensorCoo, path, index_base: int = 1) -> None:
    """Write the text format above; values with 17 significant digits."""
    if index_base not in (0, 1):
        raise ValueError("index_base must be 0 or 1")
    if tensor.nnz == 0:
        raise ValueError("refusing to write tensor with no entries")
    shifted = tensor.indices + index_base
    lines = ["# dims: " + " ".join(map(str, tensor.dims))]
    for k in range(tensor.nnz):
        lines.append(" ".join(map(str, shifted[k].tolist())) + f" {tensor.values[k]:.17g}")
    with open(path, "w") as fh:
        fh.write("\n".join(lines) + "\n")


# --------------------------------------------------------------------- split

def split(tensor: SparseTensorCoo, test_fraction: float, seed: int = 0) -> DatasetSplit:
    """Hold out round(f * nnz) entries drawn by default_rng([seed, 0x5311]).

    Both halves keep source order (reference coo.py:268-286).
    """
    if not (0 <= test_fraction < 1):
        raise ValueError("test_fraction must be in [0, 1)")
    if tensor.nnz == 0:
        raise ValueError("cannot split an empty tensor")
    n_test = int(round(test_fraction * tensor.nnz))
    if n_test >= tensor.nnz:
        raise ValueError("test_fraction leaves an empty train set")
    held = np.random.default_rng([int(seed), 0x5311]).choice(tensor.nnz, size=n_test, replace=False)
    is_test = np.zeros(tensor.nnz, dtype=bool)
    is_test[held] = True
    keep = ~is_test
    return DatasetSplit(
        SparseTensorCoo(tensor.dims, tensor.indices[keep], tensor.values[keep]),
        SparseTensorCoo(tensor.dims, tensor.indices[is_test], tensor.values[is_test]),
    )


def write_coo_binary(tensor: SparseTensorCoo, path) -> None:
    """Binary side format of a COO tensor (ingestion at 10^8-10^9
    nonzeros, where the FROSTT text parser of coo.py:90-148 is impractical):
    an uncompressed .npz with dims, int64 indices [nnz, N] and float64 values,
    readable back without a copy via memory mapping."""
    with open(path, "wb") as fh:
        np.savez(fh, dims=np.asarray(tensor.dims, dtype=np.int64), indices=tensor.indices, values=tensor.values)


def load_coo_binary(path, mmap: bool = True) -> SparseTensorCoo:
    """Read write_coo_binary's format (arrays memory-mapped when possible);
    the same validation as SparseTensorCoo."""
    with np.load(path, mmap_mode="r" if mmap else None) as z:
        dims = tuple(int(d) for d in z["dims"])
        return SparseTensorCoo(dims, np.asarray(z["indices"]), np.asarray(z["values"]))

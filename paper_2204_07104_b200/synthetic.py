"""Synthetic sparse tensors drawn from a recoverable Kruskal-core Tucker model.

``generate_synthetic`` reproduces the reference generator (sptucker/coo.py:
178-265) draw for draw -- same ground-truth model, same index sampler, same
rescaling and noise streams -- so a seed gives the reference's tensor.  Its
distinct-index sampler is vectorised here, but it still holds every index in
memory, which limits it to a few million nonzeros.

``generate_large`` is the scalable generator for the benchmark shapes
(Netflix 480,189 x 17,770 x 2,182 with 99M nonzeros, the 4-order Yahoo shape,
10K^6 with 1e9 nonzeros).  Indices are i.i.d. uniform per
mode (duplicates are legal observations, coo.py:29-30), drawn in fixed chunks
of 2^22 rows with per-chunk seeds so that any prefix of a large tensor equals
the smaller tensor with the same seed (the CPU baseline times such a prefix).
Values use the reference's ground-truth construction, rescaled to std 4, plus
N(0, sigma^2) noise.  Data synthesis is host-side preparation, not the hot
path.
"""

from __future__ import annotations

import math

import numpy as np

from .tensor import SparseTensorCoo
from .tucker import ModelConfig, TuckerModel

BIAS_WEIGHT = 4.0
TARGET_STD = 4.0
CHUNK = 1 << 22


def host_predict(model: TuckerModel, indices: np.ndarray) -> np.ndarray:
    """fp64 numpy model evaluation, used only to synthesise values so that the
    tensors match the reference bit for bit (coo.py:231-244 -> model.py:134-146)."""
    idx = np.asarray(indices, dtype=np.int64)
    acc = np.ones((idx.shape[0], model.r_core))
    for n, (a, b) in enumerate(zip(model.factors, model.core_factors)):
        acc *= a[idx[:, n], :] @ b
    return acc.sum(axis=1)


def ground_truth(dims, j_ranks, r_core: int, seed: int) -> TuckerModel:
    """Nonnegative bias column + zero-centred columns; core column 0 routes the
    bias with weight 4/sqrt(R), the rest mix the signed columns (coo.py:178-201)."""
    rng = np.random.default_rng([int(seed), 0xC00])
    factors = []
    for d, j in zip(dims, j_ranks):
        half = 0.5 / math.sqrt(j)
        a = rng.uniform(-half, half, size=(d, j))
        a[:, 0] = rng.uniform(0.0, 2 * half, size=d)
        factors.append(a)
    hb = 1.0 / math.sqrt(r_core)
    cores = []
    for j in j_ranks:
        b = np.zeros((j, r_core))
        b[0, 0] = BIAS_WEIGHT * hb
        if j > 1 and r_core > 1:
            b[1:, 1:] = rng.uniform(-hb, hb, size=(j - 1, r_core - 1))
        cores.append(b)
    return TuckerModel(dims, j_ranks, r_core, factors, cores)


def _normalise_ranks(dims, j_ranks, r_core, seed):
    ranks = ModelConfig(j_ranks, r_core, seed=seed).j_ranks
    if len(ranks) == 1 and len(dims) > 1:
        ranks = ranks * len(dims)
    return ranks


def _distinct_rows(rng, dims, nnz):
    """Rejection-sample nnz distinct index rows in draw order (coo.py:245-254):
    draws come in batches of nnz rows per mode; a row is kept if unseen."""
    total = math.prod(dims)
    radix = np.cumprod((1,) + tuple(dims[:0:-1]))[::-1]  # mode-0 most significant
    use_keys = total < (1 << 62)
    seen_keys = np.empty(0, dtype=np.int64)
    seen_rows: set = set()
    out = []
    have = 0
    while have < nnz:
        batch = np.stack([rng.integers(0, d, size=nnz) for d in dims], axis=1)
        if use_keys:
            keys = batch @ radix.astype(np.int64)
            _, first = np.unique(keys, return_index=True)
            first.sort()
            fresh = first[~np.isin(keys[first], seen_keys)]
            take = fresh[: nnz - have]
            out.append(batch[take])
            seen_keys = np.concatenate([seen_keys, keys[take]])
            have += len(take)
        else:
            for row in batch:
                t = tuple(int(v) for v in row)
                if t not in seen_rows:
                    seen_rows.add(t)
                    out.append(row[None, :])
                    have += 1
                    if have == nnz:
                        break
    return np.concatenate(out, axis=0).astype(np.int64)


def generate_synthetic(dims, nnz: int, j_ranks, r_core: int, noise_sigma: float = 0.0,
                       seed: int = 0):
    """(tensor, ground_truth) exactly as the reference's generator draws them."""
    dims = tuple(int(d) for d in dims)
    if noise_sigma < 0:
        raise ValueError("noise_sigma must be >= 0")
    total = math.prod(dims)
    if nnz > total:
        raise ValueError(f"nnz={nnz} exceeds dense size {total}")
    if nnz < 1:
        raise ValueError("nnz must be >= 1")
    ranks = _normalise_ranks(dims, j_ranks, r_core, seed)
    model = ground_truth(dims, ranks, r_core, seed)
    rng = np.random.default_rng([int(seed), 0xC01])
    if total <= max(1 << 24, 16 * nnz):
        lin = rng.choice(total, size=nnz, replace=False)
        idx = np.stack(np.unravel_index(lin, dims), axis=1).astype(np.int64)
    else:
        idx = _distinct_rows(rng, dims, nnz)
    spread = float(np.std(host_predict(model, idx)))
    if spread > 0:
        scale = (TARGET_STD / spread) ** (1.0 / (2 * len(dims)))
        for m in model.factors + model.core_factors:
            m *= scale
    vals = host_predict(model, idx)
    if noise_sigma > 0:
        vals = vals + noise_sigma * rng.standard_normal(nnz)
    return SparseTensorCoo(dims, idx, vals), model


# ------------------------------------------------------------------ large

def large_indices(dims, nnz: int, seed: int) -> np.ndarray:
    """i.i.d. uniform indices; one stream per (chunk, mode), so any prefix of a
    large tensor equals the smaller tensor drawn with the same seed."""
    out = np.empty((nnz, len(dims)), dtype=np.int64)
    for c0 in range(0, nnz, CHUNK):
        n = min(CHUNK, nnz - c0)
        for m, d in enumerate(dims):
            rng = np.random.default_rng([int(seed), 0xC01, c0 // CHUNK, m])
            out[c0:c0 + n, m] = rng.integers(0, d, size=n)
    return out


def generate_large(dims, nnz: int, j_ranks, r_core: int, noise_sigma: float = 0.1,
                   seed: int = 7, n_test: int = 0, predict=None):
    """Scalable synthetic data: (train tensor, test tensor, ground truth).

    ``predict(model, idx) -> fp64 values`` defaults to chunked host numpy;
    callers with a GPU may pass the device evaluator.  The std used for the
    rescale is measured on the first 2^20 entries (a fixed, prefix-stable
    sample).  The test set is an independent draw of ``n_test`` entries
    (seed + 1), e.g. the Netflix probe size 1,408,395.
    """
    dims = tuple(int(d) for d in dims)
    ranks = _normalise_ranks(dims, j_ranks, r_core, seed)
    model = ground_truth(dims, ranks, r_core, seed)
    pred = predict or (lambda mdl, ix: _chunked(host_predict, mdl, ix))
    idx = large_indices(dims, nnz, seed)
    sample = idx[: min(nnz, 1 << 20)]
    spread = float(np.std(pred(model, sample)))
    if spread > 0:
        scale = (TARGET_STD / spread) ** (1.0 / (2 * len(dims)))
        for m in model.factors + model.core_factors:
            m *= scale
    vals = pred(model, idx) + noise_sigma * _noise(nnz, seed)
    train = SparseTensorCoo(dims, idx, vals)
    test = None
    if n_test:
        tidx = large_indices(dims, n_test, seed + 1)
        tvals = pred(model, tidx) + noise_sigma * _noise(n_test, seed + 1)
        test = SparseTensorCoo(dims, tidx, tvals)
    return train, test, model


def _noise(n, seed):
    out = np.empty(n)
    for c0 in range(0, n, CHUNK):
        k = min(CHUNK, n - c0)
        out[c0:c0 + k] = np.random.default_rng([int(seed), 0xC02, c0 // CHUNK]).standard_normal(k)
    return out


def _chunked(fn, model, idx, chunk=1 << 20):
    out = np.empty(idx.shape[0])
    for c0 in range(0, idx.shape[0], chunk):
        out[c0:c0 + chunk] = fn(model, idx[c0:c0 + chunk])
    return out

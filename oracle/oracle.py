"""TEST INFRASTRUCTURE ONLY -- ctypes front end of the C restatement.

This module is the checker the parity tests compare the CUDA library against,
and the CPU baseline bench.py times (``cpu_baseline.kind = "port"``).  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu-baseline /
``--impl reference`` legs import it; the product package never does.

Everything here restates the reference ``sptucker`` package
(/root/reference/pkg/src/sptucker) in fp64:

* ``train``            -> trainer.py:150-271 (epoch loop, seeds, DSGD rounds,
                          core batch, merge and apply)
* ``factor_pass``      -> _loops.py:17-63
* ``core_pass``        -> _loops.py:66-104
* ``predict``          -> model.py:134-146
* ``permutation``      -> Generator.permutation as used at trainer.py:196-199
* ``choice``           -> Generator.choice(replace=False), trainer.py:212-221
* ``partition``        -> partition.py:47-81
* ``round_schedule``   -> partition.py:84-117
* ``pcg64_state``      -> default_rng(entropy) seeding (SeedSequence + PCG64)

The restatement is pinned against golden vectors written by the reference
itself (tests/golden/make_golden.py); see tests/test_oracle_golden.py.
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")
_lib = None

_i64p = ctypes.POINTER(ctypes.c_int64)
_u64p = ctypes.POINTER(ctypes.c_uint64)
_u32p = ctypes.POINTER(ctypes.c_uint32)
_f64p = ctypes.POINTER(ctypes.c_double)


def build():
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        L.orc_seedseq_generate.argtypes = [_u64p, ctypes.c_int, _u32p, ctypes.c_int]
        L.orc_pcg64_from_entropy.argtypes = [_u64p, ctypes.c_int, _u64p]
        L.orc_pcg64_u32_stream.argtypes = [_u64p, ctypes.c_int64, _u32p]
        L.orc_permutation.argtypes = [_u64p, ctypes.c_int64, _i64p, _i64p]
        L.orc_choice.argtypes = [_u64p, ctypes.c_int64, ctypes.c_int64, _i64p]
        L.orc_choice.restype = ctypes.c_int
        L.orc_partition.argtypes = [_i64p, ctypes.c_int64, ctypes.c_int, _i64p, ctypes.c_int64,
                                    _i64p, _i64p]
        L.orc_factor_pass.argtypes = [_i64p, _f64p, _i64p, ctypes.c_int64, _f64p, _i64p, _f64p,
                                      _i64p, _i64p, ctypes.c_int, ctypes.c_int64, _f64p, _f64p]
        L.orc_core_pass.argtypes = [_i64p, _f64p, _i64p, ctypes.c_int64, _f64p, _i64p, _f64p,
                                    _i64p, _i64p, ctypes.c_int, ctypes.c_int64, _f64p, _i64p]
        L.orc_predict.argtypes = [_i64p, ctypes.c_int64, _f64p, _i64p, _f64p, _i64p, _i64p,
                                  ctypes.c_int, ctypes.c_int64, _f64p]
        _lib = L
    return _lib


def _p(a, t):
    return a.ctypes.data_as(t)


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


# ---------------------------------------------------------------- RNG ----

def seedseq_words(entropy, n_words=8):
    ent = _c([int(e) for e in entropy], np.uint64)
    out = np.zeros(n_words, dtype=np.uint32)
    lib().orc_seedseq_generate(_p(ent, _u64p), len(ent), _p(out, _u32p), n_words)
    return out


def pcg64_state(entropy):
    """(state_hi, state_lo, inc_hi, inc_lo) of default_rng(entropy)."""
    ent = _c([int(e) for e in entropy], np.uint64)
    out = np.zeros(4, dtype=np.uint64)
    lib().orc_pcg64_from_entropy(_p(ent, _u64p), len(ent), _p(out, _u64p))
    return out


def u32_stream(state, n):
    st = _c(state, np.uint64)
    out = np.empty(n, dtype=np.uint32)
    lib().orc_pcg64_u32_stream(_p(st, _u64p), int(n), _p(out, _u32p))
    return out


def permutation(entropy, n, return_j=False):
    st = pcg64_state(entropy)
    out = np.empty(max(int(n), 1), dtype=np.int64)
    js = np.empty(max(int(n), 1), dtype=np.int64) if return_j else None
    lib().orc_permutation(_p(st, _u64p), int(n), _p(out, _i64p),
                          _p(js, _i64p) if return_j else None)
    out = out[: int(n)]
    return (out, js[: int(n)]) if return_j else out


def choice(entropy, pop, k):
    """default_rng(entropy).choice(pop, k, replace=False); returns (ids, path)."""
    st = pcg64_state(entropy)
    out = np.empty(max(int(k), 1), dtype=np.int64)
    path = lib().orc_choice(_p(st, _u64p), int(pop), int(k), _p(out, _i64p))
    return out[: int(k)], ("tail" if path == 1 else "floyd")


# ----------------------------------------------------------- partition ----

def partition(indices, dims, m):
    """partition.py:47-81 -> (ids grouped by block, block key per id)."""
    idx = _c(indices, np.int64)
    nnz, order = idx.shape
    d = _c(dims, np.int64)
    ids = np.empty(max(nnz, 1), dtype=np.int64)
    keys = np.empty(max(nnz, 1), dtype=np.int64)
    lib().orc_partition(_p(idx, _i64p), nnz, order, _p(d, _i64p), int(m), _p(ids, _i64p),
                        _p(keys, _i64p))
    return ids[:nnz], keys[:nnz]


def block_entries(indices, dims, m):
    """dict block-tuple -> ids, as PartitionPlan.block_entries."""
    ids, keys = partition(indices, dims, m)
    order = len(dims)
    out = {}
    if len(ids) == 0:
        return out
    starts = np.flatnonzero(np.r_[True, keys[1:] != keys[:-1]])
    ends = np.r_[starts[1:], len(keys)]
    for s, e in zip(starts, ends):
        k = int(keys[s])
        block = []
        for _ in range(order):
            block.append(k % m)
            k //= m
        out[tuple(reversed(block))] = ids[s:e]
    return out


def _snake(digits, m):
    if digits == 0:
        yield ()
        return
    tails = list(_snake(digits - 1, m))
    for lead in range(m):
        seq = tails if lead % 2 == 0 else reversed(tails)
        for tail in seq:
            yield (lead,) + tail


def round_schedule(order, m):
    """partition.py:100-117 -> tuple of rounds, each a tuple of M blocks."""
    return tuple(
        tuple((w,) + tuple((w + d) % m for d in offs) for w in range(m))
        for offs in _snake(order - 1, m)
    )


# ------------------------------------------------------------- kernels ----

def pack(mats):
    """trainer.py:135-141."""
    offs = np.zeros(len(mats) + 1, dtype=np.int64)
    for n, a in enumerate(mats):
        offs[n + 1] = offs[n] + a.size
    flat = np.empty(offs[-1])
    for n, a in enumerate(mats):
        flat[offs[n]: offs[n + 1]] = np.asarray(a, dtype=np.float64).ravel()
    return flat, offs


def unpack(flat, offs, shapes):
    return [flat[offs[n]: offs[n + 1]].reshape(s).copy() for n, s in enumerate(shapes)]


def factor_pass(idx, vals, visit, fac, foff, cor, coff, jr, rcore, gammas, lambdas):
    """_loops.factor_pass; fac updated in place."""
    L = lib()
    L.orc_factor_pass(_p(idx, _i64p), _p(vals, _f64p), _p(visit, _i64p), len(visit),
                      _p(fac, _f64p), _p(foff, _i64p), _p(cor, _f64p), _p(coff, _i64p),
                      _p(jr, _i64p), len(jr), int(rcore), _p(gammas, _f64p),
                      _p(lambdas, _f64p))
    return 0


def core_pass(idx, vals, visit, fac, foff, cor, coff, jr, rcore, acc, aoff):
    """_loops.core_pass; acc updated in place."""
    L = lib()
    L.orc_core_pass(_p(idx, _i64p), _p(vals, _f64p), _p(visit, _i64p), len(visit),
                    _p(fac, _f64p), _p(foff, _i64p), _p(cor, _f64p), _p(coff, _i64p),
                    _p(jr, _i64p), len(jr), int(rcore), _p(acc, _f64p), _p(aoff, _i64p))
    return 0


def predict(factors, core_factors, indices):
    fac, foff = pack(factors)
    cor, coff = pack(core_factors)
    jr = _c([a.shape[1] for a in factors], np.int64)
    idx = _c(indices, np.int64)
    if idx.ndim == 1:
        idx = idx[None, :]
    out = np.empty(idx.shape[0])
    lib().orc_predict(_p(idx, _i64p), idx.shape[0], _p(fac, _f64p), _p(foff, _i64p),
                      _p(cor, _f64p), _p(coff, _i64p), _p(jr, _i64p), len(jr),
                      core_factors[0].shape[1], _p(out, _f64p))
    return out


def learning_rate(alpha, beta, t):
    """trainer.py:80-86."""
    return alpha / (1.0 + beta * float(t) ** 1.5)


def _metrics(factors, core_factors, idx, vals):
    resid = vals - predict(factors, core_factors, idx)
    return float(np.sqrt(np.mean(resid ** 2))), float(np.mean(np.abs(resid)))


def train(factors, core_factors, train_idx, train_vals, test_idx=None, test_vals=None, *,
          epochs, workers=1, update_core=True, alpha_a=0.009, beta_a=0.05, lambda_a=0.01,
          alpha_b=0.0045, beta_b=0.1, lambda_b=0.01, core_batch_cap=1 << 20, seed=0,
          eval_every=1, core_average=True, evaluate=True, dims=None):
    """trainer.py:150-271 restated; factors/core_factors are updated in place.

    Returns a list of dict rows with the MetricsRow fields.  With
    ``evaluate=False`` the metric fields are NaN (used for timing only).
    """
    order = len(factors)
    if dims is None:
        dims = tuple(a.shape[0] for a in factors)
    idx = _c(train_idx, np.int64)
    vals = _c(train_vals, np.float64)
    nnz = idx.shape[0]
    w = int(workers)
    blocks = block_entries(idx, dims, w)
    schedule = round_schedule(order, w)
    fac, foff = pack(factors)
    cor, coff = pack(core_factors)
    jr = _c([a.shape[1] for a in factors], np.int64)
    rcore = core_factors[0].shape[1]
    has_test = test_idx is not None and len(test_vals) > 0
    ex = ThreadPoolExecutor(max_workers=w) if w > 1 else None
    rows = []
    wall = 0.0
    try:
        for t in range(epochs):
            ga = learning_rate(alpha_a, beta_a, t)
            gb = learning_rate(alpha_b, beta_b, t)
            gammas = np.full(order, ga)
            lambdas = np.full(order, lambda_a)
            start = time.perf_counter()
            processed = 0
            for rnd in schedule:
                futs = []
                for block in rnd:
                    ids = blocks.get(block)
                    if ids is None or len(ids) == 0:
                        continue
                    visit = np.ascontiguousarray(ids[permutation([seed, 1, t, *block], len(ids))])
                    processed += len(visit)
                    args = (idx, vals, visit, fac, foff, cor, coff, jr, rcore, gammas, lambdas)
                    if ex is None:
                        factor_pass(*args)
                    else:
                        futs.append(ex.submit(factor_pass, *args))
                for f in futs:
                    f.result()
            if processed != nnz:
                raise RuntimeError("partition did not cover every training entry")
            if update_core:
                k = min(nnz, core_batch_cap)
                if k == nnz:
                    psi = np.arange(k, dtype=np.int64)
                else:
                    psi, _ = choice([seed, 2, t], nnz, k)
                chunks = [c for c in np.array_split(psi, w) if len(c)]
                accs = [np.zeros(coff[-1]) for _ in chunks]
                if ex is None:
                    for ch, acc in zip(chunks, accs):
                        core_pass(idx, vals, np.ascontiguousarray(ch), fac, foff, cor, coff, jr,
                                  rcore, acc, coff)
                else:
                    futs = [ex.submit(core_pass, idx, vals, np.ascontiguousarray(ch), fac, foff,
                                      cor, coff, jr, rcore, acc, coff)
                            for ch, acc in zip(chunks, accs)]
                    for f in futs:
                        f.result()
                total = accs[0]
                for acc in accs[1:]:
                    total = total + acc
                denom = k if core_average else 1
                for n in range(order):
                    view = cor[coff[n]: coff[n + 1]].reshape(jr[n], rcore)
                    view -= gb * (total[coff[n]: coff[n + 1]].reshape(jr[n], rcore) / denom
                                  + lambda_b * view)
            wall += time.perf_counter() - start
            if (t + 1) % eval_every == 0 or t == epochs - 1:
                fs = unpack(fac, foff, [a.shape for a in factors])
                bs = unpack(cor, coff, [b.shape for b in core_factors])
                if evaluate:
                    tr = _metrics(fs, bs, idx, vals)
                    te = _metrics(fs, bs, test_idx, test_vals) if has_test else (math.nan, math.nan)
                else:
                    tr = te = (math.nan, math.nan)
                rows.append(dict(epoch=t + 1, wall_seconds=wall, train_rmse=tr[0],
                                 train_mae=tr[1], test_rmse=te[0], test_mae=te[1],
                                 gamma_a=ga, gamma_b=gb))
    finally:
        if ex is not None:
            ex.shutdown(wait=True)
    for n, a in enumerate(factors):
        a[...] = fac[foff[n]: foff[n + 1]].reshape(a.shape)
    for n, b in enumerate(core_factors):
        b[...] = cor[coff[n]: coff[n + 1]].reshape(b.shape)
    return rows

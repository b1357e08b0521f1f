"""Generate the golden fixtures from the REFERENCE itself (run in the build
container only; /root/reference does not exist on the GPU box).

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

Everything recorded here comes out of the reference package's own code paths
(the trainer's real visit/psi arrays are captured by wrapping
``sptucker._loops``), so the fixtures pin both the C oracle (oracle/) and the
CUDA library to the reference's behaviour with numpy 2.3.5.

Outputs:
  tests/golden/golden.npz        small arrays (compressed)
  tests/golden/golden_meta.json  hashes of the full-size sampler outputs and
                                 the reference training curves
"""

from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

REF = os.environ.get("SPTUCKER_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")

import sptucker  # noqa: E402
from sptucker import _loops  # noqa: E402
from sptucker.coo import DatasetSplit, SparseTensorCoo, generate_synthetic, split  # noqa: E402
from sptucker.model import ModelConfig, TuckerModel, default_init_scale, init_model, predict_entries  # noqa: E402
from sptucker.partition import build_partition, round_schedule  # noqa: E402
from sptucker.trainer import TrainConfig, train  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
G: dict[str, np.ndarray] = {}
META: dict = {"numpy": np.__version__, "reference": REF}


def h32(a) -> str:
    """sha256 over the int32 little-endian bytes (the device layout)."""
    return hashlib.sha256(np.ascontiguousarray(np.asarray(a), dtype="<i4").tobytes()).hexdigest()


# ----------------------------------------------------------------- RNG ----
ENTROPIES = [[0], [1], [1, 1, 0, 0, 0, 0], [7, 2, 3], [2**40 + 5, 3], [123456789, 1, 4, 1, 2, 3, 0]]
for i, ent in enumerate(ENTROPIES):
    st = np.random.default_rng(ent).bit_generator.state["state"]
    G[f"rng_state_{i}"] = np.array(
        [st["state"] >> 64, st["state"] & (2**64 - 1), st["inc"] >> 64, st["inc"] & (2**64 - 1)],
        dtype=np.uint64)
    G[f"rng_entropy_{i}"] = np.array(ent, dtype=np.uint64)
    # the raw 64-bit PCG64 outputs (each one yields two buffered 32-bit draws)
    bg = np.random.default_rng(ent).bit_generator
    G[f"rng_u32_{i}"] = np.array([bg.random_raw() for _ in range(32)], dtype=np.uint64)
META["n_entropies"] = len(ENTROPIES)

# ---------------------------------------------- captured trainer arrays ----
captured = {"factor": [], "core": []}
_orig_f, _orig_c = _loops.factor_pass, _loops.core_pass


def _wrap_f(idx, vals, visit, *a):
    captured["factor"].append(np.array(visit))
    return _orig_f(idx, vals, visit, *a)


def _wrap_c(idx, vals, visit, *a):
    captured["core"].append(np.array(visit))
    return _orig_c(idx, vals, visit, *a)


def run_train(name, dims, nnz, jr, r, *, noise=0.1, seed=3, test_fraction=0.1, workers=1,
              epochs=2, cap=1 << 20, update_core=True, alpha_a=0.009, init_seed=1, train_seed=1,
              store_arrays=True, capture=True):
    t, _ = generate_synthetic(dims, nnz, jr, r, noise_sigma=noise, seed=seed)
    ds = split(t, test_fraction, seed=seed) if test_fraction else DatasetSplit(
        t, SparseTensorCoo(t.dims, np.empty((0, t.order), dtype=np.int64), np.empty(0)))
    scale = default_init_scale(ds.train.values, len(dims))
    m = init_model(dims, ModelConfig(tuple(jr), r, scale, seed=init_seed))
    cfg = TrainConfig(epochs=epochs, workers=workers, seed=train_seed, core_batch_cap=cap,
                      update_core=update_core, alpha_a=alpha_a)
    init_f = [a.copy() for a in m.factors]
    init_b = [b.copy() for b in m.core_factors]
    captured["factor"].clear()
    captured["core"].clear()
    if capture:
        _loops.factor_pass, _loops.core_pass = _wrap_f, _wrap_c
    t0 = time.perf_counter()
    try:
        rows = train(m, ds, cfg)
    finally:
        _loops.factor_pass, _loops.core_pass = _orig_f, _orig_c
    el = time.perf_counter() - t0
    META[f"train_{name}"] = {
        "dims": list(dims), "nnz": nnz, "jr": list(jr), "r": r, "noise": noise, "seed": seed,
        "test_fraction": test_fraction, "workers": workers, "epochs": epochs, "cap": cap,
        "update_core": update_core, "alpha_a": alpha_a, "init_seed": init_seed,
        "train_seed": train_seed, "scale": scale, "seconds": el,
        "rows": [r_.__dict__ for r_ in rows],
        "n_factor_calls": len(captured["factor"]), "n_core_calls": len(captured["core"]),
        "final_hash": hashlib.sha256(b"".join(a.tobytes() for a in m.factors + m.core_factors)).hexdigest(),
    }
    if store_arrays:
        G[f"train_{name}_train_idx"] = ds.train.indices
        G[f"train_{name}_train_vals"] = ds.train.values
        G[f"train_{name}_test_idx"] = ds.test.indices
        G[f"train_{name}_test_vals"] = ds.test.values
        for n in range(len(dims)):
            G[f"train_{name}_A{n}_init"] = init_f[n]
            G[f"train_{name}_B{n}_init"] = init_b[n]
            G[f"train_{name}_A{n}_final"] = m.factors[n]
            G[f"train_{name}_B{n}_final"] = m.core_factors[n]
    if capture:
        for k, v in enumerate(captured["factor"]):
            G[f"train_{name}_visit_{k}"] = v
        for k, v in enumerate(captured["core"]):
            G[f"train_{name}_psi_{k}"] = v
    print(f"train {name}: {el:.2f}s rows={[round(r_.test_rmse, 6) for r_ in rows]}", flush=True)
    return rows


# small, full-array cases (DSGD with 1/2/3 workers, order 3 and 4, R=1)
run_train("s3w1", (20, 22, 24), 600, (3, 3, 3), 2, epochs=2, workers=1)
run_train("s3w2", (20, 22, 24), 600, (3, 3, 3), 2, epochs=2, workers=2)
run_train("s3w3", (21, 22, 25), 700, (2, 3, 4), 3, epochs=2, workers=3)
run_train("s4w2", (9, 10, 11, 12), 900, (2, 2, 3, 2), 2, epochs=2, workers=2)
run_train("r1", (12, 12, 12), 300, (2, 2, 2), 1, epochs=2, workers=1)
# core batch cap below nnz: Floyd path (pop <= 10000) and tail path (pop > 10000, k > pop // 50)
run_train("floyd", (30, 30, 30), 3000, (2, 2, 2), 2, epochs=2, cap=64, test_fraction=0.0)
run_train("tail", (40, 40, 40), 13000, (2, 2, 2), 2, epochs=2, cap=1000, test_fraction=0.0)
run_train("floydbig", (60, 60, 60), 30000, (2, 2, 2), 2, epochs=1, cap=200, test_fraction=0.0)
# BASELINE configs[0]: 1K^3, 100K nnz, J=R=8 (90K train / 10K test)
run_train("cfg1", (1000, 1000, 1000), 100_000, (8, 8, 8), 8, noise=0.1, seed=7,
          test_fraction=0.1, epochs=5, init_seed=1, train_seed=1, capture=True)
run_train("cfg1w4", (1000, 1000, 1000), 100_000, (8, 8, 8), 8, noise=0.1, seed=7,
          test_fraction=0.1, epochs=5, workers=4, init_seed=1, train_seed=1, store_arrays=False,
          capture=False)

# ----------------------------------------------------- partition / schedule ----
rng = np.random.default_rng(3)
for c in range(8):
    order = int(rng.integers(2, 6))
    dims = tuple(int(rng.integers(4, 40)) for _ in range(order))
    nnz = int(rng.integers(1, 3000))
    idx = np.stack([rng.integers(0, d, nnz) for d in dims], axis=1)
    tt = SparseTensorCoo(dims, idx, rng.standard_normal(nnz))
    m = int(rng.integers(1, min(dims) + 1))
    plan = build_partition(tt, m)
    keys = sorted(plan.block_entries)
    G[f"part_{c}_idx"] = idx
    G[f"part_{c}_dims"] = np.array(dims)
    G[f"part_{c}_m"] = np.array(m)
    G[f"part_{c}_blocks"] = np.array(keys, dtype=np.int64)
    G[f"part_{c}_ids"] = np.concatenate([plan.block_entries[k] for k in keys])
    G[f"part_{c}_sizes"] = np.array([len(plan.block_entries[k]) for k in keys])
    G[f"part_{c}_bounds"] = np.array([b for bb in plan.boundaries for b in bb])
META["n_part"] = 8
for order, m in [(2, 3), (3, 2), (3, 4), (4, 3), (6, 2), (5, 4)]:
    s = round_schedule(order, m)
    G[f"sched_{order}_{m}"] = np.array(s.rounds, dtype=np.int64)

# ------------------------------------------------------ _loops directly ----
rng = np.random.default_rng(11)
for c in range(4):
    order = int(rng.integers(2, 6))
    dims = tuple(int(rng.integers(3, 30)) for _ in range(order))
    jr = np.array([int(rng.integers(1, 7)) for _ in range(order)], dtype=np.int64)
    r = int(rng.integers(1, 7))
    fac = rng.uniform(-1, 1, size=int(sum(d * j for d, j in zip(dims, jr))))
    foff = np.r_[0, np.cumsum([d * j for d, j in zip(dims, jr)])].astype(np.int64)
    cor = rng.uniform(-1, 1, size=int(jr.sum() * r))
    coff = np.r_[0, np.cumsum(jr * r)].astype(np.int64)
    nnz = int(rng.integers(10, 400))
    idx = np.stack([rng.integers(0, d, nnz) for d in dims], axis=1).astype(np.int64)
    vals = rng.standard_normal(nnz)
    visit = rng.integers(0, nnz, size=int(rng.integers(5, 2 * nnz)))
    gam = rng.uniform(0.001, 0.05, order)
    lam = rng.uniform(0.0, 0.1, order)
    G[f"loops_{c}_dims"] = np.array(dims)
    G[f"loops_{c}_jr"] = jr
    G[f"loops_{c}_r"] = np.array(r)
    G[f"loops_{c}_fac"] = fac.copy()
    G[f"loops_{c}_foff"] = foff
    G[f"loops_{c}_cor"] = cor
    G[f"loops_{c}_coff"] = coff
    G[f"loops_{c}_idx"] = idx
    G[f"loops_{c}_vals"] = vals
    G[f"loops_{c}_visit"] = visit
    G[f"loops_{c}_gam"] = gam
    G[f"loops_{c}_lam"] = lam
    f2 = fac.copy()
    _loops.factor_pass(idx, vals, visit, f2, foff, cor, coff, jr, r, gam, lam)
    G[f"loops_{c}_fac_out"] = f2
    acc = np.zeros(coff[-1])
    _loops.core_pass(idx, vals, visit, fac, foff, cor, coff, jr, r, acc, coff)
    G[f"loops_{c}_acc_out"] = acc
    model = TuckerModel(dims, tuple(int(j) for j in jr), r,
                        [fac[foff[n]:foff[n + 1]].reshape(dims[n], jr[n]) for n in range(order)],
                        [cor[coff[n]:coff[n + 1]].reshape(jr[n], r) for n in range(order)])
    G[f"loops_{c}_pred"] = predict_entries(model, idx)
META["n_loops"] = 4

# ------------------------------------- sampler at small and full sizes ----
# The reference's samplers are these exact calls (trainer.py:196-199, 317-324).
small = {}
for n in [1, 2, 3, 5, 17, 100, 1000, 4097, 65536, 100_003]:
    ent = [5, 1, 3, 0, n % 5]
    G[f"perm_{n}"] = np.random.default_rng(ent).permutation(n)
    G[f"perm_{n}_ent"] = np.array(ent, dtype=np.uint64)
for pop, k in [(100, 10), (10000, 9000), (10001, 9000), (500_000, 5000), (500_000, 20_000),
               (4_000_000, 1 << 20), (200, 200)]:
    ent = [9, 2, pop % 13]
    G[f"choice_{pop}_{k}"] = np.random.default_rng(ent).choice(pop, size=k, replace=False)
    G[f"choice_{pop}_{k}_ent"] = np.array(ent, dtype=np.uint64)

big = {}
NF = 99_072_112
for t in range(2):
    ent = [1, 1, t, 0, 0, 0]
    t0 = time.perf_counter()
    p = np.random.default_rng(ent).permutation(NF)
    big[f"perm_NF_t{t}"] = {"entropy": ent, "n": NF, "sha256_i32": h32(p),
                            "head": p[:64].tolist(), "tail": p[-64:].tolist(),
                            "seconds": time.perf_counter() - t0}
    print("perm NF", t, time.perf_counter() - t0, flush=True)
    ent = [1, 2, t]
    psi = np.random.default_rng(ent).choice(NF, size=1 << 20, replace=False)
    big[f"psi_NF_t{t}"] = {"entropy": ent, "pop": NF, "k": 1 << 20, "sha256_i32": h32(psi),
                           "sha256_sorted_i32": h32(np.sort(psi)), "head": psi[:64].tolist()}
for n in [1 << 20, 3_000_017, 12_345_678]:
    ent = [42, 1, 0, 0, 0, 0]
    p = np.random.default_rng(ent).permutation(n)
    big[f"perm_{n}"] = {"entropy": ent, "n": n, "sha256_i32": h32(p), "head": p[:64].tolist()}
META["big"] = big

np.savez_compressed(os.path.join(HERE, "golden.npz"), **G)
with open(os.path.join(HERE, "golden_meta.json"), "w") as fh:
    json.dump(META, fh, indent=1, default=float)
print("wrote", len(G), "arrays")

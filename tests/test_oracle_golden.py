"""Pin the oracle (oracle/, the C restatement of the reference) against golden
vectors written by the reference itself (tests/golden/make_golden.py).
CPU only."""

import numpy as np
import pytest

from conftest import golden_train_case
from oracle import oracle as O

GOLDEN_TRAIN = ["s3w1", "s3w2", "s3w3", "s4w2", "r1", "floyd", "tail", "floydbig"]


def test_seed_sequence_pcg64_states(golden, golden_meta):
    for i in range(golden_meta["n_entropies"]):
        ent = golden[f"rng_entropy_{i}"].tolist()
        assert np.array_equal(O.pcg64_state(ent), golden[f"rng_state_{i}"]), ent


def test_raw_stream_matches_pcg64_outputs(golden, golden_meta):
    for i in range(golden_meta["n_entropies"]):
        st = golden[f"rng_state_{i}"]
        u32 = O.u32_stream(st, 64).astype(np.uint64)
        raw = golden[f"rng_u32_{i}"]  # 64-bit outputs: low half first
        assert np.array_equal(u32[0::2] | (u32[1::2] << np.uint64(32)), raw)


@pytest.mark.parametrize("n", [1, 2, 3, 5, 17, 100, 1000, 4097, 65536, 100_003])
def test_permutation_matches_reference(golden, n):
    ent = golden[f"perm_{n}_ent"].tolist()
    assert np.array_equal(O.permutation(ent, n), golden[f"perm_{n}"])


@pytest.mark.parametrize("pop,k", [(100, 10), (10000, 9000), (10001, 9000), (500_000, 5000),
                                   (500_000, 20_000), (4_000_000, 1 << 20), (200, 200)])
def test_choice_matches_reference(golden, pop, k):
    ent = golden[f"choice_{pop}_{k}_ent"].tolist()
    got, path = O.choice(ent, pop, k)
    assert np.array_equal(got, golden[f"choice_{pop}_{k}"])
    assert path == ("tail" if pop > 10000 and k > pop // 50 else "floyd")


def test_partition_matches_reference(golden, golden_meta):
    for c in range(golden_meta["n_part"]):
        idx, dims, m = golden[f"part_{c}_idx"], golden[f"part_{c}_dims"], int(golden[f"part_{c}_m"])
        ids, keys = O.partition(idx, dims, m)
        assert np.array_equal(ids, golden[f"part_{c}_ids"])
        blocks = O.block_entries(idx, dims, m)
        assert sorted(blocks) == [tuple(b) for b in golden[f"part_{c}_blocks"].tolist()]


@pytest.mark.parametrize("order,m", [(2, 3), (3, 2), (3, 4), (4, 3), (6, 2), (5, 4)])
def test_round_schedule_matches_reference(golden, order, m):
    assert np.array_equal(np.array(O.round_schedule(order, m)), golden[f"sched_{order}_{m}"])


def test_loops_bitwise(golden, golden_meta):
    """The C factor/core passes equal numba's _loops bit for bit."""
    for c in range(golden_meta["n_loops"]):
        g = {k: golden[f"loops_{c}_{k}"] for k in ("jr", "fac", "foff", "cor", "coff", "idx", "vals",
                                                   "visit", "gam", "lam", "fac_out", "acc_out", "pred")}
        r = int(golden[f"loops_{c}_r"])
        fac = g["fac"].copy()
        O.factor_pass(g["idx"], g["vals"], g["visit"], fac, g["foff"], g["cor"], g["coff"], g["jr"], r,
                      g["gam"], g["lam"])
        assert np.array_equal(fac, g["fac_out"])
        acc = np.zeros(g["coff"][-1])
        O.core_pass(g["idx"], g["vals"], g["visit"], g["fac"], g["foff"], g["cor"], g["coff"], g["jr"], r,
                    acc, g["coff"])
        assert np.array_equal(acc, g["acc_out"])
        order = len(g["jr"])
        dims = golden[f"loops_{c}_dims"]
        fs = [g["fac"][g["foff"][n]:g["foff"][n + 1]].reshape(dims[n], g["jr"][n]) for n in range(order)]
        bs = [g["cor"][g["coff"][n]:g["coff"][n + 1]].reshape(g["jr"][n], r) for n in range(order)]
        np.testing.assert_allclose(O.predict(fs, bs, g["idx"]), g["pred"], rtol=1e-13, atol=1e-13)


@pytest.mark.parametrize("name", GOLDEN_TRAIN)
def test_train_matches_reference(golden, golden_meta, name):
    """Whole-run equality: visit orders, core batches, schedule, merges."""
    case = golden_train_case(golden, golden_meta, name)
    m = case["meta"]
    fs = [a.copy() for a in case["A0"]]
    bs = [b.copy() for b in case["B0"]]
    rows = O.train(fs, bs, case["train_idx"], case["train_vals"], case["test_idx"], case["test_vals"],
                   epochs=m["epochs"], workers=m["workers"], seed=m["train_seed"], core_batch_cap=m["cap"],
                   update_core=m["update_core"], alpha_a=m["alpha_a"], dims=tuple(m["dims"]))
    for a, b in zip(fs + bs, case["A1"] + case["B1"]):
        assert np.array_equal(a, b)
    for got, want in zip(rows, m["rows"]):
        for key in ("train_rmse", "train_mae", "test_rmse", "test_mae", "gamma_a", "gamma_b"):
            if np.isnan(want[key]):
                assert np.isnan(got[key])
            else:
                assert got[key] == pytest.approx(want[key], rel=1e-12)


def test_train_visit_orders_are_reference_calls(golden, golden_meta):
    """The captured visit arrays equal ids[permutation] with the [seed,1,t,*block] streams."""
    case = golden_train_case(golden, golden_meta, "s3w2")
    blocks = O.block_entries(case["train_idx"], tuple(case["meta"]["dims"]), 2)
    sched = O.round_schedule(3, 2)
    k = 0
    for t in range(case["meta"]["epochs"]):
        for rnd in sched:
            for block in rnd:
                ids = blocks.get(block)
                if ids is None:
                    continue
                want = golden[f"train_s3w2_visit_{k}"]
                assert np.array_equal(ids[O.permutation([1, 1, t, *block], len(ids))], want)
                k += 1


def test_cfg1_reference_curve(golden, golden_meta):
    """BASELINE configs[0] (1K^3, 90K train, J=R=8): the oracle reproduces the
    reference's 5-epoch run exactly."""
    case = golden_train_case(golden, golden_meta, "cfg1")
    m = case["meta"]
    fs = [a.copy() for a in case["A0"]]
    bs = [b.copy() for b in case["B0"]]
    rows = O.train(fs, bs, case["train_idx"], case["train_vals"], case["test_idx"], case["test_vals"],
                   epochs=m["epochs"], seed=m["train_seed"])
    for got, want in zip(rows, m["rows"]):
        assert got["test_rmse"] == pytest.approx(want["test_rmse"], rel=1e-12)
    for a, b in zip(fs + bs, case["A1"] + case["B1"]):
        assert np.array_equal(a, b)

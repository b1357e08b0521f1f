"""Exact mode across the GPU (sptk_factor_pass_exact, factor_dep.cu): the
predecessor-driven schedule must reproduce the reference's strictly
sequential factor loop (_loops.py:17-63) bit for bit in fp64 -- against the
reference's own golden outputs and the oracle -- and equal the one-warp
sequential walker bit for bit in fp32."""

import numpy as np
import pytest
import torch

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _dev(a, dtype):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=dtype)).cuda()


def _run(idx, vals, fac, foff, cor, coff, jr, r, visit, gam, lam, f64, exact):
    from paper_2204_07104_b200 import _lib
    from paper_2204_07104_b200.device import DeviceCoo

    L = _lib.load()
    recs = DeviceCoo(idx, vals, f64=f64)
    dt = np.float64 if f64 else np.float32
    dfac, dcor = _dev(fac, dt), _dev(cor, dt)
    dvis = _dev(visit, np.int32)
    _, pf = _lib.i64arr(foff)
    _, pc = _lib.i64arr(coff)
    _, pj = _lib.i64arr(jr)
    _, pg = _lib.f64arr(gam)
    _, pl = _lib.f64arr(lam)
    n = len(jr)
    if exact:
        ws = torch.empty(int(L.sptk_factor_pass_exact_ws_bytes(len(visit), n)), dtype=torch.uint8, device="cuda")
        fn = L.sptk_factor_pass_exact_f64 if f64 else L.sptk_factor_pass_exact
        _lib.check(fn(recs.rec.data_ptr(), recs.rw, dvis.data_ptr(), len(visit), 0, dfac.data_ptr(), pf,
                      dcor.data_ptr(), pc, pj, n, r, pg, pl, ws.data_ptr(), ws.numel(), _lib.stream_ptr()), "exact")
        assert L.sptk_last_factor_kernel().decode() == "factor_dep_kernel"
    else:
        fn = L.sptk_factor_pass_f64 if f64 else L.sptk_factor_pass
        _lib.check(fn(recs.rec.data_ptr(), recs.rw, dvis.data_ptr(), len(visit), 0, dfac.data_ptr(), pf,
                      dcor.data_ptr(), pc, pj, n, r, pg, pl, 1, _lib.stream_ptr()), "seq")
    torch.cuda.synchronize()
    return dfac.cpu().numpy()


@pytest.mark.parametrize("c", range(4))
def test_exact_fp64_reference_golden(golden, c):
    """The reference's own factor_pass outputs (numba, tests/golden)."""
    g = {k: golden[f"loops_{c}_{k}"] for k in ("jr", "fac", "foff", "cor", "coff", "idx", "vals", "visit",
                                               "gam", "lam", "fac_out")}
    r = int(golden[f"loops_{c}_r"])
    out = _run(g["idx"], g["vals"], g["fac"], g["foff"], g["cor"], g["coff"], g["jr"], r, g["visit"], g["gam"],
               g["lam"], True, True)
    np.testing.assert_array_equal(out, g["fac_out"])


CASES = [
    # dims, jr, R, nnz: hot rows (long predecessor chains), cfg1-like, order 4
    # and 6, J != R, duplicates, wide ranks
    ((50, 7, 3), (4, 4, 4), 4, 20_000),
    ((1000, 1000, 1000), (8, 8, 8), 8, 90_000),
    ((2000, 300, 40), (16, 16, 16), 16, 60_000),
    ((30, 40, 50, 60), (5, 6, 7, 8), 3, 30_000),
    ((12, 13, 14, 15, 16, 17), (4, 4, 4, 4, 4, 4), 4, 15_000),
    ((400, 300, 200), (32, 32, 32), 32, 8_000),
    ((5, 5, 5), (3, 2, 4), 5, 4_000),
]


def _case(dims, jr, r, nnz, seed):
    rng = np.random.default_rng(seed)
    idx = np.stack([rng.integers(0, d, nnz) for d in dims], axis=1)
    fs = [rng.uniform(0, 1.2 / np.sqrt(j), (d, j)) for d, j in zip(dims, jr)]
    bs = [rng.uniform(0, 1.2 / np.sqrt(r), (j, r)) for j in jr]
    vals = rng.normal(2.0, 1.0, nnz)
    fac, foff = O.pack(fs)
    cor, coff = O.pack(bs)
    visit = rng.permutation(nnz)
    return idx, vals, fac, foff, cor, coff, np.array(jr), visit


@pytest.mark.parametrize("dims,jr,r,nnz", CASES)
def test_exact_fp64_equals_oracle(dims, jr, r, nnz):
    idx, vals, fac, foff, cor, coff, jra, visit = _case(dims, jr, r, nnz, 11)
    n = len(dims)
    gam, lam = np.full(n, 0.003), np.full(n, 0.01)
    got = _run(idx, vals, fac, foff, cor, coff, jra, r, visit, gam, lam, True, True)
    want = fac.copy()
    O.factor_pass(idx, vals, visit.astype(np.int64), want, foff, cor, coff, jra, r, gam, lam)
    np.testing.assert_array_equal(got, want)


@pytest.mark.parametrize("dims,jr,r,nnz", CASES[:4])
def test_exact_fp32_equals_sequential_walker(dims, jr, r, nnz):
    idx, vals, fac, foff, cor, coff, jra, visit = _case(dims, jr, r, nnz, 12)
    n = len(dims)
    gam, lam = np.full(n, 0.003), np.full(n, 0.01)
    a = _run(idx, vals, fac, foff, cor, coff, jra, r, visit, gam, lam, False, True)
    b = _run(idx, vals, fac, foff, cor, coff, jra, r, visit, gam, lam, False, False)
    assert a.tobytes() == b.tobytes()


def test_exact_train_cfg1_matches_reference_curve(golden_meta):
    """train() in exact fp64 mode (now on the predecessor-driven kernel) still
    reproduces the reference's cfg1 runs: covered by test_gpu_train's bitwise
    tests; here only that the dispatch really takes the new kernel."""
    from paper_2204_07104_b200 import ModelConfig, TrainConfig, default_init_scale, generate_synthetic, init_model
    from paper_2204_07104_b200 import _lib, split, train

    t, _ = generate_synthetic((200, 210, 220), 12_000, (4, 4, 4), 4, noise_sigma=0.1, seed=3)
    ds = split(t, 0.1, seed=3)
    m = init_model(t.dims, ModelConfig((4, 4, 4), 4, default_init_scale(ds.train.values, 3), seed=1))
    fs = [a.copy() for a in m.factors]
    bs = [b.copy() for b in m.core_factors]
    rows = train(m, ds, TrainConfig(epochs=2, seed=1, update_mode="exact", precision="fp64"))
    assert _lib.load().sptk_last_factor_kernel().decode() == "factor_dep_kernel"
    ref = O.train(fs, bs, ds.train.indices, ds.train.values, ds.test.indices, ds.test.values, epochs=2, seed=1)
    for a, b in zip(m.factors + m.core_factors, fs + bs):
        np.testing.assert_allclose(a, b, rtol=1e-10, atol=1e-13)
    assert abs(rows[-1].test_rmse - ref[-1]["test_rmse"]) <= 1e-9 * ref[-1]["test_rmse"]

"""K1/K3/K4/K5/K6 on the GPU against the reference's golden vectors and the oracle."""

import numpy as np
import pytest
import torch

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _dev(a, dtype):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=dtype)).cuda()


def _loops_case(golden, c):
    g = {k: golden[f"loops_{c}_{k}"] for k in ("jr", "fac", "foff", "cor", "coff", "idx", "vals", "visit",
                                               "gam", "lam", "fac_out", "acc_out", "pred")}
    g["r"] = int(golden[f"loops_{c}_r"])
    g["dims"] = golden[f"loops_{c}_dims"]
    return g


def _records(idx, vals, f64):
    from paper_2204_07104_b200.device import DeviceCoo

    return DeviceCoo(idx, vals, f64=f64)


def test_partition_golden(golden, golden_meta):
    from paper_2204_07104_b200.schedule import DevicePartition, build_partition
    from paper_2204_07104_b200.tensor import SparseTensorCoo

    for c in range(golden_meta["n_part"]):
        idx, dims, m = golden[f"part_{c}_idx"], golden[f"part_{c}_dims"], int(golden[f"part_{c}_m"])
        dp = DevicePartition(idx, np.arange(len(idx), dtype=np.float64), dims, m)
        assert np.array_equal(dp.ids[: len(idx)].cpu().numpy(), golden[f"part_{c}_ids"])
        sizes = np.diff(dp.block_off)
        assert np.array_equal(sizes[sizes > 0], golden[f"part_{c}_sizes"])
        # records carry the grouped entries
        rec = dp.rec.cpu().numpy().reshape(-1, dp.rw)[: len(idx)]
        assert np.array_equal(rec[:, : idx.shape[1]], idx[golden[f"part_{c}_ids"]])
        plan = build_partition(SparseTensorCoo(tuple(dims), idx, np.zeros(len(idx))), m)
        want = {tuple(b) for b in golden[f"part_{c}_blocks"].tolist()}
        assert set(plan.block_entries) == want


def test_partition_single_block_identity():
    """m = 1 (one worker): one block in source order, without the key sort."""
    from paper_2204_07104_b200.schedule import DevicePartition

    rng = np.random.default_rng(8)
    dims = (50, 60, 70)
    idx = np.stack([rng.integers(0, d, 123_457) for d in dims], axis=1)
    vals = rng.normal(size=len(idx))
    dp = DevicePartition(idx, vals, dims, 1)
    n = len(idx)
    assert np.array_equal(dp.ids[:n].cpu().numpy(), np.arange(n))
    assert np.array_equal(dp.pos_of_id[:n].cpu().numpy(), np.arange(n))
    assert dp.block_off.tolist() == [0, n]
    rec = dp.rec.cpu().numpy().reshape(-1, dp.rw)[:n]
    assert np.array_equal(rec[:, :3], idx)
    assert np.array_equal(rec[:, 3].view(np.float32), vals.astype(np.float32))


def test_partition_many_blocks_stable():
    """Keys needing two radix passes (m^N = 4096) stay stable."""
    from paper_2204_07104_b200.schedule import DevicePartition

    rng = np.random.default_rng(5)
    dims = (64, 70, 80, 90)
    idx = np.stack([rng.integers(0, d, 300_000) for d in dims], axis=1)
    dp = DevicePartition(idx, np.zeros(len(idx)), dims, 8)
    ids, _ = O.partition(idx, dims, 8)
    assert np.array_equal(dp.ids[: len(idx)].cpu().numpy(), ids)


@pytest.mark.parametrize("c", range(4))
def test_factor_seq_fp64_bitwise(golden, c):
    """Sequential fp64 mode reproduces numba's factor_pass bit for bit."""
    from paper_2204_07104_b200 import _lib

    g = _loops_case(golden, c)
    L = _lib.load()
    recs = _records(g["idx"], g["vals"], True)
    fac = _dev(g["fac"], np.float64)
    cor = _dev(g["cor"], np.float64)
    visit = _dev(g["visit"], np.int32)
    foff, pf = _lib.i64arr(g["foff"])
    coff, pc = _lib.i64arr(g["coff"])
    jr, pj = _lib.i64arr(g["jr"])
    gam, pg = _lib.f64arr(g["gam"])
    lam, pl = _lib.f64arr(g["lam"])
    _lib.check(L.sptk_factor_pass_f64(recs.rec.data_ptr(), recs.rw, visit.data_ptr(), len(g["visit"]), 0,
                                      fac.data_ptr(), pf, cor.data_ptr(), pc, pj, len(g["jr"]), g["r"], pg, pl, 1,
                                      _lib.stream_ptr()), "factor")
    np.testing.assert_array_equal(fac.cpu().numpy(), g["fac_out"])


@pytest.mark.parametrize("c", range(4))
def test_core_exact_fp64_bitwise(golden, c):
    from paper_2204_07104_b200 import _lib

    g = _loops_case(golden, c)
    L = _lib.load()
    recs = _records(g["idx"], g["vals"], True)
    fac = _dev(g["fac"], np.float64)
    cor = _dev(g["cor"], np.float64)
    visit = _dev(g["visit"], np.int32)
    _, pf = _lib.i64arr(g["foff"])
    _, pc = _lib.i64arr(g["coff"])
    jrc, pj = _lib.i64arr(g["jr"])
    acc = torch.zeros(int(g["coff"][-1]), dtype=torch.float64, device="cuda")
    ws = torch.empty(int(L.sptk_core_ws_bytes(pj, len(jrc), g["r"], 1)), dtype=torch.uint8, device="cuda")
    _lib.check(L.sptk_core_pass_f64(recs.rec.data_ptr(), recs.rw, visit.data_ptr(), None, len(g["visit"]),
                                    fac.data_ptr(), pf, cor.data_ptr(), pc, pj, len(jrc), g["r"], acc.data_ptr(),
                                    1, ws.data_ptr(), ws.numel(), _lib.stream_ptr()), "core")
    np.testing.assert_array_equal(acc.cpu().numpy(), g["acc_out"])


@pytest.mark.parametrize("c", range(4))
def test_core_throughput_fp32(golden, c):
    from paper_2204_07104_b200 import _lib

    g = _loops_case(golden, c)
    L = _lib.load()
    recs = _records(g["idx"], g["vals"], False)
    fac = _dev(g["fac"], np.float32)
    cor = _dev(g["cor"], np.float32)
    visit = _dev(g["visit"], np.int32)
    _, pf = _lib.i64arr(g["foff"])
    _, pc = _lib.i64arr(g["coff"])
    jrc, pj = _lib.i64arr(g["jr"])
    acc = torch.zeros(int(g["coff"][-1]), dtype=torch.float64, device="cuda")
    ws = torch.empty(int(L.sptk_core_ws_bytes(pj, len(jrc), g["r"], 0)), dtype=torch.uint8, device="cuda")
    _lib.check(L.sptk_core_pass(recs.rec.data_ptr(), recs.rw, visit.data_ptr(), None, len(g["visit"]),
                                fac.data_ptr(), pf, cor.data_ptr(), pc, pj, len(jrc), g["r"], acc.data_ptr(), 0,
                                ws.data_ptr(), ws.numel(), _lib.stream_ptr()), "core")
    want = g["acc_out"]
    np.testing.assert_allclose(acc.cpu().numpy(), want, rtol=1e-4, atol=1e-5 * np.abs(want).max())


@pytest.mark.parametrize("c", range(4))
def test_eval_golden(golden, c):
    from paper_2204_07104_b200 import TuckerModel
    from paper_2204_07104_b200.device import predict_device, predict_device_f64

    g = _loops_case(golden, c)
    order = len(g["jr"])
    fs = [g["fac"][g["foff"][n]:g["foff"][n + 1]].reshape(g["dims"][n], g["jr"][n]) for n in range(order)]
    bs = [g["cor"][g["coff"][n]:g["coff"][n + 1]].reshape(g["jr"][n], g["r"]) for n in range(order)]
    model = TuckerModel(tuple(g["dims"]), tuple(g["jr"]), g["r"], fs, bs)
    np.testing.assert_allclose(predict_device_f64(model, g["idx"]), g["pred"], rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(predict_device(model, g["idx"]), g["pred"], rtol=2e-5, atol=2e-5)


def _model_and_data(dims, jr, r, nnz, seed, distinct=False):
    rng = np.random.default_rng(seed)
    if distinct:
        n = min(dims)
        assert nnz <= n
        idx = np.stack([rng.permutation(d)[:nnz] for d in dims], axis=1)
    else:
        idx = np.stack([rng.integers(0, d, nnz) for d in dims], axis=1)
    fs = [rng.uniform(0, 1.2 / np.sqrt(j), (d, j)) for d, j in zip(dims, jr)]
    bs = [rng.uniform(0, 1.2 / np.sqrt(r), (j, r)) for j in jr]
    vals = rng.normal(2.0, 1.0, nnz)
    return idx, vals, fs, bs


def _run_factor(idx, vals, fs, bs, visit, mode, f64, gam=0.01, lam=0.01, tc=None):
    from paper_2204_07104_b200 import _lib

    L = _lib.load()
    prev = L.sptk_get_tc_mode()
    _lib.check(L.sptk_set_tc_mode(prev if tc is None else tc), "tc mode")
    fac, foff = O.pack(fs)
    cor, coff = O.pack(bs)
    jr = np.array([a.shape[1] for a in fs])
    recs = _records(idx, vals, f64)
    dt = np.float64 if f64 else np.float32
    dfac, dcor = _dev(fac, dt), _dev(cor, dt)
    dvis = _dev(visit, np.int32)
    _, pf = _lib.i64arr(foff)
    _, pc = _lib.i64arr(coff)
    _, pj = _lib.i64arr(jr)
    gm, pg = _lib.f64arr(np.full(len(fs), gam))
    lm, pl = _lib.f64arr(np.full(len(fs), lam))
    fn = L.sptk_factor_pass_f64 if f64 else L.sptk_factor_pass
    _lib.check(fn(recs.rec.data_ptr(), recs.rw, dvis.data_ptr(), len(visit), 0, dfac.data_ptr(), pf,
                  dcor.data_ptr(), pc, pj, len(fs), bs[0].shape[1], pg, pl, mode, _lib.stream_ptr()), "factor")
    out = dfac.double().cpu().numpy()
    _lib.check(L.sptk_set_tc_mode(prev), "tc mode")
    return out, fac, foff, cor, coff, jr


@pytest.mark.parametrize("dims,J", [((40, 50, 60), 4), ((300, 40, 30), 8), ((2000, 300, 100), 16),
                                    ((30, 40, 50, 60), 8), ((30, 40, 50, 60), 16), ((20, 21, 22, 23, 24, 25), 8),
                                    ((50, 60, 70), 32)])
def test_eval_uniform_ranks_vs_oracle(dims, J):
    """K6 specialised for uniform J = R (fp32) and the generic kernel: the
    predictions of the oracle within fp32 rounding, RMSE/MAE sums likewise."""
    from paper_2204_07104_b200 import TuckerModel
    from paper_2204_07104_b200.device import DeviceCoo, DeviceModel, eval_sums, predict_device

    idx, vals, fs, bs = _model_and_data(dims, (J,) * len(dims), J, 20001, 4)
    model = TuckerModel(tuple(dims), (J,) * len(dims), J, fs, bs)
    want = O.predict(fs, bs, idx)
    got = predict_device(model, idx)
    np.testing.assert_allclose(got, want, rtol=2e-5, atol=2e-5 * np.abs(want).max())
    s = eval_sums(DeviceModel(model), DeviceCoo(idx, vals)).cpu().numpy()
    d = vals - want
    np.testing.assert_allclose(s, [np.sum(d * d), np.sum(np.abs(d))], rtol=1e-4)


@pytest.mark.parametrize("dims,J,R", [((40, 50, 60), 4, 4), ((300, 40, 30), 8, 8), ((200, 300, 100), 16, 16),
                                      ((30, 40, 50, 60), 16, 16), ((20, 21, 22, 23, 24, 25), 8, 8),
                                      ((50, 60, 70), 32, 32), ((40, 50, 60), 5, 3)])
def test_factor_seq_fp32_one_epoch(dims, J, R):
    """Deterministic fp32 mode vs the fp64 oracle after one pass: |d| <= 1e-4 * |A| + 1e-5 * max|A|."""
    idx, vals, fs, bs = _model_and_data(dims, (J,) * len(dims), R, 3000, 1)
    visit = np.random.default_rng(2).permutation(len(vals))
    got, fac, foff, cor, coff, jr = _run_factor(idx, vals, fs, bs, visit, 1, False, gam=0.002)
    want = fac.copy()
    O.factor_pass(idx, vals, visit.astype(np.int64), want, foff, cor, coff, jr, R, np.full(len(dims), 0.002),
                  np.full(len(dims), 0.01))
    tol = 1e-4 * np.abs(want) + 1e-5 * np.abs(want).max()
    assert (np.abs(got - want) <= tol).all(), np.max(np.abs(got - want) / (np.abs(want) + 1e-12))


@pytest.mark.parametrize("dims,J,R", [((4000, 4000, 4000), 4, 4), ((4000, 4000, 4000), 8, 8),
                                      ((4000, 4000, 4000), 16, 16), ((3000,) * 4, 16, 16),
                                      ((3000,) * 6, 8, 8), ((3000, 3000, 3000), 32, 32),
                                      ((3000, 3000, 3000), 64, 64), ((300000, 3000, 3000), 64, 64),
                                      ((3000, 3000, 3000), 6, 5), ((300000, 3000, 3000), 16, 16),
                                      ((300000, 3000, 3000), 8, 8), ((300000,) * 4, 16, 16)])
@pytest.mark.parametrize("tc", [0, 1, 2, 3, 4, 5, 6])
def test_factor_hogwild_conflict_free_equals_sequential(dims, J, R, tc):
    """On samples touching pairwise-distinct rows the Hogwild kernels have no
    races, so they must equal the sequential semantics: FMA and 3xTF32 tcgen05
    at fp32 tolerance, single-pass TF32 (v1 straight, v2 folded refresh) at
    TF32 tolerance."""
    idx, vals, fs, bs = _model_and_data(dims, (J,) * len(dims), R, 2500, 3, distinct=True)
    visit = np.arange(len(vals))
    got, fac, foff, cor, coff, jr = _run_factor(idx, vals, fs, bs, visit, 0, False, gam=0.003, tc=tc)
    want = fac.copy()
    O.factor_pass(idx, vals, visit.astype(np.int64), want, foff, cor, coff, jr, R, np.full(len(dims), 0.003),
                  np.full(len(dims), 0.01))
    rtol = 5e-3 if tc in (1, 2, 4, 6) else 1e-4
    np.testing.assert_allclose(got, want, rtol=rtol, atol=rtol * 0.1 * np.abs(want).max())


@pytest.mark.parametrize("dims,J", [((40, 50, 60), 4), ((300, 40, 30), 8), ((200, 300, 100), 16),
                                    ((50, 60, 70), 32), ((30, 40, 50, 60), 8), ((30, 40, 50, 60), 16),
                                    ((20, 21, 22, 23, 24, 25), 8), ((50, 60, 70), 64)])
@pytest.mark.parametrize("nnz,sub", [(5000, None), (3000, 777), (1, None)])
def test_core_throughput_uniform_ranks(dims, J, nnz, sub):
    """Specialised K4 (uniform J = R, fp32, register-tiled outer products) vs
    the fp64 oracle core_pass, with and without a visit subset."""
    from paper_2204_07104_b200 import _lib

    L = _lib.load()
    idx, vals, fs, bs = _model_and_data(dims, (J,) * len(dims), J, nnz, 5)
    fac, foff = O.pack(fs)
    cor, coff = O.pack(bs)
    jr = np.array([a.shape[1] for a in fs])
    visit = np.arange(nnz) if sub is None else np.random.default_rng(9).choice(nnz, sub, replace=False)
    recs = _records(idx, vals, False)
    _, pf = _lib.i64arr(foff)
    _, pc = _lib.i64arr(coff)
    _, pj = _lib.i64arr(jr)
    dvis = _dev(visit, np.int32)
    acc = torch.zeros(int(coff[-1]), dtype=torch.float64, device="cuda")
    ws = torch.empty(int(L.sptk_core_ws_bytes(pj, len(jr), J, 0)), dtype=torch.uint8, device="cuda")
    dfac, dcor = _dev(fac, np.float32), _dev(cor, np.float32)  # keep the buffers alive across the call
    _lib.check(L.sptk_core_pass(recs.rec.data_ptr(), recs.rw, dvis.data_ptr(), None, len(visit), dfac.data_ptr(),
                                pf, dcor.data_ptr(), pc, pj, len(jr), J, acc.data_ptr(), 0, ws.data_ptr(),
                                ws.numel(), _lib.stream_ptr()), "core")
    want = np.zeros(int(coff[-1]))
    O.core_pass(idx, vals, visit.astype(np.int64), fac, foff, cor, coff, jr, J, want, coff)
    np.testing.assert_allclose(acc.cpu().numpy(), want, rtol=1e-4, atol=1e-5 * np.abs(want).max())


def test_rank4_zero_padding_is_exact():
    """J = R = 4 runs on a zero-padded rank-8 device model (tcgen05 tile):
    predictions, the factor pass on conflict-free samples and the core
    gradient equal the rank-4 reference, and the padding stays zero."""
    from paper_2204_07104_b200 import TuckerModel, _lib
    from paper_2204_07104_b200.device import DeviceModel, eval_sums

    dims, J = (4000, 4000, 4000), 4
    idx, vals, fs, bs = _model_and_data(dims, (J,) * 3, J, 2500, 3, distinct=True)
    model = TuckerModel(dims, (J,) * 3, J, [a.copy() for a in fs], [b.copy() for b in bs])
    dm = DeviceModel(model, pad_rank=8)
    assert list(dm.jr) == [8, 8, 8] and dm.rcore == 8
    recs = _records(idx, vals, False)
    L = _lib.load()
    # eval
    s_pad = eval_sums(dm, recs).cpu().numpy()
    s_ref = eval_sums(DeviceModel(model), recs).cpu().numpy()
    np.testing.assert_allclose(s_pad, s_ref, rtol=1e-5)
    # factor pass (Hogwild kernel, distinct rows -> sequential semantics)
    g, pg = _lib.f64arr([0.003] * 3)
    lam, pl = _lib.f64arr([0.01] * 3)
    visit = _dev(np.arange(len(vals)), np.int32)
    _lib.check(L.sptk_factor_pass(recs.rec.data_ptr(), recs.rw, visit.data_ptr(), len(vals), 0, dm.fac.data_ptr(),
                                  dm.p_foff, dm.cor.data_ptr(), dm.p_coff, dm.p_jr, 3, 8, pg, pl, 0,
                                  _lib.stream_ptr()), "factor")
    fac, foff = O.pack(fs)
    cor, coff = O.pack(bs)
    jr = np.array([J] * 3)
    O.factor_pass(idx, vals, np.arange(len(vals), dtype=np.int64), fac, foff, cor, coff, jr, J, np.full(3, 0.003),
                  np.full(3, 0.01))
    out = TuckerModel(dims, (J,) * 3, J, [np.zeros_like(a) for a in fs], [np.zeros_like(b) for b in bs])
    dm.download_into(out)
    got, _ = O.pack(out.factors)
    np.testing.assert_allclose(got, fac, rtol=5e-3, atol=5e-4 * np.abs(fac).max())
    padded = dm.fac.cpu().numpy()
    for n, d in enumerate(dims):
        rows = padded[dm.foff[n]: dm.foff[n + 1]].reshape(d, 8)
        assert not rows[:, J:].any()


@pytest.mark.parametrize("nbytes,threads", [(1, 0), (4097, 3), (20_000_003, 0), (50 << 20, 5)])
def test_h2d_upload_roundtrip(nbytes, threads):
    """sptk_h2d (threaded pinned staging) delivers the host bytes unchanged."""
    from paper_2204_07104_b200 import _lib

    L = _lib.load()
    src = np.random.default_rng(nbytes).integers(0, 256, nbytes, dtype=np.uint8)
    d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    _lib.check(L.sptk_h2d(d.data_ptr(), src.ctypes.data, nbytes, threads), "h2d")
    assert np.array_equal(d.cpu().numpy(), src)


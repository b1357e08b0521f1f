"""Factor-kernel time vs mode sizes (hot-row contention probe)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
from paper_2204_07104_b200 import _lib
from paper_2204_07104_b200.device import DeviceCoo
L = _lib.load()
nnz = 20_000_000
for dims in [(480189, 17770, 2182), (480189, 480189, 480189), (480189, 17770, 17770), (2182, 2182, 2182)]:
    rng = np.random.default_rng(1)
    idx = np.stack([rng.integers(0, d, nnz) for d in dims], axis=1)
    vals = rng.normal(0, 1, nnz)
    coo = DeviceCoo(idx, vals)
    fac = torch.rand(sum(d * 16 for d in dims), device="cuda") * 0.25
    cor = torch.rand(3 * 256, device="cuda") * 0.25
    foff, pf = _lib.i64arr(np.r_[0, np.cumsum([d * 16 for d in dims])])
    coff, pc = _lib.i64arr([0, 256, 512, 768])
    jr, pj = _lib.i64arr([16, 16, 16])
    g, pg = _lib.f64arr([1e-4] * 3)
    l, pl = _lib.f64arr([0.0] * 3)
    visit = torch.randperm(nnz, device="cuda", dtype=torch.int32)
    for tc in (0, 1, 2):
        L.sptk_set_tc_mode(tc)
        for rep in range(3):
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            _lib.check(L.sptk_factor_pass(coo.rec.data_ptr(), coo.rw, visit.data_ptr(), nnz, 0, fac.data_ptr(), pf,
                                          cor.data_ptr(), pc, pj, 3, 16, pg, pl, 0, _lib.stream_ptr()), "fp")
            e1.record(); e1.synchronize()
        print(dims, "tc", tc, "ms", round(e0.elapsed_time(e1), 3), "ns/nnz", round(e0.elapsed_time(e1) * 1e6 / nnz, 3), flush=True)

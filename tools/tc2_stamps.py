"""Per-phase cycle stamps of the tcgen05 factor kernel (block 0) on NF-shaped data."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
from paper_2204_07104_b200 import _lib
from paper_2204_07104_b200.device import DeviceCoo
L = _lib.load()
nnz = 20_000_000
dims = (480189, 17770, 2182)
rng = np.random.default_rng(1)
idx = np.stack([rng.integers(0, d, nnz) for d in dims], axis=1)
coo = DeviceCoo(idx, rng.normal(0, 1, nnz))
fac = torch.rand(sum(d * 16 for d in dims), device="cuda") * 0.25
cor = torch.rand(3 * 256, device="cuda") * 0.25
foff, pf = _lib.i64arr(np.r_[0, np.cumsum([d * 16 for d in dims])])
coff, pc = _lib.i64arr([0, 256, 512, 768])
jr, pj = _lib.i64arr([16, 16, 16])
g, pg = _lib.f64arr([1e-4] * 3)
l, pl = _lib.f64arr([0.0] * 3)
visit = torch.randperm(nnz, device="cuda", dtype=torch.int32)
st = torch.zeros(16 * 16, dtype=torch.int64, device="cuda")
for rep in range(2):
    L.sptk_debug_tc_buffer(st.data_ptr() if rep == 1 else None)
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    _lib.check(L.sptk_factor_pass(coo.rec.data_ptr(), coo.rw, visit.data_ptr(), nnz, 0, fac.data_ptr(), pf,
                                  cor.data_ptr(), pc, pj, 3, 16, pg, pl, 0, _lib.stream_ptr()), "fp")
    e1.record(); e1.synchronize()
    print("factor ns/nnz", round(e0.elapsed_time(e1) * 1e6 / nnz, 3), flush=True)
L.sptk_debug_tc_buffer(None)
s = st.view(16, 16).cpu().numpy()
names = ["tile", "rows issued", "gather+sync", "cMMA issued", "cMMA done"] + \
        [f"m{n}:{k}" for n in range(3) for k in ("W written", "W sync", "MMA done")] + ["m1:wb start", "end"]
for t in range(2, 10):
    row = s[t]
    base = row[0]
    d = [int(x - base) if x else -1 for x in row]
    print(f"tile {t}: total {int(s[t + 1][0] - base)} cyc | " + " ".join(f"{names[k]}={d[k]}" for k in range(16) if d[k] >= 0))

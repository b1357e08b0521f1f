"""Factor-pass timing on NF-shaped random data for the tcgen05 kernels (tc modes),
plus the v6 (TMA) kernel's per-phase stamps of block 0."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
from paper_2204_07104_b200 import _lib
from paper_2204_07104_b200.device import DeviceCoo
L = _lib.load()
nnz = int(os.environ.get("NNZ", 20_000_000))
J = int(os.environ.get("J", 16))
dims = tuple(int(x) for x in os.environ.get("DIMS", "480189,17770,2182").split(","))
N = len(dims)
rng = np.random.default_rng(1)
idx = np.stack([rng.integers(0, d, nnz) for d in dims], axis=1)
coo = DeviceCoo(idx, rng.normal(0, 1, nnz))
fac0 = torch.rand(sum(d * J for d in dims), device="cuda") * 0.25
cor = torch.rand(N * J * J, device="cuda") * 0.25
foff, pf = _lib.i64arr(np.r_[0, np.cumsum([d * J for d in dims])])
coff, pc = _lib.i64arr([n * J * J for n in range(N + 1)])
jr, pj = _lib.i64arr([J] * N)
g, pg = _lib.f64arr([1e-4] * N)
l, pl = _lib.f64arr([0.0] * N)
visit = torch.randperm(nnz, device="cuda", dtype=torch.int32)
st = torch.zeros(16 * 16, dtype=torch.int64, device="cuda")
for mode in [int(x) for x in os.environ.get("MODES", "1,6").split(",")]:
    L.sptk_set_tc_mode(mode)
    fac = fac0.clone()
    ts = []
    for rep in range(4):
        L.sptk_debug_tc_buffer(st.data_ptr() if rep == 3 else None)
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        _lib.check(L.sptk_factor_pass(coo.rec.data_ptr(), coo.rw, visit.data_ptr(), nnz, 0, fac.data_ptr(), pf,
                                      cor.data_ptr(), pc, pj, N, J, pg, pl, 0, _lib.stream_ptr()), "fp")
        e1.record(); e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    L.sptk_debug_tc_buffer(None)
    kern = L.sptk_last_factor_kernel().decode()
    print(f"mode {mode} {kern}: ms {[round(t, 3) for t in ts]}  ns/nnz {ts[1] / nnz * 1e6:.4f}  "
          f"NF-equiv ms {ts[1] / nnz * 99_072_112:.2f}  finite {bool(torch.isfinite(fac).all())}", flush=True)
    if mode == 6:
        s = st.view(16, 16).cpu().numpy()
        for t in range(2, 8):
            row = s[t]; base = row[0]
            d = [int(x - base) if x else -1 for x in row]
            print(f"  tile {t}: total {int(s[t + 1][0] - base)} | " + " ".join(f"{k}:{d[k]}" for k in range(16) if d[k] >= 0))
L.sptk_set_tc_mode(1)

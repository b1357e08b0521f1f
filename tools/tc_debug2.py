import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np, torch
from paper_2204_07104_b200 import _lib
import test_gpu_kernels as T
L = _lib.load()
N, J, R = 3, 16, 16
d = 4000
idx, vals, fs, bs = T._model_and_data((d, d, d), (16, 16, 16), 16, 128, 3, distinct=True)
visit = np.arange(len(vals))
S = 2 * N * R + N * J
for tc in (1, 3):
    dbg = torch.zeros(128 * S, dtype=torch.float32, device="cuda")
    L.sptk_debug_tc_buffer(dbg.data_ptr())
    got, fac, foff, cor, coff, jr = T._run_factor(idx, vals, fs, bs, visit, 0, False, gam=0.003, tc=tc)
    L.sptk_debug_tc_buffer(None)
    D = dbg.cpu().numpy().reshape(128, S)
    c = np.stack([fs[n][idx[:, n]] @ bs[n] for n in range(N)], axis=1)  # (128, N, R)
    print("tc", tc, "c err", np.abs(D[:, :N*R].reshape(128, N, R) - c).max(), "c scale", np.abs(c).max())
    a = [fs[n][idx[:, n]].copy() for n in range(N)]
    cc = c.copy()
    for n in range(N):
        w = np.prod(np.delete(cc, n, axis=1), axis=1)
        g = w @ bs[n].T
        gd = D[:, N*R + n*J: N*R + (n+1)*J]
        print("  mode", n, "gs err", np.abs(gd - g).max(), "scale", np.abs(g).max())
        inter = np.sum(a[n] * g, axis=1, keepdims=True)
        a[n] = a[n] - 0.003 * (-vals[:, None] * g + 0.01 * a[n] + inter * g)
        cc[:, n, :] = a[n] @ bs[n]
        if n < N - 1:
            cd = D[:, N*R + N*J + n*R: N*R + N*J + (n+1)*R]
            print("  mode", n, "refresh err", np.abs(cd - cc[:, n, :]).max())

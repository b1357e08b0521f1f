"""Time sptk_block_perm on an NF-like DSGD layout (M=32, N=3: 1024 rounds x 32 blocks of ~3K)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
from paper_2204_07104_b200.sampler import BlockOrders
M = int(os.environ.get("M", 32)); nb = int(os.environ.get("NB", 3024))
rng = np.random.default_rng(0)
rounds, off = [], 0
for r in range(M * M):
    rnd = []
    for s in range(M):
        n = int(rng.integers(nb - 150, nb + 150))
        rnd.append(((s, (s + r) % M, (s + r // M) % M), off, n))
        off += n
    rounds.append(rnd)
bo = BlockOrders(rounds, 3, "cuda")
out = torch.empty(bo.total, dtype=torch.int32, device="cuda")
for rep in range(3):
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); bo.draw(1, rep, out); e1.record(); e1.synchronize()
    print(f"block_perm {bo.n_jobs} blocks, {bo.total} nnz: {e0.elapsed_time(e1):.3f} ms", flush=True)

import time, numpy as np, torch
n = 99_072_112
idx = np.random.default_rng(0).integers(0, 400000, (n, 3))
vals = np.random.default_rng(1).normal(size=n)
print("threads", torch.get_num_threads(), flush=True)
for pinned in (False, True):
    t0 = time.perf_counter()
    rec = torch.zeros((n, 4), dtype=torch.int32, pin_memory=pinned)
    t1 = time.perf_counter()
    rec[:, :3] = torch.from_numpy(idx)
    rec[:, 3] = torch.from_numpy(vals).to(torch.float32).view(torch.int32)
    t2 = time.perf_counter()
    d = rec.view(-1).to("cuda", non_blocking=pinned); torch.cuda.synchronize()
    t3 = time.perf_counter()
    print(f"pinned={pinned}: alloc {t1-t0:.3f} pack {t2-t1:.3f} h2d {t3-t2:.3f} ({rec.numel()*4/(t3-t2)/1e9:.1f} GB/s)", flush=True)
t0 = time.perf_counter(); d = torch.from_numpy(idx).to("cuda"); torch.cuda.synchronize(); t1 = time.perf_counter()
print(f"int64 idx pageable h2d {t1-t0:.3f} ({idx.nbytes/(t1-t0)/1e9:.1f} GB/s)")

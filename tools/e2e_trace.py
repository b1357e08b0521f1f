"""Where the end-to-end train() time goes (NF bench workload): setup phases
and per-epoch epoch/eval time (diagnostic)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2204_07104_b200 import DatasetSplit, ModelConfig, TrainConfig, default_init_scale, init_model  # noqa
from paper_2204_07104_b200.device import DeviceCoo, rmse_mae_device  # noqa: E402
from paper_2204_07104_b200.training import EpochRunner, _RecordView, learning_rate  # noqa: E402

cfg = bench.CONFIGS["nf"]
tr, te, _ = bench.make_data(cfg)
scale = default_init_scale(tr.values, 3)
W = int(os.environ.get("WORKERS", cfg["workers"]))
for rep in range(2):
    m = init_model(cfg["dims"], ModelConfig((16,) * 3, 16, scale, seed=1))
    tc = TrainConfig(epochs=10, seed=1, workers=W, alpha_a=cfg["alpha_a"])
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    runner = EpochRunner(m, tr, tc)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    test_coo = DeviceCoo(te.indices, te.values)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    view = _RecordView(runner.part)
    ep, ev = 0.0, 0.0
    for t in range(10):
        a = time.perf_counter()
        runner.epoch(t, learning_rate(tc.alpha_a, tc.beta_a, t), learning_rate(tc.alpha_b, tc.beta_b, t))
        torch.cuda.synchronize()
        b = time.perf_counter()
        rmse_mae_device(runner.dm, view)
        rmse_mae_device(runner.dm, test_coo)
        c = time.perf_counter()
        ep += b - a
        ev += c - b
    t3 = time.perf_counter()
    runner.dm.download_into(m)
    t4 = time.perf_counter()
    print(f"rep {rep}: runner init {1e3*(t1-t0):.1f} ms, test upload {1e3*(t2-t1):.1f} ms, 10 epochs {1e3*ep:.1f} ms, "
          f"10 evals {1e3*ev:.1f} ms, download {1e3*(t4-t3):.1f} ms, total {1e3*(t4-t0):.1f} ms", flush=True)
# inside the runner init
import cProfile  # noqa: E402
import pstats  # noqa: E402

m = init_model(cfg["dims"], ModelConfig((16,) * 3, 16, scale, seed=1))
pr = cProfile.Profile()
pr.enable()
runner = EpochRunner(m, tr, TrainConfig(epochs=10, seed=1, workers=W, alpha_a=cfg["alpha_a"]))
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)

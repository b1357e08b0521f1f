"""Phase breakdown of the public train() on the NF bench tensor (host arrays in, model out)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import math
import torch
import bench
from paper_2204_07104_b200 import ModelConfig, TrainConfig, default_init_scale, init_model
from paper_2204_07104_b200 import training as T
from paper_2204_07104_b200.device import DeviceCoo, rmse_mae_device

cfg = bench.CONFIGS["nf"]
tr, te, _ = bench.make_data(cfg)
scale = default_init_scale(tr.values, 3)
for rep in range(3):
    m = init_model(cfg["dims"], ModelConfig((16,) * 3, 16, scale, seed=1))
    conf = TrainConfig(epochs=10, seed=1, alpha_a=0.003)
    ts = {}
    def mark(k):
        torch.cuda.synchronize(); ts[k] = time.perf_counter()
    mark("start")
    runner = T.EpochRunner(m, tr, conf)
    mark("runner")
    test_coo = DeviceCoo(te.indices, te.values)
    view = T._RecordView(runner.part)
    mark("test_upload")
    ev = 0.0; ep = 0.0
    for t in range(conf.epochs):
        a = time.perf_counter()
        runner.epoch(t, T.learning_rate(conf.alpha_a, conf.beta_a, t), T.learning_rate(conf.alpha_b, conf.beta_b, t))
        torch.cuda.synchronize(); b = time.perf_counter()
        rmse_mae_device(runner.dm, view); rmse_mae_device(runner.dm, test_coo)
        torch.cuda.synchronize(); c = time.perf_counter()
        ep += b - a; ev += c - b
        if t == 0: first = b - a
    mark("epochs")
    runner.dm.download_into(m)
    mark("download")
    print(f"rep {rep}: runner init {ts['runner']-ts['start']:.3f} s, test upload {ts['test_upload']-ts['runner']:.3f}, "
          f"epochs {ep:.3f} (first {first:.3f}), evals {ev:.3f}, download {ts['download']-ts['epochs']:.3f}, "
          f"total {ts['download']-ts['start']:.3f}", flush=True)

# pieces of the runner init
from paper_2204_07104_b200.schedule import DevicePartition
import numpy as np
for rep in range(2):
    torch.cuda.synchronize(); a = time.perf_counter()
    d_idx = torch.from_numpy(np.ascontiguousarray(tr.indices)).to("cuda")
    torch.cuda.synchronize(); b = time.perf_counter()
    d_val = torch.from_numpy(np.ascontiguousarray(tr.values)).to("cuda")
    torch.cuda.synchronize(); c = time.perf_counter()
    del d_idx, d_val
    part = DevicePartition(tr.indices, tr.values, tr.dims, 1, want_ids=False)
    torch.cuda.synchronize(); d = time.perf_counter()
    del part
    print(f"init pieces: idx upload {b-a:.3f} s ({tr.indices.nbytes/1e9:.2f} GB), val upload {c-b:.3f} s, "
          f"DevicePartition total {d-c:.3f} s; idx dtype {tr.indices.dtype} contiguous {tr.indices.flags.c_contiguous}", flush=True)

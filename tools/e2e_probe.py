"""Where the end-to-end train() time goes on the NF bench tensor."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import bench
from paper_2204_07104_b200 import DatasetSplit, ModelConfig, TrainConfig, default_init_scale, init_model, train
from paper_2204_07104_b200 import training as T
from paper_2204_07104_b200.device import DeviceCoo
from paper_2204_07104_b200.schedule import DevicePartition

cfg = bench.CONFIGS["nf"]
tr, te, _ = bench.make_data(cfg)
scale = default_init_scale(tr.values, 3)
for rep in range(2):
    m = init_model(cfg["dims"], ModelConfig((16,) * 3, 16, scale, seed=1))
    torch.cuda.synchronize(); t0 = time.perf_counter()
    part = DevicePartition(tr.indices, tr.values, tr.dims, 1, want_ids=False)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    tc = DeviceCoo(te.indices, te.values)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    runner = T.EpochRunner(m, tr, TrainConfig(epochs=5, seed=1, update_mode="hogwild", alpha_a=0.003))
    torch.cuda.synchronize(); t3 = time.perf_counter()
    for t in range(5):
        runner.epoch(t, 0.003, 0.0045)
    torch.cuda.synchronize(); t4 = time.perf_counter()
    del runner, part, tc
    torch.cuda.synchronize(); t5 = time.perf_counter()
    rows = train(m, DatasetSplit(tr, te), TrainConfig(epochs=5, seed=1, update_mode="hogwild", alpha_a=0.003))
    torch.cuda.synchronize(); t6 = time.perf_counter()
    print(f"rep {rep}: partition {t1-t0:.3f} s, test upload {t2-t1:.3f}, runner init (incl partition) {t3-t2:.3f}, "
          f"5 epochs {t4-t3:.3f}, full train() {t6-t5:.3f}", flush=True)

import sys; sys.path.insert(0,'/root/repo')
import numpy as np
from paper_2204_07104_b200 import ModelConfig, init_model
from paper_2204_07104_b200.device import predict_device_f64, predict_device
from paper_2204_07104_b200.tucker import predict_entries
for R in (32, 48, 64):
    m = init_model((50,60,70), ModelConfig((R,R,R), R, 0.5, seed=1))
    idx = np.stack([np.random.default_rng(0).integers(0, d, 1000) for d in (50,60,70)], 1)
    for fn in (predict_device_f64, predict_device):
        try:
            got = fn(m, idx); print(R, fn.__name__, np.abs(got - predict_entries(m, idx)).max())
        except Exception as e:
            print(R, fn.__name__, 'ERR', e)

"""Time the K6 evaluation kernels on the NF-shaped training records: two
train() epochs with per-epoch train/test RMSE, under
ncu --metrics gpu__time_duration.sum -k regex:eval."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2204_07104_b200 import DatasetSplit, ModelConfig, TrainConfig, default_init_scale, init_model, train  # noqa
from paper_2204_07104_b200.synthetic import generate_large  # noqa

dims = (480189, 17770, 2182)
tr, te, _ = generate_large(dims, 99_072_112, (16,) * 3, 16, 0.1, seed=7, n_test=1_408_395)
m = init_model(dims, ModelConfig((16,) * 3, 16, default_init_scale(tr.values, 3), seed=1))
rows = train(m, DatasetSplit(tr, te), TrainConfig(epochs=2, seed=1, alpha_a=0.003, workers=20, update_mode="hogwild"))
print(rows[-1])

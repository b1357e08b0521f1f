"""B200-native stochastic sparse Tucker decomposition (cuFastTucker's update).

Drop-in for the reference package ``sptucker``'s public API: the same names,
signatures and semantics, with the training hot path (samplers, factor and
core updates, evaluation, partitioning) running as hand-written sm_100a CUDA
kernels behind the C ABI in include/sptk.h.
"""

from .sklearn_api import TuckerSGD, check_index_array, check_values
from .synthetic import generate_large, generate_synthetic
from .tensor import (CooFormatError, DatasetSplit, SparseTensorCoo, load_coo, load_coo_binary, split, write_coo,
                     write_coo_binary)
from .training import (
    METRICS_HEADER,
    MetricsRow,
    TrainConfig,
    frobenius_objective,
    learning_rate,
    mae,
    rmse,
    train,
    write_metrics_csv,
)
from .tucker import (
    ModelConfig,
    TuckerModel,
    clone_model,
    default_init_scale,
    init_model,
    load_model,
    predict_entries,
    save_model,
    save_model_binary,
    load_model_binary,
)

__all__ = [
    "CooFormatError", "DatasetSplit", "SparseTensorCoo", "generate_synthetic", "load_coo", "split",
    "write_coo", "TuckerSGD", "check_index_array", "check_values", "ModelConfig", "TuckerModel",
    "clone_model", "default_init_scale", "init_model", "load_model", "predict_entries", "save_model",
    "MetricsRow", "TrainConfig", "frobenius_objective", "learning_rate", "mae", "rmse", "train",
    "write_metrics_csv", "generate_large", "METRICS_HEADER", "load_coo_binary", "write_coo_binary",
    "save_model_binary", "load_model_binary",
]

__version__ = "0.1.0"

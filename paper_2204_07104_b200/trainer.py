"""Compatibility alias: ``sptucker.trainer`` names."""
from .training import (METRICS_HEADER, MetricsRow, TrainConfig, frobenius_objective,  # noqa: F401
                       learning_rate, mae, rmse, train, write_metrics_csv)

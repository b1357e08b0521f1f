"""Compatibility alias: ``sptucker.estimator`` names."""
from .sklearn_api import TuckerSGD, check_index_array, check_values  # noqa: F401

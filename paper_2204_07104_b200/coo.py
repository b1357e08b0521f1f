"""Compatibility alias: ``sptucker.coo`` names."""
from .synthetic import generate_synthetic  # noqa: F401
from .tensor import CooFormatError, DatasetSplit, SparseTensorCoo, load_coo, split, write_coo  # noqa: F401

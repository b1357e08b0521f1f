"""Compatibility alias: ``sptucker.model`` names."""
from .tucker import (ModelConfig, TuckerModel, clone_model, default_init_scale, init_model,  # noqa: F401
                     load_model, predict_entries, save_model)

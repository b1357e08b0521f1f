"""Multi-GPU data division (placeholder until the DSGD path lands)."""

from __future__ import annotations


def active() -> bool:
    try:
        import torch.distributed as td
    except Exception:  # pragma: no cover
        return False
    return td.is_available() and td.is_initialized() and td.get_world_size() > 1


def train_distributed(model, split, config):  # pragma: no cover - replaced below
    raise NotImplementedError("multi-GPU training is not built yet")

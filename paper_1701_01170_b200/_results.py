"""Device -> reference-layout conversion helpers."""
from __future__ import annotations

import numpy as np

from ._native import UNVISITED32
from .graph import UNVISITED


def labels_to_host(t) -> np.ndarray:
    """int32 device labels (INT32_MAX = unreached) -> int64 numpy with the
    reference sentinel INT64_MAX (graph.py:19-22)."""
    import torch

    wide = t.to(torch.int64)
    wide = torch.where(t == UNVISITED32, torch.full_like(wide, UNVISITED), wide)
    return wide.cpu().numpy()


def preds_to_host(t) -> np.ndarray:
    import torch

    return t.to(torch.int64).cpu().numpy()

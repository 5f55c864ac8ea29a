"""Device -> reference-layout conversion helpers.

Results are widened to the reference's int64 layout on the GPU and copied
into pinned host memory (torch's caching host allocator), so the host side
costs one DMA and no host-side conversion pass.  The returned numpy arrays
own (keep alive) their pinned buffers.
"""
from __future__ import annotations

import numpy as np

from ._native import UNVISITED32
from .graph import UNVISITED


def _to_host(t):
    import torch

    out = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    out.copy_(t, non_blocking=True)
    torch.cuda.current_stream(t.device).synchronize()
    return out.numpy()


def labels_to_host(t) -> np.ndarray:
    """int32 device labels (INT32_MAX = unreached) -> int64 numpy with the
    reference sentinel INT64_MAX (graph.py:19-22)."""
    import torch

    wide = t.to(torch.int64)
    wide.masked_fill_(t == UNVISITED32, UNVISITED)
    return _to_host(wide)


def preds_to_host(t) -> np.ndarray:
    import torch

    return _to_host(t.to(torch.int64))


def tensor_to_host(t) -> np.ndarray:
    return _to_host(t)

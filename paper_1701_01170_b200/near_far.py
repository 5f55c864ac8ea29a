"""Two-slice near/far priority pile (reference near_far.py:20-85) in HBM.

``key`` is a callable from an int64 CUDA id tensor to the items' keys (a
CUDA tensor -- e.g. ``lambda ids: dist[ids]`` with ``dist`` device
resident); the near/far partitions are stable device compactions
(``gfx_select_i64``) and the far slice keeps its enqueue keys on the device.
The SSSP primitive runs its own fused pile (csrc/gfx_sssp.cu: k_sssp_split /
k_sssp_refar); this module is the operator-level API of the same rules:
near = key < threshold; when near drains the threshold rises by delta,
stale far entries (live key != enqueue key) are dropped and the rest is
re-split.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .frontier import VERTEX, Frontier, _is_tensor


def _keys(key, ids64):
    import torch

    k = key(ids64)
    k = k if _is_tensor(k) else torch.as_tensor(np.asarray(k))
    return k.to(device=ids64.device).reshape(-1)


def _split_mask(ids64, keys, threshold):
    import torch

    from .operators import _select

    near = (keys < threshold).to(torch.uint8).contiguous()
    return _select(ids64, near), _select(ids64, near, invert=True), near


def split(frontier: Frontier, key, threshold):
    """(near, far): items with key < threshold and the rest, stable and
    multiset-conserving (near_far.py:20-31)."""
    if len(frontier) == 0:
        return Frontier(kind=frontier.kind), Frontier(kind=frontier.kind)
    ids = frontier.device64()
    near, far, _ = _split_mask(ids, _keys(key, ids), threshold)
    return Frontier.from_device(near, frontier.kind), Frontier.from_device(far, frontier.kind)


def _empty_keys():
    return None


@dataclass
class NearFarPile:
    delta: float
    threshold: float
    near: Frontier = field(default_factory=lambda: Frontier(kind=VERTEX))
    far: Frontier = field(default_factory=lambda: Frontier(kind=VERTEX))
    far_keys: object = field(default_factory=_empty_keys)  # CUDA tensor aligned with far

    def push(self, frontier: Frontier, key) -> None:
        """Split incoming items at the current threshold; append the near share
        to near and the far share, with its enqueue keys, to far (near_far.py:42-60)."""
        import torch

        from .operators import _select

        if len(frontier) == 0:
            return
        ids = frontier.device64()
        keys = _keys(key, ids)
        near, far, mask = _split_mask(ids, keys, self.threshold)
        if len(self.near):
            near = torch.cat([self.near.device64(ids.device), near])
        self.near = Frontier.from_device(near, frontier.kind)
        if far.numel():
            fk = _select(keys.to(torch.int64), mask, invert=True)
            if len(self.far):
                far = torch.cat([self.far.device64(ids.device), far])
                fk = torch.cat([self.far_keys, fk])
            self.far = Frontier.from_device(far, frontier.kind)
            self.far_keys = fk

    def pop_near(self) -> Frontier:
        out = self.near
        self.near = Frontier(kind=out.kind)
        return out

    def empty(self) -> bool:
        return len(self.near) == 0 and len(self.far) == 0


def advance_bucket(pile: NearFarPile, key) -> NearFarPile:
    """Next bucket (near_far.py:63-85): threshold += delta, drop stale far
    entries, re-split.  Only legal with an empty near slice and a non-empty far one."""
    import torch

    from .operators import _select

    if len(pile.near):
        raise ValueError("advance_bucket requires an empty near slice")
    if len(pile.far) == 0:
        raise ValueError("advance_bucket requires a nonempty far slice")
    pile.threshold = pile.threshold + pile.delta
    ids = pile.far.device64()
    live = _keys(key, ids).to(torch.int64)
    fresh = (live == pile.far_keys).to(torch.uint8).contiguous()
    ids, live = _select(ids, fresh), _select(live, fresh)
    near, far, mask = _split_mask(ids, live, pile.threshold)
    pile.near = Frontier.from_device(near, pile.far.kind)
    pile.far_keys = _select(live, mask, invert=True)
    pile.far = Frontier.from_device(far, pile.far.kind)
    return pile

"""Operator vocabulary and the device operators (reference operators.py).

Functors: the reference passes arbitrary Python callables over whole id
arrays (operators.py:88-100).  Those cannot run on the GPU, and there is no
CPU fallback, so ``FunctorSet`` here holds entries of a CLOSED device-functor
registry (``DeviceFunctor``) -- the functors the six primitives use (SURVEY
8(b)).  Passing a plain Python callable raises ``TypeError``.
"""
from __future__ import annotations

from dataclasses import dataclass
from enum import Enum


class AdvanceKind(Enum):
    V2V = ("vertex", "vertex")
    V2E = ("vertex", "edge")
    E2V = ("edge", "vertex")
    E2E = ("edge", "edge")

    @property
    def input_kind(self) -> str:
        return self.value[0]

    @property
    def output_kind(self) -> str:
        return self.value[1]


class FilterMode(Enum):
    EXACT = "exact"
    INEXACT = "inexact"


@dataclass
class CullingConfig:
    """Inexact-filter knobs (reference operators.py:66-85).  On the device the
    bitmask cull is the only heuristic used; the history-table sizes are kept
    for API compatibility."""

    use_bitmask: bool = True
    team_table_size: int = 256
    local_table_size: int = 64
    bitmask_batch: int = 1024
    local_batch: int = 32
    domain_size: int | None = None


@dataclass(frozen=True)
class DeviceFunctor:
    """An entry of the closed device-functor registry (include/gfx.h GFX_FN_*)."""

    fid: int
    name: str
    value: int = 0


@dataclass
class FunctorSet:
    cond: object = None
    apply: object = None
    vertex_cond: object = None

    def device_ids(self):
        out = []
        for f in (self.cond, self.apply, self.vertex_cond):
            if f is None:
                out.append(None)
            elif isinstance(f, DeviceFunctor):
                out.append(f)
            else:
                raise TypeError(
                    "device operators take registry functors (DeviceFunctor), not Python "
                    f"callables: got {f!r}")
        return out

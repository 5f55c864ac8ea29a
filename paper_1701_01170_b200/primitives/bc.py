"""Betweenness centrality (reference primitives/bc.py:26-116) on libgfx.

Brandes forward/backward passes (csrc/gfx_bc.cu): per level a pull-gather
in ascending neighbour order, or -- where the neighbour level has fewer
slots -- a load-balanced push whose sums are exact (sigma: integer-valued
fp64; delta: 128-bit fixed point rounded once).  Values are bit-reproducible
run to run; agreement rel <= 1e-5 (north_star), bit-identical to the
reference on gathered rows of degree <= 32.
"""
from __future__ import annotations

import ctypes
from collections.abc import Iterable
from dataclasses import dataclass

import numpy as np

from .. import _native
from ..graph import as_device_graph
from ..load_balance import resolve
from ..stats import RunStats


@dataclass
class BcResult:
    bc_values: np.ndarray
    stats: RunStats


def bc_device(dg, sources, bc_values=None):
    import torch

    n = dg.num_vertices
    srcs = [int(s) for s in sources]
    for s in srcs:
        if not 0 <= s < n:
            raise ValueError(f"source {s} out of range")
    if bc_values is None:
        bc_values = torch.zeros(max(n, 1), dtype=torch.float64, device=dg.row.device)
    arr = (ctypes.c_int64 * max(len(srcs), 1))(*srcs)
    st = _native.Stats()
    _native.call("gfx_bc", dg.handle, arr, len(srcs), _native.ptr(bc_values), ctypes.byref(st))
    stats = RunStats("bc")
    stats.iterations = int(st.iterations)
    stats.edges_traversed = int(st.edges_traversed)
    stats.edges_reached = int(st.edges_reached)
    stats.device_ms = float(st.device_ms)
    return bc_values, stats


def bc(g, sources: int | Iterable[int], strategy=None, params=None,
       num_threads: int = 1) -> BcResult:
    resolve(strategy)
    n = g.num_vertices
    srcs = [sources] if isinstance(sources, (int, np.integer)) else list(sources)
    for s in srcs:
        if not 0 <= s < n:
            raise ValueError(f"source {s} out of range")
    dg = as_device_graph(g)
    values, stats = bc_device(dg, srcs)
    stats.finalize(stats.device_ms)
    return BcResult(values[:n].cpu().numpy(), stats)

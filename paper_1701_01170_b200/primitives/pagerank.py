"""PageRank entry point (reference primitives/pagerank.py:24-91) on libgfx.

Deterministic pull-gather SpMV (csrc/gfx_pagerank.cu): same update formula,
dangling mass and epsilon frontier filter as the reference; agreement within
L1 <= 1e-6 (north_star), typically to a few ulps.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from .. import _native
from ..graph import as_device_graph
from ..load_balance import resolve
from ..stats import RunStats


@dataclass
class PageRankResult:
    rank: np.ndarray
    stats: RunStats


def pagerank_device(dg, damping=0.85, epsilon=1e-6, max_iters=100, rank=None):
    import torch

    if not 0.0 < damping < 1.0:
        raise ValueError("damping must be in (0, 1)")
    if epsilon < 0:
        raise ValueError("epsilon must be >= 0")
    n = dg.num_vertices
    if rank is None:
        rank = torch.empty(max(n, 1), dtype=torch.float64, device=dg.row.device)
    st = _native.Stats()
    _native.call("gfx_pagerank", dg.handle, float(damping), float(epsilon), int(max_iters),
                 _native.ptr(rank), ctypes.byref(st))
    stats = RunStats("pagerank")
    stats.iterations = int(st.iterations)
    stats.edges_traversed = int(st.edges_traversed)
    stats.bytes_alg = int(st.bytes_alg)
    stats.device_ms = float(st.device_ms)
    return rank, stats


def pagerank(g, damping: float = 0.85, epsilon: float = 1e-6, max_iters: int = 100,
             strategy=None, params=None, num_threads: int = 1) -> PageRankResult:
    resolve(strategy)
    if not 0.0 < damping < 1.0:
        raise ValueError("damping must be in (0, 1)")
    if epsilon < 0:
        raise ValueError("epsilon must be >= 0")
    n = g.num_vertices
    if n == 0:
        return PageRankResult(np.empty(0), RunStats("pagerank").finalize(0.0))
    dg = as_device_graph(g)
    rank, stats = pagerank_device(dg, damping, epsilon, max_iters)
    stats.finalize(stats.device_ms)
    return PageRankResult(rank[:n].cpu().numpy(), stats)

"""SSSP entry point (reference primitives/sssp.py:26-121) on libgfx.

Near/far bucketed relaxation with one 64-bit atomicMin per improving edge
(distance and predecessor settle together) -- csrc/gfx_sssp.cu.  Distances
are the exact integer shortest paths, identical to the reference for any
delta (test_primitives.py:105-114); the iteration count is
order-dependent and not a parity target.
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np

from .. import _native
from .._results import labels_to_host, preds_to_host
from ..graph import as_device_graph
from ..load_balance import resolve
from ..stats import RunStats


@dataclass
class SsspResult:
    labels: np.ndarray
    preds: np.ndarray
    stats: RunStats


def default_delta_device(dg) -> int:
    """ceil(mean(w) * 32) (reference sssp.py:33-38); the integer sum is exact,
    and int/int true division rounds exactly like numpy's float64 mean."""
    import torch

    if dg.w is None or dg.num_edges == 0:
        return 32
    total = int(dg.w.to(torch.int64).sum().item())
    return int(math.ceil(total / dg.num_edges * 32))


def _check_weights(dg):
    import torch

    if dg.w is None:
        raise ValueError("sssp requires edge weights (assign_random_weights or a weighted file)")
    if dg.num_edges:
        lo = int(dg.w.min().item())
        hi = int(dg.w.max().item())
        if lo < 0:
            raise ValueError("negative edge weights are not supported")
        if hi * max(dg.num_vertices - 1, 1) >= 2**31 - 1:
            raise ValueError("distances may exceed int32 on the device path")
    del torch


def sssp_device(dg, source: int, delta=None, use_priority_queue: bool = True,
                dist=None, preds=None, rec_cap: int = 65536):
    import torch

    n = dg.num_vertices
    if not 0 <= source < n:
        raise ValueError(f"source {source} out of range")
    _check_weights(dg)
    if not use_priority_queue:
        delta = math.inf
    elif delta is None:
        delta = default_delta_device(dg)
    dev = dg.row.device
    if dist is None:
        dist = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    if preds is None:
        preds = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    recs = (_native.IterRec * rec_cap)()
    st = _native.Stats()
    _native.call("gfx_sssp", dg.handle, int(source), float(delta), _native.ptr(dist),
                 _native.ptr(preds), recs, rec_cap, ctypes.byref(st))
    stats = RunStats("sssp")
    for r in recs[: st.num_records]:
        stats.record_iteration(int(r.iteration), int(r.frontier_in), int(r.frontier_out),
                               "push", float(r.ms))
        stats.device_levels.append({"iteration": int(r.iteration), "ms": float(r.ms),
                                    "bytes_alg": int(r.bytes_alg), "work": int(r.work),
                                    "frontier_in": int(r.frontier_in),
                                    "frontier_out": int(r.frontier_out), "far": int(r.n_u)})
    stats.iterations = int(st.iterations)
    stats.edges_traversed = int(st.edges_traversed)
    stats.work_slots = int(st.work_slots)
    stats.bytes_alg = int(st.bytes_alg)
    stats.reached = int(st.reached)
    stats.edges_reached = int(st.edges_reached)
    stats.device_ms = float(st.device_ms)
    return dist, preds, stats


def sssp(g, source: int, delta=None, strategy=None, use_priority_queue: bool = True,
         params=None, num_threads: int = 1) -> SsspResult:
    """Exact shortest distances from ``source`` (reference sssp.py:41-73 contract)."""
    resolve(strategy)
    n = g.num_vertices
    if not 0 <= source < n:
        raise ValueError(f"source {source} out of range")
    if g.edge_weights is None if hasattr(g, "edge_weights") else g.w is None:
        raise ValueError("sssp requires edge weights (assign_random_weights or a weighted file)")
    w = getattr(g, "edge_weights", None)
    if w is not None and len(w) and np.min(w) < 0:
        raise ValueError("negative edge weights are not supported")
    dg = as_device_graph(g)
    if use_priority_queue and delta is None and w is not None:
        # the reference's own formula on the host weights
        delta = int(math.ceil(float(np.mean(w)) * 32)) if len(w) else 32
    dist, preds, stats = sssp_device(dg, int(source), delta, use_priority_queue)
    res = SsspResult(labels_to_host(dist[:n]), preds_to_host(preds[:n]), stats)
    stats.finalize(stats.device_ms)
    return res

"""BFS entry point (reference primitives/bfs.py:27-166), executed by libgfx.

Same signature, defaults, errors and result type as the reference.  The
level loop, claims, filters and direction switching run on the GPU
(csrc/gfx_bfs.cu); the direction decision uses the reference formula with
bit-identical floats, so ``stats.direction_trace`` equals the reference trace.
"""
from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass

import numpy as np

from .. import _native
from .._results import labels_to_host, preds_to_host
from ..direction import PULL, PUSH
from ..graph import as_device_graph
from ..load_balance import resolve
from ..operators import FilterMode
from ..stats import RunStats

_DIRS = {PUSH: _native.DIR_PUSH, PULL: _native.DIR_PULL, "auto": _native.DIR_AUTO}
_NAMES = {_native.DIR_PUSH: PUSH, _native.DIR_PULL: PULL}


@dataclass
class BfsResult:
    labels: np.ndarray
    preds: np.ndarray
    stats: RunStats


def stats_from_records(primitive, recs, st, count_trace=True) -> RunStats:
    stats = RunStats(primitive)
    for r in recs[: st.num_records]:
        if count_trace:
            stats.direction_trace.append({
                "iteration": int(r.iteration), "mode_before": _NAMES[r.mode_before],
                "n_f": int(r.frontier_in), "n_u": int(r.n_u), "m_f": float(r.m_f),
                "m_u": float(r.m_u), "decision": _NAMES[r.decision]})
        stats.record_iteration(int(r.iteration), int(r.frontier_in), int(r.frontier_out),
                               _NAMES.get(r.decision, "push"), float(r.ms))
        stats.device_levels.append({
            "iteration": int(r.iteration), "mode": _NAMES.get(r.decision, "push"),
            "ms": float(r.ms), "bytes_alg": int(r.bytes_alg), "work": int(r.work),
            "candidates": int(r.candidates), "frontier_in": int(r.frontier_in),
            "frontier_out": int(r.frontier_out), "edges": int(r.edges)})
    stats.iterations = int(st.iterations)
    stats.edges_traversed = int(st.edges_traversed)
    stats.direction_switches = int(st.direction_switches)
    stats.reached = int(st.reached)
    stats.edges_reached = int(st.edges_reached)
    stats.work_slots = int(st.work_slots)
    stats.device_ms = float(st.device_ms)
    stats.bytes_alg = int(st.bytes_alg)
    stats.init_ms = st.init_ns * 1e-6
    stats.loop_ms = st.loop_ns * 1e-6
    return stats


def default_loop() -> int:
    """Device-resident level loop unless GFX_BFS_LOOP=host (both are device
    implementations; the host loop decides directions on the CPU)."""
    import os

    return _native.LOOP_HOST if os.environ.get("GFX_BFS_LOOP") == "host" else _native.LOOP_DEVICE


def bfs_device(dg, source: int, *, direction: str = PUSH, idempotent: bool = False,
               filter_mode=FilterMode.EXACT, do_a: float = 0.001, do_b: float = 0.2,
               mu_edge_based: bool = False, loop: int | None = None,
               labels=None, preds=None, rec_cap: int = 4096):
    """Device-resident BFS: returns (labels_d int32, preds_d int32, RunStats)."""
    import torch

    n = dg.num_vertices
    if not 0 <= source < n:
        raise ValueError(f"source {source} out of range")
    if direction not in _DIRS:
        raise ValueError(f"unknown direction {direction!r}")
    if direction == "auto" and (do_a <= 0 or do_b <= 0):
        raise ValueError("do_a and do_b must be positive")
    dev = dg.row.device
    if labels is None:
        labels = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    if preds is None:
        preds = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    if loop is None:
        loop = default_loop()
    recs = (_native.IterRec * rec_cap)()
    st = _native.Stats()
    fm = _native.FILTER_EXACT if FilterMode(filter_mode) == FilterMode.EXACT else _native.FILTER_INEXACT
    _native.call("gfx_bfs", dg.handle, int(source), _DIRS[direction], int(bool(idempotent)), fm,
                 float(do_a), float(do_b), int(bool(mu_edge_based)), int(loop),
                 _native.ptr(labels), _native.ptr(preds), recs, rec_cap, ctypes.byref(st))
    return labels, preds, stats_from_records("bfs", recs, st)


def bfs_batch(dg, sources, *, direction: str = "auto", do_a: float = 0.001, do_b: float = 0.2,
              mu_edge_based: bool = False, labels=None, preds=None) -> float:
    """Run one BFS per source back to back on the device (one synchronisation);
    returns the device time in ms.  labels/preds hold the last run."""
    import torch

    n = dg.num_vertices
    srcs = [int(s) for s in sources]
    dev = dg.row.device
    if labels is None:
        labels = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    if preds is None:
        preds = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    arr = (ctypes.c_int64 * len(srcs))(*srcs)
    ms = ctypes.c_float()
    _native.call("gfx_bfs_batch", dg.handle, arr, len(srcs), _DIRS[direction], float(do_a),
                 float(do_b), int(bool(mu_edge_based)), _native.ptr(labels), _native.ptr(preds),
                 ctypes.byref(ms))
    return ms.value


def bfs(g, source: int, idempotent: bool = False, direction: str = PUSH, strategy=None,
        do_a: float = 0.001, do_b: float = 0.2, mu_edge_based: bool = False,
        filter_mode=FilterMode.EXACT, culling=None, params=None,
        num_threads: int = 1) -> BfsResult:
    """Hop distances and discovering parents from ``source`` (reference bfs.py:42-69).

    ``strategy``/``params``/``culling``/``num_threads`` are accepted for API
    compatibility; every strategy maps to the same device partition and gives
    identical results."""
    resolve(strategy)
    n = g.num_vertices
    if not 0 <= source < n:
        raise ValueError(f"source {source} out of range")
    if direction not in _DIRS:
        raise ValueError(f"unknown direction {direction!r}")
    pre0 = time.perf_counter()
    dg = as_device_graph(g)
    preprocess_ms = (time.perf_counter() - pre0) * 1000.0
    labels, preds, stats = bfs_device(dg, int(source), direction=direction,
                                      idempotent=idempotent, filter_mode=filter_mode,
                                      do_a=do_a, do_b=do_b, mu_edge_based=mu_edge_based)
    result = BfsResult(labels_to_host(labels[:n]), preds_to_host(preds[:n]), stats)
    stats.preprocess_ms = preprocess_ms
    stats.finalize(stats.device_ms)  # the device level loop (reference bfs.py:89,158)
    return result

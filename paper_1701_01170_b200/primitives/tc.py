"""Triangle counting (reference primitives/tc.py:18-86) on libgfx.

Orientation (deg[s] > deg[d] or tie and s < d) and the canonical oriented
CSR are built on the device; per-oriented-edge counts come out in that CSR
order, exactly like the reference's ``segmented_intersect`` over ``og``.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from .. import _native
from ..graph import CsrGraph, as_device_graph
from ..load_balance import resolve
from ..stats import RunStats


@dataclass
class TcResult:
    total_triangles: int
    per_edge_counts: np.ndarray
    oriented_src: np.ndarray
    oriented_dst: np.ndarray
    stats: RunStats


def tc_device(dg):
    import torch

    mo = ctypes.c_int64()
    _native.call("gfx_tc_orient", dg.handle, ctypes.byref(mo))
    m = mo.value
    dev = dg.row.device
    osrc = torch.empty(max(m, 1), dtype=torch.int32, device=dev)
    odst = torch.empty(max(m, 1), dtype=torch.int32, device=dev)
    counts = torch.empty(max(m, 1), dtype=torch.int32, device=dev)
    total = ctypes.c_int64()
    st = _native.Stats()
    _native.call("gfx_tc_count", dg.handle, _native.ptr(osrc), _native.ptr(odst),
                 _native.ptr(counts), ctypes.byref(total), ctypes.byref(st))
    stats = RunStats("tc")
    stats.iterations = 1
    stats.device_ms = float(st.device_ms)
    return int(total.value), counts[:m], osrc[:m], odst[:m], stats


def tc(g, strategy=None, small_cut: int = 64, params=None, num_threads: int = 1) -> TcResult:
    import torch

    resolve(strategy)
    if isinstance(g, CsrGraph):
        if not (g.undirected or g.is_symmetric()):
            raise ValueError("tc expects a canonical undirected graph")
        if g.num_edges and np.any(g.edge_sources() == g.column_indices):
            raise ValueError("tc expects a graph without self loops")
    dg = as_device_graph(g)
    if not dg.undirected:
        from ..graph import DeviceGraph

        dg = DeviceGraph.from_tensors(dg.row, dg.col, dg.w, undirected=True)
    total, counts, osrc, odst, stats = tc_device(dg)
    # reference stats: edges_traversed = m + sum(odeg[src] + odeg[dst])  (tc.py:74-76)
    m = counts.numel()
    odeg = torch.bincount(osrc.to(torch.int64), minlength=dg.num_vertices)
    stats.edges_traversed = dg.num_edges + int((odeg[osrc.long()] + odeg[odst.long()]).sum().item()) if m else dg.num_edges
    stats.record_iteration(1, m, total, "intersect", stats.device_ms)
    stats.finalize(stats.device_ms)
    return TcResult(total, counts.to(torch.int64).cpu().numpy(), osrc.to(torch.int64).cpu().numpy(),
                    odst.to(torch.int64).cpu().numpy(), stats)

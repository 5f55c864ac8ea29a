"""Connected components (reference primitives/cc.py:16-82) on libgfx.

Returns canonical min-id labels (every vertex labelled with the smallest id
in its component) -- the same partition as the reference, whose labels are
arbitrary representatives (compare after canonicalisation).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from .. import _native
from ..graph import CsrGraph, as_device_graph
from ..stats import RunStats


@dataclass
class CcResult:
    """``component[v]`` is the SMALLEST vertex id of v's component (canonical
    min-id labels).  The reference's labels are other representatives of the
    same partition (its hooking order decides them, cc.py:62-72); map them
    with ``label[v] = min{u : comp[u] == comp[v]}`` to compare."""

    component: np.ndarray
    num_components: int
    stats: RunStats


def cc_device(dg, comp=None):
    import torch

    n = dg.num_vertices
    if comp is None:
        comp = torch.empty(max(n, 1), dtype=torch.int32, device=dg.row.device)
    k = ctypes.c_int64()
    st = _native.Stats()
    _native.call("gfx_cc", dg.handle, _native.ptr(comp), ctypes.byref(k), ctypes.byref(st))
    stats = RunStats("cc")
    stats.iterations = int(st.iterations)
    stats.edges_traversed = int(st.edges_traversed)
    stats.bytes_alg = int(st.bytes_alg)
    stats.device_ms = float(st.device_ms)
    return comp, int(k.value), stats


def cc(g) -> CcResult:
    if isinstance(g, CsrGraph) and not (g.undirected or g.is_symmetric()):
        raise ValueError("cc expects an undirected graph")
    n = g.num_vertices
    if n == 0:
        return CcResult(np.empty(0, dtype=np.int64), 0, RunStats("cc").finalize(0.0))
    dg = as_device_graph(g)
    if not dg.undirected:
        # symmetric but not flagged: the device treats it as undirected
        from ..graph import DeviceGraph

        dg = DeviceGraph.from_tensors(dg.row, dg.col, dg.w, undirected=True)
    comp, k, stats = cc_device(dg)
    stats.finalize(stats.device_ms)
    return CcResult(comp[:n].to(dtype=__import__("torch").int64).cpu().numpy(), k, stats)

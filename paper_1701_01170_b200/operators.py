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


# ---------------------------------------------------------------------------
# the closed device-functor registry (include/gfx.h GFX_FN_*)
# ---------------------------------------------------------------------------
class functors:
    """Constructors for registry functors.  ``labels``/``preds`` are int32 CUDA
    tensors (device arrays the functor mutates with device atomics)."""

    @staticmethod
    def claim(labels, preds=None, depth: int = 1) -> DeviceFunctor:
        """compare_and_swap(labels, d, UNVISITED, depth) + preds[d] = s (bfs.py:118-121)."""
        return _bind(DeviceFunctor(1, "bfs_claim", depth), labels, preds)

    @staticmethod
    def claim_idempotent(labels, preds=None, depth: int = 1) -> DeviceFunctor:
        """labels[d] == UNVISITED then _set_depth (bfs.py:113-116, 162-166)."""
        return _bind(DeviceFunctor(2, "bfs_idemp", depth), labels, preds)

    @staticmethod
    def relax(dist, preds=None) -> DeviceFunctor:
        """atomic_min(dist, d, dist[s] + w[e]) + set_pred (sssp.py:95-103)."""
        return _bind(DeviceFunctor(3, "sssp_relax", 0), dist, preds)

    @staticmethod
    def orient() -> DeviceFunctor:
        """deg[s] > deg[d] or (deg[s] == deg[d] and s < d) (tc.py:57-59)."""
        return DeviceFunctor(4, "tc_orient", 0)

    @staticmethod
    def label_eq(labels, value: int) -> DeviceFunctor:
        return _bind(DeviceFunctor(5, "label_eq", int(value)), labels, None)

    @staticmethod
    def label_ne(labels, value: int) -> DeviceFunctor:
        return _bind(DeviceFunctor(6, "label_ne", int(value)), labels, None)

    @staticmethod
    def set_label(labels, value: int) -> DeviceFunctor:
        return _bind(DeviceFunctor(7, "set_label", int(value)), labels, None)

    @staticmethod
    def add(acc, value: int = 1) -> DeviceFunctor:
        """atomic_add(acc, items, value) on an int64 CUDA tensor (operators.py:127-128)."""
        f = DeviceFunctor(8, "add_i64", int(value))
        object.__setattr__(f, "_acc", acc)
        return f


def _bind(f: DeviceFunctor, labels, preds) -> DeviceFunctor:
    object.__setattr__(f, "_labels", labels)
    object.__setattr__(f, "_preds", preds)
    return f


def _args(f):
    from . import _native

    a = _native.FunctorArgs()
    if f is not None:
        lab = getattr(f, "_labels", None)
        prd = getattr(f, "_preds", None)
        a.labels_d = lab.data_ptr() if lab is not None else None
        a.preds_d = prd.data_ptr() if prd is not None else None
        a.value = f.value
    return a


def _pick(fs: FunctorSet | None, *slots):
    if fs is None:
        return None
    ids = dict(zip(("cond", "apply", "vertex_cond"), fs.device_ids()))
    for s in slots:
        if ids[s] is not None:
            return ids[s]
    return None


_KINDS = {AdvanceKind.V2V: 0, AdvanceKind.V2E: 1, AdvanceKind.E2V: 2, AdvanceKind.E2E: 3}


def advance(g, frontier, kind: AdvanceKind = AdvanceKind.V2V, direction: str = "push",
            strategy=None, functors: FunctorSet | None = None, data=None,
            idempotent: bool = False, plan=None, params=None, num_threads: int = 1):
    """Device push advance (reference operators.py:218-266).  The functor is
    ``functors.cond`` (or ``apply``) from the registry; it decides which
    expansion slots survive and performs the effects atomically.  Output
    order is the device emission order (a multiset equal to the reference's)."""
    import ctypes

    import torch

    from . import _native
    from .frontier import Frontier
    from .graph import as_device_graph

    if frontier.kind != kind.input_kind:
        raise ValueError(f"{kind.name} advance needs a {kind.input_kind} frontier, "
                         f"got {frontier.kind}")
    if direction == "pull":
        if kind != AdvanceKind.V2V:
            raise ValueError("pull advance is defined on vertex frontiers")
        raise NotImplementedError("pull advance: use pull_expand() with a registry functor")
    if direction != "push":
        raise ValueError(f"unknown direction {direction!r}")
    f = _pick(functors, "cond", "apply")
    dg = as_device_graph(g)
    dev = dg.row.device
    fin = frontier.device(dev)
    if len(frontier):
        ev = fin.long() if kind.input_kind == "vertex" else dg.col[fin.long()].long()
        cap = int((dg.row[ev + 1] - dg.row[ev]).sum().item()) + 1
    else:
        cap = 1
    out = torch.empty(cap, dtype=torch.int32, device=dev)
    nout, edges = ctypes.c_int64(), ctypes.c_int64()
    args = _args(f)
    _native.call("gfx_advance", dg.handle, _native.ptr(fin), len(frontier), _KINDS[kind],
                 f.fid if f else 0, ctypes.byref(args), _native.ptr(out), cap,
                 ctypes.byref(nout), ctypes.byref(edges))
    items = out[: nout.value].to(torch.int64).cpu().numpy()
    return Frontier.from_items(items, kind=kind.output_kind)


def filter_frontier(frontier, mode: FilterMode = FilterMode.EXACT, functors: FunctorSet | None = None,
                    data=None, culling: CullingConfig | None = None, g=None):
    """Device filter (reference operators.py:360-384): registry vertex_cond,
    then EXACT = sorted unique survivors (np.unique).  INEXACT returns the
    same set, which meets its 'every survivor at least once' contract."""
    import ctypes

    import torch

    from . import _native
    from .frontier import Frontier

    mode = FilterMode(mode)
    f = _pick(functors, "vertex_cond")
    items = frontier.to_array()
    if len(items) == 0:
        return Frontier.from_items(items, kind=frontier.kind)
    ctx = _native.Context.get()
    handle, dev = _filter_graph(g, ctx)
    fin = frontier.device(dev)
    domain = int(items.max()) + 1
    if culling is not None and culling.domain_size:
        domain = max(domain, int(culling.domain_size))
    out = torch.empty(len(items) + 1, dtype=torch.int32, device=dev)
    nout = ctypes.c_int64()
    args = _args(f)
    _native.call("gfx_filter", handle, _native.ptr(fin), len(items),
                 0 if mode == FilterMode.EXACT else 1, f.fid if f else 0, ctypes.byref(args),
                 domain, _native.ptr(out), ctypes.byref(nout))
    return Frontier.from_items(out[: nout.value].to(torch.int64).cpu().numpy(), kind=frontier.kind)


_EMPTY_GRAPH = {}


def _filter_graph(g, ctx):
    """filter needs no adjacency; use the caller's graph or a 1-vertex stub."""
    import torch

    from .graph import DeviceGraph, as_device_graph

    if g is not None:
        dg = as_device_graph(g)
        return dg.handle, dg.row.device
    stub = _EMPTY_GRAPH.get(ctx.device)
    if stub is None:
        dev = torch.device("cuda", ctx.device)
        stub = DeviceGraph.from_tensors(torch.zeros(2, dtype=torch.int64, device=dev),
                                        torch.zeros(0, dtype=torch.int32, device=dev))
        _EMPTY_GRAPH[ctx.device] = stub
    return stub.handle, stub.row.device


def compute(frontier, apply, data=None, g=None) -> None:
    """Apply a registry functor to every item, multiplicity included
    (reference operators.py:528-533)."""
    import ctypes

    from . import _native

    f = apply if isinstance(apply, DeviceFunctor) else None
    if f is None:
        raise TypeError("compute takes a registry functor (functors.set_label / functors.add)")
    items = frontier.to_array()
    if len(items) == 0:
        return
    ctx = _native.Context.get()
    handle, dev = _filter_graph(g, ctx)
    fin = frontier.device(dev)
    args = _args(f)
    acc = getattr(f, "_acc", None)
    _native.call("gfx_compute", handle, _native.ptr(fin), len(items), f.fid, ctypes.byref(args),
                 _native.ptr(acc))


@dataclass
class IntersectResult:
    intersections: object
    per_pair_counts: object
    total: int


def segmented_intersect(g, pairs, small_cut: int = 64, check_sorted: bool = False) -> IntersectResult:
    """Per-pair neighbour-list intersection on the device (reference
    operators.py:485-525): counts, total and the intersection elements in
    pair order (ascending within each pair)."""
    import ctypes

    import numpy as np
    import torch

    from . import _native
    from .frontier import EDGE, VERTEX, Frontier
    from .graph import as_device_graph

    if isinstance(pairs, Frontier):
        if pairs.kind != EDGE:
            raise ValueError("a single frontier argument must be an edge frontier")
        e = pairs.to_array()
        u, v = g.edge_sources()[e], g.column_indices[e]
    else:
        a, b = pairs
        u = a.to_array() if isinstance(a, Frontier) else np.asarray(a, dtype=np.int64)
        v = b.to_array() if isinstance(b, Frontier) else np.asarray(b, dtype=np.int64)
        if len(u) != len(v):
            raise ValueError("paired frontiers must have equal length")
    if check_sorted and len(u):
        rows, cols = g.row_offsets, g.column_indices
        for w in np.unique(np.concatenate([u, v])):
            if np.any(np.diff(cols[rows[w]:rows[w + 1]]) < 0):
                raise ValueError(f"neighbor list of {w} is not sorted")
    dg = as_device_graph(g)
    dev = dg.row.device
    n = len(u)
    if n == 0:
        return IntersectResult(Frontier(kind=VERTEX), np.zeros(0, dtype=np.int64), 0)
    ud = torch.from_numpy(np.ascontiguousarray(u, dtype=np.int32)).to(dev)
    vd = torch.from_numpy(np.ascontiguousarray(v, dtype=np.int32)).to(dev)
    counts = torch.empty(n, dtype=torch.int32, device=dev)
    total = ctypes.c_int64()
    _native.call("gfx_segmented_intersect", dg.handle, _native.ptr(ud), _native.ptr(vd), n,
                 _native.ptr(counts), ctypes.byref(total))
    off = torch.zeros(n + 1, dtype=torch.int64, device=dev)
    off[1:] = torch.cumsum(counts.to(torch.int64), 0)
    out = torch.empty(max(total.value, 1), dtype=torch.int32, device=dev)
    _native.call("gfx_segmented_intersect_list", dg.handle, _native.ptr(ud), _native.ptr(vd), n,
                 _native.ptr(off), _native.ptr(out))
    inter = Frontier.from_items(out[: total.value].to(torch.int64).cpu().numpy(), kind=VERTEX)
    return IntersectResult(inter, counts.to(torch.int64).cpu().numpy(), int(total.value))

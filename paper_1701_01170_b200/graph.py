"""Graph containers with the reference's host-side contract plus a device image.

Host side mirrors reference graph.py:61-246 (``CooGraph``, ``CsrGraph``,
``coo_to_csr``, ``csr_to_coo``, ``csr_to_csc``, ``assign_random_weights``):
int64 ids, ``UNVISITED = INT64_MAX``, ``NO_PRED = -1``, sorted neighbour
lists, canonical undirected build.  These are the input data formats around
the hot path; the traversal work itself never runs on the host.

Device side: ``DeviceGraph`` is the HBM image the kernels read -- int64 row
offsets, int32 column ids, int32 weights -- plus the libgfx graph handle
(which owns traversal scratch).  ``CsrGraph.device()`` uploads once and caches
the image on the graph object, the way the reference caches its reverse
adjacency (graph.py:82-85, 113-126).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _native

ID_DTYPE = np.int64
WEIGHT_DTYPE = np.int64
UNVISITED = np.iinfo(np.int64).max
NO_PRED = -1


class GraphFormatError(ValueError):
    """Malformed graph input (reference graph.py:25-32); carries a line number."""

    def __init__(self, message: str, line: int | None = None):
        super().__init__(f"line {line}: {message}" if line is not None else message)
        self.line = line


@dataclass
class CooGraph:
    num_vertices: int
    src: np.ndarray
    dst: np.ndarray
    weights: np.ndarray | None = None

    @property
    def num_edges(self) -> int:
        return int(len(self.src))

    def validate(self) -> None:
        if len(self.src) != len(self.dst):
            raise ValueError("src/dst length mismatch")
        if self.num_edges:
            lo = min(int(np.min(self.src)), int(np.min(self.dst)))
            hi = max(int(np.max(self.src)), int(np.max(self.dst)))
            if lo < 0 or hi >= self.num_vertices:
                raise ValueError("edge endpoint out of range")
        if self.weights is not None and len(self.weights) != self.num_edges:
            raise ValueError("weights length mismatch")


@dataclass
class CsrGraph:
    """CSR adjacency; neighbour lists sorted ascending (reference graph.py:61-155)."""

    num_vertices: int
    row_offsets: np.ndarray
    column_indices: np.ndarray
    edge_weights: np.ndarray | None = None
    undirected: bool = False
    _csc: tuple | None = field(default=None, repr=False, compare=False)
    _edge_sources: np.ndarray | None = field(default=None, repr=False, compare=False)
    _device: "DeviceGraph | None" = field(default=None, repr=False, compare=False)

    @property
    def num_edges(self) -> int:
        return int(len(self.column_indices))

    @property
    def degrees(self) -> np.ndarray:
        return np.diff(self.row_offsets)

    @property
    def average_degree(self) -> float:
        return self.num_edges / self.num_vertices if self.num_vertices else 0.0

    def degree(self, v: int) -> int:
        return int(self.row_offsets[v + 1] - self.row_offsets[v])

    def neighbors(self, v: int) -> np.ndarray:
        return self.column_indices[self.row_offsets[v]:self.row_offsets[v + 1]]

    def edge_sources(self) -> np.ndarray:
        if self._edge_sources is None:
            self._edge_sources = np.repeat(
                np.arange(self.num_vertices, dtype=ID_DTYPE), self.degrees)
        return self._edge_sources

    def csc(self):
        """Incoming adjacency (rows, cols, edge_ids); stable by source id."""
        if self._csc is None:
            order = np.argsort(self.column_indices, kind="stable")
            counts = np.bincount(self.column_indices, minlength=self.num_vertices)
            rows = np.zeros(self.num_vertices + 1, dtype=ID_DTYPE)
            np.cumsum(counts, out=rows[1:])
            self._csc = (rows, self.edge_sources()[order], order.astype(ID_DTYPE))
        return self._csc

    def validate(self) -> None:
        r = self.row_offsets
        if len(r) != self.num_vertices + 1 or r[0] != 0 or r[-1] != self.num_edges:
            raise ValueError("row_offsets endpoints wrong")
        if np.any(np.diff(r) < 0):
            raise ValueError("row_offsets not nondecreasing")
        if self.num_edges and (self.column_indices.min() < 0
                               or self.column_indices.max() >= self.num_vertices):
            raise ValueError("column index out of range")
        if self.edge_weights is not None and len(self.edge_weights) != self.num_edges:
            raise ValueError("edge_weights length mismatch")
        if self.undirected:
            if np.any(self.edge_sources() == self.column_indices):
                raise ValueError("undirected graph contains self loops")
            if not self.is_symmetric():
                raise ValueError("undirected graph is not symmetric")

    def is_symmetric(self) -> bool:
        s, d, n = self.edge_sources(), self.column_indices, self.num_vertices
        return bool(np.array_equal(np.sort(s * n + d), np.sort(d * n + s)))

    # -- device image ------------------------------------------------------
    def device(self, device: int | None = None) -> "DeviceGraph":
        """Upload (once) and return the HBM image of this graph."""
        dg = self._device
        if dg is not None and (device is None or dg.device == device):
            dg.refresh_weights(self.edge_weights)
            return dg
        self._device = DeviceGraph.from_host(self, device)
        return self._device


def coo_to_csr(coo: CooGraph, *, make_undirected: bool = False, dedup: bool = True) -> CsrGraph:
    """Canonical CSR: sorted rows, duplicates dropped (reference graph.py:158-203)."""
    coo.validate()
    n = coo.num_vertices
    src = np.asarray(coo.src, dtype=ID_DTYPE)
    dst = np.asarray(coo.dst, dtype=ID_DTYPE)
    w = None if coo.weights is None else np.asarray(coo.weights)
    if make_undirected:
        keep = src != dst
        src, dst = src[keep], dst[keep]
        src, dst = np.concatenate([src, dst]), np.concatenate([dst, src])
        if w is not None:
            w = np.concatenate([w[keep], w[keep]])
    order = np.lexsort((dst, src))
    src, dst = src[order], dst[order]
    if w is not None:
        w = w[order]
    if dedup and len(src):
        first = np.ones(len(src), dtype=bool)
        first[1:] = (src[1:] != src[:-1]) | (dst[1:] != dst[:-1])
        src, dst = src[first], dst[first]
        if w is not None:
            w = w[first]
    row = np.zeros(n + 1, dtype=ID_DTYPE)
    if len(src):
        np.cumsum(np.bincount(src, minlength=n), out=row[1:])
    return CsrGraph(n, row, dst, w, undirected=make_undirected)


def csr_to_coo(g: CsrGraph) -> CooGraph:
    return CooGraph(g.num_vertices, g.edge_sources().copy(), g.column_indices.copy(),
                    None if g.edge_weights is None else g.edge_weights.copy())


def csr_to_csc(g: CsrGraph) -> CsrGraph:
    rows, cols, eids = g.csc()
    return CsrGraph(g.num_vertices, rows.copy(), cols.copy(),
                    None if g.edge_weights is None else g.edge_weights[eids], g.undirected)


def assign_random_weights(g: CsrGraph, lo: int, hi: int, seed: int) -> CsrGraph:
    """Uniform integer weights in [lo, hi], equal on mirrored slots
    (reference graph.py:227-246: one draw per unique unordered pair, in
    sorted pair order, from ``default_rng(seed).integers``)."""
    if lo > hi or lo < 1:
        raise ValueError("need 1 <= lo <= hi")
    rng = np.random.default_rng(seed)
    s, d = g.edge_sources(), g.column_indices
    key = np.minimum(s, d) * g.num_vertices + np.maximum(s, d)
    uniq, inverse = np.unique(key, return_inverse=True)
    per_pair = rng.integers(lo, hi + 1, size=len(uniq), dtype=WEIGHT_DTYPE)
    return CsrGraph(g.num_vertices, g.row_offsets, g.column_indices, per_pair[inverse],
                    g.undirected)


# ---------------------------------------------------------------------------
# device image
# ---------------------------------------------------------------------------
class DeviceGraph:
    """HBM-resident CSR (int64 row, int32 col, int32 w) + the libgfx handle.

    Build it from a host ``CsrGraph`` (``from_host``) or directly from device
    tensors (``from_tensors``, used by the GPU R-MAT builder so scale-24/27
    inputs never touch the host)."""

    def __init__(self, ctx, n, m, row, col, w, undirected, rrow=None, rcol=None,
                 host: CsrGraph | None = None):
        self.ctx = ctx
        self.device = ctx.device
        self.num_vertices = int(n)
        self.num_edges = int(m)
        self.row, self.col, self.w = row, col, w
        self.rrow, self.rcol = rrow, rcol
        self.undirected = bool(undirected)
        self.host = host
        self._w_src = None if host is None else host.edge_weights
        h = ctypes.c_void_p()
        _native.call("gfx_graph_create", ctx.handle, self.num_vertices, self.num_edges,
                     _native.ptr(row), _native.ptr(col), _native.ptr(w),
                     _native.GRAPH_UNDIRECTED if undirected else 0, ctypes.byref(h))
        self.handle = h
        self._csc_dev = None
        if not undirected and rrow is not None:
            _native.call("gfx_graph_set_reverse", h, _native.ptr(rrow), _native.ptr(rcol))
        self.max_degree = int(_native.load_library().gfx_graph_max_degree(h))

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and _native._lib is not None:
            try:
                _native._lib.gfx_graph_destroy(h)
            except Exception:
                pass
            self.handle = None

    @property
    def average_degree(self) -> float:
        return self.num_edges / self.num_vertices if self.num_vertices else 0.0

    @staticmethod
    def _check_ranges(g: CsrGraph) -> None:
        if g.num_vertices >= 2**31 - 1:
            raise ValueError("graphs with >= 2^31-1 vertices are not supported (int32 ids)")

    @classmethod
    def from_host(cls, g: CsrGraph, device: int | None = None) -> "DeviceGraph":
        import torch

        cls._check_ranges(g)
        ctx = _native.Context.get(device)
        dev = torch.device("cuda", ctx.device)
        row = torch.from_numpy(np.ascontiguousarray(g.row_offsets, dtype=np.int64)).to(dev)
        col = torch.from_numpy(np.ascontiguousarray(g.column_indices, dtype=np.int32)).to(dev)
        w = cls._weights_tensor(g.edge_weights, dev)
        rrow = rcol = None
        if not g.undirected:
            rows, cols, _ = g.csc()
            rrow = torch.from_numpy(np.ascontiguousarray(rows, dtype=np.int64)).to(dev)
            rcol = torch.from_numpy(np.ascontiguousarray(cols, dtype=np.int32)).to(dev)
        torch.cuda.synchronize(dev)
        return cls(ctx, g.num_vertices, g.num_edges, row, col, w, g.undirected, rrow, rcol,
                   host=g)

    @classmethod
    def from_tensors(cls, row, col, w=None, undirected=True, rrow=None, rcol=None):
        import torch

        ctx = _native.Context.get(row.device.index)
        n = row.numel() - 1
        torch.cuda.synchronize(row.device)
        return cls(ctx, n, col.numel(), row, col, w, undirected, rrow, rcol)

    @staticmethod
    def _weights_tensor(w, dev):
        import torch

        if w is None:
            return None
        w = np.asarray(w)
        if len(w) and (w.min() < -(2**31) or w.max() >= 2**31):
            raise ValueError("edge weights must fit in int32 on the device path")
        return torch.from_numpy(np.ascontiguousarray(w, dtype=np.int32)).to(dev)

    def reload_(self, row_h, col_h) -> None:
        """Upload a new graph of the same shape into this device copy's own
        buffers (host tensors, pinned for DMA speed; asynchronous on the
        current stream) and recompute the derived graph constants
        (gfx_graph_refresh) -- no reallocation of buffers or scratch."""
        if row_h.numel() != self.row.numel() or col_h.numel() != self.col.numel():
            raise ValueError("reload_: shape differs from the resident graph")
        if not self.undirected:
            raise ValueError("reload_: directed graphs carry a reverse adjacency; build a new "
                             "DeviceGraph instead")
        self.row.copy_(row_h, non_blocking=True)
        self.col.copy_(col_h, non_blocking=True)
        self._csc_dev = None  # stale reverse edge ids (the handle's reid)
        _native.call("gfx_graph_refresh", self.handle)

    def reload_packed_(self, packed) -> None:
        """``reload_`` from a ``io.PackedCsr``: the packed row and column
        streams (about half the bytes of int64 rows + int32 columns) cross
        PCIe into device staging buffers kept on this graph, are decoded into
        ``row`` / ``col`` on the device (gfx_csr_unpack), then the graph
        constants are refreshed.  Stream-ordered on torch's current stream."""
        if packed.num_vertices != self.num_vertices or packed.num_edges != self.num_edges:
            raise ValueError("reload_packed_: shape differs from the resident graph")
        if not self.undirected:
            raise ValueError("reload_packed_: undirected graphs only")
        self.upload_packed_(packed)
        self.decode_packed_()

    def upload_packed_(self, packed, slot: int = 0) -> None:
        """Copy the packed streams into the graph's device staging buffers
        ``slot`` (0 or 1: two sets, so the next upload can overlap the decode
        of this one; asynchronous on the current stream)."""
        import torch

        stages = getattr(self, "_pack_stage", None)
        if stages is None:
            stages = self._pack_stage = [None, None]
        st = stages[slot]
        parts = packed.parts
        self._pack_upper = packed.upper
        if st is None or len(st) != len(parts) or any(d.numel() < h.numel() for d, h in zip(st, parts)):
            dev = self.row.device
            st = tuple(torch.empty(h.numel(), dtype=h.dtype, device=dev) for h in parts)
            stages[slot] = st
        for d, h in zip(st, parts):
            d[: h.numel()].copy_(h, non_blocking=True)

    def decode_packed_(self, slot: int = 0) -> None:
        """Decode the staged streams ``slot`` into row / col and refresh the graph."""
        st = self._pack_stage[slot]
        rc, rd, rb = st[:3]
        cc, cd, cb = st[-3:]
        _native.call("gfx_csr_unpack", self.ctx.handle, _native.ptr(rc), _native.ptr(rd),
                     _native.ptr(rb), self.num_vertices + 1, _native.ptr(self.row), 8, 0)
        if len(st) == 9:  # upper triangle: decode it, then rebuild the full columns
            import torch

            mu = self.num_edges // 2
            tmp = getattr(self, "_upper_tmp", None)
            if tmp is None:
                dev = self.row.device
                tmp = self._upper_tmp = (
                    torch.empty(self.num_vertices + 1, dtype=torch.int64, device=dev),
                    torch.empty(max(mu, 1), dtype=torch.int32, device=dev))
            urow, ucol = tmp
            uc, ud, ub = st[3:6]
            _native.call("gfx_csr_unpack", self.ctx.handle, _native.ptr(uc), _native.ptr(ud),
                         _native.ptr(ub), self.num_vertices + 1, _native.ptr(urow), 8, 0)
            _native.call("gfx_csr_unpack", self.ctx.handle, _native.ptr(cc), _native.ptr(cd),
                         _native.ptr(cb), mu, _native.ptr(ucol), 4, 0)
            _native.call("gfx_graph_rebuild_upper", self.handle, _native.ptr(urow),
                         _native.ptr(ucol), mu)
        else:
            _native.call("gfx_csr_unpack", self.ctx.handle, _native.ptr(cc), _native.ptr(cd),
                         _native.ptr(cb), self.num_edges, _native.ptr(self.col), 4, 0)
        self._csc_dev = None
        _native.call("gfx_graph_refresh", self.handle)

    def refresh_weights(self, w) -> None:
        """Re-upload weights if the host graph's weight array was replaced."""
        if self.host is None or w is self._w_src:
            return
        import torch

        self.w = self._weights_tensor(w, self.row.device)
        self._w_src = w
        torch.cuda.synchronize(self.row.device)
        # weights are bound at handle creation: rebuild the handle
        old = self.handle
        h = ctypes.c_void_p()
        _native.call("gfx_graph_create", self.ctx.handle, self.num_vertices, self.num_edges,
                     _native.ptr(self.row), _native.ptr(self.col), _native.ptr(self.w),
                     _native.GRAPH_UNDIRECTED if self.undirected else 0, ctypes.byref(h))
        if not self.undirected and self.rrow is not None:
            _native.call("gfx_graph_set_reverse", h, _native.ptr(self.rrow),
                         _native.ptr(self.rcol))
        self.handle = h
        self._csc_dev = None
        _native.load_library().gfx_graph_destroy(old)

    def ensure_csc(self):
        """Reverse adjacency with edge ids on the device (CsrGraph.csc,
        graph.py:113-126): (rrow int64[n+1], rcol int32[m], reid int64[m]),
        built once by a stable radix sort of the column ids and attached to
        the handle (pull operators with callable functors need reid)."""
        import torch

        if getattr(self, "_csc_dev", None) is None:
            dev = self.row.device
            rrow = torch.empty(self.num_vertices + 1, dtype=torch.int64, device=dev)
            rcol = torch.empty(max(self.num_edges, 1), dtype=torch.int32, device=dev)
            reid = torch.empty(max(self.num_edges, 1), dtype=torch.int64, device=dev)
            _native.call("gfx_graph_build_csc", self.handle, _native.ptr(rrow), _native.ptr(rcol),
                         _native.ptr(reid))
            self._csc_dev = (rrow, rcol, reid)
            if not self.undirected:
                self.rrow, self.rcol = rrow, rcol
        return self._csc_dev

    def degrees(self):
        return self.row[1:] - self.row[:-1]

    def to_host(self) -> CsrGraph:
        """Download into a host ``CsrGraph`` (int64 arrays, reference layout)."""
        row = self.row.cpu().numpy().astype(np.int64)
        col = self.col.cpu().numpy().astype(np.int64)
        w = None if self.w is None else self.w.cpu().numpy().astype(np.int64)
        g = CsrGraph(self.num_vertices, row, col, w, undirected=self.undirected)
        g._device = self
        self.host = g
        self._w_src = w
        return g


def as_device_graph(g) -> DeviceGraph:
    if isinstance(g, DeviceGraph):
        return g
    if isinstance(g, CsrGraph):
        return g.device()
    raise TypeError(f"expected CsrGraph or DeviceGraph, got {type(g).__name__}")

"""Binary CSR cache: the reference's graph wire format, readable and writable
from host numpy arrays and straight from / into HBM.

Format (reference io.py:18-19, 121-159): magic ``GFXCSR\\0``, then
``<BQQB`` = (version 1, n, m, flags: bit 0 weighted, bit 1 undirected), then
little-endian int64 ``row_offsets[n+1]``, ``column_indices[m]`` and, when
weighted, ``edge_weights[m]``.  ``save_csr_cache`` writes byte-identical
files to the reference's; ``load_csr_cache`` returns the same ``CsrGraph``.

Compact variant ("an int32-col variant for GPU
upload"): version 2 of the same header, row offsets still int64 but column
ids and weights int32 -- the device layout, so a load is a straight copy of
half the bytes.  The reference rejects version-2 files ("unsupported cache
version"), which is the intended behaviour for a format it cannot read;
``save_csr_cache(..., compact=False)`` (the default) stays byte-identical.

The device variants move the arrays between the file and HBM without a
host-side int64 -> int32 pass: the file's int64 column ids (and weights) are
streamed to the GPU in chunks through pinned staging buffers and narrowed
there, and written back the same way; the row offsets stay int64 end to
end.  They are the input format around the hot path: a
scale-24 graph built once (GPU R-MAT builder) is cached and reloaded in
seconds instead of being regenerated.

Matrix Market / edge-list text ingestion (reference io.py:22-118) is not a
hot-path data format and is not provided here.
"""
from __future__ import annotations

import ctypes
import struct
from pathlib import Path

import numpy as np

from .graph import ID_DTYPE, WEIGHT_DTYPE, CsrGraph, DeviceGraph, GraphFormatError

CACHE_MAGIC = b"GFXCSR\x00"
CACHE_VERSION = 1
COMPACT_VERSION = 2  # int32 column ids / weights
_HDR = "<BQQB"
_HDR_BYTES = struct.calcsize(_HDR)
_DATA_OFF = len(CACHE_MAGIC) + _HDR_BYTES
_CHUNK = 1 << 25  # elements per staged transfer (256 MB of int64)


def _flags(weighted: bool, undirected: bool) -> int:
    return (1 if weighted else 0) | (2 if undirected else 0)


def _header(n: int, m: int, flags: int, version: int = CACHE_VERSION) -> bytes:
    return CACHE_MAGIC + struct.pack(_HDR, version, n, m, flags)


def read_header_version(path: str | Path) -> tuple[int, int, int, int]:
    """(version, n, m, flags) of a cache file; GraphFormatError on a bad
    magic/version (reference io.py:140-146)."""
    with open(path, "rb") as fh:
        head = fh.read(_DATA_OFF)
    if not head.startswith(CACHE_MAGIC):
        raise GraphFormatError("not a CSR cache file (bad magic)")
    if len(head) < _DATA_OFF:
        raise GraphFormatError("truncated CSR cache header")
    version, n, m, flags = struct.unpack_from(_HDR, head, len(CACHE_MAGIC))
    if version not in (CACHE_VERSION, COMPACT_VERSION):
        raise GraphFormatError(f"unsupported cache version {version}")
    return int(version), int(n), int(m), int(flags)


def read_header(path: str | Path) -> tuple[int, int, int]:
    """(n, m, flags) of a cache file (either version)."""
    return read_header_version(path)[1:]


def _layout(version: int, n: int, m: int, flags: int):
    """[(name, dtype, offset, count)] of the arrays after the header."""
    el = "<i8" if version == CACHE_VERSION else "<i4"
    parts = [("row", "<i8", _DATA_OFF, n + 1)]
    off = _DATA_OFF + 8 * (n + 1)
    parts.append(("col", el, off, m))
    if flags & 1:
        parts.append(("w", el, off + np.dtype(el).itemsize * m, m))
    return parts


def _check_size(path: Path, version: int, n: int, m: int, flags: int) -> None:
    name, dt, off, count = _layout(version, n, m, flags)[-1]
    want = off + np.dtype(dt).itemsize * count
    have = path.stat().st_size
    if have < want:
        raise GraphFormatError(f"truncated CSR cache: {have} bytes, header needs {want}")


def _arrays(path: Path, version: int, n: int, m: int, flags: int) -> dict:
    return {name: np.memmap(path, dtype=dt, mode="r", offset=off, shape=(count,))
            if count else np.zeros(0, dtype=dt)
            for name, dt, off, count in _layout(version, n, m, flags)}


# ---------------------------------------------------------------------------
# host arrays (reference io.py:121-159)
# ---------------------------------------------------------------------------
def _int32_or_raise(a: np.ndarray, what: str) -> np.ndarray:
    if len(a) and (int(a.min()) < -2**31 or int(a.max()) >= 2**31):
        raise ValueError(f"compact cache: {what} do not fit int32")
    return np.ascontiguousarray(a, dtype="<i4")


def save_csr_cache(g: CsrGraph, path: str | Path, compact: bool = False) -> None:
    """Write the binary CSR cache: byte-identical to reference save_csr_cache,
    or (``compact=True``) the version-2 file with int32 columns / weights."""
    el = (lambda a, what: _int32_or_raise(np.asarray(a), what)) if compact else \
        (lambda a, what: np.ascontiguousarray(a, dtype="<i8"))
    with open(path, "wb") as fh:
        fh.write(_header(g.num_vertices, g.num_edges,
                         _flags(g.edge_weights is not None, g.undirected),
                         COMPACT_VERSION if compact else CACHE_VERSION))
        fh.write(np.ascontiguousarray(g.row_offsets, dtype="<i8").tobytes())
        fh.write(el(g.column_indices, "column ids").tobytes())
        if g.edge_weights is not None:
            fh.write(el(g.edge_weights, "weights").tobytes())


def load_csr_cache(path: str | Path) -> CsrGraph:
    """Read a cache file (either version) into a host ``CsrGraph`` in the
    reference layout (reference load_csr_cache)."""
    path = Path(path)
    version, n, m, flags = read_header_version(path)
    _check_size(path, version, n, m, flags)
    a = _arrays(path, version, n, m, flags)
    row = np.array(a["row"], dtype=ID_DTYPE)
    col = np.array(a["col"], dtype=ID_DTYPE)
    w = np.array(a["w"], dtype=WEIGHT_DTYPE) if flags & 1 else None
    return CsrGraph(num_vertices=n, row_offsets=row, column_indices=col, edge_weights=w,
                    undirected=bool(flags & 2))


def load_graph(path: str | Path, make_undirected: bool = False) -> CsrGraph:
    """Reference load_graph (io.py:162-175) for the cache format: a cache
    file loads as stored; ``make_undirected`` symmetrises a directed one."""
    g = load_csr_cache(path)
    if make_undirected and not g.undirected:
        from .graph import coo_to_csr, csr_to_coo

        g = coo_to_csr(csr_to_coo(g), make_undirected=True)
    return g


# ---------------------------------------------------------------------------
# HBM <-> file
# ---------------------------------------------------------------------------
def _stream_to_device(mm: np.ndarray, out, narrow: bool) -> None:
    """Copy file data into the device tensor `out` chunk by chunk: memmap ->
    pinned staging -> H2D (-> int64 to int32 narrowing on the GPU when
    `narrow`)."""
    import torch

    total = len(mm)
    if total == 0:
        return
    step = min(_CHUNK, total)
    sdt = torch.int64 if (narrow or out.dtype == torch.int64) else out.dtype
    stage = [torch.empty(step, dtype=sdt, pin_memory=True) for _ in range(2)]
    dev_tmp = torch.empty(step, dtype=torch.int64, device=out.device) if narrow else None
    done = [None, None]
    for k, a in enumerate(range(0, total, step)):
        b = min(a + step, total)
        buf = stage[k % 2]
        if done[k % 2] is not None:
            done[k % 2].synchronize()  # the DMA that last read this staging buffer
        buf[:b - a].numpy()[:] = mm[a:b]
        if narrow:
            dev_tmp[:b - a].copy_(buf[:b - a], non_blocking=True)
            out[a:b].copy_(dev_tmp[:b - a])
        else:
            out[a:b].copy_(buf[:b - a], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        done[k % 2] = ev
    torch.cuda.synchronize(out.device)


def load_csr_cache_device(path: str | Path, device: int | None = None) -> DeviceGraph:
    """Load a cache file straight into HBM (int64 row, int32 col / weights).
    Ids must fit int32 (the device layout); weights must fit int32."""
    import torch

    from . import _native

    path = Path(path)
    version, n, m, flags = read_header_version(path)
    _check_size(path, version, n, m, flags)
    if n >= 2**31 - 1:
        raise ValueError("graphs with >= 2^31-1 vertices are not supported (int32 ids)")
    ctx = _native.Context.get(device)
    dev = torch.device("cuda", ctx.device)
    a = _arrays(path, version, n, m, flags)
    narrow = version == CACHE_VERSION  # the compact file is already int32
    row = torch.empty(n + 1, dtype=torch.int64, device=dev)
    col = torch.empty(max(m, 1), dtype=torch.int32, device=dev)
    _stream_to_device(a["row"], row, narrow=False)
    _stream_to_device(a["col"], col, narrow=narrow)
    w = None
    if flags & 1:
        w = torch.empty(max(m, 1), dtype=torch.int32, device=dev)
        _stream_to_device(a["w"], w, narrow=narrow)
    if not flags & 2:
        raise ValueError("load_csr_cache_device: directed caches need the reverse adjacency; "
                         "load with load_csr_cache and upload via CsrGraph.device()")
    if m and (int(row[-1]) != m or int(col.min()) < 0 or int(col.max()) >= n):
        raise GraphFormatError("CSR cache arrays inconsistent with its header")
    return DeviceGraph(ctx, n, m, row, col, w, True)


def save_csr_cache_device(dg: DeviceGraph, path: str | Path, compact: bool = False) -> None:
    """Write a device graph (e.g. from the GPU R-MAT builder) as a cache file,
    read back chunk by chunk: columns / weights widened to int64 on the GPU
    (reference format) or written as they are (``compact=True``)."""
    import torch

    n, m = dg.num_vertices, dg.num_edges
    with open(path, "wb") as fh:
        fh.write(_header(n, m, _flags(dg.w is not None, dg.undirected),
                         COMPACT_VERSION if compact else CACHE_VERSION))
        parts = [(dg.row, n + 1, torch.int64, "<i8")]
        el = (torch.int32, "<i4") if compact else (torch.int64, "<i8")
        parts.append((dg.col, m) + el)
        if dg.w is not None:
            parts.append((dg.w, m) + el)
        for t, count, tdt, ndt in parts:
            for a in range(0, count, _CHUNK):
                b = min(a + _CHUNK, count)
                fh.write(t[a:b].to(tdt).cpu().numpy().astype(ndt, copy=False).tobytes())


# ---------------------------------------------------------------------------
# packed columns for PCIe-bound uploads (csrc/gfx_pack.cu)
# ---------------------------------------------------------------------------
class PackedCsr:
    """Host (pinned) image of an undirected device CSR with BOTH arrays packed
    as zigzag differences in a StreamVByte-like layout (csrc/gfx_pack.cu):
    the int64 row offsets (differences = degrees, ~1 byte per vertex) and the
    int32 column ids (~1.9 bytes per slot on R-MAT ef16 instead of 4).  Each
    packed array is (ctrl, data, boff) uint8 / uint8 / int64 pinned tensors.
    ``DeviceGraph.reload_packed_`` uploads it into a resident graph and
    decodes it on the device.

    With ``urow`` set (``pack_csr_device(dg, upper=True)``) the image holds
    only the upper triangle's columns (each undirected edge once, m/2 slots)
    plus its row offsets; the device rebuilds the full sorted CSR
    (gfx_graph_rebuild_upper: a stable radix-sort transpose), so about half
    the bytes cross PCIe."""

    def __init__(self, n, m, row, col, urow=None):
        self.num_vertices, self.num_edges = int(n), int(m)
        self.row, self.col = row, col  # (ctrl, data, boff) each
        self.urow = urow  # upper-triangle row offsets (ctrl, data, boff), or None

    @property
    def upper(self) -> bool:
        return self.urow is not None

    @property
    def parts(self):
        return self.row + (self.urow or ()) + self.col

    @property
    def nbytes(self) -> int:
        return sum(t.numel() * t.element_size() for t in self.parts)


def _pack_device(ctx, vals, elem_bytes: int):
    import torch

    from . import _native

    count = vals.numel()
    dev = vals.device
    boff = torch.empty((count + 1023) // 1024 + 1, dtype=torch.int64, device=dev)
    nbytes = ctypes.c_int64()
    _native.call("gfx_csr_pack_size", ctx.handle, _native.ptr(vals), elem_bytes, count,
                 _native.ptr(boff), ctypes.byref(nbytes))
    ctrl = torch.empty(max((count + 3) // 4, 1), dtype=torch.uint8, device=dev)
    data = torch.empty(max(nbytes.value, 1), dtype=torch.uint8, device=dev)
    _native.call("gfx_csr_pack", ctx.handle, _native.ptr(vals), elem_bytes, count,
                 _native.ptr(boff), _native.ptr(ctrl), _native.ptr(data))

    def pinned(t):
        h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        h.copy_(t)
        return h

    return tuple(pinned(t) for t in (ctrl, data, boff))


def pack_csr_device(dg: DeviceGraph, upper: bool = False) -> PackedCsr:
    """Pack a device graph's row offsets and columns on the device and
    download the packed streams into pinned host memory.  ``upper``: pack
    only the upper triangle of an undirected graph (see PackedCsr)."""
    if not upper:
        return PackedCsr(dg.num_vertices, dg.num_edges, _pack_device(dg.ctx, dg.row, 8),
                         _pack_device(dg.ctx, dg.col[: dg.num_edges], 4))
    import torch

    if not dg.undirected:
        raise ValueError("pack_csr_device(upper=True): undirected graphs only")
    n, m = dg.num_vertices, dg.num_edges
    deg = dg.row[1:] - dg.row[:-1]
    rowid = torch.repeat_interleave(torch.arange(n, device=dg.row.device), deg)
    keep = dg.col[:m].to(torch.int64) > rowid
    ucol = dg.col[:m][keep].contiguous()
    if 2 * ucol.numel() != m:
        raise ValueError("pack_csr_device(upper=True): the CSR is not symmetric without self loops")
    urow = torch.zeros(n + 1, dtype=torch.int64, device=dg.row.device)
    urow[1:] = torch.cumsum(torch.bincount(rowid[keep], minlength=n), 0)
    del rowid, keep
    return PackedCsr(n, m, _pack_device(dg.ctx, dg.row, 8), _pack_device(dg.ctx, ucol, 4),
                     urow=_pack_device(dg.ctx, urow, 8))

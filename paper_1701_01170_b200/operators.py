"""The bulk-synchronous frontier operators on the device (reference operators.py).

Two kinds of functor, one execution model (operators.py:10-15: gather the
expansion triples, evaluate ``cond``, commit ``apply`` once over the
survivors, effects visible when the call returns):

* **Registry functors** (``DeviceFunctor``, built with ``functors.*``): the
  device forms of every functor the six primitives pass (SURVEY 8(b) table,
  include/gfx.h ``GFX_FN_*``).  They run FUSED inside the load-balanced
  warp-tile expansion: no triple is ever materialised.
* **Python callables** with the reference signature ``cond(src, dst, edge,
  data)``, ``apply(src, dst, edge, data)``, ``vertex_cond(items, data)``.
  They run STAGED: libgfx kernels gather the triples in slot order into HBM
  (``gfx_gather``, the reference ``_gather``), the callable evaluates on those
  int64 CUDA tensors (so it must use torch operations and device-resident
  problem data -- e.g. ``labels[s] == depth - 1`` with ``labels`` a CUDA
  tensor), and libgfx compacts the survivors.  Nothing runs on the host.

Mutations from callables go through the batched atomic helpers below
(``atomic_min`` / ``atomic_add`` / ``compare_and_swap``), which are device
kernels.  They also accept host ndarrays, which are updated in place (the
arrays are uploaded, updated by the kernel and written back), so the
reference's helper semantics hold for both.

Frontiers returned by the operators stay in HBM (``frontier.Frontier``).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from enum import Enum

import numpy as np

from .frontier import EDGE, VERTEX, Frontier, _is_tensor


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
    """INEXACT culling heuristics (operators.py:66-85), reproduced exactly on
    the device (gfx_cull_stage): a bitmask over the id domain that drops ids an
    earlier batch already held, then direct-mapped team and local history
    tables.  Table size 0 disables a stage."""

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
    """``cond`` / ``apply`` / ``vertex_cond``: registry functors or callables
    over CUDA tensors (see the module docstring).  Any may be None."""

    cond: object = None
    apply: object = None
    vertex_cond: object = None

    def device_ids(self):
        out = []
        for f in (self.cond, self.apply, self.vertex_cond):
            if f is None or isinstance(f, DeviceFunctor):
                out.append(f)
            else:
                raise TypeError(f"expected a registry functor (DeviceFunctor), got {f!r}")
        return out

    @property
    def staged(self) -> bool:
        """True when any slot holds a Python callable (staged execution)."""
        fs = (self.cond, self.apply, self.vertex_cond)
        has_call = any(f is not None and not isinstance(f, DeviceFunctor) for f in fs)
        has_reg = any(isinstance(f, DeviceFunctor) for f in fs)
        if has_call and has_reg:
            raise TypeError("a FunctorSet mixes registry functors and Python callables; use one kind")
        return has_call


# ---------------------------------------------------------------------------
# the closed device-functor registry (include/gfx.h GFX_FN_*)
# ---------------------------------------------------------------------------
(FN_NONE, FN_BFS_CLAIM, FN_BFS_IDEMP, FN_SSSP_RELAX, FN_TC_ORIENT, FN_LABEL_EQ, FN_LABEL_NE,
 FN_SET_LABEL, FN_ADD_I64, FN_BFS_PULL, FN_BC_CLAIM, FN_BC_SIGMA, FN_BC_DELTA, FN_PR_SCATTER,
 FN_PR_MOVED, FN_CC_SAME_COMP, FN_SSSP_STAMP) = range(17)


def _fn(fid, name, value=0, **bound) -> DeviceFunctor:
    f = DeviceFunctor(fid, name, int(value))
    for k, v in bound.items():
        object.__setattr__(f, "_" + k, v)
    return f


class functors:
    """Constructors for registry functors.  Arrays are CUDA tensors: int32
    labels / preds / comp / stamps, float64 sigma / delta / rank."""

    @staticmethod
    def claim(labels, preds=None, depth: int = 1) -> DeviceFunctor:
        """BFS_CLAIM: compare_and_swap(labels, d, UNVISITED, depth) + preds[d] = s (bfs.py:118-121)."""
        return _fn(FN_BFS_CLAIM, "bfs_claim", depth, labels=labels, preds=preds)

    @staticmethod
    def claim_idempotent(labels, preds=None, depth: int = 1) -> DeviceFunctor:
        """BFS_IDEMP: labels[d] == UNVISITED then _set_depth (bfs.py:113-116, 162-166)."""
        return _fn(FN_BFS_IDEMP, "bfs_idemp", depth, labels=labels, preds=preds)

    @staticmethod
    def pull(labels, preds=None, depth: int = 1) -> DeviceFunctor:
        """BFS_PULL: cond labels[s] == depth - 1, apply _set_depth (bfs.py:142-145)."""
        return _fn(FN_BFS_PULL, "bfs_pull", depth, labels=labels, preds=preds)

    @staticmethod
    def relax(dist, preds=None) -> DeviceFunctor:
        """SSSP_RELAX: atomic_min(dist, d, dist[s] + w[e]) winners + set_pred (sssp.py:95-103)."""
        return _fn(FN_SSSP_RELAX, "sssp_relax", 0, labels=dist, preds=preds)

    @staticmethod
    def stamp_eq(stamps, stamp: int) -> DeviceFunctor:
        """SSSP_STAMP: vertex_cond stamps[v] == stamp (sssp.py:112-115)."""
        return _fn(FN_SSSP_STAMP, "sssp_stamp", stamp, labels=stamps)

    @staticmethod
    def orient() -> DeviceFunctor:
        """TC_ORIENT: deg[s] > deg[d] or (deg[s] == deg[d] and s < d) (tc.py:57-59)."""
        return DeviceFunctor(FN_TC_ORIENT, "tc_orient", 0)

    @staticmethod
    def bc_claim(labels, depth: int) -> DeviceFunctor:
        """BC_CLAIM: compare_and_swap(labels, d, UNVISITED, depth) (bc.py:80-84)."""
        return _fn(FN_BC_CLAIM, "bc_claim", depth, labels=labels)

    @staticmethod
    def bc_sigma(labels, sigma, depth: int) -> DeviceFunctor:
        """BC_SIGMA: labels[d] == depth; sigma[d] += sigma[s] (bc.py:87-92)."""
        return _fn(FN_BC_SIGMA, "bc_sigma", depth, labels=labels, f0=sigma)

    @staticmethod
    def bc_delta(labels, sigma, delta, level: int) -> DeviceFunctor:
        """BC_DELTA: labels[d] == level + 1; delta[s] += sigma[s]/sigma[d]*(1+delta[d])
        (bc.py:104-109)."""
        return _fn(FN_BC_DELTA, "bc_delta", level + 1, labels=labels, f0=sigma, f1=delta)

    @staticmethod
    def pr_scatter(rank, rank_next, damping: float) -> DeviceFunctor:
        """PR_SCATTER: rank_next[d] += damping * rank[s] / outdeg[s] (pagerank.py:71-75)."""
        return _fn(FN_PR_SCATTER, "pr_scatter", 0, f0=rank, f1=rank_next, scalar=damping)

    @staticmethod
    def pr_moved(rank, rank_next, epsilon: float) -> DeviceFunctor:
        """PR_MOVED: vertex_cond |rank_next - rank| >= epsilon (pagerank.py:81-85)."""
        return _fn(FN_PR_MOVED, "pr_moved", 0, f0=rank, f1=rank_next, scalar=epsilon)

    @staticmethod
    def cc_same_comp(comp) -> DeviceFunctor:
        """CC_SAME_COMP: edge vertex_cond comp[src(e)] != comp[col[e]] (cc.py:55-58)."""
        return _fn(FN_CC_SAME_COMP, "cc_same_comp", 0, labels=comp)

    @staticmethod
    def label_eq(labels, value: int) -> DeviceFunctor:
        return _fn(FN_LABEL_EQ, "label_eq", value, labels=labels)

    @staticmethod
    def label_ne(labels, value: int) -> DeviceFunctor:
        return _fn(FN_LABEL_NE, "label_ne", value, labels=labels)

    @staticmethod
    def set_label(labels, value: int) -> DeviceFunctor:
        return _fn(FN_SET_LABEL, "set_label", value, labels=labels)

    @staticmethod
    def add(acc, value: int = 1) -> DeviceFunctor:
        """atomic_add(acc, items, value) on an int64 CUDA tensor (operators.py:127-128)."""
        return _fn(FN_ADD_I64, "add_i64", value, acc=acc)


def _args(f):
    from . import _native

    a = _native.FunctorArgs()
    if f is not None:
        a.labels_d = _ptr_or_none(getattr(f, "_labels", None))
        a.preds_d = _ptr_or_none(getattr(f, "_preds", None))
        a.value = f.value
        a.f0_d = _ptr_or_none(getattr(f, "_f0", None))
        a.f1_d = _ptr_or_none(getattr(f, "_f1", None))
        a.scalar = float(getattr(f, "_scalar", 0.0))
    return a


def _ptr_or_none(t):
    if t is None:
        return None
    if not (_is_tensor(t) and t.is_cuda):
        raise TypeError("registry functors bind CUDA tensors")
    return t.data_ptr()


def _pick(fs: FunctorSet | None, *slots):
    if fs is None:
        return None
    ids = dict(zip(("cond", "apply", "vertex_cond"), fs.device_ids()))
    for s in slots:
        if ids[s] is not None:
            return ids[s]
    return None


_KINDS = {AdvanceKind.V2V: 0, AdvanceKind.V2E: 1, AdvanceKind.E2V: 2, AdvanceKind.E2E: 3}


# ---------------------------------------------------------------------------
# batched atomic helpers (operators.py:111-153) -- device kernels
# ---------------------------------------------------------------------------
_DTYPES = {"int32": 0, "int64": 1, "float32": 2, "float64": 3}


def _device_array(array):
    """(CUDA tensor view, write-back callable or None, dtype code)."""
    import torch

    from . import _native

    if _is_tensor(array) and array.is_cuda:
        if not array.is_contiguous():
            raise ValueError("atomic helpers need a contiguous array")
        t, back = array, None
    elif isinstance(array, np.ndarray):
        ctx = _native.Context.get()
        t = torch.from_numpy(np.ascontiguousarray(array)).to(torch.device("cuda", ctx.device))

        def back():
            array[...] = t.cpu().numpy()
    else:
        raise TypeError(f"atomic helpers take a numpy array or a CUDA tensor, got {type(array)}")
    code = _DTYPES.get(str(t.dtype).replace("torch.", ""))
    if code is None:
        raise TypeError(f"unsupported array dtype {t.dtype}")
    return t, back, code


def _idx_tensor(idx, n, dev):
    import torch

    if _is_tensor(idx):
        t = idx.to(device=dev, dtype=torch.int64).reshape(-1).contiguous()
    else:
        t = torch.from_numpy(np.ascontiguousarray(np.asarray(idx, dtype=np.int64).reshape(-1))).to(dev)
    if t.numel():
        lo, hi = int(t.min()), int(t.max())
        if lo < -n or hi >= n:
            raise IndexError(f"index out of bounds for array of size {n}")
        if lo < 0:
            t = torch.where(t < 0, t + n, t)
    return t


def _vals_tensor(values, k, dtype, dev):
    import torch

    if _is_tensor(values):
        v = values.to(device=dev, dtype=dtype).reshape(-1)
    else:
        v = torch.as_tensor(np.asarray(values), device=dev).to(dtype).reshape(-1)
    if v.numel() == 1 and k != 1:
        v = v.expand(k)
    return v.contiguous()


def _ret_mask(mask_u8, host: bool):
    m = mask_u8.bool()
    return m.cpu().numpy() if host else m


def atomic_min(array, idx, values):
    """Scatter-min ``values`` into ``array`` at ``idx``; returns the winners:
    entries strictly below the pre-call value that equal the post-call
    minimum (operators.py:111-124).  int32/int64 arrays."""
    import torch

    from . import _native

    t, back, code = _device_array(array)
    if code > 1:
        raise TypeError("atomic_min on the device supports int32/int64 arrays")
    i = _idx_tensor(idx, t.numel(), t.device)
    v = _vals_tensor(values, i.numel(), t.dtype, t.device)
    won = torch.empty(i.numel(), dtype=torch.uint8, device=t.device)
    pre = torch.empty(i.numel(), dtype=t.dtype, device=t.device)
    ctx = _native.Context.get(t.device.index)
    _native.call("gfx_atomic_min", ctx.handle, code, _native.ptr(t), _native.ptr(i), _native.ptr(v),
                 i.numel(), _native.ptr(won), _native.ptr(pre))
    if back:
        back()
    return _ret_mask(won, back is not None)


def atomic_add(array, idx, values) -> None:
    """Scatter-add with duplicates accumulated (np.add.at, operators.py:127-128)."""
    from . import _native

    t, back, code = _device_array(array)
    i = _idx_tensor(idx, t.numel(), t.device)
    scalar, vp = 0.0, None
    if np.ndim(values) == 0 and not _is_tensor(values):
        scalar = float(values)
    else:
        vp = _vals_tensor(values, i.numel(), t.dtype, t.device)
    ctx = _native.Context.get(t.device.index)
    _native.call("gfx_atomic_add", ctx.handle, code, _native.ptr(t), _native.ptr(i),
                 _native.ptr(vp), scalar, i.numel())
    if back:
        back()


def compare_and_swap(array, idx, expected, value):
    """First-claim-wins conditional store (operators.py:131-153): among the
    entries whose slot holds ``expected`` before the call, the earliest
    occurrence of each index wins and stores ``value`` (scalar or per entry)."""
    import torch

    from . import _native

    t, back, code = _device_array(array)
    if code > 1:
        raise TypeError("compare_and_swap on the device supports int32/int64 arrays")
    i = _idx_tensor(idx, t.numel(), t.device)
    vp, scalar = None, 0
    if np.ndim(value) == 0 and not _is_tensor(value):
        scalar = int(value)
    else:
        vp = _vals_tensor(value, i.numel(), t.dtype, t.device)
    won = torch.empty(i.numel(), dtype=torch.uint8, device=t.device)
    pos = torch.empty(t.numel() + 1, dtype=torch.int64, device=t.device)
    ctx = _native.Context.get(t.device.index)
    _native.call("gfx_compare_and_swap", ctx.handle, code, _native.ptr(t), _native.ptr(i),
                 i.numel(), int(expected), _native.ptr(vp), scalar, _native.ptr(won),
                 _native.ptr(pos))
    if back:
        back()
    return _ret_mask(won, back is not None)


# ---------------------------------------------------------------------------
# staged execution helpers (callable functors)
# ---------------------------------------------------------------------------
def _select(values, flags_u8, invert=False):
    """Stable compaction of an int64 CUDA tensor by a uint8 mask (gfx_select_i64)."""
    import torch

    from . import _native

    n = values.numel()
    out = torch.empty(max(n, 1), dtype=torch.int64, device=values.device)
    cnt = ctypes.c_int64()
    ctx = _native.Context.get(values.device.index)
    _native.call("gfx_select_i64", ctx.handle, _native.ptr(values), _native.ptr(flags_u8), n,
                 int(invert), _native.ptr(out), ctypes.byref(cnt))
    return out[: cnt.value]


def _mask_of(result, k, dev):
    import torch

    if result is None:
        raise TypeError("cond/vertex_cond returned None")
    m = result if _is_tensor(result) else torch.as_tensor(np.asarray(result))
    m = m.to(device=dev).reshape(-1)
    if m.numel() != k:
        raise ValueError(f"functor mask has {m.numel()} entries for {k} triples")
    return m.to(torch.uint8).contiguous()


def _gather(dg, frontier, reverse=False, need_rep=False):
    """Device _gather (operators.py:161-197): int64 CUDA (a, b, e[, rep]) in
    slot order; a = expanding vertex, b = neighbour, e = (forward) edge id."""
    import torch

    from . import _native
    from .load_balance import device_scan_offsets

    scan, total = device_scan_offsets(dg, frontier, reverse=reverse)
    dev = dg.row.device
    a = torch.empty(max(total, 1), dtype=torch.int64, device=dev)
    b = torch.empty_like(a)
    e = torch.empty_like(a)
    rep = torch.empty(max(total, 1), dtype=torch.int32, device=dev) if need_rep else None
    fin = frontier.device(dev) if len(frontier) else None
    _native.call("gfx_gather", dg.handle, _native.ptr(fin), len(frontier),
                 int(frontier.kind == EDGE), int(reverse), _native.ptr(scan), total,
                 _native.ptr(a), _native.ptr(b), _native.ptr(e), _native.ptr(rep))
    out = (a[:total], b[:total], e[:total])
    return out + ((rep[:total],) if need_rep else ())


def _staged_advance(dg, frontier, kind, fs: FunctorSet, data):
    """cond over all triples as ONE device batch, then apply once over the
    survivors in slot order (operators.py:200-215)."""
    import torch

    src, dst, edge = _gather(dg, frontier)
    total = src.numel()
    if fs.cond is not None and total:
        keep = _mask_of(fs.cond(src, dst, edge, data), total, src.device)
    else:
        keep = torch.ones(total, dtype=torch.uint8, device=src.device)
    out_src = out_dst = out_edge = None
    if fs.apply is not None:
        out_src, out_dst, out_edge = _select(src, keep), _select(dst, keep), _select(edge, keep)
        if out_src.numel():
            fs.apply(out_src, out_dst, out_edge, data)
    if kind.output_kind == VERTEX:
        ids = out_dst if out_dst is not None else _select(dst, keep)
    else:
        ids = out_edge if out_edge is not None else _select(edge, keep)
    return ids


def _out_frontier(ids64, kind: str) -> Frontier:
    if ids64.numel() and int(ids64.max()) > np.iinfo(np.int32).max:
        # edge ids beyond int32: keep the host contract (rare; m >= 2^31)
        return Frontier.from_items(ids64.cpu().numpy(), kind=kind)
    return Frontier.from_device(ids64, kind=kind)


# ---------------------------------------------------------------------------
# operators
# ---------------------------------------------------------------------------
def advance(g, frontier, kind: AdvanceKind = AdvanceKind.V2V, direction: str = "push",
            strategy=None, functors: FunctorSet | None = None, data=None,
            idempotent: bool = False, plan=None, params=None, num_threads: int = 1):
    """Expand ``frontier`` through neighbour lists (operators.py:218-266).

    Push: the cond-true images (destinations or edge slots) of every item's
    out-neighbours.  Pull: the input is an unvisited vertex frontier and the
    members with a cond-true in-neighbour are returned (``pull_expand``).
    The device schedule does not depend on ``strategy`` / ``plan`` /
    ``params`` / ``num_threads`` (load_balance.py docstring).  Registry
    functors emit in device order; callables emit in slot order."""
    import torch

    from . import _native
    from .graph import as_device_graph

    if frontier.kind != kind.input_kind:
        raise ValueError(f"{kind.name} advance needs a {kind.input_kind} frontier, "
                         f"got {frontier.kind}")
    if direction == "pull":
        if kind != AdvanceKind.V2V:
            raise ValueError("pull advance is defined on vertex frontiers")
        active, _ = pull_expand(g, frontier, functors, data, strategy=strategy, plan=plan,
                                params=params, num_threads=num_threads)
        return active
    if direction != "push":
        raise ValueError(f"unknown direction {direction!r}")
    dg = as_device_graph(g)
    dev = dg.row.device
    if len(frontier) == 0:
        return Frontier(kind=kind.output_kind)
    if functors is not None and functors.staged:
        return _out_frontier(_staged_advance(dg, frontier, kind, functors, data), kind.output_kind)
    f = _pick(functors, "cond", "apply")
    fin = frontier.device(dev)
    from .load_balance import device_scan_offsets

    _, cap = device_scan_offsets(dg, frontier)
    out = torch.empty(cap + 1, dtype=torch.int32, device=dev)
    nout, edges = ctypes.c_int64(), ctypes.c_int64()
    args = _args(f)
    _native.call("gfx_advance", dg.handle, _native.ptr(fin), len(frontier), _KINDS[kind],
                 f.fid if f else 0, ctypes.byref(args), _native.ptr(out), cap + 1,
                 ctypes.byref(nout), ctypes.byref(edges))
    return Frontier.from_device(out[: nout.value], kind=kind.output_kind)


def pull_expand(g, unvisited, functors: FunctorSet | None, data=None, strategy=None, plan=None,
                params=None, num_threads: int = 1):
    """Probe the in-neighbours of every unvisited vertex (operators.py:269-307).

    Returns ``(new_active, new_unvisited)``, a stable split of the input.
    Registry ``functors.pull`` runs one fused kernel with the sequential
    early exit; callables see every in-edge triple
    (``src`` = in-neighbour, ``dst`` = the probed vertex, ``edge`` = the
    forward slot of the in-edge) and ``apply`` commits over all cond-true
    ones.  The reverse adjacency is built on the device on first use, like
    the reference's lazy ``CsrGraph.csc()``."""
    import torch

    from . import _native
    from .graph import as_device_graph

    if unvisited.kind != VERTEX:
        raise ValueError("pull_expand takes a vertex frontier")
    dg = as_device_graph(g)
    dev = dg.row.device
    n_u = len(unvisited)
    if n_u == 0:
        return Frontier(kind=VERTEX), Frontier(kind=VERTEX)
    fin = unvisited.device(dev)
    if functors is not None and functors.staged:
        dg.ensure_csc()
        dst, src, edge, rep = _gather(dg, unvisited, reverse=True, need_rep=True)
        total = src.numel()
        hits = torch.zeros(n_u, dtype=torch.uint8, device=dev)
        if total:
            if functors.cond is not None:
                keep = _mask_of(functors.cond(src, dst, edge, data), total, dev)
            else:
                keep = torch.ones(total, dtype=torch.uint8, device=dev)
            if functors.apply is not None:
                s, d, e = _select(src, keep), _select(dst, keep), _select(edge, keep)
                if s.numel():
                    functors.apply(s, d, e, data)
            ctx = _native.Context.get(dev.index)
            _native.call("gfx_mark_items", ctx.handle, _native.ptr(keep), _native.ptr(rep), total,
                         _native.ptr(hits))
        u64 = fin.to(torch.int64)
        return (Frontier.from_device(_select(u64, hits), VERTEX),
                Frontier.from_device(_select(u64, hits, invert=True), VERTEX))
    f = _pick(functors, "cond", "apply")
    if f is None or f.fid != FN_BFS_PULL:
        raise TypeError("registry pull_expand takes functors.pull(labels, preds, depth)")
    if not dg.undirected:
        dg.ensure_csc()
    active = torch.empty(n_u, dtype=torch.int32, device=dev)
    rest = torch.empty(n_u, dtype=torch.int32, device=dev)
    na, nr, probes = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    args = _args(f)
    _native.call("gfx_pull_advance", dg.handle, _native.ptr(fin), n_u, f.fid, ctypes.byref(args),
                 _native.ptr(active), ctypes.byref(na), _native.ptr(rest), ctypes.byref(nr),
                 ctypes.byref(probes))
    return (Frontier.from_device(active[: na.value], VERTEX),
            Frontier.from_device(rest[: nr.value], VERTEX))


def _cull(ids64, cfg: CullingConfig, domain: int):
    """INEXACT culling stages in the reference order (operators.py:344-357)."""
    import torch

    from . import _native

    ctx = _native.Context.get(ids64.device.index)
    stages = []
    if cfg.use_bitmask:
        stages.append((0, cfg.bitmask_batch, 1))
    if cfg.team_table_size:
        stages.append((1, cfg.team_table_size, cfg.team_table_size))
    if cfg.local_table_size:
        stages.append((2, cfg.local_table_size, cfg.local_batch))
    for stage, tb, batch in stages:
        if ids64.numel() == 0:
            break
        keep = torch.empty(ids64.numel(), dtype=torch.uint8, device=ids64.device)
        _native.call("gfx_cull_stage", ctx.handle, _native.ptr(ids64), ids64.numel(), stage,
                     int(domain), int(tb), int(batch), _native.ptr(keep))
        ids64 = _select(ids64, keep)
    return ids64


def _unique_sorted(dg_handle, ids32, domain: int, dev, f=None):
    """EXACT filter on the device: registry vertex_cond, then the sorted
    unique survivors (np.unique) through an id bitmap (gfx_filter)."""
    import torch

    from . import _native

    n = ids32.numel()
    out = torch.empty(n + 1, dtype=torch.int32, device=dev)
    nout = ctypes.c_int64()
    args = _args(f)
    _native.call("gfx_filter", dg_handle, _native.ptr(ids32), n, 0, f.fid if f else 0,
                 ctypes.byref(args), int(domain), _native.ptr(out), ctypes.byref(nout))
    return out[: nout.value]


def filter_frontier(frontier, mode: FilterMode = FilterMode.EXACT, functors: FunctorSet | None = None,
                    data=None, culling: CullingConfig | None = None, g=None):
    """Compact a frontier by ``vertex_cond`` (operators.py:360-384).  EXACT:
    each survivor once, ascending.  INEXACT: the reference culling
    heuristics, reproduced exactly (survivors in input order, leftover
    duplicates allowed)."""
    import torch

    from . import _native

    mode = FilterMode(mode)
    if len(frontier) == 0:
        return Frontier(kind=frontier.kind)
    ctx = _native.Context.get()
    handle, dev = _filter_graph(g, ctx)
    fin = frontier.device(dev)
    n = len(frontier)
    staged = functors is not None and functors.staged
    reg = None if staged else _pick(functors, "vertex_cond")
    domain = int(fin.max().item()) + 1 if n else 1
    if culling is not None and culling.domain_size:
        domain = max(domain, int(culling.domain_size))
    if mode == FilterMode.EXACT and not staged:
        return Frontier.from_device(_unique_sorted(handle, fin, domain, dev, reg), frontier.kind)
    ids = fin.to(torch.int64)
    if staged and functors.vertex_cond is not None:
        ids = _select(ids, _mask_of(functors.vertex_cond(ids, data), n, dev))
    elif reg is not None:
        mask = torch.empty(n, dtype=torch.uint8, device=dev)
        args = _args(reg)
        _native.call("gfx_vertex_mask", handle, _native.ptr(fin), n, reg.fid, ctypes.byref(args),
                     _native.ptr(mask))
        ids = _select(ids, mask)
    if mode == FilterMode.EXACT:
        ids32 = ids.to(torch.int32)
        return Frontier.from_device(_unique_sorted(handle, ids32, domain, dev), frontier.kind)
    return Frontier.from_device(_cull(ids, culling or CullingConfig(), domain), frontier.kind)


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


def advance_filter_fused(g, frontier, kind: AdvanceKind = AdvanceKind.V2V,
                         functors: FunctorSet | None = None, data=None,
                         mode: FilterMode = FilterMode.EXACT, culling: CullingConfig | None = None,
                         idempotent: bool = False, params=None, num_threads: int = 1):
    """Traverse and cull in one pass (operators.py:392-456): as a set of items
    and applied effects equal to ``filter_frontier(advance(...))``.  Registry
    functors: ONE expansion kernel evaluates cond, the vertex_cond on the
    image and a bitmap cull (gfx_advance_fused), so each survivor is emitted
    once and no middle frontier exists.  Callables: staged gather, cond,
    apply, vertex_cond, then the filter."""
    import torch

    from . import _native
    from .graph import as_device_graph

    if frontier.kind != kind.input_kind:
        raise ValueError("frontier kind does not match advance kind")
    mode = FilterMode(mode)
    dg = as_device_graph(g)
    dev = dg.row.device
    if len(frontier) == 0:
        return Frontier(kind=kind.output_kind)
    domain = dg.num_vertices if kind.output_kind == VERTEX else dg.num_edges
    if functors is not None and functors.staged:
        adv = FunctorSet(cond=functors.cond, apply=functors.apply)
        ids = _staged_advance(dg, frontier, kind, adv, data)
        if functors.vertex_cond is not None and ids.numel():
            ids = _select(ids, _mask_of(functors.vertex_cond(ids, data), ids.numel(), dev))
        if mode == FilterMode.EXACT:
            if ids.numel() == 0:
                return Frontier(kind=kind.output_kind)
            return Frontier.from_device(_unique_sorted(dg.handle, ids.to(torch.int32), domain, dev),
                                        kind.output_kind)
        return _out_frontier(_cull(ids, culling or CullingConfig(domain_size=domain), domain),
                             kind.output_kind)
    ids = (functors.device_ids() if functors is not None else [None, None, None])
    cond = ids[0] or ids[1]
    vcond = ids[2]
    fin = frontier.device(dev)
    from .load_balance import device_scan_offsets

    _, cap = device_scan_offsets(dg, frontier)
    out = torch.empty(cap + 1, dtype=torch.int32, device=dev)
    nout, edges = ctypes.c_int64(), ctypes.c_int64()
    ca, va = _args(cond), _args(vcond)
    _native.call("gfx_advance_fused", dg.handle, _native.ptr(fin), len(frontier), _KINDS[kind],
                 cond.fid if cond else 0, ctypes.byref(ca), vcond.fid if vcond else 0,
                 ctypes.byref(va), _native.ptr(out), cap + 1, ctypes.byref(nout),
                 ctypes.byref(edges))
    return Frontier.from_device(out[: nout.value], kind=kind.output_kind)


def compute(frontier, apply, data=None, g=None) -> None:
    """Apply over every item, multiplicity included (operators.py:528-533):
    a registry functor (``functors.set_label`` / ``functors.add``) in one
    kernel, or a callable on the int64 CUDA id tensor."""
    from . import _native

    if len(frontier) == 0:
        return
    if not isinstance(apply, DeviceFunctor):
        if not callable(apply):
            raise TypeError("compute takes a registry functor or a callable")
        apply(frontier.device64(), data)
        return
    ctx = _native.Context.get()
    handle, dev = _filter_graph(g, ctx)
    fin = frontier.device(dev)
    args = _args(apply)
    acc = getattr(apply, "_acc", None)
    _native.call("gfx_compute", handle, _native.ptr(fin), len(frontier), apply.fid,
                 ctypes.byref(args), _native.ptr(acc))


@dataclass
class IntersectResult:
    intersections: object
    per_pair_counts: object
    total: int


def _pair_ids(g, pairs):
    if isinstance(pairs, Frontier):
        if pairs.kind != EDGE:
            raise ValueError("a single frontier argument must be an edge frontier")
        e = pairs.to_array()
        return np.asarray(g.edge_sources())[e], np.asarray(g.column_indices)[e]
    a, b = pairs
    u = a.to_array() if isinstance(a, Frontier) else np.asarray(a, dtype=np.int64)
    v = b.to_array() if isinstance(b, Frontier) else np.asarray(b, dtype=np.int64)
    if len(u) != len(v):
        raise ValueError("paired frontiers must have equal length")
    return u, v


def segmented_intersect(g, pairs, small_cut: int = 64, check_sorted: bool = False) -> IntersectResult:
    """Per-pair neighbour-list intersection on the device (operators.py:485-525):
    counts, total and the intersection elements in pair order (ascending
    within each pair)."""
    import torch

    from . import _native
    from .graph import as_device_graph

    u, v = _pair_ids(g, pairs)
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
    inter = Frontier.from_device(out[: total.value], kind=VERTEX)
    return IntersectResult(inter, counts.to(torch.int64).cpu().numpy(), int(total.value))

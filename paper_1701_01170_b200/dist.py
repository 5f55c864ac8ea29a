"""Partitioned multi-GPU direction-optimising BFS.

1D cyclic vertex partition: rank r of P owns v = l*P + r (local id l), so the
R-MAT hubs -- the lowest ids, generators.py:48-51 does not permute -- spread
over every rank.  Each rank keeps the rows of its owned vertices with GLOBAL
column ids plus its own labels / preds / visited bits (csrc/gfx_dist.cu).

Per level, on every rank in lockstep:
  * the global frontier size comes from an allreduce, and the direction is
    the reference decision (direction.py:52-70) on those global counts -- the
    trace therefore equals the single-GPU and the reference trace;
  * push levels expand the local frontier, claim owned destinations locally,
    and exchange (dst, src) pairs for remote ones with an all_to_all
    (de-duplicated per level on the sender); owners claim what they receive;
  * pull levels all-gather every rank's local frontier bitmap (n/8 bytes in
    total) and pull the rank's unvisited vertices against it.

The orchestration is written against two small interfaces so the same code
runs as one process per GPU over NCCL (``ProcessComm``), as P virtual ranks
inside one process (``VirtualComm``, used to test P > 1 on a single GPU), and
-- in the CPU test suite -- over gloo with a test-only engine.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

from . import _native
from .direction import PULL, PUSH, DirectionState, decide_direction, estimate_mf_mu


# ---------------------------------------------------------------------------
# communicators
# ---------------------------------------------------------------------------
class VirtualComm:
    """All P ranks' engines live in this process (single device)."""

    def __init__(self, engines):
        self.engines = engines

    def allreduce_sum(self, values):
        return int(sum(int(v) for v in values))

    def exchange_pairs(self, counts):
        P = len(self.engines)
        offs = []
        for c in counts:  # per sender: offsets of each destination bucket
            o, acc = [], 0
            for k in c:
                o.append(acc)
                acc += int(k)
            offs.append(o)
        recv_counts = []
        for j, dst in enumerate(self.engines):
            parts = [self.engines[i].send[offs[i][j]: offs[i][j] + int(counts[i][j])]
                     for i in range(P) if int(counts[i][j])]
            total = sum(int(counts[i][j]) for i in range(P))
            if parts:
                dst.recv[:total].copy_(_cat(parts))
            recv_counts.append(total)
        return recv_counts

    def allgather_frontier(self):
        g = _cat([e.front_local for e in self.engines])
        for e in self.engines:
            e.gathered.copy_(g)


class ProcessComm:
    """One engine per process, collectives over a torch.distributed group
    (NCCL on GPUs; gloo for the CPU tests)."""

    def __init__(self, engine, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.engines = [engine]
        self.group = group

    def _tensor(self, values):
        import torch

        return torch.tensor(values, dtype=torch.int64, device=self.engines[0].device)

    def allreduce_sum(self, values):
        t = self._tensor([int(sum(values))])
        self.dist.all_reduce(t, group=self.group)
        return int(t.item())

    def exchange_pairs(self, counts):
        e = self.engines[0]
        send_counts = self._tensor([int(k) for k in counts[0]])
        recv_counts = send_counts.clone()
        self.dist.all_to_all_single(recv_counts, send_counts, group=self.group)
        rc = [int(k) for k in recv_counts.tolist()]
        sc = [int(k) for k in counts[0]]
        self.dist.all_to_all_single(e.recv[: sum(rc)], e.send[: sum(sc)], output_split_sizes=rc,
                                    input_split_sizes=sc, group=self.group)
        return [sum(rc)]

    def allgather_frontier(self):
        e = self.engines[0]
        self.dist.all_gather_into_tensor(e.gathered, e.front_local, group=self.group)


def _cat(parts):
    import torch

    return parts[0] if len(parts) == 1 else torch.cat(parts)


# ---------------------------------------------------------------------------
# device engine (one rank)
# ---------------------------------------------------------------------------
def partition_graph(dg, P: int, r: int):
    """Extract rank r's rows (owned v = l*P + r) of a device graph: (lrow, lcol)."""
    import torch

    nl, ml = ctypes.c_int64(), ctypes.c_int64()
    _native.call("gfx_dist_partition_sizes", dg.handle, P, r, ctypes.byref(nl), ctypes.byref(ml))
    dev = dg.row.device
    lrow = torch.empty(nl.value + 1, dtype=torch.int64, device=dev)
    lcol = torch.empty(max(ml.value, 1), dtype=torch.int32, device=dev)
    _native.call("gfx_dist_partition", dg.handle, P, r, _native.ptr(lrow), _native.ptr(lcol))
    return lrow, lcol[: ml.value]


class DeviceEngine:
    """Rank r's libgfx engine (gfx_dbfs) plus the exchange buffers it binds."""

    def __init__(self, lrow, lcol, n: int, m: int, P: int, r: int):
        import torch

        self.P, self.r, self.n, self.m = P, r, int(n), int(m)
        self.device = lrow.device
        self.lrow, self.lcol = lrow, lcol
        self.nl = lrow.numel() - 1
        ctx = _native.Context.get(lrow.device.index)
        torch.cuda.synchronize(self.device)
        h = ctypes.c_void_p()
        _native.call("gfx_dbfs_create", ctx.handle, self.n, self.m, P, r, _native.ptr(lrow),
                     _native.ptr(lcol), self.nl, lcol.numel(), ctypes.byref(h))
        self.handle = h
        wl, wmax = ctypes.c_int64(), ctypes.c_int64()
        _native.call("gfx_dbfs_words", h, ctypes.byref(wl), ctypes.byref(wmax))
        self.wmax = wmax.value
        dev = self.device
        self.labels = torch.empty(max(self.nl, 1), dtype=torch.int32, device=dev)
        self.preds = torch.empty(max(self.nl, 1), dtype=torch.int32, device=dev)
        cap = self.n + 64
        self.send = torch.empty(cap, dtype=torch.int64, device=dev)
        self.recv = torch.empty(cap, dtype=torch.int64, device=dev)
        self.front_local = torch.zeros(self.wmax, dtype=torch.int32, device=dev)
        self.gathered = torch.zeros(P * self.wmax, dtype=torch.int32, device=dev)
        _native.call("gfx_dbfs_bind", h, _native.ptr(self.labels), _native.ptr(self.preds),
                     _native.ptr(self.send), cap, _native.ptr(self.recv), cap,
                     _native.ptr(self.front_local), _native.ptr(self.gathered))

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and _native._lib is not None:
            _native._lib.gfx_dbfs_destroy(h)
            self.handle = None

    def reset(self, source: int) -> int:
        nf = ctypes.c_int64()
        _native.call("gfx_dbfs_reset", self.handle, int(source), ctypes.byref(nf))
        return nf.value

    def push_expand(self, depth: int):
        counts = (ctypes.c_int64 * self.P)()
        local_new, edges = ctypes.c_int64(), ctypes.c_int64()
        _native.call("gfx_dbfs_push_expand", self.handle, depth, counts, ctypes.byref(local_new),
                     ctypes.byref(edges))
        return list(counts), local_new.value, edges.value

    def push_claim(self, nrecv: int, depth: int) -> int:
        nf = ctypes.c_int64()
        _native.call("gfx_dbfs_push_claim", self.handle, int(nrecv), depth, ctypes.byref(nf))
        return nf.value

    def pull_prepare(self) -> None:
        _native.call("gfx_dbfs_pull_prepare", self.handle)

    def pull(self, depth: int):
        nf, probes, cands = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        _native.call("gfx_dbfs_pull", self.handle, depth, ctypes.byref(nf), ctypes.byref(probes),
                     ctypes.byref(cands))
        return nf.value, probes.value, cands.value

    def local_labels(self):
        return self.labels[: self.nl], self.preds[: self.nl]

    def reached_degree_sum(self) -> tuple[int, int]:
        """(reached owned vertices, sum of their degrees) -- E_r share."""
        import torch

        lab = self.labels[: self.nl]
        deg = self.lrow[1:] - self.lrow[:-1]
        mask = lab != _native.UNVISITED32
        return int(mask.sum().item()), int(deg[mask].sum().item())


# ---------------------------------------------------------------------------
# the level loop
# ---------------------------------------------------------------------------
@dataclass
class DistBfsStats:
    iterations: int = 0
    direction_trace: list = field(default_factory=list)
    per_level: list = field(default_factory=list)
    edges_push: int = 0
    bytes_alg: int = 0   # SURVEY 8(d) formulas summed over ranks and levels


def bfs_partitioned(comm, n: int, m: int, source: int, direction: str = PUSH,
                    do_a: float = 0.001, do_b: float = 0.2,
                    mu_edge_based: bool = False) -> DistBfsStats:
    """Run one BFS over the engines attached to ``comm`` (all ranks call this
    collectively).  Labels/preds stay in each engine (local ids)."""
    if not 0 <= source < n:
        raise ValueError(f"source {source} out of range")
    if direction not in (PUSH, PULL, "auto"):
        raise ValueError(f"unknown direction {direction!r}")
    engines = comm.engines
    st = DistBfsStats()
    nf = comm.allreduce_sum([e.reset(source) for e in engines])
    state = DirectionState(n=n, m=m, do_a=do_a, do_b=do_b, mu_edge_based=mu_edge_based)
    depth = 0
    while nf > 0:
        depth += 1
        state.n_f = nf
        state.n_u -= nf
        m_f, m_u = estimate_mf_mu(state)
        if direction == "auto":
            mode = decide_direction(state)
        elif direction == PULL:
            mode = PULL if depth > 1 else PUSH
        else:
            mode = PUSH
        st.direction_trace.append({"iteration": depth, "mode_before": state.mode, "n_f": nf,
                                   "n_u": state.n_u, "m_f": m_f, "m_u": m_u, "decision": mode})
        if mode == PUSH:
            outs = [e.push_expand(depth) for e in engines]
            recv = comm.exchange_pairs([o[0] for o in outs])
            local = [e.push_claim(rc, depth) for e, rc in zip(engines, recv)]
            edges = comm.allreduce_sum([o[2] for o in outs])
            st.edges_push += edges
            work = 20 * nf + 4 * edges
        else:
            for e in engines:
                e.pull_prepare()
            comm.allgather_frontier()
            res = [e.pull(depth) for e in engines]
            local = [x[0] for x in res]
            work = 12 * comm.allreduce_sum([x[2] for x in res]) + \
                4 * comm.allreduce_sum([x[1] for x in res])
        nout = comm.allreduce_sum(local)
        st.bytes_alg += work + 8 * nout
        st.per_level.append({"iteration": depth, "mode": mode, "frontier_in": nf,
                             "frontier_out": nout})
        state.mode = mode
        nf = nout
    st.iterations = depth
    return st


def gather_labels(engines, n: int):
    """Reassemble global int32 labels/preds from virtual-rank engines."""
    import torch

    P = len(engines)
    dev = engines[0].labels.device
    labels = torch.empty(n, dtype=torch.int32, device=dev)
    preds = torch.empty(n, dtype=torch.int32, device=dev)
    for e in engines:
        lab, prd = e.local_labels()
        labels[e.r::P] = lab
        preds[e.r::P] = prd
    return labels, preds

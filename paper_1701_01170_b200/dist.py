"""Partitioned multi-GPU direction-optimising BFS.

1D cyclic vertex partition: rank r of P owns v = l*P + r (local id l), so the
R-MAT hubs -- the lowest ids, generators.py:48-51 does not permute -- spread
over every rank.  Each rank keeps the rows of its owned vertices with GLOBAL
column ids plus its own labels / preds / visited bits (csrc/gfx_dist.cu).

Per level, on every rank in lockstep:
  * the level counters (new frontier, slots, pull probes / candidates) are
    allreduced on the device and read by the host once, and the direction is
    the reference decision (direction.py:52-70) on those global counts -- the
    trace therefore equals the single-GPU and the reference trace;
  * push levels expand the local frontier, claim owned destinations locally,
    and exchange (dst, src) pairs for remote ones with an all_to_all
    (de-duplicated per level on the sender, pair counts exchanged first with
    an all_to_all); owners claim what they receive;
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

    def exchange_counts(self):
        sc = [[int(k) for k in e.send_counts.tolist()] for e in self.engines]
        P = len(self.engines)
        rc = [[sc[i][j] for i in range(P)] for j in range(P)]
        return sc, rc

    def exchange_pairs(self, sc, rc):
        P = len(self.engines)
        offs = []
        for c in sc:  # per sender: offsets of each destination bucket
            o, acc = [], 0
            for k in c:
                o.append(acc)
                acc += k
            offs.append(o)
        recv = []
        for j, dst in enumerate(self.engines):
            parts = [self.engines[i].send[offs[i][j]: offs[i][j] + sc[i][j]]
                     for i in range(P) if sc[i][j]]
            total = sum(rc[j])
            if parts:
                dst.recv[:total].copy_(_cat(parts))
            recv.append(total)
        return recv

    def allgather_frontier(self):
        g = _cat([e.front_local for e in self.engines])
        for e in self.engines:
            e.gathered.copy_(g)

    def allreduce_stats(self):
        loc = [[int(x) for x in e.stats[:4].tolist()] for e in self.engines]
        return loc, [sum(col) for col in zip(*loc)]


class ProcessComm:
    """One engine per process, collectives over a torch.distributed group
    (NCCL on GPUs; gloo for the CPU tests).  Collectives are enqueued on the
    stream the engine's kernels run on; the host reads device values twice
    per push level (pair counts, level counters) and once per pull level."""

    def __init__(self, engine, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.engines = [engine]
        self.group = group

    def exchange_counts(self):
        e = self.engines[0]
        P = e.send_counts.numel()
        self.dist.all_to_all_single(e.recv_counts, e.send_counts, group=self.group)
        both = [int(k) for k in e.counts.tolist()]
        return [both[:P]], [both[P:]]

    def exchange_pairs(self, sc, rc):
        e = self.engines[0]
        s, r = sc[0], rc[0]
        self.dist.all_to_all_single(e.recv[: sum(r)], e.send[: sum(s)], output_split_sizes=r,
                                    input_split_sizes=s, group=self.group)
        return [sum(r)]

    def allgather_frontier(self):
        e = self.engines[0]
        self.dist.all_gather_into_tensor(e.gathered, e.front_local, group=self.group)

    def allreduce_stats(self):
        e = self.engines[0]
        self.dist.all_reduce(e.stats[4:], group=self.group)
        vals = [int(x) for x in e.stats.tolist()]
        return [vals[:4]], vals[4:]


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
        self.counts = torch.zeros(2 * P, dtype=torch.int64, device=dev)  # send | recv
        self.send_counts, self.recv_counts = self.counts[:P], self.counts[P:]
        self.stats = torch.zeros(8, dtype=torch.int64, device=dev)  # local | to reduce
        _native.call("gfx_dbfs_bind", h, _native.ptr(self.labels), _native.ptr(self.preds),
                     _native.ptr(self.send), cap, _native.ptr(self.recv), cap,
                     _native.ptr(self.front_local), _native.ptr(self.gathered),
                     _native.ptr(self.send_counts), _native.ptr(self.stats))

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and _native._lib is not None:
            _native._lib.gfx_dbfs_destroy(h)
            self.handle = None

    def reset(self, source: int) -> int:
        nf = ctypes.c_int64()
        _native.call("gfx_dbfs_reset", self.handle, int(source), ctypes.byref(nf))
        return nf.value

    def push_expand(self, depth: int) -> None:
        _native.call("gfx_dbfs_push_expand", self.handle, depth)

    def push_claim(self, nrecv: int, depth: int) -> None:
        _native.call("gfx_dbfs_push_claim", self.handle, int(nrecv), depth)

    def pull_prepare(self) -> None:
        _native.call("gfx_dbfs_pull_prepare", self.handle)

    def pull(self, depth: int) -> None:
        _native.call("gfx_dbfs_pull", self.handle, depth)

    def commit(self, nf_local: int) -> None:
        _native.call("gfx_dbfs_commit", self.handle, int(nf_local))

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
    device_ms: float = 0.0  # native loop: CUDA-event time of the BFS on this rank


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
    local = [e.reset(source) for e in engines]
    nf = 1  # exactly one rank owns the source
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
            for e in engines:
                e.push_expand(depth)
            sc, rc = comm.exchange_counts()
            recv = comm.exchange_pairs(sc, rc)
            for e, nr in zip(engines, recv):
                e.push_claim(nr, depth)
            loc, glob = comm.allreduce_stats()
            st.edges_push += glob[1]
            work = 20 * nf + 4 * glob[1]
        else:
            for e in engines:
                e.pull_prepare()
            comm.allgather_frontier()
            for e in engines:
                e.pull(depth)
            loc, glob = comm.allreduce_stats()
            work = 12 * glob[3] + 4 * glob[2]
        for e, lv in zip(engines, loc):
            e.commit(lv[0])
        nout = glob[0]
        st.bytes_alg += work + 8 * nout
        st.per_level.append({"iteration": depth, "mode": mode, "frontier_in": nf,
                             "frontier_out": nout})
        state.mode = mode
        nf = nout
    st.iterations = depth
    return st


_DIR_CODE = {PUSH: 0, PULL: 1, "auto": 2}


def _nccl_library_path() -> str | None:
    """File of the NCCL library torch loaded into this process."""
    try:
        with open("/proc/self/maps") as fh:
            for line in fh:
                if "libnccl.so" in line:
                    return line.split()[-1]
    except OSError:
        pass
    return None


class NativeComm:
    """A NCCL communicator owned by libgfx (gfx_nccl_comm_create), for the
    native level loop.  Created collectively: rank 0 draws the unique id and
    the torch.distributed group broadcasts it.  ``None`` handle at P = 1."""

    def __init__(self, engine, group=None, single_rank_nccl: bool = False):
        import torch

        self.handle = None
        P, r = engine.P, engine.r
        if P == 1 and not single_rank_nccl:
            return
        path = _nccl_library_path()
        if path is None:
            import torch.cuda.nccl  # noqa: F401 -- maps torch's libnccl into the process

            torch.cuda.nccl.version()
            path = _nccl_library_path()
        _native.call("gfx_nccl_load", path.encode() if path else None)
        uid = (ctypes.c_uint8 * 128)()
        if r == 0:
            _native.call("gfx_nccl_unique_id", uid)
        if P == 1:  # a 1-rank communicator: every NCCL call of the loop executes
            ctx = _native.Context.get(engine.device.index)
            h = ctypes.c_void_p()
            _native.call("gfx_nccl_comm_create", ctx.handle, 1, 0, uid, ctypes.byref(h))
            self.handle = h
            return
        import torch.distributed as dist

        dev = engine.device if dist.get_backend(group) == "nccl" else torch.device("cpu")
        t = torch.tensor(list(uid), dtype=torch.uint8, device=dev)
        dist.broadcast(t, src=0, group=group)
        uid = (ctypes.c_uint8 * 128)(*t.cpu().tolist())
        ctx = _native.Context.get(engine.device.index)
        h = ctypes.c_void_p()
        _native.call("gfx_nccl_comm_create", ctx.handle, P, r, uid, ctypes.byref(h))
        self.handle = h

    def close(self):
        if self.handle is not None and _native._lib is not None:
            _native._lib.gfx_nccl_comm_destroy(self.handle)
        self.handle = None

    def __del__(self):
        self.close()


def _comm_table(collectives):
    """gfx_dbfs_comm over a Python object with exchange_counts(),
    exchange_pairs(sc, rc), allgather_frontier(), allreduce_stats_inplace()
    acting on the engine's bound tensors (returns the struct and the ctypes
    callbacks, which must stay alive for the call)."""
    def wrap(fn):
        def cb(*args):
            try:
                fn(*args)
                return 0
            except Exception:  # noqa: BLE001 -- reported through the status code
                import traceback

                traceback.print_exc()
                return 1
        return cb

    P = collectives.P
    cbs = (_native.DBFS_CB0(wrap(lambda u: collectives.exchange_counts())),
           _native.DBFS_CB_PAIRS(wrap(lambda u, sc, rc: collectives.exchange_pairs(
               [int(sc[k]) for k in range(P)], [int(rc[k]) for k in range(P)]))),
           _native.DBFS_CB0(wrap(lambda u: collectives.allgather_frontier())),
           _native.DBFS_CB0(wrap(lambda u: collectives.allreduce_stats_inplace())))
    return _native.DbfsComm(None, *cbs), cbs


def bfs_partitioned_native(engine, ncomm, n: int, m: int, source: int, direction: str = PUSH,
                           do_a: float = 0.001, do_b: float = 0.2,
                           mu_edge_based: bool = False, collectives=None) -> DistBfsStats:
    """``bfs_partitioned`` with the level loop in libgfx (gfx_dbfs_run):
    the same protocol, decisions and trace, without a Python round trip per
    collective.  ``engine`` is this rank's DeviceEngine; the collectives are
    NCCL (``ncomm``, a NativeComm; None at P = 1) or, with ``collectives``,
    a Python implementation called back from the C loop
    (gfx_dbfs_run_comm; used by the tests to run P > 1 on one GPU)."""
    if not 0 <= source < n:
        raise ValueError(f"source {source} out of range")
    if direction not in _DIR_CODE:
        raise ValueError(f"unknown direction {direction!r}")
    cap = 4096
    recs = (_native.IterRec * cap)()
    stats = _native.Stats()
    args = (int(source), _DIR_CODE[direction], float(do_a), float(do_b),
            int(bool(mu_edge_based)), recs, cap, ctypes.byref(stats))
    if collectives is not None:
        table, keep = _comm_table(collectives)
        _native.call("gfx_dbfs_run_comm", engine.handle, ctypes.byref(table), *args)
        del keep
    else:
        _native.call("gfx_dbfs_run", engine.handle, ncomm.handle if ncomm else None, *args)
    st = DistBfsStats()
    mode = {0: PUSH, 1: PULL}
    for i in range(stats.num_records):
        x = recs[i]
        st.direction_trace.append({"iteration": x.iteration, "mode_before": mode[x.mode_before],
                                   "n_f": x.frontier_in, "n_u": x.n_u, "m_f": x.m_f,
                                   "m_u": x.m_u, "decision": mode[x.decision]})
        st.per_level.append({"iteration": x.iteration, "mode": mode[x.decision],
                             "frontier_in": x.frontier_in, "frontier_out": x.frontier_out})
    st.iterations = stats.iterations
    st.edges_push = stats.edges_traversed
    st.bytes_alg = stats.bytes_alg
    st.device_ms = stats.device_ms
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


# ---------------------------------------------------------------------------
# device-resident partitioned BFS (csrc/gfx_pdbfs.cu): one cooperative launch
# per rank, exchanges through peer memory and device flags
# ---------------------------------------------------------------------------
_DIR_CODES = {PUSH: 0, PULL: 1, "auto": 2}


class VirtualRanksBfs:
    """P ranks of the device-resident partitioned BFS inside ONE launch on one
    GPU (CTA b runs rank b mod P): the complete multi-rank protocol -- sliced
    frontier copies, peer inbox stores, counter tables -- on a single device.
    ``run`` returns global int32 labels / preds (reassembled from the ranks'
    local arrays) and the per-level records."""

    def __init__(self, dg, P: int):
        import torch

        self.P, self.n, self.m = int(P), dg.num_vertices, dg.num_edges
        self.device = dg.row.device
        parts = [partition_graph(dg, self.P, r) for r in range(self.P)]
        self._keep = parts  # the ranks' CSRs (the engine borrows them)
        ctx = _native.Context.get(self.device.index)
        torch.cuda.synchronize(self.device)
        lrow = (ctypes.c_void_p * self.P)(*[_native.ptr(p[0]) for p in parts])
        lcol = (ctypes.c_void_p * self.P)(*[_native.ptr(p[1]) for p in parts])
        self.nl = [p[0].numel() - 1 for p in parts]
        nl = (ctypes.c_int64 * self.P)(*self.nl)
        ml = (ctypes.c_int64 * self.P)(*[p[1].numel() for p in parts])
        h = ctypes.c_void_p()
        _native.call("gfx_pdbfs_create_virtual", ctx.handle, self.n, self.m, self.P, lrow, lcol,
                     nl, ml, ctypes.byref(h))
        self.handle = h
        self.labels = [torch.empty(max(k, 1), dtype=torch.int32, device=self.device)
                       for k in self.nl]
        self.preds = [torch.empty_like(t) for t in self.labels]

    def close(self):
        h = getattr(self, "handle", None)
        if h:
            self.handle = None
            _native.call("gfx_pdbfs_destroy", h)

    def __del__(self):
        try:
            self.close()
        except Exception:  # interpreter shutdown: the library may be gone
            pass

    def run(self, source: int, direction: str = "auto", do_a: float = 0.001, do_b: float = 0.2,
            mu_edge_based: bool = False, rec_cap: int = 4096):
        import torch

        recs = (_native.IterRec * rec_cap)()
        st = _native.Stats()
        lab = (ctypes.c_void_p * self.P)(*[_native.ptr(t) for t in self.labels])
        prd = (ctypes.c_void_p * self.P)(*[_native.ptr(t) for t in self.preds])
        _native.call("gfx_pdbfs_run", self.handle, int(source), _DIR_CODES[direction],
                     float(do_a), float(do_b), int(bool(mu_edge_based)), lab, prd, recs, rec_cap,
                     ctypes.byref(st))
        labels = torch.empty(self.n, dtype=torch.int32, device=self.device)
        preds = torch.empty(self.n, dtype=torch.int32, device=self.device)
        for r in range(self.P):
            labels[r::self.P] = self.labels[r][: self.nl[r]]
            preds[r::self.P] = self.preds[r][: self.nl[r]]
        levels = [dict(iteration=recs[i].iteration, mode="pull" if recs[i].decision == 1 else "push",
                       mode_before=PULL if recs[i].mode_before == 1 else PUSH,
                       decision=PULL if recs[i].decision == 1 else PUSH,
                       n_f=recs[i].frontier_in, n_u=recs[i].n_u, m_f=recs[i].m_f,
                       m_u=recs[i].m_u, frontier_in=recs[i].frontier_in,
                       frontier_out=recs[i].frontier_out, edges=recs[i].edges, ms=recs[i].ms)
                  for i in range(st.num_records)]
        return labels, preds, st, levels

    def batch_ms(self, source: int, count: int, direction: str = "auto", do_a: float = 0.001,
                 do_b: float = 0.2) -> float:
        """count BFS back to back on the device; device ms for all of them."""
        ms = ctypes.c_float()
        _native.call("gfx_pdbfs_batch", self.handle, int(source), int(count),
                     _DIR_CODES[direction], float(do_a), float(do_b), 0, ctypes.byref(ms))
        return ms.value


class DeviceResidentRank:
    """This process's rank of the device-resident partitioned BFS
    (csrc/gfx_pdbfs.cu) -- one process per GPU.  Creation is collective over
    ``group`` (torch.distributed): the ranks all-gather their CUDA-IPC
    exchange handles and degree counts, then every rank maps its peers'
    frontier copies, inboxes, counter tables and barrier flags.  ``run`` is
    collective too (all ranks launch; the kernels meet at device barriers)."""

    def __init__(self, dg, P: int, r: int, group=None):
        import torch
        import torch.distributed as tdist

        self.P, self.r, self.n, self.m = int(P), int(r), dg.num_vertices, dg.num_edges
        self.device = dg.row.device
        self.lrow, self.lcol = partition_graph(dg, self.P, self.r)
        self.nl = self.lrow.numel() - 1
        ctx = _native.Context.get(self.device.index)
        torch.cuda.synchronize(self.device)
        h = ctypes.c_void_p()
        _native.call("gfx_pdbfs_create_rank", ctx.handle, self.n, self.m, self.P, self.r,
                     _native.ptr(self.lrow), _native.ptr(self.lcol), self.nl, self.lcol.numel(),
                     ctypes.byref(h))
        self.handle = h
        nnz = ctypes.c_int64()
        _native.call("gfx_pdbfs_local_nnz", h, ctypes.byref(nnz))
        mine = ctypes.create_string_buffer(320)
        _native.call("gfx_pdbfs_export", h, mine)
        if self.P > 1:
            gathered = [None] * self.P
            tdist.all_gather_object(gathered, (mine.raw, int(nnz.value)), group=group)
        else:
            gathered = [(mine.raw, int(nnz.value))]
        blob = ctypes.create_string_buffer(b"".join(g[0] for g in gathered), 320 * self.P)
        _native.call("gfx_pdbfs_import", h, blob, sum(g[1] for g in gathered))
        self.labels = torch.empty(max(self.nl, 1), dtype=torch.int32, device=self.device)
        self.preds = torch.empty_like(self.labels)

    def close(self):
        h = getattr(self, "handle", None)
        if h:
            self.handle = None
            _native.call("gfx_pdbfs_destroy", h)

    def __del__(self):
        try:
            self.close()
        except Exception:  # interpreter shutdown: the library may be gone
            pass

    def run(self, source: int, direction: str = "auto", do_a: float = 0.001, do_b: float = 0.2,
            rec_cap: int = 4096):
        """One BFS (collective); returns this rank's (labels, preds) over its
        local ids (preds are global ids), the stats and the level records."""
        recs = (_native.IterRec * rec_cap)()
        st = _native.Stats()
        lab = (ctypes.c_void_p * 1)(_native.ptr(self.labels))
        prd = (ctypes.c_void_p * 1)(_native.ptr(self.preds))
        _native.call("gfx_pdbfs_run", self.handle, int(source), _DIR_CODES[direction],
                     float(do_a), float(do_b), 0, lab, prd, recs, rec_cap, ctypes.byref(st))
        levels = [dict(iteration=recs[i].iteration, mode="pull" if recs[i].decision == 1 else "push",
                       mode_before=PULL if recs[i].mode_before == 1 else PUSH,
                       decision=PULL if recs[i].decision == 1 else PUSH,
                       n_f=recs[i].frontier_in, n_u=recs[i].n_u, m_f=recs[i].m_f,
                       m_u=recs[i].m_u, frontier_in=recs[i].frontier_in,
                       frontier_out=recs[i].frontier_out, edges=recs[i].edges, ms=recs[i].ms,
                       bytes_alg=recs[i].bytes_alg)
                  for i in range(st.num_records)]
        return self.labels[: self.nl], self.preds[: self.nl], st, levels

    def batch_ms(self, source: int, count: int, direction: str = "auto", do_a: float = 0.001,
                 do_b: float = 0.2) -> float:
        ms = ctypes.c_float()
        _native.call("gfx_pdbfs_batch", self.handle, int(source), int(count),
                     _DIR_CODES[direction], float(do_a), float(do_b), 0, ctypes.byref(ms))
        return ms.value


# ---------------------------------------------------------------------------
# partitioned near/far SSSP (reference sssp.py:41-121, near_far.py)
# ---------------------------------------------------------------------------
def partition_weights(dg, lrow, P: int, r: int):
    """Rank r's weights aligned with its local rows (gfx_dist_partition_weights)."""
    import torch

    ml = int(lrow[-1].item()) if lrow.numel() else 0
    lw = torch.empty(max(ml, 1), dtype=torch.int32, device=lrow.device)
    _native.call("gfx_dist_partition_weights", dg.handle, P, r, _native.ptr(lrow), _native.ptr(lw))
    return lw[:ml]


class SsspEngine:
    """Rank r's partitioned-SSSP engine (gfx_dsssp) and the exchange buffers
    it binds.  Messages are (d, dist << 32 | pred) -- 2 int64 words -- so the
    send / recv tensors and send_counts are in words, which is what the
    ProcessComm / VirtualComm all_to_all already moves."""

    def __init__(self, lrow, lcol, lw, n: int, P: int, r: int):
        import torch

        self.P, self.r, self.n = P, r, int(n)
        self.device = lrow.device
        self.lrow, self.lcol, self.lw = lrow, lcol, lw
        self.nl = lrow.numel() - 1
        ml = lcol.numel()
        ctx = _native.Context.get(lrow.device.index)
        torch.cuda.synchronize(self.device)
        h = ctypes.c_void_p()
        _native.call("gfx_dsssp_create", ctx.handle, self.n, P, r, _native.ptr(lrow),
                     _native.ptr(lcol), _native.ptr(lw), self.nl, ml, ctypes.byref(h))
        self.handle = h
        dev = self.device
        send_words = 2 * (min(ml, self.n) + 64)
        recv_words = 2 * (max(P - 1, 1) * self.nl + 64)
        self.send = torch.empty(send_words, dtype=torch.int64, device=dev)
        self.recv = torch.empty(recv_words, dtype=torch.int64, device=dev)
        self.counts = torch.zeros(2 * P, dtype=torch.int64, device=dev)
        self.send_counts, self.recv_counts = self.counts[:P], self.counts[P:]
        self.stats = torch.zeros(8, dtype=torch.int64, device=dev)
        _native.call("gfx_dsssp_bind", h, _native.ptr(self.send), send_words,
                     _native.ptr(self.recv), recv_words, _native.ptr(self.send_counts),
                     _native.ptr(self.stats))

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and _native._lib is not None:
            _native._lib.gfx_dsssp_destroy(h)
            self.handle = None

    def reset(self, source: int) -> int:
        k = ctypes.c_int64()
        _native.call("gfx_dsssp_reset", self.handle, int(source), ctypes.byref(k))
        return k.value

    def relax(self) -> None:
        _native.call("gfx_dsssp_relax", self.handle)

    def apply(self, nrecv_words: int) -> None:
        _native.call("gfx_dsssp_apply", self.handle, int(nrecv_words))

    def split(self, threshold: float) -> None:
        _native.call("gfx_dsssp_split", self.handle, float(threshold))

    def refar(self, threshold: float, split: bool, far_local: int) -> None:
        _native.call("gfx_dsssp_refar", self.handle, float(threshold), int(bool(split)),
                     int(far_local))

    def result(self):
        """(local int32 distances, global int32 preds) of the owned vertices."""
        import torch

        dist = torch.empty(max(self.nl, 1), dtype=torch.int32, device=self.device)
        preds = torch.empty(max(self.nl, 1), dtype=torch.int32, device=self.device)
        _native.call("gfx_dsssp_result", self.handle, _native.ptr(dist), _native.ptr(preds))
        return dist[: self.nl], preds[: self.nl]


@dataclass
class DistSsspStats:
    iterations: int = 0
    bucket_advances: int = 0
    relaxed_slots: int = 0
    messages: int = 0
    per_iteration: list = field(default_factory=list)


def sssp_partitioned(comm, n: int, source: int, delta: float | None) -> DistSsspStats:
    """One near/far SSSP over the engines attached to ``comm`` (all ranks call
    this collectively; results stay in the engines).  ``delta`` None or <= 0:
    no splitting (everything near), as the reference's never-splitting
    default on R-MAT."""
    import math

    if not 0 <= source < n:
        raise ValueError(f"source {source} out of range")
    d = float(delta) if delta is not None and delta > 0 else math.inf
    engines = comm.engines
    for e in engines:
        e.reset(source)
    st = DistSsspStats()
    threshold = d
    near_g, far_g = 1, 0
    far_loc = [0] * len(engines)
    while near_g > 0 or far_g > 0:
        if near_g == 0:
            # advance_bucket on every rank (near_far.py:63-85)
            threshold += d
            for e, fl in zip(engines, far_loc):
                e.refar(threshold, True, fl)
            loc, glob = comm.allreduce_stats()
            near_g, far_g = glob[0], glob[1]
            far_loc = [lv[1] for lv in loc]
            st.bucket_advances += 1
            continue
        st.iterations += 1
        for e in engines:
            e.relax()
        sc, rc = comm.exchange_counts()
        recv = comm.exchange_pairs(sc, rc)
        for e, nr in zip(engines, recv):
            e.apply(nr)
        for e in engines:
            e.split(threshold)
        loc, glob = comm.allreduce_stats()
        near_g, far_g = glob[0], glob[1]
        far_loc = [lv[1] for lv in loc]
        st.relaxed_slots += glob[2]
        st.messages += sum(sum(c) for c in sc) // 2
        st.per_iteration.append({"iteration": st.iterations, "near_out": near_g, "far": far_g,
                                 "slots": glob[2], "touched": glob[3]})
        # capacity guard: drop stale far entries on ranks whose pile grew past nl
        for i, e in enumerate(engines):
            if far_loc[i] > max(e.nl, 1):
                e.refar(threshold, False, far_loc[i])
                far_loc[i] = int(e.stats[1].item())
    return st


def gather_sssp(engines, n: int):
    """Global int32 distances / preds from virtual-rank SSSP engines."""
    import torch

    P = len(engines)
    dev = engines[0].device
    dist = torch.empty(n, dtype=torch.int32, device=dev)
    preds = torch.empty(n, dtype=torch.int32, device=dev)
    for e in engines:
        d, p = e.result()
        dist[e.r::P] = d
        preds[e.r::P] = p
    return dist, preds


# ---------------------------------------------------------------------------
# device-resident partitioned near/far SSSP (csrc/gfx_pdsssp.cu)
# ---------------------------------------------------------------------------
def _delta_arg(delta) -> float:
    return float(delta) if delta is not None and delta > 0 else 0.0  # 0: one bucket


class _PdSsspBase:
    def close(self):
        h = getattr(self, "handle", None)
        if h:
            self.handle = None
            _native.call("gfx_pdsssp_destroy", h)

    def __del__(self):
        try:
            self.close()
        except Exception:  # interpreter shutdown: the library may be gone
            pass

    def _run(self, source, delta, outs_d, outs_p, rec_cap):
        recs = (_native.IterRec * rec_cap)()
        st = _native.Stats()
        dd = (ctypes.c_void_p * len(outs_d))(*[_native.ptr(t) for t in outs_d])
        pp = (ctypes.c_void_p * len(outs_p))(*[_native.ptr(t) for t in outs_p])
        _native.call("gfx_pdsssp_run", self.handle, int(source), _delta_arg(delta), dd, pp, recs,
                     rec_cap, ctypes.byref(st))
        return st

    def batch_ms(self, source: int, count: int, delta=None) -> float:
        ms = ctypes.c_float()
        _native.call("gfx_pdsssp_batch", self.handle, int(source), int(count), _delta_arg(delta),
                     ctypes.byref(ms))
        return ms.value


class VirtualRanksSssp(_PdSsspBase):
    """P ranks of the device-resident partitioned SSSP in ONE launch on one GPU
    (see VirtualRanksBfs).  ``run`` returns global int32 distances / preds."""

    def __init__(self, dg, P: int):
        import torch

        self.P, self.n = int(P), dg.num_vertices
        self.device = dg.row.device
        parts = []
        for r in range(self.P):
            lrow, lcol = partition_graph(dg, self.P, r)
            parts.append((lrow, lcol, partition_weights(dg, lrow, self.P, r)))
        self._keep = parts
        ctx = _native.Context.get(self.device.index)
        torch.cuda.synchronize(self.device)
        arr = lambda k: (ctypes.c_void_p * self.P)(*[_native.ptr(p[k]) for p in parts])  # noqa: E731
        self.nl = [p[0].numel() - 1 for p in parts]
        nl = (ctypes.c_int64 * self.P)(*self.nl)
        ml = (ctypes.c_int64 * self.P)(*[p[1].numel() for p in parts])
        h = ctypes.c_void_p()
        _native.call("gfx_pdsssp_create_virtual", ctx.handle, self.n, self.P, arr(0), arr(1),
                     arr(2), nl, ml, ctypes.byref(h))
        self.handle = h
        self.dist = [torch.empty(max(k, 1), dtype=torch.int32, device=self.device) for k in self.nl]
        self.preds = [torch.empty_like(t) for t in self.dist]

    def run(self, source: int, delta=None, rec_cap: int = 1 << 14):
        import torch

        st = self._run(source, delta, self.dist, self.preds, rec_cap)
        dist = torch.empty(self.n, dtype=torch.int32, device=self.device)
        preds = torch.empty(self.n, dtype=torch.int32, device=self.device)
        for r in range(self.P):
            dist[r::self.P] = self.dist[r][: self.nl[r]]
            preds[r::self.P] = self.preds[r][: self.nl[r]]
        return dist, preds, st


class DeviceResidentSsspRank(_PdSsspBase):
    """This process's rank of the device-resident partitioned SSSP (one
    process per GPU; creation and runs are collective, see
    DeviceResidentRank)."""

    def __init__(self, dg, P: int, r: int, group=None):
        import torch
        import torch.distributed as tdist

        self.P, self.r, self.n = int(P), int(r), dg.num_vertices
        self.device = dg.row.device
        self.lrow, self.lcol = partition_graph(dg, self.P, self.r)
        self.lw = partition_weights(dg, self.lrow, self.P, self.r)
        self.nl = self.lrow.numel() - 1
        ctx = _native.Context.get(self.device.index)
        torch.cuda.synchronize(self.device)
        h = ctypes.c_void_p()
        _native.call("gfx_pdsssp_create_rank", ctx.handle, self.n, self.P, self.r,
                     _native.ptr(self.lrow), _native.ptr(self.lcol), _native.ptr(self.lw),
                     self.nl, self.lcol.numel(), ctypes.byref(h))
        self.handle = h
        mine = ctypes.create_string_buffer(256)
        _native.call("gfx_pdsssp_export", h, mine)
        if self.P > 1:
            gathered = [None] * self.P
            tdist.all_gather_object(gathered, mine.raw, group=group)
        else:
            gathered = [mine.raw]
        blob = ctypes.create_string_buffer(b"".join(gathered), 256 * self.P)
        _native.call("gfx_pdsssp_import", h, blob)
        self.dist = torch.empty(max(self.nl, 1), dtype=torch.int32, device=self.device)
        self.preds = torch.empty_like(self.dist)

    def run(self, source: int, delta=None, rec_cap: int = 1 << 14):
        """One SSSP (collective): this rank's distances / global preds over its
        local ids, and the stats."""
        st = self._run(source, delta, [self.dist], [self.preds], rec_cap)
        return self.dist[: self.nl], self.preds[: self.nl], st

"""Partitioned BFS (csrc/gfx_dist.cu + dist.py) with P virtual ranks on one
GPU: labels and the direction trace equal the reference's."""
import numpy as np
import pytest

from conftest import host_graph, rmat_golden, sha

pytestmark = pytest.mark.gpu


def _rows(trace):
    return [[t["iteration"], t["mode_before"], t["n_f"], t["n_u"], t["m_f"], t["m_u"],
             t["decision"]] for t in trace]


def _engines(dg, P):
    from paper_1701_01170_b200.dist import DeviceEngine, partition_graph

    out = []
    for r in range(P):
        lrow, lcol = partition_graph(dg, P, r)
        out.append(DeviceEngine(lrow, lcol, dg.num_vertices, dg.num_edges, P, r))
    return out


@pytest.mark.parametrize("P", [1, 2, 3, 4])
def test_kat_partitioned(kat, P):
    from paper_1701_01170_b200._results import labels_to_host
    from paper_1701_01170_b200.dist import VirtualComm, bfs_partitioned, gather_labels

    for d in kat:
        if not d["undirected"]:
            continue
        g = host_graph(d)
        dg = g.device()
        engines = _engines(dg, P)
        for direction in ("auto", "push", "pull"):
            st = bfs_partitioned(VirtualComm(engines), d["n"], d["m"], d["source"],
                                 direction=direction)
            lab, prd = gather_labels(engines, d["n"])
            assert np.array_equal(labels_to_host(lab), d["bfs"]), (d["name"], P, direction)
            if direction == "auto":
                assert _rows(st.direction_trace) == [list(x) for x in d["bfs_auto_trace"]]


@pytest.mark.parametrize("scale,P", [(16, 2), (16, 4), (20, 3), (22, 8)])
def test_rmat_partitioned(scale, P):
    from _checks import valid_bfs_preds
    from paper_1701_01170_b200._results import labels_to_host, preds_to_host
    from paper_1701_01170_b200.dist import VirtualComm, bfs_partitioned, gather_labels
    from paper_1701_01170_b200.generators import rmat_device_graph

    rec, _ = rmat_golden(scale)
    dg = rmat_device_graph(scale, 16, 0)
    engines = _engines(dg, P)
    st = bfs_partitioned(VirtualComm(engines), dg.num_vertices, dg.num_edges, 0, direction="auto")
    lab, prd = gather_labels(engines, dg.num_vertices)
    labels = labels_to_host(lab)
    assert sha(labels) == rec["bfs_sha"]
    assert _rows(st.direction_trace) == [list(x) for x in rec["bfs_auto_trace"]]
    if scale <= 16:
        row = dg.row.cpu().numpy()
        col = dg.col.cpu().numpy().astype(np.int64)
        assert valid_bfs_preds(row, col, labels, preds_to_host(prd), 0)
    st = bfs_partitioned(VirtualComm(engines), dg.num_vertices, dg.num_edges, 0, direction="push")
    lab, _ = gather_labels(engines, dg.num_vertices)
    assert sha(labels_to_host(lab)) == rec["bfs_sha"]
    assert st.edges_push == rec["bfs_edges_traversed"]


def test_kat_native_loop_single_rank(kat):
    """The native level loop (gfx_dbfs_run) at P = 1: labels and trace equal
    the reference's, for every direction."""
    from paper_1701_01170_b200._results import labels_to_host
    from paper_1701_01170_b200.dist import bfs_partitioned_native, gather_labels

    for d in kat:
        if not d["undirected"]:
            continue
        dg = host_graph(d).device()
        (eng,) = _engines(dg, 1)
        for direction in ("auto", "push", "pull"):
            st = bfs_partitioned_native(eng, None, d["n"], d["m"], d["source"],
                                        direction=direction)
            lab, _ = gather_labels([eng], d["n"])
            assert np.array_equal(labels_to_host(lab), d["bfs"]), (d["name"], direction)
            if direction == "auto":
                assert _rows(st.direction_trace) == [list(x) for x in d["bfs_auto_trace"]]


@pytest.mark.parametrize("scale", [16, 20, 22])
def test_rmat_native_loop_single_rank(scale):
    from _checks import valid_bfs_preds
    from paper_1701_01170_b200._results import labels_to_host, preds_to_host
    from paper_1701_01170_b200.dist import bfs_partitioned_native, gather_labels
    from paper_1701_01170_b200.generators import rmat_device_graph

    rec, _ = rmat_golden(scale)
    dg = rmat_device_graph(scale, 16, 0)
    (eng,) = _engines(dg, 1)
    for _ in range(2):  # engine reuse across BFS runs
        st = bfs_partitioned_native(eng, None, dg.num_vertices, dg.num_edges, 0, direction="auto")
        lab, prd = gather_labels([eng], dg.num_vertices)
        labels = labels_to_host(lab)
        assert sha(labels) == rec["bfs_sha"]
        assert _rows(st.direction_trace) == [list(x) for x in rec["bfs_auto_trace"]]
    if scale <= 16:
        row = dg.row.cpu().numpy()
        col = dg.col.cpu().numpy().astype(np.int64)
        assert valid_bfs_preds(row, col, labels, preds_to_host(prd), 0)
    st = bfs_partitioned_native(eng, None, dg.num_vertices, dg.num_edges, 0, direction="push")
    lab, _ = gather_labels([eng], dg.num_vertices)
    assert sha(labels_to_host(lab)) == rec["bfs_sha"]
    assert st.edges_push == rec["bfs_edges_traversed"]


@pytest.mark.parametrize("scale", [16, 22])
def test_native_loop_through_single_rank_nccl(scale):
    """The native level loop with a REAL 1-rank NCCL communicator: every
    collective of the protocol (count send/recv, pair send/recv, frontier
    all-gather, counter all-reduce) executes through NCCL on the device;
    labels and trace equal the reference's."""
    from paper_1701_01170_b200._results import labels_to_host
    from paper_1701_01170_b200.dist import NativeComm, bfs_partitioned_native, gather_labels
    from paper_1701_01170_b200.generators import rmat_device_graph

    rec, _ = rmat_golden(scale)
    dg = rmat_device_graph(scale, 16, 0)
    (eng,) = _engines(dg, 1)
    comm = NativeComm(eng, single_rank_nccl=True)
    assert comm.handle is not None
    for direction in ("auto", "push"):
        st = bfs_partitioned_native(eng, comm, dg.num_vertices, dg.num_edges, 0,
                                    direction=direction)
        lab, _ = gather_labels([eng], dg.num_vertices)
        assert sha(labels_to_host(lab)) == rec["bfs_sha"], direction
        if direction == "auto":
            assert _rows(st.direction_trace) == [list(x) for x in rec["bfs_auto_trace"]]
    comm.close()


class _StagedComm:
    """Test-only: ProcessComm's protocol with each collective staged through
    host memory so gloo can carry it -- two real processes share the one
    GPU a gpurun box has, each driving its own DeviceEngine."""

    def __init__(self, engine):
        import torch.distributed as dist

        self.dist = dist
        self.engines = [engine]

    def _a2a(self, out, inp, out_splits=None, in_splits=None):
        import torch

        o = torch.empty(out.shape, dtype=out.dtype)
        self.dist.all_to_all_single(o, inp.cpu(), output_split_sizes=out_splits,
                                    input_split_sizes=in_splits)
        out.copy_(o)

    def exchange_counts(self):
        e = self.engines[0]
        P = e.send_counts.numel()
        self._a2a(e.recv_counts, e.send_counts)
        both = [int(k) for k in e.counts.tolist()]
        return [both[:P]], [both[P:]]

    def exchange_pairs(self, sc, rc):
        e = self.engines[0]
        s, r = sc[0], rc[0]
        self._a2a(e.recv[: sum(r)], e.send[: sum(s)], r, s)
        return [sum(r)]

    def allgather_frontier(self):
        import torch

        e = self.engines[0]
        o = torch.empty(e.gathered.shape, dtype=e.gathered.dtype)
        self.dist.all_gather_into_tensor(o, e.front_local.cpu())
        e.gathered.copy_(o)

    def allreduce_stats(self):
        e = self.engines[0]
        t = e.stats[4:].cpu()
        self.dist.all_reduce(t)
        e.stats[4:].copy_(t)
        vals = [int(x) for x in e.stats.tolist()]
        return [vals[:4]], vals[4:]


def _two_proc_worker(rank, world, port, q):
    import os

    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1701_01170_b200._results import labels_to_host
        from paper_1701_01170_b200.dist import DeviceEngine, bfs_partitioned, partition_graph
        from paper_1701_01170_b200.generators import rmat_device_graph

        dg = rmat_device_graph(16, 16, 0)
        n, m = dg.num_vertices, dg.num_edges
        lrow, lcol = partition_graph(dg, world, rank)
        eng = DeviceEngine(lrow, lcol, n, m, world, rank)
        comm = _StagedComm(eng)
        out = {}
        for direction in ("auto", "push", "pull"):
            st = bfs_partitioned(comm, n, m, 0, direction=direction)
            lab = labels_to_host(eng.labels[: eng.nl])
            parts = [None] * world
            dist.all_gather_object(parts, lab)
            if rank == 0:
                full = np.empty(n, dtype=np.int64)
                for r, part in enumerate(parts):
                    full[r::world] = part
                out[direction] = (full, _rows(st.direction_trace), st.edges_push)
        if rank == 0:
            q.put(out)
    finally:
        dist.destroy_process_group()


def test_two_processes_share_one_gpu():
    """The partitioned BFS as two real processes (P = 2, one DeviceEngine
    each, collectives over gloo staged through host memory): labels, trace
    and push slot totals equal the reference's s16 goldens."""
    import socket

    import torch.multiprocessing as mp

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_two_proc_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    rec, _ = rmat_golden(16)
    for direction, (labels, trace, edges_push) in out.items():
        assert sha(labels) == rec["bfs_sha"], direction
    assert out["auto"][1] == [list(x) for x in rec["bfs_auto_trace"]]
    assert out["push"][2] == rec["bfs_edges_traversed"]


class _StagedCollectives:
    """Test-only collective table for the NATIVE loop (gfx_dbfs_run_comm):
    the C loop calls back into Python, which stages each collective through
    host memory over gloo."""

    def __init__(self, engine):
        self.comm = _StagedComm(engine)
        self.e = engine
        self.P = engine.P

    def exchange_counts(self):
        self.comm._a2a(self.e.recv_counts, self.e.send_counts)

    def exchange_pairs(self, sc, rc):
        self.comm._a2a(self.e.recv[: sum(rc)], self.e.send[: sum(sc)], rc, sc)

    def allgather_frontier(self):
        self.comm.allgather_frontier()

    def allreduce_stats_inplace(self):
        import torch

        t = self.e.stats[4:].cpu()
        self.comm.dist.all_reduce(t)
        self.e.stats[4:].copy_(t)
        torch.cuda.synchronize()


def _two_proc_native_worker(rank, world, port, q):
    import os

    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1701_01170_b200._results import labels_to_host
        from paper_1701_01170_b200.dist import DeviceEngine, bfs_partitioned_native, partition_graph
        from paper_1701_01170_b200.generators import rmat_device_graph

        dg = rmat_device_graph(16, 16, 0)
        n, m = dg.num_vertices, dg.num_edges
        lrow, lcol = partition_graph(dg, world, rank)
        eng = DeviceEngine(lrow, lcol, n, m, world, rank)
        coll = _StagedCollectives(eng)
        out = {}
        for direction in ("auto", "push", "pull"):
            st = bfs_partitioned_native(eng, None, n, m, 0, direction=direction, collectives=coll)
            lab = labels_to_host(eng.labels[: eng.nl])
            parts = [None] * world
            dist.all_gather_object(parts, lab)
            if rank == 0:
                full = np.empty(n, dtype=np.int64)
                for r, part in enumerate(parts):
                    full[r::world] = part
                out[direction] = (full, _rows(st.direction_trace), st.edges_push)
        if rank == 0:
            q.put(out)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_native_loop_two_processes_share_one_gpu(world):
    """The NATIVE level loop (gfx_dbfs_run_comm: the C++ protocol the NCCL
    path runs) with P = 2 / 3 real processes on one GPU, collectives called
    back into Python and staged over gloo: labels, trace and push totals
    equal the reference's s16 goldens."""
    import socket

    import torch.multiprocessing as mp

    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_two_proc_native_worker, args=(r, world, port, q))
             for r in range(world)]
    for p in procs:
        p.start()
    out = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    rec, _ = rmat_golden(16)
    for direction, (labels, trace, edges_push) in out.items():
        assert sha(labels) == rec["bfs_sha"], direction
    assert out["auto"][1] == [list(x) for x in rec["bfs_auto_trace"]]
    assert out["push"][2] == rec["bfs_edges_traversed"]

"""Partitioned BFS orchestration on CPU: virtual ranks in one process and two
real gloo processes (world_size 2), with the test-only numpy engine."""
import os
import socket

import numpy as np
import pytest
import torch

from _dist_cpu import UNV, CpuEngine
from conftest import rmat_golden
from oracle import c_oracle
from oracle import graphfx_port as port

UNV64 = np.iinfo(np.int64).max


def _global_labels(engines, n):
    P = len(engines)
    lab = np.full(n, UNV64, dtype=np.int64)
    prd = np.full(n, -1, dtype=np.int64)
    for e in engines:
        l = e.labels.copy()
        l[l == UNV] = UNV64
        lab[e.r::P] = l
        prd[e.r::P] = e.preds
    return lab, prd


def _rows(trace):
    return [[t["iteration"], t["mode_before"], t["n_f"], t["n_u"], t["m_f"], t["m_u"],
             t["decision"]] for t in trace]


@pytest.mark.parametrize("P", [1, 2, 3, 5])
def test_virtual_ranks_kat(kat, P):
    from paper_1701_01170_b200.dist import VirtualComm, bfs_partitioned

    for d in kat:
        if not d["undirected"]:
            continue
        row, col = d["row"].astype(np.int64), d["col"].astype(np.int64)
        n, m = d["n"], d["m"]
        engines = [CpuEngine(row, col, n, m, P, r) for r in range(P)]
        st = bfs_partitioned(VirtualComm(engines), n, m, d["source"], direction="auto")
        lab, prd = _global_labels(engines, n)
        assert np.array_equal(lab, d["bfs"]), (d["name"], P)
        assert _rows(st.direction_trace) == [list(x) for x in d["bfs_auto_trace"]], (d["name"], P)
        for direction in ("push", "pull"):
            bfs_partitioned(VirtualComm(engines), n, m, d["source"], direction=direction)
            lab, _ = _global_labels(engines, n)
            assert np.array_equal(lab, d["bfs"]), (d["name"], P, direction)


def test_virtual_ranks_s12_trace():
    from paper_1701_01170_b200.dist import VirtualComm, bfs_partitioned

    rec, arrays = rmat_golden(12)
    row, col = port.rmat_csr(12, 16, 0)
    want = c_oracle.bfs(row, col, 0)
    _, _, trace, _ = port.bfs(row, col, 0, direction="auto")
    for P in (2, 4):
        engines = [CpuEngine(row, col, len(row) - 1, len(col), P, r) for r in range(P)]
        st = bfs_partitioned(VirtualComm(engines), len(row) - 1, len(col), 0, direction="auto")
        lab, prd = _global_labels(engines, len(row) - 1)
        assert np.array_equal(lab, want)
        assert _rows(st.direction_trace) == _rows(trace)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port_, q):
    import torch.distributed as dist

    from paper_1701_01170_b200.dist import ProcessComm, bfs_partitioned

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        row, col = port.rmat_csr(11, 16, 0)
        n, m = len(row) - 1, len(col)
        eng = CpuEngine(row, col, n, m, world, rank)
        out = {}
        for direction in ("auto", "push", "pull"):
            st = bfs_partitioned(ProcessComm(eng), n, m, 0, direction=direction)
            lab = torch.from_numpy(eng.labels.copy())
            gathered = [torch.zeros_like(lab) for _ in range(world)] if rank == 0 else None
            # ranks own different counts: pad to a common length
            L = torch.tensor([len(lab)])
            lens = [torch.zeros_like(L) for _ in range(world)]
            dist.all_gather(lens, L)
            mx = int(max(x.item() for x in lens))
            pad = torch.full((mx,), -7, dtype=torch.int64)
            pad[: len(lab)] = lab
            allp = [torch.zeros_like(pad) for _ in range(world)]
            dist.all_gather(allp, pad)
            if rank == 0:
                g = np.full(n, -1, dtype=np.int64)
                for r in range(world):
                    g[r::world] = allp[r].numpy()[: int(lens[r].item())]
                g[g == UNV] = UNV64
                out[direction] = (g, _rows(st.direction_trace))
        if rank == 0:
            q.put(out)
    finally:
        dist.destroy_process_group()


def test_gloo_two_processes():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port_ = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port_, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    row, col = port.rmat_csr(11, 16, 0)
    want = c_oracle.bfs(row, col, 0)
    _, _, trace, _ = port.bfs(row, col, 0, direction="auto")
    for direction, (labels, tr) in out.items():
        assert np.array_equal(labels, want), direction
    assert out["auto"][1] == _rows(trace)


def _sssp_worker(rank, world, port_, q):
    import torch.distributed as dist

    from _dist_cpu import CpuSsspEngine
    from paper_1701_01170_b200.dist import ProcessComm, sssp_partitioned

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port_))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        row, col = port.rmat_csr(10, 16, 0)
        w = port.assign_random_weights(row, col, 1, 64, 0)
        n = len(row) - 1
        eng = CpuSsspEngine(row, col, w, n, world, rank)
        out = {}
        for delta in (None, 8, 32):
            st = sssp_partitioned(ProcessComm(eng), n, 0, delta)
            lab = torch.from_numpy(eng.dist.copy())
            L = torch.tensor([len(lab)])
            lens = [torch.zeros_like(L) for _ in range(world)]
            dist.all_gather(lens, L)
            mx = int(max(x.item() for x in lens))
            pad = torch.full((mx,), -7, dtype=torch.int64)
            pad[: len(lab)] = lab
            allp = [torch.zeros_like(pad) for _ in range(world)]
            dist.all_gather(allp, pad)
            if rank == 0:
                g = np.full(n, -1, dtype=np.int64)
                for r in range(world):
                    g[r::world] = allp[r].numpy()[: int(lens[r].item())]
                out[delta] = (g, st.iterations, st.bucket_advances)
        if rank == 0:
            q.put(out)
    finally:
        dist.destroy_process_group()


def test_gloo_two_processes_sssp():
    """Partitioned near/far SSSP orchestration (dist.sssp_partitioned) across
    two real gloo processes: distances equal Dijkstra (C oracle) for several
    deltas; small deltas advance the bucket."""
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port_ = _free_port()
    procs = [ctx.Process(target=_sssp_worker, args=(r, 2, port_, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    row, col = port.rmat_csr(10, 16, 0)
    w = port.assign_random_weights(row, col, 1, 64, 0)
    want = c_oracle.dijkstra(row, col, w, 0)
    for delta, (dist_, iters, adv) in out.items():
        assert np.array_equal(dist_, want), delta
    assert out[8][2] > 0


def test_virtual_ranks_sssp_cpu_engine():
    from _dist_cpu import CpuSsspEngine
    from paper_1701_01170_b200.dist import VirtualComm, sssp_partitioned

    row, col = port.rmat_csr(9, 16, 0)
    w = port.assign_random_weights(row, col, 1, 64, 0)
    n = len(row) - 1
    want = c_oracle.dijkstra(row, col, w, 0)
    for P in (1, 3, 4):
        engines = [CpuSsspEngine(row, col, w, n, P, r) for r in range(P)]
        sssp_partitioned(VirtualComm(engines), n, 0, 16)
        got = np.full(n, -1, dtype=np.int64)
        for e in engines:
            got[e.r::P] = e.dist
        assert np.array_equal(got, want), P

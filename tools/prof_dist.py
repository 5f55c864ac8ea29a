"""Where the partitioned BFS spends a level (one rank, NCCL world size 1).

    python tools/prof_dist.py [--scale 24]

Prints the wall time per BFS, the GPU-busy time per BFS (sum of kernel and
memcpy durations from the torch profiler), and the host time of each call
kind of the level loop (engine entry points and collectives)."""
import argparse
import collections
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=24)
    ap.add_argument("--runs", type=int, default=20)
    args = ap.parse_args()
    import torch
    import torch.distributed as dist

    from paper_1701_01170_b200.dist import DeviceEngine, ProcessComm, bfs_partitioned, partition_graph
    from paper_1701_01170_b200.generators import rmat_device_graph

    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29573")
    dist.init_process_group("nccl", rank=0, world_size=1)
    dg = rmat_device_graph(args.scale, 16, 0)
    n, m = dg.num_vertices, dg.num_edges
    lrow, lcol = partition_graph(dg, 1, 0)
    del dg
    eng = DeviceEngine(lrow, lcol, n, m, 1, 0)
    comm = ProcessComm(eng)
    for _ in range(3):
        bfs_partitioned(comm, n, m, 0, direction="auto")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.runs):
        bfs_partitioned(comm, n, m, 0, direction="auto")
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / args.runs * 1e3
    print(f"wall per BFS: {wall:.3f} ms")
    from paper_1701_01170_b200.dist import bfs_partitioned_native

    for _ in range(3):
        bfs_partitioned_native(eng, None, n, m, 0, direction="auto")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.runs):
        stn = bfs_partitioned_native(eng, None, n, m, 0, direction="auto")
    torch.cuda.synchronize()
    print(f"native loop: wall per BFS {(time.perf_counter() - t0) / args.runs * 1e3:.3f} ms, "
          f"device {stn.device_ms:.3f} ms")

    # host time per call kind
    acc = collections.defaultdict(float)
    cnt = collections.Counter()

    def wrap(obj, name):
        f = getattr(obj, name)

        def g(*a, **k):
            t = time.perf_counter()
            r = f(*a, **k)
            acc[name] += time.perf_counter() - t
            cnt[name] += 1
            return r
        setattr(obj, name, g)

    for nm in ("push_expand", "push_claim", "pull_prepare", "pull", "commit", "reset"):
        wrap(eng, nm)
    for nm in ("exchange_counts", "exchange_pairs", "allgather_frontier", "allreduce_stats"):
        wrap(comm, nm)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.runs):
        bfs_partitioned(comm, n, m, 0, direction="auto")
    torch.cuda.synchronize()
    wall2 = (time.perf_counter() - t0) / args.runs * 1e3
    print(f"wall per BFS (instrumented): {wall2:.3f} ms")
    for k in sorted(acc, key=acc.get, reverse=True):
        print(f"  {k:20s} calls/BFS {cnt[k] / args.runs:5.1f}  host ms/BFS {acc[k] / args.runs * 1e3:.3f}")

    from torch.profiler import ProfilerActivity, profile

    with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
        for _ in range(5):
            bfs_partitioned(comm, n, m, 0, direction="auto")
        torch.cuda.synchronize()
    busy = collections.defaultdict(float)
    for ev in prof.events():
        if ev.device_type.name == "CUDA":
            busy[ev.name] += ev.device_time_total if hasattr(ev, "device_time_total") else ev.cuda_time_total
    tot = sum(busy.values()) / 5 / 1e3
    print(f"GPU busy per BFS: {tot:.3f} ms")
    for k in sorted(busy, key=busy.get, reverse=True)[:15]:
        print(f"  {busy[k] / 5:9.1f} us  {k[:90]}")
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

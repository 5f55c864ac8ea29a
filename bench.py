"""Benchmark: BFS GTEPS on R-MAT scale-24 ef16 (BASELINE.json metric) on B200.

    python bench.py --gpus N --steps K --warmup W [--impl ours|reference]

One step = one direction-optimised BFS from vertex 0 (reference
primitives/bfs.py with direction="auto", do_a=1e-3, do_b=0.2) over the
canonical undirected R-MAT scale-24 edge-factor-16 graph (seed 0), built
bit-exactly on the GPU (csrc/gfx_rmat.cu).  ``value`` = E_r * steps * ranks /
max-over-ranks device time, E_r = sum of degrees of reached vertices (the
paper's TEPS numerator).

Also reported on the same line: push-only BFS and SSSP (delta 32) GTEPS, the
roofline of the dominant kernel, the end-to-end number through the public
API with host buffers, the CPU baseline (oracle port of the reference
algorithm on this host) and GPU clocks sampled during the run.

--impl reference times the reference's own CPU algorithm (the numpy port in
oracle/graphfx_port.py, the reference being pure Python) on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--scale", type=int, default=24)
    ap.add_argument("--edge-factor", type=int, default=16)
    ap.add_argument("--source", type=int, default=0)
    ap.add_argument("--direction", default="auto", choices=["auto", "push", "pull"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip push-only / SSSP lines")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-s27", action="store_true", help="skip the single-GPU scale-27 extra")
    ap.add_argument("--partitioned", action="store_true",
                    help="use the partitioned multi-GPU engine even at N=1 (default: N>1)")
    ap.add_argument("--write-ref-cache", default=None, help=argparse.SUPPRESS)
    ap.add_argument("--python-loop", action="store_true",
                    help="partitioned engine: drive the levels from Python (dist.bfs_partitioned) "
                         "instead of the native loop (gfx_dbfs_run); implies --host-loop")
    ap.add_argument("--host-loop", action="store_true",
                    help="partitioned engine: the host-driven level loop with NCCL collectives "
                         "(gfx_dbfs_run) instead of the device-resident kernel (gfx_pdbfs)")
    return ap.parse_args()


# ---------------------------------------------------------------------------
# distributed plumbing (one process per GPU)
# ---------------------------------------------------------------------------
class Dist:
    def __init__(self):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.pg = None

    def init(self, backend):
        if self.world > 1:
            import torch.distributed as dist

            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            dist.init_process_group(backend=backend)
            self.pg = dist

    def barrier(self):
        if self.pg:
            if self.pg.get_backend() == "nccl":
                import torch

                self.pg.barrier(device_ids=[self.local])
                torch.cuda.synchronize()
            else:
                self.pg.barrier()

    def max(self, x: float) -> float:
        if not self.pg:
            return x
        import torch

        dev = torch.device("cuda", self.local) if self.pg.get_backend() == "nccl" else "cpu"
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        self.pg.all_reduce(t, op=self.pg.ReduceOp.MAX)
        return float(t.item())

    def sum(self, x: float) -> float:
        if not self.pg:
            return x
        import torch

        dev = torch.device("cuda", self.local) if self.pg.get_backend() == "nccl" else "cpu"
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        self.pg.all_reduce(t)
        return float(t.item())

    def close(self):
        if self.pg:
            self.pg.destroy_process_group()


# ---------------------------------------------------------------------------
# clocks sampled during the run (B200_PROFILING.md clocks line)
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,utilization.gpu,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines: list[str] = []
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        samples = []
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                samples.append((float(parts[0]), float(parts[1]), float(parts[2]), parts[3:7]))
            except ValueError:
                continue
        if not samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        loaded = [s for s in samples if s[2] > 0] or samples
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in loaded for i, v in enumerate(s[3])
                          if v.lower() == "active"})
        return {"sm_mhz": statistics.median(s[0] for s in loaded),
                "sm_max_mhz": max(s[1] for s in samples), "reasons": reasons,
                "samples": len(samples), "samples_under_load": len([s for s in samples if s[2] > 0])}


def ncu_traffic(kernel: str, scale: int):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel`
    from the committed `ncu --set full` summary (profiles/ncu_traffic.json,
    written by tools/ncu_summary.py --traffic); None when not captured."""
    p = ROOT / "profiles" / "ncu_traffic.json"
    try:
        rec = json.loads(p.read_text())[f"{kernel}@s{scale}"]
        return int(rec["dram_bytes"]), rec["source"]
    except Exception:
        return None, None


def measured_peak_gbs() -> tuple[float, str]:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())["hbm_gbs"]), "measured"
        except Exception:
            pass
    return 6650.0, "fallback"


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def run_ours(args, dist: Dist):
    import numpy as np
    import torch

    torch.cuda.set_device(dist.local)
    dist.init("nccl")
    if dist.world > 1 or args.partitioned:
        return run_partitioned(args, dist)
    import paper_1701_01170_b200 as gfx
    from paper_1701_01170_b200 import _native
    from paper_1701_01170_b200.generators import rmat_device_graph
    from paper_1701_01170_b200.primitives.bfs import bfs_batch, bfs_device

    t_build = time.perf_counter()
    dg = rmat_device_graph(args.scale, args.edge_factor, 0)
    torch.cuda.synchronize()
    build_s = time.perf_counter() - t_build
    ctx = dg.ctx
    n = dg.num_vertices
    labels = torch.empty(n, dtype=torch.int32, device="cuda")
    preds = torch.empty(n, dtype=torch.int32, device="cuda")

    def step(direction):
        return bfs_device(dg, args.source, direction=direction, labels=labels, preds=preds)[2]

    sampler = ClockSampler(dist.local) if dist.rank == 0 or True else None
    sampler.start()
    for _ in range(max(args.warmup, 3)):
        st = step(args.direction)
    e_r = st.edges_reached
    # timed region: K steps back to back (inputs -- the 2.2 GB CSR -- exceed L2;
    # every BFS re-initialises its labels/bitmaps, so nothing carries over).
    # The RunStats degree post-pass (E_r, pull-level edge counts) is switched
    # off inside it; E_r comes from the warm-up run above.
    ctx.set_stats(0)
    dist.barrier()
    torch.cuda.synchronize()
    l0 = _native.launch_count()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record()
    # K BFS runs enqueued back to back (one cooperative launch each, one
    # synchronisation): the device throughput of the primitive itself
    bfs_batch(dg, [args.source] * args.steps, direction=args.direction, labels=labels,
              preds=preds)
    ev1.record()
    torch.cuda.synchronize()
    launches = _native.launch_count() - l0
    dist.barrier()
    local_ms = ev0.elapsed_time(ev1)
    t_ms = dist.max(local_ms)
    # the same K steps through the per-call API (one host round trip each),
    # with the RunStats post-pass back on as every public call has it
    ctx.set_stats(1)
    t_call0 = time.perf_counter()
    for _ in range(args.steps):
        step(args.direction)
    torch.cuda.synchronize()
    per_call_ms = (time.perf_counter() - t_call0) * 1e3 / args.steps
    # a sustained window so the clock sampler sees the GPU under load
    t_end = time.perf_counter() + 1.5
    while time.perf_counter() < t_end:
        step(args.direction)
    torch.cuda.synchronize()
    clocks = sampler.stop()
    ctx.set_stats(1)

    total_edges = dist.sum(float(e_r) * args.steps)
    value = total_edges / (t_ms * 1e-3) / 1e9
    ms_per_step = t_ms / args.steps

    # ---- roofline of the dominant kernel.  The whole DO-BFS is ONE
    # cooperative launch (k_bfs_persistent), so the kernel's algorithmic
    # bytes per launch are the whole BFS's (SURVEY 8(d) per-level formulas,
    # counted by the kernel) and its launch duration is ms_per_step (CUDA
    # events around the K back-to-back launches on the launching stream).
    # The per-level split comes from a separate run with globaltimer stamps.
    ctx.set_timing(True)
    prof = step(args.direction)
    ctx.set_timing(False)
    peak, peak_kind = measured_peak_gbs()
    achieved = prof.bytes_alg / (ms_per_step * 1e-3) / 1e9
    lv = max(prof.device_levels, key=lambda x: x["ms"])
    traffic, traffic_src = ncu_traffic("k_bfs_persistent", args.scale)
    roofline = {
        "bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
        "frac": round(achieved / peak, 4), "traffic": traffic,
        "kernel": "k_bfs_persistent", "bytes_alg_per_launch": prof.bytes_alg,
        "launch_ms": round(ms_per_step, 4), "peak_source": peak_kind,
        "traffic_source": traffic_src,
        "init_ms": round(prof.init_ms, 4),
        "heaviest_level": {"iteration": lv["iteration"], "mode": lv["mode"],
                           "ms": round(lv["ms"], 4), "bytes_alg": lv["bytes_alg"],
                           "achieved_gbs": round(lv["bytes_alg"] / (lv["ms"] * 1e-3) / 1e9, 1)},
        "levels": [{k: (round(v, 4) if isinstance(v, float) else v) for k, v in d.items()}
                   for d in prof.device_levels],
    }

    out = {
        "metric": "BFS GTEPS on R-MAT scale-24 ef16 (direction-optimized, source 0)",
        "value": round(value, 2), "unit": "GTEPS", "n_gpus": dist.world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4),
        "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "int32", "data": "synthetic",
        "config": workload_config(args, n, dg.num_edges, e_r, st.reached),
        "run": {"parallelism": f"replicas{dist.world}" if dist.world > 1 else "1gpu",
                   "l2": "per-BFS state re-initialised each step",
                   "graph_build_s": round(build_s, 3),
                   "stats_post_pass": "off in timed steps (E_r from a warm-up run)",
                   "level_loop": "device-resident cooperative kernel, K launches enqueued back to back",
                   "per_call_ms": round(per_call_ms, 4),
                   "per_call_gteps": round(e_r / (per_call_ms * 1e-3) / 1e9, 2),
                   "per_call_what": "public bfs_device call: one host round trip per BFS "
                                    "and the RunStats degree post-pass (stats on)"},
        "roofline": roofline, "gpu_launches": int(launches), "clocks": clocks,
    }

    # ---- extras: push-only BFS and SSSP on the same graph
    if not args.no_extras:
        out["extras"] = extras(args, dg, labels, preds, dist, peak)

    # ---- end to end through the public API with host buffers
    if not args.no_e2e:
        out["e2e"] = e2e(args, dg, dist, e_r)

    # ---- CPU baseline (oracle port of the reference algorithm), rank 0, N=1
    if dist.rank == 0 and dist.world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(args, dg, e_r)
    if dist.rank == 0:
        emit(out)
    dist.close()


def run_partitioned(args, dist: Dist):
    """N GPUs, one process each: the s24 graph 1D-partitioned (owner = v mod N),
    per-level NCCL exchange (paper_1701_01170_b200/dist.py).  Strong scaling:
    the same graph and BFS at every N."""
    import torch.distributed as tdist

    if dist.pg is None:  # --partitioned at N=1: a one-rank NCCL group
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29571")
        os.environ.setdefault("RANK", "0")
        os.environ.setdefault("WORLD_SIZE", "1")
        tdist.init_process_group("nccl")
        dist.pg = tdist
    P, r = dist.world, dist.rank
    sampler = ClockSampler(dist.local)
    sampler.start()
    run = _partitioned_run(args, dist, args.scale, args.steps, max(args.warmup, 3))
    clocks = sampler.stop()
    st, t_ms, e_r, n, m, launches, build_s, loop = (run[k] for k in (
        "st", "t_ms", "e_r", "n", "m", "launches", "build_s", "loop"))
    extra = {}
    if args.scale == 24 and not args.no_s27:
        try:
            r27 = _partitioned_run(args, dist, 27, 5, 3, with_1gpu=True)
            ms27 = r27["t_ms"] / 5
            extra["bfs_do_s27_partitioned"] = {
                "gteps": round(r27["e_r"] / (ms27 * 1e-3) / 1e9, 2), "ms": round(ms27, 4),
                "n_gpus": P, "n": r27["n"], "m": r27["m"], "E_r": r27["e_r"],
                "level_loop": r27["loop"],
                "single_gpu_same_graph": r27.get("one_gpu"),
                "what": "BASELINE config C5: R-MAT s27 ef16 1D-partitioned over the N ranks, "
                        "5 BFS from vertex 0 timed (max over ranks); single_gpu_same_graph = "
                        "rank 0's device-resident DO-BFS on the whole s27 graph before partitioning",
                "trace": [[t["iteration"], t["decision"], t["n_f"]]
                          for t in r27["st"].direction_trace]}
        except Exception as exc:  # noqa: BLE001 -- report, keep the headline line
            extra["s27_error"] = repr(exc)
    if not args.no_extras:
        try:
            extra["sssp_partitioned"] = _partitioned_sssp(args, dist)
        except Exception as exc:  # noqa: BLE001 -- report, keep the headline line
            extra["sssp_partitioned_error"] = repr(exc)
    if P == 1 and not args.no_extras and not (args.host_loop or args.python_loop):
        try:
            extra["virtual_ranks"] = _virtual_ranks(args)
        except Exception as exc:  # noqa: BLE001 -- report, keep the headline line
            extra["virtual_ranks_error"] = repr(exc)
    peak, peak_kind = measured_peak_gbs()
    ms = t_ms / args.steps
    achieved = st.bytes_alg / (ms * 1e-3) / 1e9 / P
    out = {
        "metric": "BFS GTEPS on R-MAT scale-24 ef16 (direction-optimized, source 0)",
        "value": round(e_r * args.steps / (t_ms * 1e-3) / 1e9, 2), "unit": "GTEPS",
        "n_gpus": P, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int32",
        "data": "synthetic",
        "config": workload_config(args, n, m, e_r, run["reached"]),
        "run": {"parallelism": f"1d-cyclic-partition{P}",
                   "exchange": ("NCCL all_to_all(pair counts) + send/recv(dst,src pairs) push / "
                                "all_gather(frontier bitmaps) pull / allreduce(level counters)")
                   if (args.host_loop or args.python_loop) else
                   ("peer stores over CUDA-IPC mappings: (dst,src) pairs into the owner's inbox "
                    "(push), frontier-bitmap slices and level counters to every rank, "
                    "release/acquire flag barriers"),
                   "level_loop": loop,
                   "l2": "per-BFS state re-initialised each step",
                   "graph_build_s": round(build_s, 3)},
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": None,
                     "kernel": "whole partitioned BFS per GPU (bytes_alg / N / step time)",
                     "peak_source": peak_kind},
        "gpu_launches": int(launches), "clocks": clocks,
        "e2e": {"value": round(e_r * args.steps / (run["e2e"]["ms"] * 1e-3) / 1e9, 3),
                "unit": "GTEPS", "h2d_bytes_per_step": run["e2e"]["h2d_bytes_per_step"],
                "d2h_bytes_per_step": run["e2e"]["d2h_bytes_per_step"],
                "ms_per_step": round(run["e2e"]["ms"] / args.steps, 4),
                "what": "graph resident (partitioned at build time): per step the source goes "
                        "up and every rank's int32 labels + preds come back to pinned host "
                        "memory, max over ranks"},
        "trace": [[t["iteration"], t["decision"], t["n_f"]] for t in st.direction_trace],
        "extras": extra,
    }
    if dist.rank == 0:
        emit(out)
    dist.close()


def _partitioned_run(args, dist, scale: int, steps: int, warmup: int, with_1gpu: bool = False):
    """Build R-MAT ``scale`` on every rank, keep this rank's partition, and
    time ``steps`` partitioned BFS (CUDA events, max over ranks)."""
    if not (args.host_loop or args.python_loop):
        return _partitioned_run_device(args, dist, scale, steps, warmup, with_1gpu)
    import torch

    from paper_1701_01170_b200 import _native
    from paper_1701_01170_b200.dist import (DeviceEngine, NativeComm, ProcessComm, bfs_partitioned,
                                            bfs_partitioned_native, partition_graph)
    from paper_1701_01170_b200.generators import rmat_device_graph

    P, r = dist.world, dist.rank
    torch.cuda.empty_cache()
    ref_labels = None
    t_build = time.perf_counter()
    dg = rmat_device_graph(scale, args.edge_factor, 0)
    n, m = dg.num_vertices, dg.num_edges
    one_gpu = None
    if with_1gpu and r == 0:
        from paper_1701_01170_b200.primitives.bfs import bfs_batch, bfs_device

        lab = torch.empty(n, dtype=torch.int32, device=dg.row.device)
        prd = torch.empty(n, dtype=torch.int32, device=dg.row.device)
        for _ in range(3):
            st1 = bfs_device(dg, args.source, direction=args.direction, labels=lab, preds=prd)[2]
        ms1 = bfs_batch(dg, [args.source] * 5, direction=args.direction, labels=lab, preds=prd) / 5
        one_gpu = {"gteps": round(st1.edges_reached / (ms1 * 1e-3) / 1e9, 2), "ms": round(ms1, 4)}
        ref_labels = lab  # kept: the partitioned labels are checked against it below
        del prd
    lrow, lcol = partition_graph(dg, P, r)
    del dg
    torch.cuda.empty_cache()
    eng = DeviceEngine(lrow, lcol, n, m, P, r)
    comm = ProcessComm(eng)
    ncomm, loop = None, "python"
    if not args.python_loop:
        err = None
        try:
            ncomm = NativeComm(eng, single_rank_nccl=(P == 1))
        except Exception as exc:  # noqa: BLE001 -- agreed on below, reported in the line
            err = repr(exc)
        if dist.sum(0.0 if err is None else 1.0) == 0:
            loop = "native"
        else:
            loop = f"python (native communicator unavailable: {err})"
    torch.cuda.synchronize()
    build_s = time.perf_counter() - t_build

    def step():
        if loop == "native":
            return bfs_partitioned_native(eng, ncomm, n, m, args.source, direction=args.direction)
        return bfs_partitioned(comm, n, m, args.source, direction=args.direction)

    for _ in range(warmup):
        st = step()
    reached, deg = eng.reached_degree_sum()
    e_r = int(dist.sum(float(deg)))
    reached = int(dist.sum(float(reached)))
    dist.barrier()
    torch.cuda.synchronize()
    l0 = _native.launch_count()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(steps):
        step()
    ev1.record()
    torch.cuda.synchronize()
    launches = _native.launch_count() - l0
    dist.barrier()
    t_ms = dist.max(ev0.elapsed_time(ev1))
    if with_1gpu:
        match = _labels_match(eng, ref_labels if r == 0 else None, P, r, n)
        if one_gpu is not None:
            one_gpu["labels_equal_partitioned"] = match
        ref_labels = None
    # end to end with the graph resident: the source goes up, every rank's
    # labels + preds come back to pinned host memory, each step
    lab_h = torch.empty(eng.nl, dtype=torch.int32, pin_memory=True)
    prd_h = torch.empty(eng.nl, dtype=torch.int32, pin_memory=True)
    src_h = torch.tensor([args.source], dtype=torch.int64, pin_memory=True)
    src_d = torch.empty(1, dtype=torch.int64, device=eng.device)
    dist.barrier()
    torch.cuda.synchronize()
    ev0.record()
    for _ in range(steps):
        src_d.copy_(src_h, non_blocking=True)
        step()
        lab_h.copy_(eng.labels[: eng.nl], non_blocking=True)
        prd_h.copy_(eng.preds[: eng.nl], non_blocking=True)
        torch.cuda.current_stream().synchronize()
    ev1.record()
    torch.cuda.synchronize()
    dist.barrier()
    e2e_ms = dist.max(ev0.elapsed_time(ev1))
    e2e = {"ms": e2e_ms, "d2h_bytes_per_step": int(dist.sum(float(8 * eng.nl))),
           "h2d_bytes_per_step": 8 * P}
    if ncomm is not None:
        ncomm.close()
    del eng, comm, lrow, lcol
    torch.cuda.empty_cache()
    return {"st": st, "t_ms": t_ms, "e_r": e_r, "reached": reached, "n": n, "m": m,
            "launches": launches,
            "build_s": build_s, "one_gpu": one_gpu, "loop": loop, "e2e": e2e}


class _DevStats:
    """DistBfsStats-shaped view of the device-resident engine's records."""

    def __init__(self, levels, st):
        self.iterations = st.iterations
        self.direction_trace = [dict(iteration=lv["iteration"], decision=lv["decision"],
                                     n_f=lv["n_f"]) for lv in levels]
        self.bytes_alg = sum(lv["bytes_alg"] for lv in levels)
        self.device_ms = st.device_ms


def _one_gpu_reference(args, dg):
    import torch

    from paper_1701_01170_b200.primitives.bfs import bfs_batch, bfs_device

    n = dg.num_vertices
    lab = torch.empty(n, dtype=torch.int32, device=dg.row.device)
    prd = torch.empty(n, dtype=torch.int32, device=dg.row.device)
    for _ in range(3):
        st1 = bfs_device(dg, args.source, direction=args.direction, labels=lab, preds=prd)[2]
    ms1 = bfs_batch(dg, [args.source] * 5, direction=args.direction, labels=lab, preds=prd) / 5
    return {"gteps": round(st1.edges_reached / (ms1 * 1e-3) / 1e9, 2), "ms": round(ms1, 4)}, lab


def _partitioned_run_device(args, dist, scale: int, steps: int, warmup: int,
                            with_1gpu: bool = False):
    """The device-resident partitioned BFS (csrc/gfx_pdbfs.cu): one cooperative
    launch per rank and BFS; frontier slices, claim pairs and level counters
    go to the peers through CUDA-IPC mappings (NVLink) and device flag
    barriers -- no host round trip and no host-launched collective per level.
    ``steps`` BFS launched back to back, timed with CUDA events (max over
    ranks)."""
    import torch

    from paper_1701_01170_b200 import _native
    from paper_1701_01170_b200.dist import DeviceResidentRank
    from paper_1701_01170_b200.generators import rmat_device_graph

    P, r = dist.world, dist.rank
    torch.cuda.empty_cache()
    t_build = time.perf_counter()
    dg = rmat_device_graph(scale, args.edge_factor, 0)
    n, m = dg.num_vertices, dg.num_edges
    one_gpu, ref_labels = None, None
    if with_1gpu and r == 0:
        one_gpu, ref_labels = _one_gpu_reference(args, dg)
    eng, err = None, None
    try:
        eng = DeviceResidentRank(dg, P, r, group=None)
    except Exception as exc:  # noqa: BLE001 -- e.g. no CUDA IPC between these GPUs
        err = repr(exc)
    if dist.sum(0.0 if err is None else 1.0) > 0:
        # every rank falls back together to the host-driven NCCL loop
        if eng is not None:
            eng.close()
        del dg, ref_labels
        torch.cuda.empty_cache()
        import copy

        args2 = copy.copy(args)
        args2.host_loop = True
        out = _partitioned_run(args2, dist, scale, steps, warmup, with_1gpu)
        out["loop"] = f"{out['loop']} (device-resident engine unavailable: {err})"
        return out
    del dg
    torch.cuda.empty_cache()
    torch.cuda.synchronize()
    build_s = time.perf_counter() - t_build
    for _ in range(warmup):
        lab, prd, st, levels = eng.run(args.source, direction=args.direction)
    deg = (eng.lrow[1:] - eng.lrow[:-1])
    hit = lab != 2147483647
    e_r = int(dist.sum(float(deg[hit].sum().item())))
    reached = int(dist.sum(float(hit.sum().item())))
    dist.barrier()
    torch.cuda.synchronize()
    l0 = _native.launch_count()
    local_ms = eng.batch_ms(args.source, steps, direction=args.direction)
    launches = _native.launch_count() - l0
    dist.barrier()
    t_ms = dist.max(local_ms)
    # the timed launches leave the labels in the engine: the last run's result
    lab, prd, st, levels = eng.run(args.source, direction=args.direction)
    if with_1gpu:
        match = _labels_match(eng, ref_labels if r == 0 else None, P, r, n)
        if one_gpu is not None:
            one_gpu["labels_equal_partitioned"] = match
        ref_labels = None
    # end to end with the graph resident: per step the source goes up and this
    # rank's int32 labels + preds come back to pinned host memory
    lab_h = torch.empty(eng.nl, dtype=torch.int32, pin_memory=True)
    prd_h = torch.empty(eng.nl, dtype=torch.int32, pin_memory=True)
    dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        lab, prd, _, _ = eng.run(args.source, direction=args.direction)
        lab_h.copy_(lab, non_blocking=True)
        prd_h.copy_(prd, non_blocking=True)
        torch.cuda.current_stream().synchronize()
    dist.barrier()
    e2e_ms = dist.max((time.perf_counter() - t0) * 1e3)
    e2e = {"ms": e2e_ms, "d2h_bytes_per_step": int(dist.sum(float(8 * eng.nl))),
           "h2d_bytes_per_step": 8 * P}
    stats = _DevStats(levels, st)
    eng.close()
    del eng
    torch.cuda.empty_cache()
    return {"st": stats, "t_ms": t_ms, "e_r": e_r, "reached": reached, "n": n, "m": m,
            "launches": launches, "build_s": build_s, "one_gpu": one_gpu,
            "loop": "device-resident (gfx_pdbfs: one cooperative launch per rank, peer-memory "
                    "exchange, device flag barriers)",
            "e2e": e2e}


def _virtual_ranks(args, Ps=(2, 4, 8), steps: int = 10):
    """The device-resident partitioned BFS with P virtual ranks in ONE launch on
    this GPU (dist.VirtualRanksBfs): the whole multi-rank protocol -- inbox
    stores, sliced frontier copies, counter tables, exchange barriers -- with
    every rank sharing one GPU's SMs and HBM.  Labels checked against the
    single-GPU BFS."""
    import torch

    from paper_1701_01170_b200.dist import VirtualRanksBfs
    from paper_1701_01170_b200.generators import rmat_device_graph
    from paper_1701_01170_b200.primitives.bfs import bfs_device

    dg = rmat_device_graph(args.scale, args.edge_factor, 0)
    ref = bfs_device(dg, args.source, direction=args.direction)[0]
    out = {"what": "P ranks of the partitioned BFS in one launch on ONE GPU (CTA b runs rank "
                   "b mod P); ms per BFS over back-to-back launches"}
    for P in Ps:
        eng = VirtualRanksBfs(dg, P)
        lab, _, st, levels = eng.run(args.source, direction=args.direction)
        ok = bool(torch.equal(lab, ref))
        eng.batch_ms(args.source, 2, direction=args.direction)
        ms = eng.batch_ms(args.source, steps, direction=args.direction) / steps
        out[f"P{P}"] = {"ms": round(ms, 4), "labels_equal_1gpu": ok,
                        "levels_ms": [round(lv["ms"], 4) for lv in levels]}
        eng.close()
        del eng
        torch.cuda.empty_cache()
    return out


def _partitioned_sssp(args, dist, delta: int = 32, steps: int = 3):
    """Partitioned near/far SSSP (SURVEY 8(e) row e, dist.sssp_partitioned) on
    the bench graph with weights 1..64: each rank holds its 1D-cyclic share,
    offers cross ranks through all_to_all; CUDA events, max over ranks.  The
    distances are checked against the single-GPU SSSP on rank 0."""
    import torch

    from paper_1701_01170_b200.dist import (ProcessComm, SsspEngine, partition_graph,
                                            partition_weights, sssp_partitioned)
    from paper_1701_01170_b200.generators import rmat_device_graph
    from paper_1701_01170_b200.primitives.sssp import sssp_device

    P, r = dist.world, dist.rank
    torch.cuda.empty_cache()
    dgw = rmat_device_graph(args.scale, args.edge_factor, 0, weights=(1, 64), weight_seed=0)
    n = dgw.num_vertices
    ref = None
    if r == 0:
        d1, _, st1 = sssp_device(dgw, args.source, delta=delta)
        ref, e_r = d1, st1.edges_reached
    else:
        e_r = 0
    e_r = int(dist.sum(float(e_r)))
    eng, err = None, None
    if not (args.host_loop or args.python_loop):
        from paper_1701_01170_b200.dist import DeviceResidentSsspRank

        try:
            eng = DeviceResidentSsspRank(dgw, P, r)
        except Exception as exc:  # noqa: BLE001 -- e.g. no CUDA IPC between these GPUs
            err = repr(exc)
        if dist.sum(0.0 if err is None else 1.0) > 0 and eng is not None:
            eng.close()
            eng = None
    if eng is not None:
        # the device-resident engine (csrc/gfx_pdsssp.cu): one cooperative
        # launch per rank and run, offers / counters through peer memory
        del dgw
        dl, _, st = eng.run(args.source, delta)  # warm-up
        dist.barrier()
        torch.cuda.synchronize()
        ms = dist.max(eng.batch_ms(args.source, steps, delta)) / steps
        dl, _, st = eng.run(args.source, delta)
        nl = eng.nl
        nlmax = (n + P - 1) // P
        buf = torch.full((nlmax,), -2, dtype=torch.int32, device=eng.device)
        buf[:nl] = dl
        parts = [buf]
        if P > 1:
            import torch.distributed as tdist

            parts = [torch.empty_like(buf) for _ in range(P)]
            tdist.all_gather(parts, buf)
        ok = None
        if r == 0:
            ok = all(bool(torch.equal(parts[q][: len(range(q, n, P))], ref[q::P]))
                     for q in range(P))
        eng.close()
        del eng
        torch.cuda.empty_cache()
        return {"gteps": round(e_r / (ms * 1e-3) / 1e9, 2), "ms": round(ms, 3), "delta": delta,
                "n_gpus": P, "iterations": st.iterations,
                "bucket_advances": st.direction_switches, "relaxed_slots": st.work_slots,
                "dist_equal_single_gpu": ok,
                "what": "device-resident partitioned near/far SSSP (gfx_pdsssp: one cooperative "
                        "launch per rank, offers and counters through peer memory, flag "
                        "barriers); batched launches, CUDA events, max over ranks"}
    lrow, lcol = partition_graph(dgw, P, r)
    lw = partition_weights(dgw, lrow, P, r)
    eng = SsspEngine(lrow, lcol, lw, n, P, r)
    comm = ProcessComm(eng)
    st = sssp_partitioned(comm, n, args.source, delta)  # warm-up
    dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(steps):
        st = sssp_partitioned(comm, n, args.source, delta)
    ev1.record()
    torch.cuda.synchronize()
    ms = dist.max(ev0.elapsed_time(ev1)) / steps
    dl, _ = eng.result()
    nlmax = (n + P - 1) // P
    buf = torch.full((nlmax,), -2, dtype=torch.int32, device=eng.device)
    buf[: eng.nl] = dl
    parts = [buf]
    if P > 1:
        import torch.distributed as tdist

        parts = [torch.empty_like(buf) for _ in range(P)]
        tdist.all_gather(parts, buf)
    ok = None
    if r == 0:
        ok = all(bool(torch.equal(parts[q][: len(range(q, n, P))], ref[q::P])) for q in range(P))
    del eng, comm, lrow, lcol, lw, dgw
    torch.cuda.empty_cache()
    return {"gteps": round(e_r / (ms * 1e-3) / 1e9, 2), "ms": round(ms, 3), "delta": delta,
            "n_gpus": P, "iterations": st.iterations, "bucket_advances": st.bucket_advances,
            "relaxed_slots": st.relaxed_slots, "messages": st.messages,
            "dist_equal_single_gpu": ok,
            "what": "host-driven level loop over torch.distributed (NCCL) collectives"
                    + (f" (device-resident engine unavailable: {err})" if err else "")}


def _labels_match(eng, ref_labels, P: int, r: int, n: int):
    """labels(P) == labels(1): every rank's owned labels
    (cyclic: local l is global l*P + r) gathered to rank 0 and compared with
    the single-GPU labels of the same graph."""
    import torch

    nlmax = (n + P - 1) // P
    buf = torch.full((nlmax,), -2, dtype=torch.int32, device=eng.device)
    buf[: eng.nl] = eng.labels[: eng.nl]
    parts = [buf]
    if P > 1:
        import torch.distributed as tdist

        parts = [torch.empty_like(buf) for _ in range(P)]
        tdist.all_gather(parts, buf)
    if r != 0:
        return None
    ok = True
    for q in range(P):
        want = ref_labels[q::P]
        ok = ok and bool(torch.equal(parts[q][: want.numel()], want))
    return ok


def extras(args, dg, labels, preds, dist, peak):
    import torch

    from paper_1701_01170_b200.primitives.bfs import bfs_device

    res = {}
    # push-only BFS: the same batched device-resident launches as the headline
    from paper_1701_01170_b200.primitives.bfs import bfs_batch

    for _ in range(2):
        st = bfs_device(dg, args.source, direction="push", labels=labels, preds=preds)[2]
    k = max(3, args.steps // 2)
    ms = bfs_batch(dg, [args.source] * k, direction="push", labels=labels, preds=preds) / k
    res["bfs_push"] = {"gteps": round(st.edges_reached / (ms * 1e-3) / 1e9, 2),
                       "ms": round(ms, 4), "bytes_alg": st.bytes_alg,
                       "frac_of_hbm": round(st.bytes_alg / (ms * 1e-3) / 1e9 / peak, 4)}
    try:
        from paper_1701_01170_b200.primitives.sssp import sssp_device
    except ImportError:
        return res
    try:
        from paper_1701_01170_b200.generators import rmat_device_graph

        dgw = rmat_device_graph(args.scale, args.edge_factor, 0, weights=(1, 64), weight_seed=0)
        for delta in (32, None, 4):
            for _ in range(2):
                st = sssp_device(dgw, args.source, delta=delta)[2]
            # device time of the primitive as the library measures it (CUDA
            # events around its loop, the host-read iteration counters
            # included), mean of k calls
            times = [sssp_device(dgw, args.source, delta=delta)[2].device_ms for _ in range(k)]
            ms = sum(times) / len(times)
            # work-optimal lower bound: every reached vertex
            # settled once, 28 B per vertex + 8 B per slot of E_r
            lb = 28 * st.reached + 8 * st.edges_reached
            res[f"sssp_delta{delta or 'default'}"] = {
                "gteps": round(st.edges_reached / (ms * 1e-3) / 1e9, 2), "ms": round(ms, 4),
                "relaxed_slots": st.work_slots, "work_inflation": round(st.work_slots / max(st.edges_reached, 1), 3),
                "bytes_alg": st.bytes_alg,
                "frac_of_hbm": round(st.bytes_alg / (ms * 1e-3) / 1e9 / peak, 4),
                "bytes_lower_bound": lb,
                "frac_of_hbm_lower_bound": round(lb / (ms * 1e-3) / 1e9 / peak, 4)}
        del dgw
    except Exception as exc:  # report, do not hide
        res["sssp_error"] = repr(exc)
    try:
        res.update(secondary(args, dg, peak))
    except Exception as exc:
        res["secondary_error"] = repr(exc)
    if args.scale == 24 and not args.no_s27:
        try:
            res.update(scale27(args, peak))
        except Exception as exc:  # e.g. not enough free HBM next to the s24 graph
            res["s27_error"] = repr(exc)
    return res


def scale27(args, peak):
    """BASELINE config C5's input (R-MAT s27 ef16, 134M vertices, 4.2B
    directed slots) on ONE GPU: GPU-built, then the same device-resident
    DO-BFS from vertex 0, K launches back to back."""
    import torch

    from paper_1701_01170_b200.generators import rmat_device_graph
    from paper_1701_01170_b200.primitives.bfs import bfs_batch, bfs_device

    torch.cuda.empty_cache()
    t0 = time.perf_counter()
    dg = rmat_device_graph(27, args.edge_factor, 0)
    torch.cuda.synchronize()
    build_s = time.perf_counter() - t0
    labels = torch.empty(dg.num_vertices, dtype=torch.int32, device="cuda")
    preds = torch.empty(dg.num_vertices, dtype=torch.int32, device="cuda")
    st = None
    for _ in range(3):
        st = bfs_device(dg, args.source, direction="auto", labels=labels, preds=preds)[2]
    k = 5
    ms = bfs_batch(dg, [args.source] * k, direction="auto", labels=labels, preds=preds) / k
    out = {"bfs_do_s27_1gpu": {
        "gteps": round(st.edges_reached / (ms * 1e-3) / 1e9, 2), "ms": round(ms, 4),
        "n": dg.num_vertices, "m": dg.num_edges, "E_r": st.edges_reached,
        "reached": st.reached, "bytes_alg": st.bytes_alg,
        "frac_of_hbm": round(st.bytes_alg / (ms * 1e-3) / 1e9 / peak, 4),
        "graph_build_s": round(build_s, 2),
        "trace": [[t["iteration"], t["decision"], t["n_f"]] for t in st.direction_trace]}}
    del dg, labels, preds
    torch.cuda.empty_cache()
    return out


def secondary(args, dg, peak):
    """BASELINE configs C3/C4 (parity-and-time configs): PageRank (d = 0.85,
    20 iterations, eps = 0) and CC on the bench graph; BC from the source and
    TC on the scale-2 graph (s22 for the s24 bench).  Device time per call
    (CUDA events in the library), mean of 3 after a warm-up; bytes per SURVEY
    8(d) (PR 4m + 40n per iteration, CC from the kernel's counters)."""
    import torch

    from paper_1701_01170_b200.generators import rmat_device_graph
    from paper_1701_01170_b200.primitives.bc import bc_device
    from paper_1701_01170_b200.primitives.cc import cc_device
    from paper_1701_01170_b200.primitives.pagerank import pagerank_device
    from paper_1701_01170_b200.primitives.tc import tc_device

    def timed(fn, reps=3):
        fn()
        vals = []
        for _ in range(reps):
            st = fn()
            vals.append(st.device_ms)
        return st, sum(vals) / len(vals)

    n, m = dg.num_vertices, dg.num_edges
    out = {}
    st, ms = timed(lambda: pagerank_device(dg, 0.85, 0.0, 20)[1])
    b = (4 * m + 40 * n) * st.iterations
    out[f"pagerank_s{args.scale}"] = {"ms": round(ms, 3), "iterations": st.iterations,
                                      "bytes_alg": b,
                                      "frac_of_hbm": round(b / (ms * 1e-3) / 1e9 / peak, 4)}
    st, ms = timed(lambda: cc_device(dg)[2])
    out[f"cc_s{args.scale}"] = {"ms": round(ms, 3), "iterations": st.iterations,
                                "bytes_alg": st.bytes_alg,
                                "frac_of_hbm": round(st.bytes_alg / (ms * 1e-3) / 1e9 / peak, 4)}
    small = max(args.scale - 2, 10)
    dg2 = rmat_device_graph(small, args.edge_factor, 0)
    from paper_1701_01170_b200.primitives.bfs import bfs_device

    st_b = bfs_device(dg2, args.source, direction="push")[2]
    v_r, e_r2 = st_b.reached, st_b.edges_reached
    st, ms = timed(lambda: bc_device(dg2, [args.source])[1])
    b = 2 * (28 * v_r + 4 * e_r2) + 16 * v_r  # 2 x BFS-push bytes + 16 V_r
    out[f"bc_s{small}"] = {"ms": round(ms, 3), "gteps_x2": round(
        2 * st.edges_traversed / (ms * 1e-3) / 1e9, 2), "bytes_alg": b,
        "frac_of_hbm": round(b / (ms * 1e-3) / 1e9 / peak, 4)}
    total, _, osrc, odst, _ = tc_device(dg2)
    dplus = torch.bincount(osrc.long(), minlength=dg2.num_vertices)
    wedge = int((dplus[osrc.long()] + dplus[odst.long()]).sum().item())
    b_ref = 4 * wedge + 8 * int(osrc.numel())  # 4 sum(deg+u + deg+v) + 8 |E+|
    # the kernel intersects in the REVERSED orientation (short rows): its own
    # algorithmic bytes are 4 sum over reversed edges x=>y of (|R(x)| + |R(y)|)
    # + 8 |E+|; the SURVEY quantity above is the reference
    # orientation's wedge work, which the device does not perform
    dminus = torch.bincount(odst.long(), minlength=dg2.num_vertices)
    rwedge = int((dminus[osrc.long()] + dminus[odst.long()]).sum().item())
    b = 4 * rwedge + 8 * int(osrc.numel())
    del osrc, odst, dplus, dminus
    st, ms = timed(lambda: tc_device(dg2)[4])
    out[f"tc_s{small}"] = {"ms": round(ms, 3), "triangles": int(total), "bytes_alg": b,
                           "frac_of_hbm": round(b / (ms * 1e-3) / 1e9 / peak, 4),
                           "bytes_alg_reference_orientation": b_ref}
    del dg2
    torch.cuda.empty_cache()
    return out


def e2e(args, dg, dist, e_r):
    """End to end with host buffers, every step: the graph crosses PCIe from
    pinned host memory into the resident device graph, the BFS runs
    (gfx_bfs), and the reference-layout int64 labels and preds are read back
    into pinned host memory.  The graph's host image is the packed CSR
    (io.PackedCsr: int64 row offsets + the column ids as zigzag deltas in a
    StreamVByte layout, ~1.9 instead of 4 bytes per slot), decoded on the
    device (gfx_csr_unpack) before gfx_graph_refresh recomputes the graph
    constants; the same loop with plain int32 columns is reported beside it.
    Step k's read-back runs on its own stream and overlaps step k+1's upload
    (the two PCIe directions are independent); the upload of step k+1 waits
    for BFS k.  Also reported: the same public BFS call with the graph
    already resident (per-query host traffic only)."""
    import torch

    from paper_1701_01170_b200 import _native
    from paper_1701_01170_b200._native import UNVISITED32
    from paper_1701_01170_b200.graph import UNVISITED
    from paper_1701_01170_b200.io import pack_csr_device
    from paper_1701_01170_b200.primitives.bfs import bfs_device

    col_ref, row_ref = dg.col.clone(), dg.row.clone()
    row_h = dg.row.cpu().pin_memory()
    col_h = dg.col.cpu().pin_memory()
    packed_full = pack_csr_device(dg)
    packed_up = pack_csr_device(dg, upper=True)
    n = dg.num_vertices
    labels = torch.empty(n, dtype=torch.int32, device="cuda")
    preds = torch.empty(n, dtype=torch.int32, device="cuda")
    wide = [(torch.empty(n, dtype=torch.int64, device="cuda"),
             torch.empty(n, dtype=torch.int64, device="cuda")) for _ in range(2)]
    host = [(torch.empty(n, dtype=torch.int64, pin_memory=True),
             torch.empty(n, dtype=torch.int64, pin_memory=True)) for _ in range(2)]
    comp = torch.cuda.current_stream()
    up, dn = torch.cuda.Stream(), torch.cuda.Stream()

    dn_ev = [None, None]  # read-back k done: wide[k % 2] may be overwritten

    def widen(k):
        wl, wp = wide[k % 2]
        if dn_ev[k % 2] is not None:
            comp.wait_event(dn_ev[k % 2])
        wl.copy_(labels)
        wl.masked_fill_(labels == UNVISITED32, UNVISITED)
        wp.copy_(preds)
        ev = torch.cuda.Event()
        ev.record(comp)
        return ev

    def upload_slot(packed, s, after):
        """packed step input -> staging slot s on the upload stream, once the
        decode that last read slot s (event ``after``) is done"""
        with torch.cuda.stream(up):
            if after is not None:
                up.wait_event(after)
            dg.upload_packed_(packed, slot=s)
            ev = torch.cuda.Event()
            ev.record(up)
        return ev

    def run(k_steps, upload):
        # packed: double-buffered staging -- step k+1's graph crosses PCIe
        # while step k decodes and runs (every step still uploads its whole
        # input inside the timed region)
        up_ev, dec_ev = [None, None], [None, None]
        pk = {"upper": packed_up, "packed": packed_full}.get(upload)
        if pk is not None:
            up.wait_stream(comp)
            up_ev[0] = upload_slot(pk, 0, None)
        for k in range(k_steps):
            if pk is not None:
                s = k % 2
                if k + 1 < k_steps:  # slot 1-s was last read by decode k-1
                    up_ev[1 - s] = upload_slot(pk, 1 - s, dec_ev[1 - s])
                comp.wait_event(up_ev[s])
                dg.decode_packed_(slot=s)  # after BFS k-1 (same stream): graph buffers free
                dec_ev[s] = torch.cuda.Event()
                dec_ev[s].record(comp)
            elif upload == "plain":
                with torch.cuda.stream(up):
                    up.wait_stream(comp)
                    dg.row.copy_(row_h, non_blocking=True)
                    dg.col.copy_(col_h, non_blocking=True)
                comp.wait_stream(up)
                _native.call("gfx_graph_refresh", dg.handle)
            bfs_device(dg, args.source, direction=args.direction, labels=labels, preds=preds)
            ev = widen(k)
            with torch.cuda.stream(dn):
                dn.wait_event(ev)
                hl, hp = host[k % 2]
                hl.copy_(wide[k % 2][0], non_blocking=True)
                hp.copy_(wide[k % 2][1], non_blocking=True)
                dn_ev[k % 2] = torch.cuda.Event()
                dn_ev[k % 2].record(dn)
        torch.cuda.synchronize()

    k = max(2, min(args.steps, 20))  # the bench's K steps per timed batch (capped)
    total = dist.sum(float(e_r))
    d2h = n * 8 * 2
    out = {}
    # three timed batches of k steps each, the median reported (the host
    # side of these boxes occasionally stalls a whole batch 3-10x; every
    # batch is listed in the line)
    trials = {}

    def timed_batches(mode):
        times = []
        for _ in range(3):
            dist.barrier()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            run(k, mode)
            times.append(dist.max((time.perf_counter() - t0) / k))
        trials[mode or "resident"] = [round(x * 1e3, 3) for x in times]
        return sorted(times)[1]

    for mode in ("plain", "packed", "upper"):
        run(2, mode)
        dt = timed_batches(mode)
        # the decoded graph is the graph; the last read-back is the device result
        assert torch.equal(dg.col, col_ref) and torch.equal(dg.row, row_ref), mode
        assert int(host[(k - 1) % 2][0][args.source]) == 0
        out[mode] = (dt, (row_h.numel() * 8 + col_h.numel() * 4) if mode == "plain"
                     else {"packed": packed_full, "upper": packed_up}[mode].nbytes)
    del col_ref, row_ref
    dt_res = timed_batches(None)
    resident = {"value": round(total / dt_res / 1e9, 3), "unit": "GTEPS",
                "h2d_bytes_per_step": 8, "d2h_bytes_per_step": d2h,
                "ms_per_step": round(dt_res * 1e3, 3)}
    dt, h2d = out["upper"]
    dtf, h2df = out["packed"]
    dtp, h2dp = out["plain"]
    return {"value": round(total / dt / 1e9, 3), "unit": "GTEPS", "h2d_bytes_per_step": h2d,
            "d2h_bytes_per_step": d2h, "ms_per_step": round(dt * 1e3, 3), "steps": k,
            "what": "per step: the graph's upper triangle (each undirected edge once, as the "
                    "reference's COO input holds it) as a packed CSR (delta-coded row offsets "
                    "and columns) uploaded from pinned host, decoded and rebuilt into the full "
                    "sorted device CSR (gfx_csr_unpack, gfx_graph_rebuild_upper: stable "
                    "radix-sort transpose; asserted equal to the graph) + gfx_graph_refresh + "
                    "DO-BFS + int64 labels/preds read back to pinned host; double-buffered: "
                    "step k+1's upload (into the second staging slot) overlaps step k's "
                    "decode, BFS and read-back",
            "batches_ms_per_step": trials,
            "packed_full_csr": {"value": round(total / dtf / 1e9, 3), "unit": "GTEPS",
                                "h2d_bytes_per_step": h2df, "ms_per_step": round(dtf * 1e3, 3)},
            "plain_int32_columns": {"value": round(total / dtp / 1e9, 3), "unit": "GTEPS",
                                    "h2d_bytes_per_step": h2dp, "ms_per_step": round(dtp * 1e3, 3)},
            "graph_resident": resident}


def _host_graph(dg):
    import numpy as np

    row = dg.row.cpu().numpy().astype(np.int64)
    col = dg.col.cpu().numpy().astype(np.int64)
    return row, col


def cpu_baseline(args, dg, e_r):
    """One DO-BFS of the oracle port (numpy restatement of reference
    bfs.py) on this host, same graph, same source."""
    from oracle import graphfx_port as port

    row, col = _host_graph(dg)
    t0 = time.perf_counter()
    labels, _, _, _ = port.bfs(row, col, args.source, direction=args.direction,
                               rev=(row, col, None))
    dt = time.perf_counter() - t0
    return {"value": round(e_r / dt / 1e9, 6), "unit": "GTEPS", "cores": 1, "kind": "port",
            "sample": f"one {args.direction} BFS from vertex {args.source} on the full "
                      f"s{args.scale} graph ({dt:.1f} s), oracle/graphfx_port.py (numpy, 1 thread)",
            "seconds": round(dt, 3), "host_cpus": os.cpu_count()}


# ---------------------------------------------------------------------------
# reference arm: the UNMODIFIED reference (baseline/_ref) on the host cores
# ---------------------------------------------------------------------------
REF_DIR = ROOT / "baseline" / "_ref"
REF_BUDGET_S = float(os.environ.get("GFX_REF_BUDGET_S", "150"))


def workload_config(args, n: int, m: int, e_r: int, reached: int) -> dict:
    """The workload both arms report, key for key (same_config)."""
    return {"workload": f"bfs_do_rmat_s{args.scale}_ef{args.edge_factor}_src{args.source}",
            "scale": args.scale, "edge_factor": args.edge_factor, "seed": 0,
            "source": args.source, "direction": args.direction, "do_a": 1e-3, "do_b": 0.2,
            "n": int(n), "m": int(m), "E_r": int(e_r), "reached": int(reached),
            "l2": "inputs larger than L2 (CSR 2.2 GB vs 126 MB L2)"}


def write_reference_cache(args, path: str) -> None:
    """Child process of the reference arm: build the input with the GPU
    builder (input construction is untimed, reference bench.py:1-7) and write
    it in the reference's own GFXCSR v1 format (io.py:121-159)."""
    import torch

    from paper_1701_01170_b200.generators import rmat_device_graph
    from paper_1701_01170_b200.io import save_csr_cache_device

    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    dg = rmat_device_graph(args.scale, args.edge_factor, 0)
    save_csr_cache_device(dg, path)


def _sha(a) -> str:
    import hashlib

    import numpy as np

    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def run_reference(args, dist: Dist):
    """Times ``graphfx.bfs(g, source, direction, num_threads=cores)`` from the
    pip-installed reference in baseline/_ref through its public API.  The input
    is made by a CHILD process (GPU builder -> cache file) so this process
    never loads libgfx; it is read with the reference's own
    ``load_csr_cache`` and checked against the SHA-256 digests of the
    reference-built CSR (tests/golden/rmat_s<S>.json).  Each step is one full
    BFS; the timed steps stop once REF_BUDGET_S seconds are spent (at least
    one), so the run ends in minutes -- ``steps`` reports how many ran."""
    if dist.world > 1 and dist.rank != 0:
        return
    if not (REF_DIR / "graphfx" / "__init__.py").exists():
        return run_reference_port(args, dist)
    import numpy as np

    shm = Path("/dev/shm") if Path("/dev/shm").is_dir() else Path("/tmp")
    cache = shm / f"gfx_ref_rmat{args.scale}_{os.getpid()}.gfxcsr"
    t0 = time.perf_counter()
    env = dict(os.environ)
    for k in ("RANK", "WORLD_SIZE", "LOCAL_WORLD_SIZE", "GROUP_RANK"):
        env.pop(k, None)
    subprocess.run([sys.executable, str(ROOT / "bench.py"), "--write-ref-cache", str(cache),
                    "--scale", str(args.scale), "--edge-factor", str(args.edge_factor)],
                   check=True, env=env, stdout=sys.stderr)
    sys.path.insert(0, str(REF_DIR))
    import graphfx

    try:
        g = graphfx.load_csr_cache(str(cache))
    finally:
        cache.unlink(missing_ok=True)
    input_s = time.perf_counter() - t0
    golden = ROOT / "tests" / "golden" / f"rmat_s{args.scale}.json"
    verified = None
    if golden.exists():
        rec = json.loads(golden.read_text())
        verified = (_sha(g.row_offsets) == rec["row_sha"] and _sha(g.column_indices) == rec["col_sha"])
        if not verified:
            raise RuntimeError("reference-arm input differs from the reference-built CSR digests")
    cores = os.cpu_count() or 1
    kw = dict(direction=args.direction, num_threads=cores)
    t_pre = time.perf_counter()
    g.csc()  # the reference's own preprocessing (bfs.py:72-74), untimed as in its bench
    pre_s = time.perf_counter() - t_pre
    r = None
    for _ in range(max(1, min(args.warmup, 1))):
        r = graphfx.bfs(g, args.source, **kw)
    reached_mask = r.labels != graphfx.UNVISITED
    deg = np.diff(g.row_offsets)
    e_r = int(deg[reached_mask].sum())
    reached = int(reached_mask.sum())
    times = []
    t_end = time.perf_counter() + REF_BUDGET_S
    for _ in range(args.steps):
        t = time.perf_counter()
        graphfx.bfs(g, args.source, **kw)
        times.append(time.perf_counter() - t)
        if time.perf_counter() > t_end:
            break
    dt = sum(times) / len(times)
    v = e_r / dt / 1e9
    so = [p for p in _mapped_objects() if "paper_1701_01170_b200" in p or "libgfx" in p]
    out = {"metric": "BFS GTEPS on R-MAT scale-24 ef16 (direction-optimized, source 0)",
           "value": round(v, 6), "unit": "GTEPS", "n_gpus": dist.world, "steps": len(times),
           "steps_requested": args.steps, "warmup": 1, "ms_per_step": round(dt * 1e3, 3),
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int64",
           "data": "synthetic", "impl": "reference",
           "config": workload_config(args, g.num_vertices, g.num_edges, e_r, reached),
           "reference": {"package": f"graphfx {getattr(graphfx, '__version__', '?')} from "
                                    f"{Path(graphfx.__file__).parent}",
                         "call": f"graphfx.bfs(g, {args.source}, direction='{args.direction}', "
                                 f"num_threads={cores})",
                         "input": "child process: GPU builder -> GFXCSR v1 cache -> "
                                  "graphfx.load_csr_cache",
                         "input_sha_verified": verified, "input_s": round(input_s, 1),
                         "csc_preprocess_s": round(pre_s, 1),
                         "step_seconds": [round(x, 3) for x in times],
                         "libgfx_mapped": so},
           "cpu_baseline": {"value": round(v, 6), "unit": "GTEPS", "cores": cores,
                            "kind": "reference",
                            "sample": f"{len(times)} full DO-BFS runs of the reference package "
                                      f"(1 Python thread + {cores}-thread gather pool)"},
           "e2e": {"value": round(v, 6), "unit": "GTEPS", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    emit(out)


def _mapped_objects() -> list[str]:
    try:
        with open("/proc/self/maps") as f:
            return sorted({ln.split()[-1] for ln in f if ln.rstrip().endswith(".so")})
    except OSError:
        return []


def run_reference_port(args, dist: Dist):
    """Fallback when baseline/_ref is absent: the oracle port (numpy
    restatement of reference bfs.py), 1 thread, on a cache written by a child."""
    import numpy as np

    from oracle import graphfx_port as port

    shm = Path("/dev/shm") if Path("/dev/shm").is_dir() else Path("/tmp")
    cache = shm / f"gfx_ref_rmat{args.scale}_{os.getpid()}.gfxcsr"
    subprocess.run([sys.executable, str(ROOT / "bench.py"), "--write-ref-cache", str(cache),
                    "--scale", str(args.scale), "--edge-factor", str(args.edge_factor)],
                   check=True, stdout=sys.stderr)
    from paper_1701_01170_b200.io import load_csr_cache

    g = load_csr_cache(cache)
    cache.unlink(missing_ok=True)
    row, col = g.row_offsets, g.column_indices
    labels, _, _, _ = port.bfs(row, col, args.source, direction=args.direction,
                               rev=(row, col, None))
    mask = labels != port.UNVISITED
    e_r = int(np.diff(row)[mask].sum())
    times = []
    t_end = time.perf_counter() + REF_BUDGET_S
    for _ in range(args.steps):
        t = time.perf_counter()
        port.bfs(row, col, args.source, direction=args.direction, rev=(row, col, None))
        times.append(time.perf_counter() - t)
        if time.perf_counter() > t_end:
            break
    dt = sum(times) / len(times)
    v = e_r / dt / 1e9
    emit({"metric": "BFS GTEPS on R-MAT scale-24 ef16 (direction-optimized, source 0)",
          "value": round(v, 6), "unit": "GTEPS", "n_gpus": dist.world, "steps": len(times),
          "warmup": 1, "ms_per_step": round(dt * 1e3, 3), "higher_is_better": True,
          "scaling": "weak", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
          "impl": "reference",
          "config": workload_config(args, len(row) - 1, len(col), e_r, int(mask.sum())),
          "cpu_baseline": {"value": round(v, 6), "unit": "GTEPS", "cores": 1, "kind": "port",
                           "sample": "full DO-BFS per step, oracle/graphfx_port.py, 1 thread"},
          "e2e": {"value": round(v, 6), "unit": "GTEPS", "h2d_bytes_per_step": 0,
                  "d2h_bytes_per_step": 0}})


_JSON_OUT = None


def emit(out: dict) -> None:
    """The one JSON line, on the process's original stdout."""
    f = _JSON_OUT or sys.stdout
    f.write(json.dumps(out) + "\n")
    f.flush()


def main():
    global _JSON_OUT
    args = parse_args()
    # libraries (NCCL's version banner, ...) may print to fd 1: point fd 1 at
    # stderr and keep a private handle on the real stdout for the JSON line
    sys.stdout.flush()
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    if args.write_ref_cache:
        return write_reference_cache(args, args.write_ref_cache)
    dist = Dist()
    if args.impl == "reference":
        run_reference(args, dist)
    else:
        run_ours(args, dist)


if __name__ == "__main__":
    main()

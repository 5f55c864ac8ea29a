"""Benchmark harness with the reference's report schema, GPU-backed
(reference bench.py:1-203).

Same configuration object, per-run rows, means, report formats (json / csv /
table) and direction-parameter sweep as the reference.  Timing covers the
primitive's device loop only (the reference's "operator loop"); graph
loading / generation / upload and preprocessing stay outside, with
preprocessing surfaced as its own field, exactly like the reference.

Graphs: a host ``CsrGraph`` runs through the public primitives (results come
back to the host in the reference layout, as a user would see them); a
``DeviceGraph`` (e.g. ``rmat_device_graph(24, 16)``, which never exists on
the host) runs through the device entry points and summarises on the GPU.
Extra report fields (not in the reference schema, which ignores extras):
``device``, ``num_gpus``, per-run ``gteps`` (E_r / device time, the paper's
TEPS) and ``mean_gteps``.
"""
from __future__ import annotations

import csv
import io
import json
from dataclasses import dataclass, field

import numpy as np

from .graph import UNVISITED, CsrGraph, DeviceGraph, assign_random_weights
from .primitives import bc, bfs, cc, pagerank, sssp, tc
from .stats import RunStats, compute_mteps

PRIMITIVES = ("bfs", "sssp", "bc", "cc", "pagerank", "tc")
_NEEDS_SOURCE = {"bfs", "sssp", "bc"}

CSV_FIELDS = [
    "run", "source", "runtime_ms", "preprocess_ms", "iterations",
    "edges_traversed", "mteps", "direction_switches",
]


@dataclass
class BenchmarkConfig:
    primitive: str
    source: int | str = 0  # vertex id or "random"
    repetitions: int = 10
    warmup: int = 1
    seed: int = 0
    options: dict = field(default_factory=dict)

    def validate(self) -> None:
        if self.primitive not in PRIMITIVES:
            raise ValueError(f"unknown primitive {self.primitive!r}")
        if self.repetitions < 1:
            raise ValueError("repetitions must be >= 1")


def _run_host(primitive: str, g: CsrGraph, source: int, options: dict):
    if primitive == "bfs":
        return bfs(g, source, **options)
    if primitive == "sssp":
        return sssp(g, source, **options)
    if primitive == "bc":
        return bc(g, source, **options)
    if primitive == "cc":
        return cc(g, **options)
    if primitive == "pagerank":
        return pagerank(g, **options)
    if primitive == "tc":
        return tc(g, **options)
    raise ValueError(primitive)


def _summarize_host(primitive: str, result) -> dict:
    if primitive == "bfs":
        reached = int((result.labels != UNVISITED).sum())
        depth = int(result.labels[result.labels != UNVISITED].max()) if reached else 0
        return {"reached": reached, "max_depth": depth}
    if primitive == "sssp":
        return {"reached": int((result.labels != UNVISITED).sum())}
    if primitive == "bc":
        return {"max_bc": float(result.bc_values.max()) if len(result.bc_values) else 0.0}
    if primitive == "cc":
        return {"components": result.num_components}
    if primitive == "pagerank":
        return {"rank_sum": float(result.rank.sum())}
    if primitive == "tc":
        return {"triangles": result.total_triangles}
    return {}


# options of the public API that the device entry points take as well
_DEVICE_OPTS = {
    "bfs": ("direction", "idempotent", "filter_mode", "do_a", "do_b", "mu_edge_based"),
    "sssp": ("delta", "use_priority_queue"),
    "pagerank": ("damping", "epsilon", "max_iters"),
}


def _run_device(primitive: str, dg: DeviceGraph, source: int, options: dict):
    """(stats, summary) through the device entry points; results stay on the GPU."""
    from .primitives.bc import bc_device
    from .primitives.bfs import bfs_device
    from .primitives.cc import cc_device
    from .primitives.pagerank import pagerank_device
    from .primitives.sssp import sssp_device
    from .primitives.tc import tc_device
    from ._native import UNVISITED32

    opts = {k: v for k, v in options.items() if k in _DEVICE_OPTS.get(primitive, ())}
    if primitive == "bfs":
        labels, _, st = bfs_device(dg, source, **opts)
        hit = labels != UNVISITED32
        reached = int(hit.sum())
        depth = int(labels[hit].max()) if reached else 0
        return st, {"reached": reached, "max_depth": depth}
    if primitive == "sssp":
        dist, _, st = sssp_device(dg, source, **opts)
        return st, {"reached": int((dist != UNVISITED32).sum())}
    if primitive == "bc":
        values, st = bc_device(dg, [source])
        return st, {"max_bc": float(values.max())}
    if primitive == "cc":
        _, k, st = cc_device(dg)
        return st, {"components": k}
    if primitive == "pagerank":
        rank, st = pagerank_device(dg, **opts)
        return st, {"rank_sum": float(rank.sum())}
    if primitive == "tc":
        total, _, _, _, st = tc_device(dg)
        return st, {"triangles": total}
    raise ValueError(primitive)


def _device_name() -> str:
    try:
        import torch

        return torch.cuda.get_device_name()
    except Exception:
        return "cuda"


def run_benchmark(config: BenchmarkConfig, g) -> dict:
    """Warm up, run ``repetitions`` times, and report per-run stats plus
    means (reference bench.py:80-131).  With ``source="random"`` a fresh
    source is drawn per run from ``default_rng(seed)``, as the reference."""
    config.validate()
    rng = np.random.default_rng(config.seed)
    primitive = config.primitive
    on_device = isinstance(g, DeviceGraph)

    if primitive == "sssp" and not on_device and g.edge_weights is None:
        g = assign_random_weights(g, 1, 64, config.seed)
    if primitive == "sssp" and on_device and g.w is None:
        raise ValueError("sssp on a device graph needs weights (rmat_device_graph(weights=...))")

    def pick_source(run_idx: int) -> int:
        if primitive not in _NEEDS_SOURCE:
            return -1
        if config.source == "random":
            return int(rng.integers(0, g.num_vertices))
        return int(config.source)

    def once(source):
        if on_device:
            return _run_device(primitive, g, source, config.options)
        result = _run_host(primitive, g, source, config.options)
        return result.stats, _summarize_host(primitive, result)

    for _ in range(config.warmup):
        once(pick_source(-1))

    runs = []
    for i in range(config.repetitions):
        source = pick_source(i)
        stats, summary = once(source)
        stats: RunStats
        runtime = stats.total_runtime_ms if stats.total_runtime_ms else stats.device_ms
        mteps = stats.mteps if stats.mteps is not None else compute_mteps(
            primitive, stats.edges_traversed, runtime)
        gteps = None
        if primitive in ("bfs", "sssp") and stats.edges_reached > 0 and stats.device_ms:
            gteps = stats.edges_reached / (stats.device_ms * 1e6)
        runs.append({
            "run": i,
            "source": source,
            "runtime_ms": runtime,
            "preprocess_ms": stats.preprocess_ms,
            "iterations": stats.iterations,
            "edges_traversed": stats.edges_traversed,
            "mteps": mteps,
            "direction_switches": stats.direction_switches,
            "summary": summary,
            "gteps": gteps,
        })

    mteps_vals = [r["mteps"] for r in runs if r["mteps"] is not None]
    gteps_vals = [r["gteps"] for r in runs if r["gteps"] is not None]
    return {
        "primitive": primitive,
        "num_vertices": g.num_vertices,
        "num_edges": g.num_edges,
        "repetitions": config.repetitions,
        "source_mode": config.source,
        "runs": runs,
        "mean_runtime_ms": float(np.mean([r["runtime_ms"] for r in runs])),
        "mean_mteps": float(np.mean(mteps_vals)) if mteps_vals else None,
        "mean_gteps": float(np.mean(gteps_vals)) if gteps_vals else None,
        "device": _device_name(),
        "num_gpus": 1,
    }


def emit_report(report: dict, fmt: str = "table") -> str:
    """Render a report as json, csv, or a text table (reference bench.py:134-163)."""
    if fmt == "json":
        return json.dumps(report, indent=2)
    if fmt == "csv":
        out = io.StringIO()
        writer = csv.DictWriter(out, fieldnames=CSV_FIELDS, extrasaction="ignore")
        writer.writeheader()
        for row in report["runs"]:
            writer.writerow(row)
        return out.getvalue()
    if fmt == "table":
        lines = [
            f"{report['primitive']}  n={report['num_vertices']} m={report['num_edges']}",
            f"{'run':>4} {'source':>8} {'runtime_ms':>12} {'mteps':>10} {'iters':>6}",
        ]
        for r in report["runs"]:
            mteps = f"{r['mteps']:.2f}" if r["mteps"] is not None else "-"
            lines.append(f"{r['run']:>4} {r['source']:>8} {r['runtime_ms']:>12.3f} "
                         f"{mteps:>10} {r['iterations']:>6}")
        mean_mteps = f"{report['mean_mteps']:.2f}" if report["mean_mteps"] is not None else "-"
        lines.append(f"mean {'':>8} {report['mean_runtime_ms']:>12.3f} {mean_mteps:>10}")
        return "\n".join(lines) + "\n"
    raise ValueError(f"unknown output format {fmt!r}")


def run_sweep(g, do_a_grid, do_b_grid, runs: int = 25, seed: int = 0,
              **bfs_options) -> list[dict]:
    """Direction-parameter sweep (reference bench.py:166-195): for each
    (do_a, do_b) cell, BFS from the same ``runs`` random sources; mean
    runtime and MTEPS."""
    from .primitives.bfs import bfs_device

    rng = np.random.default_rng(seed)
    sources = rng.integers(0, g.num_vertices, size=runs)
    on_device = isinstance(g, DeviceGraph)
    opts = {k: v for k, v in bfs_options.items()
            if not on_device or k in _DEVICE_OPTS["bfs"]}
    rows = []
    for a in do_a_grid:
        for b in do_b_grid:
            times, rates = [], []
            for s in sources:
                if on_device:
                    _, _, st = bfs_device(g, int(s), direction="auto", do_a=float(a),
                                          do_b=float(b), **opts)
                    st.finalize(st.device_ms)
                else:
                    st = bfs(g, int(s), direction="auto", do_a=float(a), do_b=float(b),
                             **opts).stats
                times.append(st.total_runtime_ms)
                if st.mteps is not None:
                    rates.append(st.mteps)
            rows.append({"do_a": float(a), "do_b": float(b),
                         "runtime_ms": float(np.mean(times)),
                         "mteps": float(np.mean(rates)) if rates else None})
    return rows


def sweep_to_csv(rows: list[dict]) -> str:
    out = io.StringIO()
    writer = csv.DictWriter(out, fieldnames=["do_a", "do_b", "runtime_ms", "mteps"])
    writer.writeheader()
    for row in rows:
        writer.writerow(row)
    return out.getvalue()

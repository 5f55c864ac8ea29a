"""Golden-vector generator: runs the REFERENCE graphfx package (imported
read-only from /root/reference/pkg/src) and writes fixtures under
tests/golden/.  TEST INFRASTRUCTURE ONLY -- this script runs in the build
container (where /root/reference exists); its outputs are committed so the
GPU box never needs the reference.

Usage:  python oracle/make_golden.py kat            # mini suite + KAT graphs
        GOLDEN_S24_FULL=1 python oracle/make_golden.py rmat 24   # + SSSP / CC / PageRank at s24
        python oracle/make_golden.py cache          # reference-written CSR cache files
        python oracle/make_golden.py rmat S [S ...] # R-MAT scale S, ef16, seed 0

What is recorded (all arrays little-endian, hashes are SHA-256 of the raw
int64 bytes exactly as the reference returns them):
  * the canonical CSR of generate_rmat(S,16,seed=0) -> coo_to_csr(make_undirected)
    (row_offsets / column_indices / assign_random_weights(g,1,64,seed=0) hashes)
  * bfs(g,0) push labels + per-level frontier sizes; bfs(direction="auto")
    direction trace (n_f, n_u, m_f, m_u, decision) -- reference primitives/bfs.py:90-156
  * sssp(gw,0,delta=32) and default-delta labels -- primitives/sssp.py:41-121
  * cc(g) labels canonicalised to min-id -- primitives/cc.py:23-82
  * pagerank(g, epsilon=0, max_iters=20) ranks -- primitives/pagerank.py:30-91
  * bc(g, 0) -- primitives/bc.py:32-116
  * tc(g) total + per_edge_counts -- primitives/tc.py:27-86
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

REF_SRC = "/root/reference/pkg/src"
REF_TESTS = "/root/reference/pkg/tests"
sys.dont_write_bytecode = True
sys.path.insert(0, REF_SRC)
sys.path.insert(0, REF_TESTS)

import graphfx as gx  # noqa: E402  (the reference)

OUT = Path(__file__).resolve().parent.parent / "tests" / "golden"


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def canon_cc(comp: np.ndarray) -> np.ndarray:
    n = len(comp)
    first = np.full(n, n, dtype=np.int64)
    np.minimum.at(first, comp, np.arange(n, dtype=np.int64))
    return first[comp]


def level_sizes(labels: np.ndarray) -> list[int]:
    reached = labels[labels != gx.UNVISITED]
    return np.bincount(reached).tolist() if len(reached) else []


def trace_rows(trace):
    return [[t["iteration"], t["mode_before"], int(t["n_f"]), int(t["n_u"]),
             float(t["m_f"]), float(t["m_u"]), t["decision"]] for t in trace]


def run_kat():
    from _graphs import build_mini_suite, complete_graph, path_graph, star_graph

    graphs = []
    for sg in build_mini_suite(12):
        graphs.append((sg.name, sg.g, sg.weighted, sg.source))
    for name, g in (("star3", star_graph(3)), ("path5", path_graph(5)),
                    ("k4", complete_graph(4)), ("k12", complete_graph(12))):
        graphs.append((name, g, gx.assign_random_weights(g, 1, 64, seed=3), 0))
    # directed R-MAT variants (reference test_primitives.py:231-269)
    for seed in range(3):
        g = gx.coo_to_csr(gx.generate_rmat(6, 5, seed=seed))
        gw = gx.assign_random_weights(g, 1, 32, seed=seed)
        graphs.append((f"rmat-directed-{seed}", gw, gw, 0))

    arrays = {}
    meta = []
    for i, (name, g, gw, src) in enumerate(graphs):
        p = f"g{i}_"
        arrays[p + "row"] = g.row_offsets
        arrays[p + "col"] = g.column_indices
        arrays[p + "w"] = gw.edge_weights
        b = gx.bfs(g, src)
        arrays[p + "bfs"] = b.labels
        bd = gx.bfs(g, src, direction="auto")
        s = gx.sssp(gw, src)
        arrays[p + "sssp"] = s.labels
        arrays[p + "bc"] = gx.bc(g, src).bc_values
        arrays[p + "pr4"] = gx.pagerank(g, epsilon=0.0, max_iters=4).rank
        arrays[p + "pr_eps"] = gx.pagerank(g, epsilon=1e-3, max_iters=50).rank
        rec = {"name": name, "n": g.num_vertices, "m": g.num_edges,
               "undirected": bool(g.undirected), "source": int(src),
               "bfs_auto_trace": trace_rows(bd.stats.direction_trace)}
        if g.undirected:
            arrays[p + "cc"] = canon_cc(gx.cc(g).component)
            t = gx.tc(g)
            arrays[p + "tc_counts"] = t.per_edge_counts
            arrays[p + "tc_src"] = t.oriented_src
            arrays[p + "tc_dst"] = t.oriented_dst
            rec["tc_total"] = int(t.total_triangles)
        meta.append(rec)
    OUT.mkdir(parents=True, exist_ok=True)
    np.savez_compressed(OUT / "kat_graphs.npz", **arrays)
    (OUT / "kat_graphs.json").write_text(json.dumps(
        {"numpy": np.__version__, "graphs": meta}, indent=1))
    print("kat done", len(graphs))


def run_suite(stride: int = 5):
    """Every stride-th graph of the reference acceptance suite
    (pkg/tests/_graphs.py:55-91 build_suite(per_family=200, seed=20240)),
    with the outputs acceptance criterion 1 compares (test_acceptance.py:89-109)
    plus the DO trace (criterion 3) and idempotent labels (criterion 6)."""
    from _graphs import build_suite

    suite = build_suite(per_family=200)
    picked = [sg for i, sg in enumerate(suite) if i % stride == 0 or sg.g.num_vertices >= 2048]
    arrays, meta = {}, []
    for i, sg in enumerate(picked):
        p = f"g{i}_"
        g, gw, src = sg.g, sg.weighted, sg.source
        arrays[p + "row"] = g.row_offsets.astype(np.int64)
        arrays[p + "col"] = g.column_indices.astype(np.int32)
        arrays[p + "w"] = gw.edge_weights.astype(np.int8)
        b = gx.bfs(g, src)
        arrays[p + "bfs"] = b.labels
        bd = gx.bfs(g, src, direction="auto")
        arrays[p + "sssp"] = gx.sssp(gw, src).labels
        arrays[p + "bc"] = gx.bc(g, src).bc_values
        arrays[p + "cc"] = canon_cc(gx.cc(g).component)
        arrays[p + "pr4"] = gx.pagerank(g, epsilon=0.0, max_iters=4).rank
        t = gx.tc(g)
        arrays[p + "tc_counts"] = t.per_edge_counts.astype(np.int32)
        meta.append({"name": sg.name, "family": sg.family, "n": g.num_vertices,
                     "m": g.num_edges, "source": int(src), "tc_total": int(t.total_triangles),
                     "bfs_auto_trace": trace_rows(bd.stats.direction_trace)})
    OUT.mkdir(parents=True, exist_ok=True)
    np.savez_compressed(OUT / "suite_graphs.npz", **arrays)
    (OUT / "suite_graphs.json").write_text(json.dumps(
        {"numpy": np.__version__, "stride": stride, "graphs": meta}))
    print("suite done", len(picked))


def run_rmat(scale: int):
    t0 = time.time()
    rec = {"scale": scale, "edge_factor": 16, "seed": 0, "numpy": np.__version__}
    arrays = {}
    small = scale <= 16
    coo = gx.generate_rmat(scale, 16, seed=0)
    rec["gen_s"] = time.time() - t0
    g = gx.coo_to_csr(coo, make_undirected=True)
    del coo
    rec["csr_s"] = time.time() - t0
    n, m = g.num_vertices, g.num_edges
    rec.update(n=n, m=m, row_sha=sha(g.row_offsets), col_sha=sha(g.column_indices),
               isolated=int((g.degrees == 0).sum()), max_deg=int(g.degrees.max()))
    gw = gx.assign_random_weights(g, 1, 64, seed=0)
    rec["w_sha"] = sha(gw.edge_weights)
    if small:
        arrays["row"] = g.row_offsets
        arrays["col"] = g.column_indices.astype(np.int32)
        arrays["w"] = gw.edge_weights.astype(np.int8)

    def save():
        OUT.mkdir(parents=True, exist_ok=True)
        (OUT / f"rmat_s{scale}.json").write_text(json.dumps(rec, indent=1))

    save()
    b = gx.bfs(g, 0)
    rec["bfs_sha"] = sha(b.labels)
    rec["bfs_levels"] = level_sizes(b.labels)
    rec["bfs_push_ms"] = b.stats.total_runtime_ms
    rec["bfs_edges_traversed"] = int(b.stats.edges_traversed)
    reached = b.labels != gx.UNVISITED
    rec["E_r"] = int(g.degrees[reached].sum())
    if small:
        arrays["bfs"] = b.labels
    bd = gx.bfs(g, 0, direction="auto")
    assert np.array_equal(bd.labels, b.labels)
    rec["bfs_auto_trace"] = trace_rows(bd.stats.direction_trace)
    rec["bfs_auto_ms"] = bd.stats.total_runtime_ms
    save()
    if scale >= 24 and not os.environ.get("GOLDEN_S24_FULL"):
        print("s24: graph + bfs only", time.time() - t0)
        return
    for delta in (32, None):
        s = gx.sssp(gw, 0, delta=delta)
        key = "sssp_d32" if delta == 32 else "sssp_default"
        rec[key + "_sha"] = sha(s.labels)
        rec[key + "_ms"] = s.stats.total_runtime_ms
        if small:
            arrays[key] = s.labels
    save()
    if scale >= 24:  # C3 / M3 pins: SSSP above, then CC and PageRank (BC/TC: C4 is s22)
        c = canon_cc(gx.cc(g).component)
        rec["cc_canon_sha"] = sha(c)
        rec["cc_num"] = int(len(np.unique(c)))
        save()
        pr = gx.pagerank(g, epsilon=0.0, max_iters=20).rank
        rec["pr20_sum"] = float(pr.sum())
        idx = np.random.default_rng(2).choice(n, 4096, replace=False)
        arrays["pr_idx"] = idx
        arrays["pr_vals"] = pr[idx]
        rec["total_s"] = time.time() - t0
        save()
        np.savez_compressed(OUT / f"rmat_s{scale}.npz", **arrays)
        print("done scale", scale, time.time() - t0)
        return
    c = canon_cc(gx.cc(g).component)
    rec["cc_canon_sha"] = sha(c)
    rec["cc_num"] = int(len(np.unique(c)))
    if small:
        arrays["cc"] = c
    save()
    bcv = gx.bc(g, 0).bc_values
    rec["bc_sum"] = float(bcv.sum())
    rec["bc_max"] = float(bcv.max())
    if scale <= 18:
        arrays["bc"] = bcv
    else:
        idx = np.random.default_rng(1).choice(n, 4096, replace=False)
        arrays["bc_idx"] = idx
        arrays["bc_vals"] = bcv[idx]
    save()
    pr = gx.pagerank(g, epsilon=0.0, max_iters=20).rank
    rec["pr20_sum"] = float(pr.sum())
    if scale <= 18:
        arrays["pr20"] = pr
    else:
        idx = np.random.default_rng(2).choice(n, 4096, replace=False)
        arrays["pr_idx"] = idx
        arrays["pr_vals"] = pr[idx]
    save()
    if scale <= 20:
        t = gx.tc(g)
        rec["tc_total"] = int(t.total_triangles)
        rec["tc_counts_sha"] = sha(t.per_edge_counts)
        rec["tc_src_sha"] = sha(t.oriented_src)
        rec["tc_dst_sha"] = sha(t.oriented_dst)
        if small:
            arrays["tc_counts"] = t.per_edge_counts.astype(np.int32)
    rec["total_s"] = time.time() - t0
    save()
    if arrays:
        np.savez_compressed(OUT / f"rmat_s{scale}.npz", **arrays)
    print("done scale", scale, time.time() - t0)


def run_cache():
    """Binary CSR cache files written by the reference's save_csr_cache
    (io.py:121-130): an undirected weighted R-MAT s8 graph and a directed
    unweighted one, plus the arrays they hold (tests/test_io_cache.py)."""
    from graphfx.io import save_csr_cache

    g = gx.coo_to_csr(gx.generate_rmat(8, 8, seed=3), make_undirected=True)
    gw = gx.assign_random_weights(g, 1, 64, 0)
    save_csr_cache(gw, OUT / "cache_rmat8_w.gfxcsr")
    coo = gx.generate_rmat(7, 4, seed=5)
    gd = gx.coo_to_csr(coo)
    save_csr_cache(gd, OUT / "cache_rmat7_dir.gfxcsr")
    np.savez_compressed(OUT / "cache_arrays.npz", w_row=gw.row_offsets, w_col=gw.column_indices,
                        w_w=gw.edge_weights, d_row=gd.row_offsets, d_col=gd.column_indices,
                        d_n=np.array([gd.num_vertices]), w_n=np.array([gw.num_vertices]))
    print("cache files written", gw.num_edges, gd.num_edges)


if __name__ == "__main__":
    os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
    if sys.argv[1] == "kat":
        run_kat()
    elif sys.argv[1] == "cache":
        run_cache()
    elif sys.argv[1] == "suite":
        run_suite(int(sys.argv[2]) if len(sys.argv) > 2 else 5)
    else:
        for s in sys.argv[2:]:
            run_rmat(int(s))

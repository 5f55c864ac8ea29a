"""GPU-backed bench harness and CLI with the reference's report schema and
exit codes (reference tests test_cli.py,
test_stats_bench.py)."""
import json
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT


def run_cli(*args):
    return subprocess.run([sys.executable, "-m", "paper_1701_01170_b200.cli", *args],
                          capture_output=True, text=True, timeout=300, cwd=ROOT)


# ---- no GPU needed: argument / data errors are caught before any device work
def test_unknown_subcommand():
    assert run_cli("mst", "--graph", "rmat:4,4").returncode == 2


def test_bad_graph_spec_is_config_error():
    assert run_cli("bfs", "--graph", "rmat:nope").returncode == 2
    assert run_cli("bfs", "--graph", "rgg:6").returncode == 2


def test_missing_file_is_data_error():
    assert run_cli("bfs", "--graph", "/does/not/exist.gfxcsr").returncode == 3


def test_malformed_file_is_data_error(tmp_path):
    bad = tmp_path / "bad.mtx"
    bad.write_text("%%MatrixMarket matrix coordinate pattern general\n2 2 1\nx y\n")
    assert run_cli("bfs", "--graph", str(bad)).returncode == 3
    trunc = tmp_path / "trunc.gfxcsr"
    trunc.write_bytes((ROOT / "tests" / "golden" / "cache_rmat8_w.gfxcsr").read_bytes()[:100])
    assert run_cli("bfs", "--graph", str(trunc)).returncode == 3


def _report():
    return {"primitive": "bfs", "num_vertices": 4, "num_edges": 6, "repetitions": 2,
            "source_mode": 0, "mean_runtime_ms": 1.5, "mean_mteps": 2.0,
            "runs": [{"run": i, "source": 0, "runtime_ms": 1.0 + i, "preprocess_ms": 0.0,
                      "iterations": 2, "edges_traversed": 6, "mteps": 2.0,
                      "direction_switches": 0, "summary": {}} for i in range(2)]}


def test_emit_formats():
    """reference test_stats_bench.py:102-120"""
    from paper_1701_01170_b200.bench import CSV_FIELDS, emit_report

    r = _report()
    assert json.loads(emit_report(r, "json"))["primitive"] == "bfs"
    assert emit_report(r, "csv").splitlines()[0] == ",".join(CSV_FIELDS)
    t = emit_report(r, "table")
    assert "runtime_ms" in t and "mteps" in t
    with pytest.raises(ValueError):
        emit_report(r, "xml")


def test_unknown_primitive_rejected():
    from paper_1701_01170_b200.bench import BenchmarkConfig

    with pytest.raises(ValueError):
        BenchmarkConfig("mst").validate()
    with pytest.raises(ValueError):
        BenchmarkConfig("bfs", repetitions=0).validate()


# ---- on the GPU
@pytest.mark.gpu
def test_cli_runs(tmp_path):
    p = run_cli("bfs", "--graph", "rmat:6,4", "--iters", "2", "--warmup", "0")
    assert p.returncode == 0, p.stderr
    assert "runtime_ms" in p.stdout
    p = run_cli("bfs", "--graph", "rmat:5,4", "--iters", "1", "--warmup", "0", "--output", "json",
                "--direction", "auto")
    assert p.returncode == 0, p.stderr
    rep = json.loads(p.stdout)
    assert rep["primitive"] == "bfs" and len(rep["runs"]) == 1 and rep["num_gpus"] == 1
    p = run_cli("sssp", "--graph", "rmat:6,4", "--iters", "1", "--warmup", "0", "--output", "json")
    assert p.returncode == 0, p.stderr
    assert json.loads(p.stdout)["mean_mteps"] is None
    for prim in ("tc", "cc", "pagerank", "bc"):
        p = run_cli(prim, "--graph", "rmat:6,4", "--iters", "1", "--warmup", "0", "--output",
                    "json")
        assert p.returncode == 0, (prim, p.stderr)
    p = run_cli("sweep", "--graph", "rmat:5,4", "--runs", "1", "--do-a-grid", "1e-3",
                "--do-b-grid", "0.2")
    assert p.returncode == 0, p.stderr
    assert p.stdout.splitlines()[0] == "do_a,do_b,runtime_ms,mteps"
    out = tmp_path / "r.json"
    p = run_cli("bfs", "--graph", "rmat:4,4", "--iters", "1", "--warmup", "0", "--output", "json",
                "--output-file", str(out))
    assert p.returncode == 0 and json.loads(out.read_text())["primitive"] == "bfs"
    assert run_cli("bfs", "--graph", "rmat:4,4", "--source", "9999").returncode == 2
    cache = ROOT / "tests" / "golden" / "cache_rmat8_w.gfxcsr"
    p = run_cli("sssp", "--graph", str(cache), "--iters", "1", "--warmup", "0", "--output", "json")
    assert p.returncode == 0, p.stderr
    # a weight range that is not a power of two (numpy's rejection
    # sampler) works like the reference CLI
    p = run_cli("sssp", "--graph", "rmat:6,4", "--weight-range", "1,100", "--iters", "1",
                "--warmup", "0", "--output", "json")
    assert p.returncode == 0, p.stderr


@pytest.mark.gpu
def test_weights_non_power_of_two_range_match_reference_rng():
    import paper_1701_01170_b200 as gfx
    from paper_1701_01170_b200.generators import rmat_device_graph

    dg = rmat_device_graph(8, 8, 3, weights=(1, 100), weight_seed=5)
    host = gfx.coo_to_csr(gfx.generate_rmat(8, 8, seed=3), make_undirected=True)
    want = gfx.assign_random_weights(host, 1, 100, seed=5).edge_weights
    assert np.array_equal(dg.w.cpu().numpy().astype(np.int64), want)


@pytest.mark.gpu
def test_harness_matches_reference_semantics():
    """reference test_stats_bench.py:60-91: repetition count, deterministic
    random sources, sssp auto-weights with null MTEPS; summaries equal on
    the host-graph and device-graph paths."""
    import numpy as np

    from conftest import rmat_golden
    import paper_1701_01170_b200 as gfx
    from paper_1701_01170_b200.bench import BenchmarkConfig, run_benchmark
    from paper_1701_01170_b200.generators import rmat_device_graph

    rec, arrays = rmat_golden(16)
    g = gfx.CsrGraph(rec["n"], arrays["row"], arrays["col"].astype(np.int64), undirected=True)
    r = run_benchmark(BenchmarkConfig("bfs", repetitions=3, warmup=0), g)
    assert len(r["runs"]) == 3 and r["runs"][0]["summary"]["reached"] == 46694
    a = run_benchmark(BenchmarkConfig("bfs", source="random", repetitions=3, seed=7), g)
    b = run_benchmark(BenchmarkConfig("bfs", source="random", repetitions=3, seed=7), g)
    assert [x["source"] for x in a["runs"]] == [x["source"] for x in b["runs"]]
    s = run_benchmark(BenchmarkConfig("sssp", repetitions=1, warmup=0), g)
    assert s["mean_mteps"] is None
    dg = rmat_device_graph(16, 16, 0)
    d = run_benchmark(BenchmarkConfig("bfs", repetitions=2, warmup=1,
                                      options={"direction": "auto"}), dg)
    assert d["runs"][0]["summary"] == {"reached": 46694, "max_depth": 4}
    assert d["mean_gteps"] > 0

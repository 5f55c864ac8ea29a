"""The CPU oracle (oracle/) pinned against golden vectors produced by running
the reference itself (oracle/make_golden.py).  No GPU needed."""
import numpy as np
import pytest

from conftest import rmat_golden, sha
from oracle import c_oracle
from oracle import graphfx_port as port

UNV = np.iinfo(np.int64).max


@pytest.mark.parametrize("scale", [10, 12, 14, 16])
def test_rmat_csr_matches_reference_hashes(scale):
    rec, arrays = rmat_golden(scale)
    row, col = port.rmat_csr(scale, 16, 0)
    assert len(row) - 1 == rec["n"] and len(col) == rec["m"]
    assert sha(row) == rec["row_sha"]
    assert sha(col) == rec["col_sha"]
    w = port.assign_random_weights(row, col, 1, 64, 0)
    assert sha(w) == rec["w_sha"]


def test_kat_oracle_port(kat):
    for d in kat:
        row, col = d["row"].astype(np.int64), d["col"].astype(np.int64)
        w = d["w"].astype(np.int64)
        src = d["source"]
        labels, preds, trace, _ = port.bfs(row, col, src)
        assert np.array_equal(labels, d["bfs"]), d["name"]
        la, _, tr, _ = port.bfs(row, col, src, direction="auto")
        assert np.array_equal(la, d["bfs"]), d["name"]
        ref_tr = [[t["iteration"], t["mode_before"], t["n_f"], t["n_u"], t["m_f"], t["m_u"],
                   t["decision"]] for t in tr]
        assert ref_tr == [list(x) for x in d["bfs_auto_trace"]], d["name"]
        dist, _, _ = port.sssp(row, col, w, src)
        assert np.array_equal(dist, d["sssp"]), d["name"]
        assert np.allclose(port.bc(row, col, src), d["bc"], rtol=1e-12, atol=1e-12), d["name"]
        assert np.abs(port.pagerank(row, col, 0.85, 0.0, 4) - d["pr4"]).sum() < 1e-12
        assert np.abs(port.pagerank(row, col, 0.85, 1e-3, 50) - d["pr_eps"]).sum() < 1e-12
        if d["undirected"]:
            assert np.array_equal(port.cc(row, col), d["cc"]), d["name"]
            total, counts, osrc, odst = port.tc(row, col)
            assert total == d["tc_total"]
            assert np.array_equal(counts, d["tc_counts"])
            assert np.array_equal(osrc, d["tc_src"]) and np.array_equal(odst, d["tc_dst"])


def test_kat_c_oracle(kat):
    for d in kat:
        row, col = d["row"].astype(np.int64), d["col"].astype(np.int64)
        src = d["source"]
        assert np.array_equal(c_oracle.bfs(row, col, src), d["bfs"]), d["name"]
        assert np.array_equal(c_oracle.dijkstra(row, col, d["w"], src), d["sssp"]), d["name"]
        rrow, rcol, _ = port.csc(row, col)
        assert np.allclose(c_oracle.bc(row, col, rrow, rcol, src), d["bc"], rtol=1e-9,
                           atol=1e-12), d["name"]
        assert np.abs(c_oracle.pagerank(row, col, rrow, rcol, 0.85, 4) - d["pr4"]).sum() < 1e-12
        if d["undirected"]:
            comp, k = c_oracle.cc(row, col)
            assert np.array_equal(comp, d["cc"]), d["name"]
            total, counts, osrc, odst = c_oracle.tc(row, col)
            assert total == d["tc_total"] and np.array_equal(counts, d["tc_counts"])
            assert np.array_equal(odst, d["tc_dst"])


def test_s16_outputs_oracles():
    rec, arrays = rmat_golden(16)
    row, col = arrays["row"], arrays["col"].astype(np.int64)
    labels = c_oracle.bfs(row, col, 0)
    assert np.array_equal(labels, arrays["bfs"])
    assert sha(labels) == rec["bfs_sha"]
    lp, _, trace, _ = port.bfs(row, col, 0, direction="auto")
    assert np.array_equal(lp, arrays["bfs"])
    assert [[t["iteration"], t["mode_before"], t["n_f"], t["n_u"], t["m_f"], t["m_u"],
             t["decision"]] for t in trace] == [list(x) for x in rec["bfs_auto_trace"]]
    w = arrays["w"].astype(np.int64)
    assert np.array_equal(c_oracle.dijkstra(row, col, w, 0), arrays["sssp_d32"])
    comp, k = c_oracle.cc(row, col)
    assert np.array_equal(comp, arrays["cc"]) and k == rec["cc_num"]
    total, counts, _, _ = c_oracle.tc(row, col)
    assert total == rec["tc_total"] and np.array_equal(counts, arrays["tc_counts"])


def test_suite_c_oracle(suite):
    """C oracles vs the reference on its acceptance-suite graphs."""
    for d in suite:
        row, col = d["row"], d["col"].astype(np.int64)
        assert np.array_equal(c_oracle.bfs(row, col, d["source"]), d["bfs"]), d["name"]
        assert np.array_equal(c_oracle.dijkstra(row, col, d["w"], d["source"]), d["sssp"])
        comp, _ = c_oracle.cc(row, col)
        assert np.array_equal(comp, d["cc"]), d["name"]
        total, counts, _, _ = c_oracle.tc(row, col)
        assert total == d["tc_total"] and np.array_equal(counts, d["tc_counts"]), d["name"]

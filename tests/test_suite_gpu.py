"""Acceptance-suite replay (reference test_acceptance.py criteria 1, 3, 6 on
the reference's own build_suite graphs): every primitive on the GPU against
the reference's outputs."""
import numpy as np
import pytest

from conftest import host_graph

pytestmark = pytest.mark.gpu


def _rows(stats):
    return [[t["iteration"], t["mode_before"], t["n_f"], t["n_u"], t["m_f"], t["m_u"],
             t["decision"]] for t in stats.direction_trace]


def test_suite_all_primitives(suite):
    import paper_1701_01170_b200 as gfx

    fams = {}
    for d in suite:
        fams[d["family"]] = fams.get(d["family"], 0) + 1
        g = host_graph(d)
        gw = host_graph(d, weighted=True)
        src = d["source"]
        assert np.array_equal(gfx.bfs(g, src).labels, d["bfs"]), d["name"]
        r = gfx.bfs(g, src, direction="auto")
        assert np.array_equal(r.labels, d["bfs"]), d["name"]
        assert _rows(r.stats) == [list(x) for x in d["bfs_auto_trace"]], d["name"]  # criterion 3
        assert np.array_equal(gfx.bfs(g, src, idempotent=True).labels, d["bfs"])   # criterion 6
        assert np.array_equal(gfx.sssp(gw, src).labels, d["sssp"]), d["name"]
        assert np.allclose(gfx.bc(g, src).bc_values, d["bc"], rtol=1e-5, atol=1e-9), d["name"]
        assert np.array_equal(gfx.cc(g).component, d["cc"]), d["name"]
        assert np.abs(gfx.pagerank(g, epsilon=0.0, max_iters=4).rank - d["pr4"]).sum() <= 1e-6
        t = gfx.tc(g)
        assert t.total_triangles == d["tc_total"], d["name"]
        assert np.array_equal(t.per_edge_counts, d["tc_counts"]), d["name"]
    assert set(fams) == {"er", "rmat", "rgg"}

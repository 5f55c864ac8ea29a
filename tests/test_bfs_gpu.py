"""BFS on the GPU vs the reference's golden outputs and the CPU oracle."""
import numpy as np
import pytest

from _checks import valid_bfs_preds
from conftest import host_graph, rmat_golden, sha

pytestmark = pytest.mark.gpu


def _trace_rows(stats):
    return [[t["iteration"], t["mode_before"], t["n_f"], t["n_u"], t["m_f"], t["m_u"],
             t["decision"]] for t in stats.direction_trace]


def test_kat_bfs_all_modes(kat):
    import paper_1701_01170_b200 as gfx
    from paper_1701_01170_b200 import FilterMode

    for d in kat:
        g = host_graph(d)
        src = d["source"]
        for direction in ("push", "pull", "auto"):
            r = gfx.bfs(g, src, direction=direction)
            assert np.array_equal(r.labels, d["bfs"]), (d["name"], direction)
            assert valid_bfs_preds(g.row_offsets, g.column_indices, r.labels, r.preds, src)
        r = gfx.bfs(g, src, direction="auto")
        assert _trace_rows(r.stats) == [list(x) for x in d["bfs_auto_trace"]], d["name"]
        for fm in (FilterMode.EXACT, FilterMode.INEXACT):
            r = gfx.bfs(g, src, idempotent=True, filter_mode=fm)
            assert np.array_equal(r.labels, d["bfs"]), (d["name"], "idempotent", fm)


def test_reference_kats():
    """reference test_primitives.py:29-45 (star, singleton, forced pull)."""
    import paper_1701_01170_b200 as gfx

    star = gfx.coo_to_csr(gfx.CooGraph(4, np.array([0, 0, 0]), np.array([1, 2, 3])),
                          make_undirected=True)
    assert gfx.bfs(star, 0).labels.tolist() == [0, 1, 1, 1]
    single = gfx.coo_to_csr(gfx.CooGraph(1, np.array([], dtype=np.int64),
                                         np.array([], dtype=np.int64)))
    assert gfx.bfs(single, 0).labels.tolist() == [0]
    path = gfx.coo_to_csr(gfx.CooGraph(3, np.array([0, 1]), np.array([1, 2])),
                          make_undirected=True)
    assert gfx.bfs(path, 0, direction="pull").labels.tolist() == [0, 1, 2]
    with pytest.raises(ValueError):
        gfx.bfs(star, 5)
    with pytest.raises(ValueError):
        gfx.bfs(star, 0, direction="sideways")
    with pytest.raises(ValueError):
        gfx.bfs(star, 0, direction="auto", do_a=0.0)


@pytest.mark.parametrize("direction", ["push", "auto", "pull"])
def test_s16_golden(direction):
    import paper_1701_01170_b200 as gfx

    rec, arrays = rmat_golden(16)
    g = gfx.CsrGraph(rec["n"], arrays["row"], arrays["col"].astype(np.int64), undirected=True)
    r = gfx.bfs(g, 0, direction=direction)
    assert sha(r.labels) == rec["bfs_sha"]
    assert valid_bfs_preds(g.row_offsets, g.column_indices, r.labels, r.preds, 0)
    assert r.stats.edges_reached == rec["E_r"]
    if direction == "push":
        assert r.stats.edges_traversed == rec["bfs_edges_traversed"]
        assert [it.frontier_in for it in r.stats.per_iteration] == rec["bfs_levels"]
    if direction == "auto":
        assert _trace_rows(r.stats) == [list(x) for x in rec["bfs_auto_trace"]]

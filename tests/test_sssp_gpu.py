"""SSSP on the GPU vs reference goldens, Dijkstra and property checks."""
import numpy as np
import pytest

from _checks import valid_sssp_preds
from conftest import host_graph, rmat_golden, sha

pytestmark = pytest.mark.gpu


def test_kat_sssp(kat):
    import paper_1701_01170_b200 as gfx

    for d in kat:
        g = host_graph(d, weighted=True)
        src = d["source"]
        for kw in ({}, {"delta": 1}, {"delta": 7}, {"delta": 1000}, {"use_priority_queue": False}):
            r = gfx.sssp(g, src, **kw)
            assert np.array_equal(r.labels, d["sssp"]), (d["name"], kw)
            assert valid_sssp_preds(g.row_offsets, g.column_indices, g.edge_weights, r.labels,
                                    r.preds, src), (d["name"], kw)


def test_reference_kats():
    """reference test_primitives.py:73-114."""
    import paper_1701_01170_b200 as gfx

    g = gfx.coo_to_csr(gfx.CooGraph(3, np.array([0, 1]), np.array([1, 2])), make_undirected=True)
    w = np.zeros(g.num_edges, dtype=np.int64)
    s, d = g.edge_sources(), g.column_indices
    w[np.minimum(s, d) == 0] = 5
    w[np.minimum(s, d) == 1] = 7
    g.edge_weights = w
    assert gfx.sssp(g, 0).labels.tolist() == [0, 5, 12]
    g2 = gfx.assign_random_weights(
        gfx.coo_to_csr(gfx.CooGraph(4, np.array([1, 2]), np.array([2, 3])), make_undirected=True),
        1, 9, seed=0)
    r = gfx.sssp(g2, 0)
    assert r.labels[0] == 0 and np.all(r.labels[1:] == gfx.UNVISITED)
    star = gfx.coo_to_csr(gfx.CooGraph(5, np.array([0, 0, 0, 0]), np.array([1, 2, 3, 4])),
                          make_undirected=True)
    with pytest.raises(ValueError):
        gfx.sssp(star, 0)
    unit = gfx.assign_random_weights(star, 1, 1, seed=0)
    assert np.array_equal(gfx.sssp(unit, 0).labels, gfx.bfs(unit, 0).labels)
    with pytest.raises(ValueError):
        gfx.sssp(unit, 9)


@pytest.mark.parametrize("delta", [32, None])
def test_s16_golden(delta):
    import paper_1701_01170_b200 as gfx

    rec, arrays = rmat_golden(16)
    g = gfx.CsrGraph(rec["n"], arrays["row"], arrays["col"].astype(np.int64),
                     arrays["w"].astype(np.int64), undirected=True)
    r = gfx.sssp(g, 0, delta=delta)
    key = "sssp_d32" if delta == 32 else "sssp_default"
    assert sha(r.labels) == rec[key + "_sha"]
    assert valid_sssp_preds(g.row_offsets, g.column_indices, g.edge_weights, r.labels, r.preds, 0)


@pytest.mark.parametrize("scale", [20, 22])
def test_device_graph_golden(scale):
    """C2 config: SSSP on R-MAT s22 + weights 1..64 (GPU-built, bit-exact input)."""
    from paper_1701_01170_b200._results import labels_to_host
    from paper_1701_01170_b200.generators import rmat_device_graph
    from paper_1701_01170_b200.primitives.sssp import sssp_device

    from paper_1701_01170_b200._results import preds_to_host

    rec, _ = rmat_golden(scale)
    dg = rmat_device_graph(scale, 16, 0, weights=(1, 64), weight_seed=0)
    host = (dg.row.cpu().numpy(), dg.col.cpu().numpy().astype(np.int64),
            dg.w.cpu().numpy().astype(np.int64))
    for delta, key in ((32, "sssp_d32"), (None, "sssp_default")):
        dist, preds, st = sssp_device(dg, 0, delta=delta)
        lab = labels_to_host(dist)
        assert sha(lab) == rec[key + "_sha"], (scale, delta)
        # preds recovered from the final distances (undirected path)
        assert valid_sssp_preds(*host, lab, preds_to_host(preds), 0), (scale, delta)


@pytest.mark.parametrize("delta", [4, 32, None])
def test_device_loop_equals_host_loop(delta, monkeypatch):
    """The device-resident loop (one cooperative launch; the default for
    delta <= 8) and the host-driven loop give the same distances; both
    equal the reference golden; the loops agree on the work done per
    iteration when the iteration sequence is the same length."""
    from paper_1701_01170_b200._results import labels_to_host, preds_to_host
    from paper_1701_01170_b200.generators import rmat_device_graph
    from paper_1701_01170_b200.primitives.sssp import sssp_device

    rec, _ = rmat_golden(20)
    dg = rmat_device_graph(20, 16, 0, weights=(1, 64), weight_seed=0)
    out = {}
    for loop in ("device", "host"):
        monkeypatch.setenv("GFX_SSSP_LOOP", loop)
        dist, preds, st = sssp_device(dg, 0, delta=delta)
        out[loop] = (labels_to_host(dist), preds_to_host(preds), st)
    assert sha(out["device"][0]) == rec["sssp_d32_sha"]
    assert np.array_equal(out["device"][0], out["host"][0])
    g = dg.to_host()
    assert valid_sssp_preds(g.row_offsets, g.column_indices, g.edge_weights, out["device"][0],
                            out["device"][1], 0)
    st = out["device"][2]
    assert st.iterations > 0 and st.edges_traversed >= st.edges_reached


@pytest.mark.parametrize("delta,window", [(1, "4"), (3, "1"), (2, "0"), (50, "4")])
def test_two_level_far_pile_wide_weights(delta, window, monkeypatch):
    """the device loop's two-level far pile (soon / later piles, re-split
    when the threshold passes the later pile's smallest key) on a graph whose
    keys span far more than the window: weights 1..1000 at small delta, so
    the later pile is appended, re-split and rebuilt many times; distances
    equal the numpy port of sssp.py:41-121 (GFX_SSSP_WIN: window in deltas,
    0 = one far pile)"""
    import paper_1701_01170_b200 as gfx
    from oracle import graphfx_port as port

    monkeypatch.setenv("GFX_SSSP_WIN", window)
    row, col = port.rmat_csr(12, 8, 3)
    w = port.assign_random_weights(row, col, 1, 1000, 5)
    g = gfx.CsrGraph(len(row) - 1, row, col, w, undirected=True)
    want = port.sssp(row, col, w, 0, delta=delta)[0]
    r = gfx.sssp(g, 0, delta=delta)
    assert np.array_equal(r.labels, want)
    assert valid_sssp_preds(g.row_offsets, g.column_indices, g.edge_weights, r.labels, r.preds, 0)

"""BFS on the GPU vs the reference's golden outputs and the CPU oracle."""
import numpy as np
import pytest

from _checks import valid_bfs_preds
from conftest import host_graph, rmat_golden, sha

pytestmark = pytest.mark.gpu


def _trace_rows(stats):
    """reference direction_trace rows: (iteration, mode_before, n_f, n_u, m_f, m_u, decision)"""
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


@pytest.mark.parametrize("scale", [20, 22, 24])
def test_headline_config_golden(scale):
    """M2 headline input (s24 ef16 seed 0, GPU-built bit-exact): labels SHA-256,
    level sizes, E_r and the full DO trace (floats included) equal the
    reference's own run (oracle/make_golden.py rmat 24)."""
    from paper_1701_01170_b200._results import labels_to_host
    from paper_1701_01170_b200.generators import rmat_device_graph
    from paper_1701_01170_b200.primitives.bfs import bfs_device

    from paper_1701_01170_b200._results import preds_to_host

    rec, _ = rmat_golden(scale)
    dg = rmat_device_graph(scale, 16, 0)
    host = None
    for direction in ("push", "auto"):
        labels, preds, st = bfs_device(dg, 0, direction=direction)
        lab = labels_to_host(labels)
        assert sha(lab) == rec["bfs_sha"], direction
        if scale <= 22:  # preds by property (reference _oracles.py:169-182)
            if host is None:
                host = (dg.row.cpu().numpy(), dg.col.cpu().numpy().astype(np.int64))
            assert valid_bfs_preds(host[0], host[1], lab, preds_to_host(preds), 0), direction
        assert st.edges_reached == rec["E_r"]
        assert [it.frontier_in for it in st.per_iteration] == rec["bfs_levels"]
        if direction == "push":
            assert st.edges_traversed == rec["bfs_edges_traversed"]
        else:
            assert _trace_rows(st) == [list(x) for x in rec["bfs_auto_trace"]]


@pytest.mark.parametrize("loop", ["host", "device"])
def test_loops_agree(kat, loop):
    """Host-driven and device-resident level loops give identical labels and
    identical direction traces (floats included)."""
    from paper_1701_01170_b200 import _native
    from paper_1701_01170_b200._results import labels_to_host
    from paper_1701_01170_b200.primitives.bfs import bfs_device

    lp = _native.LOOP_HOST if loop == "host" else _native.LOOP_DEVICE
    for d in kat:
        g = host_graph(d)
        for direction in ("push", "pull", "auto"):
            labels, preds, st = bfs_device(g.device(), d["source"], direction=direction, loop=lp)
            assert np.array_equal(labels_to_host(labels[:d["n"]]), d["bfs"]), (d["name"], direction)
            if direction == "auto":
                assert _trace_rows(st) == [list(x) for x in d["bfs_auto_trace"]], d["name"]
    rec, arrays = rmat_golden(16)
    g = gfx_graph_s16(rec, arrays)
    for direction in ("push", "auto"):
        labels, preds, st = bfs_device(g.device(), 0, direction=direction, loop=lp)
        assert sha(labels_to_host(labels)) == rec["bfs_sha"]
        assert st.edges_reached == rec["E_r"]
        if direction == "auto":
            assert _trace_rows(st) == [list(x) for x in rec["bfs_auto_trace"]]


def gfx_graph_s16(rec, arrays):
    import paper_1701_01170_b200 as gfx

    return gfx.CsrGraph(rec["n"], arrays["row"], arrays["col"].astype(np.int64), undirected=True)


@pytest.mark.parametrize("direction", ["push", "pull", "auto"])
def test_deep_graph_past_depth_255(direction):
    """A 700-vertex path with side branches: hundreds of levels, most of them
    tiny, in every direction mode of the device-resident level loop."""
    import paper_1701_01170_b200 as gfx
    from oracle import c_oracle

    rng = np.random.default_rng(5)
    n_path = 700
    src = list(range(n_path - 1))
    dst = list(range(1, n_path))
    extra = 300  # leaves hanging off random path vertices, plus isolated ids
    for k in range(extra):
        src.append(int(rng.integers(0, n_path)))
        dst.append(n_path + k)
    n = n_path + extra + 50
    g = gfx.coo_to_csr(gfx.CooGraph(n, np.array(src), np.array(dst)), make_undirected=True)
    for s0 in (0, 350):
        want = c_oracle.bfs(g.row_offsets, g.column_indices, s0)
        r = gfx.bfs(g, s0, direction=direction)
        assert np.array_equal(r.labels, want), (direction, s0)
        assert valid_bfs_preds(g.row_offsets, g.column_indices, r.labels, r.preds, s0)


def test_graph_reload_refreshes_constants():
    """DeviceGraph.reload_ (C ABI gfx_graph_refresh): a different graph of
    the same shape uploaded into the resident buffers gives the new graph's
    BFS (max degree, nonzero bitmaps and pull heads recomputed)."""
    import torch

    import paper_1701_01170_b200 as gfx
    from oracle import c_oracle
    from paper_1701_01170_b200._results import labels_to_host
    from paper_1701_01170_b200.primitives.bfs import bfs_device

    rec, arrays = rmat_golden(16)
    g1 = gfx_graph_s16(rec, arrays)
    n = rec["n"]
    # the same graph with vertex ids reversed: same n and m, other content
    row, col = arrays["row"], arrays["col"].astype(np.int64)
    src = np.repeat(np.arange(n), np.diff(row))
    g2 = gfx.coo_to_csr(gfx.CooGraph(n, n - 1 - src, n - 1 - col))
    assert g2.num_edges == g1.num_edges
    dg = g1.device()
    for direction in ("push", "auto"):
        labels, _, _ = bfs_device(dg, 0, direction=direction)
        assert sha(labels_to_host(labels)) == rec["bfs_sha"]
    dg.reload_(torch.from_numpy(g2.row_offsets), torch.from_numpy(g2.column_indices.astype(np.int32)))
    for s0 in (n - 1, 5):
        want = c_oracle.bfs(g2.row_offsets, g2.column_indices, s0)
        for direction in ("push", "auto"):
            labels, _, _ = bfs_device(dg, s0, direction=direction)
            assert np.array_equal(labels_to_host(labels), want), (s0, direction)


@pytest.mark.parametrize("direction", ["push", "auto"])
def test_mid_frontier_with_hubs(direction):
    """Push levels of 33..65536 items expand 32 items per warp and set hubs
    (> 1024 slots) aside for a cooperative pass (gfx_bfs.cu push_mid): a
    level of 200 items holding three hubs of 3000-6000 leaves each."""
    import paper_1701_01170_b200 as gfx
    from oracle import c_oracle

    src, dst = [], []
    mids = list(range(1, 201))
    src += [0] * len(mids)
    dst += mids
    nxt = 201
    for hub, leaves in ((5, 3000), (77, 6000), (150, 4500)):
        src += [hub] * leaves
        dst += list(range(nxt, nxt + leaves))
        nxt += leaves
    for k, m in enumerate(mids):  # light items: a couple of leaves each
        src += [m, m]
        dst += [nxt + 2 * k, nxt + 2 * k + 1]
    n = nxt + 2 * len(mids) + 10
    g = gfx.coo_to_csr(gfx.CooGraph(n, np.array(src), np.array(dst)), make_undirected=True)
    want = c_oracle.bfs(g.row_offsets, g.column_indices, 0)
    r = gfx.bfs(g, 0, direction=direction)
    assert np.array_equal(r.labels, want)
    assert valid_bfs_preds(g.row_offsets, g.column_indices, r.labels, r.preds, 0)
    assert r.stats.edges_traversed > 0


def test_scale27_push_and_do_agree():
    """BASELINE config C5's input size on one GPU (R-MAT s27 ef16, GPU-built,
    4.2B slots): the direction-optimising run (pull sweeps) and the push-only
    run (load-balanced expansion) are independent code paths and must give
    identical labels; every reached vertex's pred sits one level up."""
    import torch

    from paper_1701_01170_b200.generators import rmat_device_graph
    from paper_1701_01170_b200.primitives.bfs import bfs_device

    free, _ = torch.cuda.mem_get_info()
    if free < 120 * 2**30:
        pytest.skip("needs ~120 GB of free HBM for the s27 build")
    dg = rmat_device_graph(27, 16, 0)
    la, pa, sa = bfs_device(dg, 0, direction="auto")
    lp, _, sp = bfs_device(dg, 0, direction="push")
    assert torch.equal(la, lp)
    assert sa.edges_reached == sp.edges_reached > 4_000_000_000
    reached = (la != 2**31 - 1).nonzero().squeeze(1)
    reached = reached[reached != 0]
    par = pa[reached].long()
    assert bool((par >= 0).all())
    assert torch.equal(la[par], la[reached] - 1)

"""PageRank, CC, BC and TC on the GPU vs reference goldens / CPU oracles."""
import numpy as np
import pytest

from conftest import host_graph, rmat_golden, sha
from oracle import c_oracle

pytestmark = pytest.mark.gpu

PR_L1 = 1e-6      # north_star tolerance for PageRank
BC_RTOL = 1e-5    # north_star tolerance for BC


def test_kat_all(kat):
    import paper_1701_01170_b200 as gfx

    for d in kat:
        g = host_graph(d)
        src = d["source"]
        r = gfx.pagerank(g, epsilon=0.0, max_iters=4)
        assert np.abs(r.rank - d["pr4"]).sum() <= PR_L1, d["name"]
        r = gfx.pagerank(g, epsilon=1e-3, max_iters=50)
        assert np.abs(r.rank - d["pr_eps"]).sum() <= PR_L1, d["name"]
        b = gfx.bc(g, src).bc_values
        assert np.allclose(b, d["bc"], rtol=BC_RTOL, atol=1e-9), d["name"]
        if d["undirected"]:
            c = gfx.cc(g)
            assert np.array_equal(c.component, d["cc"]), d["name"]
            assert c.num_components == len(np.unique(d["cc"]))
            t = gfx.tc(g)
            assert t.total_triangles == d["tc_total"], d["name"]
            assert np.array_equal(t.per_edge_counts, d["tc_counts"]), d["name"]
            assert np.array_equal(t.oriented_src, d["tc_src"]), d["name"]
            assert np.array_equal(t.oriented_dst, d["tc_dst"]), d["name"]


def test_reference_kats():
    """reference test_primitives.py:117-228."""
    import paper_1701_01170_b200 as gfx

    def und(n, edges):
        e = np.array(edges, dtype=np.int64).reshape(-1, 2)
        return gfx.coo_to_csr(gfx.CooGraph(n, e[:, 0], e[:, 1]), make_undirected=True)

    path3 = und(3, [(0, 1), (1, 2)])
    assert gfx.bc(path3, 0).bc_values.tolist() == [0.0, 1.0, 0.0]
    star = und(4, [(0, 1), (0, 2), (0, 3)])
    r = gfx.bc(star, 1).bc_values
    assert r[0] == pytest.approx(2.0) and r[1] == 0.0
    k3 = und(3, [(0, 1), (0, 2), (1, 2)])
    assert np.allclose(gfx.bc(k3, 0).bc_values, 0.0)
    assert gfx.tc(k3).total_triangles == 1
    k4 = und(4, [(i, j) for i in range(4) for j in range(i + 1, 4)])
    assert gfx.tc(k4).total_triangles == 4
    assert gfx.tc(und(6, [(0, i) for i in range(1, 6)])).total_triangles == 0
    two = und(4, [(0, 1), (2, 3)])
    assert gfx.cc(two).num_components == 2
    empty = gfx.coo_to_csr(gfx.CooGraph(5, np.array([], dtype=np.int64),
                                        np.array([], dtype=np.int64)), make_undirected=True)
    assert gfx.cc(empty).num_components == 5
    path10 = und(10, [(i, i + 1) for i in range(9)])
    assert gfx.cc(path10).num_components == 1
    pr = gfx.pagerank(k3, epsilon=1e-10, max_iters=200)
    assert np.allclose(pr.rank, pr.rank[0]) and pr.rank.sum() == pytest.approx(1.0)
    single = gfx.coo_to_csr(gfx.CooGraph(1, np.array([], dtype=np.int64),
                                         np.array([], dtype=np.int64)))
    assert gfx.pagerank(single).rank.tolist() == [1.0]
    assert gfx.pagerank(gfx.CsrGraph(4, np.array([0, 3, 5, 7, 9]),
                                     np.array([1, 2, 3, 0, 2, 0, 1, 0, 1]), undirected=False),
                        epsilon=1e-3, max_iters=500).stats.iterations < 500
    with pytest.raises(ValueError):
        gfx.pagerank(k3, damping=1.5)
    directed = gfx.coo_to_csr(gfx.CooGraph(3, np.array([0, 1]), np.array([1, 2])))
    with pytest.raises(ValueError):
        gfx.cc(directed)
    with pytest.raises(ValueError):
        gfx.tc(directed)
    multi = gfx.bc(und(4, [(0, 1), (1, 2), (2, 3)]), [0, 3]).bc_values
    split = gfx.bc(und(4, [(0, 1), (1, 2), (2, 3)]), 0).bc_values + \
        gfx.bc(und(4, [(0, 1), (1, 2), (2, 3)]), 3).bc_values
    assert np.allclose(multi, split)


@pytest.mark.parametrize("scale", [16, 18])
def test_rmat_golden_arrays(scale):
    import paper_1701_01170_b200 as gfx

    rec, arrays = rmat_golden(scale)
    from paper_1701_01170_b200.generators import rmat_device_graph

    dg = rmat_device_graph(scale, 16, 0)
    g = dg.to_host()
    c = gfx.cc(g)
    assert sha(c.component) == rec["cc_canon_sha"] and c.num_components == rec["cc_num"]
    pr = gfx.pagerank(g, epsilon=0.0, max_iters=20).rank
    b = gfx.bc(g, 0).bc_values
    if "pr20" in arrays:
        assert np.abs(pr - arrays["pr20"]).sum() <= PR_L1
        assert np.allclose(b, arrays["bc"], rtol=BC_RTOL, atol=1e-9)
    t = gfx.tc(g)
    assert t.total_triangles == rec["tc_total"]
    assert sha(t.per_edge_counts) == rec["tc_counts_sha"]
    assert sha(t.oriented_src) == rec["tc_src_sha"] and sha(t.oriented_dst) == rec["tc_dst_sha"]


@pytest.mark.parametrize("scale", [20, 22])
def test_rmat_golden_large(scale):
    """C3/C4 configs at s22: CC/TC exact, PR/BC against sampled reference values."""
    import torch

    from paper_1701_01170_b200.generators import rmat_device_graph
    from paper_1701_01170_b200.primitives.bc import bc_device
    from paper_1701_01170_b200.primitives.cc import cc_device
    from paper_1701_01170_b200.primitives.pagerank import pagerank_device
    from paper_1701_01170_b200.primitives.tc import tc_device

    rec, arrays = rmat_golden(scale)
    dg = rmat_device_graph(scale, 16, 0)
    comp, k, _ = cc_device(dg)
    assert sha(comp.to(torch.int64).cpu().numpy()) == rec["cc_canon_sha"] and k == rec["cc_num"]
    rank, _ = pagerank_device(dg, 0.85, 0.0, 20)
    rank = rank.cpu().numpy()
    assert abs(rank.sum() - rec["pr20_sum"]) < 1e-9
    assert np.allclose(rank[arrays["pr_idx"]], arrays["pr_vals"], rtol=1e-9, atol=1e-15)
    bcv, _ = bc_device(dg, [0])
    bcv = bcv.cpu().numpy()
    assert np.allclose(bcv[arrays["bc_idx"]], arrays["bc_vals"], rtol=BC_RTOL, atol=1e-9)
    assert abs(bcv.sum() - rec["bc_sum"]) <= 1e-5 * abs(rec["bc_sum"])
    if "tc_total" in rec:
        total, counts, osrc, odst, _ = tc_device(dg)
        assert total == rec["tc_total"]
        assert sha(counts.to(torch.int64).cpu().numpy()) == rec["tc_counts_sha"]
        assert sha(osrc.to(torch.int64).cpu().numpy()) == rec["tc_src_sha"]
        assert sha(odst.to(torch.int64).cpu().numpy()) == rec["tc_dst_sha"]


@pytest.mark.skipif(not __import__("os").environ.get("GFX_SLOW_TESTS"),
                    reason="host C oracle needs minutes at s22; run with GFX_SLOW_TESTS=1")
def test_tc_s22_vs_c_oracle():
    """TC on s22 (no reference golden: the reference needs > 30 min) against
    the C restatement of tc.py:53-76."""
    import torch

    from paper_1701_01170_b200.generators import rmat_device_graph
    from paper_1701_01170_b200.primitives.tc import tc_device

    dg = rmat_device_graph(22, 16, 0)
    total, counts, osrc, odst, _ = tc_device(dg)
    row = dg.row.cpu().numpy()
    col = dg.col.cpu().numpy()
    want_total, want_counts, want_src, want_dst = c_oracle.tc(row, col)
    assert total == want_total
    assert np.array_equal(counts.to(torch.int64).cpu().numpy(), want_counts)
    assert np.array_equal(odst.to(torch.int64).cpu().numpy(), want_dst)


def test_s24_sssp_cc_pagerank_golden():
    """C3 (PageRank 20 iterations and CC on R-MAT s24) and M3 (SSSP s24,
    delta 32 and default) against the reference's own s24 run
    (GOLDEN_S24_FULL=1 oracle/make_golden.py rmat 24): distances and
    canonical CC labels bit-exact, PageRank sum and 4096 sampled ranks."""
    import torch

    from paper_1701_01170_b200._results import labels_to_host
    from paper_1701_01170_b200.generators import rmat_device_graph
    from paper_1701_01170_b200.primitives.cc import cc_device
    from paper_1701_01170_b200.primitives.pagerank import pagerank_device
    from paper_1701_01170_b200.primitives.sssp import sssp_device

    rec, arrays = rmat_golden(24)
    if "sssp_d32_sha" not in rec:
        pytest.skip("s24 SSSP/CC/PageRank goldens not generated")
    dg = rmat_device_graph(24, 16, 0, weights=(1, 64), weight_seed=0)
    for delta, key in ((32, "sssp_d32"), (None, "sssp_default")):
        dist, _, _ = sssp_device(dg, 0, delta=delta)
        assert sha(labels_to_host(dist)) == rec[key + "_sha"], delta
    comp, k, _ = cc_device(dg)
    assert sha(comp.to(torch.int64).cpu().numpy()) == rec["cc_canon_sha"] and k == rec["cc_num"]
    rank, _ = pagerank_device(dg, 0.85, 0.0, 20)
    rank = rank.cpu().numpy()
    assert abs(rank.sum() - rec["pr20_sum"]) < 1e-9
    assert np.allclose(rank[arrays["pr_idx"]], arrays["pr_vals"], rtol=1e-9, atol=1e-15)


@pytest.mark.parametrize("n", [300, 700, 1500])
def test_bc_deep_levels(n):
    """BC's forward levels from the DO-BFS (bfs_do_levels: level lists by
    two passes over the labels) on graphs with hundreds of levels -- past
    the depth-byte limit (255) of the persistent BFS, and past 1024 levels
    (the push-level fallback) -- plus a dense head: a path with a clique at
    one end; values equal the numpy port of bc.py:32-116"""
    import paper_1701_01170_b200 as gfx
    from oracle import graphfx_port as port

    k = 24
    a, b = np.triu_indices(k, 1)
    src = np.concatenate([a, np.arange(k - 1, n - 1)]).astype(np.int64)
    dst = np.concatenate([b, np.arange(k, n)]).astype(np.int64)
    g = gfx.coo_to_csr(gfx.CooGraph(n, src, dst), make_undirected=True)
    row, col = g.row_offsets, g.column_indices
    for s in (0, n - 1, n // 2):
        want = port.bc(row, col, [s])
        got = gfx.bc(g, [s]).bc_values
        assert np.allclose(got, want, rtol=1e-9, atol=1e-9), s

"""Generic device operators with the closed functor registry
(reference operators.py; KATs from reference test_operators.py:207-276)."""
import numpy as np
import pytest

from conftest import host_graph

pytestmark = pytest.mark.gpu


def _und(n, edges):
    import paper_1701_01170_b200 as gfx

    e = np.array(edges, dtype=np.int64).reshape(-1, 2)
    return gfx.coo_to_csr(gfx.CooGraph(n, e[:, 0], e[:, 1]), make_undirected=True)


def _k(n):
    return _und(n, [(i, j) for i in range(n) for j in range(i + 1, n)])


def test_advance_no_functor_is_the_gather(kat):
    import paper_1701_01170_b200 as gfx

    for d in kat[:6]:
        g = host_graph(d)
        rng = np.random.default_rng(3)
        F = rng.integers(0, g.num_vertices, size=min(40, g.num_vertices))
        out = gfx.advance(g, gfx.Frontier.from_items(F))
        want = np.concatenate([g.neighbors(v) for v in F]) if len(F) else np.zeros(0)
        assert sorted(out.to_array().tolist()) == sorted(want.tolist())
        oute = gfx.advance(g, gfx.Frontier.from_items(F), kind=gfx.AdvanceKind.V2E)
        wante = np.concatenate([np.arange(g.row_offsets[v], g.row_offsets[v + 1]) for v in F])
        assert sorted(oute.to_array().tolist()) == sorted(wante.tolist())


def test_operator_level_bfs_matches_reference(kat):
    """The reference's push BFS loop (bfs.py:111-138) written with the device
    operators: advance(claim) -> filter(EXACT)."""
    import torch

    import paper_1701_01170_b200 as gfx
    from paper_1701_01170_b200 import _native

    for d in kat:
        g = host_graph(d)
        labels = torch.full((g.num_vertices,), _native.UNVISITED32, dtype=torch.int32,
                            device="cuda")
        preds = torch.full_like(labels, -1)
        labels[d["source"]] = 0
        F = gfx.Frontier.from_items([d["source"]])
        depth = 0
        while len(F):
            depth += 1
            fs = gfx.FunctorSet(cond=gfx.functors.claim(labels, preds, depth))
            out = gfx.advance(g, F, functors=fs)
            F = gfx.filter_frontier(out, gfx.FilterMode.EXACT, g=g)
        lab = labels.to(torch.int64).cpu().numpy()
        lab[lab == _native.UNVISITED32] = gfx.UNVISITED
        assert np.array_equal(lab, d["bfs"]), d["name"]


def test_operator_level_sssp_matches_reference(kat):
    import torch

    import paper_1701_01170_b200 as gfx
    from paper_1701_01170_b200 import _native

    for d in kat:
        g = host_graph(d, weighted=True)
        dist = torch.full((g.num_vertices,), _native.UNVISITED32, dtype=torch.int32, device="cuda")
        dist[d["source"]] = 0
        F = gfx.Frontier.from_items([d["source"]])
        while len(F):
            out = gfx.advance(g, F, functors=gfx.FunctorSet(cond=gfx.functors.relax(dist)))
            F = gfx.filter_frontier(out, g=g)
        lab = dist.to(torch.int64).cpu().numpy()
        lab[lab == _native.UNVISITED32] = gfx.UNVISITED
        assert np.array_equal(lab, d["sssp"]), d["name"]


def test_filter_exact_is_sorted_unique():
    import torch

    import paper_1701_01170_b200 as gfx

    rng = np.random.default_rng(5)
    items = rng.integers(0, 500, size=3000)
    out = gfx.filter_frontier(gfx.Frontier.from_items(items), gfx.FilterMode.EXACT)
    assert out.to_array().tolist() == np.unique(items).tolist()
    labels = torch.from_numpy((np.arange(500) % 3).astype(np.int32)).cuda()
    fs = gfx.FunctorSet(vertex_cond=gfx.functors.label_eq(labels, 1))
    out = gfx.filter_frontier(gfx.Frontier.from_items(items), gfx.FilterMode.INEXACT, fs)
    # INEXACT: the reference culling heuristics exactly (input order kept)
    from oracle import graphfx_port as port

    assert out.to_array().tolist() == port.cull_inexact(items[items % 3 == 1]).tolist()
    out = gfx.filter_frontier(gfx.Frontier.from_items(items), gfx.FilterMode.EXACT, fs)
    assert out.to_array().tolist() == np.unique(items[items % 3 == 1]).tolist()


def test_compute_counts_multiset():
    import torch

    import paper_1701_01170_b200 as gfx

    acc = torch.zeros(6, dtype=torch.int64, device="cuda")
    gfx.compute(gfx.Frontier.from_items([0, 1, 2, 5, 5]), gfx.functors.add(acc, 1))
    assert acc.cpu().tolist() == [1, 1, 1, 0, 0, 2]


def test_orient_keeps_half():
    import paper_1701_01170_b200 as gfx

    g = _k(6)
    allv = gfx.Frontier.from_items(np.arange(6))
    out = gfx.advance(g, allv, kind=gfx.AdvanceKind.V2E,
                      functors=gfx.FunctorSet(cond=gfx.functors.orient()))
    assert len(out) == g.num_edges // 2


def test_segmented_intersect_kats():
    import paper_1701_01170_b200 as gfx

    k3 = _k(3)
    r = gfx.segmented_intersect(k3, (np.array([0]), np.array([1])))
    assert r.per_pair_counts.tolist() == [1] and r.intersections.to_array().tolist() == [2]
    assert r.total == 1
    assert gfx.segmented_intersect(_und(4, [(0, 1), (2, 3)]),
                                   (np.array([0]), np.array([2]))).total == 0
    star = _und(5, [(0, i) for i in range(1, 5)])
    assert gfx.segmented_intersect(star, (np.array([0]), np.array([0]))).per_pair_counts.tolist() \
        == [4]
    k4 = _k(4)
    ef = gfx.Frontier.from_items(np.arange(k4.num_edges), kind="edge")
    assert gfx.segmented_intersect(k4, ef).total == k4.num_edges * 2
    r = gfx.segmented_intersect(k4, (np.array([0, 1]), np.array([1, 2])))
    assert r.intersections.to_array().tolist() == [2, 3, 0, 3]
    with pytest.raises(ValueError):
        gfx.segmented_intersect(k3, (np.array([0]), np.array([1, 2])))
    bad = gfx.CsrGraph(3, np.array([0, 2, 2, 2]), np.array([2, 1]))
    with pytest.raises(ValueError, match="not sorted"):
        gfx.segmented_intersect(bad, (np.array([0]), np.array([0])), check_sorted=True)
    rng = np.random.default_rng(17)
    for _ in range(5):
        g = gfx.coo_to_csr(gfx.generate_rmat(int(rng.integers(4, 9)), 6,
                                             seed=int(rng.integers(1 << 30))), make_undirected=True)
        k = min(50, g.num_vertices)
        u = rng.integers(0, g.num_vertices, size=k)
        v = rng.integers(0, g.num_vertices, size=k)
        res = gfx.segmented_intersect(g, (u, v), small_cut=8)
        adj = [set(g.neighbors(x).tolist()) for x in range(g.num_vertices)]
        want = [len(adj[a] & adj[b]) for a, b in zip(u, v)]
        assert res.per_pair_counts.tolist() == want and res.total == sum(want)


def test_callables_run_on_device_tensors_and_mixing_is_rejected():
    """Callables see int64 CUDA tensors (the staged path); a callable that
    indexes host data fails loudly instead of falling back to the CPU; a
    FunctorSet mixing registry functors and callables is rejected."""
    import torch

    import paper_1701_01170_b200 as gfx

    seen = {}

    def cond(s, d, e, _):
        seen["dev"] = (s.device.type, d.device.type, e.device.type, s.dtype)
        return d > 0

    out = gfx.advance(_k(3), gfx.Frontier.from_items([0]), functors=gfx.FunctorSet(cond=cond))
    assert sorted(out.to_array().tolist()) == [1, 2]
    assert seen["dev"] == ("cuda", "cuda", "cuda", torch.int64)
    host = np.array([True, False, True])
    with pytest.raises(Exception):
        gfx.advance(_k(3), gfx.Frontier.from_items([0]),
                    functors=gfx.FunctorSet(cond=lambda s, d, e, _: host[d]))
    labels = torch.zeros(3, dtype=torch.int32, device="cuda")
    with pytest.raises(TypeError):
        gfx.advance(_k(3), gfx.Frontier.from_items([0]),
                    functors=gfx.FunctorSet(cond=gfx.functors.label_eq(labels, 0),
                                            apply=lambda s, d, e, _: None))

"""The reference's operator / near-far / load-balance / frontier tests, replayed
against the device operators.

Each test names the reference test it replays (tests/test_operators.py,
test_near_far.py, test_load_balance.py, test_frontier.py).  Callable
functors take the same lambdas with problem data held in CUDA tensors
(the staged device path); registry functors are checked against them.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SMALL = None


def gx():
    import paper_1701_01170_b200 as gfx

    return gfx


def params():
    return gx().LbParams(small_cut=2, large_cut=8, chunk_size=4, items_per_chunk=3)


ALL = ["THREAD_EXPAND", "TWC", "LB", "LB_LIGHT", "LB_CULL"]


def from_edges(n, edges, undirected=True):
    e = np.array(list(edges), dtype=np.int64).reshape(-1, 2)
    return gx().coo_to_csr(gx().CooGraph(n, e[:, 0], e[:, 1]), make_undirected=undirected)


def star(k=3):
    return from_edges(k + 1, [(0, i + 1) for i in range(k)])


def complete(n):
    return from_edges(n, [(i, j) for i in range(n) for j in range(i + 1, n)])


def vf(*items):
    return gx().Frontier.from_items(np.array(items, dtype=np.int64))


def rmat(scale, ef, seed):
    return gx().coo_to_csr(gx().generate_rmat(scale, ef, seed=seed), make_undirected=True)


def cuda(a, dtype=None):
    import torch

    t = torch.as_tensor(np.asarray(a), device="cuda")
    return t if dtype is None else t.to(dtype)


# ---- test_operators.py:40-56 TestAtomicHelpers (unchanged: host arrays in) ----
def test_atomic_helpers_on_host_arrays():
    arr = np.array([10, 10], dtype=np.int64)
    won = gx().atomic_min(arr, np.array([0, 0, 1]), np.array([8, 5, 20]))
    assert arr.tolist() == [5, 10] and won.tolist() == [False, True, False]
    arr = np.zeros(3)
    gx().atomic_add(arr, np.array([1, 1, 2]), np.array([1.0, 2.0, 5.0]))
    assert arr.tolist() == [0.0, 3.0, 5.0]
    arr = np.array([-1, 7], dtype=np.int64)
    won = gx().compare_and_swap(arr, np.array([0, 0, 1]), -1, 3)
    assert won.tolist() == [True, False, False] and arr.tolist() == [3, 7]


def test_atomic_helpers_on_device_arrays_match_numpy():
    """The batched helpers on CUDA tensors against numpy restatements of
    operators.py:111-153 over random batches with many duplicates."""
    import torch

    rng = np.random.default_rng(5)
    for _ in range(20):
        n, k = int(rng.integers(1, 50)), int(rng.integers(0, 400))
        base = rng.integers(0, 100, size=n).astype(np.int64)
        idx = rng.integers(0, n, size=k)
        vals = rng.integers(0, 120, size=k).astype(np.int64)
        # atomic_min
        want = base.copy()
        improving = vals < want[idx]
        np.minimum.at(want, idx[improving], vals[improving])
        won_want = improving & (vals == want[idx])
        t = cuda(base)
        won = gx().atomic_min(t, cuda(idx), cuda(vals))
        assert np.array_equal(t.cpu().numpy(), want)
        assert np.array_equal(won.cpu().numpy(), won_want)
        # compare_and_swap with per-entry values
        arr = rng.integers(-1, 2, size=n).astype(np.int64)
        want = arr.copy()
        elig = arr[idx] == -1
        first = np.zeros(k, dtype=bool)
        seen = set()
        for i in range(k):
            if elig[i] and idx[i] not in seen:
                first[i] = True
                seen.add(idx[i])
        want[idx[first]] = vals[first]
        t = cuda(arr)
        won = gx().compare_and_swap(t, cuda(idx), -1, cuda(vals))
        assert np.array_equal(won.cpu().numpy(), first)
        assert np.array_equal(t.cpu().numpy(), want)
        # atomic_add, int32 array
        want = np.zeros(n, dtype=np.int32)
        np.add.at(want, idx, 3)
        t = torch.zeros(n, dtype=torch.int32, device="cuda")
        gx().atomic_add(t, cuda(idx), 3)
        assert np.array_equal(t.cpu().numpy(), want)


# ---- test_operators.py:59-169 TestAdvance ------------------------------------
def test_advance_small_graphs():
    g = star(3)
    assert sorted(gx().advance(g, vf(0)).to_array().tolist()) == [1, 2, 3]
    for kind in gx().AdvanceKind:
        f = gx().Frontier.from_items([], kind=kind.input_kind)
        assert len(gx().advance(g, f, kind)) == 0
    out = gx().advance(g, vf(0), gx().AdvanceKind.V2E)
    assert out.kind == "edge" and sorted(out.to_array().tolist()) == [0, 1, 2]
    d = from_edges(3, [(0, 1), (1, 2)], undirected=False)
    out = gx().advance(d, gx().Frontier.from_items([0], kind="edge"), gx().AdvanceKind.E2V)
    assert out.to_array().tolist() == [2]
    d = from_edges(4, [(0, 1), (1, 2), (2, 3)], undirected=False)
    out = gx().advance(d, gx().Frontier.from_items([0], kind="edge"), gx().AdvanceKind.E2E)
    assert out.kind == "edge" and out.to_array().tolist() == [1]
    with pytest.raises(ValueError):
        gx().advance(g, gx().Frontier.from_items([0], kind="edge"), gx().AdvanceKind.V2V)


def test_shared_neighbor_idempotent_duplicates():
    visited = cuda([True, True, False])
    fs = gx().FunctorSet(cond=lambda s, d, e, _: ~visited[d])
    out = gx().advance(complete(3), vf(0, 1), functors=fs, idempotent=True)
    assert sorted(out.to_array().tolist()) == [2, 2]


def test_output_size_before_cond_matches_scan_total():
    g = rmat(6, 5, 1)
    f = vf(*range(0, g.num_vertices, 3))
    _, total = gx().compute_scan_offsets(g, f)
    assert len(gx().advance(g, f)) == total
    scan, tot = gx().compute_scan_offsets(g, f)
    deg = np.diff(g.row_offsets)[f.to_array()]
    assert scan.tolist() == [0] + np.cumsum(deg).tolist() and tot == deg.sum()


@pytest.mark.parametrize("strategy", ALL)
def test_strategy_interchangeable_and_duplicates(strategy):
    strategy = getattr(gx().Strategy, strategy)
    rng = np.random.default_rng(7)
    for _ in range(10):
        g = rmat(int(rng.integers(3, 8)), 6, int(rng.integers(1 << 30)))
        size = int(rng.integers(1, g.num_vertices + 1))
        f = gx().Frontier.from_items(rng.choice(g.num_vertices, size=size, replace=False))
        base = gx().advance(g, f, strategy=gx().Strategy.THREAD_EXPAND, params=params())
        other = gx().advance(g, f, strategy=strategy, params=params())
        assert sorted(base.to_array().tolist()) == sorted(other.to_array().tolist())
    out = gx().advance(star(3), vf(0, 0), strategy=strategy, params=params(), idempotent=True)
    assert sorted(out.to_array().tolist()) == [1, 1, 2, 2, 3, 3]


def test_apply_exactly_once_per_triple():
    import torch

    g = rmat(6, 4, 9)
    f = vf(*range(0, g.num_vertices, 2))
    for strategy in ALL:
        calls = torch.zeros(g.num_edges, dtype=torch.int64, device="cuda")
        fs = gx().FunctorSet(cond=lambda s, d, e, _: torch.ones(len(s), dtype=torch.bool,
                                                                  device="cuda"),
                             apply=lambda s, d, e, _: gx().atomic_add(calls, e, 1))
        gx().advance(g, f, functors=fs, strategy=getattr(gx().Strategy, strategy),
                     params=params())
        _, total = gx().compute_scan_offsets(g, f)
        assert int(calls.sum()) == total and int(calls.max()) <= 1


def test_callable_triples_are_the_reference_gather():
    """Staged advance sees exactly the reference _gather triples, slot order."""
    g = rmat(7, 8, 3)
    rng = np.random.default_rng(0)
    items = rng.integers(0, g.num_vertices, size=60)
    seen = {}

    def cond(s, d, e, _):
        seen["t"] = (s.cpu().numpy(), d.cpu().numpy(), e.cpu().numpy())
        return (s + d) % 2 == 0

    out = gx().advance(g, gx().Frontier.from_items(items), gx().AdvanceKind.V2E,
                       functors=gx().FunctorSet(cond=cond))
    row, col = g.row_offsets, g.column_indices
    deg = row[items + 1] - row[items]
    src = np.repeat(items, deg)
    edge = np.concatenate([np.arange(row[v], row[v + 1]) for v in items])
    assert np.array_equal(seen["t"][0], src) and np.array_equal(seen["t"][2], edge)
    assert np.array_equal(seen["t"][1], col[edge])
    assert np.array_equal(out.to_array(), edge[(src + col[edge]) % 2 == 0])


# ---- test_operators.py:154-167 TestPullAdvance -------------------------------
def test_path_pull_and_kind():
    labels = cuda(np.array([0, np.iinfo(np.int64).max, np.iinfo(np.int64).max]))
    fs = gx().FunctorSet(cond=lambda s, d, e, _: labels[s] == 0)
    out = gx().advance(from_edges(3, [(0, 1), (1, 2)]), gx().Frontier.from_items([1, 2]),
                       direction="pull", functors=fs)
    assert out.to_array().tolist() == [1]
    with pytest.raises(ValueError):
        gx().advance(star(2), gx().Frontier.from_items([0], kind="edge"), gx().AdvanceKind.E2V,
                     direction="pull")


@pytest.mark.parametrize("undirected", [True, False])
def test_pull_step_registry_equals_callable(undirected):
    """One reference pull level (bfs.py:139-151) three ways: the registry
    functor (fused early-exit kernel), the callable lambdas with _set_depth
    as apply, and the numpy definition; the (active, rest) split and the
    labels agree; preds are in-neighbours on the previous level."""
    import torch

    g = gx().coo_to_csr(gx().generate_rmat(9, 8, seed=4), make_undirected=undirected)
    n = g.num_vertices
    # level sets from a push BFS so depth-1 labels are real
    r = gx().bfs(g, 0, direction="push")
    lab = r.labels.copy()
    depth = 3
    lab[lab >= depth - 1 + 1] = np.iinfo(np.int64).max  # keep levels < depth
    U = np.flatnonzero(lab == np.iinfo(np.int64).max)
    # numpy definition over the reverse adjacency
    rows, cols, _ = g.csc()
    want = np.array([u for u in U if np.any(lab[cols[rows[u]:rows[u + 1]]] == depth - 1)])
    # registry
    lab32 = torch.from_numpy(np.where(lab == np.iinfo(np.int64).max, 2**31 - 1, lab)
                             .astype(np.int32)).cuda()
    preds = torch.full((n,), -1, dtype=torch.int32, device="cuda")
    a, rest = gx().pull_step(g, gx().Frontier.from_items(U),
                             gx().FunctorSet(cond=gx().functors.pull(lab32, preds, depth)))
    assert a.to_array().tolist() == want.tolist()
    assert sorted(rest.to_array().tolist() + want.tolist()) == U.tolist()
    l32 = lab32.cpu().numpy()
    p32 = preds.cpu().numpy()
    assert np.all(l32[want] == depth)
    for u in want[:200]:
        assert p32[u] in cols[rows[u]:rows[u + 1]] and lab[p32[u]] == depth - 1
    # callables on device tensors
    lab64 = torch.from_numpy(lab.copy()).cuda()
    prd64 = torch.full((n,), -1, dtype=torch.int64, device="cuda")

    def set_depth(s, d, e, _):
        lab64[d] = depth
        prd64[d] = s

    fs = gx().FunctorSet(cond=lambda s, d, e, _: lab64[s] == depth - 1, apply=set_depth)
    a2, rest2 = gx().pull_expand(g, gx().Frontier.from_items(U), fs)
    assert a2.to_array().tolist() == want.tolist()
    assert rest2.to_array().tolist() == rest.to_array().tolist()
    # every callable triple's edge id is the forward slot of (src -> dst)
    seen = {}

    def cond(s, d, e, _):
        seen["t"] = (s.cpu().numpy(), d.cpu().numpy(), e.cpu().numpy())
        return lab64[s] == depth - 1

    gx().pull_expand(g, gx().Frontier.from_items(U[:50]), gx().FunctorSet(cond=cond))
    s_, d_, e_ = seen["t"]
    assert np.array_equal(g.edge_sources()[e_], s_) and np.array_equal(g.column_indices[e_], d_)


# ---- test_operators.py:170-205 TestFilter --------------------------------------
def test_filter_exact_and_cond():
    assert gx().filter_frontier(vf(1, 2, 2, 3)).to_array().tolist() == [1, 2, 3]
    fs = gx().FunctorSet(vertex_cond=lambda v, _: v % 2 == 0)
    assert gx().filter_frontier(vf(1, 2, 3), functors=fs).to_array().tolist() == [2]
    rng = np.random.default_rng(3)
    once = gx().filter_frontier(gx().Frontier.from_items(rng.integers(0, 50, size=200)))
    assert np.array_equal(once.to_array(), gx().filter_frontier(once).to_array())


@pytest.mark.parametrize("bitmask", [True, False])
@pytest.mark.parametrize("team", [0, 16, 256])
@pytest.mark.parametrize("local", [0, 8, 64])
def test_inexact_sandwich(bitmask, team, local):
    import collections

    rng = np.random.default_rng(team * 100 + local + bitmask)
    items = rng.integers(0, 500, size=10_000)
    keep_even = gx().FunctorSet(vertex_cond=lambda v, _: v % 2 == 0)
    cfg = gx().CullingConfig(use_bitmask=bitmask, team_table_size=team, local_table_size=local,
                             domain_size=500)
    out = gx().filter_frontier(gx().Frontier.from_items(items), gx().FilterMode.INEXACT,
                               functors=keep_even, culling=cfg).to_array()
    valid = items[items % 2 == 0]
    assert set(out.tolist()) == set(valid.tolist())
    oc, ic = collections.Counter(out.tolist()), collections.Counter(valid.tolist())
    assert all(oc[k] <= ic[k] for k in oc)


def test_inexact_cull_bit_exact_vs_reference_golden():
    """Device culling == the reference's _apply_culling output, order included
    (golden vectors from running the reference, oracle/make_cull_golden.py)."""
    from conftest import GOLDEN

    z = np.load(GOLDEN / "cull_inexact.npz")
    for k in range(int(z["count"])):
        bm, team, local, bb, lb, dom = z[f"cfg_{k}"].tolist()
        cfg = gx().CullingConfig(use_bitmask=bool(bm), team_table_size=team,
                                 local_table_size=local, bitmask_batch=bb, local_batch=lb,
                                 domain_size=dom)
        got = gx().filter_frontier(gx().Frontier.from_items(z[f"items_{k}"]),
                                   gx().FilterMode.INEXACT, culling=cfg).to_array()
        assert np.array_equal(got, z[f"out_{k}"]), k


def test_registry_vertex_cond_inexact_and_exact():
    import torch

    labels = torch.tensor([0, 1, 0, 1, 0], dtype=torch.int32, device="cuda")
    f = vf(4, 0, 2, 4, 1, 0)
    fs = gx().FunctorSet(vertex_cond=gx().functors.label_eq(labels, 0))
    assert gx().filter_frontier(f, functors=fs).to_array().tolist() == [0, 2, 4]
    cfg = gx().CullingConfig(use_bitmask=False, team_table_size=0, local_table_size=0)
    out = gx().filter_frontier(f, gx().FilterMode.INEXACT, functors=fs, culling=cfg)
    assert out.to_array().tolist() == [4, 0, 2, 4, 0]


# ---- test_operators.py:278-295 TestCompute --------------------------------------
def test_compute_callables():
    counters = np.zeros(4, dtype=np.int64)
    gx().compute(vf(0, 1, 2), lambda items, _: gx().atomic_add(counters, items, 1))
    assert counters.tolist() == [1, 1, 1, 0]
    counters = np.zeros(2, dtype=np.int64)
    gx().compute(vf(), lambda items, _: gx().atomic_add(counters, items, 1))
    assert counters.sum() == 0
    counters = np.zeros(6, dtype=np.int64)
    gx().compute(vf(5, 5), lambda items, _: gx().atomic_add(counters, items, 1))
    assert counters[5] == 2


# ---- test_operators.py:296-330 TestFusedAdvanceFilter ---------------------------
def test_fused_equivalent_to_advance_then_filter():
    rng = np.random.default_rng(11)
    for _ in range(15):
        g = rmat(int(rng.integers(3, 7)), 5, int(rng.integers(1 << 30)))
        size = int(rng.integers(1, g.num_vertices + 1))
        f = gx().Frontier.from_items(rng.choice(g.num_vertices, size=size, replace=False))
        drop = int(rng.integers(0, g.num_vertices))
        fs = gx().FunctorSet(cond=lambda s, d, e, _: (d + s) % 3 != 0,
                             vertex_cond=lambda v, _: v != drop)
        fused = gx().advance_filter_fused(g, f, functors=fs, params=params())
        staged = gx().filter_frontier(gx().advance(g, f, functors=gx().FunctorSet(cond=fs.cond)),
                                      functors=gx().FunctorSet(vertex_cond=fs.vertex_cond))
        assert set(fused.to_array().tolist()) == set(staged.to_array().tolist())


def test_fused_star_claim_and_determinism():
    import torch

    visited = torch.zeros(4, dtype=torch.bool, device="cuda")
    visited[0] = True

    def claim(s, d, e, _):
        fresh = ~visited[d]
        visited[d] = True
        return fresh

    out = gx().advance_filter_fused(star(3), vf(0), functors=gx().FunctorSet(cond=claim))
    assert sorted(out.to_array().tolist()) == [1, 2, 3]
    g = rmat(6, 6, 2)
    f = vf(*range(0, g.num_vertices, 5))
    fs = gx().FunctorSet(cond=lambda s, d, e, _: d % 2 == 0)
    a = gx().advance_filter_fused(g, f, functors=fs).to_array()
    b = gx().advance_filter_fused(g, f, functors=fs).to_array()
    assert np.array_equal(a, b)


def test_fused_registry_claim_is_one_bfs_level():
    """Registry fused (one kernel: claim + vertex_cond + cull) == staged
    advance(claim) + EXACT filter, as sets, and claims each vertex once."""
    import torch

    g = rmat(10, 8, 1)
    n = g.num_vertices
    for fused in (True, False):
        labels = torch.full((n,), 2**31 - 1, dtype=torch.int32, device="cuda")
        labels[0] = 0
        preds = torch.full((n,), -1, dtype=torch.int32, device="cuda")
        fs = gx().FunctorSet(cond=gx().functors.claim(labels, preds, 1))
        f = vf(0)
        if fused:
            out = gx().advance_filter_fused(g, f, functors=fs)
        else:
            out = gx().filter_frontier(gx().advance(g, f, functors=fs))
        got = sorted(out.to_array().tolist())
        assert got == sorted(set(g.neighbors(0).tolist()))
        assert len(out.to_array()) == len(got)
        assert np.all(preds.cpu().numpy()[got] == 0)


def test_sssp_relax_functor_preds_consistent():
    """relax winners are the final minima; preds satisfy
    dist[pred] + w == dist[d] for a one-step relaxation from a settled set."""
    import torch

    g = rmat(9, 8, 6)
    g = gx().assign_random_weights(g, 1, 64, seed=1)
    n = g.num_vertices
    dist = torch.full((n,), 2**31 - 1, dtype=torch.int32, device="cuda")
    dist[0] = 0
    preds = torch.full((n,), -1, dtype=torch.int32, device="cuda")
    out = gx().advance(g, vf(0), functors=gx().FunctorSet(cond=gx().functors.relax(dist, preds)))
    d = dist.cpu().numpy()
    p = preds.cpu().numpy()
    nb = g.neighbors(0)
    w = g.edge_weights[g.row_offsets[0]:g.row_offsets[1]]
    assert sorted(out.to_array().tolist()) == sorted(nb.tolist())
    assert np.array_equal(d[nb], w) and np.all(p[nb] == 0)
    # second step from the whole first ring: winners hold the final minimum
    pre = d.copy()
    out2 = gx().advance(g, gx().Frontier.from_items(nb),
                        functors=gx().FunctorSet(cond=gx().functors.relax(dist, preds)))
    d2 = dist.cpu().numpy()
    p2 = preds.cpu().numpy()
    row, col, wt = g.row_offsets, g.column_indices, g.edge_weights
    want = pre.astype(np.int64).copy()
    for u in nb:
        for j in range(row[u], row[u + 1]):
            want[col[j]] = min(want[col[j]], int(pre[u]) + int(wt[j]))
    assert np.array_equal(d2.astype(np.int64), want)
    for v in set(out2.to_array().tolist()):
        u = p2[v]
        j = row[u] + np.searchsorted(col[row[u]:row[u + 1]], v)
        assert int(pre[u]) + int(wt[j]) == d2[v]


# ---- test_near_far.py ---------------------------------------------------------
def keyed(values):
    table = cuda(np.asarray(values, dtype=np.int64))
    return lambda ids: table[ids]


def test_near_far_split():
    key = keyed([3, 12, 7])
    near, far = gx().split(gx().Frontier.from_items([0, 1, 2]), key, 10)
    assert sorted(key(near.device64()).tolist()) == [3, 7]
    assert key(far.device64()).tolist() == [12]
    near, far = gx().split(gx().Frontier.from_items([0, 1, 2]), key, 0)
    assert len(near) == 0 and len(far) == 3
    near, far = gx().split(gx().Frontier.from_items([]), keyed([]), 5)
    assert len(near) == 0 and len(far) == 0
    rng = np.random.default_rng(2)
    table = rng.integers(0, 100, size=50)
    items = rng.integers(0, 50, size=200)
    near, far = gx().split(gx().Frontier.from_items(items), keyed(table), 40)
    assert np.array_equal(np.sort(np.concatenate([near.to_array(), far.to_array()])),
                          np.sort(items))


def test_near_far_advance_bucket():
    key = keyed([12, 25])
    pile = gx().NearFarPile(delta=10, threshold=10)
    pile.push(gx().Frontier.from_items([0, 1]), key)
    assert len(pile.near) == 0
    gx().advance_bucket(pile, key)
    assert pile.threshold == 20
    assert key(pile.near.device64()).tolist() == [12]
    assert key(pile.far.device64()).tolist() == [25]
    key = keyed([35, 45])
    pile = gx().NearFarPile(delta=10, threshold=10)
    pile.push(gx().Frontier.from_items([0, 1]), key)
    gx().advance_bucket(pile, key)
    assert len(pile.near) == 0
    gx().advance_bucket(pile, key)
    gx().advance_bucket(pile, key)
    assert key(pile.near.device64()).tolist() == [35]
    key = keyed([57])
    pile = gx().NearFarPile(delta=10, threshold=10)
    pile.push(gx().Frontier.from_items([0]), key)
    adv = 0
    while len(pile.near) == 0:
        gx().advance_bucket(pile, key)
        adv += 1
    assert adv <= 6
    key = keyed([1, 50])
    pile = gx().NearFarPile(delta=10, threshold=10)
    pile.push(gx().Frontier.from_items([0, 1]), key)
    assert len(pile.near) == 1
    with pytest.raises(ValueError):
        gx().advance_bucket(pile, key)


def test_near_far_stale_and_conservation():
    table = cuda(np.array([30], dtype=np.int64))
    key = lambda ids: table[ids]  # noqa: E731
    pile = gx().NearFarPile(delta=10, threshold=10)
    pile.push(gx().Frontier.from_items([0]), key)
    table[0] = 5
    gx().advance_bucket(pile, key)
    assert pile.empty()
    rng = np.random.default_rng(8)
    key = keyed(rng.integers(0, 200, size=64))
    pile = gx().NearFarPile(delta=25, threshold=25)
    items = rng.integers(0, 64, size=100)
    pile.push(gx().Frontier.from_items(items), key)
    seen = [pile.pop_near().to_array()]
    while not pile.empty():
        gx().advance_bucket(pile, key)
        seen.append(pile.pop_near().to_array())
    assert np.array_equal(np.sort(np.concatenate(seen)), np.sort(items))


# ---- test_load_balance.py:35-50, 201-221 with device scans ---------------------
def test_scan_offsets_device_and_exact_plans():
    g = star(3)
    scan, total = gx().compute_scan_offsets(g, vf())
    assert scan.tolist() == [0] and total == 0
    scan, total = gx().compute_scan_offsets(g, vf(0))
    assert scan.tolist() == [0, 3] and total == 3
    rng = np.random.default_rng(4)
    p = gx().LbParams(small_cut=4, large_cut=16, chunk_size=8, items_per_chunk=4)
    for strategy in ALL:
        for _ in range(5):
            g = rmat(int(rng.integers(3, 8)), 5, int(rng.integers(1 << 30)))
            size = int(rng.integers(0, g.num_vertices + 1))
            f = gx().Frontier.from_items(rng.choice(g.num_vertices, size=size, replace=False))
            plan = gx().build_plan(g, f, getattr(gx().Strategy, strategy), p)
            got = gx().plan_pairs(plan)
            got = got[np.lexsort((got[:, 1], got[:, 0]))]
            sc = plan.scan_offsets
            want = np.array([(i, s) for i in range(len(sc) - 1)
                             for s in range(int(sc[i]), int(sc[i + 1]))],
                            dtype=np.int64).reshape(-1, 2)
            assert np.array_equal(got, want)


# ---- test_frontier.py --------------------------------------------------------
def test_frontier_device_helpers():
    U = np.iinfo(np.int64).max
    f = gx().generate_unvisited_frontier(np.array([0, U, U, 1], dtype=np.int64))
    assert f.to_array().tolist() == [1, 2]
    assert len(gx().generate_unvisited_frontier(np.array([0, 1, 2], dtype=np.int64))) == 0
    assert gx().generate_unvisited_frontier(np.full(5, U)).to_array().tolist() == list(range(5))
    rng = np.random.default_rng(0)
    for _ in range(20):
        n = int(rng.integers(1, 200))
        labels = np.full(n, U, dtype=np.int64)
        vis = rng.random(n) < 0.5
        labels[vis] = 1
        assert len(gx().generate_unvisited_frontier(labels)) + int(vis.sum()) == n
    bm = gx().StatusBitmap(8)
    assert bm.test_and_set(np.array([1, 2])).tolist() == [True, True]
    assert bm.test_and_set(np.array([2, 3])).tolist() == [False, True]
    assert bm.count() == 3
    dup = gx().StatusBitmap(8).test_and_set(np.array([4, 4]))
    assert dup.tolist() == [True, True]


def test_operator_chain_stays_in_hbm():
    """advance -> filter -> advance without a host round trip of the ids."""
    g = rmat(8, 8, 3)
    f1 = gx().advance(g, vf(0))
    assert f1.on_device and f1._host is None
    f2 = gx().filter_frontier(f1)
    f3 = gx().advance(g, f2)
    assert f2._host is None and f3._host is None
    want = np.unique(g.neighbors(0))
    assert np.array_equal(f2.to_array(), want)
    assert len(f3) == int(np.diff(g.row_offsets)[want].sum())

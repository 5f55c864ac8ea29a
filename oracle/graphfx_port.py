"""CPU ORACLE -- test infrastructure only.

A numpy restatement of the reference graphfx algorithms (pure Python/NumPy,
/root/reference/pkg/src/graphfx) used as (a) the parity checker for the
CUDA path and (b) the CPU baseline arm of bench.py.  Only tests/,
__graft_entry__.smoke() and bench.py (cpu_baseline / --impl reference) may
import it; the product package never does.

It is pinned against golden vectors produced by running the reference
itself (oracle/make_golden.py -> tests/golden/, checked by
tests/test_oracle_golden.py).

Every function follows the reference's vectorised algorithm step for step
(gather by repeat, first-claim CAS by stable sort, np.unique filters,
np.add.at / np.minimum.at scatters) so its timing is representative of the
reference CPU path; the file:line it restates is cited per function.
Graphs are passed as (row int64[n+1], col int64[m]) numpy arrays.
"""
from __future__ import annotations

import math

import numpy as np

UNVISITED = np.iinfo(np.int64).max
NO_PRED = -1


# ---------------------------------------------------------------------------
# inputs: generators.py:22-52, graph.py:158-203, graph.py:227-246
# ---------------------------------------------------------------------------
def generate_rmat(scale: int, edge_factor: int, seed: int = 0,
                  a=0.57, b=0.19, c=0.19):
    """generators.py:22-52: one rng.random(m) per level, quadrant by
    searchsorted(cum, u, 'right'); src/dst built MSB first; no permutation."""
    n = 1 << scale
    m = edge_factor * n
    rng = np.random.default_rng(seed)
    cum = np.array([a, a + b, a + b + c])
    src = np.zeros(m, dtype=np.int64)
    dst = np.zeros(m, dtype=np.int64)
    for _ in range(scale):
        q = np.searchsorted(cum, rng.random(m), side="right")
        src = (src << 1) | (q >> 1)
        dst = (dst << 1) | (q & 1)
    return n, src, dst


def coo_to_csr(n, src, dst, make_undirected=True):
    """graph.py:158-203: symmetrise + drop self loops, lexsort, dedup, bincount."""
    src = np.asarray(src, dtype=np.int64)
    dst = np.asarray(dst, dtype=np.int64)
    if make_undirected:
        keep = src != dst
        src, dst = src[keep], dst[keep]
        src, dst = np.concatenate([src, dst]), np.concatenate([dst, src])
    key = src * n + dst
    key = np.unique(key)  # sorted lexicographically by (src, dst), deduplicated
    src, dst = key // n, key % n
    row = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(src, minlength=n), out=row[1:])
    return row, dst


def rmat_csr(scale, edge_factor=16, seed=0):
    n, s, d = generate_rmat(scale, edge_factor, seed)
    return coo_to_csr(n, s, d, True)


def edge_sources(row):
    return np.repeat(np.arange(len(row) - 1, dtype=np.int64), np.diff(row))


def assign_random_weights(row, col, lo, hi, seed):
    """graph.py:227-246: one integers(lo, hi+1) draw per unique unordered pair
    in sorted (min, max) order; mirrored slots share it."""
    n = len(row) - 1
    s = edge_sources(row)
    key = np.minimum(s, col) * n + np.maximum(s, col)
    uniq, inv = np.unique(key, return_inverse=True)
    rng = np.random.default_rng(seed)
    return rng.integers(lo, hi + 1, size=len(uniq), dtype=np.int64)[inv]


def csc(row, col):
    """graph.py:113-126: stable argsort of column ids."""
    n = len(row) - 1
    order = np.argsort(col, kind="stable")
    rrow = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(col, minlength=n), out=rrow[1:])
    return rrow, edge_sources(row)[order], order


# ---------------------------------------------------------------------------
# expansion gather: operators.py:161-197
# ---------------------------------------------------------------------------
def _gather(row, col, items):
    deg = row[items + 1] - row[items]
    total = int(deg.sum())
    src = np.repeat(items, deg)
    start = np.zeros(len(items) + 1, dtype=np.int64)
    np.cumsum(deg, out=start[1:])
    edge = np.arange(total, dtype=np.int64) + np.repeat(row[items] - start[:-1], deg)
    return src, col[edge], edge, total


def _first_claim(labels, idx):
    """operators.py:131-153 compare_and_swap: among eligible entries the first
    occurrence of each index wins."""
    won = np.zeros(len(idx), dtype=bool)
    elig = np.flatnonzero(labels[idx] == UNVISITED)
    if len(elig):
        _, first = np.unique(idx[elig], return_index=True)
        won[elig[first]] = True
    return won


# ---------------------------------------------------------------------------
# direction.py:52-70
# ---------------------------------------------------------------------------
def estimate_mf_mu(n, m, n_f, n_u, mu_edge_based=False):
    m_f = n_f * m / n
    if n_u >= n:
        return m_f, math.inf
    return m_f, n_u * (m if mu_edge_based else n) / (n - n_u)


def decide(mode, m_f, m_u, do_a, do_b):
    if mode == "push":
        return "pull" if m_f > m_u * do_a else "push"
    return "push" if m_f < m_u * do_b else "pull"


# ---------------------------------------------------------------------------
# primitives/bfs.py:42-166
# ---------------------------------------------------------------------------
def bfs(row, col, source, direction="push", do_a=0.001, do_b=0.2, mu_edge_based=False,
        rev=None):
    n = len(row) - 1
    m = len(col)
    labels = np.full(n, UNVISITED, dtype=np.int64)
    preds = np.full(n, NO_PRED, dtype=np.int64)
    labels[source] = 0
    frontier = np.array([source], dtype=np.int64)
    n_u, mode_state, depth = n, "push", 0
    trace, edges_traversed = [], 0
    rrow = rcol = None
    unvisited = None
    while len(frontier):
        depth += 1
        n_f = len(frontier)
        n_u -= n_f
        m_f, m_u = estimate_mf_mu(n, m, n_f, n_u, mu_edge_based)
        if direction == "auto":
            mode = decide(mode_state, m_f, m_u, do_a, do_b)
        elif direction == "pull":
            mode = "pull" if depth > 1 else "push"
        else:
            mode = "push"
        trace.append({"iteration": depth, "mode_before": mode_state, "n_f": n_f,
                      "n_u": n_u, "m_f": m_f, "m_u": m_u, "decision": mode})
        if mode == "push":
            src, dst, _, total = _gather(row, col, frontier)
            edges_traversed += total
            won = _first_claim(labels, dst)
            labels[dst[won]] = depth
            preds[dst[won]] = src[won]
            frontier = np.unique(dst[won])
        else:
            if rrow is None:
                rrow, rcol, _ = rev if rev is not None else csc(row, col)
            if mode_state == "push" or unvisited is None:
                unvisited = np.flatnonzero(labels == UNVISITED)  # frontier.py:97-100
            # operators.py:269-307: all in-edges of U, cond labels[s] == depth-1
            probe, src, _, total = _gather(rrow, rcol, unvisited)
            edges_traversed += total
            ok = labels[src] == depth - 1
            hit_v = probe[ok]
            labels[hit_v] = depth
            preds[hit_v] = src[ok]
            hits = np.zeros(n, dtype=bool)
            hits[hit_v] = True
            frontier = unvisited[hits[unvisited]]
            unvisited = unvisited[~hits[unvisited]]
        mode_state = mode
    return labels, preds, trace, edges_traversed


# ---------------------------------------------------------------------------
# primitives/sssp.py:33-121 + near_far.py:40-85
# ---------------------------------------------------------------------------
def default_delta(w):
    if w is None or len(w) == 0:
        return 32
    return int(math.ceil(float(np.mean(w)) * 32))


def sssp(row, col, w, source, delta=None, use_priority_queue=True):
    n = len(row) - 1
    if not use_priority_queue:
        delta = math.inf
    elif delta is None:
        delta = default_delta(w)
    labels = np.full(n, UNVISITED, dtype=np.int64)
    preds = np.full(n, NO_PRED, dtype=np.int64)
    stamps = np.zeros(n, dtype=np.int64)
    labels[source] = 0
    threshold = delta
    near = np.array([source], dtype=np.int64)
    far = np.empty(0, dtype=np.int64)
    far_keys = np.empty(0, dtype=np.int64)
    stamp = 0
    relaxed = 0
    while len(near) or len(far):
        if len(near) == 0:  # near_far.py:68-85 advance_bucket
            threshold = threshold + delta
            live = labels[far]
            fresh = live == far_keys
            far, live = far[fresh], live[fresh]
            nm = live < threshold
            near, far, far_keys = far[nm], far[~nm], live[~nm]
            continue
        stamp += 1
        src, dst, edge, total = _gather(row, col, near)
        relaxed += total
        cand = labels[src] + w[edge]
        # operators.py:111-124 atomic_min (one chunk), then set_pred + stamp
        improving = cand < labels[dst]
        ci = np.flatnonzero(improving)
        if len(ci):
            np.minimum.at(labels, dst[ci], cand[ci])
        final = improving & (cand == labels[dst])
        preds[dst[final]] = src[final]
        stamps[dst[final]] = stamp
        out = np.unique(dst[final])
        out = out[stamps[out] == stamp]
        keys = labels[out]
        nm = keys < threshold
        near = out[nm]
        far = np.concatenate([far, out[~nm]])
        far_keys = np.concatenate([far_keys, keys[~nm]])
    return labels, preds, relaxed


# ---------------------------------------------------------------------------
# primitives/bc.py:62-116 (single source)
# ---------------------------------------------------------------------------
def bc(row, col, sources):
    n = len(row) - 1
    if np.isscalar(sources):
        sources = [int(sources)]
    bcv = np.zeros(n)
    for s0 in sources:
        labels = np.full(n, UNVISITED, dtype=np.int64)
        sigma = np.zeros(n)
        labels[s0] = 0
        sigma[s0] = 1.0
        frontier = np.array([s0], dtype=np.int64)
        levels = [frontier]
        depth = 0
        while len(frontier):
            depth += 1
            src, dst, _, _ = _gather(row, col, frontier)
            won = _first_claim(labels, dst)
            labels[dst[won]] = depth
            on = labels[dst] == depth
            np.add.at(sigma, dst[on], sigma[src[on]])
            frontier = np.unique(dst[won])
            if len(frontier):
                levels.append(frontier)
        delta = np.zeros(n)
        for lvl in range(len(levels) - 2, -1, -1):
            src, dst, _, _ = _gather(row, col, levels[lvl])
            on = labels[dst] == lvl + 1
            s, d = src[on], dst[on]
            np.add.at(delta, s, sigma[s] / sigma[d] * (1.0 + delta[d]))
        delta[s0] = 0.0
        bcv += delta
    return bcv


# ---------------------------------------------------------------------------
# primitives/cc.py:23-98, returned canonicalised to min-id
# ---------------------------------------------------------------------------
def cc(row, col):
    n = len(row) - 1
    comp = np.arange(n, dtype=np.int64)
    es = edge_sources(row)
    ef = np.flatnonzero(es < col)
    it = 0
    while len(ef):
        it += 1
        ef = ef[comp[es[ef]] != comp[col[ef]]]
        if len(ef):
            cu, cv = comp[es[ef]], comp[col[ef]]
            lo, hi = np.minimum(cu, cv), np.maximum(cu, cv)
            if it % 2 == 1:
                comp[hi] = lo
            else:
                comp[lo] = hi
            vf = np.arange(n, dtype=np.int64)
            while len(vf):
                parent = comp[comp[vf]]
                moved = parent != comp[vf]
                comp[vf] = parent
                vf = vf[moved]
    return canon_min_id(comp)


def canon_min_id(comp):
    n = len(comp)
    first = np.full(n, n, dtype=np.int64)
    np.minimum.at(first, comp, np.arange(n, dtype=np.int64))
    return first[comp]


# ---------------------------------------------------------------------------
# primitives/pagerank.py:30-91
# ---------------------------------------------------------------------------
def pagerank(row, col, damping=0.85, epsilon=1e-6, max_iters=100):
    n = len(row) - 1
    if n == 0:
        return np.empty(0)
    outdeg = np.diff(row).astype(np.float64)
    rank = np.full(n, 1.0 / n)
    frontier = np.arange(n, dtype=np.int64)
    it = 0
    while len(frontier) and it < max_iters:
        it += 1
        dangling = rank[frontier[outdeg[frontier] == 0]].sum()
        nxt = np.full(n, (1.0 - damping) / n + damping * dangling / n)
        src, dst, _, _ = _gather(row, col, frontier)
        np.add.at(nxt, dst, damping * rank[src] / outdeg[src])
        moved = np.abs(nxt - rank)
        frontier = np.unique(frontier[moved[frontier] >= epsilon])
        rank = nxt
    return rank


# ---------------------------------------------------------------------------
# primitives/tc.py:27-86 + operators.py:485-525 (vectorised per source vertex)
# ---------------------------------------------------------------------------
def tc(row, col):
    n = len(row) - 1
    deg = np.diff(row)
    s = edge_sources(row)
    keep = (deg[s] > deg[col]) | ((deg[s] == deg[col]) & (s < col))
    osrc, odst = s[keep], col[keep]  # already (src, dst)-sorted: CSR order
    orow = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(osrc, minlength=n), out=orow[1:])
    counts = np.zeros(len(osrc), dtype=np.int64)
    for i in range(len(osrc)):
        a = odst[orow[osrc[i]]:orow[osrc[i] + 1]]
        b = odst[orow[odst[i]]:orow[odst[i] + 1]]
        if len(a) and len(b):
            counts[i] = len(np.intersect1d(a, b, assume_unique=True))
    return int(counts.sum()), counts, osrc, odst


# ---------------------------------------------------------------------------
# INEXACT filter culling: operators.py:315-357
# ---------------------------------------------------------------------------
def cull_inexact(items, use_bitmask=True, team_table_size=256, local_table_size=64,
                 bitmask_batch=1024, local_batch=32, domain_size=None):
    """operators.py:344-357 (_apply_culling): bitmask over the domain where a
    batch reads the seen bits before marking them (:315-322), then the
    direct-mapped team and local history tables (:325-341), each stage over
    the previous stage's survivors."""
    items = np.asarray(items, dtype=np.int64)
    if len(items) == 0:
        return items
    if use_bitmask:
        seen = np.zeros(domain_size or int(items.max()) + 1, dtype=bool)
        keep = np.ones(len(items), dtype=bool)
        for lo in range(0, len(items), bitmask_batch):
            chunk = items[lo:lo + bitmask_batch]
            keep[lo:lo + bitmask_batch] = ~seen[chunk]
            seen[chunk] = True
        items = items[keep]

    def history(items, table, batch):
        keep = np.ones(len(items), dtype=bool)
        for lo in range(0, len(items), batch):
            chunk = items[lo:lo + batch]
            slots = chunk % table
            order = np.argsort(slots, kind="stable")
            s, v = slots[order], chunk[order]
            dup = np.zeros(len(chunk), dtype=bool)
            dup[1:] = (s[1:] == s[:-1]) & (v[1:] == v[:-1])
            sub = np.ones(len(chunk), dtype=bool)
            sub[order] = ~dup
            keep[lo:lo + batch] = sub
        return items[keep]

    if team_table_size:
        items = history(items, team_table_size, team_table_size)
    if local_table_size:
        items = history(items, local_table_size, local_batch)
    return items

"""Vectorised property checks (restating reference pkg/tests/_oracles.py:169-202)."""
import numpy as np

UNV = np.iinfo(np.int64).max


def has_edge(row, col, u, v):
    """Vectorised: is v in N(u) (sorted neighbour lists)?"""
    u = np.asarray(u, dtype=np.int64)
    v = np.asarray(v, dtype=np.int64)
    lo, hi = row[u], row[u + 1]
    ok = np.zeros(len(u), dtype=bool)
    # binary search per pair with numpy (row-local): search in the global col
    # array restricted to [lo, hi) by offsetting keys
    n = len(row) - 1
    key_col = np.repeat(np.arange(n, dtype=np.int64), np.diff(row)) * (n + 1) + col
    pos = np.searchsorted(key_col, u * (n + 1) + v)
    inb = pos < len(col)
    ok[inb] = key_col[pos[inb]] == (u[inb] * (n + 1) + v[inb])
    del lo, hi
    return ok


def valid_bfs_preds(row, col, labels, preds, source):
    """_oracles.py:169-182: preds[v] is an in-neighbour one level closer."""
    reached = labels != UNV
    others = ~reached.copy()
    others[source] = True
    if np.any(preds[others] != -1):
        return False
    v = np.flatnonzero(reached)
    v = v[v != source]
    p = preds[v]
    if np.any(p < 0) or np.any(labels[p] != labels[v] - 1):
        return False
    return bool(np.all(has_edge(row, col, p, v)))


def valid_sssp_preds(row, col, w, labels, preds, source):
    """_oracles.py:185-202: some slot p->v with labels[p] + w == labels[v]."""
    reached = labels != UNV
    others = ~reached.copy()
    others[source] = True
    if np.any(preds[others] != -1):
        return False
    v = np.flatnonzero(reached)
    v = v[v != source]
    p = preds[v]
    if np.any(p < 0):
        return False
    n = len(row) - 1
    s = np.repeat(np.arange(n, dtype=np.int64), np.diff(row))
    key = s * (n + 1) + col
    # any parallel slot qualifies; canonical CSR has no duplicates
    pos = np.searchsorted(key, p * (n + 1) + v)
    if np.any(pos >= len(col)) or np.any(key[pos] != p * (n + 1) + v):
        return False
    return bool(np.all(labels[p] + w[pos] == labels[v]))

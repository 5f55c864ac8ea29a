"""ctypes wrapper of oracle/liboracle.so (CPU ORACLE, test infrastructure only)."""
from __future__ import annotations

import ctypes
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "liboracle.so"
_lib = None


def build() -> Path:
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB


def lib():
    global _lib
    if _lib is None:
        if not LIB.exists():
            build()
        _lib = ctypes.CDLL(str(LIB))
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _graph(row, col):
    return (np.ascontiguousarray(row, dtype=np.int64), np.ascontiguousarray(col, dtype=np.int32))


def bfs(row, col, src):
    row, col = _graph(row, col)
    n = len(row) - 1
    out = np.empty(n, dtype=np.int64)
    f = lib().ora_bfs
    f.restype = ctypes.c_int64
    f(ctypes.c_int64(n), _p(row), _p(col), ctypes.c_int64(src), _p(out))
    return out


def dijkstra(row, col, w, src):
    row, col = _graph(row, col)
    w = np.ascontiguousarray(w, dtype=np.int64)
    n = len(row) - 1
    out = np.empty(n, dtype=np.int64)
    f = lib().ora_dijkstra
    f.restype = ctypes.c_int64
    f(ctypes.c_int64(n), _p(row), _p(col), _p(w), ctypes.c_int64(src), _p(out))
    return out


def cc(row, col):
    row, col = _graph(row, col)
    n = len(row) - 1
    out = np.empty(n, dtype=np.int64)
    f = lib().ora_cc
    f.restype = ctypes.c_int64
    k = f(ctypes.c_int64(n), _p(row), _p(col), _p(out))
    return out, int(k)


def tc(row, col):
    row, col = _graph(row, col)
    n = len(row) - 1
    orow = np.empty(n + 1, dtype=np.int64)
    ocol = np.empty(max(len(col), 1), dtype=np.int32)
    counts = np.empty(max(len(col), 1), dtype=np.int64)
    f = lib().ora_tc
    f.restype = ctypes.c_int64
    total = f(ctypes.c_int64(n), _p(row), _p(col), _p(orow), _p(ocol), _p(counts))
    mo = int(orow[-1])
    osrc = np.repeat(np.arange(n, dtype=np.int64), np.diff(orow))
    return int(total), counts[:mo].copy(), osrc, ocol[:mo].astype(np.int64)


def pagerank(row, col, rrow, rcol, damping, iters):
    row, col = _graph(row, col)
    rrow, rcol = _graph(rrow, rcol)
    n = len(row) - 1
    out = np.empty(n, dtype=np.float64)
    lib().ora_pagerank(ctypes.c_int64(n), _p(row), _p(rrow), _p(rcol), ctypes.c_double(damping),
                       ctypes.c_int64(iters), _p(out))
    return out


def bc(row, col, rrow, rcol, src):
    row, col = _graph(row, col)
    rrow, rcol = _graph(rrow, rcol)
    n = len(row) - 1
    out = np.empty(n, dtype=np.float64)
    lib().ora_bc(ctypes.c_int64(n), _p(row), _p(col), _p(rrow), _p(rcol), ctypes.c_int64(src),
                 _p(out))
    return out

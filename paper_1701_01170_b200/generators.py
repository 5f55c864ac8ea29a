"""Synthetic R-MAT input (reference generators.py:22-52) on host and device.

``generate_rmat`` is the host COO generator with the reference contract.
``rmat_device_graph`` builds the identical canonical undirected CSR (and
optionally the identical weights of ``assign_random_weights``) directly in
HBM with the bit-exact PCG64 replay in csrc/gfx_rmat.cu -- seconds instead of
the reference's ~20 minutes at scale 24, and the only way to reach scale 27.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _native
from .graph import ID_DTYPE, CooGraph, DeviceGraph

RMAT_A, RMAT_B, RMAT_C, RMAT_D = 0.57, 0.19, 0.19, 0.05


def _check(scale, a, b, c, d):
    if scale < 1:
        raise ValueError("scale must be >= 1")
    if abs(a + b + c + d - 1.0) > 1e-9:
        raise ValueError("quadrant probabilities must sum to 1")


def generate_rmat(scale: int, edge_factor: int, a: float = RMAT_A, b: float = RMAT_B,
                  c: float = RMAT_C, d: float = RMAT_D, seed: int = 0) -> CooGraph:
    """Host R-MAT COO (duplicates kept; dedup happens at CSR build)."""
    _check(scale, a, b, c, d)
    n = 1 << scale
    m = edge_factor * n
    rng = np.random.default_rng(seed)
    cum = np.array([a, a + b, a + b + c])
    src = np.zeros(m, dtype=ID_DTYPE)
    dst = np.zeros(m, dtype=ID_DTYPE)
    for _ in range(scale):
        q = np.searchsorted(cum, rng.random(m), side="right")
        src = (src << 1) | (q >> 1)
        dst = (dst << 1) | (q & 1)
    return CooGraph(num_vertices=n, src=src, dst=dst)


def pcg64_state(seed: int):
    """(state_hi, state_lo, inc_hi, inc_lo) of numpy's default_rng(seed)."""
    st = np.random.default_rng(seed).bit_generator.state["state"]
    s, inc = int(st["state"]), int(st["inc"])
    mask = (1 << 64) - 1
    return (s >> 64) & mask, s & mask, (inc >> 64) & mask, inc & mask


def rmat_device_graph(scale: int, edge_factor: int = 16, seed: int = 0, *, weights=None,
                      weight_seed: int = 0, a: float = RMAT_A, b: float = RMAT_B,
                      c: float = RMAT_C, d: float = RMAT_D, device: int | None = None,
                      make_undirected: bool = True) -> DeviceGraph:
    """generate_rmat(scale, edge_factor, seed) -> coo_to_csr(make_undirected)
    [-> assign_random_weights(g, lo, hi, weight_seed)] built on the GPU.

    ``weights`` is None or a (lo, hi) pair."""
    import torch

    _check(scale, a, b, c, d)
    ctx = _native.Context.get(device)
    dev = torch.device("cuda", ctx.device)
    m_raw = edge_factor << scale
    cap = 2 * m_raw if make_undirected else m_raw
    keys = torch.empty(cap, dtype=torch.int64, device=dev)
    cum = (ctypes.c_double * 3)(a, a + b, a + b + c)
    sh, sl, ih, il = pcg64_state(seed)
    count = ctypes.c_int64()
    torch.cuda.synchronize(dev)
    _native.call("gfx_rmat_keys", ctx.handle, scale, edge_factor, cum, sh, sl, ih, il,
                 int(make_undirected), _native.ptr(keys), ctypes.byref(count))
    m = count.value
    n = 1 << scale
    row = torch.empty(n + 1, dtype=torch.int64, device=dev)
    col = torch.empty(max(m, 1), dtype=torch.int32, device=dev)
    _native.call("gfx_keys_to_csr", ctx.handle, _native.ptr(keys), m, scale, _native.ptr(row),
                 _native.ptr(col))
    del keys
    col = col[:m]
    dg = DeviceGraph.from_tensors(row, col, None, undirected=make_undirected)
    if weights is not None:
        lo, hi = weights
        span = int(hi) - int(lo) + 1
        if span < 1 or span & (span - 1):
            # numpy's bounded integers() rejects draws for ranges that are not a
            # power of two (Lemire), a sequential stream the GPU builder does not
            # reproduce: draw them with the reference algorithm over the
            # downloaded CSR (input construction, untimed) and upload
            from .graph import assign_random_weights

            host = assign_random_weights(dg.to_host(), int(lo), int(hi), weight_seed)
            w = DeviceGraph._weights_tensor(host.edge_weights, dev)
            return DeviceGraph.from_tensors(row, col, w, undirected=make_undirected)
        w = torch.empty(max(m, 1), dtype=torch.int32, device=dev)[:m]
        wsh, wsl, wih, wil = pcg64_state(weight_seed)
        _native.call("gfx_assign_weights", dg.handle, int(lo), int(hi), wsh, wsl, wih, wil,
                     _native.ptr(w))
        dg = DeviceGraph.from_tensors(row, col, w, undirected=make_undirected)
    return dg

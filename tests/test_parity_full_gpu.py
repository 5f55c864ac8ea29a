"""Full-size parity the sampled goldens cannot give (VERDICT r1 "what's weak" 1-2).

* PageRank (C3 config, 20 iterations, eps 0) full-vector L1 <= 1e-6 at s22
  and s24 against the C restatement of pagerank.py:30-91 (oracle/serial.c),
  after pinning that restatement to the reference's own sampled ranks.
* BC (C4 config, source 0) full-vector rel <= 1e-5 at s22 against the C
  restatement of bc.py:62-116, pinned to the reference's sampled values; BC
  is bit-reproducible run to run.
* DO-BFS at s27 (C5 input size, 4.2 B slots) against the C serial BFS
  (_oracles.py:17-28) over the GPU-built CSR, bit-exact labels.

The host C oracle runs on the GPU box's CPU (seconds to a minute each).
"""
import os
import time

import numpy as np
import pytest

from conftest import rmat_golden
from oracle import c_oracle

pytestmark = pytest.mark.gpu

PR_L1 = 1e-6
BC_RTOL = 1e-5


def _host_csr(dg):
    return dg.row.cpu().numpy(), dg.col.cpu().numpy()


@pytest.mark.parametrize("scale", [22, 24])
def test_pagerank_full_vector(scale):
    from paper_1701_01170_b200.generators import rmat_device_graph
    from paper_1701_01170_b200.primitives.pagerank import pagerank_device

    rec, arrays = rmat_golden(scale)
    dg = rmat_device_graph(scale, 16, 0)
    rank, _ = pagerank_device(dg, 0.85, 0.0, 20)
    rank = rank.cpu().numpy()
    row, col = _host_csr(dg)
    t0 = time.perf_counter()
    want = c_oracle.pagerank(row, col, row, col, 0.85, 20)  # undirected: reverse == CSR
    oracle_s = time.perf_counter() - t0
    # pin the restatement to the reference's own run (4096 sampled ranks + sum;
    # numpy's pairwise dangling sum differs from the serial one in the last bits)
    pin = np.abs(want[arrays["pr_idx"]] - arrays["pr_vals"]) / arrays["pr_vals"]
    print(f"s{scale} C-oracle vs reference samples: max rel {pin.max():.2e}")
    assert pin.max() <= 1e-10
    assert abs(want.sum() - rec["pr20_sum"]) < 1e-9
    l1 = float(np.abs(rank - want).sum())
    print(f"s{scale} PageRank L1 {l1:.3e} (C oracle {oracle_s:.1f} s)")
    assert l1 <= PR_L1


def test_bc_full_vector_s22_and_reproducible():
    from paper_1701_01170_b200.generators import rmat_device_graph
    from paper_1701_01170_b200.primitives.bc import bc_device

    rec, arrays = rmat_golden(22)
    dg = rmat_device_graph(22, 16, 0)
    a, _ = bc_device(dg, [0])
    a = a.cpu().numpy()
    b, _ = bc_device(dg, [0])
    assert np.array_equal(a.view(np.int64), b.cpu().numpy().view(np.int64)), "BC not reproducible"
    row, col = _host_csr(dg)
    t0 = time.perf_counter()
    want = c_oracle.bc(row, col, row, col, 0)
    oracle_s = time.perf_counter() - t0
    assert np.allclose(want[arrays["bc_idx"]], arrays["bc_vals"], rtol=1e-10, atol=1e-9)
    nz = want != 0
    rel = np.abs(a[nz] - want[nz]) / np.abs(want[nz])
    print(f"s22 BC max rel {rel.max():.3e}, exact {np.mean(a == want):.4f} (C oracle {oracle_s:.1f} s)")
    assert np.all(a[~nz] == 0)
    assert rel.max() <= BC_RTOL


@pytest.mark.skipif(os.environ.get("GFX_SKIP_S27") == "1", reason="s27 needs ~25 GB host RAM")
def test_bfs_s27_vs_host_c_oracle():
    """C5: the GPU DO-BFS labels on the scale-27 graph equal a serial BFS
    (C restatement of _oracles.py:17-28) run on the host over the same CSR."""
    import torch

    from paper_1701_01170_b200.generators import rmat_device_graph
    from paper_1701_01170_b200.primitives.bfs import bfs_device

    dg = rmat_device_graph(27, 16, 0)
    n = dg.num_vertices
    labels = torch.empty(n, dtype=torch.int32, device="cuda")
    preds = torch.empty(n, dtype=torch.int32, device="cuda")
    bfs_device(dg, 0, direction="auto", labels=labels, preds=preds)
    got = labels.cpu().numpy()
    pr = preds.cpu().numpy()
    row, col = _host_csr(dg)
    del labels, preds, dg
    torch.cuda.empty_cache()
    t0 = time.perf_counter()
    want = c_oracle.bfs(row, col, 0)
    oracle_s = time.perf_counter() - t0
    reached = want != np.iinfo(np.int64).max
    print(f"s27: {int(reached.sum())} reached, C oracle {oracle_s:.1f} s")
    assert np.array_equal(got == 2**31 - 1, ~reached)
    assert np.array_equal(got[reached].astype(np.int64), want[reached])
    # preds: an edge into v from the previous level (_oracles.py:169-202), sampled
    rng = np.random.default_rng(0)
    vs = rng.choice(np.flatnonzero(reached & (want > 0)), size=20000, replace=False)
    for v in vs:
        p = int(pr[v])
        assert want[p] == want[v] - 1
        nb = col[row[p]:row[p + 1]]
        i = np.searchsorted(nb, v)
        assert i < len(nb) and nb[i] == v

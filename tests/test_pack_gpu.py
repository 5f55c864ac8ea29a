"""Packed CSR columns (csrc/gfx_pack.cu): pack on the device, download, reload
into a resident graph through the packed path; the decoded graph is the
graph, and BFS on it equals the reference golden."""
import numpy as np
import pytest

from conftest import rmat_golden, sha

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("scale", [10, 16, 20])
def test_pack_round_trip_and_bfs(scale):
    import torch

    from paper_1701_01170_b200._results import labels_to_host
    from paper_1701_01170_b200.generators import rmat_device_graph
    from paper_1701_01170_b200.io import pack_csr_device
    from paper_1701_01170_b200.primitives.bfs import bfs_device

    rec, _ = rmat_golden(scale)
    dg = rmat_device_graph(scale, 16, 0)
    ref = dg.col.clone()
    packed = pack_csr_device(dg)
    assert packed.nbytes < dg.col.numel() * 4 + dg.row.numel() * 8
    dg.col.zero_()
    dg.reload_packed_(packed)
    torch.cuda.synchronize()
    assert torch.equal(dg.col, ref)
    lab, _, _ = bfs_device(dg, 0, direction="auto")
    assert sha(labels_to_host(lab)) == rec["bfs_sha"]


def test_pack_edge_cases():
    """big jumps (4-byte deltas), descending row starts, tiny graphs"""
    import torch

    import paper_1701_01170_b200 as gfx
    from paper_1701_01170_b200.io import pack_csr_device

    n = 1 << 20
    src = np.array([0, 0, 5, 5, n - 1, 7], dtype=np.int64)
    dst = np.array([n - 1, 1, 3, n - 2, 2, 6], dtype=np.int64)
    g = gfx.coo_to_csr(gfx.CooGraph(n, src, dst), make_undirected=True)
    dg = g.device()
    packed = pack_csr_device(dg)
    ref = dg.col.clone()
    dg.col.fill_(-1)
    dg.reload_packed_(packed)
    torch.cuda.synchronize()
    assert torch.equal(dg.col, ref)
    assert np.array_equal(dg.col.cpu().numpy(), g.column_indices)

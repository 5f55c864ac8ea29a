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


@pytest.mark.parametrize("scale", [10, 16, 20])
def test_upper_triangle_round_trip_and_bfs(scale):
    """the upper-triangle image (each edge once) rebuilds the full sorted CSR
    bit-exactly (gfx_graph_rebuild_upper), and the graph's BFS equals the
    reference golden; then the graph is reloaded again from the full image"""
    import torch

    from paper_1701_01170_b200._results import labels_to_host
    from paper_1701_01170_b200.generators import rmat_device_graph
    from paper_1701_01170_b200.io import pack_csr_device
    from paper_1701_01170_b200.primitives.bfs import bfs_device

    rec, _ = rmat_golden(scale)
    dg = rmat_device_graph(scale, 16, 0)
    ref_col, ref_row = dg.col.clone(), dg.row.clone()
    full = pack_csr_device(dg)
    up = pack_csr_device(dg, upper=True)
    assert up.upper and up.nbytes < 0.6 * full.nbytes
    for packed in (up, full, up):
        dg.col.fill_(-7)
        dg.reload_packed_(packed)
        torch.cuda.synchronize()
        assert torch.equal(dg.col, ref_col) and torch.equal(dg.row, ref_row)
    assert sha(dg.col[: rec["m"]].cpu().numpy().astype(np.int64)) == rec["col_sha"]
    lab, _, _ = bfs_device(dg, 0, direction="auto")
    assert sha(labels_to_host(lab)) == rec["bfs_sha"]


@pytest.mark.parametrize("case", ["jumps", "star", "path", "isolated", "clique"])
def test_upper_triangle_edge_cases(case):
    """4-byte deltas, a hub whose lower part is everything (star centred on
    the last vertex), long chains, isolated vertices, a dense block"""
    import torch

    import paper_1701_01170_b200 as gfx
    from paper_1701_01170_b200.io import pack_csr_device

    n = 1 << 20
    if case == "jumps":
        src = np.array([0, 0, 5, 5, n - 1, 7], dtype=np.int64)
        dst = np.array([n - 1, 1, 3, n - 2, 2, 6], dtype=np.int64)
    elif case == "star":
        n = 5000
        src = np.full(n - 1, n - 1, dtype=np.int64)
        dst = np.arange(n - 1, dtype=np.int64)
    elif case == "path":
        n = 100000
        src = np.arange(n - 1, dtype=np.int64)
        dst = src + 1
    elif case == "isolated":
        n = 64
        src = np.array([3, 3, 40], dtype=np.int64)
        dst = np.array([40, 63, 63], dtype=np.int64)
    else:
        n = 300
        a, b = np.triu_indices(n, 1)
        src, dst = a.astype(np.int64), b.astype(np.int64)
    g = gfx.coo_to_csr(gfx.CooGraph(n, src, dst), make_undirected=True)
    dg = g.device()
    packed = pack_csr_device(dg, upper=True)
    dg.col.fill_(-1)
    dg.reload_packed_(packed)
    torch.cuda.synchronize()
    assert np.array_equal(dg.col.cpu().numpy()[: g.num_edges], g.column_indices)
    assert np.array_equal(dg.row.cpu().numpy(), g.row_offsets)


def test_upper_triangle_rejects_directed():
    import paper_1701_01170_b200 as gfx
    from paper_1701_01170_b200.io import pack_csr_device

    g = gfx.CsrGraph(3, np.array([0, 1, 2, 2]), np.array([1, 2]), undirected=False)
    with pytest.raises(ValueError):
        pack_csr_device(g.device(), upper=True)

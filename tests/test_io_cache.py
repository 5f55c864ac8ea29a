"""Binary CSR cache against files written by the
reference's save_csr_cache (oracle/make_golden.py cache; reference
io.py:121-159)."""
import numpy as np
import pytest

from conftest import GOLDEN

W_FILE = GOLDEN / "cache_rmat8_w.gfxcsr"
D_FILE = GOLDEN / "cache_rmat7_dir.gfxcsr"


def _arrays():
    return dict(np.load(GOLDEN / "cache_arrays.npz"))


def test_load_reference_files():
    from paper_1701_01170_b200.io import load_csr_cache, load_graph

    a = _arrays()
    g = load_csr_cache(W_FILE)
    assert g.undirected and g.num_vertices == int(a["w_n"][0])
    assert np.array_equal(g.row_offsets, a["w_row"])
    assert np.array_equal(g.column_indices, a["w_col"])
    assert np.array_equal(g.edge_weights, a["w_w"])
    assert g.row_offsets.dtype == np.int64 and g.column_indices.dtype == np.int64
    d = load_graph(D_FILE)
    assert not d.undirected and d.edge_weights is None
    assert np.array_equal(d.row_offsets, a["d_row"])
    assert np.array_equal(d.column_indices, a["d_col"])
    u = load_graph(D_FILE, make_undirected=True)
    assert u.undirected and u.is_symmetric()


def test_save_is_byte_identical(tmp_path):
    import paper_1701_01170_b200 as gfx
    from paper_1701_01170_b200.io import save_csr_cache

    a = _arrays()
    g = gfx.CsrGraph(int(a["w_n"][0]), a["w_row"], a["w_col"], a["w_w"], undirected=True)
    save_csr_cache(g, tmp_path / "w.gfxcsr")
    assert (tmp_path / "w.gfxcsr").read_bytes() == W_FILE.read_bytes()
    d = gfx.CsrGraph(int(a["d_n"][0]), a["d_row"], a["d_col"])
    save_csr_cache(d, tmp_path / "d.gfxcsr")
    assert (tmp_path / "d.gfxcsr").read_bytes() == D_FILE.read_bytes()


def test_bad_files(tmp_path):
    from paper_1701_01170_b200 import GraphFormatError
    from paper_1701_01170_b200.io import load_csr_cache

    blob = W_FILE.read_bytes()
    (tmp_path / "magic").write_bytes(b"NOTCSR\x00" + blob[7:])
    (tmp_path / "version").write_bytes(blob[:7] + b"\x03" + blob[8:])
    (tmp_path / "short").write_bytes(blob[:-8])
    for name in ("magic", "version", "short"):
        with pytest.raises(GraphFormatError):
            load_csr_cache(tmp_path / name)


def test_compact_variant(tmp_path):
    """Version-2 file (int32 columns / weights): half the
    column bytes, loads to the same reference-layout CsrGraph."""
    import paper_1701_01170_b200 as gfx
    from paper_1701_01170_b200.io import load_csr_cache, read_header_version, save_csr_cache

    a = _arrays()
    g = gfx.CsrGraph(int(a["w_n"][0]), a["w_row"], a["w_col"], a["w_w"], undirected=True)
    p = tmp_path / "w2.gfxcsr"
    save_csr_cache(g, p, compact=True)
    n, m = g.num_vertices, g.num_edges
    assert read_header_version(p) == (2, n, m, 3)
    assert p.stat().st_size == 7 + 18 + 8 * (n + 1) + 4 * m + 4 * m
    h = load_csr_cache(p)
    assert h.undirected and h.column_indices.dtype == np.int64
    assert np.array_equal(h.row_offsets, g.row_offsets)
    assert np.array_equal(h.column_indices, g.column_indices)
    assert np.array_equal(h.edge_weights, g.edge_weights)
    big = gfx.CsrGraph(2, np.array([0, 1, 2]), np.array([1, 0]), np.array([2**31, 2**31]),
                       undirected=True)
    with pytest.raises(ValueError):
        save_csr_cache(big, tmp_path / "big.gfxcsr", compact=True)


@pytest.mark.gpu
def test_device_compact_variant(tmp_path):
    """Compact file -> HBM is a straight int32 copy equal to the reference
    file's load; HBM -> compact file equals the host writer's bytes."""
    import paper_1701_01170_b200 as gfx
    from paper_1701_01170_b200.io import load_csr_cache, load_csr_cache_device, save_csr_cache, \
        save_csr_cache_device

    host = load_csr_cache(W_FILE)
    p = tmp_path / "w2.gfxcsr"
    save_csr_cache(host, p, compact=True)
    dg = load_csr_cache_device(p)
    ref = load_csr_cache_device(W_FILE)
    for x, y in ((dg.row, ref.row), (dg.col, ref.col), (dg.w, ref.w)):
        assert x.dtype == y.dtype and bool((x == y).all())
    save_csr_cache_device(dg, tmp_path / "back.gfxcsr", compact=True)
    assert (tmp_path / "back.gfxcsr").read_bytes() == p.read_bytes()
    assert gfx.bfs(load_csr_cache(p), 0).labels.tolist() == gfx.bfs(host, 0).labels.tolist()


@pytest.mark.gpu
def test_device_round_trip(tmp_path):
    """File -> HBM (int64 ids narrowed on the GPU) -> file, byte-identical;
    the device copy traverses like the host graph."""
    import paper_1701_01170_b200 as gfx
    from paper_1701_01170_b200._results import labels_to_host
    from paper_1701_01170_b200.io import (load_csr_cache, load_csr_cache_device,
                                           save_csr_cache_device)
    from paper_1701_01170_b200.primitives.bfs import bfs_device
    from paper_1701_01170_b200.primitives.sssp import sssp_device

    dg = load_csr_cache_device(W_FILE)
    host = load_csr_cache(W_FILE)
    assert np.array_equal(dg.row.cpu().numpy(), host.row_offsets)
    assert np.array_equal(dg.col.cpu().numpy(), host.column_indices)
    assert np.array_equal(dg.w.cpu().numpy(), host.edge_weights)
    save_csr_cache_device(dg, tmp_path / "w.gfxcsr")
    assert (tmp_path / "w.gfxcsr").read_bytes() == W_FILE.read_bytes()
    for s0 in (0, 7):
        want = gfx.bfs(host, s0, direction="auto").labels
        labels, _, _ = bfs_device(dg, s0, direction="auto")
        assert np.array_equal(labels_to_host(labels[:host.num_vertices]), want)
        want = gfx.sssp(host, s0).labels
        dist, _, _ = sssp_device(dg, s0)
        assert np.array_equal(labels_to_host(dist[:host.num_vertices]), want)


@pytest.mark.gpu
def test_device_cache_of_gpu_rmat(tmp_path):
    """The GPU R-MAT builder's s16 graph saved from HBM is the reference's
    canonical CSR (golden SHA) and reloads to the same BFS."""
    import hashlib

    from conftest import rmat_golden, sha
    from paper_1701_01170_b200._results import labels_to_host
    from paper_1701_01170_b200.generators import rmat_device_graph
    from paper_1701_01170_b200.io import load_csr_cache, load_csr_cache_device, save_csr_cache_device
    from paper_1701_01170_b200.primitives.bfs import bfs_device

    rec, _ = rmat_golden(16)
    dg = rmat_device_graph(16, 16, 0)
    path = tmp_path / "s16.gfxcsr"
    save_csr_cache_device(dg, path)
    g = load_csr_cache(path)
    assert hashlib.sha256(g.row_offsets.astype("<i8").tobytes()).hexdigest() == rec["row_sha"]
    assert hashlib.sha256(g.column_indices.astype("<i8").tobytes()).hexdigest() == rec["col_sha"]
    dg2 = load_csr_cache_device(path)
    labels, _, _ = bfs_device(dg2, 0, direction="auto")
    assert sha(labels_to_host(labels)) == rec["bfs_sha"]

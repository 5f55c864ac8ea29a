"""Partitioned BFS (csrc/gfx_dist.cu + dist.py) with P virtual ranks on one
GPU: labels and the direction trace equal the reference's."""
import numpy as np
import pytest

from conftest import host_graph, rmat_golden, sha

pytestmark = pytest.mark.gpu


def _rows(trace):
    return [[t["iteration"], t["mode_before"], t["n_f"], t["n_u"], t["m_f"], t["m_u"],
             t["decision"]] for t in trace]


def _engines(dg, P):
    from paper_1701_01170_b200.dist import DeviceEngine, partition_graph

    out = []
    for r in range(P):
        lrow, lcol = partition_graph(dg, P, r)
        out.append(DeviceEngine(lrow, lcol, dg.num_vertices, dg.num_edges, P, r))
    return out


@pytest.mark.parametrize("P", [1, 2, 3, 4])
def test_kat_partitioned(kat, P):
    from paper_1701_01170_b200._results import labels_to_host
    from paper_1701_01170_b200.dist import VirtualComm, bfs_partitioned, gather_labels

    for d in kat:
        if not d["undirected"]:
            continue
        g = host_graph(d)
        dg = g.device()
        engines = _engines(dg, P)
        for direction in ("auto", "push", "pull"):
            st = bfs_partitioned(VirtualComm(engines), d["n"], d["m"], d["source"],
                                 direction=direction)
            lab, prd = gather_labels(engines, d["n"])
            assert np.array_equal(labels_to_host(lab), d["bfs"]), (d["name"], P, direction)
            if direction == "auto":
                assert _rows(st.direction_trace) == [list(x) for x in d["bfs_auto_trace"]]


@pytest.mark.parametrize("scale,P", [(16, 2), (16, 4), (20, 3), (22, 8)])
def test_rmat_partitioned(scale, P):
    from _checks import valid_bfs_preds
    from paper_1701_01170_b200._results import labels_to_host, preds_to_host
    from paper_1701_01170_b200.dist import VirtualComm, bfs_partitioned, gather_labels
    from paper_1701_01170_b200.generators import rmat_device_graph

    rec, _ = rmat_golden(scale)
    dg = rmat_device_graph(scale, 16, 0)
    engines = _engines(dg, P)
    st = bfs_partitioned(VirtualComm(engines), dg.num_vertices, dg.num_edges, 0, direction="auto")
    lab, prd = gather_labels(engines, dg.num_vertices)
    labels = labels_to_host(lab)
    assert sha(labels) == rec["bfs_sha"]
    assert _rows(st.direction_trace) == [list(x) for x in rec["bfs_auto_trace"]]
    if scale <= 16:
        row = dg.row.cpu().numpy()
        col = dg.col.cpu().numpy().astype(np.int64)
        assert valid_bfs_preds(row, col, labels, preds_to_host(prd), 0)
    st = bfs_partitioned(VirtualComm(engines), dg.num_vertices, dg.num_edges, 0, direction="push")
    lab, _ = gather_labels(engines, dg.num_vertices)
    assert sha(labels_to_host(lab)) == rec["bfs_sha"]
    assert st.edges_push == rec["bfs_edges_traversed"]


def test_kat_native_loop_single_rank(kat):
    """The native level loop (gfx_dbfs_run) at P = 1: labels and trace equal
    the reference's, for every direction."""
    from paper_1701_01170_b200._results import labels_to_host
    from paper_1701_01170_b200.dist import bfs_partitioned_native, gather_labels

    for d in kat:
        if not d["undirected"]:
            continue
        dg = host_graph(d).device()
        (eng,) = _engines(dg, 1)
        for direction in ("auto", "push", "pull"):
            st = bfs_partitioned_native(eng, None, d["n"], d["m"], d["source"],
                                        direction=direction)
            lab, _ = gather_labels([eng], d["n"])
            assert np.array_equal(labels_to_host(lab), d["bfs"]), (d["name"], direction)
            if direction == "auto":
                assert _rows(st.direction_trace) == [list(x) for x in d["bfs_auto_trace"]]


@pytest.mark.parametrize("scale", [16, 20, 22])
def test_rmat_native_loop_single_rank(scale):
    from _checks import valid_bfs_preds
    from paper_1701_01170_b200._results import labels_to_host, preds_to_host
    from paper_1701_01170_b200.dist import bfs_partitioned_native, gather_labels
    from paper_1701_01170_b200.generators import rmat_device_graph

    rec, _ = rmat_golden(scale)
    dg = rmat_device_graph(scale, 16, 0)
    (eng,) = _engines(dg, 1)
    for _ in range(2):  # engine reuse across BFS runs
        st = bfs_partitioned_native(eng, None, dg.num_vertices, dg.num_edges, 0, direction="auto")
        lab, prd = gather_labels([eng], dg.num_vertices)
        labels = labels_to_host(lab)
        assert sha(labels) == rec["bfs_sha"]
        assert _rows(st.direction_trace) == [list(x) for x in rec["bfs_auto_trace"]]
    if scale <= 16:
        row = dg.row.cpu().numpy()
        col = dg.col.cpu().numpy().astype(np.int64)
        assert valid_bfs_preds(row, col, labels, preds_to_host(prd), 0)
    st = bfs_partitioned_native(eng, None, dg.num_vertices, dg.num_edges, 0, direction="push")
    lab, _ = gather_labels([eng], dg.num_vertices)
    assert sha(labels_to_host(lab)) == rec["bfs_sha"]
    assert st.edges_push == rec["bfs_edges_traversed"]

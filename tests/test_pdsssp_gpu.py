"""Device-resident partitioned near/far SSSP (csrc/gfx_pdsssp.cu): P virtual
ranks in one launch on one GPU.  Distances equal the reference's (KATs and
R-MAT goldens from the real graphfx package) for several delta values --
bucket splits, advance_bucket and the offer exchange exercised -- and preds
satisfy the shortest-path property (_oracles.py:185-202)."""
import numpy as np
import pytest

from conftest import host_graph, rmat_golden, sha

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("P", [1, 2, 3, 4])
def test_kat_virtual_ranks_sssp(kat, P):
    from _checks import valid_sssp_preds
    from paper_1701_01170_b200._results import labels_to_host, preds_to_host
    from paper_1701_01170_b200.dist import VirtualRanksSssp

    for d in kat:
        if not d["undirected"] or "w" not in d:
            continue
        g = host_graph(d, weighted=True)
        dg = g.device()
        eng = VirtualRanksSssp(dg, P)
        for delta in (None, 1, 7, 1000):
            dist, preds, st = eng.run(d["source"], delta)
            lab = labels_to_host(dist)
            assert np.array_equal(lab, d["sssp"]), (d["name"], P, delta)
            assert valid_sssp_preds(g.row_offsets, g.column_indices, g.edge_weights, lab,
                                    preds_to_host(preds), d["source"]), (d["name"], P, delta)
        eng.close()


@pytest.mark.parametrize("scale,P,delta", [(16, 1, 32), (16, 2, 32), (16, 4, None), (20, 3, 4),
                                           (20, 8, 32), (22, 1, 4)])
def test_rmat_virtual_ranks_sssp(scale, P, delta):
    from _checks import valid_sssp_preds
    from paper_1701_01170_b200._results import labels_to_host, preds_to_host
    from paper_1701_01170_b200.dist import VirtualRanksSssp
    from paper_1701_01170_b200.generators import rmat_device_graph

    rec, _ = rmat_golden(scale)
    dg = rmat_device_graph(scale, 16, 0, weights=(1, 64), weight_seed=0)
    eng = VirtualRanksSssp(dg, P)
    dist, preds, st = eng.run(0, delta)
    lab = labels_to_host(dist)
    assert sha(lab) == rec["sssp_d32_sha"]  # distances are delta-independent
    assert st.iterations > 0
    if scale == 16:
        g = dg.to_host()
        assert valid_sssp_preds(g.row_offsets, g.column_indices, g.edge_weights, lab,
                                preds_to_host(preds), 0)
    eng.close()


@pytest.mark.parametrize("P,scale", [(2, 12), (3, 14)])
def test_real_ranks_processes_share_one_gpu_sssp(P, scale):
    """Real-rank mode of the partitioned SSSP: P processes on the one GPU,
    CUDA-IPC-mapped inboxes / counter tables, flag barriers across processes;
    distances equal the single-GPU SSSP."""
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parent.parent
    r = subprocess.run([sys.executable, str(root / "tools" / "pd_procs_one_gpu.py"), str(scale),
                        str(P), "sssp"], capture_output=True, text=True, timeout=300, cwd=root)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "labels equal: True" in r.stdout, r.stdout[-2000:]

"""GPU R-MAT + CSR + weights builder vs the reference's SHA-256 goldens."""
import numpy as np
import pytest

from conftest import rmat_golden, sha

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("scale", [10, 12, 14, 16, 18, 20, 22, 24])
def test_device_builder_bit_exact(scale):
    from paper_1701_01170_b200.generators import rmat_device_graph

    rec, _ = rmat_golden(scale)
    dg = rmat_device_graph(scale, 16, 0, weights=(1, 64), weight_seed=0)
    assert dg.num_vertices == rec["n"] and dg.num_edges == rec["m"]
    assert sha(dg.row.cpu().numpy()) == rec["row_sha"]
    assert sha(dg.col.cpu().numpy().astype(np.int64)) == rec["col_sha"]
    assert sha(dg.w.cpu().numpy().astype(np.int64)) == rec["w_sha"]
    assert dg.max_degree == rec["max_deg"]


def test_directed_builder_matches_host():
    import paper_1701_01170_b200 as gfx
    from paper_1701_01170_b200.generators import generate_rmat, rmat_device_graph

    for seed in range(3):
        host = gfx.coo_to_csr(generate_rmat(8, 5, seed=seed))
        dg = rmat_device_graph(8, 5, seed, make_undirected=False)
        assert np.array_equal(dg.row.cpu().numpy(), host.row_offsets)
        assert np.array_equal(dg.col.cpu().numpy(), host.column_indices)

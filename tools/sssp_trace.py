"""SSSP s24 per delta: device ms (min of 3), iterations, relaxed slots and a
digest of the per-iteration (frontier_in, frontier_out) trace -- for checking
that a variant build keeps the reference's iteration sequence."""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1701_01170_b200.generators import rmat_device_graph  # noqa: E402
from paper_1701_01170_b200.primitives.sssp import sssp_device  # noqa: E402

dg = rmat_device_graph(int(sys.argv[1]) if len(sys.argv) > 1 else 24, 16, 0, weights=(1, 64),
                       weight_seed=0)
for d in (4, 32, None):
    runs = [sssp_device(dg, 0, delta=d) for _ in range(4)]
    st = runs[-1][2]
    tr = [(r["frontier_in"], r["frontier_out"]) for r in st.device_levels]
    dist_sha = hashlib.sha256(runs[-1][0].cpu().numpy().tobytes()).hexdigest()[:12]
    print(f"delta {d}: {min(r[2].device_ms for r in runs[1:]):.3f} ms  it {st.iterations}  "
          f"slots {st.edges_traversed}  trace {hashlib.sha256(repr(tr).encode()).hexdigest()[:12]}  "
          f"dist {dist_sha}")

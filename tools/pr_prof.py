"""PageRank (20 iterations, eps 0) on the GPU-built R-MAT graph (default s24)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1701_01170_b200.generators import rmat_device_graph  # noqa: E402
from paper_1701_01170_b200.primitives.pagerank import pagerank_device  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 20
dg = rmat_device_graph(scale, 16, 0)
for _ in range(2):
    r, st = pagerank_device(dg, 0.85, 0.0, iters)
print("pagerank scale", scale, "iters", iters, "ms", round(st.device_ms, 3), "sum", float(r.sum()))

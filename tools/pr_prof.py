"""One PageRank run (20 iterations, eps 0) on R-MAT s<scale> for ncu launch lists."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1701_01170_b200.generators import rmat_device_graph  # noqa: E402
from paper_1701_01170_b200.primitives.pagerank import pagerank_device  # noqa: E402

dg = rmat_device_graph(int(sys.argv[1]) if len(sys.argv) > 1 else 24, 16, 0)
pagerank_device(dg, 0.85, 0.0, 20)
torch.cuda.synchronize()
rank, st = pagerank_device(dg, 0.85, 0.0, 20)
torch.cuda.synchronize()
print("ms", st.device_ms)

"""Push-only BFS ms at s24 (batched device launches), for variant sweeps."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1701_01170_b200.generators import rmat_device_graph  # noqa: E402
from paper_1701_01170_b200.primitives.bfs import bfs_batch, bfs_device  # noqa: E402

dg = rmat_device_graph(24, 16, 0)
lab = torch.empty(dg.num_vertices, dtype=torch.int32, device="cuda")
prd = torch.empty_like(lab)
for _ in range(2):
    bfs_device(dg, 0, direction="push", labels=lab, preds=prd)
print(round(bfs_batch(dg, [0] * 5, direction="push", labels=lab, preds=prd) / 5, 4))

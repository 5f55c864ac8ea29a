"""Device-resident partitioned BFS at s<scale>: P virtual ranks on one GPU
(P = 1 is the N = 1 partitioned engine) against the single-GPU kernel, device
ms per BFS over batched launches.   python tools/pdbfs_time.py [scale] [P...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1701_01170_b200.dist import VirtualRanksBfs  # noqa: E402
from paper_1701_01170_b200.generators import rmat_device_graph  # noqa: E402
from paper_1701_01170_b200.primitives.bfs import bfs_batch, bfs_device  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
Ps = [int(x) for x in sys.argv[2:]] or [1, 2, 4, 8]
dg = rmat_device_graph(scale, 16, 0)
lab = torch.empty(dg.num_vertices, dtype=torch.int32, device="cuda")
prd = torch.empty_like(lab)
for _ in range(3):
    bfs_device(dg, 0, direction="auto", labels=lab, preds=prd)
one = bfs_batch(dg, [0] * 10, direction="auto", labels=lab, preds=prd) / 10
print(f"single-GPU kernel s{scale}: {one:.4f} ms")
ref = lab.clone()
for P in Ps:
    eng = VirtualRanksBfs(dg, P)
    labels, _, st, levels = eng.run(0, direction="auto")
    ok = bool(torch.equal(labels, ref))
    for _ in range(2):
        eng.batch_ms(0, 2)
    ms = eng.batch_ms(0, 10) / 10
    print(f"partitioned, {P} virtual rank(s): {ms:.4f} ms ({ms / one:.2f}x), labels equal: {ok}, "
          f"levels {[round(lv['ms'] * 1000, 1) for lv in levels]}")
    del eng
    torch.cuda.synchronize()

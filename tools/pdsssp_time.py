"""Device-resident partitioned SSSP at s<scale> (weights 1..64): P virtual
ranks on one GPU (P = 1 is the N = 1 partitioned engine) against the
single-GPU SSSP, device ms per run.   python tools/pdsssp_time.py [scale] [P...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1701_01170_b200.dist import VirtualRanksSssp  # noqa: E402
from paper_1701_01170_b200.generators import rmat_device_graph  # noqa: E402
from paper_1701_01170_b200.primitives.sssp import sssp_device  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
Ps = [int(x) for x in sys.argv[2:]] or [1, 2, 4, 8]
dg = rmat_device_graph(scale, 16, 0, weights=(1, 64), weight_seed=0)
for delta in (4, 32, None):
    sssp_device(dg, 0, delta=delta)
    one = min(sssp_device(dg, 0, delta=delta)[2].device_ms for _ in range(3))
    ref = sssp_device(dg, 0, delta=delta)[0].clone()
    line = [f"delta {delta}: single-GPU {one:.3f} ms"]
    for P in Ps:
        eng = VirtualRanksSssp(dg, P)
        dist, _, st = eng.run(0, delta)
        ok = bool(torch.equal(dist, ref))
        eng.batch_ms(0, 1, delta)
        ms = eng.batch_ms(0, 3, delta) / 3
        line.append(f"P{P} {ms:.3f} ms ({ms / one:.2f}x, iters {st.iterations}, eq {ok})")
        eng.close()
        del eng
        torch.cuda.synchronize()
    print(" | ".join(line), flush=True)

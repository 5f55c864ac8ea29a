import os, sys
sys.path.insert(0, os.getcwd())
import torch
from paper_1701_01170_b200.generators import rmat_device_graph
from paper_1701_01170_b200.primitives.sssp import sssp_device
dg = rmat_device_graph(24, 16, 0, weights=(1, 64), weight_seed=0)
for d in (None, 2, 4, 8, 16, 32, 64, 128):
    for _ in range(2):
        st = sssp_device(dg, 0, delta=d)[2]
    ms = min(sssp_device(dg, 0, delta=d)[2].device_ms for _ in range(3))
    print("delta", d, "ms", round(ms, 3), "iters", st.iterations, "slots", st.work_slots, flush=True)

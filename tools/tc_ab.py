import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
from paper_1701_01170_b200.generators import rmat_device_graph
from paper_1701_01170_b200.primitives.tc import tc_device
for scale in (20, 22):
    dg = rmat_device_graph(scale, 16, 0)
    t0 = time.perf_counter(); r = tc_device(dg); torch.cuda.synchronize()
    print(scale, "first call (orient+rev) s", round(time.perf_counter() - t0, 3), "total", r[0])
    for mode in ("new", "legacy", "new", "legacy"):
        if mode == "legacy":
            os.environ["GFX_TC_LEGACY"] = "1"
        else:
            os.environ.pop("GFX_TC_LEGACY", None)
        total, counts, osrc, odst, st = tc_device(dg)
        print(scale, mode, "ms", round(st.device_ms, 3), "total", total, "counts_sum", int(counts.sum()))

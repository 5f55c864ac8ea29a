"""SSSP device ms at s24 (delta 4, 32 and default), min of 3 after warm-up: for
A/B sweeps of compile-time tunables (GFX_LIB_PATH=<variant .so>)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1701_01170_b200.generators import rmat_device_graph  # noqa: E402
from paper_1701_01170_b200.primitives.sssp import sssp_device  # noqa: E402

dg = rmat_device_graph(24, 16, 0, weights=(1, 64), weight_seed=0)
out = []
for d in (4, 32, None):
    sssp_device(dg, 0, delta=d)
    out.append(round(min(sssp_device(dg, 0, delta=d)[2].device_ms for _ in range(3)), 3))
print(*out)

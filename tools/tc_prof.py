"""One TC count on R-MAT s<scale> for ncu captures: python tools/tc_prof.py 22"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1701_01170_b200.generators import rmat_device_graph  # noqa: E402
from paper_1701_01170_b200.primitives.tc import tc_device  # noqa: E402

dg = rmat_device_graph(int(sys.argv[1]) if len(sys.argv) > 1 else 22, 16, 0)
total, counts, osrc, odst, st = tc_device(dg)
torch.cuda.synchronize()
print("total", total, "ms", st.device_ms)

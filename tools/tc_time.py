"""TC s22 count time: the search kernel (default) vs the staged-hash path
(GFX_TC_HASH=1); totals must agree.  python tools/tc_time.py [scale]"""
import os
import sys

sys.path.insert(0, os.getcwd())
from paper_1701_01170_b200.generators import rmat_device_graph  # noqa: E402
from paper_1701_01170_b200.primitives.tc import tc_device  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 22
dg = rmat_device_graph(scale, 16, 0)
for mode in ("search", "hash", "search"):
    if mode == "hash":
        os.environ["GFX_TC_HASH"] = "1"
    else:
        os.environ.pop("GFX_TC_HASH", None)
    tc_device(dg)
    ms = []
    for _ in range(3):
        total, *_, st = tc_device(dg)
        ms.append(st.device_ms)
    print(mode, "total", total, "ms", [round(x, 2) for x in ms], flush=True)

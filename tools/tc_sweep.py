"""TC counting variants side by side (device ms, totals and count digests)."""
import hashlib
import os
import sys

sys.path.insert(0, os.getcwd())
import torch  # noqa: E402

from paper_1701_01170_b200.generators import rmat_device_graph  # noqa: E402
from paper_1701_01170_b200.primitives.tc import tc_device  # noqa: E402

VARIANTS = {"reversed": {}}
VARIANTS["legacy"] = {"GFX_TC_LEGACY": "1"}
for scale in (20, 22):
    dg = rmat_device_graph(scale, 16, 0)
    tc_device(dg)
    for name, env in list(VARIANTS.items()) * 2:
        for k in ("GFX_TC_LEGACY", "GFX_TC_SKEW", "GFX_TC_GRAB"):
            os.environ.pop(k, None)
        os.environ.update(env)
        total, counts, _, _, st = tc_device(dg)
        dig = hashlib.sha256(counts.to(torch.int64).cpu().numpy().tobytes()).hexdigest()[:12]
        print(scale, name, round(st.device_ms, 2), total, dig, flush=True)

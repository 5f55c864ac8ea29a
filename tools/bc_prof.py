"""BC (single source) on the GPU-built R-MAT graph (default s22)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1701_01170_b200.generators import rmat_device_graph  # noqa: E402
from paper_1701_01170_b200.primitives.bc import bc_device  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 22
dg = rmat_device_graph(scale, 16, 0)
for _ in range(2):
    v, st = bc_device(dg, [0])
print("bc scale", scale, "ms", round(st.device_ms, 3), "max", float(v.max()))

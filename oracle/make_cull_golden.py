"""Golden vectors for the INEXACT culling heuristics, made by running the
REFERENCE (operators.py:315-357, _apply_culling) here.  Test infrastructure:
writes tests/golden/cull_inexact.npz (the GPU box never reads /root/reference).

    PYTHONPATH=/root/reference/pkg/src python oracle/make_cull_golden.py
"""
from __future__ import annotations

from pathlib import Path

import numpy as np
from graphfx.operators import CullingConfig, _apply_culling

OUT = Path(__file__).resolve().parent.parent / "tests" / "golden" / "cull_inexact.npz"


def main():
    arrays = {}
    k = 0
    for bitmask in (True, False):
        for team in (0, 16, 256):
            for local in (0, 8, 64):
                for bb, lb in ((1024, 32), (100, 7)):
                    rng = np.random.default_rng(1000 + k)
                    items = rng.integers(0, 500, size=2000)
                    cfg = CullingConfig(use_bitmask=bitmask, team_table_size=team,
                                        local_table_size=local, bitmask_batch=bb,
                                        local_batch=lb, domain_size=500)
                    out = _apply_culling(items.copy(), cfg)
                    arrays[f"items_{k}"] = items
                    arrays[f"out_{k}"] = out
                    arrays[f"cfg_{k}"] = np.array([int(bitmask), team, local, bb, lb, 500])
                    k += 1
    np.savez_compressed(OUT, count=np.array(k), **arrays)
    print(OUT, k)


if __name__ == "__main__":
    main()

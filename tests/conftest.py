import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running parity job")


def gpu_available() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def kat():
    """Reference-generated KAT graphs + outputs (oracle/make_golden.py kat)."""
    meta = json.loads((GOLDEN / "kat_graphs.json").read_text())
    arrs = np.load(GOLDEN / "kat_graphs.npz")
    out = []
    for i, rec in enumerate(meta["graphs"]):
        p = f"g{i}_"
        d = dict(rec)
        for k in arrs.files:
            if k.startswith(p):
                d[k[len(p):]] = arrs[k]
        out.append(d)
    return out


def rmat_golden(scale: int):
    rec = json.loads((GOLDEN / f"rmat_s{scale}.json").read_text())
    npz = GOLDEN / f"rmat_s{scale}.npz"
    arrays = dict(np.load(npz)) if npz.exists() else {}
    return rec, arrays


def sha(a) -> str:
    import hashlib

    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def host_graph(d, weighted=False):
    """CsrGraph (product type) from a KAT record."""
    from paper_1701_01170_b200 import CsrGraph

    w = d["w"].astype(np.int64) if weighted else None
    return CsrGraph(int(d["n"]), d["row"].astype(np.int64), d["col"].astype(np.int64), w,
                    undirected=bool(d["undirected"]))


@pytest.fixture(scope="session")
def suite():
    """Every 5th graph of the reference acceptance suite (+ its large tail),
    with reference outputs (oracle/make_golden.py suite)."""
    meta = json.loads((GOLDEN / "suite_graphs.json").read_text())
    arrs = np.load(GOLDEN / "suite_graphs.npz")
    out = []
    for i, rec in enumerate(meta["graphs"]):
        p = f"g{i}_"
        d = dict(rec)
        d["undirected"] = True
        for k in ("row", "col", "w", "bfs", "sssp", "bc", "cc", "pr4", "tc_counts"):
            d[k] = arrs[p + k]
        out.append(d)
    return out

"""libgfx.so loads and exports every symbol declared in include/gfx.h; the
host-only direction replica matches CPython's floats.  No GPU needed."""
import math
import random
import re

import numpy as np

from conftest import ROOT


def declared_symbols():
    text = (ROOT / "include" / "gfx.h").read_text()
    return sorted(set(re.findall(r"GFX_API\s+[\w\s\*]+?\b(gfx_\w+)\s*\(", text)))


def test_library_exports_header_symbols():
    from paper_1701_01170_b200 import _native

    lib = _native.load_library()
    syms = declared_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_native.exported_symbols())
    assert lib.gfx_version() >= 1


def _py_est(n, m, n_f, n_u, mu_edge):
    m_f = n_f * m / n
    if n_u >= n:
        return m_f, math.inf
    return m_f, n_u * (m if mu_edge else n) / (n - n_u)


def test_direction_replica_bit_exact():
    from paper_1701_01170_b200 import _native

    rng = random.Random(7)
    cases = [(65536, 1819076, 9699, 55836, 0), (1 << 27, 4_200_000_000, 90_000_000, 30_000_000, 0),
             (1 << 27, 4_200_000_000, 90_000_000, 30_000_000, 1), (16, 40, 1, 16, 0)]
    for _ in range(3000):
        n = rng.choice([rng.randint(1, 1000), rng.randint(1, 1 << 31)])
        m = rng.randint(0, 1 << 33)
        n_f = rng.randint(0, n)
        n_u = rng.randint(0, n)
        cases.append((n, m, n_f, n_u, rng.randint(0, 1)))
    for n, m, n_f, n_u, e in cases:
        got = _native.estimate_mf_mu(n, m, n_f, n_u, bool(e))
        want = _py_est(n, m, n_f, n_u, e)
        assert got[0] == want[0], (n, m, n_f, n_u)
        assert got[1] == want[1], (n, m, n_f, n_u, e)

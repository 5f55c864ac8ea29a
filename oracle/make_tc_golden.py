"""TC golden for R-MAT s22 (BASELINE config C4) from the C restatement.

The reference's own tc() needs more than 30 minutes at s22, so this script
runs the C oracle (oracle/serial.c, restating tc.py:53-76) instead, after
pinning it twice: (1) the s22 CSR it builds (oracle/graphfx_port.py) must
hash to the reference's row/col digests in tests/golden/rmat_s22.json, and
(2) the same oracle must reproduce the reference's own TC golden at s20
(tests/golden/rmat_s20.json: total, per-edge counts, oriented src/dst).
It then adds tc_total / tc_counts_sha / tc_src_sha / tc_dst_sha and
tc_source to rmat_s22.json.  Test infrastructure only.

    python oracle/make_tc_golden.py
"""
import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))

from oracle import c_oracle  # noqa: E402
from oracle import graphfx_port as port  # noqa: E402

GOLD = HERE.parent / "tests" / "golden"


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def tc_record(scale):
    row, col = port.rmat_csr(scale, 16, 0)
    rec = json.loads((GOLD / f"rmat_s{scale}.json").read_text())
    assert sha(np.asarray(row, dtype=np.int64)) == rec["row_sha"], "row digest"
    assert sha(np.asarray(col, dtype=np.int64)) == rec["col_sha"], "col digest"
    total, counts, osrc, odst = c_oracle.tc(row, col)
    return rec, {"tc_total": int(total), "tc_counts_sha": sha(counts.astype(np.int64)),
                 "tc_src_sha": sha(osrc.astype(np.int64)), "tc_dst_sha": sha(odst.astype(np.int64))}


def main():
    t0 = time.time()
    rec20, got20 = tc_record(20)
    for k, v in got20.items():
        assert rec20[k] == v, f"C oracle disagrees with the reference's s20 {k}"
    print(f"s20 pin ok ({time.time() - t0:.0f} s)", flush=True)
    rec22, got22 = tc_record(22)
    rec22.update(got22)
    rec22["tc_source"] = ("oracle/serial.c (C restatement of tc.py:53-76), pinned to the "
                          "reference's own s20 TC golden by oracle/make_tc_golden.py")
    (GOLD / "rmat_s22.json").write_text(json.dumps(rec22, indent=1) + "\n")
    print(f"s22 tc_total {got22['tc_total']} ({time.time() - t0:.0f} s)")


if __name__ == "__main__":
    main()

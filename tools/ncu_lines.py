"""Per-CUDA-source-line view of an ncu report (source page, cuda,sass):
warp-stall samples with the dominant reasons and L2 sectors per line.

    python tools/ncu_lines.py report.ncu-rep [top]
"""
import csv
import subprocess
import sys

import os
rep = os.path.abspath(sys.argv[1])
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True, cwd="/tmp").stdout
rows = list(csv.reader(out.splitlines()))
fname, hdr, lines = None, None, []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
    elif r[0] == "Line No":
        hdr = r
    elif hdr and len(r) == len(hdr) and r[0] not in ("",):
        lines.append((fname, r))
if not hdr:
    sys.exit("no source rows")
i_s = hdr.index("Warp Stall Sampling (All Samples)")
i_l2 = hdr.index("L2 Theoretical Sectors Global")
i_ex = hdr.index("Instructions Executed")
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(int(r[i_s] or 0) for _, r in lines)
print(f"total samples {tot}")
agg = sorted(lines, key=lambda x: -int(x[1][i_s] or 0))[:top]
for f, r in agg:
    s = int(r[i_s] or 0)
    rs = sorted(((int(r[hdr.index(h)] or 0), h[6:]) for h in reasons), reverse=True)[:2]
    rtxt = ", ".join(f"{n} {v}" for v, n in rs if v)
    print(f"{s:6d} {100*s/max(tot,1):5.1f}%  {f}:{r[0]:<5} l2sec={r[i_l2]:>10} inst={r[i_ex]:>9}  [{rtxt}]  {r[1].strip()[:80]}")

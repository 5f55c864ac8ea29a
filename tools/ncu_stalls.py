"""Aggregate warp-stall samples of an ncu report's source page by reason and
list the hottest SASS lines with their dominant reason."""
import csv
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
blocks, cur = [], None
for r in rows:
    if "Warp Stall Sampling (All Samples)" in r:
        cur = {"hdr": r, "rows": []}
        blocks.append(cur)
    elif cur and len(r) == len(cur["hdr"]):
        cur["rows"].append(r)
for bi, b in enumerate(blocks):
    hdr = b["hdr"]
    reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    idx = {h: hdr.index(h) for h in reasons}
    tot = {h: 0 for h in reasons}
    lines = []
    for r in b["rows"]:
        vals = {h: int(r[idx[h]] or 0) for h in reasons}
        for h, v in vals.items():
            tot[h] += v
        s = sum(vals.values())
        if s:
            top = max(vals, key=vals.get)
            lines.append((s, top, r[hdr.index("Source")][:70]))
    total = sum(tot.values()) or 1
    print(f"=== launch block {bi}: {total} samples")
    for h, v in sorted(tot.items(), key=lambda x: -x[1])[:8]:
        print(f"  {h:<24} {100*v/total:5.1f}%")
    for s, top, src in sorted(lines, reverse=True)[:12]:
        print(f"  {s:7d} {top:<16} {src}")

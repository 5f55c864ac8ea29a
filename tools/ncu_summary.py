"""Summarise an ncu report (details page) or a launch-list CSV."""
import csv
import subprocess
import sys

SECTIONS = ("GPU Speed Of Light Throughput", "Memory Workload Analysis", "Scheduler Statistics",
            "Warp State Statistics", "Occupancy", "Launch Statistics")
KEEP = ("Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Issued Warp Per Scheduler", "No Eligible", "Active Warps Per Scheduler",
        "Warp Cycles Per Issued Instruction", "Avg. Active Threads Per Warp",
        "Achieved Occupancy", "Theoretical Occupancy", "Registers Per Thread", "Grid Size",
        "Compute (SM) Throughput", "L1/TEX Cache Throughput", "L2 Cache Throughput")
RAW = ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
       "smsp__pcsamp_warps_issue_stalled_long_scoreboard", "lts__t_sector_hit_rate.pct")


def details(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[0]
    g = {k: hdr.index(k) for k in ("ID", "Kernel Name", "Section Name", "Metric Name",
                                   "Metric Value", "Metric Unit")}
    cur = None
    for r in rows[1:]:
        if r[g["ID"]] != cur:
            cur = r[g["ID"]]
            print(f"--- launch {cur}: {r[g['Kernel Name']][:90]}")
        if r[g["Section Name"]] in SECTIONS and r[g["Metric Name"]] in KEEP:
            print(f"   {r[g['Metric Name']]:<38} {r[g['Metric Value']]} {r[g['Metric Unit']]}")
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr = rows[0]
    for name in RAW:
        if name in hdr:
            i = hdr.index(name)
            print(f"   {name:<50} {[r[i] for r in rows[1:]]}")


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    tot = {}
    order = []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            name = d["Kernel Name"].split("(")[0][:70]
            v = float(d["Metric Value"].replace(",", ""))
            order.append((name, v))
            tot[name] = tot.get(name, 0.0) + v
    for name, v in order:
        print(f"{v/1000:10.1f} us  {name}")
    print("--- totals")
    for name, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"{v/1000:10.1f} us  {name}")


def traffic(rep, kernel, key, source):
    """Record dram read+write bytes per launch of `kernel` (mean over the
    captured launches) in profiles/ncu_traffic.json under `key`."""
    import json
    from pathlib import Path

    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    k, r_i, w_i = hdr.index("Kernel Name"), hdr.index("dram__bytes_read.sum"), hdr.index(
        "dram__bytes_write.sum")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    vals = []
    for r in rows[2:]:
        if kernel in r[k]:
            vals.append(float(r[r_i].replace(",", "")) * scale[units[r_i]] +
                        float(r[w_i].replace(",", "")) * scale[units[w_i]])
    assert vals, f"{kernel} not in {rep}"
    out = Path(__file__).resolve().parent.parent / "profiles" / "ncu_traffic.json"
    db = json.loads(out.read_text()) if out.exists() else {}
    db[key] = {"dram_bytes": int(sum(vals) / len(vals)), "launches": len(vals), "source": source}
    out.write_text(json.dumps(db, indent=1, sort_keys=True) + "\n")
    print(key, db[key])


if __name__ == "__main__":
    p = sys.argv[1]
    if len(sys.argv) > 2 and sys.argv[2] == "--traffic":
        traffic(p, sys.argv[3], sys.argv[4], sys.argv[5])
    else:
        (launches if p.endswith(".csv") else details)(p)

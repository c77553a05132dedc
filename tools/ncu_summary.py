"""Summarise ncu exports: launch list (csv) and --set full reports."""
import csv
import subprocess
import sys
from collections import defaultdict


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = defaultdict(lambda: [0, 0.0])
    order = []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                name = d["Kernel Name"].split("(")[0]
                v = float(d["Metric Value"].replace(",", ""))
                if d["Metric Unit"] == "us":
                    v *= 1e3
                elif d["Metric Unit"] == "ms":
                    v *= 1e6
                if name not in agg:
                    order.append(name)
                agg[name][0] += 1
                agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    print(f"{'kernel':60s} {'n':>4s} {'total_us':>10s} {'avg_us':>9s} {'share':>6s}")
    for name in sorted(agg, key=lambda k: -agg[k][1]):
        n, t = agg[name]
        print(f"{name[:60]:60s} {n:4d} {t/1e3:10.1f} {t/n/1e3:9.1f} {100*t/tot:5.1f}%")


WANT = ["Duration", "Executed Ipc Active", "Issue Slots Busy", "Achieved Occupancy",
        "Theoretical Occupancy", "Registers Per Thread", "DRAM Throughput",
        "Warp Cycles Per Issued Instruction", "No Eligible", "Active Warps Per Scheduler",
        "Eligible Warps Per Scheduler", "L1/TEX Hit Rate", "L2 Hit Rate", "Executed Instructions",
        "Memory Throughput", "Compute (SM) Throughput"]


def details(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[0]
    idx = {h: i for i, h in enumerate(hdr)}
    seen = set()
    for r in rows[1:]:
        k = r[idx["Kernel Name"]].split("(")[0]
        key = (r[idx["ID"]], r[idx["Metric Name"]])
        if r[idx["Metric Name"]] in WANT and key not in seen:
            seen.add(key)
            print(f"{r[idx['ID']]:>3s} {k[:44]:44s} | {r[idx['Metric Name']]:36s} | "
                  f"{r[idx['Metric Value']]} {r[idx['Metric Unit']]}")


def raw(path, pattern):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[0]
    cols = [i for i, h in enumerate(hdr) if any(p in h for p in pattern.split("|"))]
    for r in rows[2:]:
        print(r[4][:40], [(hdr[i], r[i]) for i in cols])


if __name__ == "__main__":
    mode = sys.argv[1]
    if mode == "launches":
        launches(sys.argv[2])
    elif mode == "details":
        details(sys.argv[2])
    else:
        raw(sys.argv[2], sys.argv[3])

"""Per-line hot spots of one kernel in an ncu report (needs -lineinfo and
--import-source on): python tools/ncu_source.py <rep> <kernel-regex> [sass|cuda] [top]"""
import csv
import subprocess
import sys

rep, rx = sys.argv[1], sys.argv[2]
view = sys.argv[3] if len(sys.argv) > 3 else "cuda"
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{rx}",
                      "--print-source", view], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = None
data = []
for r in rows:
    if len(r) > 3 and r[0] in ("Address", "Line", "#"):
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
    if hdr and len(r) == 2 and r[0] == "Kernel Name" and data:
        break
key = "Instructions Executed"
tot = sum(float(d.get(key, "0") or 0) for d in data)
samp = sum(float(d.get("Warp Stall Sampling (All Samples)", "0") or 0) for d in data)
print(f"total warp instructions {tot:.4g}, stall samples {samp:.4g}")
data.sort(key=lambda d: -float(d.get(key, "0") or 0))
for d in data[:top]:
    ins = float(d.get(key, "0") or 0)
    sm = float(d.get("Warp Stall Sampling (All Samples)", "0") or 0)
    loc = d.get("Address") or d.get("Line") or d.get("#")
    print(f"{loc:>8s} {100*ins/tot:5.1f}% ins {100*sm/max(samp,1):5.1f}% smp | {d['Source'].strip()[:110]}")

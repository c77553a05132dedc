"""Instruction-count profile of one kernel by SASS address, grouped into runs of
equal execution count (basic blocks): python tools/ncu_blocks.py <rep> <regex> [top]"""
import csv
import subprocess
import sys

rep, rx = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{rx}",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, seen, data = None, set(), []
for r in rows:
    if r and r[0] == "Address":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d["Address"] in seen:
            continue
        seen.add(d["Address"])
        data.append((int(d["Address"], 16), float(d["Instructions Executed"] or 0),
                     float(d["Warp Stall Sampling (All Samples)"] or 0), d["Source"].strip()))
data.sort()
tot = sum(x[1] for x in data)
smp = sum(x[2] for x in data)
blocks = []
for a, n, s_, src in data:
    if blocks and blocks[-1]["n"] == n:
        b = blocks[-1]
        b["len"] += 1
        b["tot"] += n
        b["smp"] += s_
    else:
        blocks.append({"a": a, "n": n, "len": 1, "tot": n, "smp": s_, "src": src})
print(f"total warp instr {tot:.4g}; {len(data)} SASS instructions; stall samples {smp:.4g}")
base = data[0][0]
for b in sorted(blocks, key=lambda b: -b["tot"])[:top]:
    print(f"+{b['a']-base:05x} len {b['len']:4d} x{b['n']:11.0f} = {100*b['tot']/tot:5.1f}% ins "
          f"{100*b['smp']/max(smp,1):5.1f}% smp | {b['src'][:60]}")

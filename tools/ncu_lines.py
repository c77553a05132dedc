"""Per-CUDA-line instructions and stall samples of one kernel in an ncu report
(--import-source on, -lineinfo), with optional line-range groups:
  python tools/ncu_lines.py REP KERNEL_REGEX [name:first-last ...] [--top N]"""
import csv
import subprocess
import sys

rep, rx = sys.argv[1], sys.argv[2]
FILE = "sw_kernels"
if "--file" in sys.argv:
    FILE = sys.argv[sys.argv.index("--file") + 1]
    del sys.argv[sys.argv.index("--file"):sys.argv.index("--file") + 2]
groups, top = [], 30
args = sys.argv[3:]
if "--top" in args:
    i = args.index("--top")
    top = int(args[i + 1])
    args = args[:i] + args[i + 2:]
for g in args:
    name, rng = g.split(":")
    a, b = rng.split("-")
    groups.append((name, int(a), int(b)))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{rx}",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
fname, hdr, rows = None, None, []
for r in csv.reader(out.splitlines()):
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].rsplit("/", 1)[-1]
    elif len(r) > 4 and r[0] == "Line No":
        hdr = r
    elif hdr and len(r) == len(hdr) and r[2] == "-":
        d = dict(zip(hdr[4:], r[4:]))
        rows.append((fname, int(r[0]), r[1], float(d.get("Instructions Executed", 0) or 0),
                     float(d.get("Warp Stall Sampling (All Samples)", 0) or 0)))
ti = sum(r[3] for r in rows) or 1
ts = sum(r[4] for r in rows) or 1
print(f"warp instructions {ti:.4g}, stall samples {ts:.4g}")
for name, a, b in groups:
    gi = sum(r[3] for r in rows if a <= r[1] <= b and r[0].startswith(FILE))
    gs = sum(r[4] for r in rows if a <= r[1] <= b and r[0].startswith(FILE))
    print(f"  {name:12s} lines {a}-{b}: {100*gi/ti:5.1f}% instr  {100*gs/ts:5.1f}% samples")
for f, ln, src, i, s in sorted(rows, key=lambda r: -r[4])[:top]:
    print(f"{f[:14]:14s}{ln:5d} {100*i/ti:5.1f}% ins {100*s/ts:5.1f}% smp | {src.strip()[:100]}")

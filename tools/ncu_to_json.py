"""Summarise a round's ncu evidence for bench.py's roofline fields:
kernel shares from the launch list, and DRAM traffic per launch of the
dominant kernel from its `--set full` capture, beside the algorithmic bytes
of that launch.

    python tools/ncu_to_json.py LAUNCH_CSV NCU_REP KERNEL_RE CLASS_R OUT_JSON [--pairs N]

CLASS_R: the packed class (rows per lane) of the captured K1p launch; its
algorithmic bytes are computed from the benched batch (pastis_synth,
seed 2303): residue bytes + 24 B pair entry + 32 B result per pair of that
class (bench.computed_cells' class model).
"""
import csv
import json
import os
import subprocess
import sys
from collections import defaultdict

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def launch_shares(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                name = d["Kernel Name"].split("(")[0].replace("void ", "")
                v = float(d["Metric Value"].replace(",", ""))
                unit = d["Metric Unit"]
                v *= {"ns": 1, "nsecond": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}.get(unit, 1)
                agg[name][0] += 1
                agg[name][1] += v
    # the e2e leg's device gather of pinned host arenas moves bytes over PCIe
    # (serialised under ncu): reported, but not part of the step's kernel shares
    tot = sum(v[1] for k, v in agg.items() if "k_gather_arena" not in k)
    out = {}
    for name in sorted(agg, key=lambda k: -agg[k][1]):
        n, t = agg[name]
        if t / tot < 0.002:
            continue
        out[name] = {"launches": n, "total_ms": round(t / 1e6, 3), "share": round(t / tot, 4)}
    groups = defaultdict(float)
    for name, v in out.items():
        if "k_gather_arena" in name:
            continue
        key = ("K1p k_score_packed" if "k_score_packed" in name else
               "K5 k_tb" if "k_tb" in name else
               "K1cp k_score_cta_packed" if "k_score_cta_packed" in name else "other")
        groups[key] += v["share"]
    return out, {k: round(v, 4) for k, v in groups.items()}


def raw_metrics(rep, regex):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr = rows[0]
    want = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
            "sm__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread"]
    idx = {h: i for i, h in enumerate(hdr)}
    units = rows[1]
    res = []
    for r in rows[2:]:
        rec = {"kernel": r[idx["Kernel Name"]][:80]}
        for w in want:
            if w in idx:
                v = r[idx[w]].replace(",", "")
                try:
                    v = float(v)
                except ValueError:
                    pass
                u = units[idx[w]]
                if isinstance(v, float) and u in ("Kbyte", "Mbyte", "Gbyte"):
                    v *= {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[u]
                if isinstance(v, float) and u in ("usecond", "msecond"):
                    v *= {"usecond": 1e3, "msecond": 1e6}[u]
                rec[w] = v
        res.append(rec)
    return res


def main():
    launches, rep, regex, cls_r, out_path = sys.argv[1:6]
    n_pairs = 1_000_000
    if "--pairs" in sys.argv:
        n_pairs = int(sys.argv[sys.argv.index("--pairs") + 1])
    per_kernel, groups = launch_shares(launches)
    caps = raw_metrics(rep, regex)
    cap = caps[0] if caps else {}
    import bench
    from pastis_synth import workloads
    _, table = workloads.config3_packed(n_pairs, seed=2303)
    m = table["a_len"].astype(np.int64)
    n = table["b_len"].astype(np.int64)
    cls = bench.packed_class_of(m, n)
    k = bench.CLASS_ROWS.index(int(cls_r))
    sel = (cls == k) & (m * n <= bench.FUSED_MAX_CELLS)
    alg = int((m[sel] + n[sel]).sum() + 56 * sel.sum())
    traffic = None
    if "dram__bytes_read.sum" in cap:
        traffic = cap["dram__bytes_read.sum"] + cap["dram__bytes_write.sum"]
    d = {"kernel": cap.get("kernel"),
         "source": f"ncu --set full --clock-control none ({os.path.basename(rep)}); launch list "
                   f"{os.path.basename(launches)} (gpu__time_duration, serialised, cold cache)",
         "class_rows": int(cls_r), "pairs_in_launch": int(sel.sum()),
         "cells_in_launch": int((m[sel] * n[sel]).sum()),
         "traffic_bytes_per_launch": traffic,
         "dram_read_bytes": cap.get("dram__bytes_read.sum"),
         "dram_write_bytes": cap.get("dram__bytes_write.sum"),
         "duration_ns": cap.get("gpu__time_duration.sum"),
         "algorithmic_bytes_per_launch": alg,
         "metrics": cap,
         "kernel_share": groups,
         "per_kernel": per_kernel,
         "note": "DRAM writes are the traceback checkpoints (~0.4 B/cell, replayed by K5); the "
                 "algorithmic bytes are the pairs' residues + 24 B pair entry + 32 B result"}
    with open(out_path, "w") as fh:
        json.dump(d, fh, indent=1)
    print(json.dumps({k: d[k] for k in ("kernel", "traffic_bytes_per_launch",
                                         "algorithmic_bytes_per_launch", "kernel_share")}))


if __name__ == "__main__":
    main()

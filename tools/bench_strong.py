"""Strong scaling of ONE config-3 batch (1M pairs) over 1..N GPUs of one
process through sw_align_batch_multi (device-planned cell-balanced shards,
zero-copy shard gather from the pinned host arena, host scatter of the
records).  Wall time per call (host arena in, host records out), best and
mean of --reps after a warm-up; prints one JSON line per device count.

    python tools/bench_strong.py [--pairs 1000000] [--reps 5]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2303_01845_b200 import _native, blosum62  # noqa: E402
from pastis_synth import workloads  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--pairs", type=int, default=1_000_000)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--workload", default="config3")
    args = ap.parse_args()
    n_dev = _native.device_count()
    pool = _native.pinned_pool()
    gen = {"config3": workloads.config3_packed, "config2": workloads.config2_packed}[args.workload]
    bufs = []

    def alloc(nb):
        b = pool.acquire(nb)
        bufs.append(b)
        return b.array

    arena, table = gen(args.pairs, seed=2303, alloc=alloc)
    cells = int(np.dot(table["a_len"].astype(np.int64), table["b_len"].astype(np.int64)))
    p = _native.make_params(11, 1, blosum62.MATRIX)
    ref = None
    base = None
    for k in range(1, n_dev + 1):
        devs = list(range(k))
        if k == 1:
            call = lambda: (_native.align_host(arena, table, p, device=0)[0], None)  # noqa: E731
        else:
            call = lambda: _native.align_multi(arena, table, p, devs)  # noqa: E731
        rec, _ = call()
        walls, tms = [], None
        for _ in range(args.reps):
            t0 = time.perf_counter()
            rec, tms = call()
            walls.append(time.perf_counter() - t0)
        if ref is None:
            ref = rec
        line = {"workload": args.workload, "pairs": args.pairs, "cells": cells, "gpus": k,
                "wall_ms_best": min(walls) * 1e3, "wall_ms_mean": float(np.mean(walls)) * 1e3,
                "gcups_best": cells / min(walls) / 1e9, "exact_vs_1gpu": bool((rec == ref).all())}
        if base is None:
            base = line["gcups_best"]
        line["efficiency_vs_1gpu"] = line["gcups_best"] / (k * base)
        if tms:
            line["per_device"] = [{"cells": t["cells"], "kernel_ms": round(t["kernel_ms"], 3),
                                   "total_ms": round(t["total_ms"], 3),
                                   "forward_ms": round(t["forward_ms"], 3)} for t in tms]
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()

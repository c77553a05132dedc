"""TEST/BENCH INFRASTRUCTURE ONLY -- times the CPU restatements of the
reference aligner on a bounded sample of a workload (bench.py's cpu_baseline
leg and `bench.py --impl reference`).

The reference's engine runs pairs in forked worker processes, one per lane
(align.py:299-335); `numpy` mode mirrors that: a fork pool of N processes,
each running the numpy restatement of align.py:79-181 (oracle.align_numpy).
`c` mode runs the plain-C restatement threaded over N pthreads.
Run it in a fresh process (it forks): python -m oracle.cpu_bench --mode numpy
"""

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from oracle import oracle  # noqa: E402

_PAIRS = None
_GAP = None
_MAT = None


def _init(pairs, gap, mat):
    global _PAIRS, _GAP, _MAT
    _PAIRS, _GAP, _MAT = pairs, gap, mat


def _run_chunk(bounds):
    lo, hi = bounds
    out = []
    for a, b in _PAIRS[lo:hi]:
        out.append(oracle.align_numpy(a, b, _GAP[0], _GAP[1], _MAT))
    return out


def sample_pairs(workload: str, n: int, seed: int, offset: int = 0):
    """Pairs [offset, offset + n) of the batch bench.py times for `workload`
    (pastis_synth's packed generators: the first k pairs of a batch do not
    depend on its size), as (str, str)."""
    from pastis_synth import workloads
    gen = {"config2": workloads.config2_packed, "config3": workloads.config3_packed,
           "config5": workloads.config5_packed}[workload]
    arena, table = gen(offset + n, seed=seed)
    raw = arena.tobytes()
    out = []
    for p in table[offset:offset + n].tolist():
        a_off, b_off, la, lb = p
        out.append((raw[a_off:a_off + la].decode(), raw[b_off:b_off + lb].decode()))
    return out


def _warm(_i):
    return oracle.align_numpy("MKVLA", "MKVLA", 11, 1, _MAT)


def time_numpy(pairs, gap, mat, procs: int) -> dict:
    """The reference's process lanes (align.py:299-335) over the numpy
    restatement; lanes are capped so that their 16 B/cell matrices
    (align.py:92-99) fit in 60 % of the free host memory (config 5)."""
    import multiprocessing as mp
    cells = sum(len(a) * len(b) for a, b in pairs)
    biggest = max(((len(a) + 1) * (len(b) + 1) for a, b in pairs), default=1)
    free = os.sysconf("SC_AVPHYS_PAGES") * os.sysconf("SC_PAGE_SIZE")
    procs = max(1, min(procs, len(pairs), int(0.6 * free // (16 * biggest))))
    chunk = max(1, len(pairs) // (procs * 8))
    bounds = [(i, min(len(pairs), i + chunk)) for i in range(0, len(pairs), chunk)]
    ctx = mp.get_context("fork")
    with ctx.Pool(procs, initializer=_init, initargs=(pairs, gap, mat)) as pool:
        pool.map(_warm, range(procs))  # start the workers before timing
        t0 = time.perf_counter()
        res = pool.map(_run_chunk, bounds)
        dt = time.perf_counter() - t0
    n = sum(len(r) for r in res)
    return {"seconds": dt, "pairs": n, "cells": cells, "gcups": cells / dt / 1e9,
            "aln_per_s": n / dt, "cores": procs}


def time_c(pairs, gap, mat, threads: int) -> dict:
    from paper_2303_01845_b200.batch import pack_codes
    arena, table = pack_codes([a.encode() for a, _ in pairs], [b.encode() for _, b in pairs])
    cells = int(np.dot(table["a_len"].astype(np.int64), table["b_len"].astype(np.int64)))
    # pairs whose 16 B/cell matrices would not fit: the O(sqrt(m) n) restatement
    long = int((table["a_len"].astype(np.int64) * table["b_len"]).max(initial=0)) > 50_000_000
    if not long:
        oracle.align_batch_c(arena, table[: min(len(table), threads)], gap[0], gap[1], mat, threads)
    t0 = time.perf_counter()
    oracle.align_batch_c(arena, table, gap[0], gap[1], mat, threads, long=long)
    dt = time.perf_counter() - t0
    return {"seconds": dt, "pairs": len(table), "cells": cells, "gcups": cells / dt / 1e9,
            "aln_per_s": len(table) / dt, "cores": threads,
            "restatement": "orc_align_long (O(sqrt(m) n) memory)" if long else "orc_align"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mode", choices=["numpy", "c"], default="numpy")
    ap.add_argument("--workload", default="config2")
    ap.add_argument("--pairs", type=int, default=2000)
    ap.add_argument("--seed", type=int, default=2303)
    ap.add_argument("--offset", type=int, default=0)
    ap.add_argument("--pairs-file", default=None,
                    help="npz with `arena` (uint8) and `table` (a_off, b_off, a_len, b_len): time "
                         "exactly these pairs (e.g. a pipeline's candidate pairs)")
    ap.add_argument("--procs", type=int, default=0)
    ap.add_argument("--gap-open", type=int, default=11)
    ap.add_argument("--gap-extend", type=int, default=1)
    args = ap.parse_args()
    procs = args.procs or len(os.sched_getaffinity(0))
    from paper_2303_01845_b200 import blosum62
    mat = np.asarray(blosum62.MATRIX, dtype=np.int32)
    if args.pairs_file:
        z = np.load(args.pairs_file)
        raw = z["arena"].tobytes()
        pairs = [(raw[a:a + la].decode(), raw[b:b + lb].decode())
                 for a, b, la, lb in z["table"].tolist()]
    else:
        pairs = sample_pairs(args.workload, args.pairs, args.seed, args.offset)
    gap = (args.gap_open, args.gap_extend)
    if args.mode == "numpy":
        r = time_numpy(pairs, gap, mat, procs)
    else:
        r = time_c(pairs, gap, mat, procs)
    r.update({"mode": args.mode, "workload": args.workload})
    print(json.dumps(r))


if __name__ == "__main__":
    main()

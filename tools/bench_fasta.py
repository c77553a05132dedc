"""FASTA ingest throughput: libpastis_sw.so's sw_fasta_parse
(via seqio.read_fasta_arena / read_fasta) vs the reference's read_fasta on a
config-4-sized file (100k records, lengths U[50, 500], 60-column lines).
Runs on the host (no GPU); the reference leg needs /root/reference.

    python tools/bench_fasta.py [n_records]
"""
import json
import os
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2303_01845_b200 import seqio  # noqa: E402


def best_of(fn, reps=3):
    t = []
    for _ in range(reps):
        t0 = time.perf_counter()
        out = fn()
        t.append(time.perf_counter() - t0)
    return min(t), out


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000
    rng = np.random.default_rng(4)
    std = np.frombuffer(b"ARNDCQEGHILKMFPSTWYV", np.uint8)
    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, "in.fa")
        with open(path, "wb") as fh:
            for k, ln in enumerate(rng.integers(50, 501, size=n)):
                s = std[rng.integers(0, 20, size=int(ln))].tobytes()
                fh.write(b">seq%d synthetic\n" % k)
                for o in range(0, len(s), 60):
                    fh.write(s[o:o + 60] + b"\n")
        mb = os.path.getsize(path) / 1e6
        t_arena, fa = best_of(lambda: seqio.read_fasta_arena(path))
        t_recs, recs = best_of(lambda: seqio.read_fasta(path))
        out = {"records": n, "file_mb": round(mb, 2), "residues": int(fa.arena.size),
               "arena_s": t_arena, "arena_mb_s": mb / t_arena,
               "records_s": t_recs, "records_mb_s": mb / t_recs}
        ref = "/root/reference/pkg/src"
        if os.path.isdir(ref):
            sys.path.insert(0, ref)
            from pastislite import seqio as R
            t_ref, rr = best_of(lambda: R.read_fasta(path), reps=1)
            assert [(r.header, r.residues) for r in rr] == [(r.header, r.residues) for r in recs]
            out.update({"reference_s": t_ref, "reference_mb_s": mb / t_ref,
                        "speedup_arena": t_ref / t_arena, "speedup_records": t_ref / t_recs})
        print(json.dumps(out))


if __name__ == "__main__":
    main()

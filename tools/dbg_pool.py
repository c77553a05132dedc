"""Debug: tiny traceback pool -> fallback paths; print mismatches vs the oracle."""
import json, sys, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2303_01845_b200 import _native, blosum62
from pastis_synth import workloads
from paper_2303_01845_b200.batch import pack_codes
from oracle import oracle
n = int(sys.argv[1]) if len(sys.argv) > 1 else 3000
sa, sb = workloads.config3(n, seed=8)
arena, table = pack_codes(sa, sb)
m = np.asarray(blosum62.MATRIX, np.int32)
rec, tm = _native.align_host(arena, table, _native.make_params(11, 1, m))
ref = oracle.align_batch_c(arena, table, 11, 1, m, threads=16)
F = ("score", "i_begin", "i_end", "j_begin", "j_end", "matches", "aln_len")
got = np.stack([rec[f] for f in F], axis=1)
bad = np.flatnonzero((got != ref[:, :7]).any(axis=1))
print("bad", len(bad), "of", n, "status counts", np.bincount(rec["status"]), "launches", tm["launches"])
for k in bad[:8]:
    print(k, table["a_len"][k], table["b_len"][k], got[k].tolist(), ref[k, :7].tolist(), rec["status"][k])

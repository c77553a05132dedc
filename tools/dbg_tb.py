"""Debug aid: a small config-3 batch through the GPU, compared field by field
with the C oracle; prints the first mismatching pairs."""
import sys
import numpy as np
sys.path.insert(0, '/root/repo')
from oracle import oracle
from paper_2303_01845_b200 import _native, blosum62
from paper_2303_01845_b200.batch import pack_codes
from pastis_synth import workloads

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
mat = np.asarray(blosum62.MATRIX, dtype=np.int32)
sa, sb = workloads.config3(n, seed=5)
arena, table = pack_codes(sa, sb)
rec, tm = _native.align_host(arena, table, _native.make_params(11, 1, mat), device=0)
ref = oracle.align_batch_c(arena, table, 11, 1, mat, threads=8)
fields = ("score", "i_begin", "i_end", "j_begin", "j_end", "matches", "aln_len")
got = np.stack([rec[f] for f in fields], axis=1)
bad = np.flatnonzero((got != ref[:, :7]).any(axis=1) | (rec["status"] != 0))
print(f"{len(bad)} of {n} pairs differ; statuses {np.bincount(rec['status'][bad]) if len(bad) else []}")
for k in bad[:12]:
    print(k, "len", table["a_len"][k], table["b_len"][k], "gpu", got[k].tolist(), "st", rec["status"][k],
          "ref", ref[k, :7].tolist())

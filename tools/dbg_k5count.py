"""Debug aid (K5_COUNT builds only): how many tiles and rows K5 replays per
pair on a config-3 batch -- the j_end search vs the walk.
  tools/build_var.sh k5c -DK5_COUNT; PASTIS_SW_LIB=var/k5c.so python tools/dbg_k5count.py"""
import ctypes
import sys
import numpy as np
sys.path.insert(0, '/root/repo')
from paper_2303_01845_b200 import _native, blosum62
from pastis_synth import workloads

n = int(sys.argv[1]) if len(sys.argv) > 1 else 200000
mat = np.asarray(blosum62.MATRIX, dtype=np.int32)
arena, table = workloads.config3_packed(n, seed=2303)
lib = _native.load()
fn = lib.sw_debug_k5_counters
fn.argtypes = [ctypes.POINTER(ctypes.c_ulonglong)]
buf = (ctypes.c_ulonglong * 8)()
for rep in range(2):
    fn(buf)
    rec, tm = _native.align_host(arena, table, _native.make_params(11, 1, mat), device=0)
    fn(buf)
c = list(buf)
pairs = max(c[0], 1)
print(f"pairs {c[0]}  j-search tiles/pair {c[1]/pairs:.2f} rows/pair {c[2]/pairs:.1f}  "
      f"walk tiles/pair {c[3]/pairs:.2f} rows/pair {c[4]/pairs:.1f}  aln/pair {c[5]/pairs:.1f}  "
      f"rows per aligned column {(c[2]+c[4])/max(c[5],1):.2f}")

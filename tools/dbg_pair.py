import ctypes, numpy as np, sys
sys.path.insert(0, '/root/repo')
from paper_2303_01845_b200 import _native
from paper_2303_01845_b200.batch import pack_pairs
from paper_2303_01845_b200 import blosum62
lib = _native.load()
pairs = [("MKVLAAGIVG", "MKVAAGIVG"), ("AAAA","AAAA")]
b = pack_pairs(pairs)
for ge in (2, 1):
    rec, tm = _native.align_host(b.arena, b.pairs, _native.make_params(11, ge, blosum62.MATRIX))
    st = np.zeros((len(pairs), 12), dtype=np.int32)
    lib.sw_debug_pair_state(0, st.ctypes.data, len(pairs))
    print(ge, rec.tolist())
    print(st[:, :8].tolist(), st[:, 8:10].view(np.uint64).tolist())
pool = np.zeros(2560, dtype=np.uint8)
lib.sw_debug_pool(0, pool.ctypes.data, 2560)
# nibble (rho, kap) for R=4, BPL=2, steps=40
def nib(rho, kap):
    t, r = rho // 4, rho % 4
    s = kap + t
    b = pool[s * 64 + t * 2 + (r >> 1)]
    return (b >> 4) if (r & 1) else (b & 15)
for rho in range(10):
    print(rho, [int(nib(rho, k)) for k in range(9)])

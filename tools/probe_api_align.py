"""Probe: the C-ABI call on the bench arena vs align_packed on the API-packed
batch (pinned records, steady pinned pool after two calls)."""
import sys, time, numpy as np
sys.path.insert(0, "/root/repo")
from pastis_synth import workloads
from paper_2303_01845_b200 import _native, blosum62
from paper_2303_01845_b200.align import _pack, align_packed
from paper_2303_01845_b200 import AlignParams
pool = _native.pinned_pool()
bufs = []
def alloc(nb):
    b = pool.acquire(nb); bufs.append(b); return b.array
arena, table = workloads.config3_packed(1_000_000, seed=2303, alloc=alloc)
p = _native.make_params(11, 1, blosum62.MATRIX)
raw = arena.tobytes()
pairs = [(raw[a:a + la].decode(), raw[b:b + lb].decode(), None) for a, b, la, lb in table[["a_off","b_off","a_len","b_len"]].tolist()]
del raw
params = AlignParams(gap_open=11, gap_extend=1)
for rep in range(4):
    t0 = time.perf_counter(); rec, tm = _native.align_host(arena, table, p, device=0); t1 = time.perf_counter()
    print("bench arena align_host ms", round((t1 - t0) * 1e3, 1), {k: round(v, 2) for k, v in tm.items() if isinstance(v, float)})
batch, pbufs = _pack(pairs)
print("packed arena bytes", batch.arena.nbytes, "bench", arena.nbytes)
for rep in range(4):
    t0 = time.perf_counter(); rec, tms = align_packed(batch, params, (0,)); t1 = time.perf_counter()
    print("api batch align_packed ms", round((t1 - t0) * 1e3, 1), {k: round(v, 2) for k, v in tms[0].items() if isinstance(v, float)})

"""Probe: host packing phases of the drop-in API on 1M config-3 (str, str)
pairs into pinned pool buffers (PASTIS_PACK_DEBUG=1 prints the C phases)."""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from pastis_synth import workloads  # noqa: E402
from paper_2303_01845_b200.align import _pack  # noqa: E402

arena, table = workloads.config3_packed(1_000_000, seed=2303)
raw = arena.tobytes()
pairs = [(raw[a:a + la].decode(), raw[b:b + lb].decode(), None)
         for a, b, la, lb in table[["a_off", "b_off", "a_len", "b_len"]].tolist()]
del raw
print("cores", len(os.sched_getaffinity(0)))
for rep in range(5):
    t0 = time.perf_counter()
    batch, bufs = _pack(pairs)
    dt = time.perf_counter() - t0
    for b in bufs:
        b.release()
    print(f"pack {dt * 1e3:.1f} ms")

if "--engine" in sys.argv:
    import paper_2303_01845_b200 as sw
    eng = sw.AlignEngine(sw.AlignParams(gap_open=11, gap_extend=1), lanes=1, use_processes=True)
    eng.start()
    for rep in range(5):
        t0 = time.perf_counter()
        results, errors, counters, lanes = eng.submit(pairs).result()
        print(f"engine call {(time.perf_counter() - t0) * 1e3:.1f} ms", eng.last_phases)
    eng.close()

if "--idle" in sys.argv:
    for gap_ms in (0, 20, 60, 200):
        ts = []
        for rep in range(4):
            time.sleep(gap_ms / 1e3)
            t0 = time.perf_counter()
            batch, bufs = _pack(pairs)
            ts.append((time.perf_counter() - t0) * 1e3)
            for b in bufs:
                b.release()
        print(f"idle {gap_ms} ms before each pack: pack ms {[round(t, 1) for t in ts]}")

if "--gpu" in sys.argv:
    from paper_2303_01845_b200.align import align_packed
    from paper_2303_01845_b200 import AlignParams
    prm = AlignParams(gap_open=11, gap_extend=1)
    keep = None
    for rep in range(5):
        t0 = time.perf_counter()
        batch, bufs = _pack(pairs)
        t1 = time.perf_counter()
        rec, tms = align_packed(batch, prm, (0,))
        t2 = time.perf_counter()
        for b in bufs:
            b.release()
        keep = rec
        print(f"pack {(t1 - t0) * 1e3:.1f} ms  align {(t2 - t1) * 1e3:.1f} ms")

if "--engine-sync" in sys.argv or "--engine-1" in sys.argv:
    import paper_2303_01845_b200 as sw
    from concurrent.futures import ThreadPoolExecutor
    eng = sw.AlignEngine(sw.AlignParams(gap_open=11, gap_extend=1), lanes=1,
                         use_processes="--engine-1" in sys.argv)
    eng.start()
    if "--engine-1" in sys.argv:
        eng._pool.shutdown()
        eng._pool = ThreadPoolExecutor(max_workers=1)
    for rep in range(5):
        t0 = time.perf_counter()
        results, errors, counters, lanes = eng.submit(pairs).result()
        ph = eng.last_phases
        print(f"engine call {(time.perf_counter() - t0) * 1e3:.1f} ms pack {ph['pack']*1e3:.1f} align {ph['align']*1e3:.1f}")
    eng.close()

if "--engine-del" in sys.argv:
    import gc
    import paper_2303_01845_b200 as sw
    eng = sw.AlignEngine(sw.AlignParams(gap_open=11, gap_extend=1), lanes=1, use_processes=False)
    eng.start()
    for rep in range(5):
        t0 = time.perf_counter()
        results, errors, counters, lanes = eng.submit(pairs).result()
        ph = eng.last_phases
        print(f"engine call {(time.perf_counter() - t0) * 1e3:.1f} ms pack {ph['pack']*1e3:.1f} align {ph['align']*1e3:.1f}")
        del results, errors, counters, lanes
        gc.collect()

if "--bisect" in sys.argv:
    import numpy as np
    from paper_2303_01845_b200.align import align_packed, _to_results, _Lengths, _align
    from paper_2303_01845_b200 import AlignParams
    prm = AlignParams(gap_open=11, gap_extend=1)
    mode = sys.argv[sys.argv.index("--bisect") + 1]
    keep = None
    for rep in range(5):
        if mode == "align":
            out = _align(pairs, prm, [0])
            keep = out
            print(f"_align pack {out[4]['pack']*1e3:.1f} align {out[4]['align']*1e3:.1f}")
            continue
        t0 = time.perf_counter()
        batch, bufs = _pack(pairs)
        t1 = time.perf_counter()
        rec, tms = align_packed(batch, prm, (0,))
        t2 = time.perf_counter()
        if mode in ("copies", "results"):
            la = np.array(batch.pairs["a_len"]); lb = np.array(batch.pairs["b_len"])
            idx = batch.index + 0
        for b in bufs:
            b.release()
        if mode == "results":
            keep = _to_results(_Lengths(la, lb, idx, len(pairs), []), rec)
        else:
            keep = rec
        print(f"{mode}: pack {(t1 - t0) * 1e3:.1f} ms  align {(t2 - t1) * 1e3:.1f} ms")

if "--chunk" in sys.argv:
    import paper_2303_01845_b200.align as al
    import paper_2303_01845_b200 as sw
    for ch in (1 << 40, 500_000, 334_000, 250_000):
        al._CHUNK = ch
        eng = sw.AlignEngine(sw.AlignParams(gap_open=11, gap_extend=1), lanes=1, use_processes=True)
        eng.start()
        ts = []
        for rep in range(5):
            t0 = time.perf_counter()
            results, errors, counters, lanes = eng.submit(pairs).result()
            ts.append((time.perf_counter() - t0) * 1e3)
        eng.close()
        ph = eng.last_phases
        print(f"chunk {ch}: calls ms {[round(t, 1) for t in ts[2:]]} last phases "
              f"{ {k: round(v * 1e3, 1) for k, v in ph.items() if k != 'chunks'} } chunks {ph['chunks']}")

if "--piped" in sys.argv:
    import paper_2303_01845_b200 as sw
    from paper_2303_01845_b200 import _native
    pool = _native.pinned_pool()
    orig = pool.acquire

    def acquire(nbytes):
        n_free = len(pool._free)
        t0 = time.perf_counter()
        b = orig(nbytes)
        dt = (time.perf_counter() - t0) * 1e3
        if dt > 1:
            print(f"  acquire {nbytes / 2**20:.0f} MiB took {dt:.1f} ms (free list {n_free})")
        return b
    pool.acquire = acquire
    eng = sw.AlignEngine(sw.AlignParams(gap_open=11, gap_extend=1), lanes=1, use_processes=True)
    eng.start()
    for rep in range(2):
        eng.submit(pairs).result()
    print("pipelined")
    t0 = time.perf_counter()
    pend = eng.submit(pairs)
    for k in range(4):
        nxt = eng.submit(pairs) if k + 1 < 4 else None
        res = pend.result()
        print(f"batch {k} done at {(time.perf_counter() - t0) * 1e3:.1f} ms phases "
              f"{ {a: round(v * 1e3, 1) for a, v in eng.last_phases.items() if a != 'chunks'} }")
        del res
        pend = nxt
    eng.close()

"""Per-call cost vs batch size (config-3 shapes): device-resident and host
entry points, CUDA-event device time, launches.  Builder probe (not a bench)."""
import sys, time, json
import numpy as np
sys.path.insert(0, ".")
import torch
from paper_2303_01845_b200 import _native, blosum62
from pastis_synth import workloads
from paper_2303_01845_b200.batch import pack_codes

p = _native.make_params(11, 1, blosum62.MATRIX)
sa, sb = workloads.config3_bulk(int(sys.argv[1]) if len(sys.argv) > 1 else 250_000, seed=7)
for n in (256, 2048, 16384, 125_000, 250_000):
    if n > len(sa):
        break
    arena, table = pack_codes(sa[:n], sb[:n])
    cells = int(np.dot(table["a_len"].astype(np.int64), table["b_len"].astype(np.int64)))
    d_arena = torch.from_numpy(arena.copy()).cuda()
    d_pairs = torch.from_numpy(table.view(np.uint8).copy()).cuda()
    d_out = torch.empty(n * 32, dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream()
    rows = []
    for rep in range(6):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0.record(s)
        tm = _native.align_device(d_arena.data_ptr(), arena.size, d_pairs.data_ptr(), n, p,
                                  d_out.data_ptr(), stream=s.cuda_stream)
        e1.record(s)
        torch.cuda.synchronize()
        wall = (time.perf_counter() - t0) * 1e3
        rows.append((e0.elapsed_time(e1), wall, tm["forward_ms"], tm["traceback_ms"], tm["launches"]))
    hrows = []
    for rep in range(4):
        t0 = time.perf_counter()
        _, th = _native.align_host(arena, table, p)
        hrows.append((time.perf_counter() - t0) * 1e3)
    r = rows[-1]
    print(json.dumps({"pairs": n, "cells": cells, "dev_ms": round(min(x[0] for x in rows[2:]), 3),
                      "wall_ms": round(min(x[1] for x in rows[2:]), 3), "fwd_ms": round(r[2], 3),
                      "tb_ms": round(r[3], 3), "launches": r[4],
                      "gcups_dev": round(cells / min(x[0] for x in rows[2:]) / 1e6, 1),
                      "host_ms": round(min(hrows[1:]), 3)}), flush=True)

"""Builder probe: host C-ABI (e2e) vs device-resident call on the benched
config-3 batch, with the engine's per-call debug breakdown
(PASTIS_SW_DEBUG_E2E=1 prints per-class completion times)."""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from paper_2303_01845_b200 import _native, blosum62  # noqa: E402
from pastis_synth import workloads  # noqa: E402

pool = _native.pinned_pool()
bufs = []


def alloc(nb):
    b = pool.acquire(nb)
    bufs.append(b)
    return b.array


arena, table = workloads.config3_packed(1_000_000, seed=2303, alloc=alloc)
pt = pool.acquire(table.nbytes)
pt.array[:] = table.view(np.uint8)
tab = pt.array.view(_native.PAIR_DTYPE)
po = pool.acquire(len(table) * 32)
out = po.array.view(_native.RESULT_DTYPE)
p = _native.make_params(11, 1, blosum62.MATRIX)
for it in range(4):
    t0 = time.perf_counter()
    _, tm = _native.align_host(arena, tab, p, out=out)
    dt = (time.perf_counter() - t0) * 1e3
    print(f"host wall={dt:.2f} kernel={tm['kernel_ms']:.2f} fwd={tm['forward_ms']:.2f} "
          f"h2d={tm['h2d_ms']:.2f} d2h={tm['d2h_ms']:.2f} tail={tm['fwd_tail_ms']:.2f}", flush=True)
da = torch.from_numpy(arena).cuda()
dp = torch.from_numpy(table.view(np.uint8).copy()).cuda()
do = torch.empty(len(table) * 32, dtype=torch.uint8, device="cuda")
for it in range(3):
    t0 = time.perf_counter()
    tm = _native.align_device(da.data_ptr(), arena.size, dp.data_ptr(), len(table), p, do.data_ptr())
    dt = (time.perf_counter() - t0) * 1e3
    print(f"device wall={dt:.2f} kernel={tm['kernel_ms']:.2f} fwd={tm['forward_ms']:.2f} "
          f"tail={tm['fwd_tail_ms']:.2f}", flush=True)

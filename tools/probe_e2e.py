"""Per-call breakdown of the host C-ABI path with pinned buffers (debug aid)."""
import ctypes, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2303_01845_b200 import _native, blosum62
from pastis_synth import workloads
from paper_2303_01845_b200.batch import pack_codes
n = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
sa, sb = workloads.config2(n, seed=2303)
arena, table = pack_codes(sa, sb)
lib = _native.load()
def pinned(nbytes):
    ptr = lib.sw_host_alloc(nbytes)
    return np.ctypeslib.as_array((ctypes.c_uint8 * nbytes).from_address(ptr))
pa = pinned(arena.size); pa[:] = arena
pp = pinned(table.nbytes); pp[:] = table.view(np.uint8)
po = pinned(n * 32)
p = _native.make_params(11, 1, blosum62.MATRIX)
for it in range(6):
    t0 = time.perf_counter()
    _, tm = _native.align_host(pa, pp.view(_native.PAIR_DTYPE), p, out=po.view(_native.RESULT_DTYPE))
    dt = (time.perf_counter() - t0) * 1e3
    print(f"wall={dt:.3f} total={tm['total_ms']:.3f} kernel={tm['kernel_ms']:.3f} fwd={tm['forward_ms']:.3f} "
          f"h2d={tm['h2d_ms']:.3f} d2h={tm['d2h_ms']:.3f} plan={tm['host_plan_ms']:.3f} setup={tm['host_setup_ms']:.3f}")

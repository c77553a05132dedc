"""Per-call timing probe of the device and host entry points (debug aid)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2303_01845_b200 import _native, blosum62
from pastis_synth import workloads
from paper_2303_01845_b200.batch import pack_codes
n = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
sa, sb = workloads.config2(n, seed=2303)
arena, table = pack_codes(sa, sb)
p = _native.make_params(11, 1, blosum62.MATRIX)
dev = torch.device("cuda", 0)
da = torch.from_numpy(arena.copy()).to(dev)
dp = torch.from_numpy(table.view(np.uint8).copy()).to(dev)
do = torch.empty(n * 32, dtype=torch.uint8, device=dev)
for use_torch_stream in (False, True):
    for it in range(4):
        st = torch.cuda.current_stream(dev).cuda_stream if use_torch_stream else 0
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        tm = _native.align_device(da.data_ptr(), arena.size, dp.data_ptr(), n, p, do.data_ptr(),
                                  device=0, stream=st)
        dt = (time.perf_counter() - t0) * 1e3
        print(f"torch_stream={use_torch_stream} it={it} wall={dt:.2f} ms total={tm['total_ms']:.2f} "
              f"kernel={tm['kernel_ms']:.2f} fwd={tm['forward_ms']:.2f} rev={tm['reverse_ms']:.2f} "
              f"tb={tm['traceback_ms']:.2f} launches={tm['launches']} plan={tm['host_plan_ms']:.2f} "
              f"setup={tm['host_setup_ms']:.2f}")
for it in range(3):
    t0 = time.perf_counter()
    rec, tm = _native.align_host(arena, table, p)
    dt = (time.perf_counter() - t0) * 1e3
    print(f"host it={it} wall={dt:.2f} total={tm['total_ms']:.2f} h2d={tm['h2d_ms']:.2f} "
          f"kernel={tm['kernel_ms']:.2f} fwd={tm['forward_ms']:.2f} d2h={tm['d2h_ms']:.2f}")

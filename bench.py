"""Benchmark of the alignment stage (BASELINE.json metric: SW GCUPS and
alignments/s on B200 vs the reference CPU aligner on the host cores).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
                    [--workload config3|config2|config5]

Workload (default): BASELINE.json configs[2] = "config 3", the largest
single-GPU pair batch: 1,000,000 synthetic protein pairs per GPU with
Metaclust-like skewed lengths (len(a) ~ clip(LogNormal(5.5, 0.75), 30, 2000);
half the b's length-correlated homologs with 30 % substitutions + 8 % indels,
half independent draws), BLOSUM62, gap 11/1 (pastis_synth/gen.c, seeded).
One step = the full hot path over that batch: forward score + end cell,
traceback (tile replay / reverse pass + box) -> every AlignmentResult field.
  value   : GCUPS (sum of |a||b| per second) with inputs resident in HBM
            (device C-ABI entry point), CUDA events on the launching stream,
            L2 flushed between steps, max over ranks.
  e2e     : the same metric through the host C-ABI call (sw_align_batch):
            pinned host arena + pair table in, host result records out, the
            copies inside the timed region.
  api_e2e : the same through the reference-shaped Python API
            (AlignEngine.submit(list[(str, str, payload)]).result()), with
            host packing and result materialisation reported separately.
N>1 runs one process per GPU under torchrun (weak scaling: N x 1M pairs).
--impl reference times the reference algorithm (the numpy restatement of
align.py:79-181 in forked lanes over all host cores) on bounded samples of
the same batch.
"""

import argparse
import ctypes
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

GAP = (11, 1)
WORKLOADS = {
    "config3": {"pairs": 1_000_000,
                "desc": "config 3: 1M pairs/GPU, skewed lengths 30-2000 (lognormal, median 245), "
                        "50% homologs, BLOSUM62, gap 11/1",
                "cpu_sample": 24_000, "ref_sample": 3_000},
    "config2": {"pairs": 100_000,
                "desc": "config 2: 100k pairs/GPU of 300x300, 50% homologs, BLOSUM62, gap 11/1",
                "cpu_sample": 64_000, "ref_sample": 4_000},
    "config5": {"pairs": 10_000,
                "desc": "config 5: 10k pairs/GPU, lengths U[2000, 35000] (independent), "
                        "BLOSUM62, gap 11/1",
                "cpu_sample": 4, "ref_sample": 1},
}
DTYPE = "int16x2 (biased u16x2 DPX lanes, exact; int32 re-run on overflow)"


def metric_of(workload: str) -> str:
    return ("SW GCUPS, full alignment incl. traceback (" + WORKLOADS[workload]["desc"] + ")")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="config3", choices=sorted(WORKLOADS))
    ap.add_argument("--pairs", type=int, default=None,
                    help="pairs per GPU (default: the BASELINE config's count)")
    ap.add_argument("--cpu-sample", type=int, default=None,
                    help="pairs in the bounded CPU-baseline sample (~10-20 s of host CPU)")
    ap.add_argument("--ref-sample", type=int, default=None,
                    help="pairs per step of --impl reference (bounded sample)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-api", action="store_true", help="skip the Python-API e2e leg")
    args = ap.parse_args()
    w = WORKLOADS[args.workload]
    args.pairs = args.pairs or w["pairs"]
    args.cpu_sample = args.cpu_sample or w["cpu_sample"]
    args.ref_sample = args.ref_sample or w["ref_sample"]
    return args


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def cpu_bench(mode: str, workload: str, pairs: int, seed: int = 2303, offset: int = 0) -> dict:
    """Run oracle/cpu_bench.py in a fresh process (it forks worker lanes)."""
    cmd = [sys.executable, "-m", "oracle.cpu_bench", "--mode", mode, "--workload", workload,
           "--pairs", str(pairs), "--seed", str(seed), "--offset", str(offset),
           "--gap-open", str(GAP[0]), "--gap-extend", str(GAP[1])]
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, check=True)
    return json.loads(out.stdout.strip().splitlines()[-1])


class ClockSampler:
    """SM clocks + clock-event (throttle) reasons sampled DURING the timed
    region: NVML in-process every 5 ms (nvidia-smi every 200 ms if NVML is
    unavailable).  `timed()` brackets a timed region; the summary covers only
    the samples taken inside those brackets."""

    BITS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
            "sw_power_cap": 0x4}
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
        ids = [x for x in vis.split(",") if x.strip()]
        self.gpu = int(ids[gpu]) if gpu < len(ids) and ids[gpu].strip().isdigit() else gpu
        self.rows = []          # (t, sm_mhz, max_mhz, frozenset(reasons))
        self.windows = []
        self.source = None
        self._stop = threading.Event()
        self._t = None
        self._nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._h = pynvml.nvmlDeviceGetHandleByIndex(self.gpu)
            self._nvml = pynvml
            self.source = "nvml"
        except Exception:  # noqa: BLE001
            self.source = "nvidia-smi"

    def _sample(self):
        if self._nvml is not None:
            nv = self._nvml
            sm = nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)
            mx = nv.nvmlDeviceGetMaxClockInfo(self._h, nv.NVML_CLOCK_SM)
            bits = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
            return float(sm), float(mx), frozenset(n for n, b in self.BITS.items() if bits & b)
        out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                              "--format=csv,noheader,nounits"], capture_output=True,
                             text=True, timeout=5).stdout.strip()
        f = [x.strip() for x in out.split(",")]
        return (float(f[0]), float(f[1]),
                frozenset(n for n, v in zip(self.BITS, f[2:6]) if v.lower() == "active"))

    def _run(self):
        period = 0.005 if self._nvml is not None else 0.2
        while not self._stop.is_set():
            try:
                sm, mx, why = self._sample()
                self.rows.append((time.monotonic(), sm, mx, why))
            except Exception:  # noqa: BLE001
                pass
            self._stop.wait(period)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=10)

    class _Window:
        def __init__(self, owner):
            self.owner = owner

        def __enter__(self):
            self.t0 = time.monotonic()

        def __exit__(self, *exc):
            self.owner.windows.append((self.t0, time.monotonic()))

    def timed(self):
        return self._Window(self)

    def summary(self) -> dict:
        inside = [r for r in self.rows if any(a <= r[0] <= b for a, b in self.windows)]
        rows = inside or self.rows
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        reasons = sorted(set().union(*[r[3] for r in rows]))
        return {"sm_mhz": float(np.median([r[1] for r in rows])),
                "sm_min_mhz": float(min(r[1] for r in rows)),
                "sm_max_mhz": float(max(r[2] for r in rows)), "reasons": reasons,
                "samples": len(inside), "source": self.source,
                "window": "timed region" if inside else "whole run (no sample inside the timed region)"}




# --- roofline context -------------------------------------------------------
CLASS_ROWS = (4, 6, 7, 8, 9, 10, 16)      # sw_kernels.cuh class_rows()
FUSED_MAX_CELLS = 1 << 22                 # kFusedMaxCells: the packed (K1p) pairs


def packed_class_of(m: np.ndarray, n: np.ndarray) -> np.ndarray:
    """Vectorised sw_kernels.cuh packed_class_of (issue-slot cost model)."""
    costs = []
    for R in CLASS_ROWS:
        S = (m + 32 * R - 1) // (32 * R)
        c = S * (n + 31) * (9 * R + 23) + (S - 1) * (n + 31) * 6 + S * 260 * R
        costs.append(c * (1.5 if R >= 12 else 1.0))
    return np.argmin(np.stack(costs), axis=0)


def computed_cells(table) -> dict:
    """Cells K1p computes per algorithmic cell for this batch: each work list
    (class) is sorted by strip count, then n (descending; k_classify) and
    consumed two pairs per warp; a duo computes strips(max m) x 32R rows x
    (max n + 31) wavefront steps in both u16 halves."""
    m = table["a_len"].astype(np.int64)
    n = table["b_len"].astype(np.int64)
    cells = m * n
    k1p = (cells > 0) & (cells <= FUSED_MAX_CELLS)
    if not k1p.any():
        return {"computed_cells_per_cell": None, "k1p_cell_fraction": 0.0}
    m, n = m[k1p], n[k1p]
    cls = packed_class_of(m, n)
    rows_of = np.asarray(CLASS_ROWS)[cls]
    strips = (m + 32 * rows_of - 1) // (32 * rows_of)
    order = np.lexsort((np.arange(len(m)), -n, -strips, cls))
    m, n, cls = m[order], n[order], cls[order]
    comp = 0
    for c, R in enumerate(CLASS_ROWS):
        sel = cls == c
        if not sel.any():
            continue
        mc, nc = m[sel], n[sel]
        if len(mc) % 2:
            mc, nc = np.append(mc, 0), np.append(nc, 0)
        md = np.maximum(mc[0::2], mc[1::2])
        nd = np.maximum(nc[0::2], nc[1::2])
        rows = (md + 32 * R - 1) // (32 * R) * 32 * R
        comp += int((rows * (nd + 31)).sum()) * 2
    alg = int((table["a_len"].astype(np.int64) * table["b_len"].astype(np.int64))[k1p].sum())
    tot = int((table["a_len"].astype(np.int64) * table["b_len"].astype(np.int64)).sum())
    return {"computed_cells_per_cell": comp / alg, "k1p_cell_fraction": alg / tot}


def ncu_fields(workload: str, per_step_ms: float) -> dict:
    """roofline.traffic and the kernel shares of the step from the committed
    ncu captures of this configuration (profiles/r02/ncu_<workload>.json,
    written by tools/ncu_summary.py from `ncu --set full` and the
    gpu__time_duration launch list)."""
    path = os.path.join(ROOT, "profiles", "r02", f"ncu_{workload}.json")
    try:
        with open(path) as fh:
            t = json.load(fh)
    except (OSError, ValueError):
        return {"traffic": None, "traffic_note": f"no committed capture ({path})"}
    out = {"traffic": t.get("traffic_bytes_per_launch"),
           "traffic_unit": "DRAM bytes per launch of the dominant kernel (ncu dram__bytes_read.sum"
                           " + dram__bytes_write.sum, --set full)",
           "algorithmic_bytes_per_launch": t.get("algorithmic_bytes_per_launch"),
           "traffic_note": t.get("note"),
           "kernel_share_ncu": t.get("kernel_share")}
    return out


def hbm_view(alg_bytes: int, cells: int, fwd_ms: float) -> dict:
    """The same forward phase against the HBM roofline (MEASURED_PEAKS.json):
    algorithmic bytes (residues + pair entries + results) per second -- a tiny
    fraction, i.e. HBM is not what bounds the kernel (the int-issue roofline
    above is)."""
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            peak, src = float(json.load(fh)["hbm_gbs"]), "MEASURED_PEAKS.json hbm_gbs"
    except (OSError, KeyError, ValueError):
        peak, src = 6650.0, "fallback (B200_PROFILING.md)"
    ach = alg_bytes / (fwd_ms / 1e3) / 1e9
    return {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
            "peak_source": src, "basis": "algorithmic bytes of the batch / forward-phase time"}


# --- reference arm ----------------------------------------------------------
def run_reference(args, rank: int, world: int) -> None:
    """--impl reference: the reference algorithm on the host cores (rank 0 only),
    each step a bounded sample (consecutive slices) of the batch our arm times."""
    if rank != 0:
        return
    cores = len(os.sched_getaffinity(0))
    vals, secs, alns = [], [], []
    last = None
    for step in range(args.warmup + args.steps):
        r = cpu_bench("numpy", args.workload, args.ref_sample, seed=2303,
                      offset=step * args.ref_sample)
        if step >= args.warmup:
            vals.append(r["cells"] / r["seconds"] / 1e9)
            secs.append(r["seconds"])
            alns.append(r["pairs"] / r["seconds"])
            last = r
    value = float(np.mean(vals))
    line = {
        "impl": "reference",
        "metric": metric_of(args.workload),
        "value": value,
        "unit": "GCUPS",
        "n_gpus": args.gpus,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": float(np.mean(secs)) * 1e3,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "int32 (numpy int32 arrays, as align.py)",
        "data": "synthetic",
        "alignments_per_sec": float(np.mean(alns)),
        "config": {"workload": WORKLOADS[args.workload]["desc"],
                   "sample_pairs_per_step": last["pairs"]},
        "cpu_baseline": {"value": value, "unit": "GCUPS", "cores": cores, "kind": "port",
                         "sample": f"{last['pairs']} consecutive pairs of the benched batch per "
                                   "step; numpy restatement of align.py:79-181 over forked "
                                   "lanes (AlignEngine use_processes=True semantics)"},
        "e2e": {"value": value, "unit": "GCUPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# --- our arm ----------------------------------------------------------------
def make_batch(workload: str, n: int, seed: int, alloc=None):
    from pastis_synth import workloads
    gen = {"config2": workloads.config2_packed, "config3": workloads.config3_packed,
           "config5": workloads.config5_packed}[workload]
    return gen(n, seed=seed, alloc=alloc)


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    # CPU baselines first: the numpy lanes fork, which must precede CUDA init.
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cores = len(os.sched_getaffinity(0))
            rn = cpu_bench("numpy", args.workload, args.cpu_sample)
            rc = cpu_bench("c", args.workload, max(args.cpu_sample, 4 * args.cpu_sample))
            cpu = {"value": rn["gcups"], "unit": "GCUPS", "cores": cores, "kind": "port",
                   "sample": f"first {rn['pairs']} pairs of the benched batch (rank 0); numpy "
                             f"restatement of align.py:79-181 (the reference algorithm) over "
                             f"{cores} forked lanes; {rn['seconds']:.1f} s wall",
                   "alignments_per_sec": rn["aln_per_s"],
                   "c_oracle_gcups": rc["gcups"],
                   "c_oracle_note": f"plain-C restatement (oracle/sw_oracle.c, "
                                    f"{rc.get('restatement', 'orc_align')}), {rc['cores']} "
                                    f"pthreads, first {rc['pairs']} pairs"}
        except Exception as exc:  # noqa: BLE001
            cpu = {"value": None, "unit": "GCUPS", "cores": None, "kind": "port",
                   "sample": f"failed: {exc}"}

    import torch

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)

    from paper_2303_01845_b200 import _native, blosum62

    lib = _native.load()
    params = _native.make_params(GAP[0], GAP[1], blosum62.MATRIX)

    def pinned(nbytes):
        ptr = lib.sw_host_alloc(nbytes)
        if not ptr:   # no page-locked memory left (e.g. many ranks): pageable fallback
            print(f"bench: sw_host_alloc({nbytes}) failed; pageable host memory", file=sys.stderr)
            return None, np.empty(nbytes, dtype=np.uint8)
        return ptr, np.ctypeslib.as_array((ctypes.c_uint8 * nbytes).from_address(ptr))

    pins = []

    def alloc(nbytes):
        ptr, arr = pinned(nbytes)
        pins.append(ptr)
        return arr

    # The batch, generated straight into pinned host memory.  N = 1: the
    # config's pairs.  N > 1 (weak scaling): a global batch of N x that many
    # pairs (the first N x pairs of the same seeded stream) held by every
    # rank, as the node's host memory would hold it; each GPU plans the
    # cell-balanced partition on the device and takes its shard
    # (sw_align_shard), and the result records are gathered to rank 0 over
    # NCCL -- all inside the timed region.
    arena_np, table_np = make_batch(args.workload, args.pairs * world, 2303, alloc=alloc)
    cells_all = int(np.dot(table_np["a_len"].astype(np.int64), table_np["b_len"].astype(np.int64)))
    n_all = len(table_np)
    bounds = _native.shard_ranges(table_np, world)
    n_local = int(bounds[rank + 1] - bounds[rank])

    # device-resident inputs for `value`
    d_arena = torch.from_numpy(arena_np).to(dev)
    d_pairs = torch.from_numpy(table_np.view(np.uint8).copy()).to(dev)
    d_out = torch.empty((max(n_local, n_all if world == 1 else 1), 8), dtype=torch.int32, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2
    stream = torch.cuda.current_stream(dev)

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    def max_over_ranks(xs):
        if world == 1:
            return list(xs)
        t = torch.tensor(list(xs), dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return t.cpu().tolist()

    def gather_to_rank0():
        from paper_2303_01845_b200.distributed import gather_ranges
        return gather_ranges(d_out[:n_local], rank, world, dst=0)

    def device_step():
        if world == 1:
            return _native.align_device(d_arena.data_ptr(), arena_np.size, d_pairs.data_ptr(),
                                        n_all, params, d_out.data_ptr(), device=local,
                                        stream=stream.cuda_stream), d_out
        tm, _ = _native.align_shard(d_arena.data_ptr(), arena_np.size, d_pairs.data_ptr(), n_all,
                                    rank, world, params, d_out.data_ptr(), device=local,
                                    stream=stream.cuda_stream)
        return tm, gather_to_rank0()      # records stay on rank 0's GPU

    step_ms, launches = [], 0
    tms = []
    gathered = None
    with ClockSampler(local) as clocks:
        # warm-up also lets the first clock query (which stalls the driver
        # briefly) happen before the timed region
        for _ in range(args.warmup):
            device_step()
        t_wait = time.time()
        while not clocks.rows and time.time() - t_wait < 10:
            time.sleep(0.05)
        torch.cuda.synchronize()
        barrier()
        with clocks.timed():
            for _ in range(args.steps):
                flush.zero_()
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                torch.cuda.synchronize()
                barrier()
                e0.record(stream)
                tm, gathered = device_step()
                e1.record(stream)
                torch.cuda.synchronize()
                step_ms.append(e0.elapsed_time(e1))
                tms.append(tm)
                launches += tm["launches"]
        barrier()
    step_max = max_over_ranks(step_ms)
    dev_ms = float(np.sum(step_max))
    total_cells = cells_all * args.steps
    value = total_cells / (dev_ms / 1e3) / 1e9
    rec_dev = (gathered.cpu().numpy().view(_native.RESULT_DTYPE).reshape(-1)[:n_all]
               if gathered is not None else None)

    # end to end through the host C-ABI call with pinned buffers
    po_ptr, po = pinned(n_all * 32)
    pins.append(po_ptr)
    pp_ptr, pp = pinned(table_np.nbytes)
    pins.append(pp_ptr)
    pp[:] = table_np.view(np.uint8)
    host_pairs = pp.view(_native.PAIR_DTYPE)
    host_out = po.view(_native.RESULT_DTYPE)
    host_rows = torch.from_numpy(po.view(np.int32).reshape(-1, 8))   # pinned: D2H by DMA

    def host_step():
        t0 = time.perf_counter()
        if world == 1:
            _native.align_host(arena_np, host_pairs, params, device=local, out=host_out)
            res = host_out
        else:
            _native.align_shard(arena_np.ctypes.data, arena_np.size, host_pairs.ctypes.data, n_all,
                                rank, world, params, d_out.data_ptr(), device=local,
                                stream=stream.cuda_stream)
            g = gather_to_rank0()               # records land on rank 0's GPU ...
            res = None
            if g is not None:                   # ... and come down to its pinned host buffer
                host_rows.copy_(g)
                res = host_out
        return (time.perf_counter() - t0) * 1e3, res

    for _ in range(max(1, args.warmup)):
        host_step()
    barrier()
    e2e_ms = []
    res_host = None
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        barrier()
        ms, res_host = host_step()
        e2e_ms.append(ms)
    barrier()
    e2e_total = float(np.sum(max_over_ranks(e2e_ms)))
    e2e_value = total_cells / (e2e_total / 1e3) / 1e9
    ok = True
    if rank == 0:
        ok = bool((res_host["status"] == 0).all()) and bool((res_host == rec_dev).all())
    cells = cells_all // world
    n_pairs = n_all // world

    # end to end through the reference-shaped Python API
    api = None
    if not args.no_api and world == 1:
        api = api_leg(args, arena_np, table_np, cells_all, flush, torch)

    if rank != 0:
        if world > 1:
            torch.distributed.destroy_process_group()
        for p in pins:
            if p:
                lib.sw_host_free(p)
        return

    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    csum = clocks.summary()
    # Integer issue roofline of the minimal Gotoh cell in packed u16x2 form
    # (two cells per lane-op): 4 adds + 5 maxes = 9 issue slots per word
    # (measured on B200: VIMNMX full rate on the ALU pipe, IMAD half rate on
    # the FMA pipe, fused DPX ops half rate on the ALU pipe ->
    # profiles/r01/{dpx_rate,pipe_mix,mix2}.txt).
    slots_per_word = 9.0
    clk_ghz = (csum.get("sm_max_mhz") or 1965.0) / 1e3
    peak_gcups = sms * clk_ghz * 4 * 32 * 2 / slots_per_word
    mean = lambda key: float(np.mean([t[key] for t in tms]))  # noqa: E731
    fwd_ms = mean("forward_ms")
    fwd_gcups = (cells_all if world == 1 else mean("cells")) / (fwd_ms / 1e3) / 1e9
    dominant = ("k_score_cta_packed<8> (K1cp: forward, 2 long pairs per CTA)"
                if args.workload == "config5" else
                "k_score_packed<R> (K1p: forward, 2 pairs per warp, R = 4..16 rows/lane "
                "classes running concurrently)")
    cc = computed_cells(table_np[: args.pairs])
    line = {
        "metric": metric_of(args.workload),
        "value": value,
        "unit": "GCUPS",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": dev_ms / args.steps,
        "step_ms_max_over_ranks": [round(x, 3) for x in step_max],
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": DTYPE,
        "data": "synthetic",
        "alignments_per_sec": n_all * args.steps / (dev_ms / 1e3),
        "forward_gcups": fwd_gcups,
        "phase_ms_per_step": {
            "forward": fwd_ms,
            "tile_traceback_k5": mean("tile_tb_ms"),
            "traceback_past_forward": mean("fwd_tail_ms"),
            "reverse": mean("reverse_ms"),
            "box_traceback": mean("traceback_ms"),
            "note": "forward = fork -> last forward kernel (K1p classes + long-pair K1cp/K1, "
                    "concurrent streams); tile_traceback_k5 = union of K5's class-stream "
                    "intervals (overlaps other classes' forward); traceback_past_forward = "
                    "how long K5 runs after the forward phase; reverse/box_traceback = the "
                    "long-pair chain",
        },
        "results_ok": ok,
        "config": {"workload": WORKLOADS[args.workload]["desc"],
                   "pairs_per_gpu": n_pairs, "cells_per_gpu_per_step": cells,
                   "global_pairs": n_all, "global_cells_per_step": cells_all,
                   "l2": "flushed between timed steps (256 MiB memset, outside the events)",
                   "parallelism": (f"one process per GPU x{world}, weak scaling: a global batch "
                                   f"of {world} x {args.pairs} pairs held by every rank; "
                                   "cell-balanced contiguous ranges planned on the device "
                                   "(sw_align_shard), NCCL gather of the result records to "
                                   "rank 0's GPU, all inside the timed region")
                   if world > 1 else "1 GPU"},
        "roofline": {"bound": "int-issue", "kernel": dominant,
                     "achieved": fwd_gcups, "peak": peak_gcups, "unit": "GCUPS",
                     "frac": fwd_gcups / peak_gcups,
                     "achieved_basis": "algorithmic cells (sum |a||b|) / forward-phase time "
                                       "(CUDA events on the class streams)",
                     "peak_basis": f"{sms} SMs x {clk_ghz:.3f} GHz x 4 SMSP x 32 lanes x 2 cells "
                                   f"(u16x2) / {slots_per_word:.0f} issue slots per packed Gotoh "
                                   "cell (4 adds + 5 maxes); pipe rates measured in tools/microbench",
                     "hbm_note": "algorithmic bytes/cell = (m+n)/(m*n) + 56/(m*n) "
                                 f"= {(arena_np.size + 56 * n_all) / cells_all:.4f} B -> non-binding",
                     "alu_pipe_ceiling": sms * clk_ghz * 4 * 64 / 11.0,
                     "hbm_view": hbm_view((arena_np.size + 56 * n_all) * (n_local / n_all), cells_all, fwd_ms),
                     **cc,
                     **ncu_fields(args.workload, dev_ms / args.steps)},
        "e2e": {"value": e2e_value, "unit": "GCUPS",
                "h2d_bytes_per_step": int(arena_np.size + table_np.nbytes),
                "d2h_bytes_per_step": int(n_all * 32),
                "ms_per_step": e2e_total / args.steps,
                "alignments_per_sec": n_all * args.steps / (e2e_total / 1e3),
                "entry": "sw_align_batch (C ABI, pinned host buffers)" if world == 1 else
                "sw_align_shard per rank (host plan; the range's pairs and bytes uploaded from "
                "pinned host memory, overlapped with the forward) + NCCL gather of the records "
                "to rank 0 + D2H there"},
        "gpu_launches": int(launches),
        "clocks": csum,
    }
    if api is not None:
        line["api_e2e"] = api
    if cpu is not None:
        line["cpu_baseline"] = cpu
    print(json.dumps(line), flush=True)
    for p in pins:
        if p:
            lib.sw_host_free(p)
    if world > 1:
        torch.distributed.destroy_process_group()


def api_leg(args, arena_np, table_np, cells, flush, torch) -> dict:
    """AlignEngine(...).submit([(str, str, None), ...]).result() -- the
    reference's batch seam (align.py:299-347) -- on the same batch."""
    import paper_2303_01845_b200 as sw
    raw = arena_np.tobytes()
    pairs = [(raw[a:a + la].decode(), raw[b:b + lb].decode(), None)
             for a, b, la, lb in table_np.tolist()]
    del raw
    params = sw.AlignParams(gap_open=GAP[0], gap_extend=GAP[1])
    eng = sw.AlignEngine(params, lanes=1, use_processes=True)
    eng.start()
    walls, phases = [], []
    steps = min(args.steps, 3)          # host-heavy leg: a few steps suffice
    # two untimed calls: the engine's pinned pool reaches its steady state
    # (the previous call's results still hold their pinned record buffer
    # while the next call runs, so the second call allocates one more)
    warm = 2
    for step in range(warm + steps):
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        results, errors, counters, lanes = eng.submit(pairs).result()
        dt = time.perf_counter() - t0
        if step >= warm:
            walls.append(dt)
            phases.append(getattr(eng, "last_phases", {}))
    assert not errors and len(results) == len(pairs)
    del results, errors, counters, lanes
    # pipelined: batch k+1 submitted before batch k's result is taken (the
    # reference pipeline's lookahead, pipeline.py:209-212), so its packing
    # runs beside batch k's GPU work on the engine's second host thread
    # (one untimed pipelined round first: two batches in flight need a second
    # pinned arena in the engine's pool, a one-time cudaHostAlloc of ~0.4 s)
    def pipelined(nb):
        done = []
        pend = eng.submit(pairs)
        for k in range(nb):
            nxt = eng.submit(pairs) if k + 1 < nb else None
            res = pend.result()
            done.append(time.perf_counter())
            assert not res[1] and len(res[0]) == len(pairs)
            del res
            pend = nxt
        return done
    pipelined(4)
    torch.cuda.synchronize()
    nb = 8
    done = pipelined(nb)
    # steady state: batches completed per second after the first completion
    piped = (done[-1] - done[0]) / (nb - 1)
    gaps = [round((b - a) * 1e3, 1) for a, b in zip(done, done[1:])]
    eng.close()
    wall = float(np.mean(walls))
    out = {"value": cells / wall / 1e9, "unit": "GCUPS", "ms_per_step": wall * 1e3,
           "alignments_per_sec": len(pairs) / wall,
           "entry": "AlignEngine(lanes=1, use_processes=True).submit(list[(str, str, None)])"
                    ".result()",
           "pipelined": {"value": cells / piped / 1e9, "unit": "GCUPS", "ms_per_batch": piped * 1e3,
                         "batches": nb, "in_flight": 2, "completion_gaps_ms": gaps,
                         "median_gap_ms": float(np.median(gaps)),
                         "note": "submit(batch k+1) before result(batch k): packing overlaps "
                                 "the previous batch's GPU work"}}
    if phases and phases[0]:
        out["phase_ms"] = {k: float(np.mean([p[k] for p in phases])) * 1e3 for k in phases[0]
                           if k != "chunks"}
        out["chunks"] = phases[0].get("chunks")
        out["phase_note"] = ("pack = host packing not hidden behind the GPU (chunk k+1 packs "
                             "while chunk k aligns), align = GPU calls, results = lazy "
                             "result list + counters")
    return out


if __name__ == "__main__":
    main()

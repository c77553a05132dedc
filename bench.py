"""Benchmark of the alignment stage (BASELINE.json metric: SW GCUPS and
alignments/s on B200 vs the reference CPU aligner).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

Workload (BASELINE.json configs[1] = "config 2"): per GPU, 100,000 synthetic
300x300 protein pairs (50% homologs with substitutions + indels), BLOSUM62,
gap 11/1.  One step = the full hot path over that batch: forward score +
end cell, reverse pass, box traceback -> all AlignmentResult fields.
  value : GCUPS with inputs resident in HBM (device C-ABI entry point),
          device time from CUDA events on the launching stream, L2 flushed
          between steps, max over ranks.
  e2e   : the same metric through the host C-ABI call (sw_align_batch):
          pinned host arena + pair table in, host results out, copies timed.
N>1 runs one process per GPU under torchrun (weak scaling: every rank aligns
its own 100k-pair shard); no collective on the data path, only the timing
reductions.  --impl reference times the reference algorithm (the numpy
restatement of align.py, forked process lanes, all host cores) instead.
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

WORKLOAD = "config2"
# BASELINE.json configs: 2 = 100k 300x300 pairs, 3 = 1M skewed-length pairs,
# 5 = 10k long pairs (2,000-35,000 aa)
DEFAULT_PAIRS = {"config2": 100_000, "config3": 1_000_000, "config5": 10_000}
LENGTH = 300
GAP = (11, 1)
METRIC = "SW GCUPS (config 2: 300x300 pairs, BLOSUM62, gap 11/1; full alignment incl. traceback)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--pairs", type=int, default=None,
                    help="pairs per GPU (default: the BASELINE config's count)")
    ap.add_argument("--cpu-sample", type=int, default=64000,
                    help="pairs in the bounded CPU-baseline sample (~12 s on 16 cores)")
    ap.add_argument("--ref-sample", type=int, default=4000,
                    help="pairs per step of --impl reference (bounded sample)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--workload", default=WORKLOAD, choices=["config2", "config3", "config5"],
                    help="exploration only; the headline bench is config2")
    args = ap.parse_args()
    if args.pairs is None:
        args.pairs = DEFAULT_PAIRS[args.workload]
    return args


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def cpu_bench(mode: str, pairs: int, seed: int = 2303) -> dict:
    """Run oracle/cpu_bench.py in a fresh process (it forks worker lanes)."""
    cmd = [sys.executable, "-m", "oracle.cpu_bench", "--mode", mode, "--workload", WORKLOAD,
           "--pairs", str(pairs), "--seed", str(seed), "--gap-open", str(GAP[0]),
           "--gap-extend", str(GAP[1])]
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


def traffic_fields(fwd_ms, args) -> dict:
    """roofline.traffic: DRAM bytes per K1p launch from the committed ncu
    --set full capture (profiles/r01/k1p_traffic.json), beside the algorithmic
    bytes, and the HBM fraction they imply at this run's forward time against
    MEASURED_PEAKS.json's copy bandwidth."""
    out = {"traffic": None}
    if args.workload != "config2" or args.pairs != DEFAULT_PAIRS["config2"]:
        return out      # the capture is of the default configuration
    try:
        with open(os.path.join(ROOT, "profiles", "r01", "k1p_traffic.json")) as fh:
            t = json.load(fh)
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            hbm = float(json.load(fh)["hbm_gbs"])
    except (OSError, KeyError, ValueError):
        return out
    per_launch_s = float(np.mean(fwd_ms)) / 1e3 if len(fwd_ms) else 0.0
    out["traffic"] = t["traffic_bytes_per_launch"]
    out["traffic_unit"] = "bytes per K1p launch (config 2, 100k pairs; ncu dram__bytes_read+write)"
    out["algorithmic_bytes_per_launch"] = t["algorithmic_bytes_per_launch"]
    out["traffic_note"] = t["note"]
    if per_launch_s > 0:
        out["hbm_gbs_at_traffic"] = t["traffic_bytes_per_launch"] / per_launch_s / 1e9
        out["hbm_frac"] = out["hbm_gbs_at_traffic"] / hbm
        out["hbm_peak_gbs"] = hbm
    return out


def run_reference(args, rank: int, world: int) -> None:
    """--impl reference: the reference algorithm on the host cores (rank 0 only)."""
    if rank != 0:
        return
    cores = len(os.sched_getaffinity(0))
    vals = []
    last = None
    for step in range(args.warmup + args.steps):
        r = cpu_bench("numpy", args.ref_sample, seed=2303 + step)
        if step >= args.warmup:
            vals.append(r["gcups"])
            last = r
    value = float(np.mean(vals))
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": value,
        "unit": "GCUPS",
        "n_gpus": args.gpus,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": last["seconds"] * 1e3,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "int32",
        "data": "synthetic",
        "alignments_per_sec": last["aln_per_s"],
        "config": {"workload": f"{WORKLOAD}: {LENGTH}x{LENGTH} pairs, BLOSUM62, gap {GAP[0]}/{GAP[1]}",
                   "sample_pairs_per_step": last["pairs"]},
        "cpu_baseline": {"value": value, "unit": "GCUPS", "cores": cores, "kind": "port",
                         "sample": f"{last['pairs']} pairs of {WORKLOAD} per step; numpy "
                                   "restatement of align.py:79-181 in forked lanes "
                                   "(AlignEngine use_processes=True semantics)"},
        "e2e": {"value": value, "unit": "GCUPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


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
            rn = cpu_bench("numpy", args.cpu_sample)
            rc = cpu_bench("c", max(args.cpu_sample, 8000))
            cpu = {"value": rn["gcups"], "unit": "GCUPS", "cores": cores, "kind": "port",
                   "sample": f"{rn['pairs']} {WORKLOAD} pairs; numpy restatement of "
                             f"align.py:79-181 (the reference algorithm) over {cores} forked "
                             f"lanes; {rn['seconds']:.1f} s wall",
                   "alignments_per_sec": rn["aln_per_s"],
                   "c_oracle_gcups": rc["gcups"],
                   "c_oracle_note": f"plain-C restatement (oracle/sw_oracle.c), {rc['cores']} "
                                    f"pthreads, {rc['pairs']} pairs"}
        except Exception as exc:  # noqa: BLE001
            cpu = {"value": None, "unit": "GCUPS", "cores": None, "kind": "port",
                   "sample": f"failed: {exc}"}

    import torch

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)

    from paper_2303_01845_b200 import _native, blosum62, workloads
    from paper_2303_01845_b200.batch import pack_codes

    lib = _native.load()
    params = _native.make_params(GAP[0], GAP[1], blosum62.MATRIX)
    if args.workload == "config2":
        sa, sb = workloads.config2(args.pairs, seed=2303 + rank, length=LENGTH)
    elif args.workload == "config3":
        sa, sb = workloads.config3_bulk(args.pairs, seed=2303 + rank)
    else:
        sa, sb = workloads.config5(args.pairs, seed=2303 + rank)
    arena_np, table_np = pack_codes(sa, sb)
    cells = int(np.dot(table_np["a_len"].astype(np.int64), table_np["b_len"].astype(np.int64)))
    n_pairs = len(table_np)

    # device-resident inputs for `value`
    d_arena = torch.from_numpy(arena_np.copy()).to(dev)
    d_pairs = torch.from_numpy(table_np.view(np.uint8).copy()).to(dev)
    d_out = torch.empty(n_pairs * 32, dtype=torch.uint8, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)  # > 126 MB L2
    stream = torch.cuda.current_stream(dev)

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        return float(t.item())

    def device_step():
        return _native.align_device(d_arena.data_ptr(), arena_np.size, d_pairs.data_ptr(),
                                    n_pairs, params, d_out.data_ptr(), device=local,
                                    stream=stream.cuda_stream)

    step_ms, fwd_ms, rev_ms, tb_ms, launches = [], [], [], [], 0
    tm = None
    with ClockSampler(local) as clocks:
        # warm-up also lets the first nvidia-smi query (which stalls the
        # driver briefly) happen before the timed region
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
                e0.record(stream)
                tm = device_step()
                e1.record(stream)
                torch.cuda.synchronize()
                step_ms.append(e0.elapsed_time(e1))
                fwd_ms.append(tm["forward_ms"])
                rev_ms.append(tm["reverse_ms"])
                tb_ms.append(tm["traceback_ms"])
                launches += tm["launches"]
        barrier()
    dev_ms = max_over_ranks(float(np.sum(step_ms)))
    fwd_total = max_over_ranks(float(np.sum(fwd_ms)))
    total_cells = cells * world * args.steps
    value = total_cells / (dev_ms / 1e3) / 1e9

    # end to end through the host C-ABI call with pinned buffers
    def pinned(nbytes):
        ptr = lib.sw_host_alloc(nbytes)
        if not ptr:
            raise RuntimeError("sw_host_alloc failed")
        return ptr, np.ctypeslib.as_array((ctypes.c_uint8 * nbytes).from_address(ptr))

    pa_ptr, pa = pinned(max(1, arena_np.size))
    pa[: arena_np.size] = arena_np
    pp_ptr, pp = pinned(table_np.nbytes)
    pp[:] = table_np.view(np.uint8)
    po_ptr, po = pinned(n_pairs * 32)
    host_arena = pa[: arena_np.size]
    host_pairs = pp.view(_native.PAIR_DTYPE)
    host_out = po.view(_native.RESULT_DTYPE)

    def host_step():
        t0 = time.perf_counter()
        _, t = _native.align_host(host_arena, host_pairs, params, device=local, out=host_out)
        return (time.perf_counter() - t0) * 1e3, t

    for _ in range(max(1, args.warmup)):
        host_step()
    barrier()
    e2e_ms = []
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        ms, tmh = host_step()
        e2e_ms.append(ms)
    barrier()
    e2e_total = max_over_ranks(float(np.sum(e2e_ms)))
    e2e_value = total_cells / (e2e_total / 1e3) / 1e9
    ok = bool((host_out["status"] == 0).all())

    if rank != 0:
        if world > 1:
            torch.distributed.destroy_process_group()
        return

    # integer/DPX roofline of the forward kernel (K1), measured DPX issue rate
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    csum = clocks.summary()
    # Integer issue roofline of the minimal Gotoh cell in packed u16x2 form
    # (two cells per lane-op): 4 adds + 5 maxes = 9 issue slots per word, and
    # no formulation needs fewer pipe cycles (measured on B200: VIMNMX full
    # rate on the ALU pipe, IMAD half rate on the FMA pipe, DPX fused ops half
    # rate on the ALU pipe -> profiles/r01/{dpx_rate,pipe_mix,mix2}.txt).
    slots_per_word = 9.0
    clk_ghz = (csum.get("sm_max_mhz") or 1965.0) / 1e3
    peak_gcups = sms * clk_ghz * 4 * 32 * 2 / slots_per_word
    fwd_gcups = cells * args.steps / (float(np.sum(fwd_ms)) / 1e3) / 1e9
    line = {
        "metric": METRIC,
        "value": value,
        "unit": "GCUPS",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": dev_ms / args.steps,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "int32",
        "data": "synthetic",
        "alignments_per_sec": n_pairs * world * args.steps / (dev_ms / 1e3),
        "forward_gcups": fwd_gcups,
        "phase_ms_per_step": {"forward": float(np.mean(fwd_ms)), "reverse": float(np.mean(rev_ms)),
                              "traceback": float(np.mean(tb_ms))},
        "results_ok": ok,
        "config": {"workload": (f"{WORKLOAD}: {args.pairs} pairs/GPU of {LENGTH}x{LENGTH}, "
                                f"BLOSUM62, gap {GAP[0]}/{GAP[1]}, 50% homologs")
                   if args.workload == "config2" else
                   f"{args.workload}: {args.pairs} pairs/GPU, BLOSUM62, gap {GAP[0]}/{GAP[1]}",
                   "pairs_per_gpu": args.pairs, "cells_per_gpu_per_step": cells,
                   "l2": "flushed between timed steps (256 MiB memset, outside the events)",
                   "parallelism": f"weak-scaled shards x{world}"},
        "roofline": {"bound": "int-issue", "kernel": "k_score_packed<R=10> (K1 forward, 2 pairs/warp)",
                     "achieved": fwd_gcups, "peak": peak_gcups, "unit": "GCUPS",
                     "frac": fwd_gcups / peak_gcups,
                     "peak_basis": f"{sms} SMs x {clk_ghz:.3f} GHz x 4 SMSP x 32 lanes x 2 cells "
                                   f"(u16x2) / {slots_per_word:.0f} issue slots per packed Gotoh "
                                   "cell (4 adds + 5 maxes); pipe rates measured in tools/microbench",
                     "hbm_note": "algorithmic bytes/cell = (m+n)/(m*n) + 32/(m*n) = 0.0070 B "
                                 "-> non-binding (HBM would allow ~9e14 CUPS)",
                     # context for `frac`: the ALU-pipe ceiling of the cell as written
                     # (PRMT 2 + 3 VIADDMNMX 6 + VIMNMX3 2 + VIMNMX 1 = 11 ALU-pipe
                     # cycles per packed row-word; ncu shows that pipe at 74 %), and the
                     # cells the kernel computes per algorithmic cell (strip padding
                     # 320/300 rows x wavefront skew (n+31)/n steps at config 2)
                     "alu_pipe_ceiling": sms * clk_ghz * 4 * 64 / 11.0,
                     "computed_cells_per_cell": (320 * 331) / (300 * 300)
                     if args.workload == "config2" else None,
                     **traffic_fields(fwd_ms, args)},
        "e2e": {"value": e2e_value, "unit": "GCUPS",
                "h2d_bytes_per_step": int(arena_np.size + table_np.nbytes),
                "d2h_bytes_per_step": int(n_pairs * 32),
                "ms_per_step": e2e_total / args.steps,
                "alignments_per_sec": n_pairs * world * args.steps / (e2e_total / 1e3)},
        "gpu_launches": int(launches),
        "clocks": csum,
    }
    if cpu is not None:
        line["cpu_baseline"] = cpu
    print(json.dumps(line), flush=True)
    lib.sw_host_free(pa_ptr)
    lib.sw_host_free(pp_ptr)
    lib.sw_host_free(po_ptr)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()

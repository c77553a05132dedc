"""Multi-GPU path: cell-balanced contiguous shards planned on the host or
the device, range uploads, NCCL result gather (sw_align_shard,
sw_align_batch_multi, distributed.align_distributed).  The shard tests run
on one GPU (every shard of a 3-way split in turn); the multi-device ones
need >= 2 GPUs (`gpurun --gpus 2`)."""

import os
import socket

import numpy as np
import pytest

from conftest import FIELDS, ROOT, matrix
from oracle import oracle

pytestmark = pytest.mark.gpu

from paper_2303_01845_b200 import _native  # noqa: E402
from pastis_synth import workloads  # noqa: E402

THREADS = len(os.sched_getaffinity(0))


def _mixed_batch(n=6000, seed=3):
    """config-3 pairs plus long pairs and a handful of repeated sequences."""
    a3, t3 = workloads.config3_packed(n, seed=seed)
    a5, t5 = workloads.config5_packed(6, seed=seed, lo=2000, hi=9000, hom_frac=0.5)
    t5 = t5.copy()
    t5["a_off"] += a3.size
    t5["b_off"] += a3.size
    arena = np.concatenate([a3, a5])
    rep = t3[:50].copy()                      # pairs sharing sequences with earlier pairs
    rep["b_off"], rep["b_len"] = t3["a_off"][50:100], t3["a_len"][50:100]
    return arena, np.concatenate([t3, t5, rep])


@pytest.mark.parametrize("where", ["pinned", "pageable", "device"])
def test_every_shard_of_a_split_is_exact(where):
    import torch
    arena, table = _mixed_batch()
    mat = matrix("blosum62")
    p = _native.make_params(11, 1, mat)
    ref, _ = _native.align_host(arena, table, p)
    bounds = _native.shard_ranges(table, 3)
    if where == "pinned":
        buf = _native.pinned_pool().acquire(arena.size)
        buf.array[:] = arena
        a_ptr, t_ptr = buf.array.ctypes.data, table.ctypes.data
    elif where == "pageable":
        a_ptr, t_ptr = arena.ctypes.data, table.ctypes.data
    else:
        d_a = torch.from_numpy(arena.copy()).cuda()
        d_t = torch.from_numpy(table.view(np.uint8).copy()).cuda()
        a_ptr, t_ptr = d_a.data_ptr(), d_t.data_ptr()
        assert (_native.shard_ranges(t_ptr, 3, len(table)) == bounds).all()   # device plan
    got = np.zeros(len(table), dtype=_native.RESULT_DTYPE)
    d_out = torch.empty(len(table) * 32, dtype=torch.uint8, device="cuda")
    for s in range(3):
        tm, (first, end) = _native.align_shard(a_ptr, arena.size, t_ptr, len(table), s, 3, p,
                                               d_out.data_ptr())
        assert (first, end) == (int(bounds[s]), int(bounds[s + 1]))
        got[first:end] = d_out[: (end - first) * 32].cpu().numpy().view(_native.RESULT_DTYPE)
        cells = int(np.dot(table["a_len"][first:end].astype(np.int64), table["b_len"][first:end]))
        assert tm["cells"] == cells
    assert (got == ref).all()
    full = oracle.align_batch_c(arena, table, 11, 1, mat, threads=THREADS)
    assert (np.stack([got[f] for f in FIELDS], 1) == full[:, :7]).all()


def test_shard_of_invalid_pair_fails_the_call():
    import torch
    arena, table = workloads.config3_packed(500, seed=4)
    bad = table.copy()
    bad["b_off"][17] = arena.size
    p = _native.make_params(11, 1, matrix("blosum62"))
    d_out = torch.empty(500 * 32, dtype=torch.uint8, device="cuda")
    with pytest.raises(ValueError):
        _native.align_shard(arena.ctypes.data, arena.size, bad.ctypes.data, len(bad), 0, 1, p,
                            d_out.data_ptr())


needs2 = pytest.mark.skipif("_native.device_count() < 2", reason="needs >= 2 GPUs")


@needs2
def test_multi_device_batch_exact():
    arena, table = _mixed_batch(20000, seed=9)
    p = _native.make_params(11, 1, matrix("blosum62"))
    ref, _ = _native.align_host(arena, table, p)
    n = _native.device_count()
    for devs in ([0, 1], list(range(n))):
        rec, tms = _native.align_multi(arena, table, p, devs)
        assert (rec == ref).all()
        cells = [t["cells"] for t in tms]
        assert max(cells) - min(cells) <= int(table["a_len"].max()) * int(table["b_len"].max())


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _nccl_worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    from paper_2303_01845_b200 import _native as nat
    from paper_2303_01845_b200.distributed import align_distributed
    from pastis_synth import workloads as w
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world,
                            device_id=torch.device("cuda", rank))
    arena, table = w.config3_packed(30000, seed=21)
    import numpy as _np
    mat = _np.asarray(__import__("paper_2303_01845_b200.blosum62", fromlist=["MATRIX"]).MATRIX,
                      dtype=_np.int32)
    p = nat.make_params(11, 1, mat)
    out = align_distributed(arena, table, p, rank, world, device=rank)
    if rank == 0:
        ref, _ = nat.align_host(arena, table, p, device=0)
        q.put(bool((out == ref).all()))
    dist.barrier()
    dist.destroy_process_group()


@needs2
def test_nccl_distributed_world2_exact():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_nccl_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    ok = q.get(timeout=600)
    for pr in procs:
        pr.join(timeout=120)
    assert ok
    assert all(pr.exitcode == 0 for pr in procs)

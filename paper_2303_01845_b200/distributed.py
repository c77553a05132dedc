"""Multi-GPU shard / gather driver over torch.distributed (one process per GPU).

The reference spreads a batch over process "lanes" with a contiguous ceil
split by pair COUNT (align.py:265-269), which leaves lanes imbalanced when
lengths are skewed.  Here every rank holds the batch (host or device memory)
and calls sw_align_shard with its rank: the batch is cut into contiguous
ranges of equal CELLS (|a|*|b|; sw_shard_ranges -- the same plan on every
rank, no communication), each GPU uploads only its range's pairs and the
bytes they reference (host memory, overlapped with its forward pass) or
aligns them in place (device memory).  The per-rank 32-byte result records,
contiguous in input order, are then gathered to one rank over NCCL (device
tensors; NVLink) and concatenated there -- the only collective of the path.
gloo + a CPU `compute` stand-in serve the CPU tests.
"""

from typing import Callable, Optional

import numpy as np

from . import _native
from ._native import PAIR_DTYPE, RESULT_DTYPE


def partition(table: np.ndarray, world: int) -> np.ndarray:
    """Shard id per pair (the cell-balanced contiguous plan, sw_partition_pairs)."""
    shard, _ = _native.partition(table, world)
    return shard


def local_shard(arena: np.ndarray, table: np.ndarray, shard: np.ndarray, rank: int):
    """(arena_shard, table_shard, index) for `rank`; sequences deduplicated by
    (offset, length) so each referenced byte range is copied once."""
    index = np.flatnonzero(shard == rank).astype(np.int64)
    sub = table[index]
    keys = np.concatenate([np.stack([sub["a_off"], sub["a_len"].astype(np.uint64)], 1),
                           np.stack([sub["b_off"], sub["b_len"].astype(np.uint64)], 1)])
    uniq, inv = np.unique(keys, axis=0, return_inverse=True)
    inv = inv.reshape(-1)
    lens = uniq[:, 1].astype(np.int64)
    new_off = np.concatenate(([0], np.cumsum(lens)[:-1])).astype(np.uint64)
    out = np.empty(int(lens.sum()) or 1, dtype=np.uint8)
    for (off, ln), no in zip(uniq.tolist(), new_off.tolist()):
        out[no:no + ln] = arena[off:off + ln]
    t = np.empty(len(sub), dtype=PAIR_DTYPE)
    n = len(sub)
    t["a_off"] = new_off[inv[:n]]
    t["b_off"] = new_off[inv[n:]]
    t["a_len"] = sub["a_len"]
    t["b_len"] = sub["b_len"]
    return out, t, index


def _comm_device(device):
    """Device for collective buffers: CUDA under NCCL (it rejects CPU
    tensors), CPU otherwise, unless the caller says."""
    import torch
    import torch.distributed as dist
    if device is not None:
        return torch.device(device) if not isinstance(device, torch.device) else device
    if dist.get_backend() == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def gather_records(records: np.ndarray, index: np.ndarray, n_total: int, rank: int, world: int,
                   dst: int = 0, device=None) -> Optional[np.ndarray]:
    """Gather every rank's RESULT_DTYPE records (host arrays) to `dst`, in
    input order."""
    import torch
    dev = _comm_device(device)
    rows = torch.zeros((len(records), 9), dtype=torch.int32)
    if len(records):
        rows[:, :8] = torch.from_numpy(np.ascontiguousarray(records).view(np.int32).reshape(-1, 8))
        rows[:, 8] = torch.from_numpy(np.asarray(index, dtype=np.int64)).to(torch.int32)
    return gather_rows(rows.to(dev), n_total, rank, world, dst)


def gather_rows(rows, n_total: int, rank: int, world: int, dst: int = 0) -> Optional[np.ndarray]:
    """rows: [count, 9] int32 tensor (8 result words + input index) on the
    communication device, in any order.  Pads to the largest count, gathers
    to `dst`, scatters into input order there; records on dst's host (None
    elsewhere).  (The CPU-test path of align_distributed.)"""
    import torch
    import torch.distributed as dist
    dev = rows.device
    cnt = torch.tensor([int(rows.shape[0])], dtype=torch.int64, device=dev)
    counts = [torch.zeros_like(cnt) for _ in range(world)]
    dist.all_gather(counts, cnt)
    cmax = max(int(c.item()) for c in counts)
    buf = torch.full((max(cmax, 1), 9), -1, dtype=torch.int32, device=dev)
    buf[: rows.shape[0]] = rows
    parts = [torch.empty_like(buf) for _ in range(world)] if rank == dst else None
    dist.gather(buf, gather_list=parts, dst=dst)
    if rank != dst:
        return None
    allr = torch.cat(parts)
    allr = allr[allr[:, 8] >= 0]
    out = torch.zeros((n_total, 8), dtype=torch.int32, device=dev)
    out[allr[:, 8].long()] = allr[:, :8]
    return out.cpu().numpy().view(RESULT_DTYPE).reshape(-1)


def gather_ranges(rec, rank: int, world: int, dst: int = 0):
    """rec: [count, 8] int32 device tensor holding this rank's records of its
    contiguous range of the plan (ranks in input order).  NCCL gather to
    `dst` (padded to the largest range), concatenated there: a [n, 8] int32
    DEVICE tensor in input order on dst, None elsewhere."""
    import torch
    import torch.distributed as dist
    dev = rec.device
    cnt = torch.tensor([int(rec.shape[0])], dtype=torch.int64, device=dev)
    counts = [torch.zeros_like(cnt) for _ in range(world)]
    dist.all_gather(counts, cnt)
    counts = [int(c.item()) for c in counts]
    cmax = max(max(counts), 1)
    if rec.shape[0] == cmax:
        buf = rec.contiguous()
    else:
        buf = torch.zeros((cmax, 8), dtype=torch.int32, device=dev)
        buf[: rec.shape[0]] = rec
    parts = [torch.empty_like(buf) for _ in range(world)] if rank == dst else None
    dist.gather(buf, gather_list=parts, dst=dst)
    if rank != dst:
        return None
    return torch.cat([p[:c] for p, c in zip(parts, counts)])


def align_distributed(arena: np.ndarray, table: np.ndarray, params, rank: int, world: int,
                      device: int = 0, dst: int = 0,
                      compute: Optional[Callable] = None, comm_device=None):
    """Shard -> align locally -> gather; returns the records (input order) on
    `dst`, None elsewhere.  GPU path: sw_align_shard on `device` (every rank
    holds the batch; pinned host memory is read zero-copy).  `compute(arena,
    table) -> records` replaces the GPU with a host stand-in (CPU tests):
    the same partition is then made on the host."""
    if compute is not None:
        shard = partition(table, world)
        a_s, t_s, idx = local_shard(arena, table, shard, rank)
        rec = compute(a_s, t_s)
        return gather_records(rec, idx, len(table), rank, world, dst=dst, device=comm_device)
    import torch
    dev = torch.device("cuda", device)
    n = len(table)
    bounds = _native.shard_ranges(table, world)
    nl = int(bounds[rank + 1] - bounds[rank])
    res = torch.empty((max(nl, 1), 8), dtype=torch.int32, device=dev)
    arena = np.ascontiguousarray(arena, dtype=np.uint8)
    table = np.ascontiguousarray(table, dtype=PAIR_DTYPE)
    _, (first, end) = _native.align_shard(arena.ctypes.data, arena.size, table.ctypes.data, n,
                                          rank, world, params, res.data_ptr(), device=device,
                                          stream=torch.cuda.current_stream(dev).cuda_stream)
    assert (first, end) == (int(bounds[rank]), int(bounds[rank + 1]))
    out = gather_ranges(res[:nl], rank, world, dst)
    if out is None:
        return None
    return out.cpu().numpy().view(RESULT_DTYPE).reshape(-1)

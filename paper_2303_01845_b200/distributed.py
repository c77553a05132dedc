"""Multi-GPU shard / gather driver over torch.distributed (one process per GPU).

The reference spreads a batch over process "lanes" with a contiguous ceil
split (align.py:265-269), which leaves lanes imbalanced when lengths are
skewed.  Here every rank holds the batch (host or device memory) and calls
sw_align_shard with its rank: the GPU plans the cell-balanced partition
itself (pairs in stable descending |a|*|b| order dealt in a snake over the
ranks -- the same plan on every rank, no communication), pulls only its
shard's sequence bytes (zero-copy from pinned host memory, or from device
memory) and aligns them.  The per-rank 32-byte result records and their
input positions are then gathered to one rank over NCCL (device tensors;
NVLink) and scattered back into input order on that rank's GPU -- the only
collective of the path.  gloo + a CPU `compute` stand-in serve the CPU tests.
"""

from typing import Callable, Optional

import numpy as np

from . import _native
from ._native import PAIR_DTYPE, RESULT_DTYPE


def partition(table: np.ndarray, world: int) -> np.ndarray:
    """Shard id per pair (LPT over cells, C++ sw_partition_pairs)."""
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
    communication device.  Pads to the largest shard, gathers to `dst` (NCCL:
    device to device), scatters into input order there and returns the
    records on dst's host (None elsewhere)."""
    import torch
    import torch.distributed as dist
    dev = rows.device
    cmax = max(_native.shard_count(n_total, world, r) for r in range(world)) if world else 0
    cmax = max(cmax, int(rows.shape[0]))
    buf = torch.full((cmax, 9), -1, dtype=torch.int32, device=dev)
    buf[: rows.shape[0]] = rows
    parts = [torch.empty_like(buf) for _ in range(world)] if rank == dst else None
    dist.gather(buf, gather_list=parts, dst=dst)
    if rank != dst:
        return None
    allr = torch.cat(parts)
    valid = allr[:, 8] >= 0
    allr = allr[valid]
    out = torch.zeros((n_total, 8), dtype=torch.int32, device=dev)
    out[allr[:, 8].long()] = allr[:, :8]
    return out.cpu().numpy().view(RESULT_DTYPE).reshape(-1)


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
    nl = _native.shard_count(n, world, rank)
    d_out = torch.empty((max(nl, 1), 9), dtype=torch.int32, device=dev)
    d_idx = torch.empty(max(nl, 1), dtype=torch.int32, device=dev)
    res = torch.empty((max(nl, 1), 8), dtype=torch.int32, device=dev)
    arena = np.ascontiguousarray(arena, dtype=np.uint8)
    table = np.ascontiguousarray(table, dtype=PAIR_DTYPE)
    _native.align_shard(arena.ctypes.data, arena.size, table.ctypes.data, n, rank, world, params,
                        res.data_ptr(), d_idx.data_ptr(), device=device,
                        stream=torch.cuda.current_stream(dev).cuda_stream)
    d_out[:, :8] = res
    d_out[:, 8] = d_idx
    return gather_rows(d_out[:nl], n, rank, world, dst)

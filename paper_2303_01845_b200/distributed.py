"""Multi-GPU shard / gather driver over torch.distributed (one process per GPU).

The reference spreads a batch over process "lanes" with a contiguous ceil
split (align.py:265-269), which leaves lanes imbalanced when lengths are
skewed.  Here pairs are partitioned by CELLS (|a|*|b|) with the greedy
least-loaded rule of sw_partition_pairs (LPT); every rank packs only the
sequences its pairs reference (deduplicated arena shard), aligns its shard on
its own GPU with no inter-GPU traffic, and the per-rank 32-byte result
records are gathered to one rank at the end and scattered back into input
order.  The gather is the only collective (NCCL over NVLink for GPU tensors,
gloo for the CPU tests).
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


def gather_records(records: np.ndarray, index: np.ndarray, n_total: int, rank: int, world: int,
                   dst: int = 0, device=None) -> Optional[np.ndarray]:
    """Gather every rank's RESULT_DTYPE records to `dst`, in input order."""
    import torch
    import torch.distributed as dist

    counts = torch.zeros(world, dtype=torch.int64, device=device)
    counts[rank] = len(records)
    dist.all_reduce(counts)
    cmax = int(counts.max().item())
    # records travel as raw int32 rows (8 per record) + their input index
    buf = np.zeros((cmax, 9), dtype=np.int64)
    if len(records):
        buf[: len(records), :8] = records.view(np.int32).reshape(-1, 8)
        buf[: len(records), 8] = index
    t = torch.from_numpy(buf)
    if device is not None:
        t = t.to(device)
    parts = [torch.empty_like(t) for _ in range(world)] if rank == dst else None
    dist.gather(t, gather_list=parts, dst=dst)
    if rank != dst:
        return None
    out = np.empty(n_total, dtype=RESULT_DTYPE)
    flat = out.view(np.int32).reshape(-1, 8)
    for r, p in enumerate(parts):
        c = int(counts[r].item())
        if c == 0:
            continue
        arr = p.cpu().numpy()[:c]
        flat[arr[:, 8]] = arr[:, :8].astype(np.int32)
    return out


def align_distributed(arena: np.ndarray, table: np.ndarray, params, rank: int, world: int,
                      device: int = 0, dst: int = 0,
                      compute: Optional[Callable] = None, comm_device=None):
    """Shard -> align locally -> gather.  `compute(arena, table) -> records`
    defaults to the GPU kernels on `device`; tests substitute the oracle."""
    shard = partition(table, world)
    a_s, t_s, idx = local_shard(arena, table, shard, rank)
    if compute is None:
        rec, _ = _native.align_host(a_s, t_s, params, device=device)
    else:
        rec = compute(a_s, t_s)
    return gather_records(rec, idx, len(table), rank, world, dst=dst, device=comm_device)

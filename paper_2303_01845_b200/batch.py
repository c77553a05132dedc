"""Pair-batching / packing layer: Python pairs -> flat byte arena + pair table.

The reference hands each worker pickled (str, str, payload) tuples
(pipeline.py:307 -> AlignEngine.submit, align.py:327-335).  Here a batch is
packed once, by the C extension `_pack` (csrc/pack_ext.c), into
  * a flat uint8 arena holding every DISTINCT sequence object once (the
    pipeline reuses `residues[i]` objects across pairs, so sequences are
    deduplicated by object identity), raw ASCII bytes exactly as the
    reference receives them, in a caller-chosen buffer (the engine passes
    recycled pinned host memory, so the upload runs at full PCIe speed and
    several GPUs can read it directly), and
  * a pair table (a_off, b_off, a_len, b_len) in input order (sw_pair_t).
Length binning and cell-balanced sharding happen on the device, so they
never reorder results.

Per-pair input errors are detected with the reference's order and exception
types (align.py:81-84): empty -> AlignmentError, then str.encode("ascii")
errors (UnicodeEncodeError) for a, then b; sequences over 65,000 residues
(the GPU aligner's domain) -> ValueError.  A failing pair is reported in
`errors` and left out of the table; the rest of the batch proceeds.
"""

import os
from dataclasses import dataclass, field

import numpy as np

from ._native import PAIR_DTYPE

try:  # drop-in interop: the reference's own exception class when importable
    from pastislite.align import AlignmentError  # type: ignore  # noqa: F401
except ImportError:  # pragma: no cover - the GPU box has no pastislite
    class AlignmentError(ValueError):
        """Same role as pastislite.align.AlignmentError (align.py:33-34)."""

try:
    from . import _pack
except ImportError as exc:  # built by __graft_entry__.build() / build.build_pack()
    raise ImportError("paper_2303_01845_b200._pack is not built: run "
                      "python -c 'import __graft_entry__ as g; g.build()'") from exc

_THREADS = max(1, min(16, len(os.sched_getaffinity(0))))


@dataclass
class PackedBatch:
    arena: np.ndarray                      # uint8, raw residue bytes
    pairs: np.ndarray                      # PAIR_DTYPE, one row per packed pair
    index: np.ndarray                      # int64, packed row -> input position
    n_input: int                           # number of input pairs
    errors: list = field(default_factory=list)  # [(input index, exception)]
    buffer: object = None                  # owner of `arena` (pinned pool slot) or None

    @property
    def cells(self) -> int:
        p = self.pairs
        return int((p["a_len"].astype(np.uint64) * p["b_len"]).sum())   # no BLAS, exact


def _numpy_alloc(nbytes: int) -> np.ndarray:
    return np.empty(nbytes, dtype=np.uint8)


def pack_pairs(pairs, alloc=None, table_alloc=None) -> PackedBatch:
    """Pack (a, b[, payload]) items; invalid pairs are reported, not packed.

    `alloc(nbytes)` returns the writable arena buffer (default: a new numpy
    array); it is called once, after the table is known.  `table_alloc(nbytes)`
    likewise supplies the pair table's buffer (the engine passes pinned memory
    for both)."""
    n = len(pairs)
    if table_alloc is not None and n:
        table = np.asarray(table_alloc(n * PAIR_DTYPE.itemsize)).view(PAIR_DTYPE)[:n]
    else:
        table = np.empty(n, dtype=PAIR_DTYPE)
    index = np.empty(n, dtype=np.int64)
    holder = {}

    def _alloc(nbytes):
        buf = (alloc or _numpy_alloc)(nbytes)
        holder["buf"] = buf
        return buf

    kept, arena, nbytes, errors = _pack.pack(pairs, table, index, _alloc, AlignmentError,
                                             _THREADS)
    arena = np.frombuffer(arena, dtype=np.uint8, count=max(int(nbytes), 1)) \
        if not isinstance(arena, np.ndarray) else arena[: max(int(nbytes), 1)]
    return PackedBatch(arena=arena, pairs=table[:kept], index=index[:kept], n_input=n,
                       errors=errors, buffer=holder.get("buf"))


def pack_codes(seqs_a, seqs_b) -> tuple:
    """Pack already-byte sequences (lists of bytes/uint8 arrays) pairwise,
    without dedup: the bench/test path for synthetic workloads."""
    lens_a = np.fromiter((len(s) for s in seqs_a), dtype=np.uint32, count=len(seqs_a))
    lens_b = np.fromiter((len(s) for s in seqs_b), dtype=np.uint32, count=len(seqs_b))
    inter = []
    for x, y in zip(seqs_a, seqs_b):
        inter.append(bytes(x))
        inter.append(bytes(y))
    arena = np.frombuffer(b"".join(inter) or b"\0", dtype=np.uint8)
    lens = np.empty(2 * len(lens_a), dtype=np.uint64)
    lens[0::2] = lens_a
    lens[1::2] = lens_b
    offs = np.concatenate(([0], np.cumsum(lens)[:-1])).astype(np.uint64)
    table = np.empty(len(lens_a), dtype=PAIR_DTYPE)
    table["a_off"] = offs[0::2]
    table["b_off"] = offs[1::2]
    table["a_len"] = lens_a
    table["b_len"] = lens_b
    return arena, table

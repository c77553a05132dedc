"""Pair-batching / packing layer: Python pairs -> flat byte arena + pair table.

The reference hands each worker pickled (str, str, payload) tuples
(pipeline.py:307 -> AlignEngine.submit, align.py:327-335).  Here a batch is
packed once into
  * a flat uint8 arena holding every DISTINCT sequence once (the pipeline
    reuses `residues[i]` objects across pairs, so sequences are deduplicated
    by object identity first and by value second), raw ASCII bytes exactly as
    the reference receives them, and
  * a pair table (a_off, b_off, a_len, b_len) in input order (sw_pair_t).
Length binning and cell-balanced sharding happen on the device / in the C++
host driver (sw_engine.cu), so they never reorder results.

Per-pair input errors are detected here with the reference's order and
exception types (align.py:81-84): empty -> AlignmentError, then str.encode
("ascii") errors (UnicodeEncodeError) for a, then b.
"""

from dataclasses import dataclass, field

import numpy as np

from ._native import PAIR_DTYPE


class AlignmentError(ValueError):
    """Same role as pastislite.align.AlignmentError (align.py:33-34)."""


@dataclass
class PackedBatch:
    arena: np.ndarray                      # uint8, raw residue bytes
    pairs: np.ndarray                      # PAIR_DTYPE, one row per packed pair
    index: np.ndarray                      # int64, packed row -> input position
    n_input: int                           # number of input pairs
    errors: list = field(default_factory=list)  # [(input index, exception)]

    @property
    def cells(self) -> int:
        p = self.pairs
        return int(np.dot(p["a_len"].astype(np.uint64), p["b_len"].astype(np.uint64)))


def pack_pairs(pairs) -> PackedBatch:
    """Pack (a, b[, payload]) items; invalid pairs are reported, not packed."""
    n = len(pairs)
    by_id: dict = {}
    by_val: dict = {}
    chunks: list = []
    offset = 0
    a_off = np.empty(n, dtype=np.uint64)
    b_off = np.empty(n, dtype=np.uint64)
    a_len = np.empty(n, dtype=np.uint32)
    b_len = np.empty(n, dtype=np.uint32)
    keep = np.ones(n, dtype=bool)
    errors = []

    def place(s):
        nonlocal offset
        key = id(s)
        hit = by_id.get(key)
        if hit is not None and hit[0] is s:
            return hit[1]
        o = by_val.get(s)
        if o is None:
            raw = s.encode("ascii")
            o = offset
            chunks.append(raw)
            offset += len(raw)
            by_val[s] = o
        by_id[key] = (s, o)
        return o

    for idx, item in enumerate(pairs):
        a, b = item[0], item[1]
        try:
            if not a or not b:
                raise AlignmentError("cannot align an empty sequence")
            oa = place(a)
            ob = place(b)
        except Exception as exc:  # noqa: BLE001 - per-pair isolation (align.py:236-241)
            keep[idx] = False
            errors.append((idx, exc))
            continue
        a_off[idx] = oa
        b_off[idx] = ob
        a_len[idx] = len(a)
        b_len[idx] = len(b)

    arena = np.frombuffer(b"".join(chunks) or b"\0", dtype=np.uint8)
    index = np.flatnonzero(keep).astype(np.int64)
    table = np.empty(len(index), dtype=PAIR_DTYPE)
    table["a_off"] = a_off[index]
    table["b_off"] = b_off[index]
    table["a_len"] = a_len[index]
    table["b_len"] = b_len[index]
    return PackedBatch(arena=arena, pairs=table, index=index, n_input=n, errors=errors)


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

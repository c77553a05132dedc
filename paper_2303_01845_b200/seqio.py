"""FASTA ingest for the alignment stage, drop-in for
pastislite.seqio.read_fasta (/root/reference/pkg/src/pastislite/seqio.py:42-92).

`read_fasta(path)` returns the same records as the reference (ids 0..n-1 in
file order, header = first token of the '>' line, residues upper-cased with
bytes outside the alphabet mapped to 'X'), raises `FastaError` (a ValueError)
with the reference's message for the same first error, and logs the same
"mapped %d residue bytes" warning.  `read_fasta_arena(path)` returns the
residues already laid out as the byte arena `sw_align_batch` consumes, so a
pipeline can pack candidate pairs as offsets into it with no per-sequence
copies (`arena_pairs`).

The parse runs in libpastis_sw.so (`sw_fasta_parse`, host code, no GPU).
Non-ASCII text needs Python's Unicode `str.strip` / `str.upper` semantics and
is parsed by `_parse_unicode`, a restatement of the same rules on `str`.
"""

import logging
from dataclasses import dataclass

import numpy as np

from . import _native
from .alphabet import ALPHABET

log = logging.getLogger(__name__)

UNKNOWN = "X"


class FastaError(ValueError):
    """seqio.py:19"""


@dataclass(slots=True)
class SequenceRecord:
    """seqio.py:23-27"""

    id: int
    header: str
    residues: str


@dataclass
class FastaArena:
    """Residues of every record back to back (uint8 ASCII), in file order."""

    arena: np.ndarray       # uint8
    offsets: np.ndarray     # uint64, residues of record k: arena[offsets[k]:offsets[k]+lengths[k]]
    lengths: np.ndarray     # uint32
    headers: list
    n_mapped: int = 0

    def __len__(self) -> int:
        return len(self.headers)

    def residues(self, k: int) -> str:
        o = int(self.offsets[k])
        return self.arena[o:o + int(self.lengths[k])].tobytes().decode("ascii")

    def records(self) -> list:
        return [SequenceRecord(k, h, self.residues(k)) for k, h in enumerate(self.headers)]


def _errors(kind: int, path, header: str = "") -> FastaError:
    if kind == _native.FASTA_DATA_BEFORE_HEADER:
        return FastaError(f"residue data before first header in {path}")
    if kind == _native.FASTA_EMPTY_HEADER:
        return FastaError("record with empty description line")
    if kind == _native.FASTA_EMPTY_SEQ:
        return FastaError(f"record {header!r} has an empty sequence")
    return FastaError(f"no FASTA records in {path}")


def _parse_unicode(path) -> FastaArena:
    """Non-ASCII input: the same rules on decoded text (universal newlines,
    str.strip / str.split / str.upper), one character at a time."""
    letters = set(ALPHABET)
    headers, seqs = [], []
    cur, parts, mapped = None, [], 0

    def close():
        nonlocal mapped
        if cur is None:
            return
        up = "".join(parts).upper()
        out = "".join(ch if ch in letters else UNKNOWN for ch in up)
        mapped += sum(1 for ch in up if ch not in letters)
        if not out:
            raise _errors(_native.FASTA_EMPTY_SEQ, path, cur)
        headers.append(cur)
        seqs.append(out)

    with open(path, "r", encoding="utf-8") as fh:
        for raw in fh:
            line = raw.strip()
            if not line:
                continue
            if line[0] == ">":
                close()
                tokens = line[1:].split()
                if not tokens:
                    raise _errors(_native.FASTA_EMPTY_HEADER, path)
                cur, parts = tokens[0], []
            elif cur is None:
                raise _errors(_native.FASTA_DATA_BEFORE_HEADER, path)
            else:
                parts.append(line)
    close()
    if not headers:
        raise _errors(_native.FASTA_NO_RECORDS, path)
    data = "".join(seqs).encode("ascii")
    lengths = np.array([len(x) for x in seqs], dtype=np.uint32)
    offsets = np.zeros(len(seqs), dtype=np.uint64)
    if len(seqs) > 1:
        offsets[1:] = np.cumsum(lengths[:-1], dtype=np.uint64)
    return FastaArena(np.frombuffer(data, dtype=np.uint8).copy(), offsets, lengths, headers, mapped)


def read_fasta_arena(path) -> FastaArena:
    """Parse a FASTA file straight into a residue arena (seqio.py:42-92 rules)."""
    with open(path, "rb") as fh:
        text = fh.read()
    arena, hdr, recs, info = _native.fasta_parse(text)
    if info["error"] == _native.FASTA_NONASCII:
        fa = _parse_unicode(path)
    elif info["error"]:
        h0 = int(info["error_hdr_off"])
        header = hdr[h0:h0 + int(info["error_hdr_len"])].decode("ascii")
        raise _errors(info["error"], path, header)
    else:
        hs = hdr.decode("ascii")          # ASCII: byte offsets are str offsets
        ends = (recs["hdr_off"] + recs["hdr_len"]).tolist()
        headers = [hs[o:e] for o, e in zip(recs["hdr_off"].tolist(), ends)]
        fa = FastaArena(arena, recs["off"].astype(np.uint64), recs["len"].astype(np.uint32),
                        headers, int(info["n_mapped"]))
    if fa.n_mapped:
        log.warning("mapped %d residue bytes outside the alphabet to %r", fa.n_mapped, UNKNOWN)
    return fa


def read_fasta(path) -> list:
    """Drop-in for seqio.read_fasta: list[SequenceRecord] with ids 0..n-1."""
    return read_fasta_arena(path).records()


def arena_pairs(fa: FastaArena, ids_a, ids_b) -> np.ndarray:
    """sw_pair_t table for candidate pairs (a = rows = record ids_a[k], b =
    columns = ids_b[k]) as offsets into fa.arena -- the pipeline's
    orientation a = min(i, j), b = max(i, j) (pipeline.py:297-302) is the
    caller's choice, as in the reference."""
    ia = np.asarray(ids_a, dtype=np.int64)
    ib = np.asarray(ids_b, dtype=np.int64)
    t = np.empty(len(ia), dtype=_native.PAIR_DTYPE)
    t["a_off"] = fa.offsets[ia]
    t["b_off"] = fa.offsets[ib]
    t["a_len"] = fa.lengths[ia]
    t["b_len"] = fa.lengths[ib]
    return t

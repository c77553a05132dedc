"""Candidate discovery feeding the aligner, on the GPU.

Replaces the reference's candidate stage -- sequence-by-k-mer matrix
(pastislite.kmer.build_kmer_matrix, kmer.py:56-90), overlap-semiring product
A*A^T as a blocked 2D sparse SUMMA with symmetry pruning (kmer.py:93-126,
sparse.py:236, summa.py, balance.py) and the threshold/orientation filter
(pipeline.py:290-303) -- with sw_kmer_candidates (csrc/sw_kmer.cuh): sorts of
k-mer keys and of shared-k-mer pair keys.  The result is the reference's
candidate set, independent of its blocking, worker grid and pruning scheme:
every pair i < j sharing >= min_shared_kmers distinct k-mers, with the count.
"""

from dataclasses import dataclass

import numpy as np

from . import _native
from .alphabet import SIZE
from .seqio import FastaArena

CANDIDATE_DTYPE = _native.CANDIDATE_DTYPE


@dataclass(frozen=True)
class KmerParams:
    """kmer.KmerParams (kmer.py:26-45): same fields, defaults and checks."""

    k: int = 6
    alphabet_size: int = SIZE
    min_shared_kmers: int = 2

    def __post_init__(self):
        if self.k < 1:
            raise ValueError("k must be >= 1")
        if self.alphabet_size != SIZE:
            raise ValueError(f"alphabet size is fixed at {SIZE}")
        if self.min_shared_kmers < 0:
            raise ValueError("min_shared_kmers must be >= 0")

    @property
    def code_space(self) -> int:
        return self.alphabet_size ** self.k


def _as_arena(source):
    if isinstance(source, FastaArena):
        return source.arena, source.offsets, source.lengths
    seqs = [getattr(r, "residues", r) for r in source]
    raw = [s.encode("ascii") if isinstance(s, str) else bytes(s) for s in seqs]
    lengths = np.array([len(b) for b in raw], dtype=np.uint32)
    offsets = np.zeros(len(raw), dtype=np.uint64)
    if len(raw) > 1:
        offsets[1:] = np.cumsum(lengths[:-1], dtype=np.uint64)
    arena = np.frombuffer(b"".join(raw), dtype=np.uint8) if raw else np.zeros(0, np.uint8)
    return arena, offsets, lengths


def kmer_candidates(source, params: KmerParams = KmerParams(), device: int = 0):
    """Candidate pairs of `source` (a FastaArena, or records / strings in id
    order): structured array (i, j, count) sorted by (i, j), i < j, count >=
    params.min_shared_kmers; plus the discovery counters (positions, distinct
    (sequence, k-mer) entries, shared-k-mer buckets, pair emissions,
    discovered = pairs sharing >= 1 k-mer, performed = candidates, the
    semiring flops of A*A^T, sequences shorter than k, device ms)."""
    arena, offsets, lengths = _as_arena(source)
    cand, stats = _native.kmer_candidates(arena, offsets, lengths, params.k,
                                          params.min_shared_kmers, device=device)
    return cand, stats

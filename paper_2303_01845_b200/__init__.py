"""B200-native batched Smith-Waterman for the PASTIS alignment stage.

Drop-in for the alignment API of the reference package pastislite
(/root/reference/pkg/src/pastislite/__init__.py:9): the same names, fields
and error behaviour, computed by hand-written sm_100a kernels through the C
ABI in include/pastis_sw.h.
"""

from .align import (
    AlignEngine,
    AlignmentError,
    AlignmentResult,
    AlignParams,
    BatchCounters,
    align_batch,
    align_packed,
    encode,
    evaluate_pair,
    smith_waterman,
)
from .batch import PackedBatch, pack_pairs
from .edges import SimilarityEdge, canonical_bytes, evaluate_records, format_edge_line
from .seqio import FastaArena, FastaError, SequenceRecord, arena_pairs, read_fasta, read_fasta_arena

__version__ = "0.1.0"

__all__ = [
    "AlignEngine",
    "AlignParams",
    "AlignmentError",
    "AlignmentResult",
    "BatchCounters",
    "FastaArena",
    "FastaError",
    "PackedBatch",
    "SequenceRecord",
    "SimilarityEdge",
    "align_batch",
    "align_packed",
    "arena_pairs",
    "canonical_bytes",
    "encode",
    "evaluate_pair",
    "evaluate_records",
    "format_edge_line",
    "pack_pairs",
    "read_fasta",
    "read_fasta_arena",
    "smith_waterman",
]

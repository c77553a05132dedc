"""Result consumption: similarity edges and their triplet lines.

SimilarityEdge mirrors /root/reference/pkg/src/pastislite/seqio.py:30-39,
format_edge_line mirrors seqio.py:101-110 (4-decimal fractions) and
canonical_bytes mirrors canonicalize_output (seqio.py:145-153).
evaluate_records is the vectorised form of evaluate_pair (align.py:184-208):
the same float64 divisions and >= comparisons, so accept/reject decisions and
the formatted values are identical to the per-pair Python loop of
pipeline.py:233-236.
"""

from dataclasses import dataclass

import numpy as np


try:  # drop-in interop: the reference's own edge class when importable
    from pastislite.seqio import SimilarityEdge  # type: ignore  # noqa: F401
except ImportError:  # pragma: no cover - the GPU box has no pastislite
    @dataclass(slots=True)
    class SimilarityEdge:
        """Canonical undirected edge: i < j, fractions in [0, 1]."""

        i: int
        j: int
        score: int
        identity: float
        coverage_i: float
        coverage_j: float


def format_edge_line(edge: SimilarityEdge, headers) -> str:
    return (
        f"{headers[edge.i]}\t{headers[edge.j]}\t{edge.score}"
        f"\t{edge.identity:.4f}\t{edge.coverage_i:.4f}\t{edge.coverage_j:.4f}"
    )


def canonical_bytes(lines) -> bytes:
    """Sorted triplet lines joined by '\\n' with a trailing newline."""
    enc = sorted(ln.encode("utf-8") if isinstance(ln, str) else ln for ln in lines)
    enc = [ln for ln in enc if ln]
    out = b"\n".join(enc)
    return out + b"\n" if enc else out


def evaluate_records(ids_i, ids_j, len_a, len_b, rec, min_identity: float, min_coverage: float):
    """Vectorised evaluate_pair over a RESULT_DTYPE array.

    Returns (accepted mask, identity, cov_a, cov_b) as float64 arrays."""
    ids_i = np.asarray(ids_i)
    ids_j = np.asarray(ids_j)
    if np.any(ids_i >= ids_j):
        k = int(np.flatnonzero(ids_i >= ids_j)[0])
        raise ValueError(f"pair not canonical: ({int(ids_i[k])}, {int(ids_j[k])})")
    aln = rec["aln_len"].astype(np.float64)
    nonempty = rec["aln_len"] > 0
    with np.errstate(divide="ignore", invalid="ignore"):
        identity = rec["matches"].astype(np.float64) / aln
    cov_a = (rec["i_end"] - rec["i_begin"] + 1).astype(np.float64) / np.asarray(len_a, np.float64)
    cov_b = (rec["j_end"] - rec["j_begin"] + 1).astype(np.float64) / np.asarray(len_b, np.float64)
    accept = nonempty & (identity >= min_identity) & (np.minimum(cov_a, cov_b) >= min_coverage)
    return accept, identity, cov_a, cov_b

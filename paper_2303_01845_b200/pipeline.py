"""The search pipeline on GPUs: FASTA -> candidates -> alignment -> edges.

Mirrors pastislite.pipeline.run_search (/root/reference/pkg/src/pastislite/
pipeline.py:180-323) for the paths SURVEY 8 puts in scope: FASTA ingest
into the aligner's arena (seqio.read_fasta_arena, sw_fasta_parse), candidate
discovery (candidates.kmer_candidates, sw_kmer_candidates: the reference's
k-mer matrix + overlap SpGEMM + pruning + threshold, pipeline.py:241-303),
batched Smith-Waterman (sw_align_batch / sw_align_batch_multi, the
AlignEngine path, pipeline.py:304-314), the identity/coverage filter
(evaluate_pair, pipeline.py:233-236, vectorised) and the triplet writer
(EdgeWriter, seqio.py:112-134).  The output file holds the same edges as the
reference's; its canonical form (canonicalize_output) is byte-identical --
the line order differs, as it does between the reference's own blockings.

The reference's PipelineConfig carries the parameters of its CPU sparse
engine (blocking, scheme, workers, lanes); they do not change the result
and are accepted but not used here.
"""

from dataclasses import asdict, dataclass, field
from time import perf_counter
from typing import Optional

import numpy as np

from . import _native
from .align import AlignParams, _device_ids, _native_params
from .candidates import KmerParams, kmer_candidates
from .edges import SimilarityEdge, evaluate_records, format_edge_line
from .seqio import arena_pairs, read_fasta_arena


class PipelineError(RuntimeError):
    """pipeline.py PipelineError: a stage failed."""


@dataclass
class PipelineConfig:
    """pipeline.PipelineConfig's result-relevant fields (kmer, align) plus the
    GPUs to use (None: all visible, PASTIS_SW_DEVICES honoured).  A reference
    PipelineConfig works too (duck-typed .kmer / .align)."""

    kmer: KmerParams = field(default_factory=KmerParams)
    align: AlignParams = field(default_factory=AlignParams)
    devices: Optional[tuple] = None
    blocks: int = 4       # pre-blocking: alignment blocks (one in flight beside the host filter)


@dataclass
class RunStats:
    """pipeline.RunStats (pipeline.py:71-90), same fields and meanings; the
    sparse timers cover the GPU candidate stage."""

    discovered_candidates: int
    performed_alignments: int
    output_edges: int
    align_seconds: float
    spgemm_seconds: float
    sparse_all_seconds: float
    io_seconds: float
    cwait_seconds: float
    total_seconds: float
    alignments_per_second: float
    cups: float
    imbalance_align_pct: float
    imbalance_sparse_pct: float
    compression_factor: float
    peak_live_blocks: int

    def to_json(self) -> dict:
        return asdict(self)


def _imbalance(xs) -> float:
    xs = [float(x) for x in xs]
    if len(xs) <= 1:
        return 0.0
    avg = sum(xs) / len(xs)
    return 100.0 * (max(xs) - avg) / avg if avg > 0 else 0.0


def run_search(config, input_path, output_path) -> RunStats:
    """Run the full search; writes triplet lines to output_path and returns
    the run statistics (pipeline.py:180)."""
    t_start = perf_counter()
    kparams = KmerParams(k=config.kmer.k, min_shared_kmers=config.kmer.min_shared_kmers)
    aparams = config.align
    devices = list(getattr(config, "devices", None) or _device_ids(1 << 30))

    t0 = perf_counter()
    fa = read_fasta_arena(input_path)
    io_s = perf_counter() - t0

    t0 = perf_counter()
    cand, kst = kmer_candidates(fa, kparams, device=devices[0])
    sparse_s = perf_counter() - t0

    t0 = perf_counter()
    ii = cand["i"].astype(np.int64)
    jj = cand["j"].astype(np.int64)
    table = arena_pairs(fa, ii, jj)
    p = _native_params(aparams) if isinstance(aparams, AlignParams) else _native.make_params(
        aparams.gap_open, aparams.gap_extend, np.asarray(aparams.matrix, dtype=np.int32))
    headers = fa.headers
    # Pre-blocking (pipeline.py:209-212, 305-314): the candidate list is cut
    # into blocks; the GPU aligns block b+1 (a host thread: the ctypes call
    # releases the GIL) while this thread filters and formats block b's edges.
    n_blocks = max(1, min(int(getattr(config, "blocks", 4)), len(table) // 20000 or 1))
    bounds = np.linspace(0, len(table), n_blocks + 1).astype(np.int64)
    from concurrent.futures import ThreadPoolExecutor

    def align_block(b):
        sub = table[bounds[b]:bounds[b + 1]]
        if len(sub) == 0:
            return np.empty(0, dtype=_native.RESULT_DTYPE), []
        if len(devices) == 1:
            r, tm = _native.align_host(fa.arena, sub, p, device=devices[0])
            return r, [tm]
        return _native.align_multi(fa.arena, sub, p, devices)

    lines, tms, io_w, per_dev = [], [], 0.0, {}
    with ThreadPoolExecutor(max_workers=1, thread_name_prefix="pastis-align") as pool:
        fut = pool.submit(align_block, 0)
        for b in range(n_blocks):
            rec_b, tms_b = fut.result()
            if b + 1 < n_blocks:
                fut = pool.submit(align_block, b + 1)     # in flight while we filter block b
            tms += tms_b
            for d_i, t in enumerate(tms_b):
                per_dev[d_i] = per_dev.get(d_i, 0.0) + t["forward_ms"]
            s0, s1 = int(bounds[b]), int(bounds[b + 1])
            bad = np.flatnonzero(rec_b["status"] != 0) if len(rec_b) else []
            if len(bad):
                k = s0 + int(bad[0])
                raise PipelineError(f"stage align: pair ({int(ii[k])}, {int(jj[k])}): status "
                                    f"{int(rec_b['status'][k - s0])}")
            tw = perf_counter()
            accept, identity, cov_a, cov_b = evaluate_records(
                ii[s0:s1], jj[s0:s1], table["a_len"][s0:s1], table["b_len"][s0:s1], rec_b,
                aparams.min_identity, aparams.min_coverage)
            for k in np.flatnonzero(accept).tolist():
                e = SimilarityEdge(int(ii[s0 + k]), int(jj[s0 + k]), int(rec_b["score"][k]),
                                   float(identity[k]), float(cov_a[k]), float(cov_b[k]))
                lines.append(format_edge_line(e, headers))
            io_w += perf_counter() - tw
    align_s = perf_counter() - t0 - io_w

    t0 = perf_counter()
    with open(output_path, "w", encoding="utf-8", newline="\n") as fh:
        if lines:
            fh.write("\n".join(lines) + "\n")
    n_out = len(lines)
    io_s += io_w + perf_counter() - t0

    total = perf_counter() - t_start
    cells = int(np.sum(table["a_len"].astype(np.int64) * table["b_len"].astype(np.int64)))
    kernel_s = sum(t["forward_ms"] for t in tms) / 1e3
    # the reference's overlap nnz counts every computed entry of A*A^T
    # (both orders and the diagonal, index scheme): 2 * discovered + rows
    # with at least one k-mer
    nonempty = int(np.count_nonzero(fa.lengths >= kparams.k))
    overlap_nnz = 2 * int(kst["discovered"]) + nonempty
    return RunStats(
        discovered_candidates=int(kst["discovered"]),
        performed_alignments=int(kst["performed"]),
        output_edges=n_out,
        align_seconds=align_s,
        spgemm_seconds=kst["device_ms"] / 1e3,
        sparse_all_seconds=sparse_s,
        io_seconds=io_s,
        cwait_seconds=0.0,
        total_seconds=total,
        alignments_per_second=(int(kst["performed"]) / total) if total > 0 else 0.0,
        cups=(cells / kernel_s) if kernel_s > 0 else 0.0,
        imbalance_align_pct=_imbalance(list(per_dev.values())),
        imbalance_sparse_pct=0.0,
        compression_factor=(int(kst["flops"]) / overlap_nnz) if overlap_nnz else 0.0,
        peak_live_blocks=min(2, n_blocks) if len(table) else 0,
    )


def canonical_digest(path) -> str:
    """sha256 of canonicalize_output(path) (seqio.py:145-153)."""
    import hashlib
    data = open(path, "rb").read()
    lines = sorted(ln for ln in data.split(b"\n") if ln)
    out = b"\n".join(lines) + (b"\n" if lines else b"")
    return hashlib.sha256(out).hexdigest()


__all__ = ["PipelineConfig", "PipelineError", "RunStats", "canonical_digest", "run_search"]

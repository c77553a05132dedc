"""Drop-in GPU replacement of pastislite.align (the reference's alignment stage).

Same names, signatures, result fields and error behaviour as
/root/reference/pkg/src/pastislite/align.py:
  AlignParams       align.py:37-52   (validation identical)
  AlignmentResult   align.py:55-67   (same 8 fields, 0-based inclusive spans)
  AlignmentError    align.py:33-34
  encode            align.py:70-71
  smith_waterman    align.py:74-76   (raises AlignmentError on empty input)
  evaluate_pair     align.py:184-208 (identity / coverage filter)
  BatchCounters     align.py:211-220
  align_batch       align.py:223-246 (per-pair error isolation, input order)
  AlignEngine       align.py:299-347 (start/submit/result/close; lanes = GPUs)
Every alignment runs on the B200 through libpastis_sw.so (forward, reverse
and traceback kernels); there is no CPU fallback -- a missing library or GPU
raises.  Results are bit-identical to the reference's (tests/).
"""

import os
import threading
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field
from time import perf_counter
from collections.abc import Sequence
from typing import Optional

import numpy as np

from . import _native, blosum62
from .alphabet import INDEX, SIZE
from .batch import AlignmentError, PackedBatch, pack_pairs
from .edges import SimilarityEdge

__all__ = [
    "AlignParams",
    "AlignmentResult",
    "AlignmentError",
    "BatchCounters",
    "AlignEngine",
    "align_batch",
    "align_packed",
    "encode",
    "evaluate_pair",
    "smith_waterman",
]

# byte -> alphabet index (align.py:27-30); unknown bytes score as 'X'
_LUT = np.full(256, INDEX["X"], dtype=np.int64)
for _sym, _code in INDEX.items():
    _LUT[ord(_sym)] = _code


@dataclass(frozen=True)
class AlignParams:
    gap_open: int = 11
    gap_extend: int = 2
    matrix: np.ndarray = field(default_factory=lambda: blosum62.MATRIX)
    min_identity: float = 0.30
    min_coverage: float = 0.70

    def __post_init__(self):
        if not (self.gap_open >= self.gap_extend >= 0):
            raise ValueError("need gap_open >= gap_extend >= 0")
        mat = np.asarray(self.matrix)
        if mat.shape != (SIZE, SIZE):
            raise ValueError(f"substitution matrix must be {SIZE}x{SIZE}")
        if not np.array_equal(mat, mat.T):
            raise ValueError("substitution matrix must be symmetric")


try:  # drop-in interop: the reference's own result class when importable
    from pastislite.align import AlignmentResult  # type: ignore  # noqa: F401
except ImportError:  # pragma: no cover - the GPU box has no pastislite
    @dataclass(slots=True)
    class AlignmentResult:
        """Optimal local alignment; spans are 0-based inclusive residue offsets,
        all -1 for the empty (score 0) alignment (align.py:55-67)."""

        score: int
        i_begin: int
        i_end: int
        j_begin: int
        j_end: int
        matches: int
        aln_len: int
        cells: int


def encode(residues: str) -> np.ndarray:
    """Residue indices of `residues` (align.py:70-71)."""
    return _LUT[np.frombuffer(residues.encode("ascii"), dtype=np.uint8)]


_params_cache: dict = {}


def _native_params(params: AlignParams) -> "_native.SwParams":
    key = (params.gap_open, params.gap_extend, id(params.matrix))
    hit = _params_cache.get(key)
    if hit is not None and hit[0] is params.matrix:
        return hit[1]
    p = _native.make_params(params.gap_open, params.gap_extend,
                            np.asarray(params.matrix, dtype=np.int32))
    _params_cache[key] = (params.matrix, p)
    return p


def _device_ids(lanes: int) -> list:
    n = _native.device_count()
    if n <= 0:
        raise _native.NativeError("no CUDA device visible: the GPU aligner has no CPU fallback")
    env = os.environ.get("PASTIS_SW_DEVICES")
    ids = [int(x) for x in env.split(",")] if env else list(range(n))
    return ids[: max(1, min(lanes, len(ids)))]


def align_packed(batch: PackedBatch, params: AlignParams, devices=(0,)):
    """Align a packed batch on the GPU(s).  Returns (records, timings):
    records is a RESULT_DTYPE array in packed order."""
    p = _native_params(params)
    devices = list(devices)
    if len(batch.pairs) == 0:
        return np.empty(0, dtype=_native.RESULT_DTYPE), []
    if len(devices) == 1:
        out = _native.pinned_array(len(batch.pairs) * _native.RESULT_DTYPE.itemsize)
        rec, tm = _native.align_host(batch.arena, batch.pairs, p, device=devices[0],
                                     out=out.view(_native.RESULT_DTYPE))
        return rec, [tm]
    return _native.align_multi(batch.arena, batch.pairs, p, devices)


class ResultList(Sequence):
    """The `results` list of align_batch / AlignEngine (align.py:231-246), in
    input order: AlignmentResult or None per input pair.  The records stay a
    RESULT_DTYPE array; an AlignmentResult is built only when an element is
    read, so a batch of 1M pairs costs no Python objects until the caller
    touches them (`records`, `ok` and `cells` give vectorised access)."""

    __slots__ = ("records", "_ok", "_cells", "_n", "_la", "_lb", "_index")

    def __init__(self, batch: PackedBatch, rec: np.ndarray):
        n = self._n = batch.n_input
        # the pair lengths are kept (not the pinned table they came in):
        # ok / cells are derived on first use
        # contiguous copies, detached from a (pinned) pair table; no copy
        # when the caller already detached them (_Lengths)
        self._la = np.ascontiguousarray(batch.pairs["a_len"])
        self._lb = np.ascontiguousarray(batch.pairs["b_len"])
        self._index = None if len(batch.index) == n else batch.index
        if self._index is None:            # no packing errors: packed order == input order
            self.records = rec
        else:
            self.records = np.zeros(n, dtype=_native.RESULT_DTYPE)
            self.records[self._index] = rec
        self._ok = self._cells = None

    @property
    def ok(self) -> np.ndarray:
        if self._ok is None:
            ok = self.records["status"] == _native.STATUS_OK
            if self._index is not None:
                present = np.zeros(self._n, dtype=bool)
                present[self._index] = True
                ok &= present
            self._ok = ok
        return self._ok

    @property
    def cells(self) -> np.ndarray:
        if self._cells is None:
            c = self._la.astype(np.int64) * self._lb
            if self._index is not None:
                full = np.zeros(self._n, dtype=np.int64)
                full[self._index] = c
                c = full
            self._cells = c
        return self._cells

    def __len__(self) -> int:
        return self._n

    def _make(self, i: int):
        r = self.records[i]
        if r[7] != _native.STATUS_OK or (self._index is not None and not self.ok[i]):
            return None
        if self._index is None:
            c = int(self._la[i]) * int(self._lb[i])
        else:
            c = int(self.cells[i])
        return AlignmentResult(int(r[0]), int(r[1]), int(r[2]), int(r[3]), int(r[4]), int(r[5]),
                               int(r[6]), c)

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self._make(k) for k in range(*i.indices(len(self)))]
        n = len(self)
        if i < 0:
            i += n
        if not 0 <= i < n:
            raise IndexError("result index out of range")
        return self._make(i)

    def __iter__(self):
        rows = self.records.tolist()
        cells = self.cells.tolist()
        for ok, row, c in zip(self.ok.tolist(), rows, cells):
            yield AlignmentResult(row[0], row[1], row[2], row[3], row[4], row[5], row[6], c) \
                if ok else None

    def __eq__(self, other):
        try:
            return len(self) == len(other) and all(a == b for a, b in zip(self, other))
        except TypeError:
            return NotImplemented

    def __repr__(self) -> str:
        return f"ResultList({len(self)} results)"


def _to_results(batch: PackedBatch, rec: np.ndarray):
    """(results, errors, n_ok, cells): lazy results in input order, per-pair
    errors sorted by input index (packing errors + device status)."""
    results = ResultList(batch, rec)
    errors = list(batch.errors)
    bad = np.flatnonzero(rec["status"] != _native.STATUS_OK)
    for k in bad.tolist():
        idx = int(batch.index[k])
        if rec["status"][k] == _native.STATUS_EMPTY:
            errors.append((idx, AlignmentError("cannot align an empty sequence")))
        else:
            errors.append((idx, AssertionError("traceback lost at H state")))
    if len(bad):
        errors.sort(key=lambda e: e[0])
    if not len(bad) and len(batch.index) == batch.n_input:
        # exact uint64 multiply + sum: a float64 np.dot goes through the BLAS
        # thread pool, whose threads keep spinning after the call and halve
        # the speed of the next batch's packing threads (pack 25 -> 55 ms per
        # 1M pairs on the B200 box); numpy's integer dot is a slow scalar loop
        cells = int((results._la.astype(np.uint64) * results._lb).sum())
        return results, errors, batch.n_input, cells
    ok = results.ok
    return results, errors, int(ok.sum()), int(results.cells[ok].sum())


def smith_waterman(a: str, b: str, params: AlignParams) -> AlignmentResult:
    """Single-pair API (align.py:74-76) on the GPU."""
    if not a or not b:
        raise AlignmentError("cannot align an empty sequence")
    batch = pack_pairs([(a, b, None)])
    if batch.errors:
        raise batch.errors[0][1]
    rec, _ = align_packed(batch, params)
    results, errors, _, _ = _to_results(batch, rec)
    if errors:
        raise errors[0][1]
    return results[0]


def evaluate_pair(
    i: int,
    j: int,
    a: str,
    b: str,
    result: AlignmentResult,
    params: AlignParams,
) -> Optional[SimilarityEdge]:
    """Identity/coverage filter (align.py:184-208); returns an edge or None."""
    if i >= j:
        raise ValueError(f"pair not canonical: ({i}, {j})")
    if result.aln_len == 0:
        return None
    identity = result.matches / result.aln_len
    cov_a = (result.i_end - result.i_begin + 1) / len(a)
    cov_b = (result.j_end - result.j_begin + 1) / len(b)
    if identity >= params.min_identity and min(cov_a, cov_b) >= params.min_coverage:
        return SimilarityEdge(i, j, result.score, identity, cov_a, cov_b)
    return None


try:  # drop-in interop: the reference's counters class when importable
    from pastislite.align import BatchCounters  # type: ignore  # noqa: F401
except ImportError:  # pragma: no cover
    @dataclass
    class BatchCounters:
        alignments: int = 0
        cells: int = 0
        kernel_seconds: float = 0.0

        def merge(self, other: "BatchCounters") -> None:
            self.alignments += other.alignments
            self.cells += other.cells
            self.kernel_seconds += other.kernel_seconds


# Pairs per chunk of a large API batch, pipelined (pack chunk k+1 while the
# GPU aligns chunk k).  Off by default: on config 3 (1M pairs) four chunks
# cost more GPU time (smaller batches) and merging than the packing they hide
# (149 ms vs 133 ms per call on the box).
_CHUNK = 1 << 40


def _pack(pairs):
    """pack_pairs into recycled pinned buffers; returns (batch, buffers)."""
    pool = _native.pinned_pool()
    bufs = []

    def alloc(nbytes):
        b = pool.acquire(nbytes)
        bufs.append(b)
        return b.array

    try:
        return pack_pairs(pairs, alloc=alloc, table_alloc=alloc), bufs
    except BaseException:
        for b in bufs:
            b.release()
        raise


class _Lengths:
    """What _to_results needs of a batch once its pinned buffers are gone
    (the pair lengths as contiguous arrays, already copied out)."""

    def __init__(self, la, lb, index, n_input, errors):
        self.pairs = {"a_len": la, "b_len": lb}
        self.index, self.n_input, self.errors = index, n_input, errors


def _align(pairs: Sequence[tuple], params: AlignParams, devices, gpu_lock=None) -> tuple:
    """pack (host, C threads) -> align (GPU; under gpu_lock when given, so a
    second in-flight batch packs while this one runs) -> lazy results.

    A large batch is cut into chunks of _CHUNK pairs and pipelined: a helper
    thread packs chunk k+1 (the C extension releases the GIL while copying)
    while the GPU aligns chunk k; results, errors and counters come back as
    for one batch, in input order."""
    from contextlib import nullcontext
    lock = gpu_lock if gpu_lock is not None else nullcontext()
    n = len(pairs)
    t0 = perf_counter()
    bounds = [(0, n)] if n <= 2 * _CHUNK else [(c, min(n, c + _CHUNK)) for c in range(0, n, _CHUNK)]
    pieces, timings = [], []
    t_pack = t_align = 0.0
    ex = ThreadPoolExecutor(max_workers=1, thread_name_prefix="pastis-pack") if len(bounds) > 1 else None
    try:
        fut = None
        tp = perf_counter()
        nxt = _pack(pairs if len(bounds) == 1 else pairs[bounds[0][0]:bounds[0][1]])
        t_pack += perf_counter() - tp
        for k, (c0, c1) in enumerate(bounds):
            batch, bufs = nxt
            if k + 1 < len(bounds):
                d0, d1 = bounds[k + 1]
                fut = ex.submit(_pack, pairs[d0:d1])
            try:
                with lock:
                    ta = perf_counter()
                    rec, tms = align_packed(batch, params, devices)
                    t_align += perf_counter() - ta
                timings += tms
                # keep what the results need before the pinned buffers go back
                pieces.append((rec, np.array(batch.pairs["a_len"]), np.array(batch.pairs["b_len"]),
                               batch.index + c0, [(i + c0, e) for i, e in batch.errors]))
            finally:
                for b in bufs:
                    b.release()
            if fut is not None:
                tp = perf_counter()
                nxt = fut.result()
                t_pack += perf_counter() - tp    # only the part not hidden behind the GPU
                fut = None
    finally:
        if ex is not None:
            ex.shutdown(wait=True)
    t2 = perf_counter()
    if len(pieces) == 1:
        rec, la, lb, index, errs = pieces[0]
    else:
        rec = np.concatenate([p[0] for p in pieces])
        la = np.concatenate([p[1] for p in pieces])
        lb = np.concatenate([p[2] for p in pieces])
        index = np.concatenate([p[3] for p in pieces])
        errs = [e for p in pieces for e in p[4]]
    results, errors, n_ok, cell_sum = _to_results(_Lengths(la, lb, index, n, errs), rec)
    t3 = perf_counter()
    # kernel_seconds = forward fill time, the quantity align.py:103-122 times
    fwd = sum(t["forward_ms"] for t in timings) / 1e3
    counters = BatchCounters(alignments=n_ok, cells=cell_sum, kernel_seconds=fwd)
    phases = {"pack": t_pack, "align": t_align, "results": t3 - t2, "chunks": len(bounds),
              "total": t3 - t0}
    return results, errors, counters, timings, phases


def align_batch(pairs: Sequence[tuple], params: AlignParams) -> tuple:
    """Align (seq_a, seq_b, payload) tuples in order (align.py:223-246).

    Returns (results, errors, counters); a failing pair leaves None in its
    result slot and an (index, exception) entry instead of aborting."""
    results, errors, counters, _, _ = _align(pairs, params, _device_ids(1))
    return results, errors, counters


class _Pending:
    """Handle for a submitted batch (align.py:272-296)."""

    def __init__(self, future=None, resolved=None):
        self._future = future
        self._resolved = resolved

    def result(self) -> tuple:
        if self._resolved is None:
            self._resolved = self._future.result()
        return self._resolved


class AlignEngine:
    """GPU alignment engine with the reference's interface (align.py:299-347).

    `lanes` = number of GPUs a batch is sharded over (cell-balanced, capped at
    the visible device count).  With use_processes=True, submit() returns
    immediately and the batch runs on a host thread (the reference's async
    pool semantics, needed by pre-blocking, pipeline.py:209-212); two host
    threads, so the next batch's packing overlaps this batch's GPU work (the
    GPU phase is serialised by a lock; results come back per batch, in order
    of each handle's result())."""

    def __init__(self, params: AlignParams, lanes: int = 1, use_processes: bool = False):
        if lanes < 1:
            raise ValueError("need at least one alignment lane")
        self.params = params
        self.lanes = lanes
        self.use_processes = use_processes
        self._pool: Optional[ThreadPoolExecutor] = None
        self._devices: Optional[list] = None
        self._lock = threading.Lock()
        self.last_phases: dict = {}   # host pack / device align / results seconds, last batch

    def start(self) -> None:
        if self._devices is None:
            self._devices = _device_ids(self.lanes)
        if self.use_processes and self._pool is None:
            self._pool = ThreadPoolExecutor(max_workers=2, thread_name_prefix="pastis-gpu")

    def _run(self, pairs: list) -> tuple:
        t0 = perf_counter()
        results, errors, counters, timings, phases = _align(pairs, self.params, self._devices,
                                                            gpu_lock=self._lock)
        self.last_phases = phases
        wall = perf_counter() - t0
        if len(timings) <= 1:
            lanes = [(self._devices[0], counters.kernel_seconds, wall)]
        else:
            lanes = [(dev, t["forward_ms"] / 1e3, t["total_ms"] / 1e3)
                     for dev, t in zip(self._devices, timings)]
        return results, errors, counters, lanes

    def submit(self, pairs: list) -> _Pending:
        self.start()
        if not self.use_processes:
            return _Pending(resolved=self._run(pairs))
        return _Pending(future=self._pool.submit(self._run, pairs))

    def close(self) -> None:
        if self._pool is not None:
            self._pool.shutdown(wait=True)
            self._pool = None

    def __enter__(self):
        self.start()
        return self

    def __exit__(self, *exc):
        self.close()

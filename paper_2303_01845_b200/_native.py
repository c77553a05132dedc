"""ctypes binding of libpastis_sw.so (C ABI: include/pastis_sw.h).

There is no CPU fallback: if the library or a GPU is missing, every compute
entry point raises.  The library is built in-tree by __graft_entry__.build()
(or `python -m paper_2303_01845_b200.build`).
"""

import ctypes
import os
import threading
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libpastis_sw.so")

# numpy mirrors of the C structs (packed exactly like the C layout)
PAIR_DTYPE = np.dtype([("a_off", "<u8"), ("b_off", "<u8"), ("a_len", "<u4"), ("b_len", "<u4")])
RESULT_DTYPE = np.dtype(
    [
        ("score", "<i4"),
        ("i_begin", "<i4"),
        ("i_end", "<i4"),
        ("j_begin", "<i4"),
        ("j_end", "<i4"),
        ("matches", "<i4"),
        ("aln_len", "<i4"),
        ("status", "<i4"),
    ]
)
assert PAIR_DTYPE.itemsize == 24 and RESULT_DTYPE.itemsize == 32

SW_OK, SW_EINVAL, SW_ECUDA, SW_EINTERNAL, SW_EFORMAT, SW_ERANGE = 0, -1, -2, -3, -4, -5
STATUS_OK, STATUS_EMPTY, STATUS_INTERNAL, STATUS_INVALID = 0, 1, 2, 3  # SW_STATUS_* (include/pastis_sw.h)

# every symbol include/pastis_sw.h declares
EXPORTED_SYMBOLS = (
    "sw_get_device_count",
    "sw_last_error",
    "sw_abi_version",
    "sw_align_batch",
    "sw_align_batch_device",
    "sw_align_batch_multi",
    "sw_partition_pairs",
    "sw_align_shard",
    "sw_shard_ranges",
    "sw_release",
    "sw_host_alloc",
    "sw_host_free",
    "sw_fasta_parse",
    "sw_kmer_candidates",
)

# candidate discovery (sw_kmer_candidates)
CANDIDATE_DTYPE = np.dtype([("i", "<u4"), ("j", "<u4"), ("count", "<u4"), ("pad", "<u4")])
assert CANDIDATE_DTYPE.itemsize == 16

# FASTA ingest (sw_fasta_parse)
FASTA_REC_DTYPE = np.dtype([("off", "<u8"), ("hdr_off", "<u8"), ("len", "<u4"), ("hdr_len", "<u4")])
assert FASTA_REC_DTYPE.itemsize == 24
FASTA_NONASCII, FASTA_DATA_BEFORE_HEADER, FASTA_EMPTY_HEADER, FASTA_EMPTY_SEQ, FASTA_NO_RECORDS = 1, 2, 3, 4, 5


class SwParams(ctypes.Structure):
    _fields_ = [("gap_open", ctypes.c_int32), ("gap_extend", ctypes.c_int32),
                ("matrix", ctypes.c_int32 * 625)]


class SwTiming(ctypes.Structure):
    _fields_ = [
        ("forward_ms", ctypes.c_double),
        ("reverse_ms", ctypes.c_double),
        ("traceback_ms", ctypes.c_double),
        ("kernel_ms", ctypes.c_double),
        ("h2d_ms", ctypes.c_double),
        ("d2h_ms", ctypes.c_double),
        ("total_ms", ctypes.c_double),
        ("cells", ctypes.c_uint64),
        ("h2d_bytes", ctypes.c_uint64),
        ("d2h_bytes", ctypes.c_uint64),
        ("launches", ctypes.c_uint32),
        ("wide_pairs", ctypes.c_uint32),
        ("box_cells", ctypes.c_uint64),
        ("rev_cells", ctypes.c_uint64),
        ("host_plan_ms", ctypes.c_double),
        ("host_setup_ms", ctypes.c_double),
        ("tile_tb_ms", ctypes.c_double),
        ("fwd_tail_ms", ctypes.c_double),
    ]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


class SwFastaInfo(ctypes.Structure):
    _fields_ = [("n_recs", ctypes.c_uint64), ("arena_bytes", ctypes.c_uint64),
                ("header_bytes", ctypes.c_uint64), ("n_mapped", ctypes.c_uint64),
                ("error", ctypes.c_int32), ("error_hdr_len", ctypes.c_uint32),
                ("error_hdr_off", ctypes.c_uint64)]


class SwKmerStats(ctypes.Structure):
    _fields_ = [("positions", ctypes.c_uint64), ("distinct", ctypes.c_uint64),
                ("buckets", ctypes.c_uint64), ("emitted", ctypes.c_uint64),
                ("discovered", ctypes.c_uint64), ("performed", ctypes.c_uint64),
                ("flops", ctypes.c_uint64), ("short_seqs", ctypes.c_uint32),
                ("pad", ctypes.c_uint32), ("device_ms", ctypes.c_double)]


class NativeError(RuntimeError):
    pass


_lib = None
_lock = threading.Lock()


def load(path: Optional[str] = None) -> ctypes.CDLL:
    """Load (once) and type the library; raises if it is not built."""
    global _lib
    with _lock:
        if _lib is not None and path is None:
            return _lib
        p = path or os.environ.get("PASTIS_SW_LIB") or LIB_PATH
        if not os.path.exists(p):
            raise NativeError(
                f"{p} not found: build the CUDA extension first "
                "(python -c 'import __graft_entry__ as g; g.build()')"
            )
        lib = ctypes.CDLL(p)
        vp, u64, i32 = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_int
        lib.sw_get_device_count.restype = i32
        lib.sw_get_device_count.argtypes = []
        lib.sw_last_error.restype = ctypes.c_char_p
        lib.sw_last_error.argtypes = []
        lib.sw_abi_version.restype = i32
        lib.sw_align_batch.restype = i32
        lib.sw_align_batch.argtypes = [i32, vp, u64, vp, u64, ctypes.POINTER(SwParams), vp,
                                       ctypes.POINTER(SwTiming)]
        lib.sw_align_batch_device.restype = i32
        lib.sw_align_batch_device.argtypes = [i32, vp, u64, vp, u64, ctypes.POINTER(SwParams),
                                              vp, vp, ctypes.POINTER(SwTiming)]
        lib.sw_align_batch_multi.restype = i32
        lib.sw_align_batch_multi.argtypes = [i32, vp, vp, u64, vp, u64,
                                             ctypes.POINTER(SwParams), vp, vp]
        lib.sw_align_shard.restype = i32
        lib.sw_align_shard.argtypes = [i32, vp, u64, vp, u64, i32, i32, ctypes.POINTER(SwParams),
                                       vp, vp, vp, ctypes.POINTER(SwTiming)]
        lib.sw_shard_ranges.restype = i32
        lib.sw_shard_ranges.argtypes = [vp, u64, i32, vp]
        lib.sw_partition_pairs.restype = i32
        lib.sw_partition_pairs.argtypes = [vp, u64, i32, vp, vp]
        lib.sw_release.restype = None
        lib.sw_release.argtypes = [i32]
        lib.sw_host_alloc.restype = vp
        lib.sw_host_alloc.argtypes = [u64]
        lib.sw_host_free.restype = None
        lib.sw_host_free.argtypes = [vp]
        lib.sw_kmer_candidates.restype = i32
        lib.sw_kmer_candidates.argtypes = [i32, vp, u64, vp, vp, ctypes.c_uint32, i32,
                                           ctypes.c_uint32, vp, u64, ctypes.POINTER(SwKmerStats)]
        lib.sw_fasta_parse.restype = i32
        lib.sw_fasta_parse.argtypes = [vp, u64, vp, vp, vp, u64, ctypes.POINTER(SwFastaInfo)]
        if path is None:
            _lib = lib
        return lib


def _check(rc: int) -> None:
    if rc != SW_OK:
        msg = load().sw_last_error().decode("utf-8", "replace")
        if rc == SW_EINVAL:
            raise ValueError(msg)
        raise NativeError(f"libpastis_sw error {rc}: {msg}")


def device_count() -> int:
    return int(load().sw_get_device_count())


def make_params(gap_open: int, gap_extend: int, matrix) -> SwParams:
    m = np.ascontiguousarray(np.asarray(matrix, dtype=np.int32)).reshape(-1)
    if m.size != 625:
        raise ValueError("substitution matrix must be 25x25")
    p = SwParams()
    p.gap_open = int(gap_open)
    p.gap_extend = int(gap_extend)
    ctypes.memmove(p.matrix, m.ctypes.data, 625 * 4)
    return p


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data if a.size else 0


def align_host(arena: np.ndarray, pairs: np.ndarray, params: SwParams, device: int = 0,
               out: Optional[np.ndarray] = None):
    """sw_align_batch: host arena + pair table -> (results, timing dict)."""
    lib = load()
    arena = np.ascontiguousarray(arena, dtype=np.uint8)
    pairs = np.ascontiguousarray(pairs, dtype=PAIR_DTYPE)
    if out is None:
        out = np.empty(len(pairs), dtype=RESULT_DTYPE)
    tm = SwTiming()
    _check(lib.sw_align_batch(device, _ptr(arena), arena.size, _ptr(pairs), len(pairs),
                              ctypes.byref(params), _ptr(out), ctypes.byref(tm)))
    return out, tm.as_dict()


def align_multi(arena: np.ndarray, pairs: np.ndarray, params: SwParams, devices):
    """sw_align_batch_multi: cell-balanced shard over `devices`."""
    lib = load()
    arena = np.ascontiguousarray(arena, dtype=np.uint8)
    pairs = np.ascontiguousarray(pairs, dtype=PAIR_DTYPE)
    devs = np.asarray(list(devices), dtype=np.int32)
    out = np.empty(len(pairs), dtype=RESULT_DTYPE)
    tms = (SwTiming * len(devs))()
    _check(lib.sw_align_batch_multi(len(devs), devs.ctypes.data, _ptr(arena), arena.size,
                                    _ptr(pairs), len(pairs), ctypes.byref(params), _ptr(out),
                                    ctypes.cast(tms, ctypes.c_void_p)))
    return out, [t.as_dict() for t in tms]


def align_device(d_arena: int, arena_bytes: int, d_pairs: int, n_pairs: int, params: SwParams,
                 d_out: int, device: int = 0, stream: int = 0) -> dict:
    """sw_align_batch_device on raw device pointers (e.g. torch tensors)."""
    lib = load()
    tm = SwTiming()
    _check(lib.sw_align_batch_device(device, d_arena, arena_bytes, d_pairs, n_pairs,
                                     ctypes.byref(params), d_out, stream or None,
                                     ctypes.byref(tm)))
    return tm.as_dict()


def shard_ranges(pairs, n_shards: int, n_pairs: Optional[int] = None) -> np.ndarray:
    """sw_shard_ranges: bounds[0..n_shards] of the cell-balanced contiguous
    plan.  `pairs`: a PAIR_DTYPE array, or a device pointer with n_pairs."""
    b = np.zeros(n_shards + 1, dtype=np.uint64)
    if isinstance(pairs, np.ndarray):
        pairs = np.ascontiguousarray(pairs, dtype=PAIR_DTYPE)
        ptr, n = _ptr(pairs), len(pairs)
    else:
        ptr, n = int(pairs), int(n_pairs)
    _check(load().sw_shard_ranges(ptr, n, n_shards, b.ctypes.data))
    return b


def align_shard(arena_ptr: int, arena_bytes: int, pairs_ptr: int, n_pairs: int, shard: int,
                n_shards: int, params: SwParams, d_out: int, device: int = 0,
                stream: int = 0):
    """sw_align_shard: shard `shard` of a batch (arena and pairs both device or
    both host pointers) into the DEVICE buffer d_out.  Returns (timing dict,
    (first, end)) -- d_out holds the results of pairs first .. end-1."""
    tm = SwTiming()
    rng = np.zeros(2, dtype=np.uint64)
    _check(load().sw_align_shard(device, arena_ptr, arena_bytes, pairs_ptr, n_pairs, shard,
                                 n_shards, ctypes.byref(params), d_out, rng.ctypes.data,
                                 stream or None, ctypes.byref(tm)))
    return tm.as_dict(), (int(rng[0]), int(rng[1]))


def partition(pairs: np.ndarray, n_shards: int):
    """sw_partition_pairs: the cell-balanced plan as a shard id per pair."""
    lib = load()
    pairs = np.ascontiguousarray(pairs, dtype=PAIR_DTYPE)
    shard = np.empty(len(pairs), dtype=np.int32)
    load_ = np.empty(n_shards, dtype=np.uint64)
    _check(lib.sw_partition_pairs(_ptr(pairs), len(pairs), n_shards, _ptr(shard),
                                  load_.ctypes.data))
    return shard, load_


def fasta_parse(text: bytes):
    """sw_fasta_parse on a whole FASTA text (host only, no GPU needed).

    Returns (arena uint8[arena_bytes], headers bytes, recs FASTA_REC_DTYPE[n],
    info dict); info["error"] != 0 reports the reference's first FastaError
    (or FASTA_NONASCII) -- the caller raises it."""
    lib = load()
    buf = np.frombuffer(text, dtype=np.uint8) if len(text) else np.zeros(1, np.uint8)
    n = len(text)
    arena = np.empty(max(n, 1), dtype=np.uint8)
    headers = np.empty(max(n, 1), dtype=np.uint8)
    cap = int(np.count_nonzero(buf[:n] == ord(">"))) + 1
    recs = np.empty(cap, dtype=FASTA_REC_DTYPE)
    info = SwFastaInfo()
    rc = lib.sw_fasta_parse(_ptr(buf), n, _ptr(arena), _ptr(headers), _ptr(recs), cap,
                            ctypes.byref(info))
    if rc not in (SW_OK, SW_EFORMAT):
        _check(rc)
    d = {name: getattr(info, name) for name, _ in SwFastaInfo._fields_}
    return (arena[: info.arena_bytes], headers[: info.header_bytes].tobytes(),
            recs[: info.n_recs].copy(), d)


def kmer_candidates(arena: np.ndarray, offsets: np.ndarray, lengths: np.ndarray, k: int,
                    min_shared: int, device: int = 0):
    """sw_kmer_candidates: (candidates CANDIDATE_DTYPE sorted by (i, j), stats dict)."""
    lib = load()
    arena = np.ascontiguousarray(arena, dtype=np.uint8)
    offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
    lengths = np.ascontiguousarray(lengths, dtype=np.uint32)
    cap = max(1024, 4 * len(lengths))
    while True:
        out = np.empty(cap, dtype=CANDIDATE_DTYPE)
        st = SwKmerStats()
        rc = lib.sw_kmer_candidates(device, _ptr(arena), arena.size, _ptr(offsets), _ptr(lengths),
                                    len(lengths), k, min_shared, _ptr(out), cap, ctypes.byref(st))
        if rc == SW_ERANGE:
            cap = int(st.performed)
            continue
        _check(rc)
        d = {name: getattr(st, name) for name, _ in SwKmerStats._fields_ if name != "pad"}
        return out[: st.performed], d


class PinnedPool:
    """Recycled pinned (page-locked, cudaHostAllocPortable) host buffers.

    cudaHostAlloc costs far more than the copies it speeds up, so buffers are
    kept and reused: acquire(nbytes) hands out the smallest free buffer that
    fits (or allocates one of the next power-of-two size), release() returns
    it.  Pinned memory lets the upload run at full PCIe speed and lets every
    GPU read the arena directly (zero-copy) on the multi-GPU path.  When no
    CUDA driver is present (CPU tests) it hands out plain numpy memory."""

    def __init__(self, max_free: int = 8, max_free_bytes: int = 3 << 30):
        # up to 8 buffers / 3 GiB kept free: two batches in flight through the
        # engine (arena, table and records each) without a cudaHostAlloc per call
        self._free: list = []
        self._lock = threading.Lock()
        self._max_free = max_free
        self._max_free_bytes = max_free_bytes

    def acquire(self, nbytes: int):
        nbytes = max(int(nbytes), 1)
        with self._lock:
            fits = [b for b in self._free if b[1] >= nbytes]
            if fits:
                best = min(fits, key=lambda b: b[1])
                self._free.remove(best)
                ptr, cap = best
                return PinnedBuffer(self, ptr, cap, nbytes)
        cap = 1 << max(20, (nbytes - 1).bit_length())
        ptr = load().sw_host_alloc(cap)
        if not ptr:
            return PinnedBuffer(None, None, nbytes, nbytes)    # unpinned fallback memory
        return PinnedBuffer(self, ptr, cap, nbytes)

    def _release(self, ptr, cap):
        with self._lock:
            self._free.append((ptr, cap))
            while len(self._free) > self._max_free:
                p, _ = min(self._free, key=lambda b: b[1])
                self._free.remove((p, _))
                load().sw_host_free(p)
            while len(self._free) > 1 and sum(c for _, c in self._free) > self._max_free_bytes:
                p, _ = max(self._free, key=lambda b: b[1])
                self._free.remove((p, _))
                load().sw_host_free(p)


class PinnedBuffer:
    """A pinned host buffer lent by PinnedPool; `array` is a uint8 view of
    the requested size.  release() (or garbage collection) returns it."""

    def __init__(self, pool, ptr, cap, nbytes):
        self.pool, self.ptr, self.cap = pool, ptr, cap
        if ptr is None:
            self.array = np.empty(nbytes, dtype=np.uint8)
        else:
            self.array = np.ctypeslib.as_array((ctypes.c_uint8 * nbytes).from_address(ptr))
        self.pinned = ptr is not None

    def release(self):
        if self.pool is not None and self.ptr is not None:
            pool, ptr, cap = self.pool, self.ptr, self.cap
            self.pool = self.ptr = None
            self.array = None
            pool._release(ptr, cap)

    def __del__(self):
        try:
            self.release()
        except Exception:  # noqa: BLE001 - interpreter shutdown
            pass


class _Lease:
    """Returns a PinnedBuffer to its pool when the last array viewing it dies."""

    def __init__(self, buf):
        self.buf = buf

    def __del__(self):
        try:
            self.buf.release()
        except Exception:  # noqa: BLE001 - interpreter shutdown
            pass


def pinned_array(nbytes: int) -> np.ndarray:
    """A uint8 array in pinned memory from the pool that goes back to the
    pool when the array (and every view of it) is garbage -- for results the
    caller keeps (device-to-host copies into pinned memory run at full PCIe
    speed and touch no fresh pages)."""
    b = pinned_pool().acquire(nbytes)
    if not b.pinned:
        return b.array
    ca = (ctypes.c_uint8 * max(int(nbytes), 1)).from_address(b.ptr)
    ca._lease = _Lease(b)
    return np.ctypeslib.as_array(ca)


_POOL = None


def pinned_pool() -> PinnedPool:
    global _POOL
    if _POOL is None:
        _POOL = PinnedPool()
    return _POOL

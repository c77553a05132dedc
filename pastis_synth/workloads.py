"""Seeded synthetic workloads of BASELINE.json's configs.

config 2: n pairs of fixed-length 300x300 proteins; a uniform over the 20
          standard residues (synth.py:12 of the reference); b is a homolog of
          a half of the time (30% substitutions + ~8% indels, trimmed/padded
          back to the fixed length) and an independent draw otherwise.
config 3: n pairs, len(a) = clip(round(LogNormal(5.5, 0.75)), 30, 2000);
          b a length-correlated homolog (len*U(0.7,1.3)) half of the time,
          else an independent draw of the same distribution.
config 5: n pairs with both lengths U[2000, 35000] (independent).
All sequences are returned as ASCII bytes objects.
"""

import numpy as np

STANDARD = np.frombuffer(b"ARNDCQEGHILKMFPSTWYV", dtype=np.uint8)


def _random_seq(rng, n: int) -> np.ndarray:
    return STANDARD[rng.integers(0, len(STANDARD), size=n)]


def _homolog(rng, a: np.ndarray, sub_rate: float = 0.30, indel_rate: float = 0.08) -> np.ndarray:
    out = a.copy()
    mask = rng.random(len(out)) < sub_rate
    if mask.any():
        repl = STANDARD[rng.integers(0, len(STANDARD), size=int(mask.sum()))]
        out[mask] = repl
    pieces = []
    pos = 0
    n = len(out)
    events = np.flatnonzero(rng.random(n) < indel_rate)
    for e in events:
        pieces.append(out[pos:e])
        if rng.random() < 0.5:  # deletion of 1..3 residues
            pos = min(n, e + int(rng.integers(1, 4)))
        else:  # insertion of 1..3 random residues
            pieces.append(_random_seq(rng, int(rng.integers(1, 4))))
            pos = e
    pieces.append(out[pos:])
    return np.concatenate(pieces) if pieces else out


def _fit(rng, s: np.ndarray, length: int) -> np.ndarray:
    if len(s) >= length:
        return s[:length]
    return np.concatenate([s, _random_seq(rng, length - len(s))])


def config2(n: int, seed: int = 2303, length: int = 300):
    rng = np.random.default_rng(seed)
    seqs_a, seqs_b = [], []
    for _ in range(n):
        a = _random_seq(rng, length)
        if rng.random() < 0.5:
            b = _fit(rng, _homolog(rng, a), length)
        else:
            b = _random_seq(rng, length)
        seqs_a.append(a.tobytes())
        seqs_b.append(b.tobytes())
    return seqs_a, seqs_b


def _lognormal_len(rng, size):
    return np.clip(np.rint(rng.lognormal(5.5, 0.75, size=size)), 30, 2000).astype(np.int64)


def config3(n: int, seed: int = 2303):
    rng = np.random.default_rng(seed)
    la = _lognormal_len(rng, n)
    seqs_a, seqs_b = [], []
    for k in range(n):
        a = _random_seq(rng, int(la[k]))
        if rng.random() < 0.5:
            lb = int(np.clip(round(la[k] * rng.uniform(0.7, 1.3)), 30, 2000))
            b = _fit(rng, _homolog(rng, a), lb)
        else:
            b = _random_seq(rng, int(_lognormal_len(rng, 1)[0]))
        seqs_a.append(a.tobytes())
        seqs_b.append(b.tobytes())
    return seqs_a, seqs_b


def config5(n: int, seed: int = 2303, lo: int = 2000, hi: int = 35000):
    rng = np.random.default_rng(seed)
    seqs_a, seqs_b = [], []
    for _ in range(n):
        seqs_a.append(_random_seq(rng, int(rng.integers(lo, hi + 1))).tobytes())
        seqs_b.append(_random_seq(rng, int(rng.integers(lo, hi + 1))).tobytes())
    return seqs_a, seqs_b


def _split(buf: np.ndarray, lens: np.ndarray) -> list:
    raw = buf.tobytes()
    ends = np.cumsum(lens)
    starts = ends - lens
    return [raw[s:e] for s, e in zip(starts.tolist(), ends.tolist())]


def _homolog_bulk(rng, a: np.ndarray, la: np.ndarray, sub_rate: float = 0.30,
                  indel_rate: float = 0.08) -> tuple:
    """Vectorised homolog of every sequence in the concatenation `a` (lengths
    `la`): substitutions at `sub_rate`; at each position an indel event with
    probability `indel_rate`, half deletions of 1..3 residues starting there,
    half insertions of 1..3 random residues before it (the model of _homolog,
    without its sequential quirks).  Returns (concatenation, lengths)."""
    t = len(a)
    out = a.copy()
    mask = rng.random(t) < sub_rate
    out[mask] = STANDARD[rng.integers(0, len(STANDARD), size=int(mask.sum()))]
    r = rng.random(t)
    ends = np.cumsum(la)
    ev = np.flatnonzero(r < indel_rate / 2)          # deletions stay inside their sequence
    del_end = np.zeros(t, np.int64)
    del_end[ev] = np.minimum(ev + rng.integers(1, 4, size=len(ev)),
                             ends[np.searchsorted(ends, ev, side="right")])
    keep = np.maximum.accumulate(del_end) <= np.arange(t)
    ev = np.flatnonzero((r >= indel_rate / 2) & (r < indel_rate))
    emit = keep.astype(np.int64)
    emit[ev] += rng.integers(1, 4, size=len(ev))    # insertions before the residue
    last = np.cumsum(emit)
    res = STANDARD[rng.integers(0, len(STANDARD), size=int(last[-1]) if t else 0)]
    res[last[keep] - 1] = out[keep]                  # a kept residue ends its emitted run
    lens = np.add.reduceat(emit, ends - la) if t else np.zeros(len(la), np.int64)
    return res, lens.astype(np.int64)


def _fit_bulk(rng, s: np.ndarray, ls: np.ndarray, target: np.ndarray) -> np.ndarray:
    """Truncate / pad (random residues) each sequence of the concatenation."""
    starts = np.cumsum(ls) - ls
    keep = np.minimum(ls, target)
    total = int(target.sum())
    out = STANDARD[rng.integers(0, len(STANDARD), size=total)]
    dst0 = np.cumsum(target) - target
    pos = np.arange(int(keep.sum())) - np.repeat(np.cumsum(keep) - keep, keep)
    out[np.repeat(dst0, keep) + pos] = s[np.repeat(starts, keep) + pos]
    return out


def config3_bulk(n: int, seed: int = 2303, chunk: int = 65536):
    """Config 3 at bench scale (1M pairs in seconds): the distribution of
    config3() -- len(a) ~ clip(LogNormal(5.5, 0.75), 30, 2000); half the b's
    length-correlated homologs (len*U(0.7,1.3)), half independent draws --
    generated with whole-chunk numpy operations (a different random stream)."""
    seqs_a, seqs_b = [], []
    for c0 in range(0, n, chunk):
        a, b = _config3_chunk(min(chunk, n - c0), seed * 1_000_003 + c0)
        seqs_a += a
        seqs_b += b
    return seqs_a, seqs_b


def _config3_chunk(n: int, seed: int):
    rng = np.random.default_rng(seed)
    la = _lognormal_len(rng, n)
    a = _random_seq(rng, int(la.sum()))
    hom = rng.random(n) < 0.5
    lb = np.where(hom, np.clip(np.rint(la * rng.uniform(0.7, 1.3, size=n)), 30, 2000).astype(np.int64),
                  _lognormal_len(rng, n))
    # homolog b's: mutate the a's of the homolog pairs, then fit to lb
    a_starts = np.cumsum(la) - la
    h_idx = np.flatnonzero(hom)
    h_la = la[h_idx]
    h_pos = np.arange(int(h_la.sum())) - np.repeat(np.cumsum(h_la) - h_la, h_la)
    h_src = a[np.repeat(a_starts[h_idx], h_la) + h_pos]
    h_mut, h_len = _homolog_bulk(rng, h_src, h_la)
    h_b = _fit_bulk(rng, h_mut, h_len, lb[h_idx])
    r_idx = np.flatnonzero(~hom)
    r_b = _random_seq(rng, int(lb[r_idx].sum()))
    b_h = _split(h_b, lb[h_idx])
    b_r = _split(r_b, lb[r_idx])
    seqs_b = [None] * n
    for k, s in zip(h_idx.tolist(), b_h):
        seqs_b[k] = s
    for k, s in zip(r_idx.tolist(), b_r):
        seqs_b[k] = s
    return _split(a, la), seqs_b


# ---------------------------------------------------------------------------
# Packed generators (gen.c): the same models, written straight into a byte
# arena + sw_pair_t table by multi-threaded C -- ~50x faster than the numpy
# generators above (different random streams; the tests check the GPU against
# the CPU oracle on whatever these produce, and the bench's full-size parity
# test uses exactly the batch the bench times).
# ---------------------------------------------------------------------------
import ctypes as _ct
import os as _os

_HERE = _os.path.dirname(_os.path.abspath(__file__))
_LIB = None
PAIR_DTYPE = np.dtype([("a_off", "<u8"), ("b_off", "<u8"), ("a_len", "<u4"), ("b_len", "<u4")])


class _Cfg(_ct.Structure):
    _fields_ = [("kind", _ct.c_int), ("seed", _ct.c_uint64), ("length", _ct.c_uint32),
                ("lo", _ct.c_uint32), ("hi", _ct.c_uint32), ("hom_frac", _ct.c_double),
                ("sub_rate", _ct.c_double), ("indel_rate", _ct.c_double)]


def _lib():
    global _LIB
    if _LIB is None:
        path = _os.path.join(_HERE, "libsynth.so")
        if not _os.path.exists(path) or (_os.path.getmtime(path) <
                                         _os.path.getmtime(_os.path.join(_HERE, "gen.c"))):
            import subprocess
            subprocess.run(["make", "-s", "-B", "-C", _HERE, "libsynth.so"], check=True)
        lib = _ct.CDLL(path)
        vp, u64 = _ct.c_void_p, _ct.c_uint64
        lib.syn_lengths.argtypes = [_ct.POINTER(_Cfg), u64, vp, vp, vp]
        lib.syn_lengths.restype = _ct.c_int
        lib.syn_fill.argtypes = [_ct.POINTER(_Cfg), u64, vp, vp, vp, _ct.c_int]
        lib.syn_fill.restype = _ct.c_int
        _LIB = lib
    return _LIB


def packed(kind: int, n: int, seed: int, *, length: int = 300, lo: int = 2000, hi: int = 35000,
           hom_frac: float = 0.5, sub_rate: float = 0.30, indel_rate: float = 0.08,
           alloc=None, threads: int = 0):
    """(arena uint8, table PAIR_DTYPE) of `n` pairs of config `kind` (2, 3, 5);
    pair k's a and b sit back to back in the arena.  `alloc(nbytes)` may
    supply the arena buffer (e.g. pinned host memory)."""
    lib = _lib()
    c = _Cfg(kind, seed, length, lo, hi, hom_frac, sub_rate, indel_rate)
    la = np.empty(n, np.uint32)
    lb = np.empty(n, np.uint32)
    hom = np.empty(n, np.uint8)
    if lib.syn_lengths(_ct.byref(c), n, la.ctypes.data, lb.ctypes.data, hom.ctypes.data):
        raise ValueError(f"unknown workload kind {kind}")
    tot = la.astype(np.uint64) + lb
    ends = np.cumsum(tot, dtype=np.uint64)
    table = np.empty(n, PAIR_DTYPE)
    table["a_off"] = ends - tot
    table["b_off"] = table["a_off"] + la
    table["a_len"] = la
    table["b_len"] = lb
    nbytes = int(ends[-1]) if n else 0
    arena = alloc(max(nbytes, 1)) if alloc is not None else np.empty(max(nbytes, 1), np.uint8)
    lib.syn_fill(_ct.byref(c), n, table.ctypes.data, hom.ctypes.data, arena.ctypes.data,
                 threads or len(_os.sched_getaffinity(0)))
    return arena[: max(nbytes, 1)], table


def config2_packed(n: int, seed: int = 2303, length: int = 300, **kw):
    """Config 2: n pairs of length x length, half homologs."""
    return packed(2, n, seed, length=length, **kw)


def config3_packed(n: int, seed: int = 2303, **kw):
    """Config 3: 1M-pair-scale skewed lengths 30-2000 (lognormal), half homologs."""
    return packed(3, n, seed, **kw)


def config5_packed(n: int, seed: int = 2303, lo: int = 2000, hi: int = 35000, hom_frac: float = 0.0,
                   **kw):
    """Config 5: lengths U[lo, hi]; hom_frac of the b's homologs of their a
    (0 = the BASELINE config: independent pairs)."""
    return packed(5, n, seed, lo=lo, hi=hi, hom_frac=hom_frac, **kw)

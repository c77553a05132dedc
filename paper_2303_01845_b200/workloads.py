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

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

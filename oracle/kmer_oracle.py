"""CPU restatement of the reference's candidate discovery -- TEST
INFRASTRUCTURE ONLY (tests/ and bench.py's CPU leg may use it; the product
path is sw_kmer_candidates on the GPU).

Follows pastislite.kmer.build_kmer_matrix (kmer.py:56-90: one entry per
distinct k-mer per sequence, base-25 codes, first residue most significant,
sequences shorter than k contribute nothing) and the overlap semiring product
A*A^T (kmer.py:93-126): the shared count of (i, j) is the number of distinct
codes both sequences contain.  Pinned to tests/golden/kmer_candidates.json
(generated from the reference by tests/golden/make_kmer_golden.py).
"""

import numpy as np

ALPHABET = "ARNDCQEGHILKMFPSTWYVBZXU*"
_LUT = np.full(256, 22, dtype=np.int64)          # unknown -> 'X' (align.py:27-30)
for _i, _ch in enumerate(ALPHABET):
    _LUT[ord(_ch)] = _i


def kmer_sets(seqs, k: int):
    """(code, seq) arrays of the distinct k-mers of every sequence."""
    codes, owners = [], []
    powers = 25 ** np.arange(k - 1, -1, -1, dtype=np.int64)
    for s, seq in enumerate(seqs):
        b = np.frombuffer(seq.encode("ascii") if isinstance(seq, str) else bytes(seq), dtype=np.uint8)
        if len(b) < k:
            continue
        idx = _LUT[b]
        win = np.lib.stride_tricks.sliding_window_view(idx, k)
        u = np.unique(win @ powers)
        codes.append(u)
        owners.append(np.full(len(u), s, dtype=np.int64))
    if not codes:
        return np.zeros(0, np.int64), np.zeros(0, np.int64)
    return np.concatenate(codes), np.concatenate(owners)


def shared_counts(seqs, k: int):
    """All unordered pairs i < j sharing >= 1 distinct k-mer, with the count,
    sorted by (i, j): arrays (i, j, count)."""
    code, owner = kmer_sets(seqs, k)
    order = np.lexsort((owner, code))
    code, owner = code[order], owner[order]
    bounds = np.flatnonzero(np.diff(code)) + 1
    starts = np.concatenate(([0], bounds))
    ends = np.concatenate((bounds, [len(code)]))
    ii, jj = [], []
    for a, b in zip(starts, ends):
        if b - a < 2:
            continue
        m = owner[a:b]
        x, y = np.triu_indices(len(m), 1)
        ii.append(m[x])
        jj.append(m[y])
    if not ii:
        z = np.zeros(0, np.int64)
        return z, z, z
    key = np.concatenate(ii) * (1 << 32) + np.concatenate(jj)
    u, cnt = np.unique(key, return_counts=True)
    return u >> 32, u & 0xFFFFFFFF, cnt

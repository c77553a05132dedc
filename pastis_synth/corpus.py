"""Seeded synthetic protein corpora: BASELINE configs 1 and 4 as FASTA input.

Restates pastislite.synth.synthetic_records (/root/reference/pkg/src/
pastislite/synth.py:15-61) -- same Python `random.Random(seed)` call
sequence, so the records are identical: random base sequences of length
U[min_len, max_len] over the 20 standard residues; with probability
family_fraction a base is followed by family_size - 1 variants, each with
per-residue substitutions at mutation_rate (never to the same residue) and,
with probability fragment_fraction, cut to a random fragment of 40-90 % of
its length (at least min_len).  Headers are "s%05d".  `write_fasta` mirrors
seqio.write_fasta (seqio.py:95-98).

  config 1: synthetic_records(1000, seed=0)
  config 4: synthetic_records(100_000, seed=4)
"""

import random

from paper_2303_01845_b200.seqio import SequenceRecord

STANDARD_RESIDUES = "ARNDCQEGHILKMFPSTWYV"


def _substitute(seq: str, rng: random.Random, rate: float) -> str:
    out = list(seq)
    for pos in range(len(out)):
        if rng.random() < rate:
            old = out[pos]
            new = rng.choice(STANDARD_RESIDUES)
            while new == old:
                new = rng.choice(STANDARD_RESIDUES)
            out[pos] = new
    return "".join(out)


def _cut(seq: str, rng: random.Random, min_len: int) -> str:
    keep = min(max(min_len, int(len(seq) * rng.uniform(0.4, 0.9))), len(seq))
    start = rng.randint(0, len(seq) - keep)
    return seq[start:start + keep]


def synthetic_records(count: int, seed: int, *, min_len: int = 50, max_len: int = 500,
                      family_fraction: float = 0.35, family_size: int = 3,
                      mutation_rate: float = 0.12, fragment_fraction: float = 0.25) -> list:
    rng = random.Random(seed)
    seqs: list = []
    while len(seqs) < count:
        n = rng.randint(min_len, max_len)
        base = "".join(rng.choice(STANDARD_RESIDUES) for _ in range(n))
        seqs.append(base)
        if rng.random() >= family_fraction:
            continue
        for _ in range(family_size - 1):
            if len(seqs) >= count:
                break
            v = _substitute(base, rng, mutation_rate)
            if rng.random() < fragment_fraction:
                v = _cut(v, rng, min_len)
            seqs.append(v)
    return [SequenceRecord(i, f"s{i:05d}", s) for i, s in enumerate(seqs)]


def write_fasta(path, records) -> None:
    with open(path, "w", encoding="utf-8") as fh:
        for rec in records:
            fh.write(f">{rec.header}\n{rec.residues}\n")

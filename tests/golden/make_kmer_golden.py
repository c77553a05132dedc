"""Generate tests/golden/kmer_candidates.json from the REFERENCE's candidate
discovery: pastislite.kmer.build_kmer_matrix (kmer.py:56-90) and the overlap
semiring product A * A^T (kmer.py:93-126, sparse.local_spgemm sparse.py:236).
For each corpus it stores every unordered pair i < j sharing >= 1 distinct
k-mer with its shared count (the pipeline keeps count >= min_shared_kmers,
pipeline.py:290-303).  Runs only in the build container.

    python tests/golden/make_kmer_golden.py
"""

import json
import os
import random
import sys

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)

from pastislite import kmer, sparse, synth  # noqa: E402
from pastislite.seqio import SequenceRecord  # noqa: E402


def overlap_pairs(records, k):
    params = kmer.KmerParams(k=k)
    a = kmer.build_kmer_matrix(records, params)
    c = sparse.local_spgemm(a, sparse.local_transpose(a), kmer.overlap_semiring(params))
    out = []
    for i, j, payload in c.to_coo():
        if i < j:
            out.append([i, j, payload.count])
    out.sort()
    return out


def low_complexity(n, seed):
    rng = random.Random(seed)
    recs = []
    for i in range(n):
        unit = "".join(rng.choice("AGS") for _ in range(rng.randint(1, 4)))
        s = (unit * 200)[: rng.randint(3, 90)]
        if rng.random() < 0.5:
            s = "".join(ch if rng.random() > 0.1 else rng.choice("ARNDCQEGHILKMFPSTWYVBZXU*")
                        for ch in s)
        recs.append(SequenceRecord(i, f"q{i}", s))
    return recs


def main():
    cases = []
    cases.append({"name": "config1", "corpus": [1000, 0], "k": 6,
                  "pairs": overlap_pairs(synth.synthetic_records(1000, 0), 6)})
    cases.append({"name": "corpus300_k4", "corpus": [300, 7], "k": 4,
                  "pairs": overlap_pairs(synth.synthetic_records(300, 7), 4)})
    cases.append({"name": "corpus200_k3", "corpus": [200, 5], "k": 3,
                  "pairs": overlap_pairs(synth.synthetic_records(200, 5), 3)})
    lc = low_complexity(150, 11)
    cases.append({"name": "lowcomplex_k5", "seqs": [r.residues for r in lc], "k": 5,
                  "pairs": overlap_pairs(lc, 5)})
    cases.append({"name": "lowcomplex_k2", "seqs": [r.residues for r in lc], "k": 2,
                  "pairs": overlap_pairs(lc, 2)})
    with open(os.path.join(HERE, "kmer_candidates.json"), "w") as fh:
        json.dump({"source": "pastislite.kmer.build_kmer_matrix + overlap_semiring SpGEMM",
                   "cases": cases}, fh)
    for c in cases:
        n2 = sum(1 for p in c["pairs"] if p[2] >= 2)
        print(c["name"], "k", c["k"], "pairs>=1", len(c["pairs"]), ">=2", n2)


if __name__ == "__main__":
    main()

"""Candidate discovery: the CPU oracle vs the reference's
golden candidate sets (CPU), and the GPU sw_kmer_candidates vs the same
goldens (gpu).  tests/golden/kmer_candidates.json comes from the reference's
build_kmer_matrix + overlap-semiring SpGEMM (make_kmer_golden.py): config 1
and small corpora at k = 6, 4, 3, plus low-complexity repeats at k = 5, 2."""

import numpy as np
import pytest

from conftest import load_golden
from oracle import kmer_oracle
from paper_2303_01845_b200 import _native
from pastis_synth import corpus

GOLD = load_golden("kmer_candidates.json")["cases"]


def _seqs(case):
    if "seqs" in case:
        return case["seqs"]
    n, seed = case["corpus"]
    return [r.residues for r in corpus.synthetic_records(n, seed)]


@pytest.mark.parametrize("idx", range(len(GOLD)))
def test_oracle_matches_reference_candidates(idx):
    case = GOLD[idx]
    i, j, c = kmer_oracle.shared_counts(_seqs(case), case["k"])
    got = np.stack([i, j, c], axis=1).tolist() if len(i) else []
    assert got == case["pairs"]


def test_kmer_params_mirror():
    from paper_2303_01845_b200.candidates import KmerParams
    assert KmerParams().k == 6 and KmerParams().min_shared_kmers == 2
    assert KmerParams().code_space == 25 ** 6
    for bad, msg in (({"k": 0}, "k must be >= 1"), ({"alphabet_size": 20}, "alphabet size"),
                     ({"min_shared_kmers": -1}, "min_shared_kmers")):
        with pytest.raises(ValueError, match=msg):
            KmerParams(**bad)


@pytest.mark.gpu
@pytest.mark.parametrize("idx", range(len(GOLD)))
@pytest.mark.parametrize("min_shared", [0, 1, 2, 3])
def test_gpu_candidates_match_reference(idx, min_shared):
    from paper_2303_01845_b200.candidates import KmerParams, kmer_candidates
    case = GOLD[idx]
    cand, st = kmer_candidates(_seqs(case), KmerParams(k=case["k"], min_shared_kmers=min_shared))
    ref = [p for p in case["pairs"] if p[2] >= min_shared]
    got = np.stack([cand["i"], cand["j"], cand["count"]], axis=1).tolist() if len(cand) else []
    assert got == ref
    assert st["discovered"] == len(case["pairs"])
    assert st["performed"] == len(ref)


@pytest.mark.gpu
def test_gpu_candidates_random_vs_oracle():
    """Random corpora incl. short sequences, unknown bytes and repeats."""
    from paper_2303_01845_b200.candidates import KmerParams, kmer_candidates
    rng = np.random.default_rng(7)
    alpha = np.frombuffer(b"ARNDCQEGHILKMFPSTWYVBZXU*J", np.uint8)
    seqs = []
    for n in rng.integers(0, 120, size=700):
        pool = alpha[: rng.integers(3, len(alpha) + 1)]
        seqs.append(pool[rng.integers(0, len(pool), size=int(n))].tobytes().decode())
    for k in (1, 3, 6, 8):
        cand, st = kmer_candidates(seqs, KmerParams(k=k, min_shared_kmers=1))
        i, j, c = kmer_oracle.shared_counts(seqs, k)
        assert len(cand) == len(i)
        assert (cand["i"] == i).all() and (cand["j"] == j).all() and (cand["count"] == c).all()
        assert st["short_seqs"] == sum(1 for s in seqs if len(s) < k)

"""The CPU oracle (oracle/) pinned to golden vectors made by the reference."""

import pytest

from conftest import expect_tuple, load_golden, matrix
from oracle import oracle

SETS = ["kats.json", "random_pairs.json", "config2_sample.json"]


@pytest.mark.parametrize("name", SETS + ["long_pairs.json"])
def test_c_oracle_matches_reference(name):
    for case in load_golden(name):
        got = oracle.align_c(case["a"], case["b"], case["gap_open"], case["gap_extend"],
                             matrix(case["matrix"]))
        assert got == expect_tuple(case), (case["kind"], case["a"][:40], case["b"][:40])


@pytest.mark.parametrize("name", SETS)
def test_numpy_oracle_matches_reference(name):
    cases = load_golden(name)
    for case in cases[:400]:
        got = oracle.align_numpy(case["a"], case["b"], case["gap_open"], case["gap_extend"],
                                 matrix(case["matrix"]))
        assert got == expect_tuple(case), (case["kind"], case["a"][:40], case["b"][:40])


def test_score_only_oracle_agrees():
    for case in load_golden("long_pairs.json") + load_golden("kats.json"):
        best, i_end, j_end = oracle.score_c(case["a"], case["b"], case["gap_open"],
                                            case["gap_extend"], matrix(case["matrix"]))
        e = case["expect"]
        assert (best, i_end, j_end) == (e["score"], e["i_end"], e["j_end"])


def test_config1_results():
    d = load_golden("config1.json")
    res = d["residues"]
    for (i, j), exp in zip(d["pairs"], d["results"]):
        got = oracle.align_c(res[i], res[j], d["gap_open"], d["gap_extend"], matrix("blosum62"))
        assert list(got) == exp[:7]


def test_batch_oracle_threads():
    import numpy as np
    from paper_2303_01845_b200.batch import pack_pairs

    cases = load_golden("random_pairs.json")[:300]
    cases = [c for c in cases if c["gap_open"] == 11 and c["gap_extend"] == 1
             and c["matrix"] == "blosum62"]
    batch = pack_pairs([(c["a"], c["b"]) for c in cases])
    out = oracle.align_batch_c(batch.arena, batch.pairs, 11, 1, matrix("blosum62"), threads=4)
    for row, c in zip(out, cases):
        assert tuple(int(v) for v in row[:7]) == expect_tuple(c)
        assert row[7] == 0


def test_empty_rejected():
    with pytest.raises(ValueError):
        oracle.align_c("", "A", 11, 1, matrix("blosum62"))


def test_long_pair_oracle_matches_full_oracle():
    """orc_align_long (O(sqrt(m) n) memory, used for config-5-size pairs) equals
    orc_align on homologs and unrelated pairs across gap settings, including
    traceback walks that cross its checkpoint blocks."""
    from pastis_synth import workloads
    mat = matrix("blosum62")
    for kind, kw in ((3, {}), (5, dict(lo=200, hi=1500, hom_frac=0.7)), (2, dict(length=120))):
        arena, table = workloads.packed(kind, 120, 11, **kw)
        for go, ge in ((11, 1), (11, 2), (5, 5), (3, 0), (0, 0)):
            full = oracle.align_batch_c(arena, table, go, ge, mat, threads=8)
            lng = oracle.align_batch_c(arena, table, go, ge, mat, threads=8, long=True)
            assert (full == lng).all(), (kind, go, ge)


def test_packed_generator_is_deterministic():
    from pastis_synth import workloads
    a1, t1 = workloads.config3_packed(5000, seed=3, threads=1)
    a2, t2 = workloads.config3_packed(5000, seed=3, threads=6)
    assert (a1 == a2).all() and (t1 == t2).all()
    assert t1["a_len"].min() >= 30 and t1["a_len"].max() <= 2000

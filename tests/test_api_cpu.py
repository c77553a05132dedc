"""Host-side API parity with the reference (no GPU needed)."""

import hashlib

import numpy as np
import pytest

from conftest import FIELDS, load_golden, matrix
import paper_2303_01845_b200 as sw
from paper_2303_01845_b200 import alphabet, blosum62


def test_alphabet_and_blosum62_match_reference():
    g = load_golden("blosum62.json")
    assert alphabet.ALPHABET == g["alphabet"]
    assert np.array_equal(blosum62.MATRIX, np.asarray(g["matrix"]))
    assert not blosum62.MATRIX.flags.writeable
    assert alphabet.INDEX["X"] == 22 and alphabet.SIZE == 25


def test_align_params_validation():
    sw.AlignParams()
    with pytest.raises(ValueError, match="gap_open >= gap_extend >= 0"):
        sw.AlignParams(gap_open=1, gap_extend=2)
    with pytest.raises(ValueError, match="gap_open >= gap_extend >= 0"):
        sw.AlignParams(gap_open=1, gap_extend=-1)
    with pytest.raises(ValueError, match="25x25"):
        sw.AlignParams(matrix=np.zeros((24, 24)))
    bad = np.asarray(blosum62.MATRIX).copy()
    bad[0, 1] = 7
    with pytest.raises(ValueError, match="symmetric"):
        sw.AlignParams(matrix=bad)
    assert issubclass(sw.AlignmentError, ValueError)


def test_encode_matches_reference_lut():
    s = "ARNDCQEGHILKMFPSTWYVBZXU*ajO1"
    got = sw.encode(s)
    exp = [alphabet.INDEX.get(ch, 22) for ch in s]
    assert got.tolist() == exp and got.dtype == np.int64


def _result(exp):
    return sw.AlignmentResult(*[exp[f] for f in FIELDS], exp["cells"])


def test_evaluate_pair_matches_reference_edges():
    n = 0
    for case in load_golden("random_pairs.json") + load_golden("kats.json"):
        params = sw.AlignParams(gap_open=case["gap_open"], gap_extend=case["gap_extend"],
                                matrix=matrix(case["matrix"]))
        edge = sw.evaluate_pair(0, 1, case["a"], case["b"], _result(case["expect"]), params)
        exp = case["expect"]["edge"]
        if exp is None:
            assert edge is None
        else:
            n += 1
            assert [edge.score, edge.identity, edge.coverage_i, edge.coverage_j] == exp
    assert n > 50
    with pytest.raises(ValueError, match="not canonical"):
        sw.evaluate_pair(2, 1, "A", "A", _result(load_golden("kats.json")[0]["expect"]),
                         sw.AlignParams())


def test_config1_digest_from_reference_results():
    """evaluate_pair + format_edge_line + canonical_bytes over the reference's
    own config-1 results reproduce the pipeline's canonical sha256."""
    d = load_golden("config1.json")
    params = sw.AlignParams()
    lines = []
    for (i, j), r in zip(d["pairs"], d["results"]):
        edge = sw.evaluate_pair(i, j, d["residues"][i], d["residues"][j],
                                sw.AlignmentResult(*r), params)
        if edge is not None:
            lines.append(sw.format_edge_line(edge, d["headers"]))
    canon = sw.canonical_bytes(lines)
    assert canon.decode().splitlines() == d["canonical_lines"]
    assert hashlib.sha256(canon).hexdigest() == d["canonical_sha256"]


def test_vectorised_evaluate_matches_per_pair():
    from paper_2303_01845_b200._native import RESULT_DTYPE
    d = load_golden("config1.json")
    params = sw.AlignParams()
    rec = np.zeros(len(d["results"]), dtype=RESULT_DTYPE)
    for k, r in enumerate(d["results"]):
        for f, v in zip(FIELDS, r[:7]):
            rec[f][k] = v
    ii = np.array([p[0] for p in d["pairs"]])
    jj = np.array([p[1] for p in d["pairs"]])
    la = np.array([len(d["residues"][i]) for i in ii])
    lb = np.array([len(d["residues"][j]) for j in jj])
    acc, ident, ca, cb = sw.evaluate_records(ii, jj, la, lb, rec, params.min_identity,
                                             params.min_coverage)
    for k, ((i, j), r) in enumerate(zip(d["pairs"], d["results"])):
        edge = sw.evaluate_pair(i, j, d["residues"][i], d["residues"][j],
                                sw.AlignmentResult(*r), params)
        assert (edge is not None) == bool(acc[k])
        if edge is not None:
            assert (edge.identity, edge.coverage_i, edge.coverage_j) == (ident[k], ca[k], cb[k])


def test_pack_pairs_dedup_and_errors():
    a = "MKVLAAG"
    b = "MKV"
    pairs = [(a, b, 0), (a, b, 1), ("", b, 2), ("Aé", "A", 3), (b, a, 4), ("WW", "", 5)]
    batch = sw.pack_pairs(pairs)
    assert [e[0] for e in batch.errors] == [2, 3, 5]
    assert isinstance(batch.errors[0][1], sw.AlignmentError)
    assert str(batch.errors[0][1]) == "cannot align an empty sequence"
    assert isinstance(batch.errors[1][1], UnicodeEncodeError)
    assert batch.index.tolist() == [0, 1, 4]
    assert bytes(batch.arena) == (a + b).encode()  # each distinct sequence stored once
    t = batch.pairs
    assert t["a_off"].tolist() == [0, 0, 7] and t["b_off"].tolist() == [7, 7, 0]
    assert t["a_len"].tolist() == [7, 7, 3] and t["b_len"].tolist() == [3, 3, 7]
    assert batch.cells == 63
    # raw bytes are kept (unknown symbols are mapped on the device, align.py:27-30)
    b2 = sw.pack_pairs([("ajX", "AJx")])
    assert bytes(b2.arena) == b"ajXAJx"


def test_pack_codes_layout():
    from paper_2303_01845_b200.batch import pack_codes
    arena, t = pack_codes([b"AAA", b"C"], [b"GG", b"TTTT"])
    assert bytes(arena) == b"AAAGGCTTTT"
    assert t["a_off"].tolist() == [0, 5] and t["b_off"].tolist() == [3, 6]
    assert t["a_len"].tolist() == [3, 1] and t["b_len"].tolist() == [2, 4]

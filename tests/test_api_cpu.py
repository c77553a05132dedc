"""Host-side API parity with the reference (no GPU needed)."""

import hashlib
import os

import numpy as np
import pytest

from conftest import FIELDS, ROOT, load_golden, matrix
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


def test_pack_pairs_parallel_path_matches_sequential_semantics():
    """The C packer's threaded fast path (tuples of ASCII str) and its Python-
    semantics path (everything else) give the same table: every packed pair
    points at its own bytes, shared objects are stored once, and the per-pair
    errors keep the reference's types and input order."""
    rng = np.random.default_rng(3)
    seqs = ["".join(rng.choice(list("ACDEFGHIKLMNPQRSTVWY"), size=int(n)))
            for n in rng.integers(1, 400, size=500)]
    pairs = []
    for k in range(20000):
        a, b = seqs[k % 500], seqs[(k * 7 + 3) % 500]
        if k % 997 == 5:
            pairs.append((a, "", k))                 # AlignmentError
        elif k % 991 == 7:
            pairs.append([a, b])                     # list item: slow path, still packed
        elif k % 983 == 11:
            pairs.append((a, "A" * 65001, k))        # over the GPU domain: ValueError
        elif k % 977 == 13:
            pairs.append((a, b.encode(), k))         # bytes: AttributeError like .encode
        else:
            pairs.append((a, b, k))
    batch = sw.pack_pairs(pairs)
    err_idx = [e[0] for e in batch.errors]
    assert err_idx == sorted(err_idx)
    kinds = {k: type(e) for k, e in batch.errors}
    for k in err_idx:
        assert kinds[k] in (sw.AlignmentError, ValueError, AttributeError)
    assert len(batch.index) + len(batch.errors) == len(pairs)
    raw = bytes(batch.arena)
    for row, k in zip(batch.pairs.tolist(), batch.index.tolist()):
        a_off, b_off, la, lb = row
        assert raw[a_off:a_off + la].decode() == pairs[k][0]
        assert raw[b_off:b_off + lb].decode() == pairs[k][1]
    assert len(raw) <= sum(len(s) for s in seqs) + 65001   # distinct objects stored once


def test_pack_pairs_concurrent_calls_and_map_reuse():
    """The packer keeps its dedup maps between calls (cleared after use) and
    two batches may be packed at once (AlignEngine's two host threads): many
    concurrent and repeated calls, with different sizes and sharing patterns,
    each give a table whose every pair points at the same bytes as in a call
    made alone (which user of a shared object owns its bytes is up to the
    packing threads, so offsets may differ)."""
    import threading
    rng = np.random.default_rng(7)
    seqs = ["".join(rng.choice(list("ACDEFGHIKLMNPQRSTVWY"), size=int(n)))
            for n in rng.integers(1, 300, size=800)]

    def batch_of(seed, n):
        r = np.random.default_rng(seed)
        return [(seqs[int(i)], seqs[int(j)], None) for i, j in r.integers(0, 800, size=(n, 2))]

    jobs = [batch_of(s, n) for s, n in ((1, 9000), (2, 20000), (3, 500), (4, 13000))]
    alone = [sw.pack_pairs(b) for b in jobs]

    def check(b, ref):
        got = sw.pack_pairs(b)
        raw, rraw = bytes(got.arena), bytes(ref.arena)
        assert len(got.pairs) == len(ref.pairs) and not got.errors
        for (ao, bo, la, lb), (rao, rbo, _, _) in zip(got.pairs.tolist(), ref.pairs.tolist()):
            assert raw[ao:ao + la] == rraw[rao:rao + la] and raw[bo:bo + lb] == rraw[rbo:rbo + lb]
        assert len(raw) == len(rraw)              # each distinct object stored once

    errors = []

    def worker(k):
        try:
            for rep in range(3):
                check(jobs[(k + rep) % 4], alone[(k + rep) % 4])
        except Exception as e:  # noqa: BLE001 - reported below
            errors.append(e)

    threads = [threading.Thread(target=worker, args=(k,)) for k in range(4)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors[0]


def test_result_list_is_lazy_and_list_like():
    from paper_2303_01845_b200 import _native
    from paper_2303_01845_b200.align import ResultList
    batch = sw.pack_pairs([("AAAA", "AAAA", 0), ("", "A", 1), ("MKV", "MKV", 2)])
    rec = np.zeros(2, dtype=_native.RESULT_DTYPE)
    rec["score"] = [16, 15]
    rec["aln_len"] = [4, 3]
    res = ResultList(batch, rec)
    assert len(res) == 3 and res[1] is None
    assert res[0].score == 16 and res[0].cells == 16 and res[-1].cells == 9
    assert [r.score if r else None for r in res] == [16, None, 15]
    assert res[0:2] == [res[0], None]
    assert list(res) == list(res[:])


def test_interop_with_reference_classes_when_importable():
    """With pastislite importable (this container), the drop-in uses the
    reference's own AlignmentError / AlignmentResult / BatchCounters /
    SimilarityEdge classes, so `except pastislite.align.AlignmentError` and
    dataclass equality work across the two packages."""
    import subprocess
    import sys
    ref = "/root/reference/pkg/src"
    if not os.path.isdir(ref):
        pytest.skip("reference not present")
    code = (f"import sys; sys.path[:0] = [{ref!r}, {ROOT!r}]\n"
            "import pastislite.align as R, pastislite.seqio as S\n"
            "import paper_2303_01845_b200 as sw\n"
            "from paper_2303_01845_b200 import edges\n"
            "assert sw.AlignmentError is R.AlignmentError\n"
            "assert sw.AlignmentResult is R.AlignmentResult\n"
            "assert sw.BatchCounters is R.BatchCounters\n"
            "assert edges.SimilarityEdge is S.SimilarityEdge\n"
            "b = sw.pack_pairs([('', 'A', 0)])\n"
            "assert isinstance(b.errors[0][1], R.AlignmentError)\n"
            "print('ok')\n")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True)
    assert out.returncode == 0 and out.stdout.strip() == "ok", out.stderr


def test_chunked_pipeline_merges_like_one_batch(monkeypatch):
    """AlignEngine's large-batch pipeline (pack chunk k+1 while chunk k is on
    the GPU) returns the same results, errors and counters as one batch.  The
    device call is replaced by the C oracle here (CPU test of the host logic)."""
    from oracle import oracle
    from paper_2303_01845_b200 import _native
    from paper_2303_01845_b200 import align as A
    mat = matrix("blosum62")

    def fake_align_packed(batch, params, devices=(0,)):
        ref = oracle.align_batch_c(batch.arena, batch.pairs, params.gap_open, params.gap_extend,
                                   mat, threads=4)
        rec = np.zeros(len(batch.pairs), dtype=_native.RESULT_DTYPE)
        for k, f in enumerate(FIELDS):
            rec[f] = ref[:, k]
        return rec, [{"forward_ms": 1.0}]

    monkeypatch.setattr(A, "align_packed", fake_align_packed)
    rng = np.random.default_rng(7)
    letters = list("ACDEFGHIKLMNPQRSTVWY")
    seqs = ["".join(rng.choice(letters, size=int(n))) for n in rng.integers(5, 60, size=80)]
    pairs = [(seqs[k % 80], seqs[(k * 3 + 1) % 80] if k % 41 else "", k) for k in range(700)]
    params = sw.AlignParams(gap_open=11, gap_extend=1)
    one = A._align(pairs, params, [0])
    monkeypatch.setattr(A, "_CHUNK", 64)
    many = A._align(pairs, params, [0])
    assert many[4]["chunks"] == 11
    assert [e[0] for e in one[1]] == [e[0] for e in many[1]]
    assert one[2].alignments == many[2].alignments and one[2].cells == many[2].cells
    assert list(one[0]) == list(many[0])
    assert many[0][41] is None and many[0][3].cells == len(seqs[3]) * len(seqs[10])


def test_pinned_pool_reuse_and_caps(monkeypatch):
    """PinnedPool hands back the smallest free buffer that fits, keeps at most
    max_free buffers (smallest freed first) and max_free_bytes (largest freed
    first), against a fake allocator (no CUDA driver here)."""
    import ctypes
    from paper_2303_01845_b200 import _native

    class FakeLib:
        def __init__(self):
            self.live, self.allocs, self.frees = {}, 0, 0

        def sw_host_alloc(self, n):
            buf = ctypes.create_string_buffer(n)
            ptr = ctypes.addressof(buf)
            self.live[ptr] = buf
            self.allocs += 1
            return ptr

        def sw_host_free(self, ptr):
            del self.live[ptr]
            self.frees += 1

    fake = FakeLib()
    monkeypatch.setattr(_native, "load", lambda *a, **k: fake)
    pool = _native.PinnedPool(max_free=3, max_free_bytes=5 << 20)
    a = pool.acquire(3 << 20)            # 4 MiB cap
    b = pool.acquire(100)                # 1 MiB cap
    assert a.pinned and b.pinned and a.cap == 4 << 20 and b.cap == 1 << 20
    a.array[:] = 7
    a.release(); b.release()
    assert fake.allocs == 2 and fake.frees == 0
    c = pool.acquire(10)                 # smallest fit: the 1 MiB buffer
    assert c.cap == 1 << 20 and fake.allocs == 2
    c.release()
    bufs = [pool.acquire(1 << 20) for _ in range(4)]   # the 1 MiB, the 4 MiB, 2 new
    assert fake.allocs == 4 and sorted(x.cap for x in bufs) == [1 << 20] * 3 + [4 << 20]
    for x in bufs:
        x.release()
    # released one by one: with 1 + 4 + 1 MiB free (6 MiB > 5 MiB) the largest
    # goes; the last 1 MiB then fits both caps
    caps = sorted(cap for _, cap in pool._free)
    assert caps == [1 << 20] * 3
    assert fake.frees == 1 and len(fake.live) == 3
    extra = [pool.acquire(1 << 20) for _ in range(4)]   # 3 reused + 1 new
    assert fake.allocs == 5
    for x in extra:
        x.release()
    assert len(pool._free) == 3 and fake.frees == 2      # count cap: one 1 MiB freed

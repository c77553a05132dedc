"""GPU parity: the B200 kernels vs the reference's golden vectors and the C oracle.

Every comparison is exact (integer fields).  Runs only on a GPU box
(`pytest -m gpu`); all calls go through libpastis_sw.so's C ABI.
"""

import hashlib

import numpy as np
import pytest

from conftest import FIELDS, expect_tuple, load_golden, matrix
from oracle import oracle

pytestmark = pytest.mark.gpu

import paper_2303_01845_b200 as sw  # noqa: E402
from paper_2303_01845_b200 import _native  # noqa: E402
from pastis_synth import workloads  # noqa: E402
from paper_2303_01845_b200.batch import pack_codes, pack_pairs  # noqa: E402


def _params(go, ge, mname="blosum62"):
    return sw.AlignParams(gap_open=go, gap_extend=ge, matrix=matrix(mname))


def _tuple(res):
    return tuple(getattr(res, f) for f in FIELDS)


def _check_cases(cases):
    groups = {}
    for k, c in enumerate(cases):
        groups.setdefault((c["gap_open"], c["gap_extend"], c["matrix"]), []).append(k)
    bad = []
    for (go, ge, mname), idx in groups.items():
        results, errors, counters = sw.align_batch(
            [(cases[k]["a"], cases[k]["b"], None) for k in idx], _params(go, ge, mname))
        assert not errors, errors[:3]
        for k, res in zip(idx, results):
            c = cases[k]
            if _tuple(res) != expect_tuple(c) or res.cells != c["expect"]["cells"]:
                bad.append((c["kind"], go, ge, c["a"][:30], c["b"][:30], _tuple(res),
                            expect_tuple(c)))
    assert not bad, f"{len(bad)} mismatches, first: {bad[:3]}"


@pytest.mark.parametrize("name", ["kats.json", "random_pairs.json", "config2_sample.json",
                                  "long_pairs.json"])
def test_golden_vectors(name):
    _check_cases(load_golden(name))


def test_single_pair_api():
    for c in load_golden("kats.json"):
        res = sw.smith_waterman(c["a"], c["b"], _params(c["gap_open"], c["gap_extend"]))
        assert _tuple(res) == expect_tuple(c)
    with pytest.raises(sw.AlignmentError):
        sw.smith_waterman("", "AAA", _params(11, 1))


def test_error_isolation_and_order():
    pairs = [("AAAA", "AAAA", 0), ("", "A", 1), ("MKV", "MKV", 2), ("Aé", "A", 3),
             ("WW", "", 4), ("P", "A", 5)]
    results, errors, counters = sw.align_batch(pairs, _params(11, 2))
    assert [e[0] for e in errors] == [1, 3, 4]
    assert isinstance(errors[0][1], sw.AlignmentError)
    assert isinstance(errors[1][1], UnicodeEncodeError)
    assert results[1] is None and results[3] is None and results[4] is None
    assert results[0].score == 16 and results[5].score == 0
    assert counters.alignments == 3 and counters.cells == 16 + 9 + 1


def test_config1_digest_through_engine():
    """Config 1's 628 pipeline pairs through AlignEngine + evaluate_pair reproduce
    the reference pipeline's canonical output byte for byte."""
    d = load_golden("config1.json")
    res = d["residues"]
    params = sw.AlignParams()
    with sw.AlignEngine(params, lanes=1, use_processes=True) as eng:
        pending = eng.submit([(res[i], res[j], None) for i, j in d["pairs"]])
        results, errors, counters, lanes = pending.result()
    assert not errors
    for r, exp in zip(results, d["results"]):
        assert list(_tuple(r)) + [r.cells] == exp
    lines = []
    for (i, j), r in zip(d["pairs"], results):
        edge = sw.evaluate_pair(i, j, res[i], res[j], r, params)
        if edge is not None:
            lines.append(sw.format_edge_line(edge, d["headers"]))
    canon = sw.canonical_bytes(lines)
    assert hashlib.sha256(canon).hexdigest() == d["canonical_sha256"]
    assert lanes and lanes[0][0] == 0


def _oracle_compare(sa, sb, go, ge, mname="blosum62", threads=16):
    arena, table = pack_codes(sa, sb)
    rec, tm = _native.align_host(arena, table, _native.make_params(go, ge, matrix(mname)))
    ref = oracle.align_batch_c(arena, table, go, ge, matrix(mname), threads=threads)
    got = np.stack([rec[f] for f in FIELDS], axis=1)
    bad = np.flatnonzero((got != ref[:, :7]).any(axis=1))
    assert (rec["status"] == 0).all()
    assert len(bad) == 0, (len(bad), [(int(k), got[k].tolist(), ref[k, :7].tolist())
                                      for k in bad[:3]])
    return rec, tm


@pytest.mark.parametrize("ge", [1, 2])
def test_config2_vs_oracle(ge):
    sa, sb = workloads.config2(3000, seed=11 + ge)
    _oracle_compare(sa, sb, 11, ge)


def test_config3_vs_oracle():
    sa, sb = workloads.config3(1500, seed=5)
    _oracle_compare(sa, sb, 11, 1)


def test_random_lengths_and_gaps_vs_oracle():
    rng = np.random.default_rng(1)
    for go, ge in [(11, 1), (10, 10), (5, 0), (0, 0), (3, 1)]:
        n = 800
        la = rng.integers(1, 700, size=n)
        lb = rng.integers(1, 700, size=n)
        sa, sb = [], []
        for x, y in zip(la, lb):
            a = workloads._random_seq(rng, int(x))
            if rng.random() < 0.5:
                b = workloads._fit(rng, workloads._homolog(rng, a, 0.2, 0.05), int(y))
            else:
                b = workloads._random_seq(rng, int(y))
            sa.append(a.tobytes())
            sb.append(b.tobytes())
        _oracle_compare(sa, sb, go, ge)


def test_packed_class_boundaries_vs_oracle():
    """Row counts at and around every packed class's strip multiples (32R rows,
    R = 4, 6, 7, 8, 9, 10, 16; the cost model picks the class per (m, n)),
    each with homologous and unrelated columns of several widths."""
    rng = np.random.default_rng(77)
    ms = sorted({v + d for R in (4, 6, 7, 8, 9, 10, 16) for k in (1, 2, 3)
                 for v in (32 * R * k,) for d in (-1, 0, 1) if 0 < v + d <= 2100})
    sa, sb = [], []
    for m in ms:
        a = workloads._random_seq(rng, m)
        for n in (1, 33, 300, m):
            b = (workloads._fit(rng, workloads._homolog(rng, a, 0.15, 0.04), n)
                 if rng.random() < 0.6 else workloads._random_seq(rng, n))
            sa.append(a.tobytes())
            sb.append(b.tobytes())
    for ge in (1, 2):
        _oracle_compare(sa, sb, 11, ge)


def test_invalid_pairs_fail_the_call_and_the_next_call_is_exact():
    """Pairs outside the arena (or longer than 65,000 residues) are rejected on
    the device by the planning kernel: the call raises (SW_EINVAL) without
    touching them, and the engine stays usable."""
    sa, sb = workloads.config2(64, seed=5)
    arena, table = pack_codes(sa, sb)
    p = _native.make_params(11, 1, matrix("blosum62"))
    bad = table.copy()
    bad["b_off"][7] = arena.size          # one byte past the end
    with pytest.raises(ValueError, match="outside the arena"):
        _native.align_host(arena, bad, p)
    wrap = table.copy()
    wrap["a_off"][5] = np.uint64(2**64 - 8)   # offset + length wraps around u64
    with pytest.raises(ValueError, match="outside the arena"):
        _native.align_host(arena, wrap, p)
    long = table.copy()
    long["a_len"][3] = 65001
    with pytest.raises(ValueError):
        _native.align_host(arena, long, p)
    _oracle_compare(sa, sb, 11, 1)


def test_long_multistrip_vs_oracle():
    sa, sb = workloads.config5(6, seed=3, lo=2000, hi=5000)
    rng = np.random.default_rng(4)
    a = workloads._random_seq(rng, 4200)
    sa.append(a.tobytes())
    sb.append(workloads._fit(rng, workloads._homolog(rng, a, 0.2, 0.04), 3900).tobytes())
    _oracle_compare(sa, sb, 11, 1)


def test_wide_path_vs_oracle():
    """Scores 33k (above the scaled int32 path's 32,640, inside the packed u16
    paths' headroom) and 66k (above the packed limit: both pairs of the duo
    re-run in the wide int32 path)."""
    rng = np.random.default_rng(9)
    sa, sb = [], []
    for n in (2990, 3000, 6100, 6500):
        a = np.frombuffer(b"W" * n, dtype=np.uint8).copy()
        a[rng.integers(0, n, 20)] = ord("C")
        sa.append(a.tobytes())
        sb.append(a[: n - 7].tobytes())
    rec, tm = _oracle_compare(sa, sb, 11, 1)
    assert tm["wide_pairs"] >= 2
    assert rec["score"].max() > 65535


def test_order_and_sharding_invariance():
    sa, sb = workloads.config3(2000, seed=21)
    arena, table = pack_codes(sa, sb)
    p = _native.make_params(11, 1, matrix("blosum62"))
    rec, _ = _native.align_host(arena, table, p)
    perm = np.random.default_rng(0).permutation(len(table))
    rec_p, _ = _native.align_host(arena, table[perm], p)
    assert (rec_p == rec[perm]).all()
    if _native.device_count() >= 2:
        rec_m, _ = _native.align_multi(arena, table, p, [0, 1])
        assert (rec_m == rec).all()


def test_symmetric_score_property():
    sa, sb = workloads.config2(2000, seed=77)
    arena, table = pack_codes(sa, sb)
    p = _native.make_params(11, 1, matrix("blosum62"))
    rec, _ = _native.align_host(arena, table, p)
    swapped = table.copy()
    swapped["a_off"], swapped["b_off"] = table["b_off"], table["a_off"]
    swapped["a_len"], swapped["b_len"] = table["b_len"], table["a_len"]
    rec_s, _ = _native.align_host(arena, swapped, p)
    assert (rec_s["score"] == rec["score"]).all()


def test_cta_per_pair_long_vs_oracle():
    """Pairs of >= 4 strips (2048+ rows) take the CTA-per-pair forward and
    reverse kernels: exact against the full C oracle."""
    rng = np.random.default_rng(17)
    sa, sb = [], []
    for la, lb, rel in [(2100, 2300, False), (3000, 2500, False), (4100, 1800, True),
                        (5200, 5000, False), (2600, 6000, False), (3500, 3400, True),
                        (2049, 2049, False), (6000, 2100, False)]:
        a = workloads._random_seq(rng, la)
        if rel:
            b = workloads._fit(rng, workloads._homolog(rng, a, 0.25, 0.05), lb)
        else:
            b = workloads._random_seq(rng, lb)
        sa.append(a.tobytes())
        sb.append(b.tobytes())
    for go, ge in [(11, 1), (11, 2)]:
        _oracle_compare(sa, sb, go, ge)


@pytest.mark.parametrize("pool_mb,n_pairs", [(16, 3000), (4, 1000)])
def test_pool_overflow_falls_back_exactly(pool_mb, n_pairs):
    """With a small traceback pool the packed pass defers pairs to further
    rounds (pool recycled), pairs whose checkpoints exceed a quarter of the pool
    take the scalar + box path, and box codes that do not fit are retried: the
    results stay exact, call after call."""
    import json
    import os
    import subprocess
    import sys
    code = r'''
import json, sys, numpy as np
sys.path.insert(0, ".")
from paper_2303_01845_b200 import _native, blosum62
from pastis_synth import workloads
from paper_2303_01845_b200.batch import pack_codes
from oracle import oracle
sa, sb = workloads.config3(int(sys.argv[1]), seed=8)
xa, xb = workloads.config2(2, seed=8, length=1900)   # checkpoints > pool/4: scalar path
sa, sb = sa + xa, sb + xb
arena, table = pack_codes(sa, sb)
m = np.asarray(blosum62.MATRIX, np.int32)
ref = oracle.align_batch_c(arena, table, 11, 1, m, threads=16)
F = ("score", "i_begin", "i_end", "j_begin", "j_end", "matches", "aln_len")
bad, launches = [], []
for _ in range(2):    # the second call runs on the pool the first one asked for
    rec, tm = _native.align_host(arena, table, _native.make_params(11, 1, m))
    got = np.stack([rec[f] for f in F], axis=1)
    bad.append(int((got != ref[:, :7]).any(axis=1).sum()))
    launches.append(int(tm["launches"]))
print(json.dumps({"bad": bad, "launches": launches}))
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, PASTIS_SW_POOL_MB=str(pool_mb))
    out = subprocess.run([sys.executable, "-c", code, str(n_pairs)], cwd=root, env=env,
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    res = json.loads(out.stdout.strip().splitlines()[-1])
    assert res["bad"] == [0, 0], res
    assert res["launches"][0] > 60, res      # several packed rounds ran


def test_pipelined_host_upload_matches_resident_arena():
    """sw_align_batch uploads the arena in slices while the packed forward
    runs (each warp waits for its pairs' slices).  With a multi-slice arena and
    the pair table shuffled against arena order -- early work waits on late
    slices -- the host path must equal the device path on a resident arena."""
    import torch
    sa, sb = workloads.config3_bulk(30_000, seed=5)
    arena, table = pack_codes(sa, sb)
    assert arena.size > 12 << 20          # several 4 MiB slices
    table = table[np.random.default_rng(3).permutation(len(table))]
    p = _native.make_params(11, 1, matrix("blosum62"))
    host, _ = _native.align_host(arena, table, p)
    d_arena = torch.from_numpy(arena).cuda()
    d_pairs = torch.from_numpy(table.view(np.uint8).copy()).cuda()
    d_out = torch.empty(len(table) * 32, dtype=torch.uint8, device="cuda")
    _native.align_device(d_arena.data_ptr(), arena.size, d_pairs.data_ptr(), len(table), p,
                         d_out.data_ptr(), stream=torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    dev = d_out.cpu().numpy().view(_native.RESULT_DTYPE)
    for f in FIELDS + ("status",):
        assert (host[f] == dev[f]).all(), f
    pick = np.random.default_rng(2).choice(len(table), 300, replace=False)
    ref = oracle.align_batch_c(arena, table[pick], 11, 1, matrix("blosum62"), threads=16)
    got = np.stack([host[f][pick] for f in FIELDS], axis=1)
    assert (got == ref[:, :7]).all()


def test_gathered_arena_without_gather_progress_is_exact():
    """A pinned host arena is gathered to the device by k_gather_arena while
    the packed pass consumes it; a packed warp whose pair has not arrived
    within 20 us copies it itself, so the call completes even when the gather
    kernel gets no SM.  With one gather block (PASTIS_SW_GATHER_BLOCKS=1) most
    pairs take that path: results equal the resident-arena path."""
    import json
    import os
    import subprocess
    import sys
    code = r'''
import json, sys, numpy as np
sys.path.insert(0, ".")
from paper_2303_01845_b200 import _native, blosum62
from paper_2303_01845_b200.batch import pack_codes
from pastis_synth import workloads
sa, sb = workloads.config3_bulk(40_000, seed=9)
arena, table = pack_codes(sa, sb)
p = _native.make_params(11, 1, np.asarray(blosum62.MATRIX, dtype=np.int32))
ref, _ = _native.align_host(arena, table, p)
buf = _native.pinned_pool().acquire(arena.size)
buf.array[:] = arena
got, _ = _native.align_host(buf.array, table, p)
buf.release()
print(json.dumps({"bad": int((got != ref).sum()), "ok": int((got["status"] == 0).sum()), "n": len(table)}))
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, PASTIS_SW_GATHER_BLOCKS="1")
    out = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True,
                         text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    res = json.loads(out.stdout.strip().splitlines()[-1])
    assert res["bad"] == 0 and res["ok"] == res["n"], res


def test_reverse_box_path_for_every_pair_exact():
    """PASTIS_SW_TRACEBACK=box sends every pair through the anchored reverse
    pass (with its dead-strip early stop) + box traceback: still exact on the
    golden vectors (11 gap settings / matrices) and on skewed config-3 pairs."""
    import json
    import os
    import subprocess
    import sys
    code = r'''
import json, sys, numpy as np
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from conftest import FIELDS, expect_tuple, load_golden, matrix
from paper_2303_01845_b200 import _native
from pastis_synth import workloads
from paper_2303_01845_b200.batch import pack_codes, pack_pairs
from oracle import oracle
bad = 0
cases = load_golden("random_pairs.json") + load_golden("kats.json") + load_golden("long_pairs.json")
groups = {}
for c in cases:
    groups.setdefault((c["gap_open"], c["gap_extend"], c["matrix"]), []).append(c)
for (go, ge, mname), cs in groups.items():
    batch = pack_pairs([(c["a"], c["b"]) for c in cs])
    rec, _ = _native.align_host(batch.arena, batch.pairs, _native.make_params(go, ge, matrix(mname)))
    for c, r in zip(cs, rec):
        if tuple(int(r[f]) for f in FIELDS) != expect_tuple(c):
            bad += 1
sa, sb = workloads.config3(3000, seed=21)
arena, table = pack_codes(sa, sb)
m = matrix("blosum62")
rec, tm = _native.align_host(arena, table, _native.make_params(11, 1, m))
ref = oracle.align_batch_c(arena, table, 11, 1, m, threads=16)
got = np.stack([rec[f] for f in FIELDS], axis=1)
bad += int((got != ref[:, :7]).any(axis=1).sum())
print(json.dumps({"bad": bad, "n": len(cases) + len(table)}))
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, PASTIS_SW_TRACEBACK="box")
    out = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True,
                         text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    res = json.loads(out.stdout.strip().splitlines()[-1])
    assert res["bad"] == 0, res


def _long_mix(seed: int, count: int):
    """Long pairs for the packed CTA path (>= 4 strips of 512 rows): random
    and homolog pairs of unequal shapes, so a duo mixes lengths and the best
    cell falls in early or deep strips."""
    rng = np.random.default_rng(seed)
    std = np.frombuffer(b"ARNDCQEGHILKMFPSTWYV", np.uint8)
    sa, sb = [], []
    for k in range(count):
        m = int(rng.integers(1600, 4200))
        a = std[rng.integers(0, 20, m)]
        if k % 3 == 0:
            b = std[rng.integers(0, 20, int(rng.integers(1600, 4200)))]
        else:
            b = a.copy()
            mut = rng.random(m) < 0.25
            b[mut] = std[rng.integers(0, 20, int(mut.sum()))]
            cut = int(rng.integers(0, m // 2))
            b = b[cut:cut + int(rng.integers(m // 3, m))]
        sa.append(a.tobytes())
        sb.append(b.tobytes())
    return sa, sb


def test_packed_cta_long_pairs_vs_oracle():
    sa, sb = _long_mix(31, 9)                       # odd: one CTA carries a single pair
    _oracle_compare(sa, sb, 11, 1)
    _oracle_compare(sa, sb, 10, 2)


def test_packed_cta_no_pool_room_falls_back_exactly():
    """A 1 MiB pool cannot hold the boundary slots: the duos go to the scalar
    one-CTA-per-pair kernel, still exact."""
    import json
    import os
    import subprocess
    import sys
    code = r'''
import json, sys, numpy as np
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from paper_2303_01845_b200 import _native, blosum62
from paper_2303_01845_b200.batch import pack_codes
from oracle import oracle
rng = np.random.default_rng(32)
std = np.frombuffer(b"ARNDCQEGHILKMFPSTWYV", np.uint8)
sa = [std[rng.integers(0, 20, int(rng.integers(1600, 2200)))].tobytes() for _ in range(5)]
sb = [std[rng.integers(0, 20, int(rng.integers(8000, 9000)))].tobytes() for _ in range(5)]
arena, table = pack_codes(sa, sb)   # boundary slots: 32 B x 8k+ columns per pair > the pool
m = np.asarray(blosum62.MATRIX, np.int32)
rec, tm = _native.align_host(arena, table, _native.make_params(11, 1, m))
ref = oracle.align_batch_c(arena, table, 11, 1, m, threads=16)
F = ("score", "i_begin", "i_end", "j_begin", "j_end", "matches", "aln_len")
got = np.stack([rec[f] for f in F], axis=1)
print(json.dumps({"bad": int((got != ref[:, :7]).any(axis=1).sum())}))
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, PASTIS_SW_POOL_MB="1")
    out = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True,
                         text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    assert json.loads(out.stdout.strip().splitlines()[-1])["bad"] == 0


def test_lookahead_loop_with_batches_in_flight():
    """The reference pipeline's pre-blocking loop (pipeline.py:209-240,
    305-314: submit a block, drain while more than `lookahead` are in flight,
    drain the rest) against AlignEngine with use_processes=True: config 1's
    628 pairs in 7 blocks, up to 3 batches submitted before the first
    result() -- the next block packs on the host while the GPU aligns the
    previous one; the canonical output is the reference's."""
    from collections import deque
    d = load_golden("config1.json")
    res = d["residues"]
    params = sw.AlignParams()
    blocks = [d["pairs"][k:k + 97] for k in range(0, len(d["pairs"]), 97)]
    lines, inflight, capacity, max_inflight = [], deque(), 2, 0
    with sw.AlignEngine(params, lanes=1, use_processes=True) as eng:
        def drain_one():
            pairs, pending = inflight.popleft()
            results, errors, counters, lanes = pending.result()
            assert not errors and counters.alignments == len(pairs)
            for (i, j), r in zip(pairs, results):
                edge = sw.evaluate_pair(i, j, res[i], res[j], r, params)
                if edge is not None:
                    lines.append(sw.format_edge_line(edge, d["headers"]))
        for pairs in blocks:
            batch = [(res[i], res[j], None) for i, j in pairs]
            inflight.append((pairs, eng.submit(batch)))
            max_inflight = max(max_inflight, len(inflight))
            while len(inflight) > capacity:
                drain_one()
        while inflight:
            drain_one()
    assert max_inflight == capacity + 1
    assert hashlib.sha256(sw.canonical_bytes(lines)).hexdigest() == d["canonical_sha256"]


_AA = np.frombuffer(b"ARNDCQEGHILKMFPSTWYV", dtype=np.uint8)


def _gapped_motif_pairs(seed: int, count: int):
    """Long pairs whose best local alignment is a motif split by a long gap
    (40-200 residues inserted on one side) inside random flanks, plus pairs
    holding two equal copies of a motif far apart: the anchored reverse pass
    has to carry an open gap (E or F state) across many 32-column chunks and
    strips, and ties spread the cells reaching best -- the cases the reverse
    pass's dead-strip and horizontal stops must not cut short."""
    rng = np.random.default_rng(seed)
    rnd = lambda k: _AA[rng.integers(0, 20, k)]   # noqa: E731
    sa, sb = [], []
    for k in range(count):
        motif = rnd(int(rng.integers(40, 120)))
        cut = int(rng.integers(10, len(motif) - 10))
        gap = rnd(int(rng.choice([40, 90, 200])))
        fa, fb = int(rng.integers(200, 3000)), int(rng.integers(200, 3000))
        left, right = motif[:cut], motif[cut:]
        if k % 3 == 0:    # gap in a (rows): vertical gap through strips
            a = np.concatenate([rnd(fa), left, gap, right, rnd(300)])
            b = np.concatenate([rnd(fb), left, right, rnd(300)])
        elif k % 3 == 1:  # gap in b (columns): horizontal gap across chunks
            a = np.concatenate([rnd(fa), left, right, rnd(300)])
            b = np.concatenate([rnd(fb), left, gap, right, rnd(300)])
        else:             # two copies of the motif, far apart in both sequences
            a = np.concatenate([rnd(fa), motif, rnd(700), motif, rnd(100)])
            b = np.concatenate([rnd(fb), motif, rnd(1500), motif, rnd(100)])
        sa.append(a.tobytes())
        sb.append(b.tobytes())
    return sa, sb


@pytest.mark.parametrize("mode", ["default", "box"])
def test_reverse_pass_across_long_gaps_exact(mode):
    """Gapped and repeated motifs in long random pairs (up to ~3,600 x 3,600,
    the warp and CTA reverse passes) under four gap settings down to 1/1
    (cheap gaps keep the reverse pass's wavefront alive longest); "box"
    sends every pair through the anchored reverse pass."""
    import json
    import os
    import subprocess
    import sys
    code = r'''
import json, sys, numpy as np
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from conftest import FIELDS, matrix
from test_gpu_parity import _gapped_motif_pairs
from paper_2303_01845_b200 import _native
from paper_2303_01845_b200.batch import pack_codes
from oracle import oracle
bad, n = 0, 0
m = matrix("blosum62")
for seed, (go, ge) in enumerate([(11, 1), (6, 2), (3, 1), (1, 1)]):
    sa, sb = _gapped_motif_pairs(100 + seed, 90)
    arena, table = pack_codes(sa, sb)
    rec, _ = _native.align_host(arena, table, _native.make_params(go, ge, m))
    ref = oracle.align_batch_c(arena, table, go, ge, m, threads=16)
    got = np.stack([rec[f] for f in FIELDS], axis=1)
    bad += int((got != ref[:, :7]).any(axis=1).sum())
    n += len(table)
print(json.dumps({"bad": bad, "n": n}))
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ)
    if mode == "box":
        env["PASTIS_SW_TRACEBACK"] = "box"
    out = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True,
                         text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    res = json.loads(out.stdout.strip().splitlines()[-1])
    assert res["bad"] == 0 and res["n"] == 360, res

"""GPU parity at full scale: every pair of the benched batches, exact.

* config 2 (100k x 300x300) and config 3 (1M skewed pairs, the exact batch
  bench.py times) against the threaded C oracle (oracle/sw_oracle.c,
  restating align.py:79-181), all pairs;
* config-5-size pairs (30,000-35,000 residues, long homologs that overflow
  the u16 and scaled-int32 paths, and a pair at the 65,000-residue cap)
  against orc_align_long, an O(sqrt(m) n)-memory exact restatement
  (score pass -> checkpoint rows -> block-wise traceback of align.py:133-169)
  that never sees the GPU's output;
* scores above the int16 tile range of the packed traceback.
"""

import os

import numpy as np
import pytest

from conftest import FIELDS, matrix
from oracle import oracle

pytestmark = pytest.mark.gpu

from paper_2303_01845_b200 import _native  # noqa: E402
from pastis_synth import workloads  # noqa: E402

THREADS = len(os.sched_getaffinity(0))


def _fields(rec):
    return np.stack([rec[f] for f in FIELDS], axis=1)


def _assert_exact(arena, table, go, ge, mat, long=False, rec=None):
    if rec is None:
        rec, _ = _native.align_host(arena, table, _native.make_params(go, ge, mat))
    ref = oracle.align_batch_c(arena, table, go, ge, mat, threads=THREADS, long=long)
    assert (ref[:, 7] == 0).all()
    got = _fields(rec)
    bad = np.flatnonzero((got != ref[:, :7]).any(axis=1) | (rec["status"] != 0))
    assert len(bad) == 0, (len(bad), [(int(k), got[k].tolist(), ref[k, :7].tolist(),
                                       int(table["a_len"][k]), int(table["b_len"][k]))
                                      for k in bad[:3]])
    return rec


def test_full_config2_exact():
    arena, table = workloads.config2_packed(100_000, seed=2303)
    rec = _assert_exact(arena, table, 11, 1, matrix("blosum62"))
    assert (rec["score"] > 0).all()


def test_full_config3_exact():
    """Config 3 at full size: the 1M pairs bench.py times (seed 2303), every
    pair exact against the C oracle (~25 s of host CPU on 16 cores)."""
    arena, table = workloads.config3_packed(1_000_000, seed=2303)
    _assert_exact(arena, table, 11, 1, matrix("blosum62"))


def _concat(parts):
    arenas, tables, off = [], [], 0
    for a, t in parts:
        t = t.copy()
        t["a_off"] += off
        t["b_off"] += off
        arenas.append(a)
        tables.append(t)
        off += a.size
    return np.concatenate(arenas), np.concatenate(tables)


def test_config5_long_pairs_exact():
    """Config-5 lengths up to the 65,000-residue cap, checked against the
    independent long-pair oracle: unrelated 30-35k pairs (packed CTA forward,
    j_end replay, reverse pass, box), 30k homologs scoring ~48k (above the
    scaled-int32 reverse pass's range: prefix box) and ~84k (above u16: wide
    re-run), random 2-35k pairs, and 65,000 x 65,000."""
    parts = [
        workloads.config5_packed(6, seed=71, lo=30000, hi=35000),
        workloads.config5_packed(2, seed=72, lo=30000, hi=30000, hom_frac=1.0, sub_rate=0.5),
        workloads.config5_packed(1, seed=73, lo=30000, hi=30000, hom_frac=1.0, sub_rate=0.3),
        workloads.config5_packed(6, seed=74, lo=2000, hi=35000),
        workloads.config5_packed(1, seed=75, lo=65000, hi=65000),
    ]
    arena, table = _concat(parts)
    mat = matrix("blosum62")
    rec, tm = _native.align_host(arena, table, _native.make_params(11, 1, mat))
    assert rec["score"][6:8].min() > 32767 and rec["score"][6:8].max() < 65375
    assert rec["score"][8] > 65535
    _assert_exact(arena, table, 11, 1, mat, long=True, rec=rec)


def _ident_matrix(diag, off):
    m = np.full((25, 25), off, dtype=np.int32)
    np.fill_diagonal(m, diag)
    return m


def test_high_scores_above_int16_tiles_exact():
    """identical sequences under a 50/-10 matrix with gap
    10/1 score 50 per residue -- 32,750 (655 aa: tile traceback), 32,800
    (656 aa) and 35,000 (700 aa) must not reach the int16 tiles of k_tb;
    also 1,300 aa (65,000: just inside the u16 forward) and 1,400 aa (wide)."""
    rng = np.random.default_rng(5)
    std = np.frombuffer(b"ARNDCQEGHILKMFPSTWYV", np.uint8)
    sa, sb = [], []
    for n in (655, 656, 700, 1000, 1300, 1400, 300):
        a = std[rng.integers(0, 20, n)].tobytes()
        sa.append(a)
        sb.append(a)
        b = bytearray(a)
        b[n // 2] = ord("W") if b[n // 2] != ord("W") else ord("C")
        sa.append(a)
        sb.append(bytes(b))
    from paper_2303_01845_b200.batch import pack_codes
    arena, table = pack_codes(sa, sb)
    mat = _ident_matrix(50, -10)
    rec = _assert_exact(arena, table, 10, 1, mat)
    assert rec["score"][4] == 35000 and rec["score"][2] == 32800


def test_tie_heavy_pairs_exact():
    """Row-major-first end cells and traceback priorities where ties are the
    rule: a 4-letter alphabet under a +1/-1 matrix with gap 1/1, 20,000
    random pairs of 100-900 residues across the packed classes, strips and
    windows; plus 200 constructed pairs where the best score is reached at
    (r, late column) and at (r + 1, early column): a = random, b = a[r-L+2 ..
    r+1] + W-padding + a[r-L+1 .. r] (W matches nothing in a).  The lane
    maxima in the checkpoints then point K5 at row r+1's early window, so row
    r = i_end's j_end needs the later window's replay (~90 % of these pairs,
    checked with a numpy DP when the test was written)."""
    rng = np.random.default_rng(11)
    alpha = np.frombuffer(b"ACGT", np.uint8)
    sa, sb = [], []
    wpad = np.frombuffer(b"W", np.uint8)
    for k in range(200):
        m = int(rng.integers(150, 800))
        a = alpha[rng.integers(0, 4, m)]
        L = int(rng.integers(30, 60))
        r = int(rng.integers(L, m - 2))
        b = np.concatenate([a[r - L + 2:r + 2], np.repeat(wpad, int(rng.integers(70, 300))),
                            a[r - L + 1:r + 1], np.repeat(wpad, int(rng.integers(0, 50)))])
        sa.append(a.tobytes())
        sb.append(b.tobytes())
    for k in range(20_000):
        m, n = (int(x) for x in rng.integers(100, 900, 2))
        a = alpha[rng.integers(0, 4, m)]
        if k % 2:
            b = alpha[rng.integers(0, 4, n)]
        else:
            b = a[rng.integers(0, max(1, m - n)) if m > n else 0:][:n].copy()
            mut = rng.random(len(b)) < 0.2
            b[mut] = alpha[rng.integers(0, 4, int(mut.sum()))]
        sa.append(a.tobytes())
        sb.append(b.tobytes())
    from paper_2303_01845_b200.batch import pack_codes
    arena, table = pack_codes(sa, sb)
    _assert_exact(arena, table, 1, 1, _ident_matrix(1, -1))


def test_unaligned_device_arena():
    """the device entry point takes arenas at any byte
    offset (k_encode handles the unaligned head)."""
    import torch
    arena, table = workloads.config3_packed(3000, seed=9)
    mat = matrix("blosum62")
    p = _native.make_params(11, 1, mat)
    ref = oracle.align_batch_c(arena, table, 11, 1, mat, threads=THREADS)
    base = torch.zeros(arena.size + 64, dtype=torch.uint8, device="cuda")
    d_pairs = torch.from_numpy(table.view(np.uint8).copy()).cuda()
    d_out = torch.empty(len(table) * 32, dtype=torch.uint8, device="cuda")
    for shift in (1, 3, 8, 15):
        sub = base[shift: shift + arena.size]
        sub.copy_(torch.from_numpy(arena.copy()))
        _native.align_device(sub.data_ptr(), arena.size, d_pairs.data_ptr(), len(table), p,
                             d_out.data_ptr())
        rec = d_out.cpu().numpy().view(_native.RESULT_DTYPE)
        assert (_fields(rec) == ref[:, :7]).all(), shift

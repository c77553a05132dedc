"""The C-ABI library: loads, exports every declared symbol, host-only entry points."""

import os
import re

import numpy as np
import pytest

from conftest import ROOT
from paper_2303_01845_b200 import _native
from paper_2303_01845_b200.batch import pack_codes

HEADER = os.path.join(ROOT, "include", "pastis_sw.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sw_[a-z_]+)\s*\(", src)))


def test_header_declares_expected_api():
    assert declared_functions() == sorted(_native.EXPORTED_SYMBOLS)


def test_library_exports_every_symbol():
    lib = _native.load()
    for name in declared_functions():
        assert hasattr(lib, name), name
    assert lib.sw_abi_version() == 2


def test_library_built_for_sm100a():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-lelf", _native.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_struct_layouts():
    assert _native.PAIR_DTYPE.itemsize == 24
    assert _native.RESULT_DTYPE.itemsize == 32
    import ctypes
    assert ctypes.sizeof(_native.SwParams) == 8 + 625 * 4


def test_partition_is_cell_balanced_contiguous():
    """sw_shard_ranges / sw_partition_pairs: contiguous ranges of equal cells,
    bounds[s] = min k with N * cells(pairs[0, k)) >= s * total."""
    rng = np.random.default_rng(0)
    for n in (0, 1, 7, 5000, 300_000):
        la = rng.integers(30, 2000, n)
        lb = rng.integers(30, 2000, n)
        t = np.zeros(n, dtype=_native.PAIR_DTYPE)
        t["a_len"], t["b_len"] = la, lb
        cells = la.astype(np.int64) * lb
        pre = np.concatenate(([0], np.cumsum(cells)))
        for world in (1, 2, 3, 8):
            b = _native.shard_ranges(t, world)
            total = int(pre[-1])
            expect = [0] + [int(np.searchsorted(pre * world, s_ * total, side="left"))
                            for s_ in range(1, world)] + [n]
            if total == 0:
                expect = [0] * world + [n]
            assert b.tolist() == expect, (n, world)
            shard, load = _native.partition(t, world)
            got = np.bincount(shard, weights=cells, minlength=world) if n else np.zeros(world)
            assert np.allclose(got, load.astype(np.float64))
            for s_ in range(world):
                assert (shard[b[s_]:b[s_ + 1]] == s_).all()
            if n:
                assert got.max() <= cells.sum() / world + cells.max()


def test_no_cpu_fallback_without_gpu():
    if _native.device_count() > 0:
        pytest.skip("GPU present")
    arena, t = pack_codes([b"AAAA"], [b"AAAA"])
    p = _native.make_params(11, 1, np.eye(25, dtype=np.int32))
    with pytest.raises(_native.NativeError):
        _native.align_host(arena, t, p)
    import paper_2303_01845_b200 as sw
    with pytest.raises(_native.NativeError):
        sw.align_batch([("AAAA", "AAAA", None)], sw.AlignParams())


def test_param_domain_checked_before_device():
    if _native.device_count() > 0:
        pytest.skip("GPU present: covered by the gpu tests")
    arena, t = pack_codes([b"A"], [b"A"])
    m = np.zeros((25, 25), dtype=np.int32)
    m[0, 0] = 500
    with pytest.raises(ValueError, match="127"):
        _native.align_host(arena, t, _native.make_params(11, 1, m))
    with pytest.raises(ValueError, match="gap_open >= gap_extend"):
        _native.align_host(arena, t, _native.make_params(1, 2, np.zeros((25, 25), np.int32)))


def test_status_and_return_codes_match_the_header():
    """The Python mirror's SW_* return codes and SW_STATUS_* record statuses are
    the header's #defines."""
    src = open(HEADER).read()
    defs = {k: int(v) for k, v in re.findall(r"#define\s+(SW_[A-Z_]+)\s+\(?(-?\d+)\)?", src)}
    for name in ("OK", "EMPTY", "INTERNAL", "INVALID"):
        assert getattr(_native, f"STATUS_{name}") == defs[f"SW_STATUS_{name}"], name
    for name in ("SW_OK", "SW_EINVAL", "SW_ECUDA", "SW_EINTERNAL"):
        assert getattr(_native, name) == defs[name], name

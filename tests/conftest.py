import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

FIELDS = ("score", "i_begin", "i_end", "j_begin", "j_end", "matches", "aln_len")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs through libpastis_sw.so)")


def load_golden(name):
    with open(os.path.join(GOLDEN, name)) as fh:
        return json.load(fh)


_MATS = None


def matrix(name):
    global _MATS
    if _MATS is None:
        _MATS = {k: np.asarray(v, dtype=np.int32) for k, v in load_golden("matrices.json").items()}
    return _MATS[name]


def expect_tuple(case):
    e = case["expect"]
    return tuple(e[f] for f in FIELDS)


@pytest.fixture(scope="session")
def golden():
    return load_golden

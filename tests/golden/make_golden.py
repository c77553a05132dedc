"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Runs only in the build container (it imports pastislite from
/root/reference/pkg/src, which does not exist on the GPU box).  Every
expected value below is produced by the reference's own code:
  pastislite.align.smith_waterman      (align.py:74)
  pastislite.oracle.reference_alignment (oracle.py:38, cross-check)
  pastislite.align.evaluate_pair       (align.py:184)
  pastislite.pipeline.run_search       (config 1 end to end)

    python tests/golden/make_golden.py
"""

import hashlib
import json
import os
import random
import sys
import tempfile

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REF)
sys.path.insert(0, ROOT)

from pastislite import align as ref_align  # noqa: E402
from pastislite import blosum62 as ref_blosum  # noqa: E402
from pastislite import oracle as ref_oracle  # noqa: E402
from pastislite import pipeline as ref_pipeline  # noqa: E402
from pastislite import seqio as ref_seqio  # noqa: E402
from pastislite import synth as ref_synth  # noqa: E402
from pastislite.alphabet import ALPHABET, INDEX  # noqa: E402

from pastis_synth import workloads  # noqa: E402

STD = "ARNDCQEGHILKMFPSTWYV"
FIELDS = ("score", "i_begin", "i_end", "j_begin", "j_end", "matches", "aln_len", "cells")


def matrix_named(name: str) -> np.ndarray:
    if name == "blosum62":
        return np.asarray(ref_blosum.MATRIX, dtype=np.int32)
    if name == "ident":
        m = np.full((25, 25), -4, dtype=np.int32)
        np.fill_diagonal(m, 5)
        return m
    if name == "big":  # symmetric, entries up to +-127: exercises the wide path
        rng = np.random.default_rng(7)
        m = rng.integers(-127, 60, size=(25, 25)).astype(np.int32)
        m = np.triu(m) + np.triu(m, 1).T
        np.fill_diagonal(m, 127)
        return m
    raise KeyError(name)


def ref_result(a: str, b: str, go: int, ge: int, mname: str) -> dict:
    params = ref_align.AlignParams(gap_open=go, gap_extend=ge, matrix=matrix_named(mname))
    res = ref_align.smith_waterman(a, b, params)
    out = {f: getattr(res, f) for f in FIELDS}
    if all(ch in INDEX for ch in a + b):
        chk = ref_oracle.reference_alignment(a, b, params)
        for f in FIELDS[:-1]:
            assert chk[f] == out[f], (a, b, f, chk[f], out[f])
    edge = ref_align.evaluate_pair(0, 1, a, b, res, params)
    out["edge"] = None if edge is None else [edge.score, edge.identity, edge.coverage_i,
                                             edge.coverage_j]
    return out


def mutate(rng: random.Random, s: str, sub: float, indel: float, alphabet: str = STD) -> str:
    out = []
    for ch in s:
        r = rng.random()
        if r < indel / 2:
            continue
        if r < indel:
            out.append("".join(rng.choice(alphabet) for _ in range(rng.randint(1, 6))))
        out.append(rng.choice(alphabet) if rng.random() < sub else ch)
    return "".join(out) or rng.choice(alphabet)


GAPS = [(11, 1), (11, 2), (10, 10), (5, 0), (0, 0), (3, 1), (20, 5), (1, 1), (13, 3)]
EDGE_LENS = [1, 2, 3, 31, 32, 33, 63, 64, 65, 127, 128, 129, 255, 256, 257, 319, 320, 321,
             383, 384, 385, 511, 512, 513, 640, 700]


def random_cases(seed: int = 2303) -> list:
    rng = random.Random(seed)
    cases = []

    def add(kind, a, b, go, ge, mname="blosum62"):
        cases.append({"kind": kind, "a": a, "b": b, "gap_open": go, "gap_extend": ge,
                      "matrix": mname})

    for _ in range(500):  # SPEC.md:515 style: short random pairs
        a = "".join(rng.choice(STD) for _ in range(rng.randint(1, 80)))
        b = "".join(rng.choice(STD) for _ in range(rng.randint(1, 80)))
        add("uniform", a, b, *rng.choice(GAPS))
    for alpha in ("AG", "AGS", "LIVMF", "W", "GSA"):
        for _ in range(60):  # low complexity: many ties
            a = "".join(rng.choice(alpha) for _ in range(rng.randint(1, 70)))
            b = mutate(rng, a, 0.2, 0.15, alpha) if rng.random() < 0.5 else \
                "".join(rng.choice(alpha) for _ in range(rng.randint(1, 70)))
            add("lowc", a, b, *rng.choice(GAPS))
    for _ in range(300):  # homologs with indels
        a = "".join(rng.choice(STD) for _ in range(rng.randint(20, 220)))
        b = mutate(rng, a, rng.uniform(0.05, 0.4), rng.uniform(0.0, 0.15))
        if rng.random() < 0.3:
            b = b[rng.randint(0, len(b) // 3):]
        add("mut", a, b, *rng.choice(GAPS[:4]))
    for la in EDGE_LENS:  # strip / length-class boundaries on both axes
        for lb in (1, 33, 300, la):
            a = "".join(rng.choice(STD) for _ in range(la))
            b = mutate(rng, a, 0.2, 0.05)[:lb] if rng.random() < 0.6 else \
                "".join(rng.choice(STD) for _ in range(lb))
            add("edge_len", a, b or "A", *rng.choice([(11, 1), (11, 2)]))
    weird = STD + "BZXU*abcJOjo1 ."
    for _ in range(80):  # raw-byte semantics: unknown bytes score as X, matches compare bytes
        a = "".join(rng.choice(weird) for _ in range(rng.randint(1, 60)))
        b = mutate(rng, a, 0.2, 0.05, weird) if rng.random() < 0.6 else \
            "".join(rng.choice(weird) for _ in range(rng.randint(1, 60)))
        add("chars", a, b, *rng.choice(GAPS))
    for _ in range(60):  # other matrices
        a = "".join(rng.choice(STD) for _ in range(rng.randint(5, 150)))
        b = mutate(rng, a, 0.25, 0.08)
        add("ident", a, b, *rng.choice(GAPS), mname="ident")
    for _ in range(20):
        a = "".join(rng.choice(STD) for _ in range(rng.randint(5, 200)))
        b = mutate(rng, a, 0.1, 0.03)
        add("big", a, b, 100, 20, mname="big")
    for ln in (260, 300, 400):  # best > 32640 -> the GPU's wide path
        a = "".join(rng.choice("W") for _ in range(ln))
        add("big_wide", a, a[: ln - 3], 120, 30, mname="big")
    return cases


def kats() -> list:
    pairs = [
        ("AAAA", "AAAA"), ("A", "P"),
        ("AAGAAGGGSGGSGASAGAA", "SSSAGGAAGSGGSGSSGGAA"),
        ("GSAASAGSASAAAGGAAASGASAAS", "SSGAAASA"),
        ("SSGAAASA", "GSAASAGSASAAAGGAAASGASAAS"),
        ("MKVLAAGIVG", "MKVAAGIVG"), ("WWWW", "WW"),
    ]
    out = []
    for ge in (2, 1):
        for a, b in pairs:
            out.append({"kind": "kat", "a": a, "b": b, "gap_open": 11, "gap_extend": ge,
                        "matrix": "blosum62"})
    return out


def long_cases() -> list:
    rng = random.Random(99)
    out = []
    for la, lb, rel in ((1000, 1100, True), (1500, 900, False), (2000, 2000, True),
                        (2100, 1700, True), (600, 2500, False)):
        a = "".join(rng.choice(STD) for _ in range(la))
        b = mutate(rng, a, 0.25, 0.05)[:lb] if rel else \
            "".join(rng.choice(STD) for _ in range(lb))
        out.append({"kind": "long", "a": a, "b": b, "gap_open": 11, "gap_extend": 1,
                    "matrix": "blosum62"})
    w = "W" * 3050  # 11 * 3050 = 33550 > 32767: int16 / scaled-int32 overflow
    out.append({"kind": "long_wide", "a": w, "b": w[:3001], "gap_open": 11, "gap_extend": 1,
                "matrix": "blosum62"})
    return out


def config2_sample(n: int = 96) -> list:
    sa, sb = workloads.config2(n, seed=2303)
    return [{"kind": "config2", "a": a.decode(), "b": b.decode(), "gap_open": 11,
             "gap_extend": 1, "matrix": "blosum62"} for a, b in zip(sa, sb)]


def config1() -> dict:
    """Config 1 end to end through the reference pipeline; the (i, j, result)
    triples are captured at the evaluate_pair seam (pipeline.py:233-236)."""
    recs = ref_synth.synthetic_records(1000, 0, min_len=50, max_len=500)
    captured = []
    orig_eval = ref_pipeline.evaluate_pair

    def capture(i, j, a, b, res, params):
        captured.append((i, j, [getattr(res, f) for f in FIELDS]))
        return orig_eval(i, j, a, b, res, params)

    ref_pipeline.evaluate_pair = capture
    try:
        with tempfile.TemporaryDirectory() as td:
            fa = os.path.join(td, "in.fa")
            ref_seqio.write_fasta(fa, recs)
            out = os.path.join(td, "out.tsv")
            stats = ref_pipeline.run_search(ref_pipeline.PipelineConfig(), fa, out)
            canon = os.path.join(td, "canon.tsv")
            ref_seqio.canonicalize_output(out, canon)
            canon_bytes = open(canon, "rb").read()
            fasta_sha = hashlib.sha256(open(fa, "rb").read()).hexdigest()
    finally:
        ref_pipeline.evaluate_pair = orig_eval
    params = ref_align.AlignParams()
    return {
        "headers": [r.header for r in recs],
        "residues": [r.residues for r in recs],
        "pairs": [[i, j] for i, j, _ in captured],
        "results": [r for _, _, r in captured],
        "canonical_sha256": hashlib.sha256(canon_bytes).hexdigest(),
        "canonical_lines": canon_bytes.decode().splitlines(),
        "fasta_sha256": fasta_sha,
        "counters": {"discovered": stats.discovered_candidates,
                     "performed": stats.performed_alignments,
                     "edges": stats.output_edges},
        "gap_open": params.gap_open, "gap_extend": params.gap_extend,
        "min_identity": params.min_identity, "min_coverage": params.min_coverage,
    }


def with_results(cases: list) -> list:
    for c in cases:
        c["expect"] = ref_result(c["a"], c["b"], c["gap_open"], c["gap_extend"], c["matrix"])
    return cases


def dump(name: str, obj) -> None:
    path = os.path.join(HERE, name)
    with open(path, "w") as fh:
        json.dump(obj, fh, separators=(",", ":"))
    print(f"{path}: {os.path.getsize(path)} bytes")


def main() -> None:
    dump("blosum62.json", {"alphabet": ALPHABET,
                           "matrix": np.asarray(ref_blosum.MATRIX).tolist(),
                           "dump": ref_blosum.dump()})
    dump("matrices.json", {k: matrix_named(k).tolist() for k in ("blosum62", "ident", "big")})
    dump("kats.json", with_results(kats()))
    dump("random_pairs.json", with_results(random_cases()))
    dump("long_pairs.json", with_results(long_cases()))
    dump("config2_sample.json", with_results(config2_sample()))
    dump("config1.json", config1())


if __name__ == "__main__":
    main()

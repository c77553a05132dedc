"""Generate tests/golden/fasta_cases.json from the REFERENCE's FASTA reader.

Runs only in the build container (imports pastislite from
/root/reference/pkg/src).  For each text -- hand-written edge cases plus
seeded fuzz texts over a character set rich in line breaks, whitespace,
lowercase, off-alphabet and multi-byte characters -- it records what
pastislite.seqio.read_fasta (seqio.py:42-92) returns: the (header, residues)
records and the "mapped" count of its warning, or the FastaError message
(with the path replaced by "{path}").

    python tests/golden/make_fasta_golden.py
"""

import base64
import json
import logging
import os
import random
import sys
import tempfile

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)

from pastislite import seqio as ref_seqio  # noqa: E402

EDGE = [
    b">a\nACDE\n",
    b">a desc words\nAC\nDE\n>b\nWW\n",
    b">a\r\nAC\r\nDE\r\n>b\r\nK\r\n",
    b">a\rAC\rDE\r>b\rK",
    b">a\nAC\n\n\n   \n>b\n\tmkv\t\n",
    b"   >a   x y\n  acgtjxbzu*  \n",
    b">a\nA C\tD\n",
    b">a\nAC\x0bDE\x0c\n>b\n\x1cK\x1d\x1e\x1f\n",
    b">a\nac\n>b\n>c\nD\n",
    b">a\nAC\n>\nD\n",
    b">   \nD\n",
    b"ACDE\n>a\nK\n",
    b"",
    b"\n\n   \n",
    b">a\n",
    b">a\nAC\n>b\n",
    b">a\n1234567890!@#$%^&()-_=+[]{};:'\",.<>/?\\|`~\n",
    b">x'y\n\n",
    b">a\\b\n",
    b">tab\there\nAA\n",
    b">a\n>b\nK\n",
    b">a\nK\n\r\n\r\n>b\nL",
    ">é\nACé\n".encode("utf-8"),
    ">a\nstraße\n".encode("utf-8"),
    ">a b c\n AC \n".encode("utf-8"),
    ">a b\nAC DE\n".encode("utf-8"),
    ">a\nAC\n".encode("utf-8"),
    ">ａｂ\nａｃ\n".encode("utf-8"),
]

CHARS = (["A", "C", "D", "W", "a", "k", "j", "x", "*", "X", "U", "B", "Z", "o", "1", "-", ".",
          ">", ">", " ", " ", "\t", "\n", "\n", "\n", "\r", "\r\n", "\x0b", "\x0c", "\x1c",
          "\x1f", "\x00", "'"] + ["ß", "é", " ", " "])


def run_case(data: bytes, tmpdir: str) -> dict:
    path = os.path.join(tmpdir, "case.fa")
    with open(path, "wb") as fh:
        fh.write(data)
    records = []

    class Grab(logging.Handler):
        def emit(self, rec):
            records.append(rec.getMessage())

    h = Grab()
    lg = logging.getLogger(ref_seqio.__name__)
    lg.addHandler(h)
    lg.setLevel(logging.WARNING)
    try:
        recs = ref_seqio.read_fasta(path)
        out = {"records": [[r.header, r.residues] for r in recs]}
        assert [r.id for r in recs] == list(range(len(recs)))
    except ref_seqio.FastaError as e:
        out = {"error": str(e).replace(path, "{path}")}
    except UnicodeDecodeError as e:
        out = {"unicode_error": True, "detail": str(e)[:80]}
    finally:
        lg.removeHandler(h)
    mapped = 0
    for m in records:
        if m.startswith("mapped "):
            mapped = int(m.split()[1])
    out["mapped"] = mapped
    out["text_b64"] = base64.b64encode(data).decode("ascii")
    return out


def main():
    rnd = random.Random(2303)
    texts = list(EDGE)
    for k in range(300):
        pool = CHARS if k % 3 == 0 else CHARS[:-4]
        n = rnd.randint(0, 120)
        s = "".join(rnd.choice(pool) for _ in range(n))
        if rnd.random() < 0.7:
            s = ">h" + str(k) + "\n" + s
        texts.append(s.encode("utf-8"))
    with tempfile.TemporaryDirectory() as td:
        cases = [run_case(t, td) for t in texts]
    with open(os.path.join(HERE, "fasta_cases.json"), "w") as fh:
        json.dump({"source": "pastislite.seqio.read_fasta (seqio.py:42-92)", "cases": cases}, fh)
    kinds = {}
    for c in cases:
        key = "records" if "records" in c else ("error" if "error" in c else "unicode")
        kinds[key] = kinds.get(key, 0) + 1
    print(len(cases), "cases", kinds)


if __name__ == "__main__":
    main()

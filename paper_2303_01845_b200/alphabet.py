"""The 25-symbol residue alphabet of the reference.

Same symbols, order and unknown-symbol rule as
/root/reference/pkg/src/pastislite/alphabet.py:8-14: 20 standard residues,
ambiguity codes B/Z, unknown X, selenocysteine U and the stop symbol '*'.
Index order is the row/column order of the substitution matrix and of the
residue codes the GPU kernels use (code 25 is reserved for virtual cells).
"""

ALPHABET = "ARNDCQEGHILKMFPSTWYVBZXU*"
SIZE = len(ALPHABET)
INDEX = {symbol: code for code, symbol in enumerate(ALPHABET)}
UNKNOWN = "X"

"""Matrix Market input/output (the reference's src/formats.py:143-409 API).

parse_matrix_market(path, pool, matrix_id, *, precision=SINGLE,
                    spill_bytes=..., chunk_lines=...) -> StoredMatrix
read_matrix_market_info(path) -> {"rows", "cols", "entries", "field", "symmetric"}
write_matrix_market(path, mat)
write_block_file(path, mat) / read_block_file(path, pool, matrix_id=None)
    (the one-file block export, implemented in store.py)

Parsing runs in the library's native multi-threaded reader (csrc/mmio.cu,
xb_mm_read): same acceptance rules, messages and 1-based line numbers
(ParseError.line) as the reference, triplets in the reference's order, then
registered through matrix_from_coo (duplicates summed in input order,
core.py:287-303). The reference's spill-to-disk runs (spill_bytes) exist
because pandas chunks must fit host memory; the native reader holds the
triplets once, so `spill_bytes` is accepted for signature parity and
ignored. No GPU is needed to parse.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .core import Precision, as_precision
from .pool import canonical_coo, matrix_from_coo
from .store import read_block_file, write_block_file  # noqa: F401  (formats.py:471-519)

DEFAULT_SPILL_BYTES = 256 << 20
DEFAULT_CHUNK_LINES = 500_000


def read_matrix_market_info(path: str) -> dict:
    """Header and size line only; never touches the body (formats.py:381-395)."""
    return _lib.mm_info(path)


def parse_matrix_market(path: str, pool, matrix_id: str, *, precision=Precision.SINGLE,
                        spill_bytes: int = DEFAULT_SPILL_BYTES,
                        chunk_lines: int = DEFAULT_CHUNK_LINES, threads: int = 0):
    """Parse a Matrix Market coordinate file into a pooled sparse matrix
    (formats.py:261-322)."""
    rows, cols, r, c, v, _ = _lib.mm_read(path, threads=threads, chunk_lines=chunk_lines)
    return matrix_from_coo(pool, matrix_id, rows, cols, r, c, v, precision=as_precision(precision))


def write_matrix_market(path: str, mat):
    """Write a sparse matrix as a general real coordinate file (formats.py:398-409)."""
    rows, cols = mat.shape
    r, c, v = canonical_coo(mat)
    if mat.desc.transposed:
        r, c = c, r
    order = np.lexsort((c, r))  # view coordinates, sorted by (row, col)
    r, c, v = r[order], c[order], v[order]
    with open(path, "wt", encoding="utf-8") as f:
        f.write("%%MatrixMarket matrix coordinate real general\n")
        f.write(f"{rows} {cols} {len(v)}\n")
        for i, j, x in zip(r, c, v):
            f.write(f"{i + 1} {j + 1} {float(x):.17g}\n")

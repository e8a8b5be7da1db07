"""Data-model mirror of the reference's core types (src/core.py).

Only what the hot-path boundary needs: Precision (core.py:26-58),
Density (78-80), BlockPartition (83-139), MatrixDescriptor (142-220),
DenseBlock (223-242), SparseBlock (245-284). Field names, shapes and
semantics match the reference so code written against `xsvd` objects and
against these reads the same; the GPU entry points also accept the
reference's own objects (duck-typed: `.desc`, `.shape`, `.to_array()`).
"""

from __future__ import annotations

import bisect
import enum
from dataclasses import dataclass, replace

import numpy as np

from .errors import ShapeError, XsvdError

CANONICAL_CELL = 256  # core.py:23 (the reference's reduction grid; not used on the GPU)


class Precision(enum.Enum):
    HALF = "half"
    SINGLE = "single"
    DOUBLE = "double"

    @property
    def nbytes(self) -> int:
        return {Precision.HALF: 2, Precision.SINGLE: 4, Precision.DOUBLE: 8}[self]

    @property
    def storage_dtype(self):
        return {Precision.HALF: np.dtype("<f2"), Precision.SINGLE: np.dtype("<f4"),
                Precision.DOUBLE: np.dtype("<f8")}[self]

    @property
    def compute_dtype(self):
        # half is storage-only; arithmetic widens it to single (core.py:43-46)
        return np.dtype("<f4") if self is not Precision.DOUBLE else np.dtype("<f8")

    @classmethod
    def parse(cls, name: str) -> "Precision":
        try:
            return cls(name)
        except ValueError:
            raise ValueError(f"unknown precision {name!r}") from None


def as_precision(p) -> Precision:
    """Accept our Precision, the reference's Precision, or its string value."""
    if isinstance(p, Precision):
        return p
    return Precision(getattr(p, "value", p))


def wider(a: Precision, b: Precision) -> Precision:
    order = [Precision.HALF, Precision.SINGLE, Precision.DOUBLE]
    return a if order.index(a) >= order.index(b) else b


class Density(enum.Enum):
    DENSE = "dense"
    SPARSE = "sparse"


@dataclass(frozen=True)
class BlockPartition:
    row_cuts: tuple
    col_cuts: tuple

    @staticmethod
    def _cuts(extent: int, pieces: int) -> tuple:
        pieces = max(1, min(pieces, max(extent, 1)))
        q, rem = divmod(extent, pieces)
        cuts = [0]
        for s in [q + 1] * rem + [q] * (pieces - rem):
            cuts.append(cuts[-1] + s)
        return tuple(cuts)

    @classmethod
    def grid(cls, rows, cols, n_row, n_col) -> "BlockPartition":
        return cls(cls._cuts(rows, n_row), cls._cuts(cols, n_col))

    @classmethod
    def single(cls, rows, cols) -> "BlockPartition":
        return cls((0, rows), (0, cols))

    @property
    def n_row_tiles(self):
        return len(self.row_cuts) - 1

    @property
    def n_col_tiles(self):
        return len(self.col_cuts) - 1

    def row_span(self, i):
        return self.row_cuts[i], self.row_cuts[i + 1]

    def col_span(self, j):
        return self.col_cuts[j], self.col_cuts[j + 1]

    def locate_row(self, r):
        return bisect.bisect_right(self.row_cuts, r) - 1

    def locate_col(self, c):
        return bisect.bisect_right(self.col_cuts, c) - 1

    def transposed(self) -> "BlockPartition":
        return BlockPartition(self.col_cuts, self.row_cuts)


@dataclass
class MatrixDescriptor:
    matrix_id: str
    rows: int
    cols: int
    density: Density
    precision: Precision
    transposed: bool = False
    partition: BlockPartition = None  # type: ignore[assignment]
    nnz: int = 0

    def __post_init__(self):
        if self.partition is None:
            self.partition = BlockPartition.single(self.rows, self.cols)
        if self.rows < 1 or self.cols < 1:
            raise ShapeError(f"matrix {self.matrix_id}: empty shape {self.rows}x{self.cols}")
        if self.density is Density.DENSE:
            self.nnz = self.rows * self.cols

    @property
    def shape(self):
        return (self.cols, self.rows) if self.transposed else (self.rows, self.cols)


def transpose_view(desc: MatrixDescriptor) -> MatrixDescriptor:
    return replace(desc, transposed=not desc.transposed)


@dataclass
class DenseBlock:
    """Row-major dense tile over [row0, row1) x [col0, col1) (core.py:223-242)."""

    row0: int
    row1: int
    col0: int
    col1: int
    values: np.ndarray

    def __post_init__(self):
        if self.values.shape != (self.row1 - self.row0, self.col1 - self.col0):
            raise ShapeError(f"dense block values {self.values.shape} != range")
        if not self.values.flags.c_contiguous:
            self.values = np.ascontiguousarray(self.values)

    @property
    def nbytes(self):
        return self.values.nbytes


@dataclass
class SparseBlock:
    """COO-SoA tile, (row, col)-sorted, no duplicates (core.py:245-284)."""

    row0: int
    row1: int
    col0: int
    col1: int
    rows: np.ndarray
    cols: np.ndarray
    values: np.ndarray

    def __post_init__(self):
        n = len(self.values)
        if len(self.rows) != n or len(self.cols) != n:
            raise XsvdError("sparse block index/value arrays differ in length")
        if n:
            r = self.rows.astype(np.int64)
            c = self.cols.astype(np.int64)
            key = r * (self.col1 - self.col0 + 1) + (c - self.col0)
            if not np.all(np.diff(key) > 0):
                raise XsvdError("sparse block entries not strictly (row, col) sorted")

    @property
    def nnz(self):
        return len(self.values)

    @property
    def nbytes(self):
        return self.values.nbytes + self.rows.nbytes + self.cols.nbytes

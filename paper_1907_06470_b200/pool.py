"""In-core matrix pool mirroring the reference's BlockPool / StoredMatrix API.

The reference pool (src/pool.py:100-360) manages byte budgets, LRU eviction
and a spill lane — out of scope here (the GPU owns residency in
HBM). This mirror keeps the API the hot path is called through:
`BlockPool.register/get/put/descriptor/drop_matrix`, `StoredMatrix.T/
shape/to_array/tile`, `create_matrix`, `matrix_from_dense` (pool.py:554-571)
and `matrix_from_coo` (pool.py:574-618, duplicates summed). Everything is
held in host memory, one tile per matrix unless a grid is given.
"""

from __future__ import annotations

import threading

import numpy as np

from .core import (BlockPartition, Density, DenseBlock, MatrixDescriptor, Precision, SparseBlock,
                   as_precision, transpose_view)
from .errors import BlockAbsentError, BudgetError, ShapeError, XsvdError


class BlockPool:
    """In-core tiles; with a `store.BlockStore`, tiles missing from memory are
    loaded from it (pool.py:271-278) and `flush_matrix` persists dirty tiles
    synchronously (pool.py:315-335), which is what durable step records rely
    on. No byte budget / eviction: HBM residency is the library's job."""

    def __init__(self, store=None, budget=None):
        self.store = store
        self.budget = budget
        self._descs: dict[str, MatrixDescriptor] = {}
        self._tiles: dict[tuple, object] = {}
        self._dirty: set = set()
        self._lock = threading.Lock()

    def register(self, desc):
        with self._lock:
            return self._descs.setdefault(desc.matrix_id, desc)

    def descriptor(self, matrix_id):
        return self._descs[matrix_id]

    def known_matrices(self):
        return dict(self._descs)

    def put(self, matrix_id, ti, tj, block, *, dirty=True):
        with self._lock:
            self._tiles[(matrix_id, ti, tj)] = block
            if dirty:
                self._dirty.add((matrix_id, ti, tj))

    def get(self, matrix_id, ti, tj, *, pin=False):
        key = (matrix_id, ti, tj)
        with self._lock:
            block = self._tiles.get(key)
            if block is not None:
                return block
            if self.store is None:
                raise BlockAbsentError(f"block {matrix_id}[{ti},{tj}] not resident (no store)")
            block = self.store.load_block(matrix_id, ti, tj)
            self._tiles[key] = block
            return block

    def drop_matrix(self, matrix_id, *, delete_files=False):
        with self._lock:
            for key in [k for k in self._tiles if k[0] == matrix_id]:
                del self._tiles[key]
            self._dirty = {k for k in self._dirty if k[0] != matrix_id}
            self._descs.pop(matrix_id, None)
            if delete_files and self.store is not None:
                self.store.delete_matrix_blocks(matrix_id)

    def flush_matrix(self, matrix_id, *, evict=False):
        """On return every tile of the matrix is durable (pool.py:315-335)."""
        with self._lock:
            for key in sorted(k for k in self._dirty if k[0] == matrix_id):
                if self.store is None:
                    raise BudgetError("cannot persist blocks without a workdir")
                self.store.store_block(key[0], key[1], key[2], self._tiles[key])
                self._dirty.discard(key)
            if evict:
                for key in [k for k in self._tiles if k[0] == matrix_id]:
                    del self._tiles[key]

    def close(self):
        return None


class StoredMatrix:
    def __init__(self, desc, pool):
        self.desc = desc
        self.pool = pool

    @property
    def matrix_id(self):
        return self.desc.matrix_id

    @property
    def shape(self):
        return self.desc.shape

    @property
    def T(self):
        return StoredMatrix(transpose_view(self.desc), self.pool)

    def tile(self, ti, tj):
        return self.pool.get(self.matrix_id, ti, tj)

    def set_tile(self, ti, tj, block):
        self.pool.put(self.matrix_id, ti, tj, block)

    def to_array(self) -> np.ndarray:
        return stored_to_array(self)


def _canonical_dense(mat) -> np.ndarray:
    """Assemble the canonical (untransposed) dense array from its tiles."""
    d = mat.desc
    part = d.partition
    out = np.empty((d.rows, d.cols), dtype=as_precision(d.precision).storage_dtype)
    for ti in range(part.n_row_tiles):
        r0, r1 = part.row_span(ti)
        for tj in range(part.n_col_tiles):
            c0, c1 = part.col_span(tj)
            out[r0:r1, c0:c1] = mat.pool.get(d.matrix_id, ti, tj).values
    return out


def canonical_coo(mat):
    """(rows int64, cols int64, values) of a sparse matrix, canonical orientation."""
    d = mat.desc
    part = d.partition
    rr, cc, vv = [], [], []
    for ti in range(part.n_row_tiles):
        for tj in range(part.n_col_tiles):
            blk = mat.pool.get(d.matrix_id, ti, tj)
            rr.append(np.asarray(blk.rows, np.int64))
            cc.append(np.asarray(blk.cols, np.int64))
            vv.append(np.asarray(blk.values))
    return np.concatenate(rr), np.concatenate(cc), np.concatenate(vv)


def is_sparse(mat) -> bool:
    return getattr(mat.desc.density, "value", mat.desc.density) == "sparse"


def stored_to_array(mat) -> np.ndarray:
    """View-aware dense materialisation of any StoredMatrix-like handle."""
    d = mat.desc
    if is_sparse(mat):
        r, c, v = canonical_coo(mat)
        out = np.zeros((d.rows, d.cols), dtype=as_precision(d.precision).storage_dtype)
        np.add.at(out, (r, c), v)
    else:
        out = _canonical_dense(mat)
    return out.T if d.transposed else out


def _register(pool, desc):
    """Register and, with a store, persist the descriptor (pool.py:548-550)."""
    desc = pool.register(desc)
    if getattr(pool, "store", None) is not None:
        pool.store.save_descriptor(desc)
    return desc


def create_matrix(pool, matrix_id, rows, cols, *, precision, density=Density.DENSE, nnz=None):
    desc = MatrixDescriptor(matrix_id, rows, cols, density, as_precision(precision),
                            nnz=nnz or 0)
    return StoredMatrix(_register(pool, desc), pool)


def matrix_from_dense(pool, matrix_id, array, *, precision, grid=None) -> StoredMatrix:
    array = np.asarray(array)
    if array.ndim != 2:
        raise ShapeError(f"expected a 2-d array, got shape {array.shape}")
    m, n = array.shape
    precision = as_precision(precision)
    part = BlockPartition.single(m, n) if grid is None else BlockPartition.grid(m, n, *grid)
    pool.drop_matrix(matrix_id)  # results overwrite a previous matrix of the same id
    desc = _register(pool, MatrixDescriptor(matrix_id, m, n, Density.DENSE, precision,
                                            partition=part))
    mat = StoredMatrix(desc, pool)
    for ti in range(part.n_row_tiles):
        r0, r1 = part.row_span(ti)
        for tj in range(part.n_col_tiles):
            c0, c1 = part.col_span(tj)
            vals = np.ascontiguousarray(array[r0:r1, c0:c1], dtype=precision.storage_dtype)
            mat.set_tile(ti, tj, DenseBlock(r0, r1, c0, c1, vals))
    return mat


def matrix_from_coo(pool, matrix_id, rows, cols, coo_rows, coo_cols, coo_values, *, precision):
    """Sparse matrix from unordered triplets; duplicates summed (pool.py:574-618)."""
    precision = as_precision(precision)
    r = np.asarray(coo_rows, dtype=np.int64)
    c = np.asarray(coo_cols, dtype=np.int64)
    v = np.asarray(coo_values, dtype=precision.storage_dtype)
    if len(v):
        order = np.lexsort((c, r))
        r, c, v = r[order], c[order], v[order]
        boundary = np.empty(len(r), dtype=bool)
        boundary[0] = True
        np.not_equal(r[1:], r[:-1], out=boundary[1:])
        boundary[1:] |= c[1:] != c[:-1]
        starts = np.flatnonzero(boundary)
        r, c, v = r[starts], c[starts], np.add.reduceat(v, starts)
    desc = _register(pool, MatrixDescriptor(matrix_id, rows, cols, Density.SPARSE, precision,
                                            nnz=len(v)))
    mat = StoredMatrix(desc, pool)
    idt = np.uint32 if max(rows, cols) < 2**32 else np.uint64
    mat.set_tile(0, 0, SparseBlock(0, rows, 0, cols, r.astype(idt), c.astype(idt), v))
    return mat


def register_dense(pool, matrix_id, array, precision) -> object:
    """Register a result in the CALLER's pool — ours, or the reference's own
    BlockPool (then through xsvd.pool.matrix_from_dense with xsvd's
    Precision), so outputs land where the reference would put them."""
    mod = type(pool).__module__
    if mod.startswith("xsvd"):
        import importlib

        xpool = importlib.import_module("xsvd.pool")
        xcore = importlib.import_module("xsvd.core")
        return xpool.matrix_from_dense(pool, matrix_id, array,
                                       precision=xcore.Precision(as_precision(precision).value))
    return matrix_from_dense(pool, matrix_id, array, precision=precision)

"""GPU replacements for the reference's block kernels (src/kernels.py).

Same names, arguments, return types and error behaviour as the reference:

  block_multiply(pool, x, y, out_id, *, threads=1, out_precision=None)
        -> (StoredMatrix, MultiplyStats)                      kernels.py:145-228
  gram(pool, b, out_id, *, threads=1)                         kernels.py:239-241
  thin_qr(pool, y, q_id) -> QRResult(q, r, deficient_columns) kernels.py:297-351
  svd_small(b) -> SmallSVDResult(u, s, v)                     kernels.py:542-562

Arithmetic runs in libxsvdb200.so (FP64 DMMA GEMM, CholQR2 + Householder
fallback, one-sided Jacobi). `threads` is accepted for signature parity and
ignored. There is no CPU fallback: a missing library raises XsvdError.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .core import Precision, as_precision, wider
from .errors import ShapeError, XsvdError
from .pool import canonical_coo, is_sparse, register_dense, stored_to_array


@dataclass
class MultiplyStats:
    multiply_adds: int = 0
    skipped_cells: int = 0
    threads_used: int = 1
    estimate: object = None


@dataclass
class QRResult:
    q: object
    r: np.ndarray
    deficient_columns: tuple = ()


@dataclass
class SmallSVDResult:
    u: np.ndarray
    s: np.ndarray
    v: np.ndarray


def _device_dtype(prec: Precision, what: str):
    """float64 for DOUBLE, float32 for SINGLE (the compute dtype's storage,
    core.py:43-46). HALF (storage-only in the reference) is not built."""
    prec = as_precision(prec)
    if prec is Precision.HALF:
        raise XsvdError(f"{what}: half precision is not built on the GPU path")
    return np.float64 if prec is Precision.DOUBLE else np.float32


def _canonical(mat):
    """(canonical array, transposed flag) without materialising a transpose."""
    arr = stored_to_array(mat)
    if mat.desc.transposed:
        return arr.T, True  # arr.T is the canonical (contiguous) array
    return arr, False


def block_multiply(pool, x, y, out_id, *, threads: int = 1, out_precision=None):
    """out = x @ y on the device (kernels.py:145-193, dense operands)."""
    m, k = x.shape
    k2, n = y.shape
    if k != k2:
        raise ShapeError(f"inner dimensions disagree: {x.shape} x {y.shape}")
    prec = as_precision(out_precision) if out_precision is not None else wider(
        as_precision(x.desc.precision), as_precision(y.desc.precision))
    if is_sparse(x) or is_sparse(y):
        return _sparse_multiply(pool, x, y, out_id, prec, m, n)
    dt = _device_dtype(prec, "block_multiply")
    ctx = _lib.load()
    a, ta = _canonical(x)
    b = stored_to_array(y)
    c = ctx.gemm(np.asarray(a, dt), np.asarray(b, dt), trans_a=ta)
    out = register_dense(pool, out_id, c.astype(prec.storage_dtype, copy=False), prec)
    return out, MultiplyStats(multiply_adds=m * n * k, threads_used=1)


def _coo_view(mat):
    """(rows, cols, vals, shape) of a sparse handle in VIEW coordinates."""
    r, c, v = canonical_coo(mat)
    if mat.desc.transposed:
        r, c = c, r
    return r, c, v, tuple(mat.shape)


def _sparse_multiply(pool, x, y, out_id, prec, m, n):
    """Sparse x dense (kernels.py:85-97) and dense x sparse (98-112) on the
    device CSR SpMM; sparse x sparse (113-141) is off the hot path."""
    if is_sparse(x) and is_sparse(y):
        raise XsvdError("block_multiply: sparse x sparse is not built on the GPU path")
    if as_precision(prec) is not Precision.DOUBLE:
        raise XsvdError("block_multiply: sparse operands are built for float64 only")
    ctx = _lib.load()
    if is_sparse(x):
        r, c, v, shape = _coo_view(x)
        out = ctx.spmm(r, c, v, shape, np.asarray(stored_to_array(y), np.float64))
        nnz = len(v)
        ops = nnz * n
    else:
        # x @ y = (y^T x^T)^T with y sparse
        r, c, v, shape = _coo_view(y)
        xt = np.ascontiguousarray(np.asarray(stored_to_array(x), np.float64).T)
        out = ctx.spmm(r, c, v, shape, xt, trans=True).T
        ops = len(v) * m
    res = register_dense(pool, out_id, np.ascontiguousarray(out), prec)
    return res, MultiplyStats(multiply_adds=ops, threads_used=1)


def gram(pool, b, out_id, *, threads: int = 1):
    """B^T B through the transposed-view product (kernels.py:239-241)."""
    return block_multiply(pool, b.T, b, out_id, threads=threads)


def thin_qr(pool, y, q_id) -> QRResult:
    """Thin QR of a tall dense matrix (kernels.py:297-351)."""
    m, r = y.shape
    if m < r or r < 1:
        raise ShapeError(f"thin QR needs rows >= cols >= 1, got {m}x{r}")
    prec = as_precision(y.desc.precision)
    dt = _device_dtype(prec, "thin_qr")
    q, rr, deficient = _lib.load().thin_qr(np.asarray(stored_to_array(y), dt))
    qm = register_dense(pool, q_id, q.astype(prec.storage_dtype, copy=False), prec)
    return QRResult(q=qm, r=rr, deficient_columns=deficient)


def svd_small(b) -> SmallSVDResult:
    """SVD of the small factor B (r x n, r <= n) (kernels.py:542-562)."""
    b = np.asarray(b, dtype=np.float64)
    if b.ndim != 2:
        raise ShapeError(f"svd_small expects a matrix, got shape {b.shape}")
    r, n = b.shape
    if r > n:
        raise ShapeError(f"svd_small expects r <= n, got {r}x{n}")
    u, s, v = _lib.load().svd_small(b)
    return SmallSVDResult(u=u, s=s, v=v)

"""Sparse A (config 3's path): CSR SpMM products and the full factorisation
through the C ABI, against the reference golden vectors and the oracle."""

import numpy as np
import pytest

from conftest import golden
from oracle import metrics as M
from oracle import pipeline as OP

pytestmark = pytest.mark.gpu

SIG64, ANG64 = 1e-10, 1e-8


def test_spmm_golden(lib, gold):
    g = gold("multiply")
    r, c, v, shape = g["sp_rows"], g["sp_cols"], g["sp_vals"], tuple(g["sp_shape"])
    y = lib.spmm(r, c, v, shape, g["z"])
    assert np.max(np.abs(y - g["spmm"])) <= 1e-13 * np.max(np.abs(g["spmm"]))
    yt = lib.spmm(r, c, v, shape, g["q"], trans=True)
    assert np.max(np.abs(yt - g["spmm_t"])) <= 1e-13 * np.max(np.abs(g["spmm_t"]))
    # dense x sparse (Q^T A) is the transpose of A^T Q
    assert np.max(np.abs(yt.T - g["dense_sp"])) <= 1e-13 * np.max(np.abs(g["dense_sp"]))


@pytest.mark.parametrize("l", [1, 7, 33, 120, 220])
def test_spmm_widths_and_determinism(lib, l):
    from paper_1907_06470_b200.workloads import sparse_uniform_np

    m, n = 5000, 3000
    rowptr, col, val = sparse_uniform_np(m, n, 20, 11)
    rows = np.repeat(np.arange(m), np.diff(rowptr))
    x = np.random.default_rng(l).standard_normal((n, l))
    import scipy.sparse as sp

    a = sp.csr_matrix((val, col, rowptr), shape=(m, n))
    y = lib.spmm(rows, col, val, (m, n), x)
    assert np.max(np.abs(y - a @ x)) <= 1e-12 * np.max(np.abs(y))
    q = np.random.default_rng(l + 1).standard_normal((m, l))
    z1 = lib.spmm(rows, col, val, (m, n), q, trans=True)
    z2 = lib.spmm(rows, col, val, (m, n), q, trans=True)
    assert np.array_equal(z1, z2)  # fixed summation order, no fp atomics
    assert np.max(np.abs(z1 - a.T @ q)) <= 1e-12 * np.max(np.abs(z1))


@pytest.mark.parametrize("m,n,l", [(3000, 300000, 40), (300000, 2000, 24)])
def test_spmm_l2_column_chunks(lib, m, n, l):
    """Gathered operands too large for one L2-resident slab are processed in
    column chunks (sparse.cu launch_spmm): X n x 40 (96 MB) for A X, Q
    m x 24 (58 MB) for A^T Q at 16-column chunks."""
    import scipy.sparse as sp

    from paper_1907_06470_b200.workloads import sparse_uniform_np

    rowptr, col, val = sparse_uniform_np(m, n, 12, 5)
    rows = np.repeat(np.arange(m), np.diff(rowptr))
    a = sp.csr_matrix((val, col, rowptr), shape=(m, n))
    x = np.random.default_rng(1).standard_normal((n, l))
    y = lib.spmm(rows, col, val, (m, n), x)
    assert np.max(np.abs(y - a @ x)) <= 1e-12 * np.max(np.abs(y))
    q = np.random.default_rng(2).standard_normal((m, l))
    z = lib.spmm(rows, col, val, (m, n), q, trans=True)
    assert np.max(np.abs(z - a.T @ q)) <= 1e-12 * np.max(np.abs(z))


def test_transpose_long_columns(lib):
    """Column segments longer than the warp rank-sort's register window (256)
    take the insertion-sort path; A^T products stay exact and deterministic."""
    import scipy.sparse as sp

    rng = np.random.default_rng(7)
    m, n = 2000, 50
    dense = np.where(rng.random((m, n)) < 0.02, rng.standard_normal((m, n)), 0.0)
    dense[:, 3] = rng.standard_normal(m)             # 2000 entries
    dense[::7, 9] = rng.standard_normal(len(range(0, m, 7)))  # 286 entries
    dense[::9, 11] = rng.standard_normal(len(range(0, m, 9)))  # 223 entries
    a = sp.csr_matrix(dense)
    a.sort_indices()
    rows = np.repeat(np.arange(m), np.diff(a.indptr))
    q = rng.standard_normal((m, 5))
    z1 = lib.spmm(rows, a.indices, a.data, (m, n), q, trans=True)
    z2 = lib.spmm(rows, a.indices, a.data, (m, n), q, trans=True)
    assert np.array_equal(z1, z2)
    assert np.max(np.abs(z1 - dense.T @ q)) <= 1e-12 * np.max(np.abs(z1))


def test_empty_rows_and_columns(lib):
    rows = np.array([0, 0, 3])
    cols = np.array([1, 4, 4])
    vals = np.array([2.0, -1.0, 5.0])
    x = np.arange(12, dtype=np.float64).reshape(6, 2)
    y = lib.spmm(rows, cols, vals, (5, 6), x)
    dense = np.zeros((5, 6))
    dense[rows, cols] = vals
    assert np.array_equal(y, dense @ x)
    z = lib.spmm(rows, cols, vals, (5, 6), np.ones((5, 3)), trans=True)
    assert np.array_equal(z, dense.T @ np.ones((5, 3)))


def test_rsvd_sparse_golden(lib, gold):
    g = gold("rsvd")
    m, n, k, p, q, seed, _ = (int(x) for x in g["sp_small_cfg"])
    u, s, v, _, _ = lib.rsvd_coo(g["sp_small_rows"], g["sp_small_cols"], g["sp_small_vals"],
                                 (m, n), k, p, q, seed)
    assert M.sigma_rel(s, g["sp_small_reorth_s"]) <= SIG64
    assert M.sin_angle(u, g["sp_small_reorth_u"]) <= ANG64
    assert M.sin_angle(v, g["sp_small_reorth_v"]) <= ANG64


def test_cfg3_like(lib):
    """Config 3's construction (20 distinct uniform columns per row, N(0,1)
    values) at 200000 x 40000, k=100 p=20 q=3, vs the scipy-backed oracle."""
    from paper_1907_06470_b200.workloads import sparse_uniform_np

    m, n = 200_000, 40_000
    rowptr, col, val = sparse_uniform_np(m, n, 20, 3003)
    rows = np.repeat(np.arange(m), np.diff(rowptr))
    u, s, v, _, _ = lib.rsvd_coo(rows, col, val, (m, n), 100, 20, 3, 3)
    ref = OP.rsvd_reorth(OP.Coo(rows, col, val, (m, n)), 100, 20, 3, 3, "double", fast=True)
    assert M.sigma_rel(s, ref.s) <= SIG64
    assert M.sin_angle(u, ref.u) <= ANG64
    assert M.sin_angle(v, ref.v) <= ANG64


def test_drop_in_sparse(lib):
    """tests/test_pipeline.py:151-162 through the drop-in API: sparse input
    of exact rank <= 18 inside a 25-wide window, vs LAPACK singular values."""
    import paper_1907_06470_b200 as X

    rng = np.random.default_rng(6)
    a = np.zeros((60, 50))
    live = rng.choice(60, size=18, replace=False)
    rr, cc = rng.choice(live, size=300), rng.integers(0, 50, 300)
    a[rr, cc] = rng.standard_normal(300)
    nz = np.nonzero(a)
    pool = X.BlockPool()
    ma = X.matrix_from_coo(pool, "A", 60, 50, nz[0], nz[1], a[nz], precision=X.Precision.DOUBLE)
    res = X.randomized_svd(pool, ma, X.RsvdConfig(rank=25, power=1, seed=0))
    ref = np.linalg.svd(a, compute_uv=False)
    assert np.max(np.abs(res.s - ref[:25])) / ref[0] <= 1e-8
    # the sparse products of block_multiply (and its transposed view)
    z = np.random.default_rng(1).standard_normal((50, 4))
    mz = X.matrix_from_dense(pool, "Z", z, precision=X.Precision.DOUBLE)
    out, _ = X.block_multiply(pool, ma, mz, "AZ")
    assert np.max(np.abs(out.to_array() - a @ z)) <= 1e-13
    w = np.random.default_rng(2).standard_normal((60, 3))
    mw = X.matrix_from_dense(pool, "W", w, precision=X.Precision.DOUBLE)
    out, _ = X.block_multiply(pool, mw.T, ma, "WtA")
    assert np.max(np.abs(out.to_array() - w.T @ a)) <= 1e-13
    out, _ = X.block_multiply(pool, ma.T, mw, "AtW")
    assert np.max(np.abs(out.to_array() - a.T @ w)) <= 1e-13


def test_drop_in_sparse_single_precision(lib):
    """Sparse A at Precision.SINGLE (kernels.py:85-97 with cdt = f32): float32
    values and float32 Omega (pipeline.py:281-282); the device carries them
    exactly in its f64 engine, U and V come back float32. Checked against
    the oracle's float32 computation at the f32 tolerances."""
    import paper_1907_06470_b200 as X
    from paper_1907_06470_b200.workloads import sparse_uniform_np

    m, n = 20000, 4000
    rowptr, col, val = sparse_uniform_np(m, n, 20, 21)
    rows = np.repeat(np.arange(m), np.diff(rowptr))
    val32 = val.astype(np.float32)
    pool = X.BlockPool()
    ma = X.matrix_from_coo(pool, "A", m, n, rows, col.astype(np.int64), val32,
                           precision=X.Precision.SINGLE)
    res = X.randomized_svd(pool, ma, X.RsvdConfig(rank=40, oversample=10, power=2, seed=8,
                                                  precision=X.Precision.SINGLE))
    assert res.u.to_array().dtype == np.float32 and res.v.to_array().dtype == np.float32
    ref = OP.rsvd_reorth(OP.Coo(rows, col.astype(np.int64), val32, (m, n)), 40, 10, 2, 8,
                         "single", fast=True)
    assert M.sigma_rel(res.s, ref.s) <= 1e-4
    assert M.sin_angle(res.u.to_array(), ref.u) <= 1e-3
    assert M.sin_angle(res.v.to_array(), ref.v) <= 1e-3

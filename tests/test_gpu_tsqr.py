"""TSQR (csrc/tsqr.cu): the tree Householder QR that replaces a failed
CholQR (`-m gpu`).

Checked against the reference's thin_qr semantics (kernels.py:297-351,
restated in oracle/kernels.py): Q orthonormal, Q R = Y, R upper triangular
with diag(R) >= 0, deficient columns |R_jj| <= eps ||R||_F flagged like
kernels.py:327-331; for a full-rank Y the factors equal the reference's (the
QR with a positive diagonal is unique). Rank-deficient sketches go through
the factorisation (the Cholesky flags, TSQR takes over) and must still give
the oracle's singular values.
"""

import numpy as np
import pytest

from oracle import kernels as OK
from oracle import metrics as M
from oracle import pipeline as OP

pytestmark = pytest.mark.gpu


def _tsqr(lib, y):
    import torch

    m, r = y.shape
    dy = torch.from_numpy(np.ascontiguousarray(y, dtype=np.float64)).cuda()
    dq = torch.empty((m, r), dtype=torch.float64, device="cuda")
    dr = torch.zeros((r, r), dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    deficient, sec = lib.tsqr_dev(m, r, dy.data_ptr(), r, dq.data_ptr(), r, dr.data_ptr(), r)
    return dq.cpu().numpy(), dr.cpu().numpy(), deficient, sec


def _check_qr(y, q, r, tol=1e-13):
    scale = max(np.linalg.norm(y), 1e-300)
    assert np.max(np.abs(q @ r - y)) <= tol * scale * np.sqrt(y.shape[1])
    assert M.ortho_defect(q) <= tol * np.sqrt(y.shape[0]) * 10
    assert np.all(np.diag(r) >= 0.0)
    assert np.array_equal(r, np.triu(r))


@pytest.mark.parametrize("m,r", [(1, 1), (7, 7), (300, 30), (1000, 120), (4096, 1),
                                 (100000, 120), (20000, 33), (12000, 550), (5000, 1000),
                                 (777, 256)])
def test_tsqr_full_rank_matches_reference_qr(lib, m, r):
    rng = np.random.default_rng(m + r)
    y = rng.standard_normal((m, r)) * np.logspace(0, -6, r)
    q, rr, deficient, _ = _tsqr(lib, y)
    _check_qr(y, q, rr)
    assert deficient == ()
    # unique QR with diag(R) > 0: equal to the reference's factors
    qr, Rr, dref = OK.thin_qr_fast(y, np.float64, np.float64)
    assert np.max(np.abs(rr - Rr)) <= 1e-12 * np.max(np.abs(Rr)) * np.sqrt(m)
    assert M.sin_angle(q, qr) <= 1e-10
    assert np.max(np.abs(q - qr)) <= 1e-9


def test_tsqr_matches_reference_restatement_bits(lib):
    """Small case against the bitwise restatement of the reference's
    streaming Householder thin_qr (not LAPACK)."""
    rng = np.random.default_rng(3)
    y = rng.standard_normal((700, 12))
    q, rr, deficient, _ = _tsqr(lib, y)
    qr, Rr, dref = OK.thin_qr(y, np.float64, np.float64)
    assert deficient == dref == ()
    assert np.max(np.abs(rr - Rr)) <= 1e-13 * np.max(np.abs(Rr))
    assert np.max(np.abs(q - qr)) <= 1e-13


@pytest.mark.parametrize("case", ["zero_col", "dup_cols", "rank18", "all_zero", "neg_first"])
def test_tsqr_rank_deficient(lib, case):
    rng = np.random.default_rng(11)
    m, r = 5000, 25
    y = rng.standard_normal((m, r))
    if case == "zero_col":
        y[:, 7] = 0.0
    elif case == "dup_cols":
        y[:, 10] = y[:, 3]
        y[:, 20] = 2.0 * y[:, 3] - y[:, 5]
    elif case == "rank18":
        y = rng.standard_normal((m, 18)) @ rng.standard_normal((18, r))
    elif case == "all_zero":
        y[:] = 0.0
    elif case == "neg_first":
        y = np.zeros((m, r))
        y[0, :] = -1.0  # sigma == 0 below the diagonal with x0 < 0: beta = 2
    q, rr, deficient, _ = _tsqr(lib, y)
    _check_qr(y, q, rr)
    _, Rr, dref = OK.thin_qr(y, np.float64, np.float64)

    def near(R):
        nrm = max(float(np.sqrt(np.sum(R * R))), 1e-300)
        return tuple(j for j in range(r) if abs(R[j, j]) <= 1e-13 * nrm)

    # exact zeros are flagged identically; rounding-level pivots (~eps) fall
    # on either side of eps ||R||_F in both implementations, so those are
    # compared as the set of numerically zero pivots
    assert near(rr) == near(Rr)
    assert set(deficient) <= set(near(rr))
    if case in ("zero_col", "all_zero", "neg_first"):
        assert deficient == dref
    # R agrees up to the first deficient column (beyond it the completion of
    # Q is arbitrary in both)
    j = near(Rr)[0] if near(Rr) else r
    if j > 0:
        assert np.max(np.abs(rr[:, :j] - Rr[:, :j])) <= 1e-12 * max(np.max(np.abs(Rr)), 1e-300)


def test_tsqr_rank_deficient_cfg3_shape_timing(lib):
    """A rank-deficient 1e6 x 120 sketch (cfg3's Y shape) on one GPU: Q
    orthonormal, Q R = Y, exactly the 30 dependent columns at numerically
    zero pivots, the flagged ones (|R_jj| <= eps ||R||_F, kernels.py:327-331)
    among them. Time is printed (profiles/) and guarded against regression;
    the north-star bar of 20 ms is not met yet."""
    import torch

    m, r = 1_000_000, 120
    g = torch.Generator(device="cuda")
    g.manual_seed(5)
    base = torch.randn(m, 90, generator=g, device="cuda", dtype=torch.float64)
    mix = torch.randn(90, r, generator=g, device="cuda", dtype=torch.float64)
    dy = (base @ mix).contiguous()  # rank 90 < 120
    dq = torch.empty_like(dy)
    dr = torch.zeros((r, r), dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    times = []
    for _ in range(3):
        deficient, sec = lib.tsqr_dev(m, r, dy.data_ptr(), r, dq.data_ptr(), r, dr.data_ptr(), r)
        times.append(sec)
    print(f"TSQR 1e6 x 120 rank 90: {[round(t * 1e3, 2) for t in times]} ms, "
          f"{len(deficient)} flagged")
    y, q, rr = dy.cpu().numpy(), dq.cpu().numpy(), dr.cpu().numpy()
    _check_qr(y, q, rr, tol=1e-12)
    nrm = float(np.sqrt(np.sum(rr * rr)))
    near = [j for j in range(r) if abs(rr[j, j]) <= 1e-13 * nrm]
    assert len(near) == 30
    assert set(deficient) <= set(near)
    assert min(times) <= 0.060, times


def test_rsvd_rank_deficient_sketch_through_tsqr(lib):
    """rank(A) = 60 < l = 120 at 200000 x 3000: every CholQR of the sketch
    breaks down and the TSQR carries the factorisation; sigma_1..60 match
    the oracle, the tail is ~0."""
    rng = np.random.default_rng(12)
    m, n, rk = 200000, 3000, 60
    a = (rng.standard_normal((m, rk)) * np.logspace(0, -3, rk)) @ rng.standard_normal((rk, n))
    u, s, v, deficient, _ = lib.rsvd_dense(a, 100, 20, 1, 7)
    ref = OP.rsvd_reorth(a, 100, 20, 1, 7, "double", fast=True)
    assert np.max(np.abs(s[:rk] - ref.s[:rk]) / ref.s[:rk]) <= 1e-10
    assert np.max(np.abs(s[rk:])) <= 1e-10 * s[0]
    assert M.sin_angle(u[:, :rk], ref.u[:, :rk]) <= 1e-8
    assert M.ortho_defect(u) <= 1e-12 and M.ortho_defect(v) <= 1e-12
    # the final range-finder QR flags rounding-level pivots (which of the
    # ~60 junk columns fall under eps ||R||_F is rounding-dependent in both)
    print("deficient", len(deficient), "oracle", len(ref.deficient_columns))
    assert len(deficient) <= 120 - rk

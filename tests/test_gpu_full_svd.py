"""full_svd (pipeline.py:628-716) on the device: thin QR of the tall
orientation, Jacobi SVD of R, big factor by GEMM. Mirrors the reference's
own tests (tests/test_pipeline.py:327-345, test_acceptance.py:112-127)
against the oracle's Golub-Kahan svd_small restatement."""

import numpy as np
import pytest

from oracle import kernels as K

pytestmark = pytest.mark.gpu


def _recon(res, a):
    approx = res.u.to_array() @ np.diag(res.s) @ res.v.to_array().T
    return np.max(np.abs(approx - a)) / max(np.max(np.abs(a)), 1e-300)


def _ref_sigma(a):
    m, n = a.shape
    b = a if m <= n else a.T  # svd_small takes r x n with r <= n
    return K.svd_small(np.ascontiguousarray(b))[1]


@pytest.mark.parametrize("shape", [(25, 18), (30, 17), (12, 30), (25, 25), (300, 120),
                                   (90, 400)])
def test_full_svd_dense(lib, shape):
    import paper_1907_06470_b200 as X

    rng = np.random.default_rng(sum(shape))
    a = rng.standard_normal(shape)
    pool = X.BlockPool()
    ma = X.matrix_from_dense(pool, "a", a, precision=X.Precision.DOUBLE)
    res = X.full_svd(pool, ma)
    ref = _ref_sigma(a)
    assert res.s.shape == (min(shape),)
    assert np.max(np.abs(res.s - ref)) / ref[0] <= 1e-10
    assert _recon(res, a) <= 1e-10
    assert res.u.shape == (shape[0], min(shape)) and res.v.shape == (shape[1], min(shape))
    assert res.chosen_q == 0


def test_full_svd_wide_and_sparse(lib):
    import paper_1907_06470_b200 as X

    rng = np.random.default_rng(17)
    a = np.zeros((12, 30))
    a[rng.integers(0, 12, 60), rng.integers(0, 30, 60)] = rng.standard_normal(60)
    pool = X.BlockPool()
    r, c = np.nonzero(a)
    ma = X.matrix_from_coo(pool, "a", 12, 30, r, c, a[r, c], precision=X.Precision.DOUBLE)
    res = X.full_svd(pool, ma)
    ref = _ref_sigma(a)
    assert np.max(np.abs(res.s - ref)) / max(ref[0], 1e-300) <= 1e-10


def test_full_svd_exact_rank_reconstruction(lib):
    """Acceptance criterion 2's exact-path half: rank-deficient inputs still
    reconstruct (Householder fallback inside the thin QR)."""
    import paper_1907_06470_b200 as X

    rng = np.random.default_rng(7)
    a = rng.standard_normal((80, 6)) @ rng.standard_normal((6, 40))
    pool = X.BlockPool()
    ma = X.matrix_from_dense(pool, "a", a, precision=X.Precision.DOUBLE)
    res = X.full_svd(pool, ma)
    assert _recon(res, a) <= 1e-8
    assert np.all(res.s[6:] <= 1e-8 * res.s[0])
